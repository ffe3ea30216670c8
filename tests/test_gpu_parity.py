"""GPU parity: every sm_100a kernel against the golden fixtures written by the
reference (tests/golden) and against the CPU oracle on the same seeded inputs.
Bar: bit-exact for every integer/byte/verdict output and for the f64 TPT
samples; exact nearest-rank percentiles; mean within 1e-12 relative."""
import os

import numpy as np
import pytest
import torch

from oracle.oracle import (Grid, OracleLib, TUPLE_DTYPE, default_grid, default_gpu, default_model, phi14b_model,
                           sharegpt_histogram)
from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
MODELS = {"llama8b": (cs.ModelProfile(), default_model()), "phi14b": (cs.ModelProfile.phi14b_like(), phi14b_model())}
GRIDS = {"s500": (500, 500, 5), "s250": (250, 250, 5), "s100": (100, 100, 5)}
G, OG = cs.GpuProfile(), default_gpu()


@pytest.fixture(scope="module")
def ctx():
    return cs.Context(0)


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def steps_bounds(key):
    c, i, b = GRIDS[key]
    return cs.GridSteps(c, i, b), cs.GridBounds(8000, 8000, 50)


def to_dev_tuples(t):
    return torch.from_numpy(np.ascontiguousarray(t).view(np.int32).reshape(len(t), 4).copy()).cuda()


def u32(x):
    return x.cpu().numpy().view(np.uint32)


def i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()


def random_tuples(rng, n, L, hi=9000):
    t = np.zeros(n, TUPLE_DTYPE)
    t["cached"] = rng.integers(0, hi, n)
    t["incoming"] = rng.integers(0, hi, n)
    t["charged"] = rng.integers(0, hi, n)
    t["batch"] = rng.integers(0, 60, n)
    t["pending"] = rng.integers(0, L + 5, n)
    t["dev_layers"] = rng.integers(0, L + 5, n)
    return t


# ------------------------------------------------------------------- maps
def test_map_cells_match_reference(ctx):
    z = np.load(os.path.join(GOLD, "maps.npz"))
    for mn, (m, _) in MODELS.items():
        for gk in GRIDS:
            s, b = steps_bounds(gk)
            for cpa in (0, 1):
                ms = cs.MapSet.build(ctx, m, G, s, b, cs.TrainingMode(cpa))
                off, hed = ms.cells()
                assert (off == z[f"off_{mn}_{gk}_{cpa}"]).all(), (mn, gk, cpa)
                assert (hed == z[f"hed_{mn}_{gk}_{cpa}"]).all(), (mn, gk, cpa)
                assert ms.profile_hash_value == int(z[f"hash_{mn}"])
            ms = cs.MapSet.build(ctx, m, G, s, b, cs.TrainingMode.CPA, hedge_step=250, hedge_max=8000)
            assert (ms.cells()[1] == z[f"hed_{mn}_h250_1"]).all()


def test_map_lookup_mirror_on_device_cells(ctx):  # tests/test_maps.cpp:31-53, 122-139, 152-194
    maps = cs.build_maps(ctx, cs.ModelProfile(), G, mode=cs.TrainingMode.CPA)
    om, hm = maps.offload, maps.hedge
    assert om.lookup(4000, 500, 5) == cs.OffloadDecision(cs.OffloadAction.NoAction, 0)
    assert om.lookup(4000, 2000, 10) == cs.OffloadDecision(cs.OffloadAction.FreeLayers, 6)
    assert om.lookup(5000, 500, 5).action == cs.OffloadAction.AllToHost
    assert om.lookup(8001, 500, 5) is None and om.lookup(4000, 500, 51) is None
    assert hm.lookup(4000, 32) == cs.HedgeDecision.Recompute and hm.lookup(4000, 1) == cs.HedgeDecision.LoadBack
    cpt = cs.build_maps(ctx, cs.ModelProfile(), G, mode=cs.TrainingMode.CPT)
    assert cpt.hedge.lookup(4000, 16) == cs.HedgeDecision.LoadBack and hm.lookup(4000, 16) == cs.HedgeDecision.Recompute


def test_map_errors(ctx):
    with pytest.raises(cs.ColoValidationError):
        cs.MapSet.build(ctx, cs.ModelProfile(), cs.GpuProfile(capacity_bytes=cs.GIB))
    with pytest.raises(cs.ColoValidationError):
        cs.MapSet.build(ctx, cs.ModelProfile(), G, cs.GridSteps(), cs.GridBounds(max_incoming_tokens=8100))
    with pytest.raises(cs.ColoInvalidArgument):
        cs.MapSet.build(ctx, cs.ModelProfile(num_layers=300), G)
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), G)
    off, hed = ms.cells()
    h = cs.profile_hash(cs.ModelProfile(), G)
    args = (ctx, cs.ModelProfile(), G, cs.GridSteps(), cs.GridBounds(), cs.TrainingMode.CPA, 500, 8000, 128)
    with pytest.raises(cs.ColoValidationError, match="hash"):  # maps.hpp:155-157
        cs.MapSet.from_cells(*args, h + 1, off, hed)
    ld = cs.MapSet.from_cells(*args, h, off, hed)
    assert (ld.cells()[0] == off).all() and (ld.cells()[1] == hed).all()


def test_packed_map_from_cells(ctx):
    """A sweep-size grid (step 50: the packed shared-memory kernel, whose
    image the map set builds once) loaded from its cells decides exactly like
    the built map: the image is rebuilt from the loaded cells."""
    steps, bounds = cs.GridSteps(50, 50, 5), cs.GridBounds()
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), G, steps, bounds, cs.TrainingMode.CPT)
    off, hed = ms.cells()
    ld = cs.MapSet.from_cells(ctx, cs.ModelProfile(), G, steps, bounds, cs.TrainingMode.CPT, 50, 8000, 128,
                              cs.profile_hash(cs.ModelProfile(), G), off, hed)
    rng = np.random.default_rng(17)
    dt = to_dev_tuples(random_tuples(rng, 2_000_003, 32))
    assert (u32(cs.decide(ctx, ld, dt)) == u32(cs.decide(ctx, ms, dt))).all()


# ----------------------------------------------------------------- decide
@pytest.mark.parametrize("mn", list(MODELS))
def test_decide_golden(ctx, mn):
    z = np.load(os.path.join(GOLD, "verdicts.npz"))
    m, _ = MODELS[mn]
    t = z[f"tuples_{mn}"]
    dt = to_dev_tuples(t)
    for cpa in (0, 1):
        mode = cs.TrainingMode(cpa)
        ms = cs.MapSet.build(ctx, m, G, mode=mode)
        assert (u32(cs.decide(ctx, ms, dt)) == z[f"v_{mn}_{cpa}"]).all()
        ms2 = cs.MapSet.build(ctx, m, G, mode=mode, hedge_step=250, hedge_max=8000)
        assert (u32(cs.decide(ctx, ms2, dt)) == z[f"vh250_{mn}_{cpa}"]).all()
        assert (u32(cs.decide_exact(ctx, m, G, mode, dt)) == z[f"x_{mn}_{cpa}"]).all()


@pytest.mark.parametrize("gk", ["s500", "s100"])
def test_decide_random_vs_oracle(ctx, orc, gk):
    rng = np.random.default_rng(11)
    for mn, (m, om) in MODELS.items():
        t = random_tuples(rng, 1_000_003, int(om.num_layers))
        dt = to_dev_tuples(t)
        s, b = steps_bounds(gk)
        og = Grid(*GRIDS[gk], 8000, 8000, 50)
        for cpa in (0, 1):
            ms = cs.MapSet.build(ctx, m, G, s, b, cs.TrainingMode(cpa))
            v, cnt = cs.decide(ctx, ms, dt, counters=True)
            ref = orc.decide(om, OG, og, cpa, t)
            assert (u32(v) == ref).all()
            f = cs.verdict_fields(ref)
            exp = [(f["verdict"] == 0).sum(), (f["verdict"] == 1).sum(), (f["verdict"] == 2).sum(), f["offload_oor"].sum(),
                   f["hedge_oor"].sum(), f["stream"].sum(), f["stream_oor"].sum(), len(t)]
            assert list(cnt.cpu().numpy()) == [int(x) for x in exp]


def test_decide_large_grid_global_path(ctx, orc):
    # step 50: 161 x 160 x 10 = 257,600 cells, too large for shared memory -> L1/L2 path
    rng = np.random.default_rng(5)
    t = random_tuples(rng, 500_000, 32)
    s, b = cs.GridSteps(50, 50, 5), cs.GridBounds()
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), G, s, b, cs.TrainingMode.CPA)
    assert (u32(cs.decide(ctx, ms, to_dev_tuples(t))) == orc.decide(default_model(), OG, Grid(50, 50, 5, 8000, 8000, 50), 1, t)).all()


def test_decide_exact_random_vs_oracle(ctx, orc):
    rng = np.random.default_rng(12)
    for mn, (m, om) in MODELS.items():
        t = random_tuples(rng, 300_001, int(om.num_layers), hi=200_000)
        dt = to_dev_tuples(t)
        for cpa in (0, 1):
            assert (u32(cs.decide_exact(ctx, m, G, cs.TrainingMode(cpa), dt)) == orc.decide_exact(om, OG, cpa, t)).all()


def test_decide_exact_fast_range_vs_oracle(ctx, orc):
    """Values below the shared-memory tables (the branch-free fast path of
    k_decide_exact) and the C5 bench's own question stream, 2M tuples each,
    against the oracle in both modes."""
    rng = np.random.default_rng(29)
    for mn, (m, om) in MODELS.items():
        L = int(om.num_layers)
        for t in (random_tuples(rng, 2_000_003, L, hi=16_384),
                  cs.synth_tuples(ctx, 2_000_000, L, 77).cpu().numpy().view(TUPLE_DTYPE).reshape(-1)):
            dt = to_dev_tuples(t)
            for cpa in (0, 1):
                got = u32(cs.decide_exact(ctx, m, G, cs.TrainingMode(cpa), dt))
                want = orc.decide_exact(om, OG, cpa, t)
                bad = np.nonzero(got != want)[0]
                assert bad.size == 0, (mn, cpa, t[bad[:3]], got[bad[:3]], want[bad[:3]])


def test_decide_exact_quotient_edges(ctx, orc):
    """The divide-free exact path (fp32 quotient estimate + u64 correction,
    per-cached hedge thresholds) against the oracle where the ceil-divide of
    maps.hpp:227 lands exactly on integers (tiny per-layer bytes), around n = L,
    across the whole u32 range (u64 wrap in the byte products) and for
    cached values past the threshold table; models with workspace factor 1
    take the branch-free fast path (signed-remainder ceil, cmax AllToHost
    test), the others the general one."""
    rng = np.random.default_rng(31)
    small = [(cs.ModelProfile(num_layers=L, kv_bytes_per_token=kv, act_bytes_per_token_per_layer=a,
                              workspace_factor=wf, weights_bytes=w),
              cs.GpuProfile(capacity_bytes=cap, h2d_bandwidth=h2d, d2h_bandwidth=h2d, runtime_reserve_bytes=0))
             for L, kv, a, wf, w, cap, h2d in ((32, 3, 1, 0.0, 1, 400_000, 1000), (40, 5, 2, 0.5, 1000, 2_000_000, 77),
                                               (7, 1, 3, 0.25, 1, 60_000, 3), (253, 2, 1, 1.0, 1, 1_000_000, 10_000),
                                               # workspace factor 1: the branch-free fast path on tiny per-layer bytes
                                               (32, 3, 1, 1.0, 1, 400_000, 1000), (40, 5, 2, 1.0, 1000, 2_000_000, 77),
                                               (7, 1, 3, 1.0, 1, 60_000, 3), (200, 1, 7, 1.0, 5, 3_000_000, 50))]
    big = [(m, G) for m, _ in MODELS.values()]
    for m, g in small + big:
        om, og = m.to_c(), g.to_c()
        L = int(m.num_layers)
        n = 400_000
        t = np.zeros(n, TUPLE_DTYPE)
        q = n // 4
        t["cached"][:q] = rng.integers(0, 3000, q)                    # dense small values: exact quotients
        t["cached"][q:2 * q] = rng.integers(60_000, 70_000, q)        # both sides of the 65536-entry table
        t["cached"][2 * q:] = rng.integers(0, 2**32, n - 2 * q, dtype=np.uint64)  # wrap-around in acts / bytes
        t["incoming"] = np.where(rng.random(n) < 0.5, rng.integers(0, 20_000, n), rng.integers(0, 2**32, n, dtype=np.uint64))
        t["charged"] = np.where(rng.random(n) < 0.5, rng.integers(0, 20_000, n), rng.integers(0, 2**32, n, dtype=np.uint64))
        t["batch"] = np.where(rng.random(n) < 0.8, rng.integers(0, 60, n), rng.integers(0, 65536, n))
        t["pending"] = rng.integers(0, min(L + 5, 256), n)
        t["dev_layers"] = rng.integers(0, min(L + 5, 256), n)
        dt = to_dev_tuples(t)
        for cpa in (0, 1):
            got = u32(cs.decide_exact(ctx, m, g, cs.TrainingMode(cpa), dt))
            want = orc.decide_exact(om, og, cpa, t)
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (L, cpa, t[bad[:3]], got[bad[:3]], want[bad[:3]])


def test_decide_host_pipeline(ctx, orc):
    rng = np.random.default_rng(13)
    t = random_tuples(rng, 9_000_001, 32)  # > one 8M pipeline chunk
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), G)
    v, cnt = cs.decide_host(ctx, ms, t, counters=True)
    ref = orc.decide(default_model(), OG, default_grid(), 1, t)
    assert (v == ref).all() and int(cnt[7]) == len(t)


def test_decide_misaligned_rejected(ctx):
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), G)
    buf = torch.zeros(65, dtype=torch.int32, device="cuda")
    with pytest.raises(cs.ColoInvalidArgument):
        cs.decide(ctx, ms, buf[1:].view(16, 4))


# ------------------------------------------------------------ fused path
def four_sets(ctx, hedge_step=None):
    return [cs.MapSet.build(ctx, m, G, mode=mode, hedge_step=hedge_step)
            for m in (cs.ModelProfile(), cs.ModelProfile.phi14b_like()) for mode in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]


OSETS = [(default_model(), OG, 1), (default_model(), OG, 0), (phi14b_model(), OG, 1), (phi14b_model(), OG, 0)]


def test_fused_golden(ctx):
    z = np.load(os.path.join(GOLD, "fused.npz"))
    v = cs.features_decide(ctx, four_sets(ctx), i32(z["prompt"]), i32(z["output"]),
                           torch.from_numpy(z["dev_offsets"].astype(np.int64)).cuda(),
                           torch.from_numpy(z["dev_set"].astype(np.int16)).cuda())
    assert (u32(v) == z["verdicts"]).all()


def ragged_trace(rng, sizes, hi=9000):
    n = int(sum(sizes))
    prompt = rng.integers(1, hi, n).astype(np.uint32)
    output = rng.integers(1, 600, n).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
    return prompt, output, offs


@pytest.mark.parametrize("hedge_step", [None, 250])  # None: table fast path; 250: general compose path
def test_fused_ragged_vs_oracle(ctx, orc, hedge_step):
    rng = np.random.default_rng(21)
    sizes = [0, 1, 2, 3, 127, 128, 129, 0, 5000, 1, 70001, 0, 4096, 33, 200003, 7]
    prompt, output, offs = ragged_trace(rng, sizes)
    dset = np.array([d % 4 for d in range(len(sizes))], np.uint16)
    sets = four_sets(ctx, hedge_step)
    v = cs.features_decide(ctx, sets, i32(prompt), i32(output), torch.from_numpy(offs.astype(np.int64)).cuda(),
                           torch.from_numpy(dset.astype(np.int16)).cuda())
    if hedge_step is None:
        ref = orc.features_decide(OSETS, default_grid(), prompt, output, offs, dset)
    else:  # oracle per device with the 250-step hedge map
        ref = np.zeros(len(prompt), np.uint32)
        for d in range(len(sizes)):
            lo, hi_ = int(offs[d]), int(offs[d + 1])
            m, g, cpa = OSETS[dset[d]]
            p, o = prompt[lo:hi_], output[lo:hi_]
            ch = p.astype(np.uint64) + (2 * o.astype(np.uint64) if cpa else 0)
            t = np.zeros(hi_ - lo, TUPLE_DTYPE)
            t["cached"] = np.concatenate([[0], ch[:-1]]) if hi_ > lo else []
            t["incoming"] = p + o
            t["charged"] = ch
            t["batch"] = 1
            t["dev_layers"] = m.num_layers
            ref[lo:hi_] = orc.decide(m, g, default_grid(), cpa, t, hedge_step=250, hedge_max=8000)
    assert (u32(v) == ref).all()


def test_fused_host_pipeline_and_tuple_crosscheck(ctx, orc):
    """Full-size properties on a 20M-query synthetic trace (crosses the 16M
    host-pipeline chunk): host-buffer path == device path, counters consistent,
    deterministic, equal to the tuple kernel on tuples built from the trace,
    and equal to the oracle on whole sampled devices."""
    sets = four_sets(ctx)
    D, per = 16, 1_250_003
    arr, pr, ou, offs = cs.synth_trace(ctx, [per] * D, [0.05, 0.1, 0.2, 0.3] * 4, 77)
    dset = torch.tensor([d % 4 for d in range(D)], dtype=torch.int16, device="cuda")
    v1, c1 = cs.features_decide(ctx, sets, pr, ou, offs, dset, counters=True)
    v2 = cs.features_decide(ctx, sets, pr, ou, offs, dset)
    assert torch.equal(v1, v2)
    assert int(c1[7]) == D * per and int(c1[0] + c1[1] + c1[2]) == D * per
    f = cs.verdict_fields(u32(v1))  # every counter equals a recount of the verdict words
    exp = [(f["verdict"] == 0).sum(), (f["verdict"] == 1).sum(), (f["verdict"] == 2).sum(), f["offload_oor"].sum(),
           f["hedge_oor"].sum(), f["stream"].sum(), f["stream_oor"].sum(), D * per]
    assert list(c1.cpu().numpy()) == [int(x) for x in exp]
    hp, ho = pr.cpu().numpy().view(np.uint32), ou.cpu().numpy().view(np.uint32)
    hv, hc = cs.features_decide_host(ctx, sets, hp, ho, offs.cpu().numpy(), dset.cpu().numpy(), counters=True)
    assert (hv == u32(v1)).all() and (hc.astype(np.int64) == c1.cpu().numpy()).all()
    # tuple kernel on the same questions, per map set
    offs_h = offs.cpu().numpy()
    for d in (0, 1, 2, 3):
        lo, hi_ = int(offs_h[d]), int(offs_h[d + 1])
        m, g, cpa = OSETS[d % 4]
        p, o = hp[lo:hi_], ho[lo:hi_]
        ch = p.astype(np.uint64) + (2 * o.astype(np.uint64) if cpa else 0)
        t = np.zeros(hi_ - lo, TUPLE_DTYPE)
        t["cached"] = np.concatenate([[0], ch[:-1]])
        t["incoming"] = p + o
        t["charged"] = ch
        t["batch"] = 1
        t["dev_layers"] = m.num_layers
        tv = u32(cs.decide(ctx, sets[d % 4], to_dev_tuples(t)))
        assert (tv == hv[lo:hi_]).all()
        ref = orc.features_decide([OSETS[d % 4]], default_grid(), p, o, np.array([0, hi_ - lo], np.uint64),
                                  np.zeros(1, np.uint16))
        assert (ref == hv[lo:hi_]).all()


def test_features_vs_oracle(ctx, orc):
    rng = np.random.default_rng(31)
    p = rng.integers(1, 100000, 200001).astype(np.uint32)
    o = rng.integers(1, 5000, 200001).astype(np.uint32)
    for (m, om) in MODELS.values():
        for cpa in (0, 1):
            need, ch, pre = cs.features(ctx, m, cs.TrainingMode(cpa), i32(p), i32(o))
            rn, rc, rp = orc.features(om, cpa, p, o)
            assert (need.cpu().numpy().view(np.uint64) == rn).all()
            assert (ch.cpu().numpy().view(np.uint64) == rc).all()
            assert (pre.cpu().numpy().view(np.uint64) == rp.view(np.uint64)).all()


# ----------------------------------------------------------------- replay
def run_replay(ctx, a, p, o, tau, m=None, sets=None, profiles=None, offs=None, dprof=None, segment_len=0):
    profiles = profiles or [(m or cs.ModelProfile(), G)]
    offs = offs if offs is not None else np.array([0, len(p)], np.int64)
    dprof = dprof if dprof is not None else np.zeros(len(offs) - 1, np.int16)
    return cs.replay_serving(ctx, profiles, torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda(), i32(p), i32(o),
                             torch.from_numpy(np.asarray(offs, np.int64)).cuda(),
                             torch.from_numpy(np.asarray(dprof, np.int16)).cuda(), tau=tau, sets=sets, samples=True,
                             labels=True, batches=True, summary=True, segment_len=segment_len)


@pytest.mark.parametrize("segment_len", [1, 3, 17, 64, 1000000])
@pytest.mark.parametrize("qps", [0.05, 0.3, 1.0, 2.5])
def test_replay_segmented_speculation(ctx, orc, segment_len, qps):
    """The speculate/resolve/replay passes are exact for any segment length,
    from idle (0.05 qps) to saturated (2.5 qps) servers."""
    hv, hp = sharegpt_histogram()
    a, p, o = orc.generate_trace(qps, 400.0 / qps, ("histogram", hv, hp), 7)
    o = np.random.default_rng(int(qps * 100)).integers(1, 200, len(o)).astype(np.uint32)
    sets = [cs.MapSet.build(ctx, cs.ModelProfile(), G, mode=cs.TrainingMode.CPA)]
    r = run_replay(ctx, a, p, o, 0.05, sets=sets, segment_len=segment_len)
    ref = orc.replay_serving(default_model(), OG, a, p, o, tau=0.05, grid=default_grid(), cpa=1)
    assert (r["samples"].cpu().numpy().view(np.uint64) == ref["samples"].view(np.uint64)).all()
    assert (r["labels"].cpu().numpy() == ref["labels"]).all()
    S = cs.summaries_to_numpy(r["summary"])[0]
    nb = int(S["batches"])
    assert r["batches"].cpu().numpy()[:nb].tobytes() == ref["batches"].tobytes()
    assert not r["batches"].cpu().numpy()[nb:].any()  # no records left by the speculative passes
    assert S["end_time"] == ref["summary"]["end_time"] and int(S["slow_tokens"]) == ref["summary"]["slow_tokens"]
    exact = sum(int(x) for x in (ref["samples"] * 2.0**96))  # every sample is a multiple of 2^-96 here
    limbs = [int(v) for v in S["tpt_sum"]]
    assert limbs[0] + (limbs[1] << 64) + (limbs[2] << 128) == exact


@pytest.mark.parametrize("name", ["q005", "q03", "q17", "ties", "varout"])
def test_replay_golden(ctx, name):
    z = np.load(os.path.join(GOLD, "replay.npz"))
    a, p, o = z[f"{name}_arrival"], z[f"{name}_prompt"], z[f"{name}_output"]
    sets = [cs.MapSet.build(ctx, cs.ModelProfile(), G, mode=cs.TrainingMode.CPA)]
    r = run_replay(ctx, a, p, o, float(z["tau"][0]), sets=sets)
    assert (r["samples"].cpu().numpy().view(np.uint64) == z[f"{name}_samples"].view(np.uint64)).all()
    assert (r["labels"].cpu().numpy() == z[f"{name}_labels"]).all()
    S = cs.summaries_to_numpy(r["summary"])[0]
    nb = int(S["batches"])
    b = r["batches"].cpu().numpy()[:nb].reshape(-1).view(cs.BATCH_DTYPE)
    assert (b.tobytes() == z[f"{name}_batches"].tobytes())
    assert [int(S[k]) for k in ("generated_tokens", "slow_tokens", "slow_queries", "batches", "peak_device_bytes",
                                "max_batch_size")] == [int(x) for x in z[f"{name}_summary"]]
    assert S["end_time"] == z[f"{name}_end_time"][0]


def test_replay_multidevice_vs_oracle(ctx, orc):
    hv, hp = sharegpt_histogram()
    traces, prof = [], []
    for d, q in enumerate([0.05, 0.3, 1.7, 0.8, 0.2, 2.5, 0.6]):
        a, p, o = orc.generate_trace(q, 900.0, ("histogram", hv, hp), 500 + d)
        if d % 3 == 2:
            o = np.random.default_rng(d).integers(1, 400, len(o)).astype(np.uint32)
        traces.append((a, p, o))
        prof.append(d % 2)
    traces.insert(4, (np.zeros(0), np.zeros(0, np.uint32), np.zeros(0, np.uint32)))
    prof.insert(4, 0)
    a = np.concatenate([t[0] for t in traces])
    p = np.concatenate([t[1] for t in traces]).astype(np.uint32)
    o = np.concatenate([t[2] for t in traces]).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum([len(t[1]) for t in traces])]).astype(np.int64)
    profiles = [(cs.ModelProfile(), G), (cs.ModelProfile.phi14b_like(), G)]
    sets = [cs.MapSet.build(ctx, cs.ModelProfile(), G, mode=cs.TrainingMode.CPA),
            cs.MapSet.build(ctx, cs.ModelProfile.phi14b_like(), G, mode=cs.TrainingMode.CPA)]
    r = run_replay(ctx, a, p, o, 0.05, sets=sets, profiles=profiles, offs=offs, dprof=np.array(prof, np.int16))
    samples = r["samples"].cpu().numpy()
    so = r["sample_offsets"].cpu().numpy()
    labels = r["labels"].cpu().numpy()
    S = cs.summaries_to_numpy(r["summary"])
    B = r["batches"].cpu().numpy().reshape(-1).view(cs.BATCH_DTYPE)
    for d, (ta, tp, to) in enumerate(traces):
        om = [default_model(), phi14b_model()][prof[d]]
        ref = orc.replay_serving(om, OG, ta, tp, to, tau=0.05, grid=default_grid(), cpa=1)
        assert (samples[so[d]:so[d + 1]].view(np.uint64) == ref["samples"].view(np.uint64)).all()
        assert (labels[offs[d]:offs[d + 1]] == ref["labels"]).all()
        nb = int(S[d]["batches"])
        assert (B[offs[d]:offs[d] + nb].tobytes() == ref["batches"].tobytes())
        assert int(S[d]["peak_device_bytes"]) == ref["summary"]["peak_device_bytes"]
        assert int(S[d]["slow_queries"]) == ref["summary"]["slow_queries"]


def test_replay_rejects_bad_traces(ctx):
    a = np.array([0.0, 1.0, 0.5])
    p = np.array([10, 10, 10], np.uint32)
    o = np.array([5, 5, 5], np.uint32)
    with pytest.raises(cs.ColoValidationError):
        run_replay(ctx, a, p, o, 1.0)  # unsorted (workload.hpp:165-169 would reorder; SoA input must be sorted)
    with pytest.raises(cs.ColoValidationError):
        run_replay(ctx, np.array([0.0]), np.array([0], np.uint32), np.array([5], np.uint32), 1.0)
    with pytest.raises(cs.ColoValidationError):  # engine.hpp:70-74
        run_replay(ctx, np.array([0.0]), np.array([70000], np.uint32), np.array([128], np.uint32), 1.0)


def test_serving_stats_exact(ctx, orc):
    hv, hp = sharegpt_histogram()
    a, p, o = orc.generate_trace(1.1, 1500.0, ("histogram", hv, hp), 1)
    ref = orc.replay_serving(default_model(), OG, a, p, o)
    p50, p90, p99, mean = orc.finalize(ref["samples"])
    args = (ctx, [(cs.ModelProfile(), G)], torch.from_numpy(a).cuda(), i32(p), i32(o),
            torch.tensor([0, len(p)], dtype=torch.int64).cuda(), torch.zeros(1, dtype=torch.int16).cuda())
    st = cs.serving_stats(*args, tau=0.05)
    assert (st["p50"], st["p90"], st["p99"]) == (p50, p90, p99)
    assert abs(st["mean"] - mean) <= 1e-12 * mean
    pc, tot = cs.serving_stats_c(*args, tau=0.05)
    assert tuple(pc[:3]) == (p50, p90, p99) and abs(pc[3] - mean) <= 1e-12 * mean
    assert tot.generated_tokens == len(ref["samples"])


def test_serving_stats_sparse_passes(ctx, orc, monkeypatch):
    """Sparse narrowing passes (only batches whose first-pass sample-bin range
    covers a filter bin are replayed) give the same percentiles, counters and
    exact sums as full passes, in Python and through the C-ABI, and both equal
    finalize over the union of the reference's samples."""
    hv, hp = sharegpt_histogram()
    tr = [orc.generate_trace(q, 3000.0, ("histogram", hv, hp), 20 + i) for i, q in enumerate((0.05, 0.3, 1.1, 2.5))]
    a = np.concatenate([t[0] for t in tr])
    p = np.concatenate([t[1] for t in tr])
    o = np.concatenate([t[2] for t in tr])
    off = np.concatenate([[0], np.cumsum([len(t[0]) for t in tr])]).astype(np.int64)
    smp = np.concatenate([orc.replay_serving(default_model(), OG, *t)["samples"] for t in tr])
    want = orc.finalize(smp)
    args = (ctx, [(cs.ModelProfile(), G)], torch.from_numpy(a).cuda(), i32(p), i32(o), torch.from_numpy(off).cuda(),
            torch.zeros(len(tr), dtype=torch.int16).cuda())
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("COLO_SPARSE_STATS", mode)
        st = cs.serving_stats(*args, tau=0.05)
        pc, tot = cs.serving_stats_c(*args, tau=0.05)
        assert (st["p50"], st["p90"], st["p99"]) == tuple(want[:3]) == tuple(pc[:3]), mode
        got[mode] = (st, tuple(pc), tot.generated_tokens, tot.slow_tokens, list(tot.tpt_sum))
    assert got["1"] == got["0"]


def test_mapset_save_load_roundtrip(ctx, tmp_path):  # maps.hpp:118-191, 284-332 through device map sets
    for m, mode in ((cs.ModelProfile(), cs.TrainingMode.CPA), (cs.ModelProfile.phi14b_like(), cs.TrainingMode.CPT)):
        ms = cs.MapSet.build(ctx, m, G, mode=mode)
        po, ph = str(tmp_path / "o.map"), str(tmp_path / "h.map")
        cs.save_mapset(ms, po, ph)
        ld = cs.load_mapset(ctx, m, G, po, ph)
        assert (ld.cells()[0] == ms.cells()[0]).all() and (ld.cells()[1] == ms.cells()[1]).all()
        assert ld.offload.lookup(4000, 2000, 10) == ms.offload.lookup(4000, 2000, 10)
        other = cs.ModelProfile(prefill_coef_quad=3e-8, num_layers=m.num_layers)
        with pytest.raises(cs.ColoValidationError, match="hash"):
            cs.load_mapset(ctx, other, G, po, ph)
        ms.offload.save(str(tmp_path / "o2.map"))
        assert open(str(tmp_path / "o2.map"), "rb").read() == open(po, "rb").read()


def test_replay_saturated_fast_path_large(ctx, orc, monkeypatch):
    """Saturated devices long enough to span several partition segments
    (131072 queries each): the resolve pass's all-queued fast path
    (COLO_SAT, default on) gives the same bits as forming every batch
    (COLO_SAT=0) and as the oracle; outputs beyond 128 steps included."""
    hv, hp = sharegpt_histogram()
    traces = []
    for d, q in enumerate([2.5, 1.2, 3.0]):
        a, p, o = orc.generate_trace(q, 330000.0 / q, ("histogram", hv, hp), 900 + d)
        if d == 1:
            o = np.random.default_rng(5).integers(1, 300, len(o)).astype(np.uint32)
        traces.append((a, p, o))
    a = np.concatenate([t[0] for t in traces])
    p = np.concatenate([t[1] for t in traces]).astype(np.uint32)
    o = np.concatenate([t[2] for t in traces]).astype(np.uint32)
    offs = np.concatenate([[0], np.cumsum([len(t[1]) for t in traces])]).astype(np.int64)
    assert min(len(t[0]) for t in traces) > 2 * 131072
    outs = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("COLO_SAT", flag)
        r = run_replay(ctx, a, p, o, 0.05, offs=offs)
        outs[flag] = {k: r[k].cpu().numpy() for k in ("samples", "labels", "summary")}
    for k in ("samples", "labels", "summary"):
        assert outs["1"][k].tobytes() == outs["0"][k].tobytes(), k
    ctx.release_scratch()  # caches are dropped and rebuilt on demand
    monkeypatch.setenv("COLO_SAT", "1")
    r = run_replay(ctx, a, p, o, 0.05, offs=offs)
    assert r["samples"].cpu().numpy().tobytes() == outs["1"]["samples"].tobytes()
    d = 1  # the variable-output device against the oracle
    ref = orc.replay_serving(default_model(), OG, traces[d][0], traces[d][1], traces[d][2], tau=0.05)
    S = cs.summaries_to_numpy(outs["1"]["summary"])
    lo, hi = int(offs[d]), int(offs[d + 1])
    assert (outs["1"]["labels"][lo:hi] == ref["labels"]).all()
    assert S[d]["end_time"] == ref["summary"]["end_time"]
    assert int(S[d]["generated_tokens"]) == ref["summary"]["generated_tokens"]


def test_sort_f64_matches_numpy(ctx):
    """colo_sort_f64 (the device sort of TPT samples for export_tpt_cdf)."""
    import ctypes as C

    x = np.random.default_rng(3).exponential(0.05, 1_000_003)
    x[::7] = 0.0
    d_in = torch.from_numpy(x).cuda()
    d_out = torch.empty_like(d_in)
    cs.check(cs.lib().colo_sort_f64(ctx.h, C.c_void_p(d_in.data_ptr()), C.c_void_p(d_out.data_ptr()), len(x)), ctx.h)
    assert np.array_equal(d_out.cpu().numpy().view(np.uint64), np.sort(x).view(np.uint64))


def test_replay_reuse_entries_guarded(orc):
    """reuse_entries only reuses a previous replay of the same trace buffers;
    otherwise (fresh context, other buffers) the call replays in full."""
    hv, hp = sharegpt_histogram()
    fresh = cs.Context(0)
    a1, p1, o1 = orc.generate_trace(0.8, 2000.0, ("histogram", hv, hp), 21)
    a2, p2, o2 = orc.generate_trace(1.5, 2000.0, ("histogram", hv, hp), 22)

    def run(a, p, o, reuse):
        r = cs.replay_serving(fresh, [(cs.ModelProfile(), G)], torch.from_numpy(a).cuda(), i32(p), i32(o),
                              torch.tensor([0, len(a)], dtype=torch.int64, device="cuda"),
                              torch.zeros(1, dtype=torch.int16, device="cuda"), tau=0.05, samples=True,
                              reuse_entries=reuse)
        return r["samples"].cpu().numpy(), r["labels"].cpu().numpy()

    ref1 = orc.replay_serving(default_model(), OG, a1, p1, o1, tau=0.05)
    ref2 = orc.replay_serving(default_model(), OG, a2, p2, o2, tau=0.05)
    s, lab = run(a1, p1, o1, True)  # nothing to reuse on a fresh context
    assert np.array_equal(s.view(np.uint64), ref1["samples"].view(np.uint64)) and np.array_equal(lab, ref1["labels"])
    s, lab = run(a2, p2, o2, True)  # different buffers: replays in full
    assert np.array_equal(s.view(np.uint64), ref2["samples"].view(np.uint64)) and np.array_equal(lab, ref2["labels"])
    fresh.close()
