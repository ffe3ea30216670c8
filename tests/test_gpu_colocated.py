"""GPU parity of the colocated replay (colo_replay_colocated, one warp per
device) against the reference's own Simulation::run in SimMode::Colocated
(golden fixtures from oracle/_ref) and against the plain-C restatement on
fresh traces.  Bar: every MetricsReport field bit-exact (f64 fields compared
as bit patterns), TPT samples bit-exact in reference order, the batch
timeline bit-exact, InvariantBreach runs reported as breaches; exact
nearest-rank percentiles; mean within 1e-12 relative."""
import os

import numpy as np
import pytest
import torch

from oracle.oracle import (KGB, KGIB, METRICS_FIELDS, ColoReport, Gpu, Grid, Model, OracleLib, default_gpu,
                           default_grid, default_model, phi14b_model, sharegpt_histogram)
from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ctx():
    return cs.Context(0)


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "colocated.npz"))


def to_cs(m, g, grid):
    cm = cs.ModelProfile(*[getattr(m, f) for f, _ in Model._fields_])
    cg = cs.GpuProfile(*[getattr(g, f) for f, _ in Gpu._fields_])
    steps = cs.GridSteps(grid.cached_step, grid.incoming_step, grid.batch_step)
    bounds = cs.GridBounds(grid.max_cached, grid.max_incoming, grid.max_batch)
    return cm, cg, steps, bounds


def mapset(ctx, m, g, grid, cpa):
    cm, cg, steps, bounds = to_cs(m, g, grid)
    return cs.MapSet.build(ctx, cm, cg, steps, bounds, cs.TrainingMode(int(cpa)))


def case(z, name):
    m = Model.from_buffer_copy(z[f"{name}_model"].tobytes())
    g = Gpu.from_buffer_copy(z[f"{name}_gpu"].tobytes())
    grid = Grid.from_buffer_copy(z[f"{name}_grid"].tobytes())
    cpa, to, sim = z[f"{name}_cfg"]
    rep = ColoReport.from_buffer_copy(z[f"{name}_report"].tobytes())
    return (m, g, grid, int(cpa), float(to), z[f"{name}_a"], z[f"{name}_p"], z[f"{name}_o"], z[f"{name}_ld"], rep,
            ["serving-only", "colocated", "baseline"][int(sim)])


def upload(traces):
    """traces: list of (a, p, o, ld) -> device SoA + CSR offsets."""
    a = np.concatenate([t[0] for t in traces]) if traces else np.zeros(0)
    p = np.concatenate([t[1] for t in traces]).astype(np.uint32)
    o = np.concatenate([t[2] for t in traces]).astype(np.uint32)
    ld = np.concatenate([t[3] for t in traces]).astype(np.float64)
    off = np.concatenate([[0], np.cumsum([len(t[0]) for t in traces])]).astype(np.int64)
    dev = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x).view(dt)).cuda()
    return (dev(a, np.float64), dev(p, np.int32), dev(o, np.int32), dev(ld, np.float64), dev(off, np.int64), off)


def diff(report, ref):
    bad = []
    for f in METRICS_FIELDS:
        x = report[f]
        y = ref[f] if isinstance(ref, dict) else getattr(ref, f)
        if isinstance(y, float) or isinstance(x, float):
            if np.float64(x).view(np.uint64) != np.float64(y).view(np.uint64):
                bad.append((f, x, y))
        elif int(x) != int(y):
            bad.append((f, x, y))
    return bad


def batches_of(raw, lo, nb):
    b = raw.cpu().numpy()[lo:lo + nb].copy().view(cs.BATCH_DTYPE).reshape(-1)
    return b


SEG = [None, 16]  # automatic (these traces are short: one warp per device), and forced 16-query segments


@pytest.mark.parametrize("seg", SEG)
def test_golden_each_case(ctx, gold, seg):
    for name in gold["names"]:
        m, g, grid, cpa, to, a, p, o, ld, rep, sim = case(gold, name)
        ms = mapset(ctx, m, g, grid, cpa)
        da, dp, do, dld, doff, off = upload([(a, p, o, ld)])
        dset = torch.zeros(1, dtype=torch.int16, device="cuda")
        rc = int(gold[f"{name}_rc"][0])
        sm = cs.SimMode.parse(sim)
        if rc == 3:
            with pytest.raises(cs.ColoBreachError) as ei:
                cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld, cache_timeout=to, sim_mode=sm,
                                    seg_len=seg)
            assert cs.colocated_summaries(ei.value.result["summary"])[0]["status"] == 3, name
            continue
        r = cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld, cache_timeout=to, samples=True,
                                batches=True, sim_mode=sm, seg_len=seg)
        s = cs.colocated_summaries(r["summary"])[0]
        assert s["status"] == 0
        assert not diff(s, rep), (name, diff(s, rep))
        smp = r["samples"].cpu().numpy()
        assert np.array_equal(smp.view(np.uint64), gold[f"{name}_samples"].view(np.uint64)), name
        b = batches_of(r["batches"], 0, s["batches"])
        got = np.stack([b["start"], b["end"], b["first"].astype(np.float64), b["n"].astype(np.float64)], 1)
        gb = gold[f"{name}_batches"]
        assert got.shape == gb.shape and np.array_equal(got.view(np.uint64), gb.view(np.uint64)), name
        # verdict bookkeeping: one EVALUATED per apply_offload_decision, one ADMITTED per admit_to_store
        v = b["verdict"]
        assert int(((v & cs_bit("EVALUATED")) != 0).sum()) == s["offload_decisions"]
        assert int(((v & cs_bit("ADMITTED")) != 0).sum()) == s["admissions"]


def cs_bit(name):
    return {"EVALUATED": 1 << 25, "ADMITTED": 1 << 26}[name]


@pytest.mark.parametrize("seg", SEG)
def test_golden_one_launch_many_devices(ctx, gold, seg):
    """All timeout-60 non-breach fixture cases as devices of ONE launch, each
    with its own map set (profiles, grids, modes mixed), devices replicated so
    several warps share CTAs; every device's slice must equal its fixture."""
    names = [n for n in gold["names"] if int(gold[f"{n}_rc"][0]) == 0 and float(gold[f"{n}_cfg"][1]) == 60.0]
    sets, keys, traces, devs = [], {}, [], []
    for rep_i in range(3):
        for n in names:
            m, g, grid, cpa, to, a, p, o, ld, rep, sim = case(gold, n)
            k = (bytes(m), bytes(g), bytes(grid), cpa)
            if k not in keys:
                keys[k] = len(sets)
                sets.append(mapset(ctx, m, g, grid, cpa))
            traces.append((a, p, o, ld))
            devs.append((n, keys[k], rep, int(cs.SimMode.parse(sim))))
    da, dp, do, dld, doff, off = upload(traces)
    dset = torch.tensor([d[1] for d in devs], dtype=torch.int16, device="cuda")
    dmode = torch.tensor([d[3] for d in devs], dtype=torch.uint8, device="cuda")
    r = cs.replay_colocated(ctx, sets, da, dp, do, doff, dset, label_delay=dld, samples=True, batches=True,
                            sim_mode=dmode, seg_len=seg)
    S = cs.colocated_summaries(r["summary"])
    smp = r["samples"].cpu().numpy()
    so = r["sample_offsets"].cpu().numpy()
    for i, (n, _, rep, _) in enumerate(devs):
        assert not diff(S[i], rep), (n, diff(S[i], rep))
        assert np.array_equal(smp[so[i]:so[i + 1]].view(np.uint64), gold[f"{n}_samples"].view(np.uint64)), n
        b = batches_of(r["batches"], int(off[i]), S[i]["batches"])
        assert np.array_equal(b["start"].view(np.uint64), gold[f"{n}_batches"][:, 0].view(np.uint64)), n


@pytest.mark.parametrize("seg", SEG)
def test_vs_oracle_random(ctx, orc, seg):
    """Fresh traces (variable outputs, label delays, odd GPU profiles): the
    kernel equals the restatement on every field, sample, label and batch."""
    rng = np.random.default_rng(77)
    hv, hp = sharegpt_histogram()
    done = 0
    for it in range(24):
        m = default_model() if it % 2 else phi14b_model()
        g = default_gpu()
        g.capacity_bytes = int(rng.choice([60, 80])) * KGIB
        g.d2h_bandwidth = int(rng.choice([2, 24])) * KGB
        g.h2d_bandwidth = int(rng.choice([4, 24, 200])) * KGB
        grid = Grid(int(rng.choice([250, 500])), 500, 5, 8000, 8000, 50)
        cpa = it % 3 != 0
        qps = float(rng.choice([0.05, 0.2, 0.6, 1.7]))
        dist = ("histogram", hv, hp) if rng.random() < 0.5 else ("uniform", 500.0, 7500.0)
        a, p, o, ld = orc.generate_trace(qps, 60 / qps + 100, dist, 1000 + it, ("uniform", 0.0, 20.0),
                                         with_labels=True)
        if it % 4 == 1:
            o = rng.integers(1, 300, len(a)).astype(np.uint32)
        if it % 5 == 2:
            ld[::3] = -1.0
        ref = orc.replay_colocated(m, g, grid, int(cpa), a, p, o, ld, 30.0, tau=0.05)
        ms = mapset(ctx, m, g, grid, cpa)
        da, dp, do, dld, doff, off = upload([(a, p, o, ld)])
        dset = torch.zeros(1, dtype=torch.int16, device="cuda")
        if ref["rc"] == 3:
            with pytest.raises(cs.ColoBreachError):
                cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld, cache_timeout=30.0, tau=0.05,
                                    seg_len=seg)
            continue
        r = cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld, cache_timeout=30.0, tau=0.05,
                                samples=True, batches=True, seg_len=seg)
        s = cs.colocated_summaries(r["summary"])[0]
        assert not diff(s, ref["report"]), (it, diff(s, ref["report"]))
        for f in ("batches", "max_batch_size", "offload_decisions", "admissions", "slow_tokens", "slow_queries"):
            assert s[f] == ref["report"][f], (it, f)
        assert np.float64(s["end_time"]).view(np.uint64) == np.float64(ref["report"]["end_time"]).view(np.uint64)
        assert np.array_equal(r["samples"].cpu().numpy().view(np.uint64), ref["samples"].view(np.uint64))
        assert np.array_equal(r["labels"].cpu().numpy(), ref["labels"])
        b = batches_of(r["batches"], 0, s["batches"])
        for k in ("start", "end", "first", "n", "need_total", "max_incoming"):
            assert np.array_equal(b[k], ref["batches"][k]), (it, k)
        done += 1
    assert done >= 12


def test_default_label_delay_and_validation(ctx, orc):
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    a, p, o, ld = orc.generate_trace(0.3, 500.0, ("histogram", hv, hp), 5, ("fixed", 0.01), with_labels=True)
    ms = mapset(ctx, m, g, grid, 1)
    da, dp, do, dld, doff, off = upload([(a, p, o, ld)])
    dset = torch.zeros(1, dtype=torch.int16, device="cuda")
    r1 = cs.colocated_summaries(cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld)["summary"])
    r2 = cs.colocated_summaries(cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, default_label_delay=0.01)["summary"])
    assert r1 == r2
    ref = orc.replay_colocated(m, g, grid, 1, a, p, o, None)  # no label ever arrives
    r3 = cs.colocated_summaries(cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, default_label_delay=-1.0)["summary"])
    assert not diff(r3[0], ref["report"])
    bad = a.copy()
    bad[5], bad[6] = bad[6], bad[5] + 1e-3  # unsorted arrivals (validate_trace order)
    db, _, _, _, _, _ = upload([(bad, p, o, ld)])
    with pytest.raises(cs.ColoValidationError):
        cs.replay_colocated(ctx, [ms], db, dp, do, doff, dset)


def test_colocated_stats_exact(ctx, gold, orc):
    """colo_colocated_stats over a multi-device set: nearest-rank percentiles
    equal finalize over the union of the reference's samples; mean within
    1e-12 relative (exact fixed-point sum vs the sorted sequential sum)."""
    names = [n for n in gold["names"] if int(gold[f"{n}_rc"][0]) == 0 and float(gold[f"{n}_cfg"][1]) == 60.0
             and len(gold[f"{n}_samples"])]
    sets, keys, traces, dset, dmode, allsmp = [], {}, [], [], [], []
    for n in names:
        m, g, grid, cpa, to, a, p, o, ld, rep, sim = case(gold, n)
        k = (bytes(m), bytes(g), bytes(grid), cpa)
        if k not in keys:
            keys[k] = len(sets)
            sets.append(mapset(ctx, m, g, grid, cpa))
        traces.append((a, p, o, ld))
        dset.append(keys[k])
        dmode.append(int(cs.SimMode.parse(sim)))
        allsmp.append(gold[f"{n}_samples"])
    da, dp, do, dld, doff, off = upload(traces)
    dset = torch.tensor(dset, dtype=torch.int16, device="cuda")
    dmode = torch.tensor(dmode, dtype=torch.uint8, device="cuda")
    pctl, tot = cs.colocated_stats(ctx, sets, da, dp, do, doff, dset, label_delay=dld, sim_mode=dmode)
    u = np.concatenate(allsmp)
    p50, p90, p99, mean = orc.finalize(u)
    assert pctl[:3] == [p50, p90, p99]
    assert abs(pctl[3] - mean) <= 1e-12 * abs(mean)
    assert tot["generated_tokens"] == len(u)


@pytest.mark.parametrize("seg", SEG)
def test_modes_vs_oracle_random(ctx, orc, seg):
    """ServingOnly and SeparateCluster devices (constant, varying and absent
    label delays: the sorted job-stream path) mixed with Colocated devices in
    one launch; every device equals the restatement."""
    rng = np.random.default_rng(5)
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    phi = phi14b_model()
    sets = [mapset(ctx, m, g, grid, 1), mapset(ctx, m, g, grid, 0), mapset(ctx, phi, g, grid, 1)]
    models = [(m, 1), (m, 0), (phi, 1)]
    traces, dset, dmode, refs = [], [], [], []
    for it in range(36):
        si = it % 3
        mode = ["serving-only", "colocated", "baseline"][(it // 3) % 3]
        qps = float(rng.choice([0.05, 0.3, 1.0, 2.5]))
        dist = ("histogram", hv, hp) if it % 2 else ("uniform", 200.0, 7000.0)
        spec = ("fixed", 0.01) if it % 4 == 0 else ("uniform", 0.0, 100.0)
        a, p, o, ld = orc.generate_trace(qps, 40 / qps + 60, dist, 300 + it, spec, with_labels=True)
        if it % 5 == 1:
            ld[1::3] = -1.0
        if it % 7 == 3:
            o = rng.integers(1, 250, len(a)).astype(np.uint32)
        mm, cpa = models[si]
        ref = orc.replay_colocated(mm, g, grid, cpa, a, p, o, ld, 60.0, tau=0.05, sim_mode=mode)
        if ref["rc"]:
            continue
        traces.append((a, p, o, ld))
        dset.append(si)
        dmode.append(int(cs.SimMode.parse(mode)))
        refs.append(ref)
    da, dp, do, dld, doff, off = upload(traces)
    r = cs.replay_colocated(ctx, sets, da, dp, do, doff, torch.tensor(dset, dtype=torch.int16, device="cuda"),
                            label_delay=dld, tau=0.05, samples=True, batches=True, seg_len=seg,
                            sim_mode=torch.tensor(dmode, dtype=torch.uint8, device="cuda"))
    S = cs.colocated_summaries(r["summary"])
    smp = r["samples"].cpu().numpy()
    so = r["sample_offsets"].cpu().numpy()
    lab = r["labels"].cpu().numpy()
    for i, ref in enumerate(refs):
        assert not diff(S[i], ref["report"]), (i, dmode[i], diff(S[i], ref["report"]))
        assert np.array_equal(smp[so[i]:so[i + 1]].view(np.uint64), ref["samples"].view(np.uint64)), i
        assert np.array_equal(lab[off[i]:off[i + 1]], ref["labels"]), i
        b = batches_of(r["batches"], int(off[i]), S[i]["batches"])
        for k in ("start", "end", "first", "n"):
            assert np.array_equal(b[k], ref["batches"][k]), (i, k)
    assert len(refs) >= 30 and {0, 1, 2} <= set(dmode)


@pytest.mark.parametrize("qps,cpa", [(0.3, 1), (0.1, 0), (1.7, 1)])
def test_segmented_long_trace(ctx, orc, qps, cpa):
    """One long device (the C1 shape, 60k queries): the automatic segmented
    replay (speculate / resolve / replay segments, exact folds of the three
    f64 sums) equals the one-warp replay and the restatement on every report
    field, sample, label and batch.  At 1.7 QPS the server never drains, no
    segment resolves and the device runs whole."""
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    a, p, o, ld = orc.generate_trace(qps, 60000 / qps, ("histogram", hv, hp), 41, ("fixed", 0.01), with_labels=True)
    ref = orc.replay_colocated(m, g, grid, cpa, a, p, o, ld, 60.0, tau=0.05)
    ms = mapset(ctx, m, g, grid, cpa)
    da, dp, do, dld, doff, off = upload([(a, p, o, ld)])
    dset = torch.zeros(1, dtype=torch.int16, device="cuda")
    outs = []
    for seg in (None, 0, 1000):
        r = cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, label_delay=dld, tau=0.05, samples=True,
                                batches=True, seg_len=seg)
        s = cs.colocated_summaries(r["summary"])[0]
        assert not diff(s, ref["report"]), (seg, diff(s, ref["report"]))
        for f in ("batches", "max_batch_size", "offload_decisions", "admissions", "slow_tokens", "slow_queries"):
            assert s[f] == ref["report"][f], (seg, f)
        assert np.array_equal(r["samples"].cpu().numpy().view(np.uint64), ref["samples"].view(np.uint64)), seg
        assert np.array_equal(r["labels"].cpu().numpy(), ref["labels"]), seg
        b = batches_of(r["batches"], 0, s["batches"])
        for k in ("start", "end", "first", "n", "need_total", "max_incoming"):
            assert np.array_equal(b[k], ref["batches"][k]), (seg, k)
        outs.append(b["verdict"].copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


def test_segmented_stats_and_modes(ctx, orc):
    """colo_colocated_stats over two long devices (Colocated CPA at 0.3 QPS,
    SeparateCluster with varying label delays): forced segments, automatic and
    one warp per device give the same percentiles, exact sums and totals."""
    hv, hp = sharegpt_histogram()
    m, g, grid = default_model(), default_gpu(), default_grid()
    tr = []
    for seed, qps, spec in ((3, 0.3, ("fixed", 0.01)), (4, 0.2, ("uniform", 0.0, 30.0))):
        a, p, o, ld = orc.generate_trace(qps, 20000 / qps, ("histogram", hv, hp), seed, spec, with_labels=True)
        tr.append((a, p, o, ld))
    da, dp, do, dld, doff, off = upload(tr)
    sets = [mapset(ctx, m, g, grid, 1)]
    dset = torch.zeros(2, dtype=torch.int16, device="cuda")
    dmode = torch.tensor([int(cs.SimMode.COLOCATED), int(cs.SimMode.SEPARATE_CLUSTER)], dtype=torch.uint8, device="cuda")
    outs = [cs.colocated_stats(ctx, sets, da, dp, do, doff, dset, label_delay=dld, tau=0.05, sim_mode=dmode, seg_len=s)
            for s in (0, None, 700)]
    for pc, tot in outs[1:]:
        assert np.array_equal(np.array(pc).view(np.uint64), np.array(outs[0][0]).view(np.uint64))
        assert tot == outs[0][1]
    for i, (a, p, o, ld) in enumerate(tr):
        ref = orc.replay_colocated(m, g, grid, 1, a, p, o, ld, 60.0, tau=0.05, sim_mode=["colocated", "baseline"][i])
        r = cs.replay_colocated(ctx, sets, da, dp, do, doff, dset, label_delay=dld, tau=0.05, sim_mode=dmode, seg_len=700)
        s = cs.colocated_summaries(r["summary"])[i]
        assert not diff(s, ref["report"]), (i, diff(s, ref["report"]))
