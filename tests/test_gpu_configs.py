"""Parity at BASELINE.json's configuration sizes, output for output.

- C1 (configs[0]): the 1M-query single-device trace (generate_trace,
  ShareGPT-like lengths, seed 41, label delay 0.01 s) at qps 0.3 and 1.7.
  * Serving-only: TPT samples, labels, batch records, replay-derived verdicts,
    the summary and finalize (p50/p90/p99/mean) are each checked bit for bit
    against the reference's own Simulation::run (oracle/_ref).
  * Colocated: every MetricsReport field, the TPT samples, the batch timeline
    and finalize are checked against oracle/_ref, and the labels against the
    plain-C restatement.
- C3 (configs[2]): two whole bursty devices of the 1B-query set, llama8b/CPA
  and phi14b/CPT, at 7,812,500 queries each.  The full 128-device launch (the
  bench step, with verdicts) gives the same labels, summaries and verdicts as
  a launch over the two devices alone.  That launch's samples, labels, batch
  records, verdicts and summaries equal the restatement's, and its exact
  percentiles equal a sort of the restatement's samples.
- C4 (configs[3]): two sampled devices of a rank's 1B-query share at
  7,812,500 queries each.  Their trace-fused verdicts equal oracle/_ref's
  (the reference's own map lookups).  Their replays equal the restatement's,
  and the fleet statistics over the two devices equal finalize over the union
  of the restatement's samples (percentiles exact, mean within 1e-12).

The BASELINE-size devices use the restatement (oracle/colo_oracle.c) rather
than Simulation::run: the reference's event log and its finalize sort of 1e9
samples take tens of GB and minutes per device.  The restatement is pinned to
the reference on the golden fixtures and on fresh random traces
(tests/test_oracle_golden.py), and by the C1 tests above at 1M queries."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle.oracle import (METRICS_FIELDS, OracleLib, default_grid, default_gpu, default_model,
                           phi14b_model)
from paper_2503_01066_b200 import colosim as cs

from exact import exact_mean_cuda, is_nearest_rank

pytestmark = pytest.mark.gpu
TAU = 0.05
C1_QUERIES = 1_000_000
BIG_PER_DEVICE = 7_812_500


@pytest.fixture(scope="module")
def ctx():
    c = cs.Context(0)
    yield c
    c.release_scratch()


@pytest.fixture(scope="module")
def ref():
    return OracleLib("ref")


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def c1_trace(qps):
    hv, hp = cs.sharegpt_histogram()
    return cs.generate_trace(qps, C1_QUERIES / qps, ("histogram", hv, hp), 41, ("fixed", 0.01))


def to_dev(a, p, o):
    return (torch.from_numpy(np.ascontiguousarray(a)).cuda(), torch.from_numpy(p.view(np.int32)).cuda(),
            torch.from_numpy(o.view(np.int32)).cuda())


def bits(x):
    return np.ascontiguousarray(x, np.float64).view(np.uint64)


def gpu_batches(raw, lo, nb):
    return raw[lo:lo + nb].cpu().numpy().copy().view(cs.BATCH_DTYPE).reshape(-1)


def same_batches(g, r):
    assert len(g) == len(r)
    for f in ("first", "n", "need_total", "max_incoming", "verdict"):
        assert np.array_equal(g[f], r[f]), f
    for f in ("start", "end"):
        assert np.array_equal(bits(g[f]), bits(r[f])), f


def same_summary(S, R):
    for f in ("generated_tokens", "slow_tokens", "slow_queries", "batches", "peak_device_bytes", "max_batch_size"):
        assert int(S[f]) == int(R[f]), f
    assert bits([S["end_time"]])[0] == bits([R["end_time"]])[0]


@pytest.mark.parametrize("qps", [0.3, 1.7])
def test_c1_serving_full_size_vs_reference(ctx, ref, qps):
    a, p, o = c1_trace(qps)
    assert len(p) > 0.99 * C1_QUERIES
    m, g = cs.ModelProfile(), cs.GpuProfile()
    sets = [cs.MapSet.build(ctx, m, g, mode=cs.TrainingMode.CPA)]
    da, dp, do = to_dev(a, p, o)
    offs = torch.tensor([0, len(p)], dtype=torch.int64, device="cuda")
    prof = torch.zeros(1, dtype=torch.int16, device="cuda")
    r = cs.replay_serving(ctx, [(m, g)], da, dp, do, offs, prof, tau=TAU, sets=sets, samples=True, labels=True,
                          batches=True, summary=True, verdicts=True)
    R = ref.replay_serving(default_model(), default_gpu(), a, p, o, tau=TAU, grid=default_grid(), cpa=True)
    smp = r["samples"].cpu().numpy()
    assert np.array_equal(bits(smp), bits(R["samples"]))
    assert np.array_equal(r["labels"].cpu().numpy(), R["labels"])
    S = cs.summaries_to_numpy(r["summary"])[0]
    same_summary(S, R["summary"])
    nb = int(S["batches"])
    b = gpu_batches(r["batches"], 0, nb)
    same_batches(b, R["batches"])
    assert np.array_equal(r["verdicts"][:nb].cpu().numpy().view(np.uint32), R["batches"]["verdict"])
    fin = cs.finalize(ctx, r["samples"])
    assert np.array_equal(bits(fin), bits(R["pctl"])), (fin, R["pctl"])


@pytest.mark.parametrize("qps", [0.3, 1.7])
def test_c1_colocated_full_size_vs_reference(ctx, ref, orc, qps):
    a, p, o = c1_trace(qps)
    m, g = cs.ModelProfile(), cs.GpuProfile()
    sets = [cs.MapSet.build(ctx, m, g, mode=cs.TrainingMode.CPA)]
    da, dp, do = to_dev(a, p, o)
    offs = torch.tensor([0, len(p)], dtype=torch.int64, device="cuda")
    dset = torch.zeros(1, dtype=torch.int16, device="cuda")
    r = cs.replay_colocated(ctx, sets, da, dp, do, offs, dset, tau=TAU, samples=True, labels=True, batches=True)
    ld = np.full(len(a), 0.01)
    with ThreadPoolExecutor(2) as ex:
        fr = ex.submit(ref.replay_colocated, default_model(), default_gpu(), default_grid(), 1, a, p, o, ld, 60.0,
                       TAU, True, True)
        fo = ex.submit(orc.replay_colocated, default_model(), default_gpu(), default_grid(), 1, a, p, o, ld, 60.0,
                       TAU, False, False)
        R, O = fr.result(), fo.result()
    assert R["rc"] == 0 and O["rc"] == 0
    s = cs.colocated_summaries(r["summary"])[0]
    assert s["status"] == 0
    bad = []
    for f in METRICS_FIELDS:
        x, y = s[f], R["report"][f]
        if isinstance(x, float) or isinstance(y, float):
            if bits([x])[0] != bits([y])[0]:
                bad.append((f, x, y))
        elif int(x) != int(y):
            bad.append((f, x, y))
    assert not bad, bad
    assert np.array_equal(bits(r["samples"].cpu().numpy()), bits(R["samples"]))
    b = gpu_batches(r["batches"], 0, s["batches"])
    rb = R["batches"]
    assert len(b) == len(rb)
    assert np.array_equal(bits(b["start"]), bits(rb["start"])) and np.array_equal(bits(b["end"]), bits(rb["end"]))
    assert np.array_equal(b["first"], rb["first"]) and np.array_equal(b["n"], rb["n"])
    assert np.array_equal(r["labels"].cpu().numpy(), O["labels"])
    fin = cs.finalize(ctx, r["samples"])
    assert np.array_equal(bits(fin), bits(R["pctl"])), (fin, R["pctl"])


def _oracle_devices(orc, jobs):
    """jobs: list of (Model, cpa, arrival, prompt, output) -> restatement replays (samples, labels, verdicts)."""
    def one(j):
        m, cpa, a, p, o = j
        return orc.replay_serving(m, default_gpu(), a, p, o, tau=TAU, grid=default_grid(), cpa=cpa)

    with ThreadPoolExecutor(len(jobs)) as ex:
        return list(ex.map(one, jobs))


def _check_devices(ctx, profiles, sets, arr, pr, ou, offs_h, devs, dprof_of, O, full=None):
    """Replay the devices `devs` alone on the GPU and hold them to the restatement results O."""
    parts = [(int(offs_h[d]), int(offs_h[d + 1])) for d in devs]
    sa = torch.cat([arr[lo:hi] for lo, hi in parts])
    sp = torch.cat([pr[lo:hi] for lo, hi in parts])
    so = torch.cat([ou[lo:hi] for lo, hi in parts])
    soff = torch.tensor(np.cumsum([0] + [hi - lo for lo, hi in parts]), dtype=torch.int64, device="cuda")
    sprof = torch.tensor([dprof_of(d) for d in devs], dtype=torch.int16, device="cuda")
    r = cs.replay_serving(ctx, profiles, sa, sp, so, soff, sprof, tau=TAU, sets=sets, samples=True, labels=True,
                          summary=True, verdicts=True)
    S = cs.summaries_to_numpy(r["summary"])
    so_h = soff.cpu().numpy()
    smp_off = r["sample_offsets"].cpu().numpy()
    for i, d in enumerate(devs):
        lo, hi = int(so_h[i]), int(so_h[i + 1])
        Oi = O[i]
        same_summary(S[i], Oi["summary"])
        nb = int(S[i]["batches"])
        assert np.array_equal(r["labels"][lo:hi].cpu().numpy(), Oi["labels"]), d
        assert np.array_equal(r["verdicts"][lo:lo + nb].cpu().numpy().view(np.uint32), Oi["batches"]["verdict"]), d
        g = r["samples"][int(smp_off[i]):int(smp_off[i + 1])].cpu().numpy()
        assert np.array_equal(bits(g), bits(Oi["samples"])), d
        del g
        if full is not None:  # the whole-config launch computed the same device
            flo = int(offs_h[d])
            fS = full["S"][d]
            assert fS.tobytes() == S[i].tobytes(), d
            assert torch.equal(full["labels"][flo:flo + (hi - lo)], r["labels"][lo:hi]), d
            assert torch.equal(full["verdicts"][flo:flo + nb], r["verdicts"][lo:lo + nb]), d
    return r, sa, sp, so, soff, sprof


def _union_stats_check(ctx, profiles, parts, O):
    """serving_stats over the devices == nearest ranks of the sorted union of the
    restatement's samples; the mean equals the union's correctly rounded mean
    (metrics.hpp:48-69's sequential sorted sum drifts from it by its own rounding)."""
    sa, sp, so, soff, sprof = parts
    parts.clear()  # the caller's list: the trace copies go before the union is built
    st = cs.serving_stats(ctx, profiles, sa, sp, so, soff, sprof, tau=TAU)
    del sa, sp, so, soff, sprof
    ctx.release_scratch()
    torch.cuda.empty_cache()
    u = torch.cat([torch.from_numpy(x["samples"]).cuda() for x in O])
    n = u.numel()
    assert st["generated_tokens"] == n
    for q, k in ((0.50, "p50"), (0.90, "p90"), (0.99, "p99")):
        assert is_nearest_rank(u, q, st[k]), k
    assert st["mean"] == exact_mean_cuda(u)  # correctly rounded mean of the union
    assert st["slow_tokens"] == sum(int(x["summary"]["slow_tokens"]) for x in O)
    assert st["slow_queries"] == sum(int(x["summary"]["slow_queries"]) for x in O)


def test_c3_two_whole_bursty_devices_vs_oracle(ctx, orc):
    D = 128
    arr, pr, ou, offs = cs.synth_trace(ctx, [BIG_PER_DEVICE] * D, [0.1] * D, 4242, dev_qps_hi=[3.0] * D,
                                       burst_period=600.0)
    g = cs.GpuProfile()
    profiles = [(cs.ModelProfile(), g), (cs.ModelProfile.phi14b_like(), g)]
    # CPT/CPA alternate by device with the profile: llama8b/CPA even, phi14b/CPT odd
    sets = [cs.MapSet.build(ctx, profiles[0][0], g, mode=cs.TrainingMode.CPA),
            cs.MapSet.build(ctx, profiles[1][0], g, mode=cs.TrainingMode.CPT)]
    dprof = torch.tensor([d % 2 for d in range(D)], dtype=torch.int16, device="cuda")
    rf = cs.replay_serving(ctx, profiles, arr, pr, ou, offs, dprof, tau=TAU, sets=sets, labels=True, summary=True,
                           verdicts=True)
    full = {"S": cs.summaries_to_numpy(rf["summary"]), "labels": rf["labels"], "verdicts": rf["verdicts"]}
    assert int(full["S"]["generated_tokens"].sum()) == int(ou.to(torch.int64).sum())
    offs_h = offs.cpu().numpy()
    devs = [6, 101]
    jobs = []
    for d in devs:
        lo, hi = int(offs_h[d]), int(offs_h[d + 1])
        jobs.append((default_model() if d % 2 == 0 else phi14b_model(), d % 2 == 0, arr[lo:hi].cpu().numpy(),
                     pr[lo:hi].cpu().numpy().view(np.uint32), ou[lo:hi].cpu().numpy().view(np.uint32)))
    O = _oracle_devices(orc, jobs)
    del jobs
    r, *rest = _check_devices(ctx, profiles, sets, arr, pr, ou, offs_h, devs, lambda d: d % 2, O, full)
    del r, rf, full, arr, pr, ou
    torch.cuda.empty_cache()
    _union_stats_check(ctx, profiles, rest, O)


def test_c4_two_sampled_devices_vs_oracle(ctx, ref, orc):
    D = 128  # rank 0's share at 8 GPUs (bench.py run_c4: device d on rank d % world, seed 4040)
    qps = [[0.05, 0.1, 0.2, 0.3][d % 4] for d in range(D)]
    arr, pr, ou, offs = cs.synth_trace(ctx, [BIG_PER_DEVICE] * D, qps, 4040)
    g = cs.GpuProfile()
    models = (cs.ModelProfile(), cs.ModelProfile.phi14b_like())
    sets4 = [cs.MapSet.build(ctx, m, g, mode=md) for m in models for md in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]
    set_of = lambda d: (d % 2) * 2 + (0 if d % 4 < 2 else 1)
    dset = torch.tensor([set_of(d) for d in range(D)], dtype=torch.int16, device="cuda")
    v = cs.features_decide(ctx, sets4, pr, ou, offs, dset)
    offs_h = offs.cpu().numpy()
    devs = [3, 40]  # phi14b/CPT at 0.3 qps, llama8b/CPA at 0.05 qps
    osets = [(default_model(), default_gpu(), 1), (default_model(), default_gpu(), 0),
             (phi14b_model(), default_gpu(), 1), (phi14b_model(), default_gpu(), 0)]
    jobs = []
    for d in devs:
        lo, hi = int(offs_h[d]), int(offs_h[d + 1])
        hp, ho = pr[lo:hi].cpu().numpy().view(np.uint32), ou[lo:hi].cpu().numpy().view(np.uint32)
        want = ref.features_decide([osets[set_of(d)]], default_grid(), hp, ho, np.array([0, hi - lo], np.uint64),
                                   np.zeros(1, np.uint16))
        assert np.array_equal(v[lo:hi].cpu().numpy().view(np.uint32), want), d
        om, cpa = osets[set_of(d)][0], osets[set_of(d)][2]
        jobs.append((om, cpa, arr[lo:hi].cpu().numpy(), hp, ho))
    del v
    O = _oracle_devices(orc, jobs)
    del jobs
    profiles = [(m, g) for m in models]
    # the replay's map sets follow each device's profile and mode; one set per (profile, mode) pair in use
    sets = [sets4[set_of(d)] for d in devs]
    prof_sets = [(sets4[set_of(d)].model, g) for d in devs]
    r, *rest = _check_devices(ctx, prof_sets, sets, arr, pr, ou, offs_h, devs, lambda d: devs.index(d), O)
    del r, arr, pr, ou
    torch.cuda.empty_cache()
    _union_stats_check(ctx, prof_sets, rest, O)
