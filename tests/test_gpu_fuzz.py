"""Randomised parity (fixed seeds): colocated / SeparateCluster / ServingOnly
replays of random profiles, loads, output lengths, label delays and cache
timeouts, one warp per device and in forced segments of random length, against
the plain-C restatement (every report field, sample and label; breaches as
breaches), colo_finalize against numpy's sequential sum, and the exact-stats
protocol (sparse and full narrowing passes) against finalize over the union of
the reference samples of random multi-device sets."""
import math
import os

import numpy as np
import pytest
import torch

from oracle.oracle import (KGB, KGIB, Grid, OracleLib, default_gpu, default_model, phi14b_model,
                           sharegpt_histogram)
from paper_2503_01066_b200 import colosim as cs
from test_gpu_colocated import diff, mapset, upload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return cs.Context(0)


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def test_fuzz_colocated_modes_and_segments(ctx, orc):
    hv, hp = sharegpt_histogram()
    rng = np.random.default_rng(2024)
    for it in range(16):
        m = default_model() if rng.random() < 0.5 else phi14b_model()
        g = default_gpu()
        g.capacity_bytes = int(rng.choice([48, 60, 80, 96])) * KGIB
        g.d2h_bandwidth = int(rng.choice([2, 8, 24])) * KGB
        g.h2d_bandwidth = int(rng.choice([4, 24, 100])) * KGB
        grid = Grid(int(rng.choice([250, 500])), 500, 5, 8000, 8000, 50)
        cpa = bool(rng.random() < 0.6)
        qps = float(rng.choice([0.02, 0.05, 0.1, 0.3, 0.8]))
        nq = int(rng.choice([3000, 8000]))
        dist = ("histogram", hv, hp) if rng.random() < 0.6 else ("uniform", 100.0, 6000.0)
        ldspec = (("fixed", float(rng.choice([0.0, 0.01, 1.0]))) if rng.random() < 0.5
                  else ("uniform", 0.0, float(rng.choice([5.0, 60.0]))))
        a, p, o, ld = orc.generate_trace(qps, nq / qps, dist, 700 + it, ldspec, with_labels=True)
        if rng.random() < 0.3:
            o = rng.integers(1, 400, len(a)).astype(np.uint32)
        if rng.random() < 0.2:
            ld[rng.random(len(ld)) < 0.3] = -1.0
        to = float(rng.choice([5.0, 30.0, 60.0, 600.0]))
        mode = ["colocated", "baseline", "serving-only"][int(rng.integers(0, 3))]
        ref = orc.replay_colocated(m, g, grid, int(cpa), a, p, o, ld, to, tau=0.05, sim_mode=mode)
        ms = mapset(ctx, m, g, grid, cpa)
        da, dp, do, dld, doff, off = upload([(a, p, o, ld)])
        dset = torch.zeros(1, dtype=torch.int16, device="cuda")
        sm = cs.SimMode.parse(mode)
        for seg in (None, int(rng.integers(16, 900))):
            kw = dict(label_delay=dld, cache_timeout=to, tau=0.05, sim_mode=sm, seg_len=seg)
            if ref["rc"] == 3:
                with pytest.raises(cs.ColoBreachError):
                    cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, **kw)
                continue
            r = cs.replay_colocated(ctx, [ms], da, dp, do, doff, dset, samples=True, **kw)
            s = cs.colocated_summaries(r["summary"])[0]
            assert not diff(s, ref["report"]), (it, mode, seg, diff(s, ref["report"]))
            assert np.array_equal(r["samples"].cpu().numpy().view(np.uint64), ref["samples"].view(np.uint64)), (it, seg)
            assert np.array_equal(r["labels"].cpu().numpy(), ref["labels"]), (it, seg)
        if len(ref["samples"]):
            srt = np.sort(ref["samples"])
            n = len(srt)
            rk = lambda q: float(srt[max(1, math.ceil(q * n)) - 1])
            want = [rk(0.5), rk(0.9), rk(0.99), float(np.cumsum(srt)[-1]) / n]
            got = cs.finalize(ctx, torch.from_numpy(ref["samples"]).cuda())
            assert np.array_equal(np.array(got).view(np.uint64), np.array(want).view(np.uint64)), it


def test_fuzz_stats_protocol(ctx, orc, monkeypatch):
    hv, hp = sharegpt_histogram()
    rng = np.random.default_rng(77)
    profiles = [(cs.ModelProfile(), cs.GpuProfile()), (cs.ModelProfile.phi14b_like(), cs.GpuProfile())]
    omodels = [default_model(), phi14b_model()]
    for it in range(10):
        D = int(rng.integers(1, 7))
        tr = []
        for d in range(D):
            q = float(rng.choice([0.02, 0.1, 0.4, 1.2, 3.0]))
            a, p, o = orc.generate_trace(q, float(rng.choice([300, 2000])), ("histogram", hv, hp), 90 * it + d)
            if rng.random() < 0.4:
                o = rng.integers(1, 300, len(a)).astype(np.uint32)
            tr.append((a, p, o))
        prof = rng.integers(0, 2, D).astype(np.int16)
        smp = np.concatenate([orc.replay_serving(omodels[prof[d]], default_gpu(), *tr[d])["samples"] for d in range(D)])
        want = orc.finalize(smp)
        cat = lambda k, dt: torch.from_numpy(np.concatenate([t[k] for t in tr]).view(dt)).cuda()
        off = np.concatenate([[0], np.cumsum([len(t[0]) for t in tr])]).astype(np.int64)
        args = (ctx, profiles, cat(0, np.float64), cat(1, np.int32), cat(2, np.int32), torch.from_numpy(off).cuda(),
                torch.from_numpy(prof).cuda())
        outs = []
        for mode in ("1", "0"):
            monkeypatch.setenv("COLO_SPARSE_STATS", mode)
            st = cs.serving_stats(*args, tau=0.05)
            assert (st["p50"], st["p90"], st["p99"]) == tuple(want[:3]), (it, mode)
            assert abs(st["mean"] - want[3]) <= 1e-12 * abs(want[3])
            outs.append(st)
        assert outs[0] == outs[1], it
