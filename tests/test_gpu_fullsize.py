"""Parity at BASELINE.json's full sizes through size-independent properties
(the oracle itself checks whole sampled devices; the rest is held to
identities that do not depend on size):

- C2, 64 devices x 1,562,500 queries (100M): the device path and the
  reference-facing host-buffer path give the same verdicts and counters, and
  two whole devices equal the plain-C restatement.
- C3, 128 bursty devices x 7,812,500 queries (1B): generated tokens equal the
  sum of output lengths; the all-queued fast path, the idle-start blocks and
  the plain per-batch path give the same summaries bit for bit (exact TPT
  sums, end times, slow counts, batch counts) and the same labels.
- C4 stats on one rank's 1B queries: the sparse narrowing passes and full
  passes give the same exact percentiles, counters and exact sums."""
import os

import numpy as np
import pytest
import torch

from oracle.oracle import OracleLib, default_grid, default_gpu, default_model, phi14b_model
from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu
OSETS = [(default_model(), default_gpu(), 1), (default_model(), default_gpu(), 0),
         (phi14b_model(), default_gpu(), 1), (phi14b_model(), default_gpu(), 0)]


@pytest.fixture(scope="module")
def ctx():
    c = cs.Context(0)
    yield c
    c.release_scratch()


def four_sets(ctx):
    g = cs.GpuProfile()
    return [cs.MapSet.build(ctx, m, g, mode=md) for m in (cs.ModelProfile(), cs.ModelProfile.phi14b_like())
            for md in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]


def test_c2_full_size(ctx):
    orc = OracleLib("oracle")
    sets = four_sets(ctx)
    D, per = 64, 1_562_500
    qps = [[0.05, 0.1, 0.2, 0.3][d % 4] for d in range(D)]
    arr, pr, ou, offs = cs.synth_trace(ctx, [per] * D, qps, 1000)
    del arr
    dset = torch.tensor([(d % 2) * 2 + (0 if d % 4 < 2 else 1) for d in range(D)], dtype=torch.int16, device="cuda")
    v, c = cs.features_decide(ctx, sets, pr, ou, offs, dset, counters=True)
    assert int(c[7]) == D * per and int(c[0] + c[1] + c[2]) == D * per
    hp, ho = pr.cpu().numpy().view(np.uint32), ou.cpu().numpy().view(np.uint32)
    hv, hc = cs.features_decide_host(ctx, sets, hp, ho, offs.cpu().numpy(), dset.cpu().numpy(), counters=True)
    vh = v.cpu().numpy().view(np.uint32)
    assert (hv == vh).all() and (hc.astype(np.int64) == c.cpu().numpy()).all()
    offs_h = offs.cpu().numpy()
    ds = dset.cpu().numpy()
    for d in (5, 62):
        lo, hi = int(offs_h[d]), int(offs_h[d + 1])
        ref = orc.features_decide([OSETS[int(ds[d])]], default_grid(), hp[lo:hi], ho[lo:hi],
                                  np.array([0, hi - lo], np.uint64), np.zeros(1, np.uint16))
        assert (ref == vh[lo:hi]).all(), d


def _c3_trace(ctx):
    D, per = 128, 7_812_500
    arr, pr, ou, offs = cs.synth_trace(ctx, [per] * D, [0.1] * D, 4242, dev_qps_hi=[3.0] * D, burst_period=600.0)
    dprof = torch.tensor([d % 2 for d in range(D)], dtype=torch.int16, device="cuda")
    profiles = [(cs.ModelProfile(), cs.GpuProfile()), (cs.ModelProfile.phi14b_like(), cs.GpuProfile())]
    return profiles, arr, pr, ou, offs, dprof


def test_c3_full_size_paths_agree(ctx, monkeypatch):
    profiles, arr, pr, ou, offs, dprof = _c3_trace(ctx)
    want_tokens = int(ou.to(torch.int64).sum())
    runs = {}
    for name, env in (("default", {}), ("no_sat", {"COLO_SAT": "0"}), ("no_singles", {"COLO_SINGLES": "0"})):
        for k in ("COLO_SAT", "COLO_SINGLES"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        r = cs.replay_serving(ctx, profiles, arr, pr, ou, offs, dprof, tau=0.05, labels=True, summary=True)
        S = cs.summaries_to_numpy(r["summary"])
        runs[name] = (S.tobytes(), r["labels"].sum(dtype=torch.int64).item(), r["labels"])
        assert int(S["generated_tokens"].sum()) == want_tokens, name
    base = runs["default"]
    for name in ("no_sat", "no_singles"):
        assert runs[name][0] == base[0], name
        assert torch.equal(runs[name][2], base[2]), name


def test_c4_stats_full_size_sparse_equals_full(ctx, monkeypatch):
    D, per = 128, 7_812_500
    qps = [[0.05, 0.1, 0.2, 0.3][d % 4] for d in range(D)]
    arr, pr, ou, offs = cs.synth_trace(ctx, [per] * D, qps, 4040)
    dprof = torch.tensor([d % 2 for d in range(D)], dtype=torch.int16, device="cuda")
    profiles = [(cs.ModelProfile(), cs.GpuProfile()), (cs.ModelProfile.phi14b_like(), cs.GpuProfile())]
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("COLO_SPARSE_STATS", mode)
        out[mode] = cs.serving_stats(ctx, profiles, arr, pr, ou, offs, dprof, tau=0.05)
    assert out["1"] == out["0"]
    assert out["1"]["generated_tokens"] == int(ou.to(torch.int64).sum())
