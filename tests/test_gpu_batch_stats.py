"""The first stats pass through the batch structure (speculative/resolve passes
write every batch's start; k_batch_stats replays the batches from those
starts, one per lane) against the full replay pass (COLO_BATCH_STATS=0) and
the oracle, on traces that exercise every branch of the new path:

- idle-start singles and queued single-member batches (the specialised loop),
- queued batches of 2-4 members with different output lengths (alive counts
  change inside the batch) and of more than four members (the warp path),
- arrivals near t = 0, where the TPT sum does not telescope,
- saturated devices (all-queued records, the resolve pass's chain sums),
- segment lengths that cut batches (straddling starts, covered segments).

Bar: labels, summaries (every field incl. the exact fixed-point sum),
histograms equal to the full pass bit for bit; the labels and the TPT sample
count equal the oracle's.  (The narrowing passes over the recorded bin ranges
are held to the full passes by test_gpu_fuzz.py::test_fuzz_stats_protocol.)"""
import numpy as np
import pytest
import torch

from oracle.oracle import OracleLib, default_gpu, default_model, phi14b_model, sharegpt_histogram
from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu
TAU = 0.05


@pytest.fixture(scope="module")
def ctx():
    c = cs.Context(0)
    yield c
    c.release_scratch()


@pytest.fixture(scope="module")
def orc():
    return OracleLib("oracle")


def _traces(orc, rng):
    hv, hp = sharegpt_histogram()
    tr = []
    for d, (q, dur) in enumerate(((0.05, 4000.0), (0.3, 3000.0), (1.1, 1500.0), (3.0, 600.0), (0.2, 2500.0))):
        a, p, o = orc.generate_trace(q, dur, ("histogram", hv, hp), 500 + d)
        if d in (1, 2, 4):  # different output lengths inside batches
            o = rng.integers(1, 300, len(a)).astype(np.uint32)
        if d == 4:  # the first seconds: sums that do not telescope
            a = a * 1e-3
        tr.append((a, p, o))
    return tr


def _run(ctx, profiles, dev, seg, env, monkeypatch):
    monkeypatch.setenv("COLO_BATCH_STATS", env)
    arr, pr, ou, offs, prof = dev
    hist = torch.zeros(cs.HIST_BINS, dtype=torch.int64, device="cuda")
    r = cs.replay_serving(ctx, profiles, arr, pr, ou, offs, prof, tau=TAU, labels=True, summary=True, hist=hist,
                          segment_len=seg, stats_mode=1)
    torch.cuda.synchronize()
    return {"labels": r["labels"].cpu().numpy(), "summary": cs.summaries_to_numpy(r["summary"]),
            "hist": hist.cpu().numpy()}


@pytest.mark.parametrize("seg", [0, 300, 4096])
def test_batch_stats_pass_equals_full_pass(ctx, orc, monkeypatch, seg):
    rng = np.random.default_rng(5)
    tr = _traces(orc, rng)
    profiles = [(cs.ModelProfile(), cs.GpuProfile()), (cs.ModelProfile.phi14b_like(), cs.GpuProfile())]
    prof = np.array([d % 2 for d in range(len(tr))], np.int16)
    cat = lambda k, dt: torch.from_numpy(np.concatenate([t[k] for t in tr]).view(dt)).cuda()
    off = np.concatenate([[0], np.cumsum([len(t[0]) for t in tr])]).astype(np.int64)
    dev = (cat(0, np.float64), cat(1, np.int32), cat(2, np.int32), torch.from_numpy(off).cuda(),
           torch.from_numpy(prof).cuda())
    new = _run(ctx, profiles, dev, seg, "1", monkeypatch)
    old = _run(ctx, profiles, dev, seg, "0", monkeypatch)
    assert np.array_equal(new["labels"], old["labels"])
    assert new["summary"].tobytes() == old["summary"].tobytes()
    assert np.array_equal(new["hist"], old["hist"])
    S = new["summary"]
    om = [default_model(), phi14b_model()]
    for d, t in enumerate(tr):
        ref = orc.replay_serving(om[prof[d]], default_gpu(), *t, tau=TAU)
        assert int(S["generated_tokens"][d]) == len(ref["samples"]), d
        lo, hi = int(off[d]), int(off[d + 1])
        assert np.array_equal(new["labels"][lo:hi], ref["labels"]), d
