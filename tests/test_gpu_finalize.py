"""colo_finalize: finalize (metrics.hpp:56-69) on the device, bit-exact.  The
reference mean is the strictly sequential sum of the ascending-sorted samples;
the device evaluates that left fold exactly in parallel (binade-chunked
integer sums with addend-by-addend fallback at binade crossings and ties), so
the bar is bit equality with numpy's add.accumulate over np.sort, on inputs
built to hit ties-to-even, crossings, zeros, negatives and chunk padding."""
import math

import numpy as np
import pytest
import torch

from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return cs.Context(0)


def ref_finalize(x):
    s = np.sort(x)
    n = len(s)

    def rank(q):
        k = math.ceil(q * float(n))
        return float(s[(1 if k == 0 else k) - 1])

    return [rank(0.5), rank(0.9), rank(0.99), float(np.cumsum(s)[-1]) / float(n)], s


def cases():
    rng = np.random.default_rng(11)
    yield "lognormal", rng.lognormal(-3.5, 0.7, 3_000_000)
    yield "n1", np.array([0.0371])
    yield "n2048", rng.random(2048)
    yield "n2049", rng.random(2049)
    # dyadic values whose last bit falls exactly half a grid step of the running
    # sum (ties-to-even) as the sum moves through binades
    k = rng.integers(0, 64, 1_500_000)
    yield "dyadic", 1.0 + k * 2.0 ** -rng.integers(20, 45, len(k))
    yield "ones_then_tie", np.concatenate([np.ones(1 << 19), np.full(5000, 1.0 + 2.0 ** -34)])
    yield "zeros_negatives", np.concatenate([np.zeros(10000), -rng.random(3000), rng.random(7000) * 1e-300])
    yield "wide", np.concatenate([rng.random(100000) * 1e-12, rng.random(100000) * 1e12])


@pytest.mark.parametrize("name,x", list(cases()), ids=lambda v: v if isinstance(v, str) else "")
def test_finalize_bit_exact(ctx, name, x):
    want, srt = ref_finalize(x)
    d = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    so = torch.empty_like(d)
    got = cs.finalize(ctx, d, sorted_out=so)
    assert np.array_equal(np.array(got).view(np.uint64), np.array(want).view(np.uint64)), (name, got, want)
    assert np.array_equal(so.cpu().numpy().view(np.uint64), srt.view(np.uint64)), name


def test_finalize_empty_and_replay_samples(ctx):
    assert all(math.isnan(v) for v in cs.finalize(ctx, torch.empty(0, dtype=torch.float64, device="cuda")))
    # TPT samples of a serving replay (the values finalize sees in a MetricsReport)
    hv, hp = cs.sharegpt_histogram()
    a, p, o = cs.generate_trace(1.7, 200000 / 1.7, ("histogram", hv, hp), 41, ("fixed", 0.01))
    ms = cs.MapSet.build(ctx, cs.ModelProfile(), cs.GpuProfile(), cs.GridSteps(), cs.GridBounds(), cs.TrainingMode.CPA)
    da, dp, do = (torch.from_numpy(a).cuda(), torch.from_numpy(p.view(np.int32)).cuda(),
                  torch.from_numpy(o.view(np.int32)).cuda())
    offs = torch.tensor([0, len(p)], dtype=torch.int64, device="cuda")
    r = cs.replay_colocated(ctx, [ms], da, dp, do, offs, torch.zeros(1, dtype=torch.int16, device="cuda"), samples=True,
                            sim_mode=cs.SimMode.SERVING_ONLY)
    x = r["samples"]
    want, _ = ref_finalize(x.cpu().numpy())
    got = cs.finalize(ctx, x)
    assert np.array_equal(np.array(got).view(np.uint64), np.array(want).view(np.uint64))


def test_finalize_contract_and_launch_counter(ctx):
    x = torch.rand(5000, dtype=torch.float64, device="cuda")
    with pytest.raises(cs.ColoInvalidArgument):
        cs.finalize(ctx, x, sorted_out=torch.empty(10, dtype=torch.float64, device="cuda"))
    # the library's own launch counter moves with every launch this context makes
    l0 = ctx.launches()
    cs.finalize(ctx, x)
    assert ctx.launches() == l0 + 2  # k_fold_cand + k_fold_walk (the sort is CUB's)
    st = cs.lib().colo_finalize(ctx.h, cs._ptr(x), 5000, cs._ptr(x), (cs.C.c_double * 4)())  # d_sorted aliases the input
    assert st == 1  # COLO_EINVAL
