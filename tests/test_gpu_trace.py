"""validate_trace on the device (colo_validate_trace; workload.hpp:164-188).

The reference's own load_trace (oracle/_ref: validate_trace's stable sort by
(arrival_time, query_id) and its checks) orders a shuffled trace with forced
arrival ties; colo_validate_trace must order the same rows the same way, per
device of a CSR trace, and refuse what the reference refuses."""
import ctypes as C
import os

import numpy as np
import pytest
import torch

from oracle.oracle import OracleLib
from paper_2503_01066_b200 import colosim as cs

pytestmark = pytest.mark.gpu
HAVE_REF = os.path.exists(os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libcolo_ref.so"))


@pytest.fixture(scope="module")
def ctx():
    return cs.Context(0)


def _ref_order(tmp_path, a, p, o, q, ld):
    """Rows as the reference's load_trace returns them (written with the query ids given)."""
    path = str(tmp_path / "t.jsonl")
    with open(path, "w") as f:
        for i in range(len(a)):
            ldv = "null" if np.isnan(ld[i]) else repr(float(ld[i]))
            f.write(f'{{"query_id": {int(q[i])}, "arrival_time": {float(a[i])!r}, "prompt_tokens": {int(p[i])}, '
                    f'"output_tokens": {int(o[i])}, "label_delay": {ldv}}}\n')
    ref = OracleLib("ref").lib
    n = len(a)
    ra, rp, ro, rq, rl = np.empty(n), np.empty(n, np.uint32), np.empty(n, np.uint32), np.empty(n, np.uint64), np.empty(n)
    ref.ref_load_trace.restype = C.c_int64
    rn = ref.ref_load_trace(path.encode(), *[x.ctypes.data_as(C.c_void_p) for x in (ra, rp, ro, rq, rl)], C.c_size_t(n))
    assert rn == n
    return ra, rp, ro, rq, rl


def _device(*cols):
    return [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols]


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_validate_trace_orders_like_reference(ctx, tmp_path):
    rng = np.random.default_rng(5)
    sizes = [1, 0, 3000, 17, 5000]
    devs = []
    for k, n in enumerate(sizes):
        a = np.round(rng.uniform(0, 50, n), 1)  # many exact ties
        p = rng.integers(1, 4000, n).astype(np.uint32)
        o = rng.integers(1, 300, n).astype(np.uint32)
        q = rng.permutation(10 * n + 7)[:n].astype(np.uint64)
        ld = np.where(rng.random(n) < 0.3, np.nan, rng.uniform(0, 5, n))
        devs.append((a, p, o, q, ld))
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    cat = lambda i: np.concatenate([d[i] for d in devs])
    da, dp, do, dq, dl, doff = _device(cat(0), cat(1).view(np.int32), cat(2).view(np.int32), cat(3).view(np.int64),
                                       cat(4), off)
    cs.validate_trace(ctx, da, dp, do, doff, query_id=dq, label_delay=dl)
    ga, gp, go = da.cpu().numpy(), dp.cpu().numpy().view(np.uint32), do.cpu().numpy().view(np.uint32)
    gq, gl = dq.cpu().numpy().view(np.uint64), dl.cpu().numpy()
    for k, d in enumerate(devs):
        if not len(d[0]):
            continue
        lo, hi = off[k], off[k + 1]
        ra, rp, ro, rq, rl = _ref_order(tmp_path, *d)
        assert np.array_equal(ga[lo:hi].view(np.uint64), ra.view(np.uint64)), k
        assert np.array_equal(gp[lo:hi], rp) and np.array_equal(go[lo:hi], ro) and np.array_equal(gq[lo:hi], rq), k
        assert np.array_equal(np.isnan(gl[lo:hi]), np.isnan(rl)) and np.array_equal(gl[lo:hi][~np.isnan(rl)],
                                                                                      rl[~np.isnan(rl)]), k
    # already ordered: a second call changes nothing
    before = [t.clone() for t in (da, dp, do, dq, dl)]
    cs.validate_trace(ctx, da, dp, do, doff, query_id=dq, label_delay=dl)
    bitsof = lambda t: t.view(torch.int64) if t.dtype == torch.float64 else t  # NaN label delays compare by bits
    assert all(torch.equal(bitsof(x), bitsof(y)) for x, y in zip(before, (da, dp, do, dq, dl)))


def test_validate_trace_positional_ids_keep_tie_order(ctx):
    a = np.array([3.0, 1.0, 1.0, 2.0, 1.0])
    p = np.array([1, 2, 3, 4, 5], np.uint32)
    o = np.full(5, 7, np.uint32)
    da, dp, do, doff = _device(a, p.view(np.int32), o.view(np.int32), np.array([0, 5], np.int64))
    cs.validate_trace(ctx, da, dp, do, doff)
    assert da.cpu().tolist() == [1.0, 1.0, 1.0, 2.0, 3.0]
    assert dp.cpu().tolist() == [2, 3, 5, 4, 1]  # stable: equal arrivals keep their row order


def test_validate_trace_refusals(ctx):
    def run(a, p, o, q, off=None):
        n = len(a)
        off = np.array([0, n] if off is None else off, np.int64)
        da, dp, do, dq, doff = _device(np.array(a, np.float64), np.array(p, np.uint32).view(np.int32),
                                       np.array(o, np.uint32).view(np.int32), np.array(q, np.uint64).view(np.int64), off)
        cs.validate_trace(ctx, da, dp, do, doff, query_id=dq)

    with pytest.raises(cs.ColoValidationError, match="duplicate query_id: 7"):
        run([1.0, 2.0, 3.0], [1, 1, 1], [1, 1, 1], [7, 3, 7])
    with pytest.raises(cs.ColoValidationError, match="query 4: negative arrival_time"):
        run([1.0, -2.0], [1, 1], [1, 1], [3, 4])
    with pytest.raises(cs.ColoValidationError, match="query 9: prompt_tokens must be >= 1"):
        run([1.0, 2.0], [1, 0], [1, 1], [3, 9])
    with pytest.raises(cs.ColoValidationError, match="query 3: output_tokens must be >= 1"):
        run([1.0, 2.0], [1, 1], [0, 1], [3, 9])
    # the same id on two devices is fine (separate traces)
    run([1.0, 2.0, 1.0, 2.0], [1, 1, 1, 1], [1, 1, 1, 1], [5, 6, 5, 6], off=[0, 2, 4])
