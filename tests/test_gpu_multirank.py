"""World-2 fleet statistics with the GPU replay passes.

Two ranks (gloo process group; both on cuda:0, since a gpurun box has one
GPU) each hold their share of a small fleet: fleet device g on rank g % 2,
generated with the trace keyed on g (synth_trace dev_ids), in two chunk
contexts per rank that share the first pass's temporaries (fleet_stats, as
bench.py's C4 step).  The all-reduced result on both ranks must equal the
reference finalize over the union of every device's samples (restatement
replays of the same traces): p50/p90/p99 exact, slow counts exact, and the
mean equal to the correctly rounded mean of the union (the reference's
finalize sums the sorted samples sequentially and drifts from it by its own
rounding, about 1e-12 relative here); and it must equal one rank replaying
the whole fleet."""
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLEET_QPS = [0.05, 0.3, 1.7, 0.2, 0.8, 3.0, 0.1, 0.35]
PER = 150_000
SEED = 777
TAU = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _profiles(cs):
    g = cs.GpuProfile()
    return [(cs.ModelProfile(), g), (cs.ModelProfile.phi14b_like(), g)]


def _parts(cs, devices):
    """Chunk contexts over `devices` (two chunks when there are several devices)."""
    owner = cs.Context(0)
    half = max(1, len(devices) // 2)
    parts = []
    for chunk in (devices[:half], devices[half:]):
        if not chunk:
            continue
        cx = owner if not parts else cs.Context(0)
        if cx is not owner:
            cx.share_temps(owner)
        arr, pr, ou, offs = cs.synth_trace(cx, [PER] * len(chunk), [FLEET_QPS[d] for d in chunk], SEED, dev_ids=chunk)
        dprof = torch.tensor([d % 2 for d in chunk], dtype=torch.int16, device="cuda")
        parts.append((cx, arr, pr, ou, offs, dprof))
    return parts


def _worker(rank, world, port, outq):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2503_01066_b200 import colosim as cs

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = [d for d in range(len(FLEET_QPS)) if d % world == rank]
    st = cs.fleet_stats(_parts(cs, mine), _profiles(cs), tau=TAU)
    outq.put((rank, st))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_rank_gpu_fleet_stats_equal_union_finalize():
    sys.path.insert(0, ROOT)
    from oracle.oracle import OracleLib, default_gpu, default_model, phi14b_model
    from paper_2503_01066_b200 import colosim as cs

    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    # the same fleet on one rank, one chunk per device pair
    D = len(FLEET_QPS)
    one = cs.fleet_stats(_parts(cs, list(range(D))), _profiles(cs), tau=TAU)
    # the oracle over the union: every device's trace, generated alone (its id keys the RNG)
    orc = OracleLib("oracle")
    samples, slow_tok, slow_q = [], 0, 0
    c = cs.Context(0)
    for d in range(D):
        a, p, o, _ = cs.synth_trace(c, [PER], [FLEET_QPS[d]], SEED, dev_ids=[d])
        r = orc.replay_serving(default_model() if d % 2 == 0 else phi14b_model(), default_gpu(), a.cpu().numpy(),
                               p.cpu().numpy().view(np.uint32), o.cpu().numpy().view(np.uint32), tau=TAU)
        samples.append(r["samples"])
        slow_tok += int(r["summary"]["slow_tokens"])
        slow_q += int(r["summary"]["slow_queries"])
    u = np.concatenate(samples)
    p50, p90, p99, mean = orc.finalize(u)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from exact import exact_mean

    em = exact_mean(u)
    for st in (res[0], res[1], one):
        assert st["generated_tokens"] == len(u)
        assert (st["p50"], st["p90"], st["p99"]) == (p50, p90, p99)
        assert st["mean"] == em
        assert abs(st["mean"] - mean) <= 1e-10 * mean  # the sequential sorted sum's own drift
        assert st["slow_tokens"] == slow_tok and st["slow_queries"] == slow_q
        assert st["flags"] == 0 and st["mean_exact"]
    for k in ("p50", "p90", "p99", "mean", "exact_sum", "batches", "generated_tokens", "slow_tokens", "slow_queries"):
        assert res[0][k] == res[1][k] == one[k], k


def test_fleet_trace_is_position_independent():
    """A fleet device's synthetic trace depends on its id, not on its rank or
    position (C4 at 2/4/8 GPUs replays the same fleet)."""
    sys.path.insert(0, ROOT)
    from paper_2503_01066_b200 import colosim as cs

    c = cs.Context(0)
    ids = [5, 17, 1000, 3]
    a, p, o, offs = cs.synth_trace(c, [5000, 7000, 3000, 4000], [0.3, 0.05, 1.7, 0.2], 4040, dev_ids=ids)
    offs = offs.cpu().numpy()
    for i, d in enumerate(ids):
        a1, p1, o1, _ = cs.synth_trace(c, [int(offs[i + 1] - offs[i])], [[0.3, 0.05, 1.7, 0.2][i]], 4040, dev_ids=[d])
        lo, hi = int(offs[i]), int(offs[i + 1])
        assert torch.equal(a[lo:hi], a1) and torch.equal(p[lo:hi], p1) and torch.equal(o[lo:hi], o1)
        assert bool((a1[1:] >= a1[:-1]).all())
