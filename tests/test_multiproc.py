"""Multi-rank host logic on CPU (gloo, world_size 2): devices shard across
ranks (device d -> rank d % W) with no data-path exchange; the only
collective is the stats all-reduce of the radix-select protocol.  The
combined percentiles must equal the reference finalize over every sample."""
import math
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _traces():
    sys.path.insert(0, ROOT)
    from oracle.oracle import OracleLib, sharegpt_histogram

    orc = OracleLib("oracle")
    hv, hp = sharegpt_histogram()
    return [orc.generate_trace(q, 300.0, ("histogram", hv, hp), 100 + d) for d, q in enumerate([0.05, 0.3, 1.7, 0.8, 0.2])]


def _worker(rank, world, port, outq):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.oracle import OracleLib, default_gpu, default_model
    from paper_2503_01066_b200 import colosim as cs
    from test_host_logic import numpy_pass

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    orc = OracleLib("oracle")
    mine = [t for d, t in enumerate(_traces()) if d % world == rank]
    samples = [orc.replay_serving(default_model(), default_gpu(), *t)["samples"] for t in mine]
    out = cs.stats_protocol(numpy_pass(samples), reduce=lambda t: dist.all_reduce(t))
    # flags are OR-ed across ranks: only rank 1 saw a sample outside the exact sum's range
    flagged = cs.stats_protocol(numpy_pass(samples, flags=1 if rank == 1 else 0), reduce=lambda t: dist.all_reduce(t))
    out["or_flags"], out["or_mean_exact"] = flagged["flags"], flagged["mean_exact"]
    outq.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_stats_reduce():
    sys.path.insert(0, ROOT)
    from oracle.oracle import OracleLib, default_gpu, default_model

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    orc = OracleLib("oracle")
    alls = np.concatenate([orc.replay_serving(default_model(), default_gpu(), *t)["samples"] for t in _traces()])
    p50, p90, p99, mean = orc.finalize(alls)
    for r in (0, 1):
        o = res[r]
        assert o["generated_tokens"] == len(alls)
        assert (o["p50"], o["p90"], o["p99"]) == (p50, p90, p99)
        assert abs(o["mean"] - mean) <= 1e-12 * mean
        assert o["flags"] == 0 and o["mean_exact"]
        assert o["or_flags"] & 1 and not o["or_mean_exact"]
