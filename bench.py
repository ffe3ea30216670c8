"""Benchmark: per-query admission decisions/s on the C2 workload (BASELINE.json
configs[1]): a 64-device synthetic trace set of 100M queries per GPU, trace-
fused feature extraction + offload/hedge decision (colo_features_decide).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N>1).  Weak scaling: every rank owns its own
64 devices x 1,562,500 queries; there is no data-path collective, only the
final all-reduce of the decision counters (NCCL).  A step is one pass of the
hot path over the rank's 100M queries (one kernel launch).  Inputs are 1.2 GB
per step (> 126 MB L2), so no L2 flush is needed between steps.

`value` is device-timed (CUDA events on the launching stream, max over ranks);
`e2e` is the same metric through the reference-facing host-buffer C-ABI call
(colo_features_decide_host: pinned host buffers, H2D + kernel + D2H inside the
timed region, host wall clock, max over ranks).  `--impl reference` times the
reference's own code (oracle/_ref: the unchanged colosim headers compiled by
oracle/Makefile) on the host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-I/O admission decisions/sec per GPU (1/2/4/8 B200); % HBM roofline"
UNIT = "decisions/s"
DEVICES, PER_DEVICE = 64, 1_562_500
QPS = [0.05, 0.1, 0.2, 0.3]
BYTES_PER_DECISION = 12  # prompt u32 + output u32 read, verdict u32 written


def dev_set_of(d: int) -> int:
    """llama8b even / phi14b odd devices; CPA for d%4<2 else CPT.
    Map-set order: 0 llama CPA, 1 llama CPT, 2 phi CPA, 3 phi CPT."""
    return (d % 2) * 2 + (0 if d % 4 < 2 else 1)


def config(n_gpus: int) -> dict:
    return {
        "workload": "C2: 64-device synthetic trace set, 100M queries per GPU, trace-fused features + offload/hedge decision",
        "devices_per_gpu": DEVICES,
        "queries_per_gpu": DEVICES * PER_DEVICE,
        "profiles": "llama8b (even devices) / phi14b (odd); CPA for d%4<2 else CPT; default 500/500/5 grid",
        "decision_rule": "cached=charged(prev query of device), incoming=p+o, batch=1, pending=0, dev_layers=L (SURVEY §8(d) C2)",
        "l2": "inputs 1.2 GB/step > 126 MB L2; no flush",
        "parallelism": f"dp{n_gpus} (devices sharded by GPU, no data-path collective)",
    }


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def ncu_traffic() -> float | None:
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    fused kernel from the latest committed `ncu --set full` capture
    (profiles/rNN_ncu_summary.json, written by profiles/extract_ncu.py)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    if not files:
        return None
    with open(files[-1]) as f:
        d = json.load(f)
    return (d.get("k_fused_fast<0>") or d.get("k_fused_fast") or {}).get("dram_bytes_per_launch")


class ClockSampler:
    """Polls SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def report(self) -> dict:
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def init_dist(dist, torch, local):
    """NCCL over NVLink (one rank per GPU).  COLO_DIST_BACKEND=gloo exercises the
    multi-rank plumbing with several ranks sharing one GPU (test only)."""
    backend = os.environ.get("COLO_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("COLO_DIST_BACKEND", "nccl") != "nccl":
        local = 0  # test mode: every rank on GPU 0
    return world, rank, local


def host_trace(seed: int):
    """Host-side synthetic C2 trace for the reference arm (numpy RNG: prompts from
    the ShareGPT-like histogram, output 128 -- workload.hpp:214)."""
    values = np.array([64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096], np.uint32)
    probs = np.array([0.05, 0.10, 0.15, 0.15, 0.13, 0.12, 0.10, 0.08, 0.06, 0.04, 0.02])
    rng = np.random.default_rng(seed)
    n = DEVICES * PER_DEVICE
    prompt = values[rng.choice(len(values), size=n, p=probs)]
    output = np.full(n, 128, np.uint32)
    offs = (np.arange(DEVICES + 1, dtype=np.uint64) * PER_DEVICE).astype(np.uint64)
    return prompt, output, offs


def reference_decide(prompt, output, offs, devices, threads, collect=None):
    """The reference's own composition over its own OffloadingMap/HedgingMap
    (oracle/_ref, ref_features_decide), one device per task, all host threads.
    collect: optional u32 array of every query's verdict (filled per device)."""
    from oracle.oracle import OracleLib, default_gpu, default_grid, default_model, phi14b_model

    ref = OracleLib("ref")
    g = default_gpu()
    sets = [(default_model(), g, 1), (default_model(), g, 0), (phi14b_model(), g, 1), (phi14b_model(), g, 0)]
    grid = default_grid()

    def one(d):
        lo, hi = int(offs[d]), int(offs[d + 1])
        m, gg, cpa = sets[dev_set_of(d)]
        v = ref.features_decide([(m, gg, cpa)], grid, prompt[lo:hi], output[lo:hi], np.array([0, hi - lo], np.uint64),
                                np.zeros(1, np.uint16))
        if collect is not None:
            collect[lo:hi] = v
        return hi - lo

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        n = sum(ex.map(one, devices))
    return n, time.perf_counter() - t0


def run_reference(args, world, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    prompt, output, offs = host_trace(1234)
    sample_devices = list(range(DEVICES))  # the whole C2 workload per step (~0.2-2 s on a multi-core host)
    for _ in range(args.warmup):
        reference_decide(prompt, output, offs, sample_devices, threads)
    tot_n, tot_t = 0, 0.0
    for _ in range(args.steps):
        n, t = reference_decide(prompt, output, offs, sample_devices, threads)
        tot_n += n
        tot_t += t
    value = tot_n / tot_t
    sample = (f"all 64 C2 devices ({DEVICES * PER_DEVICE} queries, both profiles and modes) per step, "
              f"{threads} host threads, oracle/_ref (reference headers compiled unchanged)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config(args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "cpu": cpu_model(),
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_leg(prompt_h, output_h, offs_h, gpu_verdicts=None):
    """The reference on the host cores over the same 100M queries; also holds
    every GPU verdict to the reference's (an untimed second pass collects them)."""
    threads = os.cpu_count() or 1
    devices = list(range(DEVICES))
    reference_decide(prompt_h, output_h, offs_h, devices[:1], threads)  # warm
    n, t = reference_decide(prompt_h, output_h, offs_h, devices, threads)
    n1, t1 = reference_decide(prompt_h, output_h, offs_h, devices[:4], 1)  # the reference is single-threaded
    parity = None
    if gpu_verdicts is not None:
        want = np.empty(len(prompt_h), np.uint32)
        reference_decide(prompt_h, output_h, offs_h, devices, threads, collect=want)
        diff = int(np.count_nonzero(want != gpu_verdicts))
        parity = {"c2_verdicts_equal": diff == 0, "n": int(len(want)), "mismatches": diff,
                  "how": "every GPU verdict of the step vs oracle/_ref (the reference's own map lookups composed as "
                         "engine.hpp:434-448,513-557) on the same 100M queries"}
        if diff:
            print(f"bench: {diff} C2 verdicts differ from the reference", file=sys.stderr)
    return parity, {"value": n / t, "unit": UNIT, "cores": threads, "kind": "reference", "cpu": cpu_model(),
            "single_thread": {"value": n1 / t1, "cores": 1, "sample": f"4 devices ({n1} queries), {t1:.2f} s"},
            "sample": f"the same GPU-generated C2 arrays, all 64 devices ({n} queries), {threads} host threads, "
                      f"oracle/_ref (reference headers compiled unchanged), {t:.2f} s"}


def run_ours(args, world, rank, local):
    import torch

    from paper_2503_01066_b200 import colosim as cs

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        init_dist(dist, torch, local)
    ctx = cs.Context(local)
    stream = torch.cuda.current_stream()
    g = cs.GpuProfile()
    sets = [cs.MapSet.build(ctx, m, g, mode=md) for m in (cs.ModelProfile(), cs.ModelProfile.phi14b_like())
            for md in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]
    arrival, prompt, output, offs = cs.synth_trace(ctx, [PER_DEVICE] * DEVICES,
                                                   [QPS[d % 4] for d in range(DEVICES)], 1234 + 7919 * rank)
    del arrival
    dset = torch.tensor([dev_set_of(d) for d in range(DEVICES)], dtype=torch.int16, device="cuda")
    n = DEVICES * PER_DEVICE
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")

    def step():
        cs.features_decide(ctx, sets, prompt, output, offs, dset, out=out)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        l0 = ctx.launches()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        launches = ctx.launches() - l0
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n * args.steps / (ms_max / 1e3)
    per_launch_s = ms / 1e3 / args.steps
    achieved = BYTES_PER_DECISION * n / per_launch_s / 1e9
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)

    # decision counters once, then the one NCCL stats reduction
    cs.features_decide(ctx, sets, prompt, output, offs, dset, out=out, counters=counters)
    if dist:
        dist.all_reduce(counters)
    cnt = dict(zip(cs.COUNTER_NAMES, [int(x) for x in counters.cpu().tolist()]))

    # e2e: the reference-facing host-buffer call, H2D + kernel + D2H per step
    hp = torch.empty(n, dtype=torch.int32, pin_memory=True)
    ho = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hv = torch.empty(n, dtype=torch.int32, pin_memory=True)
    hp.copy_(prompt)
    ho.copy_(output)
    offs_h = offs.cpu().numpy().astype(np.uint64)
    dset_h = dset.cpu().numpy().astype(np.uint16)
    e2e_steps = max(1, min(args.steps, 10))
    cs.features_decide_host(ctx, sets, hp, ho, offs_h, dset_h, out=hv)  # warm (pipeline buffers)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        cs.features_decide_host(ctx, sets, hp, ho, offs_h, dset_h, out=hv)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * n * e2e_steps / float(te.item())
    assert torch.equal(hv.cuda(), out), "host-buffer path disagrees with the device path"
    # the PCIe bound of that call: pinned copies of the same bytes, each direction alone
    cs_ = torch.cuda.Stream()
    dbuf = torch.empty(2 * n, dtype=torch.int32, device="cuda")
    hin = torch.empty(2 * n, dtype=torch.int32, pin_memory=True)
    pcie = {}
    for name, dst, src in (("h2d", dbuf, hin), ("d2h", hv, dbuf[:n])):
        best = float("inf")
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(cs_):
                e0.record(cs_)
                dst.copy_(src, non_blocking=True)
                e1.record(cs_)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        pcie[name + "_gbs"] = src.numel() * 4 / best / 1e9
    # both directions at once, as the call moves them: the step's transfer floor
    cs2 = torch.cuda.Stream()
    best = float("inf")
    for _ in range(3):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(cs_)
        cs2.wait_event(e0)
        with torch.cuda.stream(cs_):
            dbuf.copy_(hin, non_blocking=True)
            e1.record(cs_)
        with torch.cuda.stream(cs2):
            hv.copy_(out, non_blocking=True)
            e2.record(cs2)
        e1.synchronize()
        e2.synchronize()
        best = min(best, max(e0.elapsed_time(e1), e0.elapsed_time(e2)) / 1e3)
    pcie["duplex_s"] = best
    del dbuf, hin
    pcie_bound = n / best

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config(world),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                             "traffic": ncu_traffic(),
                             "kernel": "k_fused<FAST> (colo_features_decide)",
                             "bytes_per_decision": BYTES_PER_DECISION,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks else "fallback"},
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n * world,
                        "d2h_bytes_per_step": 4 * n * world, "steps": e2e_steps,
                        "api": "colo_features_decide_host (pinned host buffers, wall clock)",
                        "pcie": dict(pcie, bound=pcie_bound * world, frac=e2e_value / (pcie_bound * world),
                                     how="bound = queries / duplex_s, the pinned 8 B/q h2d and 4 B/q d2h copies run concurrently; h2d_gbs/d2h_gbs each alone")},
                "gpu_launches": launches, "clocks": clk.report(), "counters": cnt}
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["parity"], line["cpu_baseline"] = cpu_baseline_leg(
                    hp.numpy().view(np.uint32), ho.numpy().view(np.uint32), offs_h, hv.numpy().view(np.uint32))
            except Exception as e:  # oracle/_ref missing on this box
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
    del out, hp, ho, hv, prompt, output
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if not args.no_sub:
        # stage 3 beside the headline (SURVEY §8(d) C3 and C4's per-rank step), device-timed on this box
        sub = {"c3": c3_measure(args, world, rank, local, dist, args.sub_steps, 3, cpu=True),
               "c4": c4_measure(args, world, rank, local, dist, C4_CHUNK, args.sub_steps, 3, cpu=True)}
        if rank == 0:
            line.update(sub)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


C3_DEVICES, C3_PER_DEVICE = 128, 7_812_500


TUPLE_DTYPE_NP = np.dtype([("cached", "<u4"), ("incoming", "<u4"), ("charged", "<u4"), ("batch", "<u2"),
                           ("pending", "u1"), ("dev_layers", "u1")])


def run_c5(args, world, rank, local):
    """C5 (BASELINE.json configs[4]): grid steps {500,250,100,50} x profiles
    {llama8b, phi14b} x modes {CPT, CPA}; per point the batched quantised map
    verdicts (colo_decide) and the exact per-query verdicts (colo_decide_exact)
    on the same question stream, plus their agreement / over-free rates.
    Per GPU: args.c5_tuples questions (default 1e9 split in 4 chunks)."""
    import torch

    from paper_2503_01066_b200 import colosim as cs

    torch.cuda.set_device(local)
    ctx = cs.Context(local)
    total = args.c5_tuples
    chunk = min(total, 250_000_000)
    g = cs.GpuProfile()
    points = []
    for step in (500, 250, 100, 50):
        for mname, m in (("llama8b", cs.ModelProfile()), ("phi14b", cs.ModelProfile.phi14b_like())):
            for mode in (cs.TrainingMode.CPT, cs.TrainingMode.CPA):
                points.append((step, mname, m, mode))
    va = torch.empty(chunk, dtype=torch.int32, device="cuda")
    vb = torch.empty(chunk, dtype=torch.int32, device="cuda")
    rows = []
    t_map = t_exact = 0.0
    n_done = 0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for step, mname, m, mode in points:
        ms = cs.MapSet.build(ctx, m, g, cs.GridSteps(step, step, 5), cs.GridBounds(), mode)
        counts = torch.zeros(5, dtype=torch.int64, device="cuda")
        tm = te = 0.0
        for c0 in range(0, total, chunk):
            k = min(chunk, total - c0)
            tup_k = cs.synth_tuples(ctx, k, m.num_layers, 1 + 7919 * rank + c0)
            if c0 == 0:  # untimed warm-up of both kernels on this point's map set / profile
                for _ in range(max(args.warmup, 1)):
                    cs.decide(ctx, ms, tup_k, out=va[:k])
                    cs.decide_exact(ctx, m, g, mode, tup_k, out=vb[:k])
            torch.cuda.synchronize()
            ev[0].record()
            cs.decide(ctx, ms, tup_k, out=va[:k])
            ev[1].record()
            cs.decide_exact(ctx, m, g, mode, tup_k, out=vb[:k])
            ev[2].record()
            cs.compare_verdicts(ctx, va[:k], vb[:k], m.num_layers, counts)
            torch.cuda.synchronize()
            tm += ev[0].elapsed_time(ev[1]) / 1e3
            te += ev[1].elapsed_time(ev[2]) / 1e3
        c = [int(x) for x in counts.cpu().tolist()]
        rows.append({"step": step, "profile": mname, "mode": mode.name, "agree": c[0] / c[4], "over_free": c[1] / c[4],
                     "under_free": c[2] / c[4], "same_outcome": c[3] / c[4], "map_decisions_per_s": total / tm,
                     "exact_decisions_per_s": total / te})
        t_map += tm
        t_exact += te
        n_done += total
        ms.close()
    if rank == 0:
        line = {"metric": "C5 sweep: map (per-I/O batched) vs exact per-query decisions/s", "value": n_done / t_map,
                "unit": "decisions/s", "n_gpus": world, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32", "data": "synthetic",
                "config": {"workload": f"C5: 16 sweep points x {total} questions (steps 500/250/100/50 x llama8b/phi14b x CPT/CPA)",
                           "parallelism": f"dp{world}"},
                "exact_value": n_done / t_exact, "points": rows}
        if world == 1 and not args.no_cpu_baseline:
            try:  # the reference's composed lookup and exact decision on 16M of the same questions, all threads
                from oracle.oracle import OracleLib, Grid, default_gpu, default_model

                ref = OracleLib("ref")
                threads = os.cpu_count() or 1
                om = default_model()
                tup = cs.synth_tuples(ctx, 16_000_000, om.num_layers, 1).cpu().numpy().view(TUPLE_DTYPE_NP).reshape(-1)
                parts = np.array_split(tup, threads)
                grid = Grid(500, 500, 5, 8000, 8000, 50)
                t0 = time.perf_counter()
                with ThreadPoolExecutor(threads) as ex:
                    list(ex.map(lambda t: ref.decide(om, default_gpu(), grid, 1, t), parts))
                tmap = time.perf_counter() - t0
                t0 = time.perf_counter()
                with ThreadPoolExecutor(threads) as ex:
                    list(ex.map(lambda t: ref.decide_exact(om, default_gpu(), 1, t), parts))
                tex = time.perf_counter() - t0
                line["cpu_baseline"] = {"value": len(tup) / tmap, "unit": "decisions/s", "cores": threads,
                                        "kind": "reference", "cpu": cpu_model(), "exact_value": len(tup) / tex,
                                        "sample": f"16M of the step-500 llama8b CPA questions, OffloadingMap/HedgingMap "
                                                  f"lookups composed as apply_offload_decision ({tmap:.2f} s) and "
                                                  f"offload_cell_decision + direct hedge ({tex:.2f} s), oracle/_ref, "
                                                  f"{threads} host threads"}
            except Exception as e:
                line["cpu_baseline"] = {"value": None, "unit": "decisions/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    ctx.close()


def run_c1(args, world, rank, local):
    """C1 (BASELINE.json configs[0]): one device trace of 1M queries
    (generate_trace, ShareGPT-like lengths, seed 41) at qps 0.3 and 1.7:
    serving replay + replay-derived verdicts on the GPU, with the reference's
    own Simulation::run (oracle/_ref) timed on the host beside it."""
    import torch

    from paper_2503_01066_b200 import colosim as cs

    torch.cuda.set_device(local)
    ctx = cs.Context(local)
    hv, hp = cs.sharegpt_histogram()
    m, g = cs.ModelProfile(), cs.GpuProfile()
    sets = [cs.MapSet.build(ctx, m, g, mode=cs.TrainingMode.CPA)]
    out = []
    for qps in (0.3, 1.7):
        a, p, o = cs.generate_trace(qps, 1_000_000 / qps, ("histogram", hv, hp), 41, ("fixed", 0.01))
        da, dp, do = torch.from_numpy(a).cuda(), torch.from_numpy(p.view(np.int32)).cuda(), torch.from_numpy(o.view(np.int32)).cuda()
        offs = torch.tensor([0, len(p)], dtype=torch.int64, device="cuda")
        prof = torch.zeros(1, dtype=torch.int16, device="cuda")
        for _ in range(max(args.warmup, 1)):
            r = cs.replay_serving(ctx, [(m, g)], da, dp, do, offs, prof, tau=0.05, sets=sets, batches=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = cs.replay_serving(ctx, [(m, g)], da, dp, do, offs, prof, tau=0.05, sets=sets, batches=True)
        torch.cuda.synchronize()
        gpu_s = (time.perf_counter() - t0) / args.steps
        cpu = None
        try:
            from oracle.oracle import OracleLib, default_gpu, default_model

            ref = OracleLib("ref")
            t0 = time.perf_counter()
            ref.replay_serving(default_model(), default_gpu(), a, p, o, tau=0.05, want_samples=False)
            cpu = time.perf_counter() - t0
        except Exception as e:  # oracle/_ref absent
            cpu = None
        out.append({"qps": qps, "queries": len(p), "gpu_s": gpu_s, "gpu_queries_per_s": len(p) / gpu_s,
                    "reference_cpu_s": cpu, "reference_queries_per_s": (len(p) / cpu) if cpu else None})
    if rank == 0:
        print(json.dumps({"metric": "C1: single-trace serving replay + replay-derived verdicts, queries/s",
                          "value": out[-1]["gpu_queries_per_s"], "unit": "queries/s", "n_gpus": 1,
                          "higher_is_better": True, "dtype": "f64", "data": "synthetic (generate_trace, bit-exact)",
                          "config": {"workload": "C1: 1M queries, one device, ShareGPT-like lengths, seed 41"},
                          "cpu_baseline": {"kind": "reference", "cores": 1, "sample": "Simulation::run ServingOnly, same trace"},
                          "runs": out}), flush=True)
    ctx.close()


def reference_colocated(dev_traces, threads):
    """The reference's own Simulation::run (SimMode::Colocated) through
    oracle/_ref, one device per task on all host threads.  dev_traces: list of
    (model, gpu, cpa, arrival, prompt, output)."""
    from oracle.oracle import OracleLib, default_grid

    ref = OracleLib("ref")
    grid = default_grid()

    def one(t):
        m, g, cpa, a, p, o = t
        ref.replay_colocated(m, g, grid, cpa, a, p, o, np.full(len(a), 0.01), 60.0, want_samples=False,
                             want_batches=False)
        return len(a)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        n = sum(ex.map(one, dev_traces))
    return n, time.perf_counter() - t0


def reference_serving(dev_traces, threads, with_stats=False):
    """The reference's own Simulation::run (SimMode::ServingOnly) through
    oracle/_ref, one device per task on all host threads; with_stats also
    keeps the TPT samples and runs finalize (sort, nearest ranks, mean) as
    run_simulation does.  dev_traces: list of (model, gpu, arrival, prompt,
    output)."""
    from oracle.oracle import OracleLib, default_grid

    ref = OracleLib("ref")
    grid = default_grid()

    def one(t):
        m, g, a, p, o = t
        ref.replay_colocated(m, g, grid, 1, a, p, o, np.full(len(a), 0.01), 60.0, tau=0.05,
                             want_samples=with_stats, want_batches=False, sim_mode="serving-only")
        return len(a)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        n = sum(ex.map(one, dev_traces))
    return n, time.perf_counter() - t0


def reference_sample(arrival, prompt, output, offs, devs, per, models):
    """Host copies of the first `per` queries of the first `devs` devices."""
    from oracle.oracle import default_gpu

    offs_h = offs.cpu().numpy()
    out = []
    for d in range(min(devs, len(offs_h) - 1)):
        lo = int(offs_h[d])
        hi = min(int(offs_h[d + 1]), lo + per)
        out.append((models[d % len(models)], default_gpu(), arrival[lo:hi].cpu().numpy(),
                    prompt[lo:hi].cpu().numpy().view(np.uint32), output[lo:hi].cpu().numpy().view(np.uint32)))
    return out


def run_colo(args, world, rank, local):
    """Colocated replay (the full admission loop).
    (1) C1 (BASELINE.json configs[0]): the 1M-query single-device trace at
        qps 0.3 and 1.7 (generate_trace, ShareGPT-like lengths, label delay
        0.01 s, seed 41), CPA: one warp on the GPU vs the reference's own
        Simulation::run (oracle/_ref, one host core).
    (2) Fleet: --colo-devices devices x --colo-per-device queries per GPU
        (synth_trace, qps 0.05/0.1/0.2/0.3, llama8b/phi14b x CPA/CPT as C2),
        device-timed replay (samples reduced to exact sums / slow counts); the reference on a bounded
        device sample across all host threads."""
    import torch

    from oracle.oracle import default_gpu, default_model, phi14b_model
    from paper_2503_01066_b200 import colosim as cs

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        init_dist(dist, torch, local)
    ctx = cs.Context(local)
    hv, hp = cs.sharegpt_histogram()
    g = cs.GpuProfile()
    models = (cs.ModelProfile(), cs.ModelProfile.phi14b_like())
    sets = [cs.MapSet.build(ctx, m, g, mode=md) for m in models for md in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]
    threads = os.cpu_count() or 1
    c1 = []
    if rank == 0 and not args.colo_skip_c1:
        for qps in (0.3, 1.7):
            a, p, o = cs.generate_trace(qps, 1_000_000 / qps, ("histogram", hv, hp), 41, ("fixed", 0.01))
            da, dp, do = (torch.from_numpy(a).cuda(), torch.from_numpy(p.view(np.int32)).cuda(),
                          torch.from_numpy(o.view(np.int32)).cuda())
            offs = torch.tensor([0, len(p)], dtype=torch.int64, device="cuda")
            dset = torch.zeros(1, dtype=torch.int16, device="cuda")
            r = cs.replay_colocated(ctx, sets[:1], da, dp, do, offs, dset, tau=0.05)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = cs.replay_colocated(ctx, sets[:1], da, dp, do, offs, dset, tau=0.05)
            torch.cuda.synchronize()
            gpu_s = time.perf_counter() - t0
            S = cs.colocated_summaries(r["summary"])[0]
            cpu_s = None
            if not args.no_cpu_baseline:
                try:
                    _, cpu_s = reference_colocated([(default_model(), default_gpu(), 1, a, p, o)], 1)
                except Exception:
                    cpu_s = None
            c1.append({"qps": qps, "queries": len(p), "gpu_s": gpu_s, "gpu_queries_per_s": len(p) / gpu_s,
                       "reference_cpu_s": cpu_s, "reference_queries_per_s": len(p) / cpu_s if cpu_s else None,
                       "completed_jobs": S["completed_jobs"], "recomputes": S["recomputes"],
                       "preemptions": S["preemptions"], "batches": S["batches"]})
    D, per = args.colo_devices, args.colo_per_device
    arrival, prompt, output, offs = cs.synth_trace(ctx, [per] * D, [QPS[d % 4] for d in range(D)],
                                                   777 + 7919 * rank)
    dset = torch.tensor([dev_set_of(d) for d in range(D)], dtype=torch.int16, device="cuda")
    n = D * per

    def step():
        return cs.replay_colocated(ctx, sets, arrival, prompt, output, offs, dset, tau=0.05, labels=False)

    for _ in range(max(args.warmup, 1)):
        r = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        l0 = ctx.launches()
        ev0.record()
        for _ in range(args.steps):
            r = step()
        ev1.record()
        launches = ctx.launches() - l0
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    S = cs.colocated_summaries(r["summary"])
    keys = ("generated_tokens", "trained_tokens", "completed_jobs", "recomputes", "preemptions", "loads",
            "layers_freed", "labels_dropped", "map_fallbacks", "batches", "offload_decisions", "admissions")
    tot = torch.tensor([sum(s[k] for s in S) for k in keys], dtype=torch.int64, device="cuda")
    if dist:
        dist.all_reduce(tot)
    sec = float(t.item()) / 1e3
    value = world * n * args.steps / sec
    if rank == 0:
        line = {"metric": "colocated replay queries/s (full admission loop, Simulation::run Colocated)",
                "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"colocated fleet: {D} devices x {per} queries per GPU (qps 0.05/0.1/0.2/0.3, "
                                       "llama8b/phi14b x CPA/CPT as C2, label delay 0.01 s, timeout 60 s)",
                           "parallelism": f"dp{world} (one warp per device)"},
                "totals": dict(zip(keys, [int(x) for x in tot.cpu().tolist()])),
                "roofline": {"bound": "latency (sequential per-device event loop)", "achieved": None,
                             "peak": None, "unit": "GB/s", "frac": None, "traffic": None},
                "gpu_launches": launches, "clocks": clk.report(), "c1": c1}
        if world == 1 and not args.no_cpu_baseline:
            try:
                k = min(D, max(threads, 8))
                offs_h = offs.cpu().numpy()
                a_h, p_h, o_h = arrival.cpu().numpy(), prompt.cpu().numpy().view(np.uint32), output.cpu().numpy().view(np.uint32)
                mods = [(default_model(), 1), (default_model(), 0), (phi14b_model(), 1), (phi14b_model(), 0)]
                tr = []
                for d in range(k):
                    lo, hi = int(offs_h[d]), int(offs_h[d + 1])
                    mm, cpa = mods[dev_set_of(d)]
                    tr.append((mm, default_gpu(), cpa, a_h[lo:hi], p_h[lo:hi], o_h[lo:hi]))
                nq, ts = reference_colocated(tr, threads)
                line["cpu_baseline"] = {"value": nq / ts, "unit": "queries/s", "cores": threads, "kind": "reference",
                                        "cpu": cpu_model(),
                                        "sample": f"{k} of the fleet's devices ({nq} queries), Simulation::run "
                                                  f"Colocated via oracle/_ref, {threads} host threads, {ts:.1f} s"}
            except Exception as e:
                line["cpu_baseline"] = {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


C4_FLEET, C4_PER_DEVICE = 1024, 7_812_500
C4_SEED = 4040
C4_CHUNK = 128  # devices per chunk context (1B queries): one rank's 8-GPU share


def profile_one_step(torch, step):
    """COLO_PROFILE_STEP=1: one extra, untimed step between cudaProfilerStart /
    Stop, so `ncu --profile-from-start off` sees exactly one step's kernels
    (profiles/step_inst.py turns that capture into the issue-rate roofline)."""
    if os.environ.get("COLO_PROFILE_STEP"):
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()


def issue_roofline(kind: str, step_s: float, clk: dict, queries: int) -> dict:
    """Issue-rate roofline of a replay step: the warp instructions one step
    executes (smsp__inst_executed.sum summed over the step's kernels, from the
    committed ncu capture profiles/r*_ncu_<kind>_step.json -- the count is a
    property of the workload, not of the clock) over the live step time,
    against 148 SMs x 4 schedulers x 1 warp-instruction/clk at the live SM
    clock."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_{kind}_step.json")))
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    peak = 148 * 4 * mhz * 1e6
    out = {"bound": "issue", "unit": "warp-inst/s", "peak": peak,
           "peak_how": f"148 SMs x 4 schedulers x {mhz:.0f} MHz (live median SM clock)"}
    if not files:
        return dict(out, achieved=None, frac=None, inst_per_step=None, source="no ncu capture committed")
    with open(files[-1]) as f:
        d = json.load(f)
    # instructions scale with the rank's queries (the capture's workload per query, the same traces' shape)
    inst = float(d["inst_per_query"]) * queries if d.get("inst_per_query") else float(d["inst_per_step"])
    ach = inst / step_s
    return dict(out, achieved=ach, frac=ach / peak, inst_per_step=inst, inst_per_query=d.get("inst_per_query"),
                source=os.path.relpath(files[-1], ROOT))


def c4_measure(args, world, rank, local, dist, devices_cap, steps, warmup, cpu=False):
    """C4 (BASELINE.json configs[3]): the 1024-device fleet, fleet device g on
    rank g % world.  Device g's trace is keyed on g (synth_trace dev_ids), so it
    is the same at every world size.  The rank's devices are held in chunks of
    C4_CHUNK devices, each with its own Context (segment entry states and sparse
    records survive between the exact-stats passes; the first pass's transient
    buffers are shared).  One step = the trace-fused decisions over all the
    rank's queries + the serving replay with slow labels + the exact TPT stats
    (three radix-select passes; counters, histograms and exact sums all-reduced
    over NCCL).  Returns the record (every rank) with the max-over-ranks time."""
    import torch

    from paper_2503_01066_b200 import colosim as cs

    mine = [d for d in range(C4_FLEET) if d % world == rank]
    if devices_cap:
        mine = mine[:devices_cap]
    per = args.c4_per_device
    g = cs.GpuProfile()
    models = (cs.ModelProfile(), cs.ModelProfile.phi14b_like())
    owner = cs.Context(local)
    sets = [cs.MapSet.build(owner, m, g, mode=md) for m in models for md in (cs.TrainingMode.CPA, cs.TrainingMode.CPT)]
    profiles = [(m, g) for m in models]
    parts, fparts = [], []
    for c0 in range(0, len(mine), C4_CHUNK):
        ch = mine[c0:c0 + C4_CHUNK]
        cx = owner if c0 == 0 else cs.Context(local)
        if cx is not owner:
            cx.share_temps(owner)
        arrival, prompt, output, offs = cs.synth_trace(cx, [per] * len(ch), [QPS[d % 4] for d in ch], C4_SEED,
                                                       dev_ids=ch)
        dset = torch.tensor([dev_set_of(d) for d in ch], dtype=torch.int16, device="cuda")
        dprof = torch.tensor([d % 2 for d in ch], dtype=torch.int16, device="cuda")
        parts.append((cx, arrival, prompt, output, offs, dprof))
        fparts.append((cx, prompt, output, offs, dset))
    nmax = max(p[1].shape[0] for p in fparts)
    n = sum(p[1].shape[0] for p in fparts)
    out = torch.empty(nmax, dtype=torch.int32, device="cuda")
    counters = torch.zeros(8, dtype=torch.int64, device="cuda")

    def step():
        counters.zero_()
        for cx, prompt, output, offs, dset in fparts:
            cs.features_decide(cx, sets, prompt, output, offs, dset, out=out[:prompt.shape[0]], counters=counters)
        st = cs.fleet_stats(parts, profiles, tau=args.c4_tau)
        if dist:
            dist.all_reduce(counters)
        return st

    for _ in range(max(warmup, 3) if steps else 0):
        st = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    profile_one_step(torch, step)
    with ClockSampler(local) as clk:
        l0 = sum(p[0].launches() for p in parts)
        ev0.record()
        for _ in range(steps):
            st = step()
        ev1.record()
        torch.cuda.synchronize()
        launches = sum(p[0].launches() for p in parts) - l0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    nt = torch.tensor([n], dtype=torch.int64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(nt)
    sec = float(t.item()) / 1e3
    total = int(nt.item())
    clocks = clk.report()
    rec = {"metric": "C4 fleet: admission decisions + serving replay labels + exact TPT stats, queries/s",
           "value": total * steps / sec, "unit": "queries/s", "n_gpus": world, "steps": steps, "warmup": max(warmup, 3),
           "ms_per_step": float(t.item()) / steps, "higher_is_better": True, "scaling": "weak",
           "per_rank_queries_per_s": n * steps / sec, "dtype": "u32+f64", "data": "synthetic",
           "config": {"workload": f"C4: 1024-device fleet x {per} queries, fleet device g on rank g % {world}; "
                                  f"{len(mine)} devices ({n} queries) per rank this run, "
                                  f"{len(parts)} chunk(s) of <= {C4_CHUNK} devices",
                      "devices_per_rank": len(mine), "queries_per_rank": n, "queries_total": total,
                      "per_step": "features_decide (all queries) + serving replay with slow labels + "
                                  "3 radix-select stats passes, NCCL all-reduce of counters/histograms/exact sums",
                      "tau_s": args.c4_tau, "trace_seed": f"{C4_SEED}, keyed on the fleet device id",
                      "l2": "inputs 16 GB/step per chunk > L2", "parallelism": f"dp{world} (devices sharded by rank)"},
           "stats": {k: st[k] for k in ("generated_tokens", "slow_tokens", "slow_queries", "batches", "p50", "p90",
                                        "p99", "mean", "mean_exact")},
           "counters": dict(zip(cs.COUNTER_NAMES, [int(x) for x in counters.cpu().tolist()])),
           "roofline": issue_roofline("c4", sec / steps, clocks, n),
           "gpu_launches": launches, "clocks": clocks}
    if cpu and world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import default_model, phi14b_model

            threads = os.cpu_count() or 1
            cx, arrival, prompt, output, offs, _ = parts[0]
            tr = reference_sample(arrival, prompt, output, offs, 16, 100_000, [default_model(), phi14b_model()])
            nq, ts = reference_serving(tr, threads, with_stats=True)
            rec["cpu_baseline"] = {"value": nq / ts, "unit": "queries/s", "cores": threads, "kind": "reference",
                                   "cpu": cpu_model(),
                                   "sample": f"first 100k queries of 16 of the rank's devices ({nq} queries), "
                                             f"Simulation::run ServingOnly + finalize via oracle/_ref, "
                                             f"{threads} host threads, {ts:.1f} s (the decision lookups "
                                             "are not included)"}
        except Exception as e:
            rec["cpu_baseline"] = {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    del parts, fparts, out
    for s_ in sets:
        s_.close()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


def run_c4(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        init_dist(dist, torch, local)
    cap = args.c4_devices if args.c4_devices is not None else (None if world > 1 else C4_CHUNK)
    rec = c4_measure(args, world, rank, local, dist, cap, args.steps, args.warmup, cpu=True)
    if rank == 0:
        print(json.dumps(rec), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def c3_measure(args, world, rank, local, dist, steps, warmup, cpu=False):
    """C3 (BASELINE.json configs[2]): 128 bursty devices x 7,812,500 queries =
    1B queries per GPU (qps 0.1 / 3.0 alternating every 600 s).  One step =
    serving replay + slow labels + the first exact-stats histogram pass + the
    replay-derived verdict of every batch (CPT/CPA alternate
    by device with the profile -- llama8b/CPA even, phi14b/CPT odd).  tau =
    serving-only p99 of device 0's first 1M queries."""
    import torch

    from paper_2503_01066_b200 import colosim as cs

    ctx = cs.Context(local)
    D, per = args.c3_devices, args.c3_per_device
    g = cs.GpuProfile()
    profiles = [(cs.ModelProfile(), g), (cs.ModelProfile.phi14b_like(), g)]
    sets = [cs.MapSet.build(ctx, profiles[0][0], g, mode=cs.TrainingMode.CPA),
            cs.MapSet.build(ctx, profiles[1][0], g, mode=cs.TrainingMode.CPT)]
    arrival, prompt, output, offs = cs.synth_trace(ctx, [per] * D, [0.1] * D, 4242 + 7919 * rank,
                                                   dev_qps_hi=[3.0] * D, burst_period=600.0)
    dprof = torch.tensor([d % 2 for d in range(D)], dtype=torch.int16, device="cuda")
    m1 = min(per, 1_000_000)
    tau_stats = cs.serving_stats(ctx, profiles, arrival[:m1], prompt[:m1], output[:m1],
                                 torch.tensor([0, m1], dtype=torch.int64, device="cuda"), dprof[:1])
    tau = tau_stats["p99"]
    hist = torch.zeros(cs.HIST_BINS, dtype=torch.int64, device="cuda")
    n = D * per
    verdicts = torch.empty(n, dtype=torch.int32, device="cuda")

    def step():
        hist.zero_()
        return cs.replay_serving(ctx, profiles, arrival, prompt, output, offs, dprof, tau=tau, labels=True,
                                 summary=True, hist=hist, sets=sets, verdicts=verdicts)

    for _ in range(max(warmup, 3)):
        r = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    profile_one_step(torch, step)
    with ClockSampler(local) as clk:
        l0 = ctx.launches()
        ev0.record()
        for _ in range(steps):
            r = step()
        ev1.record()
        torch.cuda.synchronize()
        launches = ctx.launches() - l0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    S = cs.summaries_to_numpy(r["summary"])
    # verdict outcome counts over every batch (COLO_V_OUTCOME: bits 21-22)
    nb_dev = torch.from_numpy(S["batches"].astype(np.int64)).cuda()
    offs_l = offs[:-1]
    idx = torch.arange(n, device="cuda", dtype=torch.int64)
    dev_of = torch.searchsorted(offs[1:], idx, right=True)
    valid = (idx - offs_l[dev_of]) < nb_dev[dev_of]
    outcome = ((verdicts.to(torch.int64) >> 21) & 3)[valid]
    vc = torch.bincount(outcome, minlength=3)[:3]
    del idx, dev_of, valid, outcome
    tot = torch.tensor([int(S["generated_tokens"].sum()), int(S["slow_tokens"].sum()), int(S["slow_queries"].sum()),
                        int(S["batches"].sum())] + [int(x) for x in vc.tolist()], dtype=torch.int64, device="cuda")
    if dist:
        dist.all_reduce(tot)
        dist.all_reduce(hist)
    sec = float(t.item()) / 1e3
    gen, slow_tok, slow_q, nb, v_admit, v_free, v_recomp = [int(x) for x in tot.cpu().tolist()]
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    clocks = clk.report()
    hbm = 17 * n / (sec / steps) / 1e9  # 16 B/query read + 1 B label written
    rec = {"metric": "C3: bursty serving replay + slow labels + replay-derived verdicts, queries/s",
           "value": world * n * steps / sec, "unit": "queries/s", "n_gpus": world, "steps": steps,
           "warmup": max(warmup, 3), "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
           "decisions_per_s": nb * steps / sec, "tokens_per_s": gen * steps / sec,
           "config": {"workload": f"C3: {D} bursty devices x {per} queries per GPU (qps 0.1/3.0 alternating "
                                  "every 600 s), serving-only replay + slow labels + exact-stats pass 1 + one verdict "
                                  "per batch (llama8b/CPA even devices, phi14b/CPT odd)",
                      "tau_s": tau, "tau_rule": "serving-only p99 of device 0's first 1M queries",
                      "decision_rule": "cached = charged tokens of the device's last single-query batch, incoming = "
                                       "max_incoming, batch = n, pending 0, dev_layers L (SURVEY §8(d) C3)",
                      "l2": "inputs 16 GB/step > L2", "parallelism": f"dp{world}"},
           "labels": {"tokens": gen, "slow_tokens": slow_tok, "slow_queries": slow_q, "batches": nb},
           "verdicts": {"admit": v_admit, "free_loadback": v_free, "recompute_drop": v_recomp},
           "roofline": issue_roofline("c3", sec / steps, clocks, n),
           "hbm": {"achieved": hbm, "peak": peak, "unit": "GB/s", "frac": hbm / peak,
                   "note": "17 B/query algorithmic; the replay is bound by dependent f64 time chains, not HBM"},
           "gpu_launches": launches, "clocks": clocks}
    if cpu and world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import default_model, phi14b_model

            threads = os.cpu_count() or 1
            tr = reference_sample(arrival, prompt, output, offs, 16, 250_000, [default_model(), phi14b_model()])
            nq, ts = reference_serving(tr, threads)
            rec["cpu_baseline"] = {"value": nq / ts, "unit": "queries/s", "cores": threads, "kind": "reference",
                                   "cpu": cpu_model(),
                                   "sample": f"first 250k queries of 16 of the C3 devices ({nq} queries), "
                                             f"Simulation::run ServingOnly via oracle/_ref, {threads} host "
                                             f"threads, {ts:.1f} s"}
        except Exception as e:
            rec["cpu_baseline"] = {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    del r, arrival, prompt, output, verdicts
    for s_ in sets:
        s_.close()
    ctx.release_scratch()
    ctx.close()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


def run_c3(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        init_dist(dist, torch, local)
    rec = c3_measure(args, world, rank, local, dist, args.steps, args.warmup, cpu=True)
    if rank == 0:
        print(json.dumps(rec), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c1", "c2", "c3", "c4", "c5", "colo"], default="c2",
                    help="c2 (default, the headline): trace-fused decisions; c1: single-trace replay vs the "
                         "reference Simulation; c3: 1B-query bursty replay + labels; c5: map vs exact sweep; "
                         "c4: 1024-device fleet sharded by rank (decisions + replay + exact stats, NCCL reduce); "
                         "colo: colocated replay (C1 trace + device fleet)")
    ap.add_argument("--c4-devices", type=int, default=None,
                    help="cap on devices per rank (default: all of the rank's 1024/world at world >= 2, "
                         "the 8-GPU share of 128 at world 1)")
    ap.add_argument("--sub-steps", type=int, default=3, help="timed steps of the C3/C4 sub-records of the headline")
    ap.add_argument("--no-sub", action="store_true", help="headline line without the C3/C4 sub-records")
    ap.add_argument("--c4-per-device", type=int, default=C4_PER_DEVICE)
    ap.add_argument("--c4-tau", type=float, default=0.05)
    ap.add_argument("--colo-devices", type=int, default=1184)  # 8 resident warps x 148 SMs
    ap.add_argument("--colo-per-device", type=int, default=50_000)
    ap.add_argument("--colo-skip-c1", action="store_true")
    ap.add_argument("--c3-devices", type=int, default=C3_DEVICES)
    ap.add_argument("--c3-per-device", type=int, default=C3_PER_DEVICE)
    ap.add_argument("--c5-tuples", type=int, default=1_000_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.workload == "c1":
        run_c1(args, world, rank, local)
    elif args.workload == "c3":
        run_c3(args, world, rank, local)
    elif args.workload == "c5":
        run_c5(args, world, rank, local)
    elif args.workload == "colo":
        run_colo(args, world, rank, local)
    elif args.workload == "c4":
        run_c4(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
