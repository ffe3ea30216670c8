"""The reference's experiment harness on the colo-b200 engine: configuration
files, paired colocated/baseline runs, the memory-wall search and the figure
datasets -- include/colosim/experiment.hpp, include/colosim/kvfile.hpp,
include/colosim/metrics.hpp:101-289 and tools/colosim.cpp (run / compare /
plotdata), paths relative to /root/reference/proj/.

Every simulation here is Simulation::run on the GPU (colo_replay_colocated:
one warp per run, all of a stage's runs in one fleet launch); the host only
formats, exactly as the reference writes them, so the output files are
byte-identical to the reference CLI's (pinned by tests/test_gpu_experiment.py
against tests/golden/cli/, written by the reference's own driver).
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from . import colosim as cs
from ._lib import ColoValidationError, lib

KGIB = 1024**3


# ------------------------------------------------------------------ config
class KvFile:
    """kvfile.hpp:15-136: `key = value` lines, `#` comments, dotted sections."""

    def __init__(self, values: Dict[str, str], origin: str):
        self.values, self.origin, self.consumed = values, origin, set()

    @staticmethod
    def parse_text(text: str, origin: str = "<string>") -> "KvFile":
        vals = {}
        for lineno, line in enumerate(text.split("\n"), 1):
            s = line.strip(" \t\r\n")
            if not s or s[0] == "#":
                continue
            if "=" not in s:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"{origin}:{lineno}: expected `key = value`, got: {s}")
            k, v = s.split("=", 1)
            k, v = k.strip(" \t\r\n"), v.strip(" \t\r\n")
            if not k:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"{origin}:{lineno}: empty key")
            if k in vals:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"{origin}:{lineno}: duplicate key: {k}")
            vals[k] = v
        return KvFile(vals, origin)

    @staticmethod
    def parse_file(path: str) -> "KvFile":
        try:
            text = open(path).read()
        except OSError:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"cannot open config file: {path}")
        return KvFile.parse_text(text, path)

    def has(self, k):
        return k in self.values

    def get_string(self, k):
        if k not in self.values:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"{self.origin}: missing required key: {k}")
        self.consumed.add(k)
        return self.values[k]

    def get_string_or(self, k, d):
        return self.get_string(k) if self.has(k) else d

    def get_u64(self, k):
        v = self.get_string(k)
        try:
            if any(c in v for c in "eE."):
                d = float(v)
                if d < 0:
                    raise ValueError(v)
                return int(d)
            u = int(v, 10)
            if u < 0:
                raise ValueError(v)
            return u
        except ValueError:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"{self.origin}: key {k}: not an unsigned integer: {v}")

    def get_u64_or(self, k, d):
        return self.get_u64(k) if self.has(k) else d

    def get_f64(self, k):
        v = self.get_string(k)
        try:
            return float(v)
        except ValueError:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"{self.origin}: key {k}: not a number: {v}")

    def get_f64_or(self, k, d):
        return self.get_f64(k) if self.has(k) else d

    def section(self, prefix: str) -> "KvFile":
        sub = {}
        for k, v in self.values.items():
            if k.startswith(prefix + "."):
                sub[k[len(prefix) + 1:]] = v
                self.consumed.add(k)
        return KvFile(sub, f"{self.origin} [{prefix}.*]")

    def reject_unknown(self):
        for k in sorted(self.values):
            if k not in self.consumed:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"{self.origin}: unknown key: {k}")


def parse_distribution(s: str):
    """experiment.hpp:19-33: fixed:<v> | uniform:<lo>,<hi> | histogram:<path> | none."""
    if s == "none":
        return None
    kind, _, rest = s.partition(":")
    if kind == "fixed":
        return ("fixed", float(rest))
    if kind == "uniform":
        if "," not in rest:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"distribution: uniform needs lo,hi: {s}")
        lo, hi = rest.split(",", 1)
        return ("uniform", float(lo), float(hi))
    if kind == "histogram":
        v, p = cs.load_histogram(rest)
        return ("histogram", v, p)
    raise ColoValidationError(_lib.COLO_EVALIDATION, f"unknown distribution spec: {s}")


def _model_from_kv(kv: KvFile) -> cs.ModelProfile:
    """profiles.hpp:59-75."""
    m = cs.ModelProfile(
        kv.get_u64("num_layers"), kv.get_u64("kv_bytes_per_token"), kv.get_u64("act_bytes_per_token_per_layer"),
        kv.get_f64("prefill_coef_linear"), kv.get_f64("prefill_coef_quad"), kv.get_f64("decode_coef_const"),
        kv.get_f64("decode_coef_context"), kv.get_f64("backward_to_forward_ratio"),
        kv.get_f64("record_prefill_multiplier"), kv.get_f64("record_decode_multiplier"),
        kv.get_f64("workspace_factor"), kv.get_u64("weights_bytes"))
    return m


def _gpu_from_kv(kv: KvFile) -> cs.GpuProfile:
    """profiles.hpp:110-118."""
    return cs.GpuProfile(kv.get_u64("capacity_bytes"), kv.get_u64("h2d_bandwidth"), kv.get_u64("d2h_bandwidth"),
                         kv.get_u64("runtime_reserve_bytes"))


@dataclass
class Trace:
    """workload.hpp:122-162 as SoA (label_delay < 0 or NaN = nullopt)."""

    arrival: np.ndarray
    prompt: np.ndarray
    output: np.ndarray
    label_delay: np.ndarray
    query_id: np.ndarray

    def __len__(self):
        return len(self.arrival)

    def content_hash(self) -> int:
        a = np.ascontiguousarray(self.arrival, np.float64)
        p = np.ascontiguousarray(self.prompt, np.uint32)
        o = np.ascontiguousarray(self.output, np.uint32)
        ld = np.ascontiguousarray(self.label_delay, np.float64)
        q = np.ascontiguousarray(self.query_id, np.uint64)
        return int(lib().colo_trace_hash(q.ctypes.data, a.ctypes.data, p.ctypes.data, o.ctypes.data, ld.ctypes.data,
                                         len(a)))


@dataclass
class TraceSpec:
    """experiment.hpp:35-51."""

    file: Optional[str] = None
    qps: float = 1.0
    duration: float = 100.0
    seed: int = 7
    length_dist: tuple = ("fixed", 1000.0)
    min_tokens: Optional[int] = None
    label_delay: Optional[tuple] = ("fixed", 0.01)

    def realize(self) -> Trace:
        if self.file:
            a, p, o, q, ld = cs.load_trace(self.file)
            return Trace(a, p, o, np.where(np.isnan(ld), -1.0, ld), q)
        a, p, o, ld = cs.generate_trace(self.qps, self.duration, self.length_dist, self.seed, self.label_delay,
                                        min_tokens=self.min_tokens or 0, with_labels=True)
        return Trace(a, p, o, ld, np.arange(len(a), dtype=np.uint64))


@dataclass
class ExperimentConfig:
    """experiment.hpp:53-120 (ExperimentConfig::from_file)."""

    mode: cs.SimMode = cs.SimMode.COLOCATED
    training: cs.TrainingMode = cs.TrainingMode.CPA
    model: cs.ModelProfile = field(default_factory=cs.ModelProfile)
    gpu: cs.GpuProfile = field(default_factory=cs.GpuProfile)
    cache_timeout: float = 60.0
    seed: int = 7
    trace_spec: TraceSpec = field(default_factory=TraceSpec)
    map_steps: cs.GridSteps = field(default_factory=cs.GridSteps)
    map_bounds: cs.GridBounds = field(default_factory=cs.GridBounds)
    sweep_qps: List[float] = field(default_factory=list)
    sweep_token_lengths: List[int] = field(default_factory=list)
    sweep_min_tokens: Optional[int] = None
    sweep_modes: List[cs.TrainingMode] = field(default_factory=list)

    @staticmethod
    def from_file(path: str) -> "ExperimentConfig":
        kv = KvFile.parse_file(path)
        ec = ExperimentConfig()
        mk = kv.section("model")
        ec.model = _model_from_kv(mk)
        mk.reject_unknown()
        gk = kv.section("gpu")
        ec.gpu = _gpu_from_kv(gk)
        gk.reject_unknown()
        sim = kv.section("sim")
        ec.mode = cs.SimMode.parse(sim.get_string_or("mode", "colocated"))
        ec.training = training_mode_from_string(sim.get_string_or("training", "cpa"))
        ec.cache_timeout = sim.get_f64_or("cache_timeout", 60.0)
        ec.seed = sim.get_u64_or("seed", 7)
        sim.reject_unknown()
        tr = kv.section("trace")
        ts = TraceSpec()
        if tr.has("file"):
            ts.file = tr.get_string("file")
        ts.qps = tr.get_f64_or("qps", 1.0)
        ts.duration = tr.get_f64_or("duration", 100.0)
        ts.seed = tr.get_u64_or("seed", ec.seed)
        if tr.has("length_dist"):
            d = parse_distribution(tr.get_string("length_dist"))
            if d is None:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"{path}: trace.length_dist cannot be none")
            ts.length_dist = d
        if tr.has("min_tokens"):
            ts.min_tokens = tr.get_u64("min_tokens")
        if tr.has("label_delay"):
            ts.label_delay = parse_distribution(tr.get_string("label_delay"))
        tr.reject_unknown()
        ec.trace_spec = ts
        mp = kv.section("map")
        ec.map_steps = cs.GridSteps(mp.get_u64_or("cached_step", 500), mp.get_u64_or("incoming_step", 500),
                                    mp.get_u64_or("batch_step", 5))
        ec.map_bounds = cs.GridBounds(mp.get_u64_or("max_cached", 8000), mp.get_u64_or("max_incoming", 8000),
                                      mp.get_u64_or("max_batch", 50))
        mp.reject_unknown()
        sw = kv.section("sweep")
        split = lambda s: [t for t in s.split(",") if t]
        if sw.has("qps"):
            ec.sweep_qps = [float(t) for t in split(sw.get_string("qps"))]
        if sw.has("token_lengths"):
            ec.sweep_token_lengths = [int(t) for t in split(sw.get_string("token_lengths"))]
        if sw.has("min_tokens"):
            ec.sweep_min_tokens = sw.get_u64("min_tokens")
        if sw.has("modes"):
            ec.sweep_modes = [training_mode_from_string(t) for t in split(sw.get_string("modes"))]
        sw.reject_unknown()
        kv.reject_unknown()
        return ec


def training_mode_from_string(s: str) -> cs.TrainingMode:
    """maps.hpp:20-24."""
    if s == "cpt":
        return cs.TrainingMode.CPT
    if s == "cpa":
        return cs.TrainingMode.CPA
    raise ColoValidationError(_lib.COLO_EVALIDATION, f"unknown training mode: {s} (expected cpt or cpa)")


def _tm_str(t) -> str:
    return "cpt" if int(t) == int(cs.TrainingMode.CPT) else "cpa"


def _sm_str(m) -> str:  # engine.hpp:25-32
    return {cs.SimMode.COLOCATED: "colocated", cs.SimMode.SEPARATE_CLUSTER: "baseline",
            cs.SimMode.SERVING_ONLY: "serving-only"}[cs.SimMode(int(m))]


# ---------------------------------------------------------------- engine
@dataclass
class Run:
    """One Simulation (make_sim_config, experiment.hpp:154-168)."""

    model: cs.ModelProfile
    gpu: cs.GpuProfile
    mode: cs.SimMode
    training: cs.TrainingMode
    maps: cs.MapSet
    trace: Trace
    cache_timeout: float = 60.0


def finalize_report(r: dict) -> dict:
    """metrics.hpp:56-69 on a report whose samples were finalized on the device:
    r['_finalized'] = [p50, p90, p99, mean] from colo_finalize (nearest ranks of
    the ascending sort and the strictly sequential sum of the sorted samples,
    bit-exact).  There is no host path: a report with samples and no device
    result is an error."""
    x = r["tpt_samples"]
    for k in ("tpt_p50", "tpt_p90", "tpt_p99", "tpt_mean"):
        r[k] = None
    fin = r.pop("_finalized", None)
    if len(x):
        if fin is None:
            raise cs.ColoError(_lib.COLO_EINVAL, "finalize_report: samples were not finalized on the device")
        r["tpt_p50"], r["tpt_p90"], r["tpt_p99"], r["tpt_mean"] = fin
    r["training_throughput"] = (float(r["trained_tokens"]) / r["training_busy_time"]
                                if r["training_busy_time"] > 0 else None)
    return r


def _runs_with_own_maps(ctx: cs.Context, runs: Sequence[Run]) -> List[Run]:
    """Each device runs with its map set's model, GPU profile and mode, so the
    set must be the run's own (SimConfig::validate, engine.hpp:60-68).
    Colocated runs: the maps must carry profile_hash(model, gpu) and the run's
    training mode, else ColoValidationError with the reference's message.  The
    other modes never consult the maps: they get a set built from the run's own
    (model, gpu, training), as the C++ drop-in's mapset_of does."""
    own, built = [], {}
    for r in runs:
        cs.validate_profile_pair(r.model, r.gpu)
        h = cs.profile_hash(r.model, r.gpu)
        if int(r.mode) == int(cs.SimMode.COLOCATED):
            if r.maps.profile_hash_value != h:
                raise ColoValidationError(_lib.COLO_EVALIDATION, "sim config: map profile hash does not match the profiles")
            if int(r.maps.mode) != int(r.training):
                raise ColoValidationError(_lib.COLO_EVALIDATION, "sim config: map training mode does not match sim.training")
            own.append(r)
            continue
        if r.maps.profile_hash_value == h and int(r.maps.mode) == int(r.training):
            own.append(r)
            continue
        key = (h, int(r.training))
        if key not in built:
            built[key] = cs.MapSet.build(ctx, r.model, r.gpu, mode=cs.TrainingMode(int(r.training)))
        own.append(Run(r.model, r.gpu, r.mode, r.training, built[key], r.trace, r.cache_timeout))
    return own


def run_simulations(ctx: cs.Context, runs: Sequence[Run], keep_sorted: bool = True) -> List[dict]:
    """Simulation::run for every run (engine.hpp:938-941), as GPU fleets: one
    launch per cache timeout and <= 16 map sets.  Returns MetricsReport dicts
    (metrics.hpp:17-44 field names), finalized on the device (colo_finalize);
    keep_sorted also returns each run's sorted samples for export_tpt_cdf."""
    import torch

    out: List[Optional[dict]] = [None] * len(runs)
    runs = _runs_with_own_maps(ctx, runs)
    todo = list(range(len(runs)))
    while todo:
        to = runs[todo[0]].cache_timeout
        batch, rest, sets, sidx = [], [], [], {}
        for i in todo:
            r = runs[i]
            key = id(r.maps)
            if r.cache_timeout != to or (key not in sidx and len(sets) == 16):
                rest.append(i)
                continue
            if key not in sidx:
                sidx[key] = len(sets)
                sets.append(r.maps)
            batch.append(i)
        todo = rest
        tr = [runs[i].trace for i in batch]
        cat = lambda xs, dt: np.ascontiguousarray(np.concatenate([np.asarray(x) for x in xs]) if xs else
                                                  np.zeros(0), dt)
        a = cat([t.arrival for t in tr], np.float64)
        p = cat([t.prompt for t in tr], np.uint32)
        o = cat([t.output for t in tr], np.uint32)
        ld = cat([t.label_delay for t in tr], np.float64)
        off = np.concatenate([[0], np.cumsum([len(t) for t in tr])]).astype(np.int64)
        dev = torch.device("cuda", ctx.device)
        T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x).view(dt)).to(dev)
        dset = torch.tensor([sidx[id(runs[i].maps)] for i in batch], dtype=torch.int16, device=dev)
        dmode = torch.tensor([int(runs[i].mode) for i in batch], dtype=torch.uint8, device=dev)
        try:
            res = cs.replay_colocated(ctx, sets, T(a, np.float64), T(p, np.int32), T(o, np.int32),
                                      torch.from_numpy(off).to(dev), dset, label_delay=T(ld, np.float64),
                                      cache_timeout=to, samples=True, labels=False, sim_mode=dmode)
        except cs.ColoBreachError as e:
            raise cs.ColoBreachError(_lib.COLO_EBREACH, f"invariant breach in run_simulation ({e})")
        S = cs.colocated_summaries(res["summary"])
        so = res["sample_offsets"].cpu().numpy()
        smp_dev = res["samples"]
        srt_dev = None
        fin = {}
        if smp_dev.numel():
            srt_dev = torch.empty_like(smp_dev) if keep_sorted else None
            # per run: finalize its own sample range on the device (colo_finalize: sort,
            # nearest ranks, the sequential sum of the sorted samples)
            for k in range(len(batch)):
                lo_, hi_ = int(so[k]), int(so[k + 1])
                if hi_ > lo_:
                    fin[k] = cs.finalize(ctx, smp_dev[lo_:hi_],
                                         sorted_out=srt_dev[lo_:hi_] if srt_dev is not None else None)
        smp = smp_dev.cpu().numpy()
        srt = srt_dev.cpu().numpy() if srt_dev is not None else None
        for k, i in enumerate(batch):
            s, run = S[k], runs[i]
            rep = {f: s[f] for f in cs.METRICS_FIELDS}
            rep["oom_flag"] = s["oom_jobs"] > 0
            rep["tpt_samples"] = smp[so[k]:so[k + 1]].copy()
            if srt is not None:
                rep["_sorted_for_cdf"] = srt[so[k]:so[k + 1]]
            if k in fin:
                rep["_finalized"] = fin[k]
            rep["trace_hash"] = run.trace.content_hash()
            rep["mode_tag"] = f"{_sm_str(run.mode)}/{_tm_str(run.training)}"
            out[i] = finalize_report(rep)
    return out


def run_simulation(ctx: cs.Context, run: Run) -> dict:
    return run_simulations(ctx, [run])[0]


class GpuEngine:
    """The engine the harness drives: maps and Simulation::run on one GPU.  (The
    CPU tests substitute an engine over the plain-C restatement with the same
    two methods to pin the host-side formatting without a GPU.)"""

    def __init__(self, ctx: cs.Context):
        self.ctx = ctx

    def build_maps(self, model, gpu, steps, bounds, mode):
        return cs.MapSet.build(self.ctx, model, gpu, steps, bounds, mode)

    def load_maps(self, model, gpu, offload_path, hedge_path, steps=None, bounds=None, mode=None):
        """OffloadingMap::load / HedgingMap::load of the given files; a map whose file
        is None is built from (steps, bounds, mode) as load_config does (the hedge
        grid on the offload grid's cached axis, assumed output 128)."""
        if offload_path and hedge_path:
            return cs.load_mapset(self.ctx, model, gpu, offload_path, hedge_path)
        h = cs.profile_hash(model, gpu)
        built = cs.MapSet.build(self.ctx, model, gpu, steps, bounds, mode)
        b_off, b_hed = built.cells()
        if offload_path:
            ho, off = cs.load_map_cells(offload_path, h)
            o_steps, o_bounds, o_mode = ho["steps"], ho["bounds"], ho["mode"]
            hs, hm, assumed, hed = steps.cached_token_step, bounds.max_cached_tokens, 128, b_hed
        else:
            hh, hed = cs.load_map_cells(hedge_path, h)
            o_steps, o_bounds, o_mode, off = steps, bounds, mode, b_off
            hs, hm, assumed = hh["steps"].cached_token_step, hh["bounds"].max_cached_tokens, hh["assumed_output_tokens"]
            if hh["mode"] != mode:
                o_mode = hh["mode"]
        built.close()
        if o_mode != mode:  # one map set carries one mode (engine.hpp:66-67 refuses the mix in Colocated runs)
            raise ColoValidationError(_lib.COLO_EVALIDATION, "sim config: map training mode does not match sim.training")
        return cs.MapSet.from_cells(self.ctx, model, gpu, o_steps, o_bounds, o_mode, hs, hm, assumed, h, off, hed)

    def run(self, runs: Sequence[Run], keep_sorted: bool = True) -> List[dict]:
        return run_simulations(self.ctx, runs, keep_sorted)

    def sort(self, samples) -> np.ndarray:
        """Ascending sort of f64 samples on the device (colo_sort_f64)."""
        import torch

        x = np.ascontiguousarray(samples, np.float64)
        if not len(x):
            return x
        d = torch.from_numpy(x).to(torch.device("cuda", self.ctx.device))
        o = torch.empty_like(d)
        _lib.check(lib().colo_sort_f64(self.ctx.h, cs._ptr(d), cs._ptr(o), len(x)), self.ctx.h, "sort")
        return o.cpu().numpy()

    def events(self, run: Run) -> str:
        """The run's event log (colo_colocated_events)."""
        import torch

        t = run.trace
        T = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()
        return cs.colocated_events(self.ctx, run.maps, T(t.arrival, np.float64),
                                   T(np.asarray(t.prompt, np.uint32).view(np.int32), np.int32),
                                   T(np.asarray(t.output, np.uint32).view(np.int32), np.int32),
                                   label_delay=T(t.label_delay, np.float64),
                                   query_id=T(np.asarray(t.query_id, np.uint64).view(np.int64), np.int64),
                                   cache_timeout=run.cache_timeout, sim_mode=run.mode)


def _engine(e):
    return e if hasattr(e, "run") else GpuEngine(e)


def uncontended_trace(prompt_tokens: int, queries: int, spacing: float, with_labels: bool = True) -> Trace:
    """experiment.hpp:214-230."""
    n = queries
    return Trace(np.arange(n, dtype=np.float64) * spacing, np.full(n, prompt_tokens, np.uint32),
                 np.full(n, 128, np.uint32), np.full(n, 0.01 if with_labels else -1.0), np.arange(n, dtype=np.uint64))


def run_paired(engine, m, g, training, maps, trace: Trace, cache_timeout=60.0):
    """experiment.hpp:175-185: (colocated, baseline) MetricsReports."""
    r = _engine(engine).run([Run(m, g, cs.SimMode.COLOCATED, training, maps, trace, cache_timeout),
                              Run(m, g, cs.SimMode.SEPARATE_CLUSTER, training, maps, trace, cache_timeout)])
    return r[0], r[1]


def max_trainable_tokens(engine, m, g, training, maps, mode, hi_prompt: int) -> int:
    """experiment.hpp:196-211 + supports_prompt_length (:232-242): the
    reference's binary search, with every prompt length it could probe
    evaluated in one GPU launch (one single-query run per length)."""
    extra = 256 if int(training) == int(cs.TrainingMode.CPA) else 0
    lo, hi = 16, hi_prompt
    if hi < lo:
        return 0
    lengths = list(range(lo, hi + 1))
    runs = [Run(m, g, mode, training, maps, uncontended_trace(t, 1, 1000.0), 60.0) for t in lengths]
    eng = _engine(engine)
    ok = {}
    try:
        reps = eng.run(runs, keep_sorted=False)
        for t, r in zip(lengths, reps):
            ok[t] = r["completed_jobs"] == 1 and not r["oom_flag"]
    except (cs.ColoBreachError, ColoValidationError):
        # any exception is `false` (the reference catches std::exception): one run each
        for t, run in zip(lengths, runs):
            try:
                r = eng.run([run], keep_sorted=False)[0]
                ok[t] = r["completed_jobs"] == 1 and not r["oom_flag"]
            except (cs.ColoBreachError, ColoValidationError):
                ok[t] = False
    best = 0
    while lo <= hi:
        mid = lo + (hi - lo) // 2
        if ok[mid]:
            best, lo = mid, mid + 1
        else:
            if mid == 0:
                break
            hi = mid - 1
    return 0 if best == 0 else best + extra


# ---------------------------------------------------------------- exports
def _f64(v: float) -> str:  # metrics.hpp:101-106: ostream precision 17
    return "%.17g" % v


def _opt(v) -> str:
    return _f64(v) if v is not None else ""


REPORT_CSV_HEADER = ("mode,trace_hash,generated_tokens,tpt_mean,tpt_p50,tpt_p90,tpt_p99,trained_tokens,"
                     "training_busy_time,training_throughput,peak_device_bytes,peak_training_activation_bytes,"
                     "oom_flag,preemptions,layers_freed,loads,recomputes,copy_stall_seconds,labels_dropped,"
                     "prefetch_wait_seconds,completed_jobs,oom_jobs,map_fallbacks,tpt_samples")


def export_csv(r: dict, path: str) -> None:
    """metrics.hpp:120-138."""
    row = [r["mode_tag"], str(r["trace_hash"]), str(r["generated_tokens"]), _opt(r["tpt_mean"]), _opt(r["tpt_p50"]),
           _opt(r["tpt_p90"]), _opt(r["tpt_p99"]), str(r["trained_tokens"]), _f64(r["training_busy_time"]),
           _opt(r["training_throughput"]), str(r["peak_device_bytes"]), str(r["peak_training_activation_bytes"]),
           "1" if r["oom_flag"] else "0", str(r["preemptions"]), str(r["layers_freed"]), str(r["loads"]),
           str(r["recomputes"]), _f64(r["copy_stall_seconds"]), str(r["labels_dropped"]),
           _f64(r["prefetch_wait_seconds"]), str(r["completed_jobs"]), str(r["oom_jobs"]), str(r["map_fallbacks"]),
           ";".join(_f64(v) for v in r["tpt_samples"])]
    with open(path, "w") as f:
        f.write(REPORT_CSV_HEADER + "\n" + ",".join(row) + "\n")


def json_doubles(v) -> str:
    """Doubles as nlohmann::json::dump() writes them (colo_json_doubles), comma-separated."""
    a = np.ascontiguousarray(v, np.float64)
    n = lib().colo_json_doubles(a.ctypes.data, len(a), None, 0)
    buf = C.create_string_buffer(int(n) + 1)
    lib().colo_json_doubles(a.ctypes.data, len(a), buf, int(n) + 1)
    return buf.value.decode()


def _jval(v) -> str:
    if v is None:
        return "null"
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return json_doubles([float(v)])
    if isinstance(v, str):
        return json.dumps(v)
    if isinstance(v, np.ndarray):
        return "[" + json_doubles(v) + "]"
    raise TypeError(type(v))


def _jdump(d: dict) -> str:
    """nlohmann::json::dump() of an object: keys sorted (std::map), no spaces."""
    return "{" + ",".join(f"{json.dumps(k)}:{_jval(d[k])}" for k in sorted(d)) + "}"


def save_trace(t: "Trace", path: str) -> None:
    """save_trace (workload.hpp:256-270): one nlohmann::json object per record,
    keys sorted, label_delay null when absent."""
    lines = []
    for q, a, p, o, ld in zip(t.query_id, t.arrival, t.prompt, t.output, t.label_delay):
        ldv = None if (ld != ld or ld < 0) else float(ld)
        lines.append(_jdump({"query_id": int(q), "arrival_time": float(a), "prompt_tokens": int(p),
                             "output_tokens": int(o), "label_delay": ldv}))
    with open(path, "w", newline="") as f:
        f.write("".join(ln + "\n" for ln in lines))


def export_jsonl(r: dict, path: str) -> None:
    """metrics.hpp:191-226."""
    groups = [
        {"group": "run", "mode": r["mode_tag"], "trace_hash": r["trace_hash"], "generated_tokens": r["generated_tokens"]},
        {"group": "tpt", "mean": r["tpt_mean"], "p50": r["tpt_p50"], "p90": r["tpt_p90"], "p99": r["tpt_p99"],
         "samples": np.asarray(r["tpt_samples"], np.float64)},
        {"group": "training", "trained_tokens": r["trained_tokens"], "busy_time": r["training_busy_time"],
         "throughput": r["training_throughput"], "completed_jobs": r["completed_jobs"], "oom_jobs": r["oom_jobs"]},
        {"group": "memory", "peak_device_bytes": r["peak_device_bytes"],
         "peak_training_activation_bytes": r["peak_training_activation_bytes"], "oom_flag": bool(r["oom_flag"])},
        {"group": "counters", "preemptions": r["preemptions"], "layers_freed": r["layers_freed"], "loads": r["loads"],
         "recomputes": r["recomputes"], "copy_stall_seconds": r["copy_stall_seconds"],
         "labels_dropped": r["labels_dropped"], "prefetch_wait_seconds": r["prefetch_wait_seconds"],
         "map_fallbacks": r["map_fallbacks"]},
    ]
    with open(path, "w") as f:
        for g in groups:
            f.write(_jdump(g) + "\n")


def import_jsonl(path: str) -> dict:
    """metrics.hpp:228-277."""
    r = {"tpt_samples": np.zeros(0)}
    for line in open(path):
        if not line.strip():
            continue
        j = json.loads(line)
        g = j["group"]
        if g == "run":
            r.update(mode_tag=j["mode"], trace_hash=j["trace_hash"], generated_tokens=j["generated_tokens"])
        elif g == "tpt":
            r.update(tpt_mean=j["mean"], tpt_p50=j["p50"], tpt_p90=j["p90"], tpt_p99=j["p99"],
                     tpt_samples=np.array(j["samples"], np.float64))
        elif g == "training":
            r.update(trained_tokens=j["trained_tokens"], training_busy_time=j["busy_time"],
                     training_throughput=j["throughput"], completed_jobs=j["completed_jobs"], oom_jobs=j["oom_jobs"])
        elif g == "memory":
            r.update(peak_device_bytes=j["peak_device_bytes"],
                     peak_training_activation_bytes=j["peak_training_activation_bytes"], oom_flag=j["oom_flag"])
        elif g == "counters":
            r.update({k: j[k] for k in ("preemptions", "layers_freed", "loads", "recomputes", "copy_stall_seconds",
                                        "labels_dropped", "prefetch_wait_seconds", "map_fallbacks")})
    return r


def export_tpt_cdf(r: dict, path: str) -> None:
    """metrics.hpp:280-288 (the samples sorted on the device by colo_finalize)."""
    srt = r.get("_sorted_for_cdf")
    if srt is None:
        if len(r["tpt_samples"]):
            raise cs.ColoError(_lib.COLO_EINVAL, "export_tpt_cdf: run the report with keep_sorted=True")
        srt = np.zeros(0)
    n = len(srt)
    with open(path, "w") as f:
        f.write("tpt_seconds,cumulative_fraction\n")
        f.writelines(f"{_f64(v)},{_f64(float(i + 1) / float(n))}\n" for i, v in enumerate(srt.tolist()))


# ------------------------------------------------------------------- CLI
def _out_file(d: str, name: str, force: bool) -> str:
    p = os.path.join(d, name)
    if os.path.exists(p) and not force:
        raise ColoValidationError(_lib.COLO_EVALIDATION, f"refusing to overwrite {p} (pass --force)")
    return p


def _resolve(path: str) -> str:  # tools/colosim.cpp:27-34
    if os.path.exists(path):
        return path
    d = os.environ.get("COLOSIM_PROFILE_DIR")
    if d and os.path.exists(os.path.join(d, path)):
        return os.path.join(d, path)
    return path


def load_config(engine, path, offload_map_path="", hedge_map_path=""):
    """tools/colosim.cpp:54-71: the config plus its maps for ec.training."""
    eng = _engine(engine)
    ec = ExperimentConfig.from_file(_resolve(path))
    if offload_map_path or hedge_map_path:
        # whichever file is given is loaded; the other map is built from the config (colosim.cpp:58-67)
        maps = eng.load_maps(ec.model, ec.gpu, _resolve(offload_map_path) if offload_map_path else None,
                             _resolve(hedge_map_path) if hedge_map_path else None,
                             steps=ec.map_steps, bounds=ec.map_bounds, mode=ec.training)
    else:
        maps = eng.build_maps(ec.model, ec.gpu, ec.map_steps, ec.map_bounds, ec.training)
    return ec, maps


def cmd_run(engine, config_path, out_dir, trace_path="", offload_map_path="", hedge_map_path="", seed_override=-1,
            mode_override="", emit_events=False, force=False) -> dict:
    """tools/colosim.cpp:97-131 (--emit-events: ServingOnly and Colocated runs)."""
    eng = _engine(engine)
    ec, maps = load_config(eng, config_path, offload_map_path, hedge_map_path)
    if mode_override:
        ec.mode = cs.SimMode.parse(mode_override)
    if seed_override >= 0:
        ec.seed = seed_override
        ec.trace_spec.seed = seed_override
    if trace_path:
        ec.trace_spec.file = _resolve(trace_path)
    trace = ec.trace_spec.realize()
    run = Run(ec.model, ec.gpu, ec.mode, ec.training, maps, trace, ec.cache_timeout)
    if emit_events and not hasattr(eng, "events"):
        raise ColoValidationError(_lib.COLO_EVALIDATION, "--emit-events: this engine keeps no event log")
    rep = eng.run([run])[0]
    os.makedirs(out_dir, exist_ok=True)
    export_csv(rep, _out_file(out_dir, "report.csv", force))
    export_jsonl(rep, _out_file(out_dir, "report.jsonl", force))
    export_tpt_cdf(rep, _out_file(out_dir, "tpt_cdf.csv", force))
    if emit_events:  # tools/colosim.cpp:121
        with open(_out_file(out_dir, "events.jsonl", force), "w", newline="") as f:
            f.write(eng.events(run))
    return rep


def cmd_plotdata(report_path, out_dir, force=False, engine=None):
    """tools/colosim.cpp:254-260 (the samples sorted by the engine: on the GPU, colo_sort_f64)."""
    r = import_jsonl(_resolve(report_path))
    eng = _engine(engine if engine is not None else cs.Context(0))
    r["_sorted_for_cdf"] = eng.sort(r["tpt_samples"])
    os.makedirs(out_dir, exist_ok=True)
    export_tpt_cdf(r, _out_file(out_dir, "tpt_cdf.csv", force))


def cmd_compare(engine, config_path, out_dir, force=False) -> None:
    """tools/colosim.cpp:140-250: the figure datasets.  Each stage's runs (all
    token lengths x modes x {colocated, baseline}, the memory-wall probes, all
    QPS points x {colocated, baseline, serving-only}) are one GPU fleet."""
    eng = _engine(engine)
    ec, _ = load_config(eng, config_path)
    os.makedirs(out_dir, exist_ok=True)
    modes = ec.sweep_modes or [ec.training]
    if ec.sweep_token_lengths:
        tput = ["mode,prompt_tokens,colocated_tput,baseline_tput,ratio,baseline_oom"]
        mem = ["mode,prompt_tokens,colocated_peak_bytes,baseline_peak_bytes,saving,baseline_oom"]
        maxtok = ["mode,colocated_max_tokens,baseline_max_tokens,ratio"]
        runs, keys, mapsets = [], [], {}
        for mode in modes:
            mapsets[int(mode)] = eng.build_maps(ec.model, ec.gpu, ec.map_steps, ec.map_bounds, mode)
            for tokens in ec.sweep_token_lengths:
                trace = uncontended_trace(tokens, 3, 1000.0)
                for sm in (cs.SimMode.COLOCATED, cs.SimMode.SEPARATE_CLUSTER):
                    runs.append(Run(ec.model, ec.gpu, sm, mode, mapsets[int(mode)], trace, ec.cache_timeout))
                keys.append((mode, tokens))
        reps = eng.run(runs, keep_sorted=False)
        for k, (mode, tokens) in enumerate(keys):
            colo, base = reps[2 * k], reps[2 * k + 1]
            ct, bt = colo["training_throughput"], base["training_throughput"]
            ratio = ct / bt if (ct is not None and bt is not None) else 0.0
            tput.append("%s,%d,%.6f,%.6f,%.6f,%d" % (_tm_str(mode), tokens, ct or 0.0, bt or 0.0, ratio,
                                                     1 if base["oom_flag"] else 0))
            saving = (1.0 - float(colo["peak_training_activation_bytes"]) / float(base["peak_training_activation_bytes"])
                      if base["peak_training_activation_bytes"] else 0.0)
            mem.append("%s,%d,%d,%d,%.6f,%d" % (_tm_str(mode), tokens, colo["peak_training_activation_bytes"],
                                                base["peak_training_activation_bytes"], saving,
                                                1 if base["oom_flag"] else 0))
        for mode in modes:
            hi_prompt = ec.map_bounds.max_cached_tokens - (256 if int(mode) == int(cs.TrainingMode.CPA) else 0)
            mp = mapsets[int(mode)]
            mc = max_trainable_tokens(eng, ec.model, ec.gpu, mode, mp, cs.SimMode.COLOCATED, hi_prompt)
            mb = max_trainable_tokens(eng, ec.model, ec.gpu, mode, mp, cs.SimMode.SEPARATE_CLUSTER, hi_prompt)
            maxtok.append("%s,%d,%d,%.4f" % (_tm_str(mode), mc, mb, float(mc) / float(mb) if mb else 0.0))
        for name, lines in (("tput_vs_tokens.csv", tput), ("mem_vs_tokens.csv", mem), ("max_tokens.csv", maxtok)):
            with open(_out_file(out_dir, name, force), "w") as f:
                f.write("\n".join(lines) + "\n")
    if ec.sweep_qps:
        offl = ["qps,colocated_tput,baseline_tput,layers_freed,loads,recomputes,preemptions"]
        tptq = ["qps,colocated_mean_tpt,serving_only_mean_tpt,overhead"]
        maps = eng.build_maps(ec.model, ec.gpu, ec.map_steps, ec.map_bounds, ec.training)
        runs = []
        for qps in ec.sweep_qps:
            spec = TraceSpec(None, qps, max(ec.trace_spec.duration, 80.0 / qps), ec.trace_spec.seed,
                             ec.trace_spec.length_dist,
                             ec.sweep_min_tokens if ec.sweep_min_tokens is not None else ec.trace_spec.min_tokens,
                             ec.trace_spec.label_delay)
            trace = spec.realize()
            for sm in (cs.SimMode.COLOCATED, cs.SimMode.SEPARATE_CLUSTER, cs.SimMode.SERVING_ONLY):
                runs.append(Run(ec.model, ec.gpu, sm, ec.training, maps, trace, ec.cache_timeout))
        reps = eng.run(runs)
        for k, qps in enumerate(ec.sweep_qps):
            colo, base, serve = reps[3 * k], reps[3 * k + 1], reps[3 * k + 2]
            offl.append("%.4f,%.6f,%.6f,%d,%d,%d,%d" % (qps, colo["training_throughput"] or 0.0,
                                                        base["training_throughput"] or 0.0, colo["layers_freed"],
                                                        colo["loads"], colo["recomputes"], colo["preemptions"]))
            cm, sm_ = colo["tpt_mean"], serve["tpt_mean"]
            overhead = cm / sm_ - 1.0 if (cm is not None and sm_ is not None and sm_ > 0) else 0.0
            tptq.append("%.4f,%.6f,%.6f,%.6f" % (qps, cm or 0.0, sm_ or 0.0, overhead))
            if k == len(ec.sweep_qps) - 1:
                export_tpt_cdf(colo, _out_file(out_dir, "tpt_cdf_colocated.csv", force))
                export_tpt_cdf(serve, _out_file(out_dir, "tpt_cdf_serving_only.csv", force))
        with open(_out_file(out_dir, "tput_vs_qps.csv", force), "w") as f:
            f.write("\n".join(offl) + "\n")
        with open(_out_file(out_dir, "tpt_mean_vs_qps.csv", force), "w") as f:
            f.write("\n".join(tptq) + "\n")
    if not ec.sweep_token_lengths and not ec.sweep_qps:
        raise ColoValidationError(_lib.COLO_EVALIDATION,
                                  "compare: config declares no sweep axes (sweep.token_lengths / sweep.qps)")

