"""TEST INFRASTRUCTURE ONLY -- ctypes front-end to the CPU oracle.

Two interchangeable back-ends with identical signatures:

* ``OracleLib("oracle")`` -> ``oracle/lib/libcolo_oracle.so``: the plain-C
  restatement (``colo_oracle.c``), the parity checker used by ``tests/``.
* ``OracleLib("ref")``    -> ``oracle/_ref/libcolo_ref.so``: the unchanged
  reference headers (``/root/reference/proj/include``) compiled through
  ``ref_shim.cpp``; used to pin the restatement, to write the golden fixtures
  (``tests/golden/make_golden.py``) and as bench.py's ``--impl reference`` arm.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product (``paper_2503_01066_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "oracle": os.path.join(HERE, "lib", "libcolo_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libcolo_ref.so"),
}

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
u16p = np.ctypeslib.ndpointer(np.uint16, flags="C")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")


class Model(C.Structure):
    """profiles.hpp:23-35 (ModelProfile, defaults = the Llama-8B-like profile)."""

    _fields_ = [
        ("num_layers", C.c_uint64),
        ("kv_bytes_per_token", C.c_uint64),
        ("act_bytes_per_token_per_layer", C.c_uint64),
        ("prefill_coef_linear", C.c_double),
        ("prefill_coef_quad", C.c_double),
        ("decode_coef_const", C.c_double),
        ("decode_coef_context", C.c_double),
        ("backward_to_forward_ratio", C.c_double),
        ("record_prefill_multiplier", C.c_double),
        ("record_decode_multiplier", C.c_double),
        ("workspace_factor", C.c_double),
        ("weights_bytes", C.c_uint64),
    ]


class Gpu(C.Structure):
    """profiles.hpp:98-102."""

    _fields_ = [(n, C.c_uint64) for n in ("capacity_bytes", "h2d_bandwidth", "d2h_bandwidth", "runtime_reserve_bytes")]


class Grid(C.Structure):
    """maps.hpp:63-73."""

    _fields_ = [(n, C.c_uint64) for n in ("cached_step", "incoming_step", "batch_step", "max_cached", "max_incoming", "max_batch")]


class Maps(C.Structure):
    _fields_ = [
        ("grid", Grid),
        ("offload_cells", C.c_void_p),
        ("hedge_step", C.c_uint64),
        ("hedge_max", C.c_uint64),
        ("hedge_cells", C.c_void_p),
        ("num_layers", C.c_uint64),
    ]


class Summary(C.Structure):
    _fields_ = [
        ("generated_tokens", C.c_uint64),
        ("slow_tokens", C.c_uint64),
        ("slow_queries", C.c_uint64),
        ("batches", C.c_uint64),
        ("peak_device_bytes", C.c_uint64),
        ("max_batch_size", C.c_uint64),
        ("end_time", C.c_double),
    ]


class ColoReport(C.Structure):
    """orc_colo_report (colo_oracle.h): MetricsReport fields (metrics.hpp:17-44) + replay extras."""

    _fields_ = [
        ("generated_tokens", C.c_uint64),
        ("trained_tokens", C.c_uint64),
        ("training_busy_time", C.c_double),
        ("peak_device_bytes", C.c_uint64),
        ("peak_training_activation_bytes", C.c_uint64),
        ("preemptions", C.c_uint64),
        ("layers_freed", C.c_uint64),
        ("loads", C.c_uint64),
        ("recomputes", C.c_uint64),
        ("copy_stall_seconds", C.c_double),
        ("labels_dropped", C.c_uint64),
        ("prefetch_wait_seconds", C.c_double),
        ("completed_jobs", C.c_uint64),
        ("map_fallbacks", C.c_uint64),
        ("oom_jobs", C.c_uint64),
        ("batches", C.c_uint64),
        ("max_batch_size", C.c_uint64),
        ("offload_decisions", C.c_uint64),
        ("admissions", C.c_uint64),
        ("slow_tokens", C.c_uint64),
        ("slow_queries", C.c_uint64),
        ("end_time", C.c_double),
        ("status", C.c_uint64),
    ]


# MetricsReport fields the reference itself reports (metrics.hpp:17-44)
METRICS_FIELDS = [f for f, _ in ColoReport._fields_[:15]]
SIM_MODES = {"serving-only": 0, "colocated": 1, "baseline": 2}  # engine.hpp:23-39 names


class Dist(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("fixed_value", C.c_double),
        ("lo", C.c_double),
        ("hi", C.c_double),
        ("bin_values", C.c_void_p),
        ("bin_probs", C.c_void_p),
        ("nbins", C.c_size_t),
        ("min_tokens", C.c_uint64),
    ]


TUPLE_DTYPE = np.dtype(
    [("cached", "<u4"), ("incoming", "<u4"), ("charged", "<u4"), ("batch", "<u2"), ("pending", "u1"), ("dev_layers", "u1")]
)
assert TUPLE_DTYPE.itemsize == 16
BATCH_DTYPE = np.dtype(
    [("start", "<f8"), ("end", "<f8"), ("first", "<u4"), ("n", "<u4"), ("need_total", "<u8"), ("max_incoming", "<u4"), ("verdict", "<u4")]
)
assert BATCH_DTYPE.itemsize == 40

KGIB = 1024**3
KGB = 1000**3


def default_model() -> Model:
    """profiles.hpp:23-35 defaults."""
    return Model(32, 512 * 1024, 417000, 1e-4, 2e-8, 0.020, 2e-6, 1.326, 1.21, 1.35, 1.0, 16 * KGIB)


def phi14b_model() -> Model:
    """profiles.hpp:88-95."""
    m = default_model()
    m.num_layers = 40
    m.kv_bytes_per_token = 838861
    m.act_bytes_per_token_per_layer = 667200
    m.weights_bytes = 24 * KGIB
    return m


def default_gpu() -> Gpu:
    """profiles.hpp:98-102 defaults."""
    return Gpu(80 * KGIB, 24 * KGB, 24 * KGB, 2 * KGIB)


def default_grid() -> Grid:
    """maps.hpp:63-73 defaults."""
    return Grid(500, 500, 5, 8000, 8000, 50)


def grid_shape(g: Grid):
    return (g.max_cached // g.cached_step + 1, g.max_incoming // g.incoming_step, g.max_batch // g.batch_step)


def build(quiet: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True, capture_output=quiet)


class OracleLib:
    def __init__(self, which: str = "oracle"):
        self.which = which
        path = PATHS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} missing; run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        p = "orc_" if which == "oracle" else "ref_"
        self.p = p
        MP, GP, GRP = C.POINTER(Model), C.POINTER(Gpu), C.POINTER(Grid)
        ip = C.POINTER(C.c_int)
        sig = {
            "prefill_latency": (C.c_double, [MP, C.c_uint64, C.c_uint64, C.c_int, ip]),
            "decode_step_latency": (C.c_double, [MP, C.c_uint64, C.c_uint64, C.c_int, ip]),
            "forward_layer_latency": (C.c_double, [MP, C.c_uint64, ip]),
            "backward_layer_latency": (C.c_double, [MP, C.c_uint64, ip]),
            "activation_bytes": (C.c_uint64, [MP, C.c_uint64, C.c_uint64, ip]),
            "kv_bytes": (C.c_uint64, [MP, C.c_uint64, C.c_uint64]),
            "serving_memory": (C.c_uint64, [MP, C.c_uint64, C.c_uint64, ip]),
            "transfer_time": (C.c_double, [GP, C.c_uint64, C.c_int]),
            "validate_profile_pair": (C.c_int, [MP, GP]),
            "profile_hash": (C.c_uint64, [MP, GP]),
            "round_up_bucket": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "offload_cell_decision": (None, [MP, GP, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, ip, C.POINTER(C.c_uint64)]),
            "build_offloading_map": (C.c_int, [MP, GP, GRP, C.c_int, u8p, C.c_size_t]),
            "build_hedging_map": (C.c_int, [MP, GP, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, u8p, C.c_size_t]),
            "hedge_recompute_time": (C.c_double, [MP, C.c_int, C.c_uint64, C.c_uint64, ip]),
            "hedge_residual_load_time": (C.c_double, [MP, GP, C.c_uint64, C.c_uint64, ip]),
            "finalize": (C.c_int, [f64p, C.c_size_t] + [C.POINTER(C.c_double)] * 4),
            "generate_trace": (C.c_int64, [C.c_double, C.c_double, C.POINTER(Dist), C.POINTER(Dist), C.c_uint64, f64p, u32p, u32p, C.c_void_p, C.c_size_t]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            setattr(self, "_" + name, f)

    # -- scalar cost model ------------------------------------------------------
    def _err_call(self, fn, *args):
        err = C.c_int(0)
        v = fn(*args, C.byref(err))
        return v, err.value

    def prefill_latency(self, m, tokens, batch=1, recording=False):
        return self._err_call(self._prefill_latency, C.byref(m), tokens, batch, int(recording))

    def decode_step_latency(self, m, ctx, batch=1, recording=False):
        return self._err_call(self._decode_step_latency, C.byref(m), ctx, batch, int(recording))

    def forward_layer_latency(self, m, tokens):
        return self._err_call(self._forward_layer_latency, C.byref(m), tokens)

    def backward_layer_latency(self, m, tokens):
        return self._err_call(self._backward_layer_latency, C.byref(m), tokens)

    def activation_bytes(self, m, tokens, layers):
        return self._err_call(self._activation_bytes, C.byref(m), tokens, layers)

    def kv_bytes(self, m, tokens, batch):
        return self._kv_bytes(C.byref(m), tokens, batch)

    def serving_memory(self, m, tokens, batch):
        return self._err_call(self._serving_memory, C.byref(m), tokens, batch)

    def transfer_time(self, g, nbytes, h2d=True):
        return self._transfer_time(C.byref(g), nbytes, int(h2d))

    def validate_profile_pair(self, m, g):
        return self._validate_profile_pair(C.byref(m), C.byref(g))

    def profile_hash(self, m, g):
        return self._profile_hash(C.byref(m), C.byref(g))

    def round_up_bucket(self, v, s):
        return self._round_up_bucket(v, s)

    def offload_cell_decision(self, m, g, cpa, cached, incoming, batch):
        a, lay = C.c_int(0), C.c_uint64(0)
        self._offload_cell_decision(C.byref(m), C.byref(g), int(cpa), cached, incoming, batch, C.byref(a), C.byref(lay))
        return a.value, lay.value

    def hedge_recompute_time(self, m, cpa, cached, assumed=128):
        return self._err_call(self._hedge_recompute_time, C.byref(m), int(cpa), cached, assumed)

    def hedge_residual_load_time(self, m, g, cached, freed):
        return self._err_call(self._hedge_residual_load_time, C.byref(m), C.byref(g), cached, freed)

    # -- maps --------------------------------------------------------------------
    def build_offloading_map(self, m, g, grid, cpa):
        if 0 in (grid.cached_step, grid.incoming_step, grid.batch_step):
            raise ValueError("map grid: steps must be positive")  # maps.hpp:198-199
        n = int(np.prod(grid_shape(grid)))
        cells = np.zeros(n, np.uint8)
        rc = self._build_offloading_map(C.byref(m), C.byref(g), C.byref(grid), int(cpa), cells, n)
        if rc:
            raise ValueError(f"build_offloading_map rc={rc}")
        return cells

    def build_hedging_map(self, m, g, step, maxc, cpa, assumed=128):
        n = (maxc // step) * (m.num_layers + 1)
        cells = np.zeros(n, np.uint8)
        rc = self._build_hedging_map(C.byref(m), C.byref(g), step, maxc, int(cpa), assumed, cells, n)
        if rc:
            raise ValueError(f"build_hedging_map rc={rc}")
        return cells

    # -- batched hot path ---------------------------------------------------------
    def decide(self, m, g, grid, cpa, tuples, hedge_step=None, hedge_max=None, assumed=128):
        """Composed verdicts (engine.hpp:434-448, 513-557) for a colo_tuple array."""
        hs = grid.cached_step if hedge_step is None else hedge_step
        hm = grid.max_cached if hedge_max is None else hedge_max
        t = np.ascontiguousarray(tuples, dtype=TUPLE_DTYPE)
        out = np.zeros(len(t), np.uint32)
        if self.which == "ref":
            f = self.lib.ref_decide
            f.restype = C.c_int
            rc = f(C.byref(m), C.byref(g), C.byref(grid), C.c_int(int(cpa)), C.c_uint64(hs), C.c_uint64(hm),
                   C.c_uint64(assumed), t.ctypes.data_as(C.c_void_p), C.c_size_t(len(t)), out.ctypes.data_as(C.c_void_p))
            if rc:
                raise ValueError(f"ref_decide rc={rc}")
            return out
        off = self.build_offloading_map(m, g, grid, cpa)
        hed = self.build_hedging_map(m, g, hs, hm, cpa, assumed)
        mp = Maps(grid, off.ctypes.data, hs, hm, hed.ctypes.data, m.num_layers)
        self.lib.orc_decide(C.byref(mp), t.ctypes.data_as(C.c_void_p), C.c_size_t(len(t)), out.ctypes.data_as(C.c_void_p))
        return out

    def decide_exact(self, m, g, cpa, tuples, assumed=128):
        t = np.ascontiguousarray(tuples, dtype=TUPLE_DTYPE)
        out = np.zeros(len(t), np.uint32)
        fn = getattr(self.lib, self.p + "decide_exact")
        fn(C.byref(m), C.byref(g), C.c_int(int(cpa)), C.c_uint64(assumed), t.ctypes.data_as(C.c_void_p),
           C.c_size_t(len(t)), out.ctypes.data_as(C.c_void_p))
        return out

    def features_decide(self, sets, grid, prompt, output, dev_offsets, dev_set, assumed=128):
        """sets: list of (Model, Gpu, cpa).  SURVEY §8(d) C2 rule."""
        prompt = np.ascontiguousarray(prompt, np.uint32)
        output = np.ascontiguousarray(output, np.uint32)
        dev_offsets = np.ascontiguousarray(dev_offsets, np.uint64)
        dev_set = np.ascontiguousarray(dev_set, np.uint16)
        out = np.zeros(len(prompt), np.uint32)
        ns = len(sets)
        if self.which == "ref":
            models = (Model * ns)(*[s[0] for s in sets])
            gpus = (Gpu * ns)(*[s[1] for s in sets])
            cpas = (C.c_int * ns)(*[int(s[2]) for s in sets])
            rc = self.lib.ref_features_decide(models, gpus, cpas, C.c_size_t(ns), C.byref(grid), C.c_uint64(assumed),
                                              prompt.ctypes.data_as(C.c_void_p), output.ctypes.data_as(C.c_void_p),
                                              dev_offsets.ctypes.data_as(C.c_void_p), dev_set.ctypes.data_as(C.c_void_p),
                                              C.c_size_t(len(dev_set)), out.ctypes.data_as(C.c_void_p))
        else:
            keep = []
            mps = []
            for (m, g, cpa) in sets:
                off = self.build_offloading_map(m, g, grid, cpa)
                hed = self.build_hedging_map(m, g, grid.cached_step, grid.max_cached, cpa, assumed)
                keep += [off, hed]
                mps.append(Maps(grid, off.ctypes.data, grid.cached_step, grid.max_cached, hed.ctypes.data, m.num_layers))
            arr = (Maps * ns)(*mps)
            ptrs = (C.c_void_p * ns)(*[C.addressof(arr[i]) for i in range(ns)])
            cpas = (C.c_int * ns)(*[int(s[2]) for s in sets])
            rc = self.lib.orc_features_decide(ptrs, cpas, C.c_size_t(ns), prompt.ctypes.data_as(C.c_void_p),
                                              output.ctypes.data_as(C.c_void_p), dev_offsets.ctypes.data_as(C.c_void_p),
                                              dev_set.ctypes.data_as(C.c_void_p), C.c_size_t(len(dev_set)),
                                              out.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError(f"features_decide rc={rc}")
        return out

    def features(self, m, cpa, prompt, output):
        assert self.which == "oracle"
        prompt = np.ascontiguousarray(prompt, np.uint32)
        output = np.ascontiguousarray(output, np.uint32)
        n = len(prompt)
        need, charged, prefill = np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(n, np.float64)
        rc = self.lib.orc_features(C.byref(m), C.c_int(int(cpa)), prompt.ctypes.data_as(C.c_void_p),
                                   output.ctypes.data_as(C.c_void_p), C.c_size_t(n), need.ctypes.data_as(C.c_void_p),
                                   charged.ctypes.data_as(C.c_void_p), prefill.ctypes.data_as(C.c_void_p))
        if rc:
            raise ValueError(f"features rc={rc}")
        return need, charged, prefill

    def replay_serving(self, m, g, arrival, prompt, output, tau=float("inf"), grid=None, cpa=True,
                       want_samples=True):
        """Serving-only replay.  Returns dict(samples, labels, batches, summary, pctl)."""
        arrival = np.ascontiguousarray(arrival, np.float64)
        prompt = np.ascontiguousarray(prompt, np.uint32)
        output = np.ascontiguousarray(output, np.uint32)
        n = len(prompt)
        ns = int(output.astype(np.uint64).sum())
        samples = np.zeros(max(ns, 1), np.float64) if want_samples else None
        labels = np.zeros(max(n, 1), np.uint8)
        batches = np.zeros(max(n, 1), BATCH_DTYPE)
        summ = Summary()
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        if self.which == "ref":
            pctl = np.full(4, np.nan)
            rc = self.lib.ref_replay_serving(C.byref(m), C.byref(g), vp(arrival), vp(prompt), vp(output), C.c_uint64(n),
                                             C.c_double(tau), C.byref(grid) if grid is not None else None,
                                             C.c_int(int(cpa)), vp(samples), vp(labels), vp(batches), C.byref(summ),
                                             vp(pctl))
        else:
            keep = []
            mp = None
            if grid is not None:
                off = self.build_offloading_map(m, g, grid, cpa)
                hed = self.build_hedging_map(m, g, grid.cached_step, grid.max_cached, cpa, 128)
                keep += [off, hed]
                mp = Maps(grid, off.ctypes.data, grid.cached_step, grid.max_cached, hed.ctypes.data, m.num_layers)
            rc = self.lib.orc_replay_serving(C.byref(m), C.byref(g), vp(arrival), vp(prompt), vp(output), C.c_uint64(n),
                                             C.c_double(tau), C.byref(mp) if mp is not None else None, C.c_int(int(cpa)),
                                             vp(samples), vp(labels), vp(batches), C.byref(summ))
            pctl = None
        if rc:
            raise ValueError(f"replay_serving rc={rc}")
        nb = summ.batches
        res = {
            "samples": samples[:ns] if samples is not None else None,
            "labels": labels[:n],
            "batches": batches[:nb],
            "summary": {f: getattr(summ, f) for f, _ in Summary._fields_},
        }
        if pctl is None and want_samples and ns:
            pctl = np.array(self.finalize(res["samples"]))
        res["pctl"] = pctl
        return res

    def serving_samples(self, m, g, arrival, prompt, output, want_samples=True):
        """oracle/_ref only: the reference's Simulation::run (ServingOnly) without
        its event log.  Returns dict(samples, generated_tokens, peak_device_bytes, pctl)."""
        assert self.which == "ref"
        arrival = np.ascontiguousarray(arrival, np.float64)
        prompt = np.ascontiguousarray(prompt, np.uint32)
        output = np.ascontiguousarray(output, np.uint32)
        n = len(prompt)
        ns = int(output.astype(np.uint64).sum())
        samples = np.empty(max(ns, 1), np.float64) if want_samples else None
        gen, peak = C.c_uint64(0), C.c_uint64(0)
        pctl = np.full(4, np.nan)
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        f = self.lib.ref_serving_samples
        f.restype = C.c_int
        rc = f(C.byref(m), C.byref(g), vp(arrival), vp(prompt), vp(output), C.c_uint64(n), vp(samples), C.byref(gen),
               C.byref(peak), vp(pctl))
        if rc:
            raise ValueError(f"ref_serving_samples rc={rc}")
        return {"samples": samples[:ns] if samples is not None else None, "generated_tokens": gen.value,
                "peak_device_bytes": peak.value, "pctl": pctl}

    def replay_colocated(self, m, g, grid, cpa, arrival, prompt, output, label_delay=None, cache_timeout=60.0,
                         tau=float("inf"), want_samples=True, want_batches=True, sim_mode="colocated", cells=None):
        """Simulation::run in ``sim_mode`` (colocated | baseline | serving-only; maps from build_maps).
        label_delay: per-query seconds, < 0 = nullopt (None = all nullopt).
        Returns dict(report, samples, labels, batches, pctl, rc)."""
        arrival = np.ascontiguousarray(arrival, np.float64)
        prompt = np.ascontiguousarray(prompt, np.uint32)
        output = np.ascontiguousarray(output, np.uint32)
        ld = None if label_delay is None else np.ascontiguousarray(label_delay, np.float64)
        n = len(prompt)
        ns = int(output.astype(np.uint64).sum())
        samples = np.zeros(max(ns, 1), np.float64) if want_samples else None
        labels = np.zeros(max(n, 1), np.uint8)
        batches = np.zeros(max(n, 1), BATCH_DTYPE) if want_batches else None
        rep = ColoReport()
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        pctl = None
        if self.which == "ref":
            pctl = np.full(4, np.nan)
            rc = self.lib.ref_replay_sim(C.byref(m), C.byref(g), C.byref(grid), C.c_int(SIM_MODES[sim_mode]), C.c_int(int(cpa)),
                                               C.c_double(cache_timeout), vp(arrival), vp(prompt), vp(output), vp(ld),
                                               C.c_uint64(n), vp(samples), vp(batches), C.byref(rep), vp(pctl))
            labels = None
        else:
            if cells is None:
                cells = (self.build_offloading_map(m, g, grid, cpa),
                         self.build_hedging_map(m, g, grid.cached_step, grid.max_cached, cpa, 128))
            off, hed = cells
            mp = Maps(grid, off.ctypes.data, grid.cached_step, grid.max_cached, hed.ctypes.data, m.num_layers)
            rc = self.lib.orc_replay_sim(C.byref(m), C.byref(g), C.byref(mp), C.c_int(SIM_MODES[sim_mode]), C.c_int(int(cpa)),
                                               C.c_double(cache_timeout), vp(arrival), vp(prompt), vp(output), vp(ld),
                                               C.c_uint64(n), C.c_double(tau), vp(samples), vp(labels), vp(batches),
                                               C.byref(rep))
            labels = labels[:n]
        if rc not in (0, 3):
            raise ValueError(f"replay_colocated rc={rc}")
        ng = rep.generated_tokens if rc == 0 else 0
        res = {
            "rc": rc,
            "report": {f: getattr(rep, f) for f, _ in ColoReport._fields_},
            "samples": samples[:ng] if samples is not None else None,
            "labels": labels,
            "batches": batches[: rep.batches] if batches is not None else None,
        }
        if pctl is None and samples is not None and ng:
            pctl = np.array(self.finalize(res["samples"]))
        res["pctl"] = pctl
        return res

    def finalize(self, samples):
        s = np.ascontiguousarray(samples, np.float64)
        a, b, c, d = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        rc = self._finalize(s, len(s), C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        if rc:
            raise ValueError("finalize on empty samples")
        return a.value, b.value, c.value, d.value

    def generate_trace(self, qps, duration, lengths, seed, label_delay=None, cap=None, with_labels=False):
        """lengths/label_delay: ('fixed', v) | ('uniform', lo, hi) | ('histogram', values, probs); optional min_tokens kw.
        with_labels: also return the per-query label delays (-1.0 = nullopt)."""
        keep = []

        def mk(spec):
            if spec is None:
                return None
            kind = spec[0]
            d = Dist()
            d.min_tokens = spec[-1] if kind != "histogram" and len(spec) == (3 if kind == "fixed" else 4) else 0
            if kind == "fixed":
                d.kind, d.fixed_value = 0, spec[1]
            elif kind == "uniform":
                d.kind, d.lo, d.hi = 1, spec[1], spec[2]
            else:
                v = np.ascontiguousarray(spec[1], np.float64)
                p_ = np.ascontiguousarray(spec[2], np.float64)
                keep.extend([v, p_])
                d.kind, d.bin_values, d.bin_probs, d.nbins = 2, v.ctypes.data, p_.ctypes.data, len(v)
                d.min_tokens = spec[3] if len(spec) > 3 else 0
            return d

        ld, dd = mk(lengths), mk(label_delay)
        if cap is None:
            cap = int(qps * duration * 1.5 + 1000)
        arr, pr, out = np.zeros(cap), np.zeros(cap, np.uint32), np.zeros(cap, np.uint32)
        lab = np.zeros(cap)
        n = self._generate_trace(qps, duration, C.byref(ld), C.byref(dd) if dd is not None else None, seed, arr, pr, out,
                                 lab.ctypes.data, cap)
        if n < 0:
            raise ValueError(f"generate_trace rc={n}")
        if with_labels:
            return arr[:n].copy(), pr[:n].copy(), out[:n].copy(), lab[:n].copy()
        return arr[:n].copy(), pr[:n].copy(), out[:n].copy()


def sharegpt_histogram():
    """proj/profiles/sharegpt_like_lengths.jsonl (11 bins)."""
    values = [64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096]
    probs = [0.05, 0.10, 0.15, 0.15, 0.13, 0.12, 0.10, 0.08, 0.06, 0.04, 0.02]
    return np.array(values, np.float64), np.array(probs, np.float64)
