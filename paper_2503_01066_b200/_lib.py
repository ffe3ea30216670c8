"""ctypes binding of ``libcolo_b200.so`` (the C-ABI in ``include/colo_abi.h``).

The library is built in-tree by ``__graft_entry__.build()`` / ``make``.  There
is no fallback: importing the package without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COLO_B200_LIB") or os.path.join(HERE, "libcolo_b200.so")  # override: build variants

COLO_OK, COLO_EINVAL, COLO_EVALIDATION, COLO_EBREACH, COLO_ECUDA = range(5)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "EVALIDATION", 3: "EBREACH", 4: "ECUDA"}
NCOUNTERS = 8
HIST_BITS = 21
HIST_BINS = 1 << HIST_BITS


class ColoError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"colo {STATUS_NAMES.get(status, status)}: {what}")
        self.status = status


class ColoValidationError(ColoError, ValueError):
    """COLO_EVALIDATION -- where the reference throws std::runtime_error."""


class ColoInvalidArgument(ColoError, ValueError):
    """COLO_EINVAL -- where the reference throws std::invalid_argument."""


class ColoBreachError(ColoError):
    """COLO_EBREACH -- where the reference throws InvariantBreach (engine.hpp:43-46)."""


class Model(C.Structure):
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
    _fields_ = [(n, C.c_uint64) for n in ("capacity_bytes", "h2d_bandwidth", "d2h_bandwidth", "runtime_reserve_bytes")]


class Grid(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("cached_step", "incoming_step", "batch_step", "max_cached", "max_incoming", "max_batch")]


class DeviceSummary(C.Structure):
    _fields_ = [
        ("generated_tokens", C.c_uint64),
        ("slow_tokens", C.c_uint64),
        ("slow_queries", C.c_uint64),
        ("batches", C.c_uint64),
        ("peak_device_bytes", C.c_uint64),
        ("max_batch_size", C.c_uint64),
        ("end_time", C.c_double),
        ("tpt_sum", C.c_uint64 * 3),
        ("flags", C.c_uint64),
    ]


class ReplayOpts(C.Structure):
    _fields_ = [
        ("tau", C.c_double),
        ("sets", C.c_void_p),
        ("d_samples", C.c_void_p),
        ("d_sample_offsets", C.c_void_p),
        ("d_labels", C.c_void_p),
        ("d_batches", C.c_void_p),
        ("d_summary", C.c_void_p),
        ("d_hist", C.c_void_p),
        ("nfilters", C.c_uint32),
        ("hist_shift", C.c_uint32),
        ("filter_shift", C.c_uint32),
        ("segment_len", C.c_uint32),
        ("filter_prefix", C.c_uint64 * 3),
        ("reuse_entries", C.c_uint32),
        ("stats_mode", C.c_uint32),
        ("d_verdicts", C.c_void_p),
    ]


class ColocatedSummary(C.Structure):
    """colo_colocated_summary: MetricsReport fields (metrics.hpp:17-44) + replay extras."""

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
        ("tpt_sum", C.c_uint64 * 3),
        ("flags", C.c_uint64),
    ]


class ColocatedOpts(C.Structure):
    _fields_ = [
        ("cache_timeout", C.c_double),
        ("d_label_delay", C.c_void_p),
        ("default_label_delay", C.c_double),
        ("tau", C.c_double),
        ("d_samples", C.c_void_p),
        ("d_sample_offsets", C.c_void_p),
        ("d_labels", C.c_void_p),
        ("d_batches", C.c_void_p),
        ("d_summary", C.c_void_p),
        ("d_hist", C.c_void_p),
        ("nfilters", C.c_uint32),
        ("hist_shift", C.c_uint32),
        ("filter_shift", C.c_uint32),
        ("seg_len", C.c_uint32),
        ("filter_prefix", C.c_uint64 * 3),
        ("d_dev_sim_mode", C.c_void_p),
    ]


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


assert C.sizeof(Model) == 96 and C.sizeof(Gpu) == 32 and C.sizeof(Grid) == 48
assert C.sizeof(DeviceSummary) == 88
assert C.sizeof(ColocatedSummary) == 216

# Every symbol include/colo_abi.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "colo_ctx_create", "colo_ctx_destroy", "colo_ctx_set_stream", "colo_ctx_stream", "colo_sync",
    "colo_last_error", "colo_ctx_sm_count", "colo_abi_version", "colo_dev_alloc", "colo_dev_free",
    "colo_memcpy_h2d", "colo_memcpy_d2h", "colo_validate_profile_pair", "colo_profile_hash",
    "colo_validate_grid", "colo_mapset_build", "colo_mapset_from_cells", "colo_mapset_shape",
    "colo_mapset_cells", "colo_mapset_hash", "colo_mapset_destroy", "colo_decide", "colo_decide_exact",
    "colo_features_decide", "colo_features_decide_host", "colo_decide_host", "colo_features",
    "colo_validate_trace", "colo_replay_serving", "colo_hist_select", "colo_nearest_rank_index", "colo_serving_stats",
    "colo_generate_trace", "colo_synth_trace", "colo_synth_fleet_trace", "colo_synth_tuples", "colo_compare_verdicts",
    "colo_map_save", "colo_map_load", "colo_mapset_save", "colo_mapset_load", "colo_load_trace_jsonl",
    "colo_load_histogram_jsonl", "colo_replay_colocated", "colo_colocated_stats", "colo_trace_hash",
    "colo_sort_f64", "colo_json_doubles", "colo_ctx_release_scratch", "colo_ctx_share_temps", "colo_stats_allreduce",
    "colo_serving_stats_nccl", "colo_finalize", "colo_ctx_launches", "colo_colocated_events", "colo_events_text",
]


class MapHeader(C.Structure):
    _fields_ = [("kind", C.c_int), ("mode", C.c_int), ("profile_hash", C.c_uint64), ("num_layers", C.c_uint64),
                ("grid", Grid), ("assumed_output_tokens", C.c_uint64)]

_lib = None


def lib() -> C.CDLL:
    """Load the library (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` or `make`")
    L = C.CDLL(LIB_PATH)
    vp, sz, u64, i32, dbl = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int, C.c_double
    MP, GP, GRP = C.POINTER(Model), C.POINTER(Gpu), C.POINTER(Grid)
    sig = {
        "colo_ctx_create": (i32, [i32, C.POINTER(vp)]),
        "colo_ctx_destroy": (None, [vp]),
        "colo_ctx_set_stream": (i32, [vp, vp]),
        "colo_ctx_stream": (vp, [vp]),
        "colo_sync": (i32, [vp]),
        "colo_ctx_release_scratch": (i32, [vp]),
        "colo_ctx_share_temps": (i32, [vp, vp]),
        "colo_stats_allreduce": (i32, [vp, vp, vp, sz]),
        "colo_serving_stats_nccl": (i32, [vp, vp, MP, GP, sz, vp, vp, vp, sz, vp, vp, sz, dbl, vp,
                                         C.POINTER(DeviceSummary)]),
        "colo_last_error": (C.c_char_p, [vp]),
        "colo_ctx_sm_count": (i32, [vp]),
        "colo_abi_version": (i32, []),
        "colo_dev_alloc": (i32, [vp, sz, C.POINTER(vp)]),
        "colo_dev_free": (i32, [vp, vp]),
        "colo_memcpy_h2d": (i32, [vp, vp, vp, sz]),
        "colo_memcpy_d2h": (i32, [vp, vp, vp, sz]),
        "colo_validate_profile_pair": (i32, [MP, GP]),
        "colo_profile_hash": (u64, [MP, GP]),
        "colo_validate_grid": (i32, [GRP]),
        "colo_mapset_build": (i32, [vp, MP, GP, GRP, i32, u64, u64, u64, C.POINTER(vp)]),
        "colo_mapset_from_cells": (i32, [vp, MP, GP, GRP, i32, u64, u64, u64, u64, vp, sz, vp, sz, C.POINTER(vp)]),
        "colo_mapset_shape": (i32, [vp, C.POINTER(sz), C.POINTER(sz)]),
        "colo_mapset_cells": (i32, [vp, vp, vp, sz, vp, sz]),
        "colo_mapset_hash": (u64, [vp]),
        "colo_mapset_destroy": (None, [vp]),
        "colo_decide": (i32, [vp, vp, vp, sz, vp, vp]),
        "colo_decide_exact": (i32, [vp, MP, GP, i32, u64, vp, sz, vp, vp]),
        "colo_features_decide": (i32, [vp, vp, sz, vp, vp, sz, vp, vp, sz, vp, vp]),
        "colo_features_decide_host": (i32, [vp, vp, sz, vp, vp, sz, vp, vp, sz, vp, vp]),
        "colo_decide_host": (i32, [vp, vp, vp, sz, vp, vp]),
        "colo_features": (i32, [vp, MP, i32, vp, vp, sz, vp, vp, vp]),
        "colo_validate_trace": (i32, [vp, vp, vp, vp, vp, vp, sz, vp, sz]),
        "colo_replay_serving": (i32, [vp, MP, GP, sz, vp, vp, vp, sz, vp, vp, sz, C.POINTER(ReplayOpts)]),
        "colo_hist_select": (i32, [vp, sz, u64, C.POINTER(C.c_uint32), C.POINTER(u64)]),
        "colo_nearest_rank_index": (u64, [dbl, u64]),
        "colo_serving_stats": (i32, [vp, MP, GP, sz, vp, vp, vp, sz, vp, vp, sz, dbl, vp, C.POINTER(DeviceSummary)]),
        "colo_generate_trace": (C.c_int64, [dbl, dbl, C.POINTER(Dist), C.POINTER(Dist), u64, vp, vp, vp, vp, sz]),
        "colo_trace_hash": (u64, [vp, vp, vp, vp, vp, sz]),
        "colo_sort_f64": (i32, [vp, vp, vp, sz]),
        "colo_finalize": (i32, [vp, vp, sz, vp, vp]),
        "colo_ctx_launches": (u64, [vp]),
        "colo_colocated_events": (C.c_int64, [vp, vp, i32, dbl, vp, vp, vp, vp, dbl, vp, sz, dbl]),
        "colo_events_text": (C.c_int64, [vp, C.c_char_p, sz]),
        "colo_json_doubles": (C.c_int64, [vp, sz, C.c_char_p, sz]),
        "colo_replay_colocated": (i32, [vp, vp, sz, vp, vp, vp, sz, vp, vp, sz, C.POINTER(ColocatedOpts)]),
        "colo_colocated_stats": (i32, [vp, vp, sz, vp, vp, vp, sz, vp, vp, sz, C.POINTER(ColocatedOpts), vp,
                                       C.POINTER(ColocatedSummary)]),
        "colo_synth_trace": (i32, [vp, vp, vp, sz, vp, vp, vp, dbl, sz, u64, vp, vp, vp]),
        "colo_synth_fleet_trace": (i32, [vp, vp, vp, sz, vp, vp, vp, dbl, sz, vp, u64, vp, vp, vp]),
        "colo_synth_tuples": (i32, [vp, u64, sz, C.c_uint32, vp, vp, sz, vp]),
        "colo_compare_verdicts": (i32, [vp, vp, vp, sz, C.c_uint32, vp]),
        "colo_map_save": (i32, [C.c_char_p, C.POINTER(MapHeader), vp, sz]),
        "colo_map_load": (i32, [C.c_char_p, u64, C.POINTER(MapHeader), vp, sz, C.POINTER(sz), C.c_char_p, sz]),
        "colo_mapset_save": (i32, [vp, vp, C.c_char_p, C.c_char_p]),
        "colo_mapset_load": (i32, [vp, MP, GP, C.c_char_p, C.c_char_p, C.POINTER(vp)]),
        "colo_load_trace_jsonl": (C.c_int64, [C.c_char_p, vp, vp, vp, vp, vp, sz, C.c_char_p, sz]),
        "colo_load_histogram_jsonl": (C.c_int64, [C.c_char_p, vp, vp, sz, C.c_char_p, sz]),
    }
    variant = bool(os.environ.get("COLO_B200_LIB"))  # an older build variant may lack newer entry points
    for name, (res, args) in sig.items():
        if variant and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int, ctx=None, what: str = "") -> None:
    if status == COLO_OK:
        return
    detail = what
    if ctx is not None:
        msg = lib().colo_last_error(ctx)
        if msg:
            detail = f"{what}: {msg.decode()}" if what else msg.decode()
    if status == COLO_EVALIDATION:
        raise ColoValidationError(status, detail)
    if status == COLO_EINVAL:
        raise ColoInvalidArgument(status, detail)
    if status == COLO_EBREACH:
        raise ColoBreachError(status, detail)
    raise ColoError(status, detail)
