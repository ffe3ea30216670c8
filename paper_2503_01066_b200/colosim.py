"""Host-side mirror of the colosim C++ API for the admission hot path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/colosim/*.hpp, cited per symbol); the work runs
in ``libcolo_b200.so`` (sm_100a) through the C-ABI of ``include/colo_abi.h``.
Device buffers are torch CUDA tensors (plumbing only); every computation on
them is one of this package's kernels.  There is no CPU fallback: without the
built library or without a GPU the calls raise.

Reference exceptions map to Python exceptions:
  std::runtime_error (validation)   -> ColoValidationError (ValueError subclass)
  std::invalid_argument (contract)  -> ColoInvalidArgument (ValueError subclass)
  std::nullopt (out-of-range map)   -> None from lookup(); *_OOR bits in verdicts
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import ColoBreachError, ColoError, ColoInvalidArgument, ColoValidationError, HIST_BINS, NCOUNTERS, check, lib

KIB, MIB, GIB = 1024, 1024**2, 1024**3
KB, MB, GB = 1000, 1000**2, 1000**3


# ------------------------------------------------------------------ enums
class TrainingMode(enum.IntEnum):
    """maps.hpp:16"""

    CPT = 0
    CPA = 1


class OffloadAction(enum.IntEnum):
    """maps.hpp:32 (values are the verdict-word encoding)"""

    NoAction = 0
    FreeLayers = 1
    AllToHost = 2


class HedgeDecision(enum.IntEnum):
    """maps.hpp:254"""

    LoadBack = 0
    Recompute = 1


class Verdict(enum.IntEnum):
    """Outcome of engine.hpp:513-557."""

    ADMIT = 0
    FREE_LOADBACK = 1
    RECOMPUTE_DROP = 2


COUNTER_NAMES = ["admit", "free_loadback", "recompute_drop", "offload_oor", "hedge_oor", "stream", "stream_oor", "total"]


@dataclass(frozen=True)
class OffloadDecision:
    """maps.hpp:34-49"""

    action: OffloadAction = OffloadAction.NoAction
    layers: int = 0

    def layers_to_free(self, num_layers: int) -> int:
        if self.action == OffloadAction.NoAction:
            return 0
        if self.action == OffloadAction.FreeLayers:
            return self.layers
        return num_layers


# --------------------------------------------------------------- profiles
@dataclass
class ModelProfile:
    """profiles.hpp:23-35 (defaults = the Llama-8B-like profile)."""

    num_layers: int = 32
    kv_bytes_per_token: int = 512 * KIB
    act_bytes_per_token_per_layer: int = 417000
    prefill_coef_linear: float = 1e-4
    prefill_coef_quad: float = 2e-8
    decode_coef_const: float = 0.020
    decode_coef_context: float = 2e-6
    backward_to_forward_ratio: float = 1.326
    record_prefill_multiplier: float = 1.21
    record_decode_multiplier: float = 1.35
    workspace_factor: float = 1.0
    weights_bytes: int = 16 * GIB

    def to_c(self) -> _lib.Model:
        return _lib.Model(*[getattr(self, f.name) for f in dataclasses.fields(self)])

    @staticmethod
    def mistral7b_like() -> "ModelProfile":
        """profiles.hpp:85"""
        return ModelProfile()

    @staticmethod
    def phi14b_like() -> "ModelProfile":
        """profiles.hpp:88-95"""
        return ModelProfile(num_layers=40, kv_bytes_per_token=838861, act_bytes_per_token_per_layer=667200,
                            weights_bytes=24 * GIB)

    @staticmethod
    def from_kv_text(text: str) -> "ModelProfile":
        """profiles.hpp:59-75 over a flat `key = value` text (kvfile.hpp)."""
        kv = _parse_kv(text)
        m = ModelProfile()
        for f in dataclasses.fields(m):
            if f.name not in kv:
                raise ColoValidationError(_lib.COLO_EVALIDATION, f"missing key: {f.name}")
            setattr(m, f.name, int(float(kv.pop(f.name))) if f.type in ("int", int) else float(kv.pop(f.name)))
        if kv:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"unknown key: {sorted(kv)[0]}")
        return m


@dataclass
class GpuProfile:
    """profiles.hpp:98-102"""

    capacity_bytes: int = 80 * GIB
    h2d_bandwidth: int = 24 * GB
    d2h_bandwidth: int = 24 * GB
    runtime_reserve_bytes: int = 2 * GIB

    def to_c(self) -> _lib.Gpu:
        return _lib.Gpu(self.capacity_bytes, self.h2d_bandwidth, self.d2h_bandwidth, self.runtime_reserve_bytes)


@dataclass
class GridSteps:
    """maps.hpp:63-67"""

    cached_token_step: int = 500
    incoming_token_step: int = 500
    batch_step: int = 5


@dataclass
class GridBounds:
    """maps.hpp:69-73"""

    max_cached_tokens: int = 8000
    max_incoming_tokens: int = 8000
    max_batch: int = 50


def _grid(steps: GridSteps, bounds: GridBounds) -> _lib.Grid:
    return _lib.Grid(steps.cached_token_step, steps.incoming_token_step, steps.batch_step,
                     bounds.max_cached_tokens, bounds.max_incoming_tokens, bounds.max_batch)


def _parse_kv(text: str) -> dict:
    out = {}
    for ln in text.splitlines():
        ln = ln.split("#", 1)[0].strip()
        if not ln:
            continue
        k, _, v = ln.partition("=")
        k, v = k.strip(), v.strip()
        if k in out:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"duplicate key: {k}")
        out[k] = v
    return out


def validate_profile_pair(m: ModelProfile, g: GpuProfile) -> None:
    """profiles.hpp:129-134 (raises ColoValidationError)."""
    check(lib().colo_validate_profile_pair(C.byref(m.to_c()), C.byref(g.to_c())), None,
          "profile pair rejected: invalid profile or weights + runtime reserve >= device capacity")


def profile_hash(m: ModelProfile, g: GpuProfile) -> int:
    """profiles.hpp:137-152"""
    return int(lib().colo_profile_hash(C.byref(m.to_c()), C.byref(g.to_c())))


def validate_grid(steps: GridSteps, bounds: GridBounds) -> None:
    """maps.hpp:197-208"""
    check(lib().colo_validate_grid(C.byref(_grid(steps, bounds))), None, "map grid rejected")


# ---------------------------------------------------------------- context
def _torch():
    import torch

    return torch


class Context:
    """One colo_ctx per GPU (and per host thread).  Launches go to the torch
    current stream at creation time unless ``stream`` is given."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise ColoError(_lib.COLO_ECUDA, "no CUDA device: colo-b200 has no CPU path")
        self.device = device
        torch.cuda.set_device(device)
        h = C.c_void_p()
        check(lib().colo_ctx_create(device, C.byref(h)), None, f"colo_ctx_create({device})")
        self.h = h
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.torch_stream = s
        check(lib().colo_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream)), self.h)

    @property
    def sm_count(self) -> int:
        return lib().colo_ctx_sm_count(self.h)

    def launches(self) -> int:
        """Kernels this context launched so far (colo_ctx_launches)."""
        return int(lib().colo_ctx_launches(self.h))

    def sync(self) -> None:
        check(lib().colo_sync(self.h), self.h)

    def release_scratch(self) -> None:
        """Free the context's grow-only device scratch (colo_ctx_release_scratch)."""
        check(lib().colo_ctx_release_scratch(self.h), self.h)

    def share_temps(self, owner: "Context") -> None:
        """Use ``owner``'s per-call replay temporaries (colo_ctx_share_temps):
        chunk contexts of one rank keep their own pass state but share the
        first pass's transient buffers."""
        self._temps_owner = owner  # keep the owner alive while borrowed
        check(lib().colo_ctx_share_temps(self.h, owner.h if owner is not None else None), self.h)

    def close(self) -> None:
        if getattr(self, "h", None):
            lib().colo_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _need_cuda(t, name: str, dtype_bytes: int):
    if t is None:
        return
    if not t.is_cuda:
        raise ColoInvalidArgument(_lib.COLO_EINVAL, f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ColoInvalidArgument(_lib.COLO_EINVAL, f"{name} must be contiguous")
    if t.element_size() != dtype_bytes:
        raise ColoInvalidArgument(_lib.COLO_EINVAL, f"{name} must have {dtype_bytes}-byte elements")


# ---------------------------------------------------------------- map sets
class MapSet:
    """Device-resident offloading map + hedging map of one (model, gpu, grid,
    mode) -- what experiment.hpp:139-152 calls BuiltMaps."""

    def __init__(self, ctx: Context, h, model: ModelProfile, gpu: GpuProfile, steps: GridSteps, bounds: GridBounds,
                 mode: TrainingMode, hedge_step: int, hedge_max: int, assumed_output_tokens: int):
        self.ctx, self.h = ctx, h
        self.model, self.gpu, self.steps, self.bounds = model, gpu, steps, bounds
        self.mode = TrainingMode(mode)
        self.hedge_step, self.hedge_max, self.assumed_output_tokens = hedge_step, hedge_max, assumed_output_tokens
        self.profile_hash_value = int(lib().colo_mapset_hash(h))
        self._cells = None

    @classmethod
    def build(cls, ctx: Context, model: ModelProfile, gpu: GpuProfile, steps: GridSteps = None,
              bounds: GridBounds = None, mode: TrainingMode = TrainingMode.CPA, hedge_step: Optional[int] = None,
              hedge_max: Optional[int] = None, assumed_output_tokens: int = 128) -> "MapSet":
        steps = steps or GridSteps()
        bounds = bounds or GridBounds()
        hs = steps.cached_token_step if hedge_step is None else hedge_step
        hm = bounds.max_cached_tokens if hedge_max is None else hedge_max
        h = C.c_void_p()
        check(lib().colo_mapset_build(ctx.h, C.byref(model.to_c()), C.byref(gpu.to_c()), C.byref(_grid(steps, bounds)),
                                      int(mode), hs, hm, assumed_output_tokens, C.byref(h)), ctx.h, "map build")
        return cls(ctx, h, model, gpu, steps, bounds, mode, hs, hm, assumed_output_tokens)

    @classmethod
    def from_cells(cls, ctx: Context, model: ModelProfile, gpu: GpuProfile, steps: GridSteps, bounds: GridBounds,
                   mode: TrainingMode, hedge_step: int, hedge_max: int, assumed_output_tokens: int, built_hash: int,
                   offload_cells: np.ndarray, hedge_cells: np.ndarray) -> "MapSet":
        off = np.ascontiguousarray(offload_cells, np.uint8)
        hed = np.ascontiguousarray(hedge_cells, np.uint8)
        h = C.c_void_p()
        check(lib().colo_mapset_from_cells(ctx.h, C.byref(model.to_c()), C.byref(gpu.to_c()),
                                           C.byref(_grid(steps, bounds)), int(mode), hedge_step, hedge_max,
                                           assumed_output_tokens, built_hash, off.ctypes.data, off.size,
                                           hed.ctypes.data, hed.size, C.byref(h)), ctx.h, "map load")
        return cls(ctx, h, model, gpu, steps, bounds, mode, hedge_step, hedge_max, assumed_output_tokens)

    def cells(self) -> Tuple[np.ndarray, np.ndarray]:
        """(offload codes, hedge bits) copied back from the device."""
        if self._cells is None:
            a, b = C.c_size_t(), C.c_size_t()
            check(lib().colo_mapset_shape(self.h, C.byref(a), C.byref(b)))
            off = np.zeros(a.value, np.uint8)
            hed = np.zeros(b.value, np.uint8)
            check(lib().colo_mapset_cells(self.ctx.h, self.h, off.ctypes.data, off.size, hed.ctypes.data, hed.size),
                  self.ctx.h)
            self._cells = (off, hed)
        return self._cells

    @property
    def offload(self) -> "OffloadingMap":
        return OffloadingMap(self)

    @property
    def hedge(self) -> "HedgingMap":
        return HedgingMap(self)

    def close(self):
        if getattr(self, "h", None):
            lib().colo_mapset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decode_cell(code: int) -> OffloadDecision:
    if code == 0:
        return OffloadDecision(OffloadAction.NoAction, 0)
    if code == 1:
        return OffloadDecision(OffloadAction.AllToHost, 0)
    return OffloadDecision(OffloadAction.FreeLayers, int(code) - 2)


def round_up_bucket(value: int, step: int) -> int:
    """maps.hpp:28-30"""
    return (value + step - 1) // step * step


class OffloadingMap:
    """maps.hpp:77-195, as a view of a device-built MapSet.  Scalar lookup()
    indexes the GPU-built cells; batched decisions go through decide()."""

    def __init__(self, ms: MapSet):
        self.ms = ms
        self.steps, self.bounds, self.mode = ms.steps, ms.bounds, ms.mode
        self.profile_hash_value = ms.profile_hash_value
        self.num_layers = ms.model.num_layers

    def cached_count(self) -> int:
        return self.bounds.max_cached_tokens // self.steps.cached_token_step + 1

    def incoming_count(self) -> int:
        return self.bounds.max_incoming_tokens // self.steps.incoming_token_step

    def batch_count(self) -> int:
        return self.bounds.max_batch // self.steps.batch_step

    def cell(self, ci: int, ii: int, bi: int) -> OffloadDecision:
        off, _ = self.ms.cells()
        return decode_cell(off[(ci * self.incoming_count() + ii) * self.batch_count() + bi])

    def lookup(self, cached: int, incoming: int, batch: int) -> Optional[OffloadDecision]:
        s, b = self.steps, self.bounds
        cb = round_up_bucket(cached, s.cached_token_step)
        ib = round_up_bucket(incoming, s.incoming_token_step)
        bb = round_up_bucket(batch, s.batch_step)
        if cb > b.max_cached_tokens or ib > b.max_incoming_tokens or bb > b.max_batch:
            return None
        if incoming == 0 or batch == 0:
            return None
        return self.cell(cb // s.cached_token_step, ib // s.incoming_token_step - 1, bb // s.batch_step - 1)

    def cached_bucket_value(self, ci: int) -> int:
        return ci * self.steps.cached_token_step

    def incoming_bucket_value(self, ii: int) -> int:
        return (ii + 1) * self.steps.incoming_token_step

    def batch_bucket_value(self, bi: int) -> int:
        return (bi + 1) * self.steps.batch_step

    def save(self, path: str) -> None:
        """maps.hpp:118-140 text format (colo_map_save)."""
        save_map_cells(path, "offload", self.mode, self.profile_hash_value, self.num_layers, self.steps, self.bounds,
                       self.ms.cells()[0])


class HedgingMap:
    """maps.hpp:257-336, as a view of a device-built MapSet."""

    def __init__(self, ms: MapSet):
        self.ms = ms
        self.cached_token_step = ms.hedge_step
        self.max_cached_tokens = ms.hedge_max
        self.num_layers = ms.model.num_layers
        self.mode = ms.mode
        self.assumed_output_tokens = ms.assumed_output_tokens
        self.profile_hash_value = ms.profile_hash_value

    def cached_count(self) -> int:
        return self.max_cached_tokens // self.cached_token_step

    def freed_count(self) -> int:
        return self.num_layers + 1

    def cell(self, ci: int, fi: int) -> HedgeDecision:
        _, hed = self.ms.cells()
        return HedgeDecision(int(hed[ci * self.freed_count() + fi]))

    def lookup(self, cached: int, freed_layers: int) -> Optional[HedgeDecision]:
        cb = round_up_bucket(cached, self.cached_token_step)
        if cb == 0 or cb > self.max_cached_tokens or freed_layers > self.num_layers:
            return None
        return self.cell(cb // self.cached_token_step - 1, freed_layers)

    def cached_bucket_value(self, ci: int) -> int:
        return (ci + 1) * self.cached_token_step

    def save(self, path: str) -> None:
        """maps.hpp:284-295 text format (colo_map_save)."""
        save_map_cells(path, "hedge", self.mode, self.profile_hash_value, self.num_layers,
                       GridSteps(self.cached_token_step, 1, 1), GridBounds(self.max_cached_tokens, 1, 1),
                       self.ms.cells()[1], self.assumed_output_tokens)


@dataclass
class BuiltMaps:
    """experiment.hpp:139-142"""

    offload: OffloadingMap
    hedge: HedgingMap
    mapset: MapSet


def build_maps(ctx: Context, m: ModelProfile, g: GpuProfile, steps: GridSteps = None, bounds: GridBounds = None,
               mode: TrainingMode = TrainingMode.CPA, assumed_output_tokens: int = 128) -> BuiltMaps:
    """experiment.hpp:144-152 (both maps built on the GPU)."""
    ms = MapSet.build(ctx, m, g, steps, bounds, mode, None, None, assumed_output_tokens)
    return BuiltMaps(ms.offload, ms.hedge, ms)


def build_offloading_map(ctx: Context, m: ModelProfile, g: GpuProfile, steps: GridSteps, bounds: GridBounds,
                         mode: TrainingMode) -> OffloadingMap:
    """maps.hpp:233-252"""
    return MapSet.build(ctx, m, g, steps, bounds, mode).offload


def build_hedging_map(ctx: Context, m: ModelProfile, g: GpuProfile, cached_step: int, max_cached: int,
                      mode: TrainingMode, assumed_output_tokens: int = 128) -> HedgingMap:
    """maps.hpp:358-384"""
    steps = GridSteps(cached_step, cached_step, 1)
    bounds = GridBounds(max_cached, cached_step, 1)
    return MapSet.build(ctx, m, g, steps, bounds, mode, cached_step, max_cached, assumed_output_tokens).hedge


# ------------------------------------------------------------- tuples
TUPLE_DTYPE = np.dtype([("cached", "<u4"), ("incoming", "<u4"), ("charged", "<u4"), ("batch", "<u2"),
                        ("pending", "u1"), ("dev_layers", "u1")])


def pack_tuples(cached, incoming, charged, batch, pending, dev_layers):
    """colo_tuple records as an int32 [n, 4] torch tensor (any device)."""
    torch = _torch()
    w = (batch.to(torch.int64) & 0xFFFF) | ((pending.to(torch.int64) & 0xFF) << 16) | ((dev_layers.to(torch.int64) & 0xFF) << 24)
    w = torch.where(w >= 2**31, w - 2**32, w)
    return torch.stack([cached.to(torch.int32), incoming.to(torch.int32), charged.to(torch.int32), w.to(torch.int32)], 1).contiguous()


def verdict_fields(v: np.ndarray) -> dict:
    """Decode packed verdict words (include/colo_abi.h)."""
    v = np.asarray(v).astype(np.uint32)
    return {
        "action": v & 3, "layers": (v >> 2) & 0xFF, "free_now": (v >> 10) & 0xFF, "recompute": (v >> 18) & 1,
        "offload_oor": (v >> 19) & 1, "hedge_oor": (v >> 20) & 1, "verdict": (v >> 21) & 3, "stream": (v >> 23) & 1,
        "stream_oor": (v >> 24) & 1,
    }


def _counters_tensor(counters, device):
    torch = _torch()
    if counters is None:
        return None
    if counters is True:
        return torch.zeros(NCOUNTERS, dtype=torch.int64, device=device)
    return counters


def decide(ctx: Context, maps, tuples, out=None, counters=None):
    """Quantised verdicts for colo_tuple records (int32 [n,4] CUDA tensor).
    maps: BuiltMaps or MapSet.  counters: None, True (allocate) or an int64[8] tensor (accumulated)."""
    torch = _torch()
    ms = maps.mapset if isinstance(maps, BuiltMaps) else maps
    _need_cuda(tuples, "tuples", 4)
    n = tuples.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=tuples.device)
    cnt = _counters_tensor(counters, tuples.device)
    check(lib().colo_decide(ctx.h, ms.h, _ptr(tuples), n, _ptr(out), _ptr(cnt)), ctx.h, "decide")
    return (out, cnt) if counters is not None else out


def decide_exact(ctx: Context, m: ModelProfile, g: GpuProfile, mode: TrainingMode, tuples, out=None, counters=None,
                 assumed_output_tokens: int = 128):
    """Exact (un-quantised) verdicts, maps.hpp:215-231 + 341-356 per tuple."""
    torch = _torch()
    _need_cuda(tuples, "tuples", 4)
    n = tuples.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=tuples.device)
    cnt = _counters_tensor(counters, tuples.device)
    check(lib().colo_decide_exact(ctx.h, C.byref(m.to_c()), C.byref(g.to_c()), int(mode), assumed_output_tokens,
                                  _ptr(tuples), n, _ptr(out), _ptr(cnt)), ctx.h, "decide_exact")
    return (out, cnt) if counters is not None else out


def _sets_array(sets: Sequence[MapSet]):
    arr = (C.c_void_p * len(sets))(*[s.h.value for s in sets])
    return arr


def features_decide(ctx: Context, sets: Sequence[MapSet], prompt, output, dev_offsets, dev_set, out=None,
                    counters=None):
    """Trace-fused features -> verdicts (SURVEY §8(d) C2 rule).  prompt/output:
    int32 CUDA tensors; dev_offsets int64 [ndev+1]; dev_set int16 [ndev]."""
    torch = _torch()
    for t, nm, b in ((prompt, "prompt", 4), (output, "output", 4), (dev_offsets, "dev_offsets", 8), (dev_set, "dev_set", 2)):
        _need_cuda(t, nm, b)
    n = prompt.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=prompt.device)
    cnt = _counters_tensor(counters, prompt.device)
    arr = _sets_array(sets)
    check(lib().colo_features_decide(ctx.h, arr, len(sets), _ptr(prompt), _ptr(output), n, _ptr(dev_offsets),
                                     _ptr(dev_set), dev_set.shape[0], _ptr(out), _ptr(cnt)), ctx.h, "features_decide")
    return (out, cnt) if counters is not None else out


def features_decide_host(ctx: Context, sets: Sequence[MapSet], prompt: np.ndarray, output: np.ndarray,
                         dev_offsets: np.ndarray, dev_set: np.ndarray, out: Optional[np.ndarray] = None,
                         counters: bool = False):
    """Same over host buffers (numpy or pinned CPU torch tensors): the
    reference-facing call -- H2D, kernel and D2H are inside the call."""
    def addr(a):
        return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else C.c_void_p(a.ctypes.data)

    n = len(prompt)
    if out is None:
        out = np.empty(n, np.uint32)
    cnt = np.zeros(NCOUNTERS, np.uint64) if counters else None
    offs = np.ascontiguousarray(dev_offsets, np.uint64)
    dset = np.ascontiguousarray(dev_set, np.uint16)
    arr = _sets_array(sets)
    check(lib().colo_features_decide_host(ctx.h, arr, len(sets), addr(prompt), addr(output), n, offs.ctypes.data,
                                          dset.ctypes.data, len(dset), addr(out),
                                          cnt.ctypes.data if cnt is not None else None), ctx.h, "features_decide_host")
    return (out, cnt) if counters else out


def decide_host(ctx: Context, maps, tuples: np.ndarray, out: Optional[np.ndarray] = None, counters: bool = False):
    ms = maps.mapset if isinstance(maps, BuiltMaps) else maps
    t = np.ascontiguousarray(tuples, TUPLE_DTYPE)
    if out is None:
        out = np.empty(len(t), np.uint32)
    cnt = np.zeros(NCOUNTERS, np.uint64) if counters else None
    check(lib().colo_decide_host(ctx.h, ms.h, t.ctypes.data, len(t), out.ctypes.data,
                                 cnt.ctypes.data if cnt is not None else None), ctx.h, "decide_host")
    return (out, cnt) if counters else out


def features(ctx: Context, m: ModelProfile, mode: TrainingMode, prompt, output):
    """(need u64, charged u64, prefill f64) per query (int64/int64/float64 tensors)."""
    torch = _torch()
    _need_cuda(prompt, "prompt", 4)
    _need_cuda(output, "output", 4)
    n = prompt.shape[0]
    need = torch.empty(n, dtype=torch.int64, device=prompt.device)
    charged = torch.empty(n, dtype=torch.int64, device=prompt.device)
    prefill = torch.empty(n, dtype=torch.float64, device=prompt.device)
    check(lib().colo_features(ctx.h, C.byref(m.to_c()), int(mode), _ptr(prompt), _ptr(output), n, _ptr(need),
                              _ptr(charged), _ptr(prefill)), ctx.h, "features")
    return need, charged, prefill


# ------------------------------------------------------------- replay
BATCH_DTYPE = np.dtype([("start", "<f8"), ("end", "<f8"), ("first", "<u4"), ("n", "<u4"), ("need_total", "<u8"),
                        ("max_incoming", "<u4"), ("verdict", "<u4")])


def _profiles_arrays(profiles: Sequence[Tuple[ModelProfile, GpuProfile]]):
    ms = (_lib.Model * len(profiles))(*[p[0].to_c() for p in profiles])
    gs = (_lib.Gpu * len(profiles))(*[p[1].to_c() for p in profiles])
    return ms, gs


def validate_trace(ctx: Context, arrival, prompt, output, dev_offsets, query_id=None, label_delay=None) -> None:
    """validate_trace (workload.hpp:164-188) in place on device tensors: every
    device's rows ordered by (arrival, query_id) across all given columns;
    raises ColoValidationError (the reference's message) for a negative
    arrival, zero tokens or a repeated query_id within a device."""
    _need_cuda(arrival, "arrival", 8)
    _need_cuda(prompt, "prompt", 4)
    _need_cuda(output, "output", 4)
    _need_cuda(dev_offsets, "dev_offsets", 8)
    _need_cuda(query_id, "query_id", 8)
    _need_cuda(label_delay, "label_delay", 8)
    check(lib().colo_validate_trace(ctx.h, _ptr(query_id), _ptr(arrival), _ptr(prompt), _ptr(output),
                                    _ptr(label_delay), prompt.shape[0], _ptr(dev_offsets), dev_offsets.shape[0] - 1),
          ctx.h, "validate_trace")


def replay_serving(ctx: Context, profiles: Sequence[Tuple[ModelProfile, GpuProfile]], arrival, prompt, output,
                   dev_offsets, dev_profile, tau: float = math.inf, sets: Optional[Sequence[MapSet]] = None,
                   samples: bool = False, labels: bool = True, batches: bool = False, summary: bool = True,
                   hist=None, hist_shift: int = 42, filter_shift: int = 63, filter_prefix=(0,), segment_len: int = 0,
                   reuse_entries: bool = False, stats_mode: int = 0, verdicts=None):
    """Serving-only replay of every device (engine.hpp:140-387, SimMode::ServingOnly).
    Returns a dict of device tensors: samples (f64, reference order),
    labels (u8 per query), batches (raw bytes, BATCH_DTYPE), summary (DeviceSummary bytes),
    verdicts (u32 per batch: device d's batch b at dev_offsets[d] + b; needs ``sets``;
    ``verdicts`` may be True or a caller-owned int32 tensor of n words)."""
    torch = _torch()
    dev = prompt.device
    _need_cuda(arrival, "arrival", 8)
    _need_cuda(prompt, "prompt", 4)
    _need_cuda(output, "output", 4)
    _need_cuda(dev_offsets, "dev_offsets", 8)
    _need_cuda(dev_profile, "dev_profile", 2)
    n = prompt.shape[0]
    ndev = dev_profile.shape[0]
    res = {}
    opts = _lib.ReplayOpts()
    opts.tau = tau
    opts.segment_len = segment_len
    opts.reuse_entries = 1 if reuse_entries else 0
    opts.stats_mode = int(stats_mode)  # 1: record per-batch sample-bin ranges; 2: sparse narrowing pass
    keep = []
    if sets is not None:
        arr = _sets_array(sets)
        keep.append(arr)
        opts.sets = C.cast(arr, C.c_void_p)
    if samples:
        per_dev = torch.zeros(ndev + 1, dtype=torch.int64, device=dev)
        o64 = output.to(torch.int64)
        cs = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(o64, 0)])
        per_dev = cs[dev_offsets]
        total = int(per_dev[-1].item())
        res["samples"] = torch.empty(max(total, 1), dtype=torch.float64, device=dev)[:total]
        res["sample_offsets"] = per_dev.contiguous()
        opts.d_samples = res["samples"].data_ptr() if total else torch.empty(1, dtype=torch.float64, device=dev).data_ptr()
        opts.d_sample_offsets = res["sample_offsets"].data_ptr()
    if labels:
        res["labels"] = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)[:n]
        opts.d_labels = res["labels"].data_ptr() if n else 0
    if batches:
        res["batches"] = torch.zeros((max(n, 1), BATCH_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        opts.d_batches = res["batches"].data_ptr()
    if verdicts is not None and verdicts is not False:
        if sets is None:
            raise ColoError(_lib.COLO_EINVAL, "replay-derived verdicts need map sets")
        if verdicts is True:
            verdicts = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)[:n]
        _need_cuda(verdicts, "verdicts", 4)
        if verdicts.shape[0] < n:
            raise ColoError(_lib.COLO_EINVAL, "verdicts buffer shorter than the trace")
        res["verdicts"] = verdicts
        opts.d_verdicts = verdicts.data_ptr() if n else 0
    if summary:
        res["summary"] = torch.zeros((ndev, C.sizeof(_lib.DeviceSummary)), dtype=torch.uint8, device=dev)
        opts.d_summary = res["summary"].data_ptr()
    if hist is not None:
        opts.d_hist = hist.data_ptr()
        opts.nfilters = len(filter_prefix)
        opts.hist_shift = hist_shift
        opts.filter_shift = filter_shift
        for i, p in enumerate(filter_prefix):
            opts.filter_prefix[i] = int(p)
    ms, gs = _profiles_arrays(profiles)
    check(lib().colo_replay_serving(ctx.h, ms, gs, len(profiles), _ptr(arrival), _ptr(prompt), _ptr(output), n,
                                    _ptr(dev_offsets), _ptr(dev_profile), ndev, C.byref(opts)), ctx.h, "replay_serving")
    return res


def summaries_to_numpy(summary_bytes) -> np.ndarray:
    dt = np.dtype([("generated_tokens", "<u8"), ("slow_tokens", "<u8"), ("slow_queries", "<u8"), ("batches", "<u8"),
                   ("peak_device_bytes", "<u8"), ("max_batch_size", "<u8"), ("end_time", "<f8"),
                   ("tpt_sum", "<u8", (3,)), ("flags", "<u8")])
    a = summary_bytes.cpu().numpy() if hasattr(summary_bytes, "cpu") else np.asarray(summary_bytes)
    return np.ascontiguousarray(a).view(dt).reshape(-1)


def fixed_sum_value(limbs) -> Fraction:
    """Exact value of a 192-bit little-endian fixed-point TPT sum (LSB 2^-96)."""
    v = int(limbs[0]) | (int(limbs[1]) << 64) | (int(limbs[2]) << 128)
    return Fraction(v, 1 << 96)


def nearest_rank_index(q: float, n: int) -> int:
    """metrics.hpp:48-53: max(1, ceil(q * n)) with the reference's double arithmetic."""
    return int(lib().colo_nearest_rank_index(q, n))


def serving_stats(ctx: Context, profiles, arrival, prompt, output, dev_offsets, dev_profile, tau: float = math.inf,
                  group=None, quantiles=(0.50, 0.90, 0.99)):
    """Exact nearest-rank TPT percentiles + mean over all devices (finalize,
    metrics.hpp:56-66) by three radix-select replay passes; with a
    torch.distributed ``group`` the histograms, counters and exact sums are
    all-reduced across ranks (each rank holds its own device shard)."""
    return fleet_stats([(ctx, arrival, prompt, output, dev_offsets, dev_profile)], profiles, tau, group, quantiles)


def fleet_stats(parts, profiles, tau: float = math.inf, group=None, quantiles=(0.50, 0.90, 0.99)):
    """serving_stats over a rank's devices held as several parts (chunks of
    devices, each with its own Context so its replay scratch -- segment entry
    states and the sparse passes' batch records -- survives between the three
    passes).  ``parts``: list of (ctx, arrival, prompt, output, dev_offsets,
    dev_profile); every pass replays every part into the same histogram, so
    the result equals one replay over the union of the parts' devices."""
    torch = _torch()
    dist = torch.distributed if (torch.distributed.is_available() and torch.distributed.is_initialized()) else None
    dev = parts[0][2].device
    hist = torch.zeros(len(quantiles) * HIST_BINS, dtype=torch.int64, device=dev)
    sparse = os.environ.get("COLO_SPARSE_STATS", "1") != "0"

    def run_pass(hist_shift, filter_shift, prefixes):
        h = hist[: len(prefixes) * HIST_BINS]
        h.zero_()
        first = filter_shift == 63
        tot = {"generated_tokens": 0, "slow_tokens": 0, "slow_queries": 0, "batches": 0, "flags": 0, "exact_sum": 0}
        for ctx, arrival, prompt, output, dev_offsets, dev_profile in parts:
            r = replay_serving(ctx, profiles, arrival, prompt, output, dev_offsets, dev_profile, tau=tau, labels=False,
                               summary=first, hist=h, hist_shift=hist_shift, filter_shift=filter_shift,
                               filter_prefix=tuple(prefixes), reuse_entries=not first,
                               stats_mode=(1 if first else 2) if sparse else 0)
            if not first:
                continue
            S = summaries_to_numpy(r["summary"])
            for k in ("generated_tokens", "slow_tokens", "slow_queries", "batches"):
                tot[k] += int(S[k].sum())
            tot["flags"] |= int(np.bitwise_or.reduce(S["flags"])) if len(S) else 0
            tot["exact_sum"] += sum(int(a) | (int(b) << 64) | (int(c) << 128) for a, b, c in S["tpt_sum"])
        return h, (tot if first else None)

    reduce = (lambda t: dist.all_reduce(t, group=group)) if dist is not None else None
    return stats_protocol(run_pass, reduce, quantiles)


FLAG_BITS = 8  # low flag bits OR-ed across ranks (bit 0: a sample outside the exact fixed-point sum's range)


def stats_protocol(run_pass, reduce=None, quantiles=(0.50, 0.90, 0.99)):
    """Exact nearest-rank selection over f64 bit patterns in three 21-bit
    radix passes (TPT samples are non-negative, so their bit patterns order
    like their values).  ``run_pass(hist_shift, filter_shift, prefixes)``
    returns (int64 histogram tensor [len(prefixes) * HIST_BINS], totals or
    None); ``reduce`` (e.g. a torch.distributed all_reduce) sums a tensor
    across ranks in place.  The mean is the exact fixed-point sum over n,
    correctly rounded (metrics.hpp:63-65 sums the sorted samples
    sequentially instead; the difference is bounded by that sum's rounding)."""
    torch = _torch()
    nf = len(quantiles)
    hist, tot = run_pass(42, 63, (0,))
    exact = tot["exact_sum"]
    # int64-safe all-reduce: counters, the exact sum as 32-bit chunks, and the
    # flag word OR-ed across ranks as per-bit counts (a sum-only reduction)
    fl = int(tot["flags"])
    vec = torch.tensor([tot["generated_tokens"], tot["slow_tokens"], tot["slow_queries"], tot["batches"]]
                       + [(exact >> (32 * i)) & 0xFFFFFFFF for i in range(8)]
                       + [(fl >> b) & 1 for b in range(FLAG_BITS)], dtype=torch.int64, device=hist.device)
    if reduce is not None:
        reduce(vec)
        reduce(hist)
    v = [int(x) for x in vec.cpu().tolist()]
    exact = sum(c << (32 * i) for i, c in enumerate(v[4:12]))
    flags = (fl & ~((1 << FLAG_BITS) - 1)) | sum(1 << b for b, c in enumerate(v[12:]) if c)
    n = v[0]
    out = {"generated_tokens": n, "slow_tokens": v[1], "slow_queries": v[2], "batches": v[3], "flags": flags,
           "exact_sum": exact}
    if n == 0:
        out.update({f"p{int(round(q * 100))}": None for q in quantiles})
        out["mean"] = None
        return out
    ranks = [nearest_rank_index(q, n) for q in quantiles]
    sel = _select_dev(hist.view(1, HIST_BINS).expand(nf, HIST_BINS).contiguous(), ranks)
    prefixes = []
    for f in range(nf):
        b, ranks[f] = sel[f]
        prefixes.append(b)
    for fs, hs in ((42, 21), (21, 0)):
        hist, _ = run_pass(hs, fs, tuple(prefixes))
        if reduce is not None:
            reduce(hist)
        sel = _select_dev(hist.view(nf, HIST_BINS), ranks)
        for f in range(nf):
            b, ranks[f] = sel[f]
            prefixes[f] = (prefixes[f] << 21) | b
    for q, p in zip(quantiles, prefixes):
        out[f"p{int(round(q * 100))}"] = float(np.array([p], np.uint64).view(np.float64)[0])
    out["mean"] = float(Fraction(exact, 1 << 96) / n)
    # bit 0/1: a sample below the sum's 2^-96 resolution or beyond its range on some rank -- the
    # exact-sum mean is then not exact (the percentiles and counters still are)
    out["mean_exact"] = not (flags & 3)
    return out


def _select_dev(h, ranks) -> List[Tuple[int, int]]:
    """For every row of an int64 histogram tensor [nf, bins] (bins a multiple
    of 1024), the first bin whose cumulative count reaches the row's rank and
    the rank inside it, computed where the histogram lives: block sums of 1024
    bins, their prefix, then the prefix inside the one block; two words per
    row come back to the host instead of the histogram."""
    torch = _torch()
    nf, nb = h.shape
    hb = h.reshape(nf, nb // 1024, 1024)
    csum = torch.cumsum(hb.sum(dim=2), dim=1)  # [nf, nb/1024]
    rk = torch.tensor(ranks, dtype=torch.int64, device=h.device).view(-1, 1)
    blk = torch.searchsorted(csum, rk, right=False).clamp(max=nb // 1024 - 1)  # first block reaching the rank
    base = torch.where(blk > 0, csum.gather(1, (blk - 1).clamp(min=0)), torch.zeros_like(blk))
    inner = torch.cumsum(hb[torch.arange(nf, device=h.device), blk.view(-1)], dim=1) + base  # [nf, 1024]
    b = torch.searchsorted(inner, rk, right=False)
    before = torch.where(b > 0, inner.gather(1, (b - 1).clamp(min=0)), base)
    res = torch.cat([blk * 1024 + b, before, inner[:, -1:]], dim=1).cpu().tolist()
    out = []
    for (bi, bf, last), r in zip(res, ranks):
        if bi >= nb or last < r:
            raise ColoError(_lib.COLO_EBREACH, "histogram pass lost samples")
        out.append((int(bi), int(r - bf)))
    return out


def serving_stats_c(ctx: Context, profiles, arrival, prompt, output, dev_offsets, dev_profile, tau=math.inf):
    """colo_serving_stats (single GPU, all in the C-ABI)."""
    ms, gs = _profiles_arrays(profiles)
    pctl = (C.c_double * 4)()
    tot = _lib.DeviceSummary()
    check(lib().colo_serving_stats(ctx.h, ms, gs, len(profiles), _ptr(arrival), _ptr(prompt), _ptr(output),
                                   prompt.shape[0], _ptr(dev_offsets), _ptr(dev_profile), dev_profile.shape[0], tau,
                                   pctl, C.byref(tot)), ctx.h, "serving_stats")
    return list(pctl), tot


# ------------------------------------------------------------- colocated replay

COLOCATED_FIELDS = [f for f, _ in _lib.ColocatedSummary._fields_]
# MetricsReport fields the reference reports per run (metrics.hpp:17-44; oom_flag = oom_jobs > 0)
METRICS_FIELDS = COLOCATED_FIELDS[:15]


class SimMode(enum.IntEnum):
    """engine.hpp:23 (names as sim_mode_from_string, :34-39)."""

    SERVING_ONLY = 0
    COLOCATED = 1
    SEPARATE_CLUSTER = 2

    @staticmethod
    def parse(s: str) -> "SimMode":
        m = {"serving-only": SimMode.SERVING_ONLY, "colocated": SimMode.COLOCATED, "baseline": SimMode.SEPARATE_CLUSTER}
        if s not in m:
            raise ColoValidationError(_lib.COLO_EVALIDATION, f"unknown sim mode: {s}")
        return m[s]


def _colocated_opts(ctx, sets, arrival, prompt, output, dev_offsets, dev_set, label_delay, default_label_delay,
                    cache_timeout, tau, samples, labels, batches, summary, res, keep, sim_mode=None, seg_len=None):
    torch = _torch()
    dev = prompt.device
    _need_cuda(arrival, "arrival", 8)
    _need_cuda(prompt, "prompt", 4)
    _need_cuda(output, "output", 4)
    _need_cuda(dev_offsets, "dev_offsets", 8)
    _need_cuda(dev_set, "dev_set", 2)
    n = prompt.shape[0]
    ndev = dev_set.shape[0]
    o = _lib.ColocatedOpts()
    o.cache_timeout = cache_timeout
    o.default_label_delay = default_label_delay
    o.tau = tau
    o.seg_len = 0 if seg_len is None else (0xFFFFFFFF if seg_len == 0 else int(seg_len))
    if label_delay is not None:
        _need_cuda(label_delay, "label_delay", 8)
        o.d_label_delay = label_delay.data_ptr()
    if samples:
        o64 = output.to(torch.int64)
        cs = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), torch.cumsum(o64, 0)])
        per_dev = cs[dev_offsets].contiguous()
        total = int(per_dev[-1].item())
        res["samples"] = torch.empty(max(total, 1), dtype=torch.float64, device=dev)[:total]
        res["sample_offsets"] = per_dev
        o.d_samples = res["samples"].data_ptr() if total else torch.empty(1, dtype=torch.float64, device=dev).data_ptr()
        o.d_sample_offsets = per_dev.data_ptr()
    if labels:
        res["labels"] = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)[:n]
        o.d_labels = res["labels"].data_ptr() if n else 0
    if batches:
        res["batches"] = torch.zeros((max(n, 1), BATCH_DTYPE.itemsize), dtype=torch.uint8, device=dev)
        o.d_batches = res["batches"].data_ptr()
    if summary:
        res["summary"] = torch.zeros((max(ndev, 1), C.sizeof(_lib.ColocatedSummary)), dtype=torch.uint8, device=dev)
        o.d_summary = res["summary"].data_ptr()
    if sim_mode is not None:
        if isinstance(sim_mode, (int, SimMode)):
            sm = torch.full((max(ndev, 1),), int(sim_mode), dtype=torch.uint8, device=dev)
        else:
            sm = sim_mode.to(device=dev, dtype=torch.uint8).contiguous()
        res["sim_mode"] = sm
        o.d_dev_sim_mode = sm.data_ptr()
    arr = _sets_array(sets)
    keep.append(arr)
    return o, arr, n, ndev


def replay_colocated(ctx: Context, sets: Sequence[MapSet], arrival, prompt, output, dev_offsets, dev_set,
                     label_delay=None, default_label_delay: float = 0.01, cache_timeout: float = 60.0,
                     tau: float = math.inf, samples: bool = False, labels: bool = True, batches: bool = False,
                     summary: bool = True, sim_mode=None, seg_len=None):
    """Simulation::run of every device (engine.hpp:140-903), by default in
    SimMode::Colocated; ``sim_mode`` (a SimMode for all devices or a per-device
    uint8 tensor) selects ServingOnly / Colocated / SeparateCluster.  Device d runs with map set ``sets[dev_set[d]]`` and
    that set's model, GPU profile and training mode (SimConfig::validate,
    engine.hpp:60-68).  ``label_delay``: optional f64 device tensor per query
    (< 0 or NaN = the label never arrives); otherwise every query uses
    ``default_label_delay`` (the reference's TraceSpec default is fixed 0.01 s,
    experiment.hpp:45).  Raises ColoBreachError if a device's run breaches an
    invariant (the reference throws InvariantBreach).
    ``seg_len``: None = automatic (with fewer devices than the GPU holds
    warps, long devices replay in parallel segments split at idle arrivals --
    same bits), 0 = never segment, else the segment length in queries.
    Returns a dict of device tensors: samples, labels, batches (BATCH_DTYPE
    bytes at d_dev_offsets[d] + b), summary (ColocatedSummary bytes)."""
    res, keep = {}, []
    o, arr, n, ndev = _colocated_opts(ctx, sets, arrival, prompt, output, dev_offsets, dev_set, label_delay,
                                      default_label_delay, cache_timeout, tau, samples, labels, batches, summary,
                                      res, keep, sim_mode, seg_len)
    try:
        check(lib().colo_replay_colocated(ctx.h, C.cast(arr, C.c_void_p), len(sets), _ptr(arrival), _ptr(prompt),
                                          _ptr(output), n, _ptr(dev_offsets), _ptr(dev_set), ndev, C.byref(o)),
              ctx.h, "replay_colocated")
    except ColoBreachError as e:
        e.result = res  # per-device summaries carry status COLO_EBREACH where the run broke
        raise
    return res


def colocated_summaries(summary_bytes) -> list:
    """ColocatedSummary bytes -> list of dicts (one per device)."""
    a = summary_bytes.cpu().numpy() if hasattr(summary_bytes, "cpu") else np.asarray(summary_bytes)
    a = np.ascontiguousarray(a)
    out = []
    for row in a.reshape(-1, C.sizeof(_lib.ColocatedSummary)):
        s = _lib.ColocatedSummary.from_buffer_copy(row.tobytes())
        out.append({f: (list(getattr(s, f)) if f == "tpt_sum" else getattr(s, f)) for f in COLOCATED_FIELDS})
    return out


def finalize(ctx: Context, samples, sorted_out=None) -> list:
    """colo_finalize: finalize (metrics.hpp:56-69) of a device tensor of TPT
    samples, bit-exact -- [p50, p90, p99, mean] with the mean the sequential
    sum of the ascending-sorted samples / n (NaN when empty).  ``sorted_out``
    (optional f64 device tensor of the same length) receives the sorted
    samples."""
    _need_cuda(samples, "samples", 8)
    samples = samples.contiguous()
    n = samples.numel()
    if sorted_out is not None:
        _need_cuda(sorted_out, "sorted_out", 8)
        if sorted_out.numel() != n or not sorted_out.is_contiguous():
            raise ColoInvalidArgument(_lib.COLO_EINVAL, "sorted_out must be a contiguous tensor of len(samples)")
    out = (C.c_double * 4)()
    check(lib().colo_finalize(ctx.h, _ptr(samples) if n else None, n,
                              _ptr(sorted_out) if (sorted_out is not None and n) else None, out), ctx.h, "finalize")
    return list(out)


def colocated_events(ctx: Context, mapset: MapSet, arrival, prompt, output, label_delay=None,
                     default_label_delay: float = 0.01, query_id=None, cache_timeout: float = 60.0,
                     sim_mode=None, tau: float = math.inf) -> str:
    """colo_colocated_events: the event log of one device's Simulation::run
    (tools/colosim.cpp --emit-events) in any SimMode, as the reference's JSON
    lines (LoggedEvent::to_json, engine.hpp:109-129).
    Device tensors: arrival f64, prompt/output int32, label_delay f64
    (optional), query_id int64 (optional)."""
    _need_cuda(arrival, "arrival", 8)
    _need_cuda(prompt, "prompt", 4)
    _need_cuda(output, "output", 4)
    n = prompt.shape[0]
    mode = int(SimMode.COLOCATED if sim_mode is None else sim_mode)
    ln = lib().colo_colocated_events(ctx.h, mapset.h, mode, cache_timeout, _ptr(arrival), _ptr(prompt), _ptr(output),
                                     _ptr(label_delay), default_label_delay, _ptr(query_id), n, tau)
    if ln < 0:
        check(-ln, ctx.h, "colocated_events")
    buf = C.create_string_buffer(int(ln) + 1)
    lib().colo_events_text(ctx.h, buf, int(ln) + 1)
    return buf.raw[: int(ln)].decode()


def colocated_stats(ctx: Context, sets: Sequence[MapSet], arrival, prompt, output, dev_offsets, dev_set,
                    label_delay=None, default_label_delay: float = 0.01, cache_timeout: float = 60.0,
                    tau: float = math.inf, sim_mode=None, seg_len=None):
    """colo_colocated_stats: colocated replays of every device + exact
    nearest-rank p50/p90/p99 and mean of the union of their TPT samples
    (finalize, metrics.hpp:56-69).  Returns (pctl[4], totals dict)."""
    res, keep = {}, []
    o, arr, n, ndev = _colocated_opts(ctx, sets, arrival, prompt, output, dev_offsets, dev_set, label_delay,
                                      default_label_delay, cache_timeout, tau, False, False, False, False, res, keep,
                                      sim_mode, seg_len)
    pctl = (C.c_double * 4)()
    tot = _lib.ColocatedSummary()
    check(lib().colo_colocated_stats(ctx.h, C.cast(arr, C.c_void_p), len(sets), _ptr(arrival), _ptr(prompt),
                                     _ptr(output), n, _ptr(dev_offsets), _ptr(dev_set), ndev, C.byref(o), pctl,
                                     C.byref(tot)), ctx.h, "colocated_stats")
    return list(pctl), {f: (list(getattr(tot, f)) if f == "tpt_sum" else getattr(tot, f)) for f in COLOCATED_FIELDS}


# ------------------------------------------------------------- workload
def _dist(spec):
    if spec is None:
        return None, []
    d = _lib.Dist()
    keep = []
    kind = spec[0]
    if kind == "fixed":
        d.kind, d.fixed_value = 0, float(spec[1])
    elif kind == "uniform":
        d.kind, d.lo, d.hi = 1, float(spec[1]), float(spec[2])
    elif kind == "histogram":
        v = np.ascontiguousarray(spec[1], np.float64)
        p = np.ascontiguousarray(spec[2], np.float64)
        keep = [v, p]
        d.kind, d.bin_values, d.bin_probs, d.nbins = 2, v.ctypes.data, p.ctypes.data, len(v)
    else:
        raise ColoInvalidArgument(_lib.COLO_EINVAL, f"unknown distribution {kind}")
    return d, keep


def generate_trace(qps: float, duration: float, lengths, seed: int, label_delay=None, min_tokens: int = 0,
                   with_labels: bool = False):
    """workload.hpp:193-220 on the host, bit-exact (returns arrival, prompt, output numpy arrays, plus the
    per-query label delays -- -1.0 = nullopt -- when ``with_labels``).
    lengths/label_delay: ('fixed', v) | ('uniform', lo, hi) | ('histogram', values, probs)."""
    ld, k1 = _dist(lengths)
    ld.min_tokens = min_tokens
    dd, k2 = _dist(label_delay)
    cap = int(qps * duration * 1.3 + 64 * math.sqrt(qps * duration + 1) + 1000)
    arr, pr, out, lab = np.empty(cap), np.empty(cap, np.uint32), np.empty(cap, np.uint32), np.empty(cap)
    n = lib().colo_generate_trace(qps, duration, C.byref(ld), C.byref(dd) if dd is not None else None, seed,
                                  arr.ctypes.data, pr.ctypes.data, out.ctypes.data, lab.ctypes.data, cap)
    if n == -2:
        raise ColoValidationError(_lib.COLO_EVALIDATION, "generate_trace: invalid qps/duration/distribution")
    if n < 0:
        raise ColoError(_lib.COLO_EINVAL, "generate_trace: capacity exceeded")
    if with_labels:
        return arr[:n].copy(), pr[:n].copy(), out[:n].copy(), lab[:n].copy()
    return arr[:n].copy(), pr[:n].copy(), out[:n].copy()


def sharegpt_histogram():
    """proj/profiles/sharegpt_like_lengths.jsonl (11 bins)."""
    values = [64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096]
    probs = [0.05, 0.10, 0.15, 0.15, 0.13, 0.12, 0.10, 0.08, 0.06, 0.04, 0.02]
    return np.array(values, np.float64), np.array(probs, np.float64)


def synth_tuples(ctx: Context, n: int, num_layers: int, seed: int, bins=None):
    """C5 question stream on the GPU (colo_synth_tuples): int32 [n, 4] colo_tuple records."""
    torch = _torch()
    v, p = bins if bins is not None else sharegpt_histogram()
    v = np.ascontiguousarray(v, np.float64)
    p = np.ascontiguousarray(p, np.float64)
    out = torch.empty((max(n, 1), 4), dtype=torch.int32, device=torch.device("cuda", ctx.device))[:n]
    check(lib().colo_synth_tuples(ctx.h, seed, n, num_layers, v.ctypes.data, p.ctypes.data, len(v), _ptr(out)),
          ctx.h, "synth_tuples")
    return out


def compare_verdicts(ctx: Context, map_verdicts, exact_verdicts, num_layers: int, counts=None):
    """Map-vs-exact agreement (colo_compare_verdicts): int64[5] = agree, over-free,
    under-free, same outcome, total (accumulated into ``counts`` if given)."""
    torch = _torch()
    if counts is None:
        counts = torch.zeros(5, dtype=torch.int64, device=map_verdicts.device)
    check(lib().colo_compare_verdicts(ctx.h, _ptr(map_verdicts), _ptr(exact_verdicts), map_verdicts.shape[0],
                                      num_layers, _ptr(counts)), ctx.h, "compare_verdicts")
    return counts


def synth_trace(ctx: Context, dev_sizes: Sequence[int], dev_qps: Sequence[float], seed: int, bins=None,
                dev_qps_hi: Optional[Sequence[float]] = None, burst_period: float = 0.0,
                dev_ids: Optional[Sequence[int]] = None):
    """Bench-scale synthetic device traces generated on the GPU (counter-based
    RNG); bursty when dev_qps_hi/burst_period are given (rate alternates every
    burst_period seconds).  ``dev_ids``: fleet device ids -- the RNG is then
    keyed on (id, query index in the device), so a device's trace does not
    depend on which rank or array position holds it.  Returns (arrival f64,
    prompt i32, output i32, dev_offsets i64) CUDA tensors."""
    torch = _torch()
    v, p = bins if bins is not None else sharegpt_histogram()
    dev = torch.device("cuda", ctx.device)
    offs = np.concatenate([[0], np.cumsum(np.asarray(dev_sizes, np.int64))]).astype(np.int64)
    n = int(offs[-1])
    d_off = torch.from_numpy(offs).to(dev)
    d_qps = torch.tensor(list(dev_qps), dtype=torch.float64, device=dev)
    arrival = torch.empty(max(n, 1), dtype=torch.float64, device=dev)[:n]
    prompt = torch.empty(max(n, 4), dtype=torch.int32, device=dev)[:n]
    output = torch.empty(max(n, 4), dtype=torch.int32, device=dev)[:n]
    v = np.ascontiguousarray(v, np.float64)
    p = np.ascontiguousarray(p, np.float64)
    d_hi = torch.tensor(list(dev_qps_hi), dtype=torch.float64, device=dev) if dev_qps_hi is not None else None
    if dev_ids is None:
        check(lib().colo_synth_trace(ctx.h, v.ctypes.data, p.ctypes.data, len(v), _ptr(d_off), _ptr(d_qps), _ptr(d_hi),
                                     burst_period, len(dev_qps), seed, _ptr(arrival), _ptr(prompt), _ptr(output)),
              ctx.h, "synth_trace")
    else:
        ids = torch.tensor(list(dev_ids), dtype=torch.int32, device=dev)
        if len(dev_ids) != len(dev_qps) or (len(dev_ids) and (min(dev_ids) < 0 or max(dev_ids) >= 1 << 28)):
            raise ColoInvalidArgument(_lib.COLO_EINVAL, "dev_ids: one id in [0, 2^28) per device")
        check(lib().colo_synth_fleet_trace(ctx.h, v.ctypes.data, p.ctypes.data, len(v), _ptr(d_off), _ptr(d_qps),
                                           _ptr(d_hi), burst_period, len(dev_qps), _ptr(ids), seed, _ptr(arrival),
                                           _ptr(prompt), _ptr(output)), ctx.h, "synth_trace")
    return arrival, prompt, output, d_off


# ------------------------------------------------------------ file formats
def save_map_cells(path: str, kind: str, mode: TrainingMode, profile_hash_value: int, num_layers: int,
                   steps: GridSteps, bounds: GridBounds, cells: np.ndarray, assumed_output_tokens: int = 128) -> None:
    """OffloadingMap::save / HedgingMap::save text (maps.hpp:118-140, 284-295), byte-identical."""
    h = _lib.MapHeader()
    h.kind = 0 if kind == "offload" else 1
    h.mode = int(mode)
    h.profile_hash = profile_hash_value
    h.num_layers = num_layers
    h.grid = _grid(steps, bounds)
    h.assumed_output_tokens = assumed_output_tokens
    c = np.ascontiguousarray(cells, np.uint8)
    check(lib().colo_map_save(path.encode(), C.byref(h), c.ctypes.data, c.size), None, f"cannot write map file: {path}")


def load_map_cells(path: str, expected_hash: int):
    """OffloadingMap::load / HedgingMap::load (maps.hpp:142-191, 297-332): (header dict, cells).
    Raises ColoValidationError on a profile-hash mismatch or a malformed file."""
    h = _lib.MapHeader()
    n = C.c_size_t()
    err = C.create_string_buffer(512)
    st = lib().colo_map_load(path.encode(), expected_hash, C.byref(h), None, 0, C.byref(n), err, 512)
    if st:
        raise ColoValidationError(st, err.value.decode())
    cells = np.zeros(n.value, np.uint8)
    st = lib().colo_map_load(path.encode(), expected_hash, C.byref(h), cells.ctypes.data, cells.size, C.byref(n), err, 512)
    if st:
        raise ColoValidationError(st, err.value.decode())
    g = h.grid
    hdr = {"kind": "offload" if h.kind == 0 else "hedge", "mode": TrainingMode(h.mode), "profile_hash": h.profile_hash,
           "num_layers": h.num_layers, "steps": GridSteps(g.cached_step, g.incoming_step, g.batch_step),
           "bounds": GridBounds(g.max_cached, g.max_incoming, g.max_batch),
           "assumed_output_tokens": h.assumed_output_tokens}
    return hdr, cells


def save_mapset(ms: MapSet, offload_path: Optional[str], hedge_path: Optional[str]) -> None:
    """Both maps of a device MapSet in the reference's text format."""
    check(lib().colo_mapset_save(ms.ctx.h, ms.h, offload_path.encode() if offload_path else None,
                                 hedge_path.encode() if hedge_path else None), ms.ctx.h, "map save")


def load_mapset(ctx: Context, m: ModelProfile, g: GpuProfile, offload_path: str, hedge_path: str) -> MapSet:
    """Load saved maps onto the device; refuses maps built from other profiles (maps.hpp:155-157)."""
    h = C.c_void_p()
    check(lib().colo_mapset_load(ctx.h, C.byref(m.to_c()), C.byref(g.to_c()), offload_path.encode(),
                                 hedge_path.encode(), C.byref(h)), ctx.h, "map load")
    ho, _ = load_map_cells(offload_path, profile_hash(m, g))
    hh, _ = load_map_cells(hedge_path, profile_hash(m, g))
    return MapSet(ctx, h, m, g, ho["steps"], ho["bounds"], ho["mode"], hh["steps"].cached_token_step,
                  hh["bounds"].max_cached_tokens, hh["assumed_output_tokens"])


def load_trace(path: str):
    """load_trace (workload.hpp:224-254): validated, (arrival, id)-ordered SoA arrays
    (arrival f64, prompt u32, output u32, query_id u64, label_delay f64 with NaN = null)."""
    err = C.create_string_buffer(512)
    n = lib().colo_load_trace_jsonl(path.encode(), None, None, None, None, None, 0, err, 512)
    if n == -2:
        raise ColoValidationError(_lib.COLO_EVALIDATION, err.value.decode())
    lines = sum(1 for ln in open(path) if ln.strip())  # records <= non-empty lines
    a, p, o = np.empty(lines), np.empty(lines, np.uint32), np.empty(lines, np.uint32)
    q, ld = np.empty(lines, np.uint64), np.empty(lines)
    n = lib().colo_load_trace_jsonl(path.encode(), a.ctypes.data, p.ctypes.data, o.ctypes.data, q.ctypes.data,
                                    ld.ctypes.data, lines, err, 512)
    if n < 0:
        raise ColoValidationError(_lib.COLO_EVALIDATION, err.value.decode())
    return a[:n], p[:n], o[:n], q[:n], ld[:n]


def load_histogram(path: str):
    """load_histogram (workload.hpp:274-293): (values, probabilities)."""
    err = C.create_string_buffer(512)
    v, p = np.empty(1024), np.empty(1024)
    n = lib().colo_load_histogram_jsonl(path.encode(), v.ctypes.data, p.ctypes.data, 1024, err, 512)
    if n < 0:
        raise ColoValidationError(_lib.COLO_EVALIDATION, err.value.decode() or "histogram too large")
    return v[:n], p[:n]
