// colo_common.cuh -- device-side arithmetic shared by every colo-b200 kernel.
//
// Bit-exactness rules: the whole library is compiled
// with -fmad=false so a*b+c never contracts into an FMA; every f64 expression
// keeps the reference's association; byte arithmetic is uint64_t with
// wrap-around; u64->f64 conversions are round-to-nearest (as on x86).
// Reference paths are relative to /root/reference/proj/.
#pragma once

#include <cstdint>

#include "colo_abi.h"

namespace colo {

constexpr uint32_t kMaxSets = 16;      // map sets / profiles per launch
constexpr uint32_t kMaxLayers = 253;   // offload cell code width

// ---------------------------------------------------------------- division
// Exact floor(n / d) for 32-bit n and d via a 64-bit reciprocal
// (c = ceil(2^64 / d); Lemire, Kaser & Kurz 2019, valid for every 32-bit n
// when d <= 2^32).  Two IMADs instead of a 32-bit divide.
struct FastDiv {
    uint32_t d;
    uint32_t c_lo, c_hi;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint64_t c = d > 1 ? (~0ull / d + 1ull) : 0ull;
    f.c_lo = static_cast<uint32_t>(c);
    f.c_hi = static_cast<uint32_t>(c >> 32);
    return f;
}

__device__ __forceinline__ uint32_t floor_div(const FastDiv& f, uint32_t n) {
    if (f.d == 1) return n;
    uint32_t t = __umulhi(f.c_lo, n);
    uint64_t w = static_cast<uint64_t>(f.c_hi) * n + t;
    return static_cast<uint32_t>(w >> 32);
}

// ceil(n / d); the grid validation guarantees n + d - 1 < 2^32.
__device__ __forceinline__ uint32_t ceil_div(const FastDiv& f, uint32_t n) { return floor_div(f, n + f.d - 1); }

// -------------------------------------------------------------- cost model
// cost_model.hpp:18-25 (batch = 1, unrecorded): 1.0 * (lin*t + (quad*t)*t)
__host__ __device__ __forceinline__ double prefill_latency(const colo_model& m, uint64_t tokens, uint64_t batch,
                                                            bool recording) {
    double t = static_cast<double>(tokens);
    double base = static_cast<double>(batch) * (m.prefill_coef_linear * t + m.prefill_coef_quad * t * t);
    return recording ? base * m.record_prefill_multiplier : base;
}

// cost_model.hpp:28-35
__host__ __device__ __forceinline__ double decode_step_latency(const colo_model& m, uint64_t ctx, uint64_t batch,
                                                                bool recording) {
    double base = static_cast<double>(batch) * (m.decode_coef_const + m.decode_coef_context * static_cast<double>(ctx));
    return recording ? base * m.record_decode_multiplier : base;
}

// cost_model.hpp:54-56
__host__ __device__ __forceinline__ uint64_t kv_bytes(const colo_model& m, uint64_t tokens, uint64_t batch) {
    return batch * tokens * m.kv_bytes_per_token;
}

// cost_model.hpp:59-66 (std::llround semantics: half away from zero)
__device__ __forceinline__ uint64_t serving_memory(const colo_model& m, uint64_t tokens, uint64_t batch) {
    uint64_t kv = kv_bytes(m, tokens, batch);
    uint64_t ws = static_cast<uint64_t>(llround(m.workspace_factor * static_cast<double>(kv)));
    return kv + ws;
}

// maps.hpp:215-231, the reference's exact check order.  Returns the offload
// cell code: 0 NoAction, 1 AllToHost, 2+n FreeLayers(n).
__device__ __forceinline__ uint8_t offload_cell_code(const colo_model& m, uint64_t budget, bool cpa, uint64_t cached,
                                                     uint64_t incoming, uint64_t batch) {
    uint64_t acts = cached * m.num_layers * m.act_bytes_per_token_per_layer;  // maps.hpp:54-56
    uint64_t kv = cpa ? kv_bytes(m, cached, 1) : 0ull;                       // maps.hpp:58-61
    if (acts + kv > budget) return 1;
    uint64_t headroom = budget - acts - kv;
    uint64_t need = serving_memory(m, incoming, batch);
    if (need <= headroom) return 0;
    uint64_t deficit = need - headroom;
    uint64_t per_layer = cached * m.act_bytes_per_token_per_layer;
    if (per_layer == 0) return 1;
    uint64_t n = (deficit + per_layer - 1) / per_layer;
    if (n > m.num_layers) return 1;
    return static_cast<uint8_t>(2 + n);
}

// maps.hpp:341-346
__device__ __forceinline__ double hedge_recompute_time(const colo_model& m, bool cpa, uint64_t cached,
                                                       uint64_t assumed) {
    if (cpa) return 2.0 * prefill_latency(m, assumed, 1, false);
    return prefill_latency(m, cached, 1, false);
}

// maps.hpp:349-356 with cost_model.hpp:39-52, 68-71; std::max(0.0, x)
__device__ __forceinline__ double hedge_residual_load_time(const colo_model& m, const colo_gpu& g, uint64_t cached,
                                                           uint64_t freed) {
    uint64_t bytes = cached * freed * m.act_bytes_per_token_per_layer;
    double load = static_cast<double>(bytes) / static_cast<double>(g.h2d_bandwidth);
    uint64_t c1 = cached == 0 ? 1ull : cached;
    double fwd = prefill_latency(m, c1, 1, false) / static_cast<double>(m.num_layers);
    double bwd = m.backward_to_forward_ratio * fwd;
    double credit = static_cast<double>(m.num_layers - freed) * bwd;
    double x = load - credit;
    return (0.0 < x) ? x : 0.0;
}

// ------------------------------------------------------------ map views
// Everything a kernel needs to evaluate OffloadingMap::lookup (maps.hpp:100-110)
// and HedgingMap::lookup (maps.hpp:276-280) from cell tables.
struct MapView {
    const uint8_t* off;   // offload cells, row-major (ci, ii, bi)
    const uint8_t* hed;   // hedge cells, row-major (hi, f)
    const uint32_t* tab;  // trace-fused verdict table [(C+1) x (I+1)] (fast path), may be null
    const uint32_t* str;  // stream bits per cached bucket [C+1], may be null
    uint32_t max_c, max_i, max_b;
    FastDiv fc, fi, fb, fh;
    uint32_t C, I, B;     // cell counts per axis (maps.hpp:85-87)
    uint32_t hmax, hsame; // hedge bound; hsame = hedge step == cached step
    uint32_t L;           // num_layers
    uint32_t cpa;
    uint32_t off_bytes, hed_bytes;
};

// Verdict word, include/colo_abi.h.
__host__ __device__ __forceinline__ uint32_t pack_verdict(uint32_t action, uint32_t layers, uint32_t free_now,
                                                          uint32_t recompute, uint32_t off_oor, uint32_t hedge_oor,
                                                          uint32_t verdict) {
    return action | ((layers & 0xffu) << 2) | ((free_now & 0xffu) << 10) | (recompute << 18) | (off_oor << 19) |
           (hedge_oor << 20) | (verdict << 21);
}

// Offload lookup -> cell code, or 0xff for nullopt (maps.hpp:100-110).
// The round-up bound checks reduce to value > bound because every bound is a
// multiple of its step (validate_grid, maps.hpp:202-207).
__device__ __forceinline__ uint32_t offload_lookup(const MapView& mv, const uint8_t* off, uint64_t cached,
                                                   uint64_t incoming, uint64_t batch) {
    if (cached > mv.max_c || incoming > mv.max_i || batch > mv.max_b || incoming == 0 || batch == 0) return 0xffu;
    uint32_t ci = ceil_div(mv.fc, static_cast<uint32_t>(cached));
    uint32_t ii = ceil_div(mv.fi, static_cast<uint32_t>(incoming)) - 1;
    uint32_t bi = ceil_div(mv.fb, static_cast<uint32_t>(batch)) - 1;
    return off[(ci * mv.I + ii) * mv.B + bi];
}

// Stream bits for charged tokens (engine.hpp:437-444).
__device__ __forceinline__ uint32_t stream_bits(const MapView& mv, const uint8_t* off, uint64_t charged) {
    uint32_t code = offload_lookup(mv, off, charged, 1, 1);
    if (code == 0xffu) return COLO_V_STREAM | COLO_V_STREAM_OOR;
    return code == 1 ? COLO_V_STREAM : 0u;
}

// Simulation::apply_offload_decision, decision half (engine.hpp:513-557).
__device__ __forceinline__ uint32_t compose(const MapView& mv, const uint8_t* off, const uint8_t* hed, uint64_t cached,
                                            uint64_t incoming, uint64_t batch, uint32_t pending, uint32_t dev_layers) {
    uint32_t code = offload_lookup(mv, off, cached, incoming, batch);
    uint32_t fallback = code == 0xffu;
    if (fallback) code = 1;                                       // :517-521
    if (code == 0) return pack_verdict(0, 0, 0, 0, 0, 0, COLO_VD_ADMIT);  // :522
    uint32_t action = code == 1 ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS;
    uint32_t layers = code >= 2 ? code - 2 : 0;
    uint32_t free_now = code == 1 ? dev_layers : min(layers, dev_layers);  // :524-527
    uint32_t ltf = code == 1 ? mv.L : layers;                              // maps.hpp:41-48
    uint32_t total = min(pending + ltf, mv.L);                             // :528-530
    uint32_t recompute = 1, hedge_oor = 0;                                 // :532
    if (!fallback) {
        // round_up_bucket(cached, hs) == 0 or > hmax -> nullopt (maps.hpp:278)
        if (cached == 0 || cached > mv.hmax) {
            hedge_oor = 1;                                                 // :537-538
        } else {
            uint32_t hi = ceil_div(mv.fh, static_cast<uint32_t>(cached)) - 1;
            recompute = hed[hi * (mv.L + 1) + total];
        }
    }
    return pack_verdict(action, layers, free_now, recompute, fallback, hedge_oor,
                        recompute ? COLO_VD_RECOMPUTE_DROP : COLO_VD_FREE_LOADBACK);
}

// charged tokens, engine.hpp:422-423
__device__ __forceinline__ uint64_t charged_tokens(uint32_t p, uint32_t o, uint32_t cpa) {
    return cpa ? static_cast<uint64_t>(p) + 2ull * o : static_cast<uint64_t>(p);
}

// Decision counters from a verdict word.
__device__ __forceinline__ void count_verdict(uint32_t v, uint64_t (&c)[COLO_NCOUNTERS]) {
    uint32_t vd = COLO_V_VERDICT(v);
    c[COLO_CNT_ADMIT] += vd == COLO_VD_ADMIT;
    c[COLO_CNT_FREE_LOADBACK] += vd == COLO_VD_FREE_LOADBACK;
    c[COLO_CNT_RECOMPUTE_DROP] += vd == COLO_VD_RECOMPUTE_DROP;
    c[COLO_CNT_OFFLOAD_OOR] += (v >> 19) & 1u;
    c[COLO_CNT_HEDGE_OOR] += (v >> 20) & 1u;
    c[COLO_CNT_STREAM] += (v >> 23) & 1u;
    c[COLO_CNT_STREAM_OOR] += (v >> 24) & 1u;
    c[COLO_CNT_TOTAL] += 1;
}

// Warp-aggregated counting: one ballot + popc per category per warp-wide
// verdict slot (all lanes hold the same running totals).  `valid` masks lanes
// without an element.  Totals are per warp, so u32 suffices below 2^32
// elements per warp.
__device__ __forceinline__ void count_warp(uint32_t v, bool valid, uint32_t (&c)[COLO_NCOUNTERS]) {
    const uint32_t vd = COLO_V_VERDICT(v);
    c[COLO_CNT_ADMIT] += __popc(__ballot_sync(0xffffffffu, valid && vd == COLO_VD_ADMIT));
    c[COLO_CNT_FREE_LOADBACK] += __popc(__ballot_sync(0xffffffffu, valid && vd == COLO_VD_FREE_LOADBACK));
    c[COLO_CNT_RECOMPUTE_DROP] += __popc(__ballot_sync(0xffffffffu, valid && vd == COLO_VD_RECOMPUTE_DROP));
    c[COLO_CNT_OFFLOAD_OOR] += __popc(__ballot_sync(0xffffffffu, valid && (v & COLO_V_OFFLOAD_OOR)));
    c[COLO_CNT_HEDGE_OOR] += __popc(__ballot_sync(0xffffffffu, valid && (v & COLO_V_HEDGE_OOR)));
    c[COLO_CNT_STREAM] += __popc(__ballot_sync(0xffffffffu, valid && (v & COLO_V_STREAM)));
    c[COLO_CNT_STREAM_OOR] += __popc(__ballot_sync(0xffffffffu, valid && (v & COLO_V_STREAM_OOR)));
    c[COLO_CNT_TOTAL] += __popc(__ballot_sync(0xffffffffu, valid));
}

__device__ __forceinline__ void flush_warp_counters(const uint32_t (&c)[COLO_NCOUNTERS], uint64_t* d_counters) {
    const uint32_t lane = threadIdx.x & 31;
    if (lane < COLO_NCOUNTERS) {
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) mine = lane == static_cast<uint32_t>(k) ? c[k] : mine;
        if (mine) atomicAdd(reinterpret_cast<unsigned long long*>(&d_counters[lane]), static_cast<unsigned long long>(mine));
    }
}

__device__ __forceinline__ void flush_counters(uint64_t (&c)[COLO_NCOUNTERS], uint64_t* d_counters) {
#pragma unroll
    for (int k = 0; k < COLO_NCOUNTERS; ++k) {
        uint64_t v = c[k];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(&d_counters[k]), v);
    }
}

}  // namespace colo
