// colo_decide.cu -- the admission decision kernels (K1+K2) and their launchers.
//
//   k_decide        tuple stream: one 16-B colo_tuple -> one u32 verdict
//   k_decide_exact  tuple stream, un-quantised (offload_cell_decision + direct hedge)
//   k_fused_fast    trace SoA -> features -> verdict through the per-set
//                   (cached bucket x incoming bucket) verdict table in smem
//   k_fused_gen     same through compose() (hedge grid != offload grid, or
//                   tables too large for shared memory)
//
// All three decision paths evaluate the same function (colo_common.cuh
// compose(), engine.hpp:513-557 + 437-444); tests/test_gpu_parity.py holds
// each of them to the CPU oracle and the reference's golden vectors.
// Reference paths are relative to /root/reference/proj/.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "colo_internal.h"
#include "colo_tma.cuh"

using namespace colo;

namespace {

constexpr int kThreads = 256;
constexpr unsigned FULL = 0xffffffffu;

int blocks_for(colo_ctx* ctx, const void* fn, int threads, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    return per_sm * ctx->sm_count;
}

colo_status check_align(colo_ctx* ctx, const void* p) {
    if (reinterpret_cast<uintptr_t>(p) & 15u) return set_err(ctx, COLO_EINVAL, "device buffers must be 16-byte aligned");
    return COLO_OK;
}

// --------------------------------------------------------------- tuple path
// compose() specialised to 32-bit tuple fields and written branch-free:
// every lookup index is clamped into range and the out-of-range cases are
// selected afterwards, so a warp never diverges on the data.
__device__ __forceinline__ uint32_t compose32(const MapView& mv, const uint8_t* off, const uint8_t* hed, uint32_t c,
                                              uint32_t inc, uint32_t b, uint32_t pend, uint32_t dev) {
    // OffloadingMap::lookup nullopt (maps.hpp:105-107)
    const bool oor = (c > mv.max_c) | (inc > mv.max_i) | (b > mv.max_b) | (inc == 0) | (b == 0);
    const uint32_t ci = ceil_div(mv.fc, min(c, mv.max_c));
    const uint32_t ii = ceil_div(mv.fi, max(min(inc, mv.max_i), 1u)) - 1;
    const uint32_t bi = ceil_div(mv.fb, max(min(b, mv.max_b), 1u)) - 1;
    uint32_t code = off[(ci * mv.I + ii) * mv.B + bi];
    code = oor ? 1u : code;                                   // engine.hpp:517-521
    const bool a2h = code == 1;
    const uint32_t layers = code >= 2 ? code - 2 : 0u;
    const uint32_t free_now = a2h ? dev : min(layers, dev);   // engine.hpp:524-527
    const uint32_t total = min(pend + (a2h ? mv.L : layers), mv.L);  // engine.hpp:528-530
    // HedgingMap::lookup nullopt (maps.hpp:277-278); forced Recompute on offload fallback
    const bool hoor = (c == 0) | (c > mv.hmax);
    const uint32_t hi = mv.hsame ? ci - 1 : ceil_div(mv.fh, min(max(c, 1u), mv.hmax)) - 1;
    const uint32_t hbit = hed[(oor | hoor) ? 0u : hi * (mv.L + 1) + total];
    const uint32_t recompute = (oor | hoor) ? 1u : hbit;
    const uint32_t v = (a2h ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS) | (layers << 2) | (free_now << 10) |
                       (recompute << 18) | (oor ? COLO_V_OFFLOAD_OOR : 0u) | ((!oor & hoor) ? COLO_V_HEDGE_OOR : 0u) |
                       ((recompute ? COLO_VD_RECOMPUTE_DROP : COLO_VD_FREE_LOADBACK) << 21);
    return code == 0 ? 0u : v;                                // NoAction -> ADMIT (engine.hpp:522)
}

// admit_to_store's streaming pre-commitment, lookup(charged, 1, 1) (engine.hpp:437-444)
__device__ __forceinline__ uint32_t stream32(const MapView& mv, const uint8_t* off, uint32_t ch) {
    const bool oor = ch > mv.max_c;
    const uint32_t code = off[ceil_div(mv.fc, min(ch, mv.max_c)) * mv.I * mv.B];
    return oor ? (COLO_V_STREAM | COLO_V_STREAM_OOR) : (code == 1 ? COLO_V_STREAM : 0u);
}

// compose32 for the common map shape (every step > 1, hedge step == cached
// step -- what build_maps produces, experiment.hpp:144-152): the reciprocal
// constants are hoisted into registers by the caller and the step-1 and
// separate-hedge-grid cases disappear.  Same function of the tuple as
// compose32 / compose (tests hold all of them to the oracle).
struct FastMap {
    uint32_t max_c, max_i, max_b, hmax, L, I, B;
    uint32_t cc_lo, cc_hi, ci_lo, ci_hi, cb_lo, cb_hi, dc, di, db;
};

__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t lo, uint32_t hi) {  // floor(n / d), d > 1
    const uint32_t t = __umulhi(lo, n);
    return static_cast<uint32_t>((static_cast<uint64_t>(hi) * n + t) >> 32);
}

__device__ __forceinline__ uint32_t compose32_fast(const FastMap& f, const uint8_t* off, const uint8_t* hed, uint32_t c,
                                                   uint32_t inc, uint32_t b, uint32_t pend, uint32_t dev) {
    const bool oor = (c > f.max_c) | (inc - 1u >= f.max_i) | (b - 1u >= f.max_b);  // maps.hpp:105-107, 0 wraps
    const uint32_t ci = fdiv(min(c, f.max_c) + f.dc - 1u, f.cc_lo, f.cc_hi);
    const uint32_t ii = fdiv(min(inc - 1u, f.max_i - 1u) + f.di, f.ci_lo, f.ci_hi) - 1u;  // ceil(inc/d) - 1
    const uint32_t bi = fdiv(min(b - 1u, f.max_b - 1u) + f.db, f.cb_lo, f.cb_hi) - 1u;
    uint32_t code = off[(ci * f.I + ii) * f.B + bi];
    code = oor ? 1u : code;
    const bool a2h = code == 1;
    const uint32_t layers = code >= 2 ? code - 2 : 0u;
    const uint32_t free_now = a2h ? dev : min(layers, dev);
    const uint32_t total = min(pend + (a2h ? f.L : layers), f.L);
    const bool hoor = (c - 1u >= f.hmax);  // c == 0 || c > hmax
    const bool forced = oor | hoor;
    const uint32_t hbit = hed[forced ? 0u : (ci - 1u) * (f.L + 1) + total];
    const uint32_t recompute = forced ? 1u : hbit;
    const uint32_t v = (a2h ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS) | (layers << 2) | (free_now << 10) |
                       (recompute << 18) | (oor ? COLO_V_OFFLOAD_OOR : 0u) | ((!oor & hoor) ? COLO_V_HEDGE_OOR : 0u) |
                       ((COLO_VD_FREE_LOADBACK + recompute) << 21);
    return code == 0 ? 0u : v;
}

__device__ __forceinline__ uint32_t stream32_fast(const FastMap& f, const uint8_t* off, uint32_t ch) {
    const bool oor = ch > f.max_c;
    const uint32_t code = off[fdiv(min(ch, f.max_c) + f.dc - 1u, f.cc_lo, f.cc_hi) * f.I * f.B];
    return oor ? (COLO_V_STREAM | COLO_V_STREAM_OOR) : (code == 1 ? COLO_V_STREAM : 0u);
}

struct DecideParams {
    MapView mv;
    const uint4* in;
    uint32_t* out;
    uint64_t n;
    uint64_t* counters;
    const uint8_t* img;  // k_decide_packed: the map set's shared-memory image (colo_mapset::d_img), or null
    uint32_t img_bytes;
};

template <bool SMEM, bool COUNT>
__global__ void __launch_bounds__(kThreads) k_decide(const __grid_constant__ DecideParams P) {
    extern __shared__ __align__(128) uint8_t sm[];  // (one alignment for the TU's dynamic shared memory)
    const MapView mv = P.mv;  // by value: the fields live in registers / uniform registers
    const uint8_t* off = mv.off;
    const uint8_t* hed = mv.hed;
    if (SMEM) {
        const uint32_t ob = (mv.off_bytes + 15u) & ~15u;
        for (uint32_t i = threadIdx.x; i < mv.off_bytes; i += blockDim.x) sm[i] = mv.off[i];
        for (uint32_t i = threadIdx.x; i < mv.hed_bytes; i += blockDim.x) sm[ob + i] = mv.hed[i];
        __syncthreads();
        off = sm;
        hed = sm + ob;
    }
    uint32_t cnt[COLO_NCOUNTERS] = {};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    constexpr int U = 8;
    // the trip count is warp-uniform (it depends on the warp's first lane only)
    const uint64_t wbase = tid & ~uint64_t(31);
    for (uint64_t base = tid, wb = wbase; wb < P.n; base += stride * U, wb += stride * U) {
        uint4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * stride;
            t[u] = i < P.n ? __ldcs(P.in + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * stride;
            const uint32_t v = compose32(mv, off, hed, t[u].x, t[u].y, t[u].w & 0xffffu, (t[u].w >> 16) & 0xffu,
                                         t[u].w >> 24) |
                               stream32(mv, off, t[u].z);
            if (i < P.n) __stcs(P.out + i, v);
            if (COUNT) count_warp(v, i < P.n, cnt);
        }
    }
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

// Tuple-stream decisions on grids with the fast composition (every C5 grid,
// up to the sweep-size ones whose byte cells exceed shared memory -- step 50:
// 161 x 160 x 10 = 257,600 cells): the cells are packed five 6-bit codes per
// word (codes are 0, 1 or 2 + n <= L + 2 < 64) into at most 206 KB of shared
// memory, copied by one bulk copy from the map set's prebuilt image, so every
// lookup stays on the SM instead of gathering through L1/L2.  The stream bit
// of each cached bucket (cell (ci, 0, 0)) gets a byte table of its own: those
// cells sit I*B apart, which would put a warp's packed-word reads in a few
// banks.  One 1024-thread CTA per SM streams the tuples with six loads in
// flight per thread; the composition is compose32_fast's.  It beats the TMA
// pipeline below at every C5 step (step 250: 2.74e11 vs 2.52e11/s), so the
// TMA kernel is left to grids without the fast composition.
constexpr int kPackThreads = 1024;
#ifndef COLO_PACK_FROM
#define COLO_PACK_FROM 0  // byte-cell tables above this size take the packed kernel
#endif
constexpr size_t kPackFrom = COLO_PACK_FROM;
#ifndef COLO_PACK_U
#define COLO_PACK_U 6
#endif  // byte-cell tables above this size take the packed kernel

__device__ __forceinline__ uint32_t packed_cell(const uint32_t* pk, uint32_t idx) {
    const uint32_t w = __umulhi(idx, 0xCCCCCCCDu) >> 2;  // idx / 5
    return (pk[w] >> (6u * (idx - 5u * w))) & 63u;
}

// the packed image: cells five 6-bit codes per word, the hedge bits, the
// per-cached-bucket stream bytes (cell (ci, 0, 0) == AllToHost), each part
// 16-byte aligned
__device__ __forceinline__ void pack_image(const MapView& mv, uint32_t* pk, uint8_t* hed, uint8_t* sbit, uint32_t t0,
                                           uint32_t nt) {
    const uint32_t ncells = mv.off_bytes, nw = (ncells + 4) / 5;
    for (uint32_t w = t0; w < nw; w += nt) {
        uint32_t word = 0;
#pragma unroll
        for (uint32_t r = 0; r < 5; ++r) {
            const uint32_t i = 5 * w + r;
            if (i < ncells) word |= static_cast<uint32_t>(__ldg(mv.off + i)) << (6 * r);
        }
        pk[w] = word;
    }
    for (uint32_t i = t0; i < mv.hed_bytes; i += nt) hed[i] = mv.hed[i];
    for (uint32_t ci = t0; ci < mv.C; ci += nt) sbit[ci] = __ldg(mv.off + ci * mv.I * mv.B) == 1;
}

__global__ void k_pack_image(const __grid_constant__ MapView mv, uint8_t* __restrict__ img) {
    const uint32_t nw = (mv.off_bytes + 4) / 5;
    uint32_t* pk = reinterpret_cast<uint32_t*>(img);
    uint8_t* hed = img + ((nw * 4 + 15u) & ~15u);
    uint8_t* sbit = hed + ((mv.hed_bytes + 15u) & ~15u);
    pack_image(mv, pk, hed, sbit, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// bytes of the packed image when the grid takes k_decide_packed, else 0
size_t packed_image_bytes(const MapView& mv) {
    const size_t smem = ((mv.off_bytes + 15u) & ~15u) + mv.hed_bytes;
    const bool fastgrid = mv.hsame && mv.fc.d > 1 && mv.fi.d > 1 && mv.fb.d > 1;
    const size_t packed = ((((mv.off_bytes + 4u) / 5u) * 4u + 15u) & ~size_t(15)) + ((mv.hed_bytes + 15u) & ~15u) +
                          ((mv.C + 15u) & ~15u);
    return (smem > kPackFrom && fastgrid && mv.L + 2 < 64 && packed <= 220 * 1024) ? packed : 0;
}

template <bool COUNT>
__global__ void __launch_bounds__(kPackThreads, 1) k_decide_packed(const __grid_constant__ DecideParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    const MapView& mv = P.mv;
    const uint32_t ncells = mv.off_bytes, nw = (ncells + 4) / 5;
    uint32_t* pk = reinterpret_cast<uint32_t*>(sm);
    uint8_t* hed = sm + ((nw * 4 + 15u) & ~15u);
    uint8_t* sbit = hed + ((mv.hed_bytes + 15u) & ~15u);  // [C] cell (ci, 0, 0) == AllToHost
    if (P.img) {  // the map set's prebuilt image: one bulk copy (L2-resident after the first CTA)
        __shared__ uint64_t bar;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(&bar, P.img_bytes);
            bulk_g2s(sm, P.img, P.img_bytes, &bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
    } else {
        pack_image(mv, pk, hed, sbit, threadIdx.x, blockDim.x);
        __syncthreads();
    }
    const FastMap f{mv.max_c, mv.max_i, mv.max_b, mv.hmax, mv.L, mv.I, mv.B, mv.fc.c_lo, mv.fc.c_hi, mv.fi.c_lo,
                    mv.fi.c_hi, mv.fb.c_lo, mv.fb.c_hi, mv.fc.d, mv.fi.d, mv.fb.d};
    uint32_t cnt[COLO_NCOUNTERS] = {};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    constexpr int U = COUNT ? 4 : COLO_PACK_U;  // (the counters need the registers)
    const uint64_t wbase = tid & ~uint64_t(31);  // warp-uniform trip count
    for (uint64_t base = tid, wb = wbase; wb < P.n; base += stride * U, wb += stride * U) {
      // every tuple of the warp's U in range (warp-uniform): no per-tuple guards
      auto body = [&](auto guard) {
        constexpr bool G = decltype(guard)::value;
        uint4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * stride;
            t[u] = (!G || i < P.n) ? __ldcs(P.in + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * stride;
            // compose32_fast with the cell read from the packed words
            const uint32_t c = t[u].x, inc = t[u].y, b = t[u].w & 0xffffu, pend = (t[u].w >> 16) & 0xffu,
                           dev = t[u].w >> 24;
            const bool oor = (c > f.max_c) | (inc - 1u >= f.max_i) | (b - 1u >= f.max_b);  // maps.hpp:105-107
            const uint32_t ci = fdiv(min(c, f.max_c) + f.dc - 1u, f.cc_lo, f.cc_hi);
            const uint32_t ii = fdiv(min(inc - 1u, f.max_i - 1u) + f.di, f.ci_lo, f.ci_hi) - 1u;
            const uint32_t bi = fdiv(min(b - 1u, f.max_b - 1u) + f.db, f.cb_lo, f.cb_hi) - 1u;
            uint32_t code = packed_cell(pk, (ci * f.I + ii) * f.B + bi);
            code = oor ? 1u : code;  // engine.hpp:517-521
            const bool a2h = code == 1;
            const uint32_t layers = code >= 2 ? code - 2 : 0u;
            const uint32_t free_now = a2h ? dev : min(layers, dev);
            const uint32_t total = min(pend + (a2h ? f.L : layers), f.L);
            const bool hoor = (c - 1u >= f.hmax);
            const bool forced = oor | hoor;
            const uint32_t hbit = hed[forced ? 0u : (ci - 1u) * (f.L + 1) + total];
            const uint32_t recompute = forced ? 1u : hbit;
            uint32_t v = (a2h ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS) | (layers << 2) | (free_now << 10) |
                         (recompute << 18) | (oor ? COLO_V_OFFLOAD_OOR : 0u) | ((!oor & hoor) ? COLO_V_HEDGE_OOR : 0u) |
                         ((COLO_VD_FREE_LOADBACK + recompute) << 21);
            v = code == 0 ? 0u : v;
            // admit_to_store's stream bit: lookup(charged, 1, 1) (engine.hpp:437-444)
            const uint32_t ch = t[u].z;
            const bool soor = ch > f.max_c;
            const uint32_t sb = sbit[fdiv(min(ch, f.max_c) + f.dc - 1u, f.cc_lo, f.cc_hi)];
            v |= soor ? (COLO_V_STREAM | COLO_V_STREAM_OOR) : (sb ? COLO_V_STREAM : 0u);
            const bool ok = !G || i < P.n;
            if (ok) __stcs(P.out + i, v);
            if (COUNT) count_warp(v, ok, cnt);
        }
      };
      if (wb + (U - 1) * stride + 32 <= P.n) body(std::false_type{});
      else body(std::true_type{});
    }
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

// Tuple stream through a TMA pipeline: each CTA streams 16-KB tiles of tuples
// into shared memory kStages tiles ahead with cp.async.bulk (one elected
// thread, mbarrier completion), so the compute never waits on DRAM and needs
// no register prefetch buffers.  Map cells sit in shared memory next to the
// stages.
constexpr uint32_t kTile = 1024;  // tuples per bulk copy (16 KB)
constexpr uint32_t kStages = 4;

template <bool COUNT, bool FAST, uint32_t STAGES>
__global__ void __launch_bounds__(kThreads) k_decide_tma(const __grid_constant__ DecideParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    const MapView mv = P.mv;
    uint4* tiles = reinterpret_cast<uint4*>(sm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + STAGES * kTile * 16);
    uint8_t* off = sm + STAGES * kTile * 16 + 64;
    const uint32_t ob = (mv.off_bytes + 15u) & ~15u;
    uint8_t* hed = off + ob;
    const uint64_t ntiles = (P.n + kTile - 1) / kTile;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    for (uint32_t i = threadIdx.x; i < mv.off_bytes; i += blockDim.x) off[i] = mv.off[i];
    for (uint32_t i = threadIdx.x; i < mv.hed_bytes; i += blockDim.x) hed[i] = mv.hed[i];
    __syncthreads();
    auto issue = [&](uint32_t s, uint64_t t) {
        const uint64_t rest = P.n - t * kTile;
        const uint32_t bytes = static_cast<uint32_t>(rest < kTile ? rest : kTile) * 16u;
        mbar_arrive_expect_tx(&bars[s], bytes);
        bulk_g2s(tiles + s * kTile, P.in + t * kTile, bytes, &bars[s]);
    };
    if (threadIdx.x == 0)
        for (uint32_t s = 0; s < STAGES; ++s) {
            const uint64_t t = blockIdx.x + static_cast<uint64_t>(s) * gridDim.x;
            if (t < ntiles) issue(s, t);
        }
    FastMap f;
    if (FAST) {
        f = FastMap{mv.max_c, mv.max_i, mv.max_b, mv.hmax, mv.L, mv.I, mv.B, mv.fc.c_lo, mv.fc.c_hi, mv.fi.c_lo,
                    mv.fi.c_hi, mv.fb.c_lo, mv.fb.c_hi, mv.fc.d, mv.fi.d, mv.fb.d};
    }
    uint32_t cnt[COLO_NCOUNTERS] = {};
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const uint32_t s = it % STAGES;
        mbar_wait(&bars[s], (it / STAGES) & 1u);
        const uint64_t base = t * kTile;
        const uint64_t rest = P.n - base;
        const uint32_t len = static_cast<uint32_t>(rest < kTile ? rest : kTile);
#pragma unroll
        for (uint32_t q = 0; q < kTile / kThreads; ++q) {
            const uint32_t i = threadIdx.x + q * kThreads;
            const bool valid = i < len;
            const uint4 tu = valid ? tiles[s * kTile + i] : make_uint4(0, 0, 0, 0);
            uint32_t v;
            if (FAST)
                v = compose32_fast(f, off, hed, tu.x, tu.y, tu.w & 0xffffu, (tu.w >> 16) & 0xffu, tu.w >> 24) |
                    stream32_fast(f, off, tu.z);
            else
                v = compose32(mv, off, hed, tu.x, tu.y, tu.w & 0xffffu, (tu.w >> 16) & 0xffu, tu.w >> 24) |
                    stream32(mv, off, tu.z);
            if (valid) __stcs(P.out + base + i, v);
            if (COUNT) count_warp(v, valid, cnt);
        }
        __syncthreads();  // stage s consumed by every thread
        if (threadIdx.x == 0) {
            const uint64_t nt = t + static_cast<uint64_t>(STAGES) * gridDim.x;
            if (nt < ntiles) issue(s, nt);
        }
    }
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

struct ExactParams {
    colo_model m;
    colo_gpu g;
    uint64_t budget, assumed;
    uint32_t cpa;
    const uint4* in;
    uint32_t* out;
    uint64_t n;
    uint64_t* counters;
    // launch constants of offload_cell_decision (maps.hpp:215-231), all mod 2^64
    // like the reference's own products: acts + kv = cached * (L*abpt + kvbpt[CPA])
    uint64_t ak;       // L * abpt (+ kvbpt in CPA)
    uint64_t abpt, kvbpt;
    uint32_t L;
    uint32_t wf_mode;  // 1: workspace_factor == 1.0 (need = 2 kv below 2^53), 0: generic llround
    const uint16_t* tab;  // kExactTab entries: bits 0-7 hedge threshold, bit 8 stream bit (k_exact_tab)
    // exact_verdict_fast's launch conditions (fast = 0: every lane takes exact_verdict)
    uint32_t fast;   // wf_mode 1, 1 <= abpt < 2^40, ak < 2^50
    uint32_t cmax;   // floor(budget / ak): cached * ak > budget <=> cached > cmax (no wrap below kSmemTab)
    float over_f;    // (float)(L + 2)
};

// Per-value tables for the exact path, indexed by a 16-bit token count c.
//  - bits 0-7: the hedge threshold.  For a fixed cached value the residual
//    load time is non-decreasing in the freed-layer count f (bytes grow with
//    f, the credit shrinks, and every rounding step is monotone), so
//    recompute(c, f) = residual(c, f) > recompute_time(c) (maps.hpp:341-356,
//    380) holds exactly for f >= thr[c].  The entry is found by evaluating the
//    same inequality at every f in [0, L]; an entry whose bits are not of that
//    shape (u64 wrap in the byte product) is 0xff and the kernel evaluates the
//    inequality directly.  L + 1 = never.
//  - bit 8: offload_cell_decision(c, 1, 1) == AllToHost, the stream flag of a
//    query charged c tokens (engine.hpp:437-444).
constexpr uint32_t kExactTab = 65536;

__global__ void k_exact_tab(const __grid_constant__ colo_model m, const __grid_constant__ colo_gpu g, uint32_t cpa,
                            uint64_t assumed, uint64_t budget, uint16_t* __restrict__ tab) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= kExactTab) return;
    const uint32_t L = static_cast<uint32_t>(m.num_layers);
    uint32_t t = 0xffu;
    if (c != 0) {  // c == 0: HedgingMap nullopt, never read
        const double rc = hedge_recompute_time(m, cpa != 0, c, assumed);
        t = L + 1;
        bool ok = true;
        for (uint32_t f = 0; f <= L; ++f) {
            const bool r = hedge_residual_load_time(m, g, c, f) > rc;
            if (r && t == L + 1) t = f;
            ok &= r == (t != L + 1);
        }
        if (!ok) t = 0xffu;
    }
    const uint32_t stream = offload_cell_code(m, budget, cpa != 0, c, 1, 1) == 1;
    tab[c] = static_cast<uint16_t>(t | (stream << 8));
}

// offload_cell_decision (maps.hpp:215-231) at a raw point without the u64
// divide and without data-dependent branches: every check of the reference,
// in its order, on the same mod-2^64 products, evaluated for every lane and
// selected at the end.  n = ceil(deficit / per_layer) > L is decided by the
// exact 128-bit product L * per_layer; otherwise n <= L and
// floor(deficit / per_layer) comes from an fp32 quotient estimate (relative
// error < 2^-21, so within one of the floor for quotients <= 253) corrected
// with exact u64 products.  Lanes where the reference's (deficit + per_layer
// - 1) wraps or per_layer >= 2^56 take the reference's own expression.
__device__ __forceinline__ uint32_t exact_code(const ExactParams& P, uint32_t cached, uint32_t incoming,
                                               uint32_t batch) {
    const uint64_t ak = static_cast<uint64_t>(cached) * P.ak;  // acts + kv (maps.hpp:54-61)
    const uint64_t headroom = P.budget - ak;
    const uint64_t kv = static_cast<uint64_t>(batch * static_cast<uint64_t>(incoming)) * P.kvbpt;  // cost_model.hpp:54-56
    uint64_t need = kv + kv;  // serving_memory (cost_model.hpp:59-66): llround(1.0 * (double)kv) == kv below 2^53
    if (P.wf_mode != 1 || kv >= (1ull << 53))
        need = kv + static_cast<uint64_t>(llround(P.m.workspace_factor * static_cast<double>(kv)));
    const uint64_t deficit = need - headroom;
    const uint64_t per_layer = static_cast<uint64_t>(cached) * P.abpt;
    const uint64_t sum = deficit + (per_layer - 1);
    // n > L (exact: below 2^56 per_layer * L does not wrap; above, the reference's divide decides)
    const bool over = deficit > per_layer * P.L;
    const float fq = __fmul_rz(__ull2float_rn(deficit), __frcp_rn(__ull2float_rn(per_layer)));
    uint32_t q = static_cast<uint32_t>(fq);  // (only used when n <= L, i.e. fq <= L + 1)
    uint64_t pr = q * per_layer;
    const bool hi = pr > deficit;
    const bool lo = !hi && deficit - pr >= per_layer;
    q = hi ? q - 1 : (lo ? q + 1 : q);
    pr = hi ? pr - per_layer : (lo ? pr + per_layer : pr);
    uint64_t n = q + (pr != deficit);
    const bool ref_div = sum < deficit || (per_layer >> 56) != 0;
    const bool a2h = ak > P.budget;
    const bool noact = need <= headroom;
    if (ref_div && !a2h && !noact && per_layer != 0) n = sum / per_layer;  // maps.hpp:227, wrap-around included
    else if (over) n = P.L + 1;
    const uint32_t code = n > P.L ? 1u : 2u + static_cast<uint32_t>(n);
    return a2h ? 1u : (noact ? 0u : (per_layer == 0 ? 1u : code));
}

// One exact verdict: exact_code, the hedge inequality through the threshold
// table, the stream bit (engine.hpp:437-444).  thr / sbits: the per-value
// tables of k_exact_tab staged in shared memory for values below kSmemTab.
constexpr uint32_t kSmemTab = 16384;

__device__ __forceinline__ uint32_t exact_verdict(const ExactParams& P, bool cpa, const uint4 t, const uint8_t* thr,
                                                  const uint32_t* sbits) {
    const uint32_t cached = t.x, incoming = t.y, charged = t.z;
    const uint32_t batch = t.w & 0xffffu, pending = (t.w >> 16) & 0xffu, dev = t.w >> 24;
    const uint32_t L = P.L;
    const bool fallback = incoming == 0 || batch == 0;
    const uint32_t code = fallback ? 1u : exact_code(P, cached, incoming, batch);
    const bool a2h = code == 1;
    const uint32_t layers = code >= 2 ? code - 2 : 0u;
    const uint32_t free_now = a2h ? dev : min(layers, dev);
    const uint32_t total = min(pending + (a2h ? L : layers), L);
    const bool hoor = cached == 0;  // HedgingMap nullopt at c == 0 (maps.hpp:278)
    uint32_t th = thr[min(cached, kSmemTab - 1)];
    if (cached >= kSmemTab) th = cached < kExactTab ? (__ldg(P.tab + cached) & 0xffu) : 0xffu;
    bool rec = total >= th;
    if (th == 0xffu && !fallback && !hoor) {  // not of threshold shape: the inequality itself
        const double rc = hedge_recompute_time(P.m, cpa, cached, P.assumed);
        rec = hedge_residual_load_time(P.m, P.g, cached, total) > rc;
    }
    const uint32_t recompute = (fallback || hoor) ? 1u : static_cast<uint32_t>(rec);
    const uint32_t v = (a2h ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS) | (layers << 2) | (free_now << 10) |
                       (recompute << 18) | (fallback ? COLO_V_OFFLOAD_OOR : 0u) |
                       ((!fallback && hoor) ? COLO_V_HEDGE_OOR : 0u) | ((COLO_VD_FREE_LOADBACK + recompute) << 21);
    bool stream = (sbits[min(charged, kSmemTab - 1) >> 5] >> (charged & 31)) & 1u;
    if (charged >= kSmemTab)
        stream = charged < kExactTab ? (__ldg(P.tab + charged) >> 8) != 0 : exact_code(P, charged, 1, 1) == 1;
    return (code == 0 ? 0u : v) | (stream ? COLO_V_STREAM : 0u);
}

__device__ __noinline__ uint32_t exact_verdict_slow(const ExactParams& P, bool cpa, const uint4 t, const uint8_t* thr,
                                                   const uint32_t* sbits) {
    return exact_verdict(P, cpa, t, thr, sbits);
}

// exact_verdict for the common lane, without branches and with as few
// ALU-pipe operations as the exact result allows (the kernel is bound by the
// ALU pipe: compares, selects, bit fields).  The lane's values lie below
// kSmemTab (both tables in shared memory), kv below 2^53, the hedge entry is
// threshold-shaped, and the launch satisfies ExactParams::fast; then, when
// neither AllToHost nor NoAction applies, 0 < deficit <= need < 2^54 and
// per_layer < 2^54, so sum = deficit + per_layer - 1 never wraps and the
// reference's sum / per_layer is found from the fp32 estimate q of the
// quotient (within 2^-12 of it while it is <= L + 2, so q is the floor or
// one off) by one signed remainder r = sum - q * per_layer:
//   n = q + (r >= per_layer) - (r < 0).
// An estimate above L + 2 means n > L.  Any other lane sets slow and takes
// exact_verdict afterwards.
__device__ __forceinline__ uint32_t exact_verdict_fast(const ExactParams& P, const uint4 t, const uint8_t* thr,
                                                       const uint32_t* sbits, bool& slow) {
    const uint32_t cached = t.x, incoming = t.y, charged = t.z;
    const uint32_t batch = t.w & 0xffffu, pending = (t.w >> 16) & 0xffu, dev = t.w >> 24;
    const uint32_t L = P.L;
    const bool fallback = (incoming == 0) | (batch == 0);
    const bool hoor = cached == 0;  // also per_layer == 0 (abpt >= 1, no wrap)
    const uint64_t ak = static_cast<uint64_t>(cached) * P.ak;  // acts + kv (maps.hpp:54-61)
    const uint64_t kv = static_cast<uint64_t>(batch * static_cast<uint64_t>(incoming)) * P.kvbpt;  // cost_model.hpp:54-56
    const uint64_t need = kv + kv;  // serving_memory, workspace_factor 1 (cost_model.hpp:59-66)
    const uint64_t headroom = P.budget - ak;
    const bool a2h_c = cached > P.cmax;
    const bool noact = need <= headroom;
    const uint64_t deficit = need - headroom;
    const uint64_t per_layer = static_cast<uint64_t>(cached) * P.abpt;
    // n = floor(sum / per_layer), sum = deficit + per_layer - 1 (maps.hpp:227; no wrap here)
    const uint64_t sum = deficit + (per_layer - 1);
    float rcp;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"(__ull2float_rn(per_layer)));
    const float fq = __fmul_rz(__ull2float_rn(sum), rcp);
    const bool over = fq > P.over_f;
    const uint32_t q = static_cast<uint32_t>(fq);
    const int64_t r = static_cast<int64_t>(sum - q * per_layer);
    const uint32_t n = q + (r >= static_cast<int64_t>(per_layer)) - (r < 0);
    const uint32_t ccode = (over | (n > L)) ? 1u : 2u + n;
    const uint32_t code = (fallback | a2h_c) ? 1u : (noact ? 0u : (hoor ? 1u : ccode));
    const bool a2h = code == 1;
    const uint32_t layers = code >= 2 ? code - 2 : 0u;
    const uint32_t free_now = a2h ? dev : min(layers, dev);
    const uint32_t total = min(pending + (a2h ? L : layers), L);
    const uint32_t th = thr[min(cached, kSmemTab - 1)];
    const uint32_t recompute = (fallback | hoor) ? 1u : static_cast<uint32_t>(total >= th);
    const uint32_t v = (a2h ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS) | (layers << 2) | (free_now << 10) |
                       (recompute << 18) | (fallback ? COLO_V_OFFLOAD_OOR : 0u) |
                       ((!fallback && hoor) ? COLO_V_HEDGE_OOR : 0u) | ((COLO_VD_FREE_LOADBACK + recompute) << 21);
    const bool stream = (sbits[min(charged, kSmemTab - 1) >> 5] >> (charged & 31)) & 1u;
    // (bitwise: no short-circuit branches)
    slow = (max(cached, charged) >= kSmemTab) | ((th == 0xffu) & !fallback & !hoor) | (!fallback & ((kv >> 53) != 0));
    return (code == 0 ? 0u : v) | (stream ? COLO_V_STREAM : 0u);
}

constexpr int kExactU = 4, kExactStages = 3;
template <bool COUNT>
__global__ void __launch_bounds__(kPackThreads, 1) k_decide_exact(const __grid_constant__ ExactParams P) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint32_t* sbits = reinterpret_cast<uint32_t*>(sm);
    uint8_t* thr = reinterpret_cast<uint8_t*>(sbits + kSmemTab / 32);
    uint4* ring = reinterpret_cast<uint4*>(thr + kSmemTab);  // [kExactStages][U][blockDim.x]
    for (uint32_t w = threadIdx.x; w < kSmemTab / 32; w += blockDim.x) {
        uint32_t bits = 0;
        for (uint32_t b = 0; b < 32; ++b) bits |= static_cast<uint32_t>(__ldg(P.tab + 32 * w + b) >> 8) << b;
        sbits[w] = bits;
    }
    for (uint32_t c = threadIdx.x; c < kSmemTab; c += blockDim.x) thr[c] = static_cast<uint8_t>(__ldg(P.tab + c));
    __syncthreads();
    const bool cpa = P.cpa != 0;
    const bool fast = P.fast != 0;
    uint32_t cnt[COLO_NCOUNTERS] = {};
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    constexpr int U = kExactU;
    // Each thread streams its own tuples through a kExactStages-deep cp.async
    // ring in shared memory (slot [stage][u][thread]: conflict-free 16 B
    // reads), so U * kExactStages loads per thread are in flight while it
    // computes -- register loads would be sunk to their uses by the scheduler.
    auto issue = [&](int st, uint64_t base) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + u * stride;
            uint4* dst = ring + (static_cast<uint32_t>(st) * U + u) * blockDim.x + threadIdx.x;
            if (i < P.n)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                             "l"(P.in + i)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint64_t wbase = tid & ~uint64_t(31);  // warp-uniform trip count
#pragma unroll
    for (int st = 0; st < kExactStages - 1; ++st) issue(st, tid + st * stride * U);
    int st = 0;
    for (uint64_t base = tid, wb = wbase; wb < P.n; base += stride * U, wb += stride * U) {
        issue((st + kExactStages - 1) % kExactStages, base + (kExactStages - 1) * stride * U);
        asm volatile("cp.async.wait_group %0;" ::"n"(kExactStages - 1) : "memory");
        // every tuple of the warp's U in range (warp-uniform): no per-tuple guards
        const bool full = wb + (U - 1) * stride + 32 <= P.n;
        auto body = [&](auto guard) {
            constexpr bool G = decltype(guard)::value;
            uint32_t v[U], slowm = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint4* src = ring + (static_cast<uint32_t>(st) * U + u) * blockDim.x + threadIdx.x;
                const uint4 t = (!G || base + u * stride < P.n) ? *src : make_uint4(0, 1, 0, 1);
                bool sl;
                v[u] = exact_verdict_fast(P, t, thr, sbits, sl);
                slowm |= (sl | !fast) ? 1u << u : 0u;
            }
            if (slowm) {  // (the tuples are re-read: keeping them live costs spills)
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if ((slowm >> u) & 1u) v[u] = exact_verdict_slow(P, cpa, P.in[base + u * stride], thr, sbits);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = base + u * stride;
                const bool ok = !G || i < P.n;
                if (ok) __stcs(P.out + i, v[u]);
                if (COUNT) count_warp(v[u], ok, cnt);
            }
        };
        if (full) body(std::false_type{});
        else body(std::true_type{});
        st = st + 1 == kExactStages ? 0 : st + 1;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

// --------------------------------------------------------------- fused path
struct FusedParams {
    MapView sets[kMaxSets];
    uint32_t tab_off[kMaxSets];
    uint32_t str_off[kMaxSets];
    uint32_t nsets, smem_words;
    const uint32_t* prompt;
    const uint32_t* output;
    uint32_t* out;
    const uint64_t* dev_off;
    const uint16_t* dev_set;
    uint32_t ndev;
    uint32_t prev_p, prev_o;  // element base-1 (host pipeline chunks)
    uint64_t base, n;
    uint64_t* counters;
};

// largest d with dev_off[d] <= g (dev_off[0] == 0)
__device__ __forceinline__ uint32_t find_dev(const uint64_t* __restrict__ off, uint32_t ndev, uint64_t g) {
    uint32_t lo = 0, hi = ndev;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// The map-set parameters the fast path needs, held in registers per warp.
struct SetRegs {
    uint32_t max_c, max_i, C, I, W, cpa, tab, str;
    FastDiv fc, fi;
};

__device__ __forceinline__ SetRegs load_set(const FusedParams& P, uint32_t s) {
    const MapView& mv = P.sets[s];
    SetRegs r;
    r.max_c = mv.max_c;
    r.max_i = mv.max_i;
    r.C = mv.C;
    r.I = mv.I;
    r.W = mv.I + 1;
    r.cpa = mv.cpa;
    r.tab = P.tab_off[s];
    r.str = P.str_off[s];
    r.fc = mv.fc;
    r.fi = mv.fi;
    return r;
}

// cached-axis bucket of x tokens (row C = out of range), maps.hpp:102-108
__device__ __forceinline__ uint32_t bucket_c(const SetRegs& r, uint64_t x) {
    return x > r.max_c ? r.C : ceil_div(r.fc, static_cast<uint32_t>(x));
}

// incoming-axis bucket (column I = out of range or zero), maps.hpp:103-108
__device__ __forceinline__ uint32_t bucket_i(const SetRegs& r, uint64_t inc) {
    return (inc > r.max_i || inc == 0) ? r.I : ceil_div(r.fi, static_cast<uint32_t>(inc)) - 1;
}

constexpr uint32_t kChunk = 256;  // queries per warp step: 8 consecutive per lane

// Per-element path for chunks that straddle a device boundary or the array
// end: per-element device lookup, previous query read back from memory.
template <bool FAST, bool COUNT>
__device__ __forceinline__ void fused_slow(const FusedParams& P, const uint32_t* smw, uint64_t cs, uint64_t ce,
                                           uint32_t lane, uint32_t (&cnt)[COLO_NCOUNTERS]) {
    for (uint32_t k = 0; k < 8; ++k) {  // warp-uniform trip count (ballot counting)
        const uint64_t i = cs + lane * 8 + k;
        const bool valid = i < ce;
        uint32_t v = 0;
        if (valid) {
            const uint64_t g = P.base + i;
            const uint32_t dd = find_dev(P.dev_off, P.ndev, g);
            const uint32_t ss = __ldg(P.dev_set + dd);
            const MapView& mv = P.sets[ss];
            uint64_t pc = 0;
            if (g != __ldg(P.dev_off + dd)) {
                const uint32_t pp = i ? __ldg(P.prompt + i - 1) : P.prev_p;
                const uint32_t po = i ? __ldg(P.output + i - 1) : P.prev_o;
                pc = charged_tokens(pp, po, mv.cpa);
            }
            const uint32_t p = __ldg(P.prompt + i), o = __ldg(P.output + i);
            const uint64_t ch = charged_tokens(p, o, mv.cpa);
            const uint64_t inc = static_cast<uint64_t>(p) + o;
            if (FAST) {
                const SetRegs r = load_set(P, ss);
                v = smw[r.tab + bucket_c(r, pc) * r.W + bucket_i(r, inc)] | smw[r.str + bucket_c(r, ch)];
            } else {
                v = compose(mv, mv.off, mv.hed, pc, inc, 1, 0, mv.L) | stream_bits(mv, mv.off, ch);
            }
            P.out[i] = v;
        }
        if (COUNT) count_warp(v, valid, cnt);
    }
}

// Trace-fused features -> verdict through the per-set verdict table.
// Each warp owns a contiguous run of 256-query chunks (lane = 8 consecutive
// queries = two LDG.128 per column); the next chunk's loads are issued before
// the current chunk is evaluated, and the device, its map-set parameters and
// the previous query's cached bucket ride along in registers.
template <bool COUNT>
__global__ void __launch_bounds__(kThreads) k_fused_fast(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(16) uint32_t smw[];
    // COUNT: the counters of one verdict as eight byte fields (counter k in byte
    // k), indexed by its bits 19-24 (offload / hedge nullopt, outcome, stream,
    // stream nullopt); each lane adds these to a packed word and unpacks it
    // before a byte can overflow, instead of eight warp votes per verdict
    __shared__ uint64_t inc_tab[COUNT ? 64 : 1];
    if (COUNT)
        for (uint32_t key = threadIdx.x; key < 64; key += blockDim.x) {
            const uint32_t vd = (key >> 2) & 3u;
            inc_tab[key] = (vd < 3 ? 1ull << (8 * vd) : 0ull) | (static_cast<uint64_t>(key & 1u) << (8 * COLO_CNT_OFFLOAD_OOR)) |
                           (static_cast<uint64_t>((key >> 1) & 1u) << (8 * COLO_CNT_HEDGE_OOR)) |
                           (static_cast<uint64_t>((key >> 4) & 1u) << (8 * COLO_CNT_STREAM)) |
                           (static_cast<uint64_t>((key >> 5) & 1u) << (8 * COLO_CNT_STREAM_OOR)) |
                           (1ull << (8 * COLO_CNT_TOTAL));
        }
    for (uint32_t s = 0; s < P.nsets; ++s) {
        const MapView& mv = P.sets[s];
        const uint32_t nt = (mv.C + 1) * (mv.I + 1);
        for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) smw[P.tab_off[s] + i] = mv.tab[i];
        for (uint32_t i = threadIdx.x; i <= mv.C; i += blockDim.x) smw[P.str_off[s] + i] = mv.str[i];
    }
    __syncthreads();
    uint32_t cnt[COLO_NCOUNTERS] = {};
    uint64_t pk = 0;                      // COUNT: packed byte counters of this lane's fast-path verdicts
    uint32_t pkn = 0;                     // verdicts in pk (< 256)
    uint32_t lc[COLO_NCOUNTERS] = {};     // this lane's unpacked counts
    auto unpack = [&]() {
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) lc[k] += static_cast<uint32_t>((pk >> (8 * k)) & 0xffu);
        pk = 0;
        pkn = 0;
    };
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t nchunks = (P.n + kChunk - 1) / kChunk;
    const uint64_t per = (nchunks + nwarps - 1) / nwarps;
    const uint64_t c0 = gwarp * per, c1 = min(c0 + per, nchunks);
    if (c0 < c1) {
        const uint64_t i_begin = c0 * kChunk, i_end = min(P.n, c1 * kChunk);
        const uint64_t g0 = P.base + i_begin;
        uint32_t d = find_dev(P.dev_off, P.ndev, g0);
        uint64_t hi = __ldg(P.dev_off + d + 1);
        SetRegs R = load_set(P, __ldg(P.dev_set + d));
        uint32_t prev_b = 0;  // cached bucket of the previous query (0 = nothing cached)
        if (g0 != __ldg(P.dev_off + d)) {
            const uint32_t pp = i_begin ? __ldg(P.prompt + i_begin - 1) : P.prev_p;
            const uint32_t po = i_begin ? __ldg(P.output + i_begin - 1) : P.prev_o;
            prev_b = bucket_c(R, charged_tokens(pp, po, R.cpa));
        }
        const uint4* p4 = reinterpret_cast<const uint4*>(P.prompt);
        const uint4* o4 = reinterpret_cast<const uint4*>(P.output);
        uint4 cp0, cp1, co0, co1;
        if (i_begin + kChunk <= i_end) {
            const uint64_t q = (i_begin + lane * 8) >> 2;
            cp0 = __ldcs(p4 + q);
            cp1 = __ldcs(p4 + q + 1);
            co0 = __ldcs(o4 + q);
            co1 = __ldcs(o4 + q + 1);
        }
        for (uint64_t cs = i_begin; cs < i_end; cs += kChunk) {
            const uint64_t ce = min(cs + kChunk, i_end);
            uint4 np0, np1, no0, no1;
            if (cs + 2 * kChunk <= i_end) {  // prefetch the next full chunk
                const uint64_t q = (cs + kChunk + lane * 8) >> 2;
                np0 = __ldcs(p4 + q);
                np1 = __ldcs(p4 + q + 1);
                no0 = __ldcs(o4 + q);
                no1 = __ldcs(o4 + q + 1);
            }
            if (ce - cs == kChunk && P.base + ce <= hi) {
                const uint32_t pv[8] = {cp0.x, cp0.y, cp0.z, cp0.w, cp1.x, cp1.y, cp1.z, cp1.w};
                const uint32_t ov[8] = {co0.x, co0.y, co0.z, co0.w, co1.x, co1.y, co1.z, co1.w};
                uint32_t cb[8], ib[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    cb[k] = bucket_c(R, charged_tokens(pv[k], ov[k], R.cpa));
                    ib[k] = bucket_i(R, static_cast<uint64_t>(pv[k]) + ov[k]);
                }
                const uint32_t up = __shfl_up_sync(FULL, cb[7], 1);
                uint32_t pb = lane == 0 ? prev_b : up;
                uint32_t v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    v[k] = smw[R.tab + pb * R.W + ib[k]] | smw[R.str + cb[k]];
                    pb = cb[k];
                }
                uint4* dst = reinterpret_cast<uint4*>(P.out + cs + lane * 8);
                __stcs(dst, make_uint4(v[0], v[1], v[2], v[3]));
                __stcs(dst + 1, make_uint4(v[4], v[5], v[6], v[7]));
                if (COUNT) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) pk += inc_tab[(v[k] >> 19) & 63u];
                    pkn += 8;
                    if (pkn > 240) unpack();  // (warp-uniform: every lane takes 8 per chunk)
                }
                prev_b = __shfl_sync(FULL, cb[7], 31);
            } else {
                fused_slow<true, COUNT>(P, smw, cs, ce, lane, cnt);
                if (ce < i_end) {  // re-seat the warp state on the device of the next query
                    d = find_dev(P.dev_off, P.ndev, P.base + ce);
                    hi = __ldg(P.dev_off + d + 1);
                    R = load_set(P, __ldg(P.dev_set + d));
                    prev_b = 0;
                    if (P.base + ce != __ldg(P.dev_off + d))
                        prev_b = bucket_c(R, charged_tokens(__ldg(P.prompt + ce - 1), __ldg(P.output + ce - 1), R.cpa));
                }
            }
            cp0 = np0;
            cp1 = np1;
            co0 = no0;
            co1 = no1;
        }
    }
    if (COUNT) {
        unpack();
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) cnt[k] += __reduce_add_sync(FULL, lc[k]);
    }
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

// General trace-fused path: compose() per query from the cell tables.
template <bool COUNT>
__global__ void __launch_bounds__(kThreads) k_fused_gen(const __grid_constant__ FusedParams P) {
    uint32_t cnt[COLO_NCOUNTERS] = {};
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t nchunks = (P.n + kChunk - 1) / kChunk;
    for (uint64_t c = gwarp; c < nchunks; c += nwarps)
        fused_slow<false, COUNT>(P, nullptr, c * kChunk, min((c + 1) * kChunk, P.n), lane, cnt);
    if (COUNT) flush_warp_counters(cnt, P.counters);
}

colo_status launch_fused(colo_ctx* ctx, cudaStream_t stream, const colo_mapset* const* sets, size_t nsets,
                         const uint32_t* d_prompt, const uint32_t* d_output, uint64_t base, size_t n,
                         const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev, uint32_t* d_out,
                         uint64_t* d_counters, uint32_t prev_p, uint32_t prev_o) {
    FusedParams P{};
    bool fast = true;
    uint32_t words = 0;
    for (size_t s = 0; s < nsets; ++s) {
        P.sets[s] = make_view(sets[s]);
        fast = fast && sets[s]->fast;
        P.tab_off[s] = words;
        words += (sets[s]->C + 1) * (sets[s]->I + 1);
        P.str_off[s] = words;
        words += sets[s]->C + 1;
    }
    size_t smem = static_cast<size_t>(words) * 4;
    if (!fast || smem > 160 * 1024) {
        fast = false;
        smem = 0;
    }
    P.nsets = static_cast<uint32_t>(nsets);
    P.smem_words = words;
    P.prompt = d_prompt;
    P.output = d_output;
    P.out = d_out;
    P.dev_off = d_dev_offsets;
    P.dev_set = d_dev_set;
    P.ndev = static_cast<uint32_t>(ndev);
    P.prev_p = prev_p;
    P.prev_o = prev_o;
    P.base = base;
    P.n = n;
    P.counters = d_counters;
    const void* fn;
    if (fast) fn = d_counters ? (const void*)k_fused_fast<true> : (const void*)k_fused_fast<false>;
    else fn = d_counters ? (const void*)k_fused_gen<true> : (const void*)k_fused_gen<false>;
    if (smem > 48 * 1024) COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int blocks = blocks_for(ctx, fn, kThreads, smem);
    const uint64_t need_blocks = (n + kChunk * (kThreads / 32) - 1) / (kChunk * (kThreads / 32));
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(std::max<uint64_t>(need_blocks, 1));
    void* args[] = {&P};
    COLO_LAUNCHED(ctx);
    COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), args, smem, stream));
    return COLO_OK;
}

colo_status check_sets(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets) {
    if (!sets || nsets == 0 || nsets > kMaxSets) return set_err(ctx, COLO_EINVAL, "need 1..16 map sets");
    for (size_t s = 0; s < nsets; ++s)
        if (!sets[s]) return set_err(ctx, COLO_EINVAL, "null map set");
    return COLO_OK;
}

colo_status grow_pipe(colo_ctx* ctx, size_t bytes) {
    if (ctx->pipe_bytes >= bytes) return COLO_OK;
    if (ctx->d_pipe) cudaFree(ctx->d_pipe);
    ctx->d_pipe = nullptr;
    ctx->pipe_bytes = 0;
    COLO_CK(ctx, cudaMalloc(&ctx->d_pipe, bytes));
    ctx->pipe_bytes = bytes;
    return COLO_OK;
}

colo_status launch_decide(colo_ctx* ctx, cudaStream_t stream, const colo_mapset* ms, const colo_tuple* d_in, size_t n,
                          uint32_t* d_out, uint64_t* d_counters) {
    DecideParams P{};
    P.mv = make_view(ms);
    P.in = reinterpret_cast<const uint4*>(d_in);
    P.out = d_out;
    P.n = n;
    P.counters = d_counters;
    const size_t smem = ((P.mv.off_bytes + 15u) & ~15u) + P.mv.hed_bytes;
    const bool use_smem = smem <= 96 * 1024;
    const bool fastgrid = P.mv.hsame && P.mv.fc.d > 1 && P.mv.fi.d > 1 && P.mv.fb.d > 1;
    const size_t packed = packed_image_bytes(P.mv);
    if (packed) {  // packed cells in shared memory
        if (ms->d_img && ms->img_bytes == packed) {
            P.img = ms->d_img;
            P.img_bytes = static_cast<uint32_t>(packed);
        }
        const void* fn = d_counters ? (const void*)k_decide_packed<true> : (const void*)k_decide_packed<false>;
        COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)packed));
        int blocks = blocks_for(ctx, fn, kPackThreads, packed);
        const uint64_t need_blocks = (n + kPackThreads - 1) / kPackThreads;
        if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
        void* args[] = {&P};
        COLO_LAUNCHED(ctx);
        COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kPackThreads), args, packed, stream));
        return COLO_OK;
    }
    if (use_smem && !(reinterpret_cast<uintptr_t>(d_in) & 15u)) {  // TMA pipeline
        // 4 stages while the cells are small; 2 for sweep-size grids, so two
        // CTAs still fit next to 64 KB of cells
        const bool deep = smem <= 32 * 1024;
        const size_t dyn = (deep ? kStages : 2u) * kTile * 16 + 64 + smem;
        const bool fast = P.mv.hsame && P.mv.fc.d > 1 && P.mv.fi.d > 1 && P.mv.fb.d > 1;
        const void* fn;
        if (deep)
            fn = d_counters ? (fast ? (const void*)k_decide_tma<true, true, kStages> : (const void*)k_decide_tma<true, false, kStages>)
                            : (fast ? (const void*)k_decide_tma<false, true, kStages> : (const void*)k_decide_tma<false, false, kStages>);
        else
            fn = d_counters ? (fast ? (const void*)k_decide_tma<true, true, 2> : (const void*)k_decide_tma<true, false, 2>)
                            : (fast ? (const void*)k_decide_tma<false, true, 2> : (const void*)k_decide_tma<false, false, 2>);
        COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        int blocks = blocks_for(ctx, fn, kThreads, dyn);
        const uint64_t ntiles = (n + kTile - 1) / kTile;
        if (static_cast<uint64_t>(blocks) > ntiles) blocks = static_cast<int>(ntiles);
        void* args[] = {&P};
        COLO_LAUNCHED(ctx);
        COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), args, dyn, stream));
        return COLO_OK;
    }
    const void* fn;
    if (use_smem) fn = d_counters ? (const void*)k_decide<true, true> : (const void*)k_decide<true, false>;
    else fn = d_counters ? (const void*)k_decide<false, true> : (const void*)k_decide<false, false>;
    const size_t dyn = use_smem ? smem : 0;
    if (dyn > 48 * 1024) COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    int blocks = blocks_for(ctx, fn, kThreads, dyn);
    const uint64_t need_blocks = (n + kThreads - 1) / kThreads;
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
    void* args[] = {&P};
    COLO_LAUNCHED(ctx);
    COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), args, dyn, stream));
    return COLO_OK;
}

}  // namespace

namespace colo {

colo_status build_pack_image(colo_ctx* ctx, colo_mapset* ms) {
    const MapView mv = make_view(ms);
    const size_t bytes = packed_image_bytes(mv);
    if (bytes == 0) return COLO_OK;
    if (!ms->d_img) {
        COLO_CK(ctx, cudaMalloc(&ms->d_img, bytes));
        ms->img_bytes = static_cast<uint32_t>(bytes);
    }
    COLO_CK(ctx, cudaMemsetAsync(ms->d_img, 0, bytes, ctx->stream));
    COLO_LAUNCHED(ctx);
    k_pack_image<<<148, 256, 0, ctx->stream>>>(mv, ms->d_img);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

}  // namespace colo

extern "C" {

colo_status colo_decide(colo_ctx* ctx, const colo_mapset* ms, const colo_tuple* d_in, size_t n, uint32_t* d_out,
                        uint64_t* d_counters) {
    if (!ctx || !ms || (n && (!d_in || !d_out))) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    const colo_status st = check_align(ctx, d_in);
    if (st != COLO_OK) return st;
    return launch_decide(ctx, ctx->stream, ms, d_in, n, d_out, d_counters);
}

colo_status colo_decide_exact(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, colo_mode mode, uint64_t assumed,
                              const colo_tuple* d_in, size_t n, uint32_t* d_out, uint64_t* d_counters) {
    if (!ctx || !m || !g || (n && (!d_in || !d_out))) return COLO_EINVAL;
    colo_status st = colo_validate_profile_pair(m, g);
    if (st != COLO_OK) return set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
    if (check_model_limits(m) != COLO_OK) return set_err(ctx, COLO_EINVAL, "num_layers > 253");
    if (n == 0) return COLO_OK;
    st = check_align(ctx, d_in);
    if (st != COLO_OK) return st;
    ExactParams P{};
    P.m = *m;
    P.g = *g;
    P.budget = g->capacity_bytes - g->runtime_reserve_bytes - m->weights_bytes;
    P.assumed = assumed;
    P.cpa = mode == COLO_CPA;
    P.in = reinterpret_cast<const uint4*>(d_in);
    P.out = d_out;
    P.n = n;
    P.counters = d_counters;
    P.L = static_cast<uint32_t>(m->num_layers);
    P.abpt = m->act_bytes_per_token_per_layer;
    P.kvbpt = m->kv_bytes_per_token;
    P.ak = m->num_layers * m->act_bytes_per_token_per_layer + (P.cpa ? m->kv_bytes_per_token : 0ull);
    P.wf_mode = m->workspace_factor == 1.0 ? 1u : 0u;
    P.fast = P.wf_mode == 1 && P.abpt >= 1 && P.abpt < (1ull << 40) && P.ak < (1ull << 50);
    P.cmax = P.ak == 0 ? 0xffffffffu : static_cast<uint32_t>(std::min<uint64_t>(P.budget / P.ak, 0xffffffffull));
    P.over_f = static_cast<float>(P.L + 2);
    // per-value tables: rebuilt only when (model, gpu, mode, assumed) changes
    unsigned char key[sizeof(ctx->htab_key)] = {};
    std::memcpy(key, m, sizeof(colo_model));
    std::memcpy(key + sizeof(colo_model), g, sizeof(colo_gpu));
    std::memcpy(key + sizeof(colo_model) + sizeof(colo_gpu), &P.cpa, sizeof(uint32_t));
    std::memcpy(key + sizeof(colo_model) + sizeof(colo_gpu) + 8, &assumed, sizeof(uint64_t));
    if (!ctx->d_htab) COLO_CK(ctx, cudaMalloc(&ctx->d_htab, kExactTab * sizeof(uint16_t)));
    if (!ctx->htab_valid || std::memcmp(key, ctx->htab_key, sizeof(key)) != 0) {
        COLO_LAUNCHED(ctx);
        k_exact_tab<<<kExactTab / 256, 256, 0, ctx->stream>>>(*m, *g, P.cpa, assumed, P.budget, ctx->d_htab);
        COLO_CK(ctx, cudaGetLastError());
        std::memcpy(ctx->htab_key, key, sizeof(key));
        ctx->htab_valid = true;
    }
    P.tab = ctx->d_htab;
    const void* fn = d_counters ? (const void*)k_decide_exact<true> : (const void*)k_decide_exact<false>;
    const size_t dyn = kSmemTab / 8 + kSmemTab + sizeof(uint4) * kExactStages * kExactU * kPackThreads;
    COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    int blocks = blocks_for(ctx, fn, kPackThreads, dyn);
    const uint64_t need_blocks = (n + kPackThreads - 1) / kPackThreads;
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
    void* args[] = {&P};
    COLO_LAUNCHED(ctx);
    COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kPackThreads), args, dyn, ctx->stream));
    return COLO_OK;
}

colo_status colo_features_decide(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const uint32_t* d_prompt,
                                 const uint32_t* d_output, size_t n, const uint64_t* d_dev_offsets,
                                 const uint16_t* d_dev_set, size_t ndev, uint32_t* d_out, uint64_t* d_counters) {
    if (!ctx || ndev == 0 || !d_dev_offsets || !d_dev_set) return COLO_EINVAL;
    const colo_status st = check_sets(ctx, sets, nsets);
    if (st != COLO_OK) return st;
    if (n == 0) return COLO_OK;
    if (check_align(ctx, d_prompt) || check_align(ctx, d_output) || check_align(ctx, d_out)) return COLO_EINVAL;
    return launch_fused(ctx, ctx->stream, sets, nsets, d_prompt, d_output, 0, n, d_dev_offsets, d_dev_set, ndev, d_out,
                        d_counters, 0, 0);
}

colo_status colo_features_decide_host(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets,
                                      const uint32_t* h_prompt, const uint32_t* h_output, size_t n,
                                      const uint64_t* h_dev_offsets, const uint16_t* h_dev_set, size_t ndev,
                                      uint32_t* h_out, uint64_t* h_counters) {
    if (!ctx || ndev == 0 || !h_dev_offsets || !h_dev_set || (n && (!h_prompt || !h_output || !h_out)))
        return COLO_EINVAL;
    colo_status st = check_sets(ctx, sets, nsets);
    if (st != COLO_OK) return st;
    if (h_dev_offsets[0] != 0 || h_dev_offsets[ndev] != n) return set_err(ctx, COLO_EINVAL, "device offsets must span [0, n]");
    for (size_t d = 0; d < ndev; ++d) {
        if (h_dev_offsets[d + 1] < h_dev_offsets[d]) return set_err(ctx, COLO_EINVAL, "device offsets not monotone");
        if (h_dev_set[d] >= nsets) return set_err(ctx, COLO_EINVAL, "device map-set index out of range");
    }
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    const size_t CH = size_t(1) << 24;  // queries per pipeline chunk
    const size_t chunk_bytes = CH * 12;
    const size_t meta = ((ndev + 1) * 8 + ndev * 2 + 255) & ~size_t(255);
    st = grow_pipe(ctx, 2 * chunk_bytes + meta);
    if (st != COLO_OK) return st;
    auto* base = static_cast<uint8_t*>(ctx->d_pipe);
    auto* d_off = reinterpret_cast<uint64_t*>(base + 2 * chunk_bytes);
    auto* d_set = reinterpret_cast<uint16_t*>(base + 2 * chunk_bytes + (ndev + 1) * 8);
    cudaStream_t ss[2] = {ctx->stream, ctx->aux};
    COLO_CK(ctx, cudaMemcpyAsync(d_off, h_dev_offsets, (ndev + 1) * 8, cudaMemcpyHostToDevice, ss[0]));
    COLO_CK(ctx, cudaMemcpyAsync(d_set, h_dev_set, ndev * 2, cudaMemcpyHostToDevice, ss[0]));
    uint64_t* d_cnt = h_counters ? ctx->d_counters : nullptr;
    if (d_cnt) COLO_CK(ctx, cudaMemsetAsync(d_cnt, 0, sizeof(uint64_t) * COLO_NCOUNTERS, ss[0]));
    cudaEvent_t ready;
    COLO_CK(ctx, cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    COLO_CK(ctx, cudaEventRecord(ready, ss[0]));
    COLO_CK(ctx, cudaStreamWaitEvent(ss[1], ready, 0));
    cudaEventDestroy(ready);
    for (size_t c0 = 0, k = 0; c0 < n; c0 += CH, ++k) {
        const size_t len = std::min(CH, n - c0);
        cudaStream_t s = ss[k & 1];
        auto* buf = base + (k & 1) * chunk_bytes;
        auto* dp = reinterpret_cast<uint32_t*>(buf);
        auto* dq = reinterpret_cast<uint32_t*>(buf + CH * 4);
        auto* dv = reinterpret_cast<uint32_t*>(buf + CH * 8);
        COLO_CK(ctx, cudaMemcpyAsync(dp, h_prompt + c0, len * 4, cudaMemcpyHostToDevice, s));
        COLO_CK(ctx, cudaMemcpyAsync(dq, h_output + c0, len * 4, cudaMemcpyHostToDevice, s));
        st = launch_fused(ctx, s, sets, nsets, dp, dq, c0, len, d_off, d_set, ndev, dv, d_cnt,
                          c0 ? h_prompt[c0 - 1] : 0, c0 ? h_output[c0 - 1] : 0);
        if (st != COLO_OK) return st;
        COLO_CK(ctx, cudaMemcpyAsync(h_out + c0, dv, len * 4, cudaMemcpyDeviceToHost, s));
    }
    COLO_CK(ctx, cudaStreamSynchronize(ss[1]));
    COLO_CK(ctx, cudaStreamSynchronize(ss[0]));
    if (h_counters) {
        uint64_t tmp[COLO_NCOUNTERS];
        COLO_CK(ctx, cudaMemcpy(tmp, d_cnt, sizeof tmp, cudaMemcpyDeviceToHost));
        for (int i = 0; i < COLO_NCOUNTERS; ++i) h_counters[i] += tmp[i];
    }
    return COLO_OK;
}

colo_status colo_decide_host(colo_ctx* ctx, const colo_mapset* ms, const colo_tuple* h_in, size_t n, uint32_t* h_out,
                             uint64_t* h_counters) {
    if (!ctx || !ms || (n && (!h_in || !h_out))) return COLO_EINVAL;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    const size_t CH = size_t(1) << 23;
    const size_t chunk_bytes = CH * 20;
    colo_status st = grow_pipe(ctx, 2 * chunk_bytes);
    if (st != COLO_OK) return st;
    auto* base = static_cast<uint8_t*>(ctx->d_pipe);
    cudaStream_t ss[2] = {ctx->stream, ctx->aux};
    uint64_t* d_cnt = h_counters ? ctx->d_counters : nullptr;
    cudaEvent_t ready;
    COLO_CK(ctx, cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    if (d_cnt) COLO_CK(ctx, cudaMemsetAsync(d_cnt, 0, sizeof(uint64_t) * COLO_NCOUNTERS, ss[0]));
    COLO_CK(ctx, cudaEventRecord(ready, ss[0]));
    COLO_CK(ctx, cudaStreamWaitEvent(ss[1], ready, 0));
    cudaEventDestroy(ready);
    for (size_t c0 = 0, k = 0; c0 < n; c0 += CH, ++k) {
        const size_t len = std::min(CH, n - c0);
        cudaStream_t s = ss[k & 1];
        auto* buf = base + (k & 1) * chunk_bytes;
        auto* din = reinterpret_cast<colo_tuple*>(buf);
        auto* dout = reinterpret_cast<uint32_t*>(buf + CH * 16);
        COLO_CK(ctx, cudaMemcpyAsync(din, h_in + c0, len * 16, cudaMemcpyHostToDevice, s));
        st = launch_decide(ctx, s, ms, din, len, dout, d_cnt);
        if (st != COLO_OK) return st;
        COLO_CK(ctx, cudaMemcpyAsync(h_out + c0, dout, len * 4, cudaMemcpyDeviceToHost, s));
    }
    COLO_CK(ctx, cudaStreamSynchronize(ss[1]));
    COLO_CK(ctx, cudaStreamSynchronize(ss[0]));
    if (h_counters) {
        uint64_t tmp[COLO_NCOUNTERS];
        COLO_CK(ctx, cudaMemcpy(tmp, d_cnt, sizeof tmp, cudaMemcpyDeviceToHost));
        for (int i = 0; i < COLO_NCOUNTERS; ++i) h_counters[i] += tmp[i];
    }
    return COLO_OK;
}

}  // extern "C"
