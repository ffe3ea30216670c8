// colo_runtime.cu -- map sets (K3), decide kernels (K1+K2), trace-fused
// features->decision, host-buffer pipelines, bench-scale trace synthesis.
//
// Data layout in HBM: traces are SoA (prompt u32[],
// output u32[], arrival f64[]) partitioned by device with CSR offsets; tuples
// are 16-B AoS records (one LDG.128 each); verdicts are packed u32.  Map cells
// are bytes and are staged into shared memory once per CTA.
// Reference paths are relative to /root/reference/proj/.
#include <algorithm>
#include <cstring>
#include <vector>

#include "colo_internal.h"

using namespace colo;

namespace {

constexpr int kThreads = 256;

// ---------------------------------------------------------------- map build
// build_offloading_map, maps.hpp:233-252: one thread per cell, cell (ci,ii,bi)
// evaluated at (ci*sc, (ii+1)*si, (bi+1)*sb), row-major.
__global__ void k_build_offload(colo_model m, uint64_t budget, uint32_t cpa, uint64_t sc, uint64_t si, uint64_t sb,
                                uint32_t I, uint32_t B, uint32_t ncells, uint8_t* __restrict__ out) {
    uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncells) return;
    uint32_t ci = idx / (I * B), r = idx % (I * B), ii = r / B, bi = r % B;
    out[idx] = offload_cell_code(m, budget, cpa != 0, ci * sc, (ii + 1) * si, (bi + 1) * sb);
}

// build_hedging_map, maps.hpp:358-384: cell (ci, fi) at cached = (ci+1)*step.
__global__ void k_build_hedge(colo_model m, colo_gpu g, uint32_t cpa, uint64_t step, uint64_t assumed, uint32_t F,
                              uint32_t ncells, uint8_t* __restrict__ out) {
    uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= ncells) return;
    uint32_t ci = idx / F, fi = idx % F;
    uint64_t cached = (ci + 1) * step;
    double recompute = hedge_recompute_time(m, cpa != 0, cached, assumed);
    double residual = hedge_residual_load_time(m, g, cached, fi);
    out[idx] = residual > recompute ? 1 : 0;  // maps.hpp:380 (strict; ties load back)
}

// Trace-fused verdict table: the composed verdict for
// (cached bucket ci | oor, incoming bucket ii | oor, batch 1, pending 0, dev L)
// evaluated at a representative point of each bucket with the same compose()
// every other kernel uses; valid when the hedge step equals the cached step
// (then the hedge bucket is ci - 1).  Stream bits per charged bucket likewise.
__global__ void k_build_tab(MapView mv, uint32_t* __restrict__ tab, uint32_t* __restrict__ str) {
    uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t W = mv.I + 1;
    if (idx >= (mv.C + 1) * W) return;
    uint32_t ci = idx / W, ii = idx % W;
    uint64_t cached = ci < mv.C ? static_cast<uint64_t>(ci) * mv.fc.d : static_cast<uint64_t>(mv.max_c) + 1;
    uint64_t inc = ii < mv.I ? static_cast<uint64_t>(ii + 1) * mv.fi.d : static_cast<uint64_t>(mv.max_i) + 1;
    tab[idx] = compose(mv, mv.off, mv.hed, cached, inc, 1, 0, mv.L);
    if (ii == 0) str[ci] = stream_bits(mv, mv.off, cached);
}

// --------------------------------------------------------------- decide
struct DecideParams {
    MapView mv;
    const uint4* in;
    uint32_t* out;
    uint64_t n;
    uint64_t* counters;
};

// One LDG.128 tuple -> one u32 verdict per element, cells in shared memory
// (SMEM) or read through L1/L2 (large sweep grids).  Persistent grid-stride
// loop, 4 tuples in flight per thread.
template <bool SMEM, bool COUNT>
__global__ void __launch_bounds__(kThreads) k_decide(const __grid_constant__ DecideParams P) {
    extern __shared__ __align__(16) uint8_t sm[];
    const MapView& mv = P.mv;
    const uint8_t* off = mv.off;
    const uint8_t* hed = mv.hed;
    if (SMEM) {
        uint32_t ob = (mv.off_bytes + 15u) & ~15u;
        for (uint32_t i = threadIdx.x; i < mv.off_bytes; i += blockDim.x) sm[i] = mv.off[i];
        for (uint32_t i = threadIdx.x; i < mv.hed_bytes; i += blockDim.x) sm[ob + i] = mv.hed[i];
        __syncthreads();
        off = sm;
        hed = sm + ob;
    }
    uint64_t cnt[COLO_NCOUNTERS];
    if (COUNT)
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) cnt[k] = 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    constexpr int U = 4;
    for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; base < P.n; base += stride * U) {
        uint4 t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint64_t i = base + u * stride;
            if (i < P.n) t[u] = __ldcs(P.in + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint64_t i = base + u * stride;
            if (i < P.n) {
                uint32_t batch = t[u].w & 0xffffu, pending = (t[u].w >> 16) & 0xffu, dev = t[u].w >> 24;
                uint32_t v = compose(mv, off, hed, t[u].x, t[u].y, batch, pending, dev) | stream_bits(mv, off, t[u].z);
                __stcs(P.out + i, v);
                if (COUNT) count_verdict(v, cnt);
            }
        }
    }
    if (COUNT) flush_counters(cnt, P.counters);
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
};

// Exact per-query verdicts: offload_cell_decision (maps.hpp:215-231) at the
// raw point + the hedge inequality (maps.hpp:341-356, 380) evaluated directly.
template <bool COUNT>
__global__ void __launch_bounds__(kThreads) k_decide_exact(const __grid_constant__ ExactParams P) {
    uint64_t cnt[COLO_NCOUNTERS];
    if (COUNT)
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) cnt[k] = 0;
    const uint32_t L = static_cast<uint32_t>(P.m.num_layers);
    const bool cpa = P.cpa != 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P.n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint4 t = __ldcs(P.in + i);
        uint32_t cached = t.x, incoming = t.y, charged = t.z;
        uint32_t batch = t.w & 0xffffu, pending = (t.w >> 16) & 0xffu, dev = t.w >> 24;
        uint32_t fallback = incoming == 0 || batch == 0;
        uint32_t code = fallback ? 1u : offload_cell_code(P.m, P.budget, cpa, cached, incoming, batch);
        uint32_t v;
        if (code == 0) {
            v = pack_verdict(0, 0, 0, 0, 0, 0, COLO_VD_ADMIT);
        } else {
            uint32_t layers = code >= 2 ? code - 2 : 0;
            uint32_t free_now = code == 1 ? dev : min(layers, dev);
            uint32_t total = min(pending + (code == 1 ? L : layers), L);
            uint32_t recompute = 1, hedge_oor = 0;
            if (!fallback) {
                if (cached == 0) {
                    hedge_oor = 1;
                } else {
                    double rc = hedge_recompute_time(P.m, cpa, cached, P.assumed);
                    double res = hedge_residual_load_time(P.m, P.g, cached, total);
                    recompute = res > rc;
                }
            }
            v = pack_verdict(code == 1 ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS, layers, free_now, recompute, fallback,
                             hedge_oor, recompute ? COLO_VD_RECOMPUTE_DROP : COLO_VD_FREE_LOADBACK);
        }
        if (offload_cell_code(P.m, P.budget, cpa, charged, 1, 1) == 1) v |= COLO_V_STREAM;
        __stcs(P.out + i, v);
        if (COUNT) count_verdict(v, cnt);
    }
    if (COUNT) flush_counters(cnt, P.counters);
}

// ------------------------------------------------------- trace-fused decide
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

__device__ __forceinline__ uint32_t bucket_c(const MapView& mv, uint64_t x) {
    return x > mv.max_c ? mv.C : ceil_div(mv.fc, static_cast<uint32_t>(x));
}

__device__ __forceinline__ uint32_t bucket_i(const MapView& mv, uint64_t inc) {
    return (inc > mv.max_i || inc == 0) ? mv.I : ceil_div(mv.fi, static_cast<uint32_t>(inc)) - 1;
}

// largest d with dev_off[d] <= g (dev_off[0] == 0)
__device__ __forceinline__ uint32_t find_dev(const uint64_t* __restrict__ off, uint32_t ndev, uint64_t g) {
    uint32_t lo = 0, hi = ndev;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= g) lo = mid; else hi = mid;
    }
    return lo;
}

// One element, any path: previous charged tokens (0 at a device start) -> verdict.
template <bool FAST>
__device__ __forceinline__ uint32_t fused_one(const FusedParams& P, const uint32_t* sm, uint32_t s, uint64_t prev_ch,
                                              uint32_t p, uint32_t o) {
    const MapView& mv = P.sets[s];
    uint64_t ch = charged_tokens(p, o, mv.cpa);
    uint64_t inc = static_cast<uint64_t>(p) + o;
    if (FAST) {
        const uint32_t* tab = sm + P.tab_off[s];
        const uint32_t* str = sm + P.str_off[s];
        return tab[bucket_c(mv, prev_ch) * (mv.I + 1) + bucket_i(mv, inc)] | str[bucket_c(mv, ch)];
    }
    return compose(mv, mv.off, mv.hed, prev_ch, inc, 1, 0, mv.L) | stream_bits(mv, mv.off, ch);
}

// Each warp owns a contiguous run of 128-element chunks (lane = 4 consecutive
// queries, one LDG.128 per column); the device, its map set and the previous
// query's charged tokens ride along in registers, so the common chunk costs
// two vector loads, per-element bucket arithmetic, two shared-memory table
// reads and one vector store.  Chunks that touch a device boundary or the
// array tail take the per-element path.
template <bool FAST, bool COUNT>
__global__ void __launch_bounds__(kThreads) k_fused(const __grid_constant__ FusedParams P) {
    extern __shared__ __align__(16) uint32_t smw[];
    if (FAST) {
        for (uint32_t s = 0; s < P.nsets; ++s) {
            const MapView& mv = P.sets[s];
            uint32_t nt = (mv.C + 1) * (mv.I + 1);
            for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) smw[P.tab_off[s] + i] = mv.tab[i];
            for (uint32_t i = threadIdx.x; i <= mv.C; i += blockDim.x) smw[P.str_off[s] + i] = mv.str[i];
        }
        __syncthreads();
    }
    uint64_t cnt[COLO_NCOUNTERS];
    if (COUNT)
#pragma unroll
        for (int k = 0; k < COLO_NCOUNTERS; ++k) cnt[k] = 0;

    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gwarp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint64_t nchunks = (P.n + 127) / 128;
    const uint64_t per = (nchunks + nwarps - 1) / nwarps;
    const uint64_t c0 = gwarp * per;
    const uint64_t c1 = min(c0 + per, nchunks);
    if (c0 < c1) {
        const uint64_t i_begin = c0 * 128, i_end = min(P.n, c1 * 128);
        // warp state: device, its end, its set, previous query's charged tokens
        uint64_t g0 = P.base + i_begin;
        uint32_t d = find_dev(P.dev_off, P.ndev, g0);
        uint64_t hi = __ldg(P.dev_off + d + 1);
        uint32_t s = __ldg(P.dev_set + d);
        uint64_t prev_ch = 0;
        if (g0 != __ldg(P.dev_off + d)) {
            uint32_t pp = i_begin ? __ldg(P.prompt + i_begin - 1) : P.prev_p;
            uint32_t po = i_begin ? __ldg(P.output + i_begin - 1) : P.prev_o;
            prev_ch = charged_tokens(pp, po, P.sets[s].cpa);
        }
        for (uint64_t cs = i_begin; cs < i_end; cs += 128) {
            const uint64_t ce = min(cs + 128, i_end);
            if (ce - cs == 128 && P.base + ce <= hi) {
                const MapView& mv = P.sets[s];
                const uint64_t i0 = cs + lane * 4;
                uint4 p4 = __ldcs(reinterpret_cast<const uint4*>(P.prompt + i0));
                uint4 o4 = __ldcs(reinterpret_cast<const uint4*>(P.output + i0));
                uint32_t pv[4] = {p4.x, p4.y, p4.z, p4.w}, ov[4] = {o4.x, o4.y, o4.z, o4.w};
                uint32_t v[4];
                if (FAST) {
                    const uint32_t* tab = smw + P.tab_off[s];
                    const uint32_t* str = smw + P.str_off[s];
                    const uint32_t W = mv.I + 1;
                    uint32_t prev_b = bucket_c(mv, prev_ch);
                    uint32_t cb[4], ib[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        cb[k] = bucket_c(mv, charged_tokens(pv[k], ov[k], mv.cpa));
                        ib[k] = bucket_i(mv, static_cast<uint64_t>(pv[k]) + ov[k]);
                    }
                    uint32_t up = __shfl_up_sync(0xffffffffu, cb[3], 1);
                    uint32_t pb = lane == 0 ? prev_b : up;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[k] = tab[pb * W + ib[k]] | str[cb[k]];
                        pb = cb[k];
                    }
                } else {
                    uint64_t ch[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) ch[k] = charged_tokens(pv[k], ov[k], mv.cpa);
                    uint64_t up = __shfl_up_sync(0xffffffffu, ch[3], 1);
                    uint64_t pc = lane == 0 ? prev_ch : up;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        v[k] = compose(mv, mv.off, mv.hed, pc, static_cast<uint64_t>(pv[k]) + ov[k], 1, 0, mv.L) |
                               stream_bits(mv, mv.off, ch[k]);
                        pc = ch[k];
                    }
                }
                __stcs(reinterpret_cast<uint4*>(P.out + i0), make_uint4(v[0], v[1], v[2], v[3]));
                if (COUNT)
#pragma unroll
                    for (int k = 0; k < 4; ++k) count_verdict(v[k], cnt);
                prev_ch = __shfl_sync(0xffffffffu, charged_tokens(pv[3], ov[3], mv.cpa), 31);
            } else {
                // boundary / tail chunk: element-wise with per-element device lookup
#pragma unroll 1
                for (int k = 0; k < 4; ++k) {
                    uint64_t i = cs + lane * 4 + k;
                    if (i >= ce) break;
                    uint64_t g = P.base + i;
                    uint32_t dd = find_dev(P.dev_off, P.ndev, g);
                    uint32_t ss = __ldg(P.dev_set + dd);
                    uint64_t pc = 0;
                    if (g != __ldg(P.dev_off + dd)) {
                        uint32_t pp = i ? __ldg(P.prompt + i - 1) : P.prev_p;
                        uint32_t po = i ? __ldg(P.output + i - 1) : P.prev_o;
                        pc = charged_tokens(pp, po, P.sets[ss].cpa);
                    }
                    uint32_t v = fused_one<FAST>(P, smw, ss, pc, __ldg(P.prompt + i), __ldg(P.output + i));
                    P.out[i] = v;
                    if (COUNT) count_verdict(v, cnt);
                }
                if (ce < i_end) {
                    uint64_t gl = P.base + ce - 1;
                    d = find_dev(P.dev_off, P.ndev, gl);
                    hi = __ldg(P.dev_off + d + 1);
                    s = __ldg(P.dev_set + d);
                    prev_ch = charged_tokens(__ldg(P.prompt + ce - 1), __ldg(P.output + ce - 1), P.sets[s].cpa);
                    if (P.base + ce == hi) {  // next chunk starts a new device
                        d = find_dev(P.dev_off, P.ndev, P.base + ce);
                        hi = __ldg(P.dev_off + d + 1);
                        s = __ldg(P.dev_set + d);
                        prev_ch = 0;
                    }
                }
            }
        }
    }
    if (COUNT) flush_counters(cnt, P.counters);
}

// ------------------------------------------------------------- features
// Per-query cost-model features: serving_memory(p+o, 1) (engine.hpp:297),
// charged tokens (engine.hpp:422-423), prefill_latency(p, 1, false) (engine.hpp:324).
__global__ void k_features(colo_model m, uint32_t cpa, const uint32_t* __restrict__ prompt,
                           const uint32_t* __restrict__ output, uint64_t n, uint64_t* need, uint64_t* charged,
                           double* prefill) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t p = prompt[i], o = output[i];
        if (need) need[i] = serving_memory(m, static_cast<uint64_t>(p) + o, 1);
        if (charged) charged[i] = charged_tokens(p, o, cpa);
        if (prefill) prefill[i] = prefill_latency(m, p, 1, false);
    }
}

// ------------------------------------------------------------- synthesis
struct SynthParams {
    double bin_values[32];
    double cum[32];
    uint32_t nbins;
    const uint64_t* dev_off;
    const double* dev_qps;
    uint32_t ndev;
    uint64_t seed;
    double* arrival;
    uint32_t* prompt;
    uint32_t* output;
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ double u01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

// One warp per device: exponential gaps summed with a warp scan + carry.
__global__ void k_synth(const __grid_constant__ SynthParams P) {
    uint32_t lane = threadIdx.x & 31;
    uint32_t d = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (d >= P.ndev) return;
    uint64_t lo = P.dev_off[d], hi = P.dev_off[d + 1];
    double rate = P.dev_qps[d];
    double t = 0.0;
    for (uint64_t j0 = lo; j0 < hi; j0 += 32) {
        uint64_t j = j0 + lane;
        uint64_t h = mix64(P.seed ^ mix64(j * 2 + 1));
        double gap = -log(1.0 - u01(h)) / rate;
        double x = gap;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            double y = __shfl_up_sync(0xffffffffu, x, s);
            if (lane >= s) x += y;
        }
        if (j < hi) {
            P.arrival[j] = t + x;
            double u = u01(mix64(h ^ 0xD1B54A32D192ED03ull));
            uint32_t b = 0;
            while (b + 1 < P.nbins && !(u < P.cum[b])) ++b;
            P.prompt[j] = static_cast<uint32_t>(llround(P.bin_values[b] < 1.0 ? 1.0 : P.bin_values[b]));
            P.output[j] = 128;
        }
        t += __shfl_sync(0xffffffffu, x, 31);
    }
}

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

}  // namespace

// ====================================================================== C-ABI
extern "C" {

colo_status colo_mapset_build(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const colo_grid* grid,
                              colo_mode mode, uint64_t hedge_step, uint64_t hedge_max, uint64_t assumed,
                              colo_mapset** out) {
    if (!ctx || !m || !g || !grid || !out) return COLO_EINVAL;
    *out = nullptr;
    colo_status st = colo_validate_profile_pair(m, g);
    if (st != COLO_OK) return set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
    st = colo_validate_grid(grid);
    if (st != COLO_OK) return set_err(ctx, st, "map grid rejected (maps.hpp:197-208)");
    if (hedge_step == 0 || hedge_max == 0 || hedge_max % hedge_step)
        return set_err(ctx, COLO_EVALIDATION, "hedging map: step/bound invalid (maps.hpp:362-365)");
    if (check_grid_limits(grid) != COLO_OK || check_model_limits(m) != COLO_OK || hedge_step > (1ull << 31) ||
        hedge_max + hedge_step > (1ull << 32))
        return set_err(ctx, COLO_EINVAL, "grid/model outside this build's limits (steps <= 2^31, max+step <= 2^32, L <= 253)");
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    auto* ms = new colo_mapset();
    ms->device = ctx->device;
    ms->m = *m;
    ms->g = *g;
    ms->grid = *grid;
    ms->mode = mode;
    ms->hedge_step = hedge_step;
    ms->hedge_max = hedge_max;
    ms->assumed = assumed;
    ms->hash = colo_profile_hash(m, g);
    ms->C = static_cast<uint32_t>(grid->max_cached / grid->cached_step + 1);
    ms->I = static_cast<uint32_t>(grid->max_incoming / grid->incoming_step);
    ms->B = static_cast<uint32_t>(grid->max_batch / grid->batch_step);
    ms->Hc = static_cast<uint32_t>(hedge_max / hedge_step);
    ms->F = static_cast<uint32_t>(m->num_layers + 1);
    ms->fast = hedge_step == grid->cached_step;
    uint64_t noff = static_cast<uint64_t>(ms->C) * ms->I * ms->B, nhed = static_cast<uint64_t>(ms->Hc) * ms->F;
    if (noff > (1ull << 31) || nhed > (1ull << 31)) {
        delete ms;
        return set_err(ctx, COLO_EINVAL, "map too large");
    }
    uint64_t ntab = static_cast<uint64_t>(ms->C + 1) * (ms->I + 1);
    cudaError_t e = cudaMalloc(&ms->d_off, noff);
    if (e == cudaSuccess) e = cudaMalloc(&ms->d_hed, nhed);
    if (e == cudaSuccess && ms->fast) e = cudaMalloc(&ms->d_tab, ntab * 4);
    if (e == cudaSuccess && ms->fast) e = cudaMalloc(&ms->d_str, (ms->C + 1) * 4ull);
    if (e != cudaSuccess) {
        colo_mapset_destroy(ms);
        return cuda_err(ctx, e, "cudaMalloc(mapset)");
    }
    uint64_t budget = g->capacity_bytes - g->runtime_reserve_bytes - m->weights_bytes;
    uint32_t cpa = mode == COLO_CPA;
    k_build_offload<<<static_cast<uint32_t>((noff + 255) / 256), 256, 0, ctx->stream>>>(
        *m, budget, cpa, grid->cached_step, grid->incoming_step, grid->batch_step, ms->I, ms->B,
        static_cast<uint32_t>(noff), ms->d_off);
    k_build_hedge<<<static_cast<uint32_t>((nhed + 255) / 256), 256, 0, ctx->stream>>>(
        *m, *g, cpa, hedge_step, assumed, ms->F, static_cast<uint32_t>(nhed), ms->d_hed);
    if (ms->fast) {
        MapView mv = make_view(ms);
        k_build_tab<<<static_cast<uint32_t>((ntab + 255) / 256), 256, 0, ctx->stream>>>(mv, ms->d_tab, ms->d_str);
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        colo_mapset_destroy(ms);
        return cuda_err(ctx, e, "map build");
    }
    *out = ms;
    return COLO_OK;
}

colo_status colo_mapset_from_cells(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const colo_grid* grid,
                                   colo_mode mode, uint64_t hedge_step, uint64_t hedge_max, uint64_t assumed,
                                   uint64_t built_hash, const uint8_t* h_off, size_t n_off, const uint8_t* h_hed,
                                   size_t n_hed, colo_mapset** out) {
    if (!ctx || !h_off || !h_hed || !out) return COLO_EINVAL;
    if (built_hash != colo_profile_hash(m, g))
        return set_err(ctx, COLO_EVALIDATION, "profile hash mismatch; map was built from different profiles");
    colo_status st = colo_mapset_build(ctx, m, g, grid, mode, hedge_step, hedge_max, assumed, out);
    if (st != COLO_OK) return st;
    colo_mapset* ms = *out;
    if (n_off != static_cast<size_t>(ms->C) * ms->I * ms->B || n_hed != static_cast<size_t>(ms->Hc) * ms->F) {
        colo_mapset_destroy(ms);
        *out = nullptr;
        return set_err(ctx, COLO_EINVAL, "cell array sizes do not match the grid");
    }
    for (size_t i = 0; i < n_off; ++i)
        if (h_off[i] > 2 + m->num_layers) {
            colo_mapset_destroy(ms);
            *out = nullptr;
            return set_err(ctx, COLO_EVALIDATION, "bad decision token in offload cells");
        }
    COLO_CK(ctx, cudaMemcpyAsync(ms->d_off, h_off, n_off, cudaMemcpyHostToDevice, ctx->stream));
    COLO_CK(ctx, cudaMemcpyAsync(ms->d_hed, h_hed, n_hed, cudaMemcpyHostToDevice, ctx->stream));
    if (ms->fast) {
        MapView mv = make_view(ms);
        uint64_t ntab = static_cast<uint64_t>(ms->C + 1) * (ms->I + 1);
        k_build_tab<<<static_cast<uint32_t>((ntab + 255) / 256), 256, 0, ctx->stream>>>(mv, ms->d_tab, ms->d_str);
    }
    COLO_CK(ctx, cudaGetLastError());
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

colo_status colo_mapset_shape(const colo_mapset* ms, size_t* n_off, size_t* n_hed) {
    if (!ms || !n_off || !n_hed) return COLO_EINVAL;
    *n_off = static_cast<size_t>(ms->C) * ms->I * ms->B;
    *n_hed = static_cast<size_t>(ms->Hc) * ms->F;
    return COLO_OK;
}

colo_status colo_mapset_cells(colo_ctx* ctx, const colo_mapset* ms, uint8_t* h_off, size_t n_off, uint8_t* h_hed,
                              size_t n_hed) {
    if (!ctx || !ms) return COLO_EINVAL;
    size_t a, b;
    colo_mapset_shape(ms, &a, &b);
    if ((h_off && n_off != a) || (h_hed && n_hed != b)) return set_err(ctx, COLO_EINVAL, "cell buffer size mismatch");
    if (h_off) COLO_CK(ctx, cudaMemcpyAsync(h_off, ms->d_off, a, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_hed) COLO_CK(ctx, cudaMemcpyAsync(h_hed, ms->d_hed, b, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

uint64_t colo_mapset_hash(const colo_mapset* ms) { return ms ? ms->hash : 0; }

void colo_mapset_destroy(colo_mapset* ms) {
    if (!ms) return;
    cudaSetDevice(ms->device);
    cudaFree(ms->d_off);
    cudaFree(ms->d_hed);
    cudaFree(ms->d_tab);
    cudaFree(ms->d_str);
    delete ms;
}

colo_status colo_decide(colo_ctx* ctx, const colo_mapset* ms, const colo_tuple* d_in, size_t n, uint32_t* d_out,
                        uint64_t* d_counters) {
    if (!ctx || !ms || (n && (!d_in || !d_out))) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    colo_status st = check_align(ctx, d_in);
    if (st != COLO_OK) return st;
    DecideParams P{};
    P.mv = make_view(ms);
    P.in = reinterpret_cast<const uint4*>(d_in);
    P.out = d_out;
    P.n = n;
    P.counters = d_counters;
    size_t smem = ((P.mv.off_bytes + 15u) & ~15u) + P.mv.hed_bytes;
    bool use_smem = smem <= 96 * 1024;
    const void* fn;
    if (use_smem) fn = d_counters ? (const void*)k_decide<true, true> : (const void*)k_decide<true, false>;
    else fn = d_counters ? (const void*)k_decide<false, true> : (const void*)k_decide<false, false>;
    size_t dyn = use_smem ? smem : 0;
    if (dyn > 48 * 1024) COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    int blocks = blocks_for(ctx, fn, kThreads, dyn);
    uint64_t need_blocks = (n + kThreads - 1) / kThreads;
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
    void* args[] = {&P};
    COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), args, dyn, ctx->stream));
    return COLO_OK;
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
    const void* fn = d_counters ? (const void*)k_decide_exact<true> : (const void*)k_decide_exact<false>;
    int blocks = blocks_for(ctx, fn, kThreads, 0);
    uint64_t need_blocks = (n + kThreads - 1) / kThreads;
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
    void* args[] = {&P};
    COLO_CK(ctx, cudaLaunchKernel(fn, dim3(blocks), dim3(kThreads), args, 0, ctx->stream));
    return COLO_OK;
}

}  // extern "C"

namespace {

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
    size_t smem = fast ? static_cast<size_t>(words) * 4 : 0;
    if (smem > 160 * 1024) {
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
    if (fast) fn = d_counters ? (const void*)k_fused<true, true> : (const void*)k_fused<true, false>;
    else fn = d_counters ? (const void*)k_fused<false, true> : (const void*)k_fused<false, false>;
    if (smem > 48 * 1024) COLO_CK(ctx, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int blocks = blocks_for(ctx, fn, kThreads, smem);
    uint64_t need_blocks = (n + 1023) / 1024;  // >= 128 elements per warp
    if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(std::max<uint64_t>(need_blocks, 1));
    void* args[] = {&P};
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

}  // namespace

extern "C" {

colo_status colo_features_decide(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const uint32_t* d_prompt,
                                 const uint32_t* d_output, size_t n, const uint64_t* d_dev_offsets,
                                 const uint16_t* d_dev_set, size_t ndev, uint32_t* d_out, uint64_t* d_counters) {
    if (!ctx || ndev == 0 || !d_dev_offsets || !d_dev_set) return COLO_EINVAL;
    colo_status st = check_sets(ctx, sets, nsets);
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
        size_t len = std::min(CH, n - c0);
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
    if (d_cnt) {
        COLO_CK(ctx, cudaMemsetAsync(d_cnt, 0, sizeof(uint64_t) * COLO_NCOUNTERS, ss[0]));
        COLO_CK(ctx, cudaStreamSynchronize(ss[0]));
    }
    for (size_t c0 = 0, k = 0; c0 < n; c0 += CH, ++k) {
        size_t len = std::min(CH, n - c0);
        cudaStream_t s = ss[k & 1];
        auto* buf = base + (k & 1) * chunk_bytes;
        auto* din = reinterpret_cast<colo_tuple*>(buf);
        auto* dout = reinterpret_cast<uint32_t*>(buf + CH * 16);
        COLO_CK(ctx, cudaMemcpyAsync(din, h_in + c0, len * 16, cudaMemcpyHostToDevice, s));
        cudaStream_t keep = ctx->stream;
        ctx->stream = s;
        st = colo_decide(ctx, ms, din, len, dout, d_cnt);
        ctx->stream = keep;
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

colo_status colo_features(colo_ctx* ctx, const colo_model* m, colo_mode mode, const uint32_t* d_prompt,
                          const uint32_t* d_output, size_t n, uint64_t* d_need, uint64_t* d_charged, double* d_prefill) {
    if (!ctx || !m || (n && (!d_prompt || !d_output))) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    int blocks = std::max<int>(1, static_cast<int>(std::min<uint64_t>((n + 255) / 256, ctx->sm_count * 8ull)));
    k_features<<<blocks, 256, 0, ctx->stream>>>(*m, mode == COLO_CPA, d_prompt, d_output, n, d_need, d_charged,
                                                d_prefill);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

colo_status colo_synth_trace(colo_ctx* ctx, const double* h_bin_values, const double* h_bin_probs, size_t nbins,
                             const uint64_t* d_dev_offsets, const double* d_dev_qps, size_t ndev, uint64_t seed,
                             double* d_arrival, uint32_t* d_prompt, uint32_t* d_output) {
    if (!ctx || !h_bin_values || !h_bin_probs || nbins == 0 || nbins > 32 || ndev == 0) return COLO_EINVAL;
    SynthParams P{};
    double acc = 0;
    for (size_t i = 0; i < nbins; ++i) {
        P.bin_values[i] = h_bin_values[i];
        acc += h_bin_probs[i];
        P.cum[i] = acc;
    }
    P.nbins = static_cast<uint32_t>(nbins);
    P.dev_off = d_dev_offsets;
    P.dev_qps = d_dev_qps;
    P.ndev = static_cast<uint32_t>(ndev);
    P.seed = seed;
    P.arrival = d_arrival;
    P.prompt = d_prompt;
    P.output = d_output;
    uint32_t blocks = static_cast<uint32_t>((ndev * 32 + 127) / 128);
    k_synth<<<blocks, 128, 0, ctx->stream>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

}  // extern "C"
