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
    const double* dev_qps_hi;
    double period;
    uint32_t ndev;
    uint64_t seed;
    const uint32_t* dev_ids;  // NULL: keyed on the global query index; else on (fleet device id, local index)
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
    const double rate_lo = P.dev_qps[d];
    const double rate_hi = P.period > 0.0 ? P.dev_qps_hi[d] : rate_lo;
    double t = 0.0;
    for (uint64_t j0 = lo; j0 < hi; j0 += 32) {
        const double rate = (P.period > 0.0 && (static_cast<uint64_t>(t / P.period) & 1ull)) ? rate_hi : rate_lo;
        uint64_t j = j0 + lane;
        const uint64_t key = P.dev_ids ? ((static_cast<uint64_t>(P.dev_ids[d]) << 36) | (j - lo)) : j;
        uint64_t h = mix64(P.seed ^ mix64(key * 2 + 1));
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
    COLO_LAUNCHED(ctx);
    k_build_offload<<<static_cast<uint32_t>((noff + 255) / 256), 256, 0, ctx->stream>>>(
        *m, budget, cpa, grid->cached_step, grid->incoming_step, grid->batch_step, ms->I, ms->B,
        static_cast<uint32_t>(noff), ms->d_off);
    COLO_LAUNCHED(ctx);
    k_build_hedge<<<static_cast<uint32_t>((nhed + 255) / 256), 256, 0, ctx->stream>>>(
        *m, *g, cpa, hedge_step, assumed, ms->F, static_cast<uint32_t>(nhed), ms->d_hed);
    if (ms->fast) {
        MapView mv = make_view(ms);
        COLO_LAUNCHED(ctx);
        k_build_tab<<<static_cast<uint32_t>((ntab + 255) / 256), 256, 0, ctx->stream>>>(mv, ms->d_tab, ms->d_str);
    }
    if (colo::build_pack_image(ctx, ms) != COLO_OK) {
        std::string why = ctx->err;
        colo_mapset_destroy(ms);
        return set_err(ctx, COLO_ECUDA, why);
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
        COLO_LAUNCHED(ctx);
        k_build_tab<<<static_cast<uint32_t>((ntab + 255) / 256), 256, 0, ctx->stream>>>(mv, ms->d_tab, ms->d_str);
    }
    colo_status ist = colo::build_pack_image(ctx, ms);  // from the loaded cells
    if (ist != COLO_OK) return ist;
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
    cudaFree(ms->d_img);
    delete ms;
}

}  // extern "C"
extern "C" {

colo_status colo_features(colo_ctx* ctx, const colo_model* m, colo_mode mode, const uint32_t* d_prompt,
                          const uint32_t* d_output, size_t n, uint64_t* d_need, uint64_t* d_charged, double* d_prefill) {
    if (!ctx || !m || (n && (!d_prompt || !d_output))) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    int blocks = std::max<int>(1, static_cast<int>(std::min<uint64_t>((n + 255) / 256, ctx->sm_count * 8ull)));
    COLO_LAUNCHED(ctx);
    k_features<<<blocks, 256, 0, ctx->stream>>>(*m, mode == COLO_CPA, d_prompt, d_output, n, d_need, d_charged,
                                                d_prefill);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

colo_status colo_synth_trace(colo_ctx* ctx, const double* h_bin_values, const double* h_bin_probs, size_t nbins,
                             const uint64_t* d_dev_offsets, const double* d_dev_qps, const double* d_dev_qps_hi,
                             double burst_period, size_t ndev, uint64_t seed, double* d_arrival, uint32_t* d_prompt,
                             uint32_t* d_output) {
    return colo_synth_fleet_trace(ctx, h_bin_values, h_bin_probs, nbins, d_dev_offsets, d_dev_qps, d_dev_qps_hi,
                                  burst_period, ndev, nullptr, seed, d_arrival, d_prompt, d_output);
}

colo_status colo_synth_fleet_trace(colo_ctx* ctx, const double* h_bin_values, const double* h_bin_probs, size_t nbins,
                                   const uint64_t* d_dev_offsets, const double* d_dev_qps, const double* d_dev_qps_hi,
                                   double burst_period, size_t ndev, const uint32_t* d_dev_ids, uint64_t seed,
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
    P.dev_qps_hi = d_dev_qps_hi;
    P.period = d_dev_qps_hi ? burst_period : 0.0;
    P.ndev = static_cast<uint32_t>(ndev);
    P.seed = seed;
    P.dev_ids = d_dev_ids;
    P.arrival = d_arrival;
    P.prompt = d_prompt;
    P.output = d_output;
    uint32_t blocks = static_cast<uint32_t>((ndev * 32 + 127) / 128);
    COLO_LAUNCHED(ctx);
    k_synth<<<blocks, 128, 0, ctx->stream>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

}  // extern "C"
