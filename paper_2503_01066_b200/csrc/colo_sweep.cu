// colo_sweep.cu -- C5 support: synthetic admission-question streams and the
// map-vs-exact agreement statistics (per-query exact
// offload_cell_decision vs the batched quantised map lookup).
#include <algorithm>

#include "colo_internal.h"

using namespace colo;

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct TupleSynth {
    double bin_values[32];
    double cum[32];
    uint32_t nbins, L;
    uint64_t seed, n;
    uint4* out;
};

// cached ~ U[0, 8000], incoming = p + 128 (p from the length histogram),
// batch ~ U[1, 50], pending/dev_layers ~ U[0, L], charged ~ U[0, 9000]; 1 % of
// the questions push one field out of the default grid.
__global__ void k_synth_tuples(const __grid_constant__ TupleSynth P) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P.n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t h0 = mix64(P.seed ^ mix64(i)), h1 = mix64(h0), h2 = mix64(h1);
        uint32_t cached = static_cast<uint32_t>(h0 % 8001);
        const double u = static_cast<double>(h1 >> 11) * 0x1.0p-53;
        uint32_t b = 0;
        while (b + 1 < P.nbins && !(u < P.cum[b])) ++b;
        uint32_t incoming = static_cast<uint32_t>(P.bin_values[b]) + 128;
        uint32_t batch = 1 + static_cast<uint32_t>((h0 >> 32) % 50);
        const uint32_t pending = static_cast<uint32_t>((h2 & 0xffff) % (P.L + 1));
        const uint32_t dev = static_cast<uint32_t>(((h2 >> 16) & 0xffff) % (P.L + 1));
        const uint32_t charged = static_cast<uint32_t>((h2 >> 32) % 9001);
        const uint32_t oor = static_cast<uint32_t>(h1 % 300);  // 3 of 300 -> 1 %
        if (oor == 0) cached = 8001 + (cached & 1023);
        if (oor == 1) incoming = 8001 + (incoming & 1023);
        if (oor == 2) batch = 51 + (batch & 7);
        P.out[i] = make_uint4(cached, incoming, charged, batch | (pending << 16) | (dev << 24));
    }
}

// layers released by a verdict's decision (maps.hpp:41-48; AllToHost = L)
__device__ __forceinline__ uint32_t freed(uint32_t v, uint32_t L) {
    const uint32_t a = COLO_V_ACTION(v);
    return a == COLO_ACT_NOACTION ? 0u : a == COLO_ACT_ALLTOHOST ? L : COLO_V_LAYERS(v);
}

// counts[0] agree on (action, layers), [1] map frees more layers than exact,
// [2] map frees fewer, [3] same outcome (admit / load back / recompute), [4] total
__global__ void k_compare(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n, uint32_t L,
                          uint64_t* counts) {
    uint32_t c[5] = {0, 0, 0, 0, 0};
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t x = __ldcs(a + i), y = __ldcs(b + i);
        const uint32_t fx = freed(x, L), fy = freed(y, L);
        c[0] += (x & 0x3ffu) == (y & 0x3ffu);
        c[1] += fx > fy;
        c[2] += fx < fy;
        c[3] += COLO_V_VERDICT(x) == COLO_V_VERDICT(y);
        c[4] += 1;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        uint32_t v = c[k];
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(0xffffffffu, v, s);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long*>(counts + k), v);
    }
}

}  // namespace

extern "C" {

colo_status colo_synth_tuples(colo_ctx* ctx, uint64_t seed, size_t n, uint32_t num_layers, const double* h_bin_values,
                              const double* h_bin_probs, size_t nbins, colo_tuple* d_out) {
    if (!ctx || !h_bin_values || !h_bin_probs || nbins == 0 || nbins > 32 || (n && !d_out) || num_layers > 255)
        return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    TupleSynth P{};
    double acc = 0;
    for (size_t i = 0; i < nbins; ++i) {
        P.bin_values[i] = h_bin_values[i];
        acc += h_bin_probs[i];
        P.cum[i] = acc;
    }
    P.nbins = static_cast<uint32_t>(nbins);
    P.L = num_layers;
    P.seed = seed;
    P.n = n;
    P.out = reinterpret_cast<uint4*>(d_out);
    const int blocks = static_cast<int>(std::min<uint64_t>((n + 255) / 256, ctx->sm_count * 16ull));
    COLO_LAUNCHED(ctx);
    k_synth_tuples<<<blocks, 256, 0, ctx->stream>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

colo_status colo_compare_verdicts(colo_ctx* ctx, const uint32_t* d_map, const uint32_t* d_exact, size_t n,
                                  uint32_t num_layers, uint64_t* d_counts) {
    if (!ctx || !d_counts || (n && (!d_map || !d_exact))) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    const int blocks = static_cast<int>(std::min<uint64_t>((n + 255) / 256, ctx->sm_count * 8ull));
    COLO_LAUNCHED(ctx);
    k_compare<<<blocks, 256, 0, ctx->stream>>>(d_map, d_exact, n, num_layers, d_counts);
    COLO_CK(ctx, cudaGetLastError());
    return COLO_OK;
}

}  // extern "C"
