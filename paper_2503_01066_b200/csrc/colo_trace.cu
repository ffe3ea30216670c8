// colo_trace.cu -- validate_trace (workload.hpp:164-188) on the device for
// CSR device traces.  Reference paths are relative to
// /root/reference/proj/include/colosim/.
//
// The reference stable-sorts a trace's records by (arrival_time, query_id),
// then rejects a negative arrival, zero prompt or output tokens, and a
// repeated query_id.  Here every device's rows [off[d], off[d+1]) are
// ordered the same way by LSD radix passes over a row permutation (CUB's
// radix sort is stable): by query id, by device (the id-ordered rows of one
// device are now adjacent, so a repeated id is a pair of equal neighbours),
// by arrival bits (arrivals are checked non-negative first, so their IEEE
// bit patterns order as the values), and by device again.  The permutation
// is then applied to every column.  A trace that is already ordered and has
// positional ids (d_query_id == NULL) costs one check kernel.
#include <cstdio>
#include <string>

#include <cub/device/device_radix_sort.cuh>

#include "colo_internal.h"

using namespace colo;

namespace {

constexpr uint32_t kThreads = 256;

// per row: 1 = negative or NaN arrival, 2 = zero prompt tokens, 3 = zero output
// tokens; the lowest offending row wins (atomicMin on row << 2 | code)
__global__ void k_trace_check(const double* __restrict__ a, const uint32_t* __restrict__ p,
                              const uint32_t* __restrict__ o, const uint64_t* __restrict__ qid,
                              const uint64_t* __restrict__ off, uint32_t ndev, uint64_t n,
                              unsigned long long* bad, unsigned int* unsorted) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double x = a[i];
        uint32_t code = 0;
        if (!(x >= 0.0)) code = 1;  // workload.hpp:176-178 (NaN refused too)
        else if (p[i] == 0) code = 2;  // :179-181
        else if (o[i] == 0) code = 3;  // :182-184
        if (code) atomicMin(bad, (static_cast<unsigned long long>(i) << 2) | code);
        // ordered within the device by (arrival, id)? row i+1 is in the same device unless it starts one
        if (i + 1 < n) {
            uint32_t lo = 0, hi = ndev;  // device of row i+1: last d with off[d] <= i+1
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (off[mid] <= i + 1) lo = mid;
                else hi = mid;
            }
            if (off[lo] != i + 1) {
                const double y = a[i + 1];
                const bool ok = x < y || (x == y && (qid ? qid[i] < qid[i + 1] : true));
                if (!ok) *unsorted = 1u;
            }
        }
    }
}

__global__ void k_iota(uint32_t* __restrict__ v, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<uint32_t>(i);
}

__global__ void k_dev_of(const uint64_t* __restrict__ off, uint32_t ndev, uint32_t* __restrict__ dev) {
    // one block per device: rows [off[d], off[d+1]) belong to d
    const uint32_t d = blockIdx.x;
    if (d >= ndev) return;
    for (uint64_t i = off[d] + threadIdx.x; i < off[d + 1]; i += blockDim.x) dev[i] = d;
}

template <class K>
__global__ void k_gather_key(const K* __restrict__ src, const uint32_t* __restrict__ perm, K* __restrict__ dst,
                             uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[perm[i]];
}

// adjacent rows of the (device, id) order with equal device and id: the
// lowest such position wins
__global__ void k_dup(const uint32_t* __restrict__ dev_sorted, const uint64_t* __restrict__ id_sorted, uint64_t n,
                      unsigned long long* first) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i + 1 < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (dev_sorted[i] == dev_sorted[i + 1] && id_sorted[i] == id_sorted[i + 1]) atomicMin(first, i);
}

template <class T>
__global__ void k_apply(const T* __restrict__ src, const uint32_t* __restrict__ perm, T* __restrict__ dst, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[perm[i]];
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

extern "C" colo_status colo_validate_trace(colo_ctx* ctx, uint64_t* d_query_id, double* d_arrival, uint32_t* d_prompt,
                                           uint32_t* d_output, double* d_label_delay, size_t n,
                                           const uint64_t* d_dev_offsets, size_t ndev) {
    if (!ctx || (n && (!d_arrival || !d_prompt || !d_output || !d_dev_offsets)) || ndev == 0)
        return COLO_EINVAL;
    if (n >= (1ull << 32) || ndev >= (1ull << 32))
        return set_err(ctx, COLO_EINVAL, "validate_trace: at most 2^32 - 1 rows and devices");
    if (n == 0) return COLO_OK;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const uint32_t blocks = static_cast<uint32_t>(std::min<uint64_t>((n + kThreads - 1) / kThreads,
                                                                     static_cast<uint64_t>(ctx->sm_count) * 8));
    auto* bad = reinterpret_cast<unsigned long long*>(ctx->d_counters);
    auto* unsorted = reinterpret_cast<unsigned int*>(ctx->d_flag);
    const unsigned long long none = ~0ull;
    COLO_CK(ctx, cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, st));
    COLO_CK(ctx, cudaMemsetAsync(unsorted, 0, 4, st));
    COLO_LAUNCHED(ctx);
    k_trace_check<<<blocks, kThreads, 0, st>>>(d_arrival, d_prompt, d_output, d_query_id, d_dev_offsets,
                                               static_cast<uint32_t>(ndev), n, bad, unsorted);
    unsigned long long h_bad = 0;
    unsigned int h_unsorted = 0;
    COLO_CK(ctx, cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cudaMemcpyAsync(&h_unsorted, unsorted, 4, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cudaStreamSynchronize(st));
    if (h_bad != none) {
        const uint64_t row = h_bad >> 2;
        uint64_t q = row;
        if (d_query_id) COLO_CK(ctx, cudaMemcpy(&q, d_query_id + row, 8, cudaMemcpyDeviceToHost));
        static const char* what[] = {"", ": negative arrival_time", ": prompt_tokens must be >= 1",
                                     ": output_tokens must be >= 1"};
        return set_err(ctx, COLO_EVALIDATION, "trace: query " + std::to_string(q) + what[h_bad & 3]);
    }
    if (!h_unsorted && !d_query_id) return COLO_OK;  // ordered, positional ids: nothing to do

    // scratch: two permutations, two u64 key buffers, the device of every row, CUB temp
    DevBuf perm[2], key[2], dev, tmp;
    COLO_CK(ctx, cudaMalloc(&perm[0].p, n * 4));
    COLO_CK(ctx, cudaMalloc(&perm[1].p, n * 4));
    COLO_CK(ctx, cudaMalloc(&key[0].p, n * 8));
    COLO_CK(ctx, cudaMalloc(&key[1].p, n * 8));
    COLO_CK(ctx, cudaMalloc(&dev.p, n * 4));
    auto* P0 = static_cast<uint32_t*>(perm[0].p);
    auto* P1 = static_cast<uint32_t*>(perm[1].p);
    auto* K0 = static_cast<uint64_t*>(key[0].p);
    auto* K1 = static_cast<uint64_t*>(key[1].p);
    auto* DV = static_cast<uint32_t*>(dev.p);
    size_t tb = 0, tb2 = 0;
    COLO_CK(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tb, K0, K1, P0, P1, static_cast<int64_t>(n), 0, 64, st));
    COLO_CK(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tb2, reinterpret_cast<uint32_t*>(K0),
                                                 reinterpret_cast<uint32_t*>(K1), P0, P1, static_cast<int64_t>(n), 0,
                                                 32, st));
    COLO_CK(ctx, cudaMalloc(&tmp.p, std::max(tb, tb2) + 16));
    tb = std::max(tb, tb2);
    COLO_LAUNCHED(ctx);
    k_iota<<<blocks, kThreads, 0, st>>>(P0, n);
    COLO_LAUNCHED(ctx);
    k_dev_of<<<static_cast<uint32_t>(ndev), kThreads, 0, st>>>(d_dev_offsets, static_cast<uint32_t>(ndev), DV);
    int dbits = 1;
    while ((1ull << dbits) < ndev) ++dbits;
    // stable pass: keys = column[perm], (perm) sorted by them -> P0
    auto pass64 = [&](const uint64_t* col) -> colo_status {
        COLO_LAUNCHED(ctx);
        k_gather_key<uint64_t><<<blocks, kThreads, 0, st>>>(col, P0, K0, n);
        COLO_CK(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tb, K0, K1, P0, P1, static_cast<int64_t>(n), 0, 64, st));
        COLO_CK(ctx, cudaMemcpyAsync(P0, P1, n * 4, cudaMemcpyDeviceToDevice, st));
        return COLO_OK;
    };
    auto pass_dev = [&]() -> colo_status {
        auto* k0 = reinterpret_cast<uint32_t*>(K0);
        auto* k1 = reinterpret_cast<uint32_t*>(K1);
        COLO_LAUNCHED(ctx);
        k_gather_key<uint32_t><<<blocks, kThreads, 0, st>>>(DV, P0, k0, n);
        COLO_CK(ctx, cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0, k1, P0, P1, static_cast<int64_t>(n), 0, dbits, st));
        COLO_CK(ctx, cudaMemcpyAsync(P0, P1, n * 4, cudaMemcpyDeviceToDevice, st));
        return COLO_OK;
    };
    colo_status s = COLO_OK;
    if (d_query_id) {
        if ((s = pass64(d_query_id)) != COLO_OK) return s;
        if (ndev > 1 && (s = pass_dev()) != COLO_OK) return s;
        // (device, id) order: equal neighbours are a repeated id (workload.hpp:186-188)
        auto* ids = K1;  // ids in this order
        COLO_LAUNCHED(ctx);
        k_gather_key<uint64_t><<<blocks, kThreads, 0, st>>>(d_query_id, P0, ids, n);
        auto* dvs = reinterpret_cast<uint32_t*>(K0);
        COLO_LAUNCHED(ctx);
        k_gather_key<uint32_t><<<blocks, kThreads, 0, st>>>(DV, P0, dvs, n);
        COLO_CK(ctx, cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, st));
        COLO_LAUNCHED(ctx);
        k_dup<<<blocks, kThreads, 0, st>>>(dvs, ids, n, bad);
        COLO_CK(ctx, cudaMemcpyAsync(&h_bad, bad, 8, cudaMemcpyDeviceToHost, st));
        COLO_CK(ctx, cudaStreamSynchronize(st));
        if (h_bad != none) {
            uint64_t q = 0;
            COLO_CK(ctx, cudaMemcpy(&q, ids + h_bad, 8, cudaMemcpyDeviceToHost));
            return set_err(ctx, COLO_EVALIDATION, "trace: duplicate query_id: " + std::to_string(q));
        }
        if (!h_unsorted) return COLO_OK;
    }
    // (device, arrival, id): arrival bits (all >= +0.0 here, so they order as the values), then device
    if ((s = pass64(reinterpret_cast<const uint64_t*>(d_arrival))) != COLO_OK) return s;
    if (ndev > 1 && (s = pass_dev()) != COLO_OK) return s;
    // apply the permutation to every column (through K0/K1 as staging)
    auto apply8 = [&](void* col) -> colo_status {
        COLO_LAUNCHED(ctx);
        k_apply<uint64_t><<<blocks, kThreads, 0, st>>>(static_cast<const uint64_t*>(col), P0, K0, n);
        COLO_CK(ctx, cudaMemcpyAsync(col, K0, n * 8, cudaMemcpyDeviceToDevice, st));
        return COLO_OK;
    };
    auto apply4 = [&](void* col) -> colo_status {
        COLO_LAUNCHED(ctx);
        k_apply<uint32_t><<<blocks, kThreads, 0, st>>>(static_cast<const uint32_t*>(col), P0,
                                                        reinterpret_cast<uint32_t*>(K0), n);
        COLO_CK(ctx, cudaMemcpyAsync(col, K0, n * 4, cudaMemcpyDeviceToDevice, st));
        return COLO_OK;
    };
    if ((s = apply8(d_arrival)) != COLO_OK) return s;
    if ((s = apply4(d_prompt)) != COLO_OK) return s;
    if ((s = apply4(d_output)) != COLO_OK) return s;
    if (d_query_id && (s = apply8(d_query_id)) != COLO_OK) return s;
    if (d_label_delay && (s = apply8(d_label_delay)) != COLO_OK) return s;
    COLO_CK(ctx, cudaGetLastError());
    COLO_CK(ctx, cudaStreamSynchronize(st));
    return COLO_OK;
}
