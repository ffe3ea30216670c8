// colo_replay.cuh -- device helpers shared by the replay kernels
// (colo_serving.cu: serving-only replay, colo_colocated.cu: colocated replay).
#pragma once

#include <cstdint>

namespace colo {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {  // two 32-bit warp reductions (REDUX)
    const uint32_t hi = __reduce_max_sync(kFullMask, static_cast<uint32_t>(v >> 32));
    const uint32_t lo = __reduce_max_sync(kFullMask, static_cast<uint32_t>(v >> 32) == hi ? static_cast<uint32_t>(v) : 0u);
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(kFullMask, v, s);
    return v;
}

// 192-bit fixed-point accumulation (LSB 2^-96) of s * mult.  flags bit0: a
// sample below the representable range was truncated; bit1: overflow.
__device__ __forceinline__ void add3(uint64_t (&a)[3], uint64_t w0, uint64_t w1, uint64_t w2) {
    const uint64_t t0 = a[0] + w0;
    const uint64_t c0 = t0 < w0;
    const uint64_t t1 = a[1] + w1;
    uint64_t c1 = t1 < w1;
    const uint64_t t1b = t1 + c0;
    c1 |= t1b < c0;
    a[0] = t0;
    a[1] = t1b;
    a[2] = a[2] + w2 + c1;
}

__device__ __forceinline__ void acc_fixed(uint64_t (&a)[3], uint32_t& flags, double s, uint32_t mult) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
    const uint32_t ex = static_cast<uint32_t>(bits >> 52) & 0x7ffu;
    const uint64_t frac = bits & ((1ull << 52) - 1);
    if (ex == 0) {
        if (frac) flags |= 1u;
        return;
    }
    uint64_t m = frac | (1ull << 52);
    int sh = static_cast<int>(ex) - 1075 + 96;
    if (sh < 0) {
        flags |= 1u;
        if (sh <= -53) return;
        m >>= -sh;
        sh = 0;
    }
    const uint64_t lo = m * mult, hi = __umul64hi(m, static_cast<uint64_t>(mult));
    const int q = sh >> 6, r = sh & 63;
    const uint64_t x0 = lo << r;
    const uint64_t x1 = r ? ((lo >> (64 - r)) | (hi << r)) : hi;
    const uint64_t x2 = r ? (hi >> (64 - r)) : 0ull;
    if (q == 0) {
        add3(a, x0, x1, x2);
    } else if (q == 1) {
        if (x2) flags |= 2u;
        add3(a, 0, x0, x1);
    } else if (q == 2) {
        if (x1 | x2) flags |= 2u;
        add3(a, 0, 0, x0);
    } else {
        flags |= 2u;
    }
}

// ---- the absolute-time chain without the chain ----------------------------------
// now_k = now_{k-1} + d_k (f64, in order) for K <= 128 durations held 4 per
// lane (d[r] is step 32r + lane).  While now stays in the binade
// [2^e, 2^(e+1)) of now_0 the grid is u = 2^(e-52), now is a multiple of u and
// fl(now + d) = now + RN_u(d) unless now + d is a tie; so with the integers
// r_k = RN_u(d_k) / u, now_k = now_0 + u * (r_0 + ... + r_k) exactly, and the
// whole chain is a warp scan.  Returns false (warp-uniform) when a step is a
// tie, a duration is negative / not finite / too small to scale exactly, or
// the chain would reach the next binade: the caller folds sequentially.
// binade e of a positive normal double (t in [2^e, 2^(e+1))) and 2^k, from the bits
__device__ __forceinline__ int binade_of(double t) {
    return static_cast<int>((static_cast<uint64_t>(__double_as_longlong(t)) >> 52) & 0x7ff) - 1023;
}
__device__ __forceinline__ double pow2i(int k) {  // k in [-1022, 1023]
    return __longlong_as_double(static_cast<long long>(static_cast<uint64_t>(k + 1023) << 52));
}
// RN_u(x) / u for u = 1/sc (a power of two): false on a tie, a negative / NaN
// x, or a result >= 2^51 (x*sc is exact: callers keep sc in [2^-60, 2^260]
// and x either 0 or >= 2^-700).  Adding 2^52 rounds x*sc to an integer (the
// f64 spacing there is 1) whose value is the low mantissa bits.
template <bool POS = false>  // POS: the caller guarantees x >= 2^-700 (durations of validated profiles)
__device__ __forceinline__ bool rn_units(double x, double sc, uint64_t& r) {
    const double xs = x * sc;
    if (POS ? !(xs < 2251799813685248.0) : (!(xs < 2251799813685248.0) || !(x >= 0.0) || (x != 0.0 && x < 0x1p-700)))
        return false;
    const double t = xs + 4503599627370496.0;
    r = static_cast<uint64_t>(__double_as_longlong(t)) & ((1ull << 52) - 1);
    return fabs(xs - (t - 4503599627370496.0)) != 0.5;
}
template <bool POS = false>
__device__ __forceinline__ bool chain_rk(double t0, const double (&d)[4], uint32_t K, uint64_t (&rk)[4], double& u,
                                         uint64_t& room) {
    const uint32_t lane = threadIdx.x & 31;
    if (!(t0 >= 0x1p-200) || !(t0 <= 0x1p200)) return false;
    const int e = binade_of(t0);
    const double sc = pow2i(52 - e);
    u = pow2i(e - 52);
    room = (1ull << 53) - static_cast<uint64_t>(t0 * sc);  // now_K < 2^(e+1)  <=>  sum r < room
    bool ok = true;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t i = 32 * r + lane;
        rk[r] = 0;
        if (i < K) ok &= rn_units<POS>(d[r], sc, rk[r]);
    }
    return __all_sync(kFullMask, ok);
}

// warp sum of values < 2^57 (three exact 32-bit reductions of 19-bit chunks)
__device__ __forceinline__ uint64_t warp_sum_small(uint64_t v) {
    const uint32_t c0 = __reduce_add_sync(kFullMask, static_cast<uint32_t>(v & 0x7ffff));
    const uint32_t c1 = __reduce_add_sync(kFullMask, static_cast<uint32_t>((v >> 19) & 0x7ffff));
    const uint32_t c2 = __reduce_add_sync(kFullMask, static_cast<uint32_t>(v >> 38));
    return static_cast<uint64_t>(c0) + (static_cast<uint64_t>(c1) << 19) + (static_cast<uint64_t>(c2) << 38);
}

// now_{K-1} (the batch's end) or false.  POS: every duration of the first
// K is >= 2^-700 (a decode step of a validated profile whose step constant
// is at least that), so rn_units skips its sign and range tests.
template <bool POS = false>
__device__ __forceinline__ bool chain_fast_end(double t0, const double (&d)[4], uint32_t K, double& t_end) {
    uint64_t rk[4];
    double u;
    uint64_t room;
    if (!chain_rk<POS>(t0, d, K, rk, u, room)) return false;
    const uint64_t s = warp_sum_small(rk[0] + rk[1] + rk[2] + rk[3]);  // lane sums < 2^55
    if (s >= room) return false;
    t_end = t0 + static_cast<double>(s) * u;  // exact: a multiple of u below 2^(e+1)
    return true;
}

// every now_k, k < K, stored over the durations in d (shared memory, step i at d[i])
__device__ __forceinline__ bool chain_fast_store(double t0, double* d, uint32_t K) {
    const uint32_t lane = threadIdx.x & 31;
    double x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t i = 32 * r + lane;
        x[r] = i < K ? d[i] : 0.0;
    }
    uint64_t rk[4];
    double u;
    uint64_t room;
    if (!chain_rk(t0, x, K, rk, u, room)) return false;
    uint64_t carry = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // inclusive prefix in step order
        uint64_t v = rk[r];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(kFullMask, v, o);
            if (lane >= static_cast<uint32_t>(o)) v += y;
        }
        v += carry;
        carry = __shfl_sync(kFullMask, v, 31);
        rk[r] = v;
    }
    if (carry >= room) return false;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const uint32_t i = 32 * r + lane;
        if (i < K) d[i] = t0 + static_cast<double>(rk[r]) * u;
    }
    return true;
}

// a -= fixed(s * mult) (mod 2^192; the lane partials are summed mod 2^192 and
// the total is non-negative)
__device__ __forceinline__ void acc_fixed_sub(uint64_t (&a)[3], uint32_t& flags, double s, uint32_t mult) {
    uint64_t t[3] = {0, 0, 0};
    acc_fixed(t, flags, s, mult);
    const uint64_t c0 = t[0] == 0, c1 = c0 & (t[1] == 0);
    add3(a, ~t[0] + 1, ~t[1] + c0, ~t[2] + c1);
}

// First index >= from whose arrival is > T (or N): every arrival at or before
// T has been popped by the time the batch starts (engine.hpp:146-147,184-187).
// Arrivals are sorted, so the warp gallops with 32 probes per step (stride
// x32) and then refines (stride /32): O(log32 distance) dependent loads, so a
// saturated server's backlog of millions of queued arrivals costs a handful
// of steps instead of a linear scan.
__device__ __forceinline__ uint64_t find_tail(const double* __restrict__ arr, uint64_t N, uint64_t from, double T) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t lo = from;  // every index in [from, lo) has arrival <= T
    uint64_t stride = 1;
    bool gallop = true;
    while (lo < N) {
        const uint64_t p = lo + (lane + 1) * stride - 1;
        const bool le = p < N && arr[p] <= T;
        const uint32_t bal = __ballot_sync(kFullMask, le);
        if (bal == kFullMask && gallop) {
            lo += 32 * stride;
            stride *= 32;
            continue;
        }
        gallop = false;
        const uint32_t f = __ffs(~bal) - 1;  // bal != kFullMask once refining (the answer lies in the window)
        lo += f * stride;
        if (stride == 1) break;
        stride /= 32;
    }
    return lo < N ? lo : N;
}

// hist[key] += cnt for every lane with act.  The lanes are consecutive decode
// steps of a batch, whose TPT samples rise slowly with the context, so equal
// keys come in runs of neighbouring lanes: the lane that starts a run adds the
// run's total (an inclusive scan of the counts, differenced at the run's ends),
// and every run head issues its atomic in the same instruction.  Keys that
// repeat in separate runs just add separately, so the histogram is the same
// integer sum whatever the order.  Call from all lanes.
__device__ __forceinline__ void hist_add(uint64_t* hist, uint32_t key, uint32_t cnt, bool act) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t c = act ? cnt : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += y;
    }
    const uint32_t pkey = __shfl_up_sync(kFullMask, key, 1);
    const unsigned am = __ballot_sync(kFullMask, act);
    const bool pact = lane > 0 && ((am >> (lane - 1)) & 1u);
    const bool head = act && !(pact && pkey == key);
    // a run ends just before the next head or inactive lane
    const unsigned brk = __ballot_sync(kFullMask, head || !act);
    const unsigned above = lane == 31 ? 0u : brk & (~0u << (lane + 1));
    const uint32_t last = above ? static_cast<uint32_t>(__ffs(above) - 2) : 31u;
    const uint32_t iend = __shfl_sync(kFullMask, incl, last);
    if (head) atomicAdd(reinterpret_cast<unsigned long long*>(&hist[key]), static_cast<unsigned long long>(iend - incl + c));
}

// hist_add with cnt == 1 on every active lane: a run's total is its length.
__device__ __forceinline__ void hist_add1(uint64_t* hist, uint32_t key, bool act) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pkey = __shfl_up_sync(kFullMask, key, 1);
    const unsigned am = __ballot_sync(kFullMask, act);
    const bool pact = lane > 0 && ((am >> (lane - 1)) & 1u);
    const bool head = act && !(pact && pkey == key);
    const unsigned brk = __ballot_sync(kFullMask, head || !act);
    const unsigned above = lane == 31 ? 0u : brk & (~0u << (lane + 1));
    const uint32_t end = above ? static_cast<uint32_t>(__ffs(above) - 1) : 32u;
    if (head) atomicAdd(reinterpret_cast<unsigned long long*>(&hist[key]), static_cast<unsigned long long>(end - lane));
}

// Sequential f64 fold t = (((t + d0) + d1) + ...) over K durations staged in
// 16-B aligned shared memory, on one lane.  Pairs come in with one LDS.128 and
// the K == 128 case (the default output length) is fully unrolled, so the
// chain runs at the f64 add latency (8.5 vs 15 cycles per step measured on B200).
__device__ __forceinline__ double chain_fold(double t, const double* d, uint32_t K) {
    const double2* d2 = reinterpret_cast<const double2*>(d);
    if (K == 128) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
            const double2 q = d2[i];
            t = t + q.x;
            t = t + q.y;
        }
        return t;
    }
    uint32_t i = 0;
#pragma unroll 8
    for (; i + 1 < K; i += 2) {
        const double2 q = d2[i >> 1];
        t = t + q.x;
        t = t + q.y;
    }
    if (i < K) t = t + d[i];
    return t;
}

// The same fold, storing every partial result (the absolute step times) back.
__device__ __forceinline__ double chain_fold_store(double t, double* d, uint32_t K) {
    double2* d2 = reinterpret_cast<double2*>(d);
    if (K == 128) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
            double2 q = d2[i];
            q.x = t + q.x;
            q.y = q.x + q.y;
            t = q.y;
            d2[i] = q;
        }
        return t;
    }
    uint32_t i = 0;
#pragma unroll 8
    for (; i + 1 < K; i += 2) {
        double2 q = d2[i >> 1];
        q.x = t + q.x;
        q.y = q.x + q.y;
        t = q.y;
        d2[i >> 1] = q;
    }
    if (i < K) {
        t = t + d[i];
        d[i] = t;
    }
    return t;
}

}  // namespace colo
