// colo_replay.cu -- serving-only replay (K4) and exact tail statistics (K5).
//
// One warp replays one device's trace segment (the reference's Simulation is
// strictly sequential per instance, engine.hpp:140-164; instances share no
// state).  Inside a batch the warp's lanes own decode steps:
// lane l folds step k0+l's duration over the batch members in batch order
// (engine.hpp:358-365), then the absolute-time fold now_k = now_{k-1} + d_k
// runs through the 32 lanes in order via shuffles, so every f64 operation is
// the reference's, in the reference's order (bit-exact TPT samples).
// Reference paths are relative to /root/reference/proj/.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "colo_internal.h"

using namespace colo;

namespace {

constexpr int kWarps = 4;
constexpr int kStage = 256;  // batch members staged in shared memory per warp
constexpr unsigned FULL = 0xffffffffu;

struct DevProfile {
    colo_model m;
    uint64_t budget;  // capacity - reserve - weights, engine.hpp:278-280
    uint64_t fixed;   // weights + reserve, engine.hpp:141
};

struct ReplayParams {
    DevProfile prof[kMaxSets];
    MapView sets[kMaxSets];
    uint32_t nprof, has_sets;
    const double* arr;
    const uint32_t* p;
    const uint32_t* o;
    const uint64_t* dev_off;
    const uint16_t* dev_prof;
    uint32_t ndev;
    double tau;
    double* samples;
    const uint64_t* sample_off;
    uint8_t* labels;
    colo_batch* batches;
    colo_device_summary* summary;
    uint64_t* hist;
    uint32_t nfilters, hist_shift, filter_shift;
    uint64_t prefix[3];
    int* err;
};

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v = max(v, __shfl_xor_sync(FULL, v, s));
    return v;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v += __shfl_xor_sync(FULL, v, s);
    return v;
}

// 192-bit fixed-point accumulation (LSB 2^-96) of s * mult.  flags bit0: a
// sample below the representable range was truncated; bit1: overflow.
__device__ __forceinline__ void add3(uint64_t (&a)[3], uint64_t w0, uint64_t w1, uint64_t w2) {
    uint64_t t0 = a[0] + w0;
    uint64_t c0 = t0 < w0;
    uint64_t t1 = a[1] + w1;
    uint64_t c1 = t1 < w1;
    uint64_t t1b = t1 + c0;
    c1 |= t1b < c0;
    a[0] = t0;
    a[1] = t1b;
    a[2] = a[2] + w2 + c1;
}

__device__ __forceinline__ void acc_fixed(uint64_t (&a)[3], uint32_t& flags, double s, uint32_t mult) {
    uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
    uint32_t ex = static_cast<uint32_t>(bits >> 52) & 0x7ffu;
    uint64_t frac = bits & ((1ull << 52) - 1);
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
    uint64_t lo = m * mult, hi = __umul64hi(m, static_cast<uint64_t>(mult));
    int q = sh >> 6, r = sh & 63;
    uint64_t x0 = lo << r;
    uint64_t x1 = r ? ((lo >> (64 - r)) | (hi << r)) : hi;
    uint64_t x2 = r ? (hi >> (64 - r)) : 0ull;
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

__global__ void __launch_bounds__(kWarps * 32) k_replay(const __grid_constant__ ReplayParams P) {
    __shared__ uint32_t sp[kWarps][kStage];
    __shared__ uint32_t so[kWarps][kStage];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * kWarps + warp;
    if (d >= P.ndev) return;
    const uint32_t pi = P.dev_prof[d];
    const colo_model& m = P.prof[pi].m;
    const uint64_t budget = P.prof[pi].budget;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const double* __restrict__ arr = P.arr + lo;
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;

    // Trace validation (workload.hpp:173-181 ordering/zero checks; engine.hpp:70-74 fit check).
    bool bad = false;
    for (uint64_t j = lane; j < N; j += 32) {
        uint32_t pj = pp[j], oj = po[j];
        if (pj == 0 || oj == 0) bad = true;
        else if (serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) > budget) bad = true;
        if (j > 0 && arr[j] < arr[j - 1]) bad = true;
    }
    if (__any_sync(FULL, bad)) {
        if (lane == 0) atomicOr(P.err, 1);
        return;
    }

    double T = -INFINITY;  // server idle before the first arrival (probe B4b)
    uint64_t head = 0, tail_ptr = 0;
    uint64_t slot = 0;  // charged tokens of the last single-query batch (C3 rule)
    uint64_t sample_pos = P.samples ? P.sample_off[d] : 0;
    uint64_t gen = 0, slow_tok = 0, slow_q = 0, max_need = 0, maxb = 0, nbatches = 0;
    uint64_t acc[3] = {0, 0, 0};
    uint32_t flags = 0;
    uint32_t* sP = sp[warp];
    uint32_t* sO = so[warp];
    const bool want_hist = P.hist != nullptr;

    while (head < N) {
        // ---- batch window: engine.hpp:146-147,178-188,270-276 -------------------
        uint64_t tail;
        double ah = arr[head];
        if (ah > T) {  // idle: the first popped arrival starts a batch alone
            T = ah;
            tail = head + 1;
            tail_ptr = head + 1;
        } else {       // queued: every arrival with time <= T has been popped
            if (tail_ptr < head) tail_ptr = head;
            while (tail_ptr < N) {
                uint64_t j = tail_ptr + lane;
                bool in = j < N && arr[j] <= T;
                uint32_t bal = __ballot_sync(FULL, in);
                if (bal == FULL) {
                    tail_ptr += 32;
                    continue;
                }
                tail_ptr += __ffs(~bal) - 1;
                break;
            }
            tail = tail_ptr;
        }
        // ---- batch formation: FIFO, at least one, sum(need) <= budget (engine.hpp:292-306)
        uint64_t end = head, need_total = 0, max_inc = 0;
        uint32_t maxo = 0;
        while (end < tail) {
            uint64_t j = end + lane;
            bool valid = j < tail;
            uint32_t pj = valid ? pp[j] : 0u, oj = valid ? po[j] : 0u;
            uint64_t nd = valid ? serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) : 0ull;
            uint64_t incl = nd;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                uint64_t y = __shfl_up_sync(FULL, incl, s);
                if (lane >= static_cast<uint32_t>(s)) incl += y;
            }
            incl += need_total;
            bool ok = valid && (j == head || incl <= budget);
            uint32_t bal = __ballot_sync(FULL, ok);
            uint32_t cnt = __popc(bal);
            if (ok && j - head < kStage) {
                sP[j - head] = pj;
                sO[j - head] = oj;
            }
            max_inc = max(max_inc, warp_max_u64(ok ? static_cast<uint64_t>(pj) + oj : 0ull));
            maxo = max(maxo, static_cast<uint32_t>(warp_max_u64(ok ? oj : 0u)));
            if (cnt) need_total = __shfl_sync(FULL, incl, cnt - 1);
            end += cnt;
            if (cnt < 32) break;
        }
        __syncwarp();
        const uint64_t nb = end - head;
        auto mem_p = [&](uint64_t j) -> uint32_t { return j < kStage ? sP[j] : pp[head + j]; };
        auto mem_o = [&](uint64_t j) -> uint32_t { return j < kStage ? sO[j] : po[head + j]; };

        // ---- replay-derived verdict (SURVEY §8(d) C3 rule) ----------------------
        uint32_t verdict = 0;
        if (P.has_sets) {
            const MapView& mv = P.sets[pi];
            uint64_t ch = charged_tokens(mem_p(0), mem_o(0), mv.cpa);
            if (lane == 0)
                verdict = compose(mv, mv.off, mv.hed, slot, max_inc, nb, 0, mv.L) | stream_bits(mv, mv.off, ch);
            if (nb == 1) slot = ch;
        }

        // ---- prefill: left fold in batch order (engine.hpp:321-325) -------------
        double dur = 0.0;
        for (uint64_t j = 0; j < nb; ++j) dur += prefill_latency(m, mem_p(j), 1, false);
        const double start = T + 0.0;  // prefill_start = now_ + stall, stall = 0
        double now = start + dur;      // PrefillDone time; every member's last_token_time

        // ---- decode steps (engine.hpp:358-387) ---------------------------------
        uint32_t first_slow = 0xffffffffu;
        for (uint32_t k0 = 0; k0 < maxo; k0 += 32) {
            const uint32_t k = k0 + lane;
            double dk = 0.0;
            uint32_t alive = 0;
            if (k < maxo) {
                for (uint64_t j = 0; j < nb; ++j) {
                    uint32_t oj = mem_o(j);
                    if (k < oj) {
                        dk += decode_step_latency(m, static_cast<uint64_t>(mem_p(j)) + k, 1, false);
                        ++alive;
                    }
                }
            }
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < 32; ++l) {
                double dl = __shfl_sync(FULL, dk, l);
                if (k0 + l < maxo) {
                    double nw = now + dl;
                    if (lane == static_cast<uint32_t>(l)) s = nw - now;  // now - last_token_time
                    now = nw;
                }
            }
            const bool live = k < maxo;
            const bool slow = live && s > P.tau;
            uint32_t sb = __ballot_sync(FULL, slow);
            if (sb && first_slow == 0xffffffffu) first_slow = k0 + __ffs(sb) - 1;
            gen += alive;
            if (slow) slow_tok += alive;
            if (live) {
                acc_fixed(acc, flags, s, alive);
                if (want_hist) {
                    uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
                    for (uint32_t f = 0; f < P.nfilters; ++f)
                        if ((bits >> P.filter_shift) == P.prefix[f])
                            atomicAdd(reinterpret_cast<unsigned long long*>(
                                          &P.hist[static_cast<uint64_t>(f) * COLO_HIST_BINS +
                                                  ((bits >> P.hist_shift) & (COLO_HIST_BINS - 1))]),
                                      static_cast<unsigned long long>(alive));
                }
            }
            if (P.samples) {
                // samples of step k occupy alive_k consecutive slots, steps in order
                uint32_t ex = alive;
#pragma unroll
                for (int sft = 1; sft < 32; sft <<= 1) {
                    uint32_t y = __shfl_up_sync(FULL, ex, sft);
                    if (lane >= static_cast<uint32_t>(sft)) ex += y;
                }
                uint32_t total = __shfl_sync(FULL, ex, 31);
                uint64_t pos = sample_pos + ex - alive;
                for (uint32_t a = 0; a < alive; ++a) P.samples[pos + a] = s;
                sample_pos += total;
            }
        }
        // ---- labels: a query is slow iff one of its tokens is (o_j > first slow step)
        for (uint64_t j = lane; j < nb; j += 32) {
            bool slowq = mem_o(j) > first_slow;
            slow_q += slowq;
            if (P.labels) P.labels[lo + head + j] = slowq ? 1 : 0;
        }
        if (lane == 0 && P.batches) {
            colo_batch b;
            b.start = start;
            b.end = now;
            b.first = static_cast<uint32_t>(head);
            b.n = static_cast<uint32_t>(nb);
            b.need_total = need_total;
            b.max_incoming = max_inc < 0xffffffffull ? static_cast<uint32_t>(max_inc) : 0xffffffffu;
            b.verdict = verdict;
            P.batches[lo + nbatches] = b;
        }
        max_need = max(max_need, need_total);
        maxb = max(maxb, nb);
        ++nbatches;
        T = now;
        head = end;
        __syncwarp();
    }

    // ---- per-device summary --------------------------------------------------
    gen = warp_sum_u64(gen);
    slow_tok = warp_sum_u64(slow_tok);
    slow_q = warp_sum_u64(slow_q);
    uint32_t fl = static_cast<uint32_t>(warp_max_u64(flags));
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        uint64_t b0 = __shfl_xor_sync(FULL, acc[0], s);
        uint64_t b1 = __shfl_xor_sync(FULL, acc[1], s);
        uint64_t b2 = __shfl_xor_sync(FULL, acc[2], s);
        add3(acc, b0, b1, b2);
    }
    if (lane == 0 && P.summary) {
        colo_device_summary& S = P.summary[d];
        S.generated_tokens = gen;
        S.slow_tokens = slow_tok;
        S.slow_queries = slow_q;
        S.batches = nbatches;
        S.peak_device_bytes = P.prof[pi].fixed + max_need;  // memory.hpp:28-35 watermark
        S.max_batch_size = maxb;
        S.end_time = N ? T : 0.0;
        S.tpt_sum[0] = acc[0];
        S.tpt_sum[1] = acc[1];
        S.tpt_sum[2] = acc[2];
        S.flags = fl;
    }
}

}  // namespace

extern "C" {

colo_status colo_replay_serving(colo_ctx* ctx, const colo_model* models, const colo_gpu* gpus, size_t nprofiles,
                                const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                const uint64_t* d_dev_offsets, const uint16_t* d_dev_profile, size_t ndev,
                                const colo_replay_opts* opts) {
    if (!ctx || !models || !gpus || !opts || nprofiles == 0 || nprofiles > kMaxSets || !d_dev_offsets ||
        !d_dev_profile)
        return COLO_EINVAL;
    if (ndev == 0) return COLO_OK;
    if (n && (!d_arrival || !d_prompt || !d_output)) return COLO_EINVAL;
    if (opts->d_samples && !opts->d_sample_offsets) return set_err(ctx, COLO_EINVAL, "samples need d_sample_offsets");
    if (opts->d_hist && (opts->nfilters == 0 || opts->nfilters > 3)) return set_err(ctx, COLO_EINVAL, "nfilters 1..3");
    ReplayParams P{};
    for (size_t i = 0; i < nprofiles; ++i) {
        colo_status st = colo_validate_profile_pair(&models[i], &gpus[i]);
        if (st != COLO_OK) return set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
        P.prof[i].m = models[i];
        P.prof[i].budget = gpus[i].capacity_bytes - gpus[i].runtime_reserve_bytes - models[i].weights_bytes;
        P.prof[i].fixed = models[i].weights_bytes + gpus[i].runtime_reserve_bytes;
        if (opts->sets) {
            if (!opts->sets[i]) return set_err(ctx, COLO_EINVAL, "null map set");
            P.sets[i] = make_view(opts->sets[i]);
        }
    }
    P.nprof = static_cast<uint32_t>(nprofiles);
    P.has_sets = opts->sets ? 1u : 0u;
    P.arr = d_arrival;
    P.p = d_prompt;
    P.o = d_output;
    P.dev_off = d_dev_offsets;
    P.dev_prof = d_dev_profile;
    P.ndev = static_cast<uint32_t>(ndev);
    P.tau = opts->tau;
    P.samples = opts->d_samples;
    P.sample_off = opts->d_sample_offsets;
    P.labels = opts->d_labels;
    P.batches = opts->d_batches;
    P.summary = opts->d_summary;
    P.hist = opts->d_hist;
    P.nfilters = opts->d_hist ? opts->nfilters : 0;
    P.hist_shift = opts->hist_shift;
    P.filter_shift = opts->filter_shift;
    for (int f = 0; f < 3; ++f) P.prefix[f] = opts->filter_prefix[f];
    P.err = ctx->d_flag;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    COLO_CK(ctx, cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
    uint32_t blocks = static_cast<uint32_t>((ndev + kWarps - 1) / kWarps);
    k_replay<<<blocks, kWarps * 32, 0, ctx->stream>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    int flag = 0;
    COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (flag)
        return set_err(ctx, COLO_EVALIDATION,
                       "trace rejected: unsorted arrivals, zero tokens, or a query that cannot fit the device alone");
    return COLO_OK;
}

colo_status colo_serving_stats(colo_ctx* ctx, const colo_model* models, const colo_gpu* gpus, size_t nprofiles,
                               const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                               const uint64_t* d_dev_offsets, const uint16_t* d_dev_profile, size_t ndev, double tau,
                               double* pctl, colo_device_summary* totals) {
    if (!ctx || !pctl || !totals) return COLO_EINVAL;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    const size_t hbytes = sizeof(uint64_t) * 3 * COLO_HIST_BINS;
    uint64_t* d_hist = nullptr;
    colo_device_summary* d_sum = nullptr;
    COLO_CK(ctx, cudaMalloc(&d_hist, hbytes));
    cudaError_t e = cudaMalloc(&d_sum, sizeof(colo_device_summary) * std::max<size_t>(ndev, 1));
    if (e != cudaSuccess) {
        cudaFree(d_hist);
        return cuda_err(ctx, e, "cudaMalloc(summary)");
    }
    std::vector<uint64_t> h(3 * static_cast<size_t>(COLO_HIST_BINS));
    std::vector<colo_device_summary> sums(ndev);
    colo_status st = COLO_OK;
    const double qs[3] = {0.50, 0.90, 0.99};
    uint64_t rank[3], b1[3], b2[3];
    uint64_t ntot = 0;
    *totals = colo_device_summary{};
    for (int pass = 0; pass < 3 && st == COLO_OK; ++pass) {
        colo_replay_opts o{};
        o.tau = tau;
        o.d_hist = d_hist;
        o.d_summary = pass == 0 ? d_sum : nullptr;
        if (pass == 0) {
            o.nfilters = 1;
            o.filter_shift = 63;
            o.hist_shift = 42;
        } else {
            o.nfilters = 3;
            o.filter_shift = pass == 1 ? 42 : 21;
            o.hist_shift = pass == 1 ? 21 : 0;
            for (int f = 0; f < 3; ++f) o.filter_prefix[f] = pass == 1 ? b1[f] : ((b1[f] << 21) | b2[f]);
        }
        e = cudaMemsetAsync(d_hist, 0, hbytes, ctx->stream);
        if (e != cudaSuccess) {
            st = cuda_err(ctx, e, "cudaMemset(hist)");
            break;
        }
        st = colo_replay_serving(ctx, models, gpus, nprofiles, d_arrival, d_prompt, d_output, n, d_dev_offsets,
                                 d_dev_profile, ndev, &o);
        if (st != COLO_OK) break;
        e = cudaMemcpy(h.data(), d_hist, sizeof(uint64_t) * o.nfilters * COLO_HIST_BINS, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            st = cuda_err(ctx, e, "hist D2H");
            break;
        }
        if (pass == 0) {
            e = cudaMemcpy(sums.data(), d_sum, sizeof(colo_device_summary) * ndev, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                st = cuda_err(ctx, e, "summary D2H");
                break;
            }
            for (const auto& s : sums) {
                totals->generated_tokens += s.generated_tokens;
                totals->slow_tokens += s.slow_tokens;
                totals->slow_queries += s.slow_queries;
                totals->batches += s.batches;
                totals->peak_device_bytes = std::max(totals->peak_device_bytes, s.peak_device_bytes);
                totals->max_batch_size = std::max(totals->max_batch_size, s.max_batch_size);
                totals->end_time = std::max(totals->end_time, s.end_time);
                fixed_add(totals->tpt_sum, s.tpt_sum);
                totals->flags |= s.flags;
            }
            ntot = totals->generated_tokens;
            if (ntot == 0) {
                for (int i = 0; i < 4; ++i) pctl[i] = std::nan("");
                break;
            }
            for (int f = 0; f < 3; ++f) rank[f] = colo_nearest_rank_index(qs[f], ntot);
        }
        for (int f = 0; f < 3; ++f) {
            uint32_t bin;
            uint64_t rin;
            const uint64_t* hf = h.data() + static_cast<size_t>(pass == 0 ? 0 : f) * COLO_HIST_BINS;
            st = colo_hist_select(hf, COLO_HIST_BINS, rank[f], &bin, &rin);
            if (st != COLO_OK) {
                st = set_err(ctx, COLO_EBREACH, "histogram pass lost samples");
                break;
            }
            rank[f] = rin;
            if (pass == 0) b1[f] = bin;
            else if (pass == 1) b2[f] = bin;
            else {
                uint64_t bits = (b1[f] << 42) | (b2[f] << 21) | bin;
                double v;
                std::memcpy(&v, &bits, 8);
                pctl[f] = v;
            }
        }
    }
    if (st == COLO_OK && ntot) pctl[3] = fixed_mean(totals->tpt_sum, ntot);
    cudaFree(d_hist);
    cudaFree(d_sum);
    return st;
}

}  // extern "C"
