// colo_serving.cu -- serving-only replay (K4) and exact tail statistics (K5).
//
// The reference's Simulation is strictly sequential per instance
// (engine.hpp:140-164); instances share no state.  A device
// trace is therefore cut into segments and replayed in passes so the GPU is
// not limited to one warp per device:
//
//   A  speculate  every segment in parallel, assuming the server is idle when
//                 the segment's first query arrives; records the exit state
//                 and the first kRegen idle batch starts ("regeneration
//                 points": at an idle start the whole replay state is reset to
//                 (head, T = arrival[head]), so two runs that share one agree
//                 from there on).
//   B  resolve    one warp per device walks its segments in order: the true
//                 entry state of segment k is the exit of k-1; the segment is
//                 re-run only until the true run reaches an idle start that the
//                 speculative run also had, then the speculative exit is taken.
//   C  replay     every segment in parallel from its true entry state, writing
//                 samples, labels, batch records, histograms and partial sums.
//   D  finalize   per-device summaries from the segment partials; dense batch
//                 lists and the replay-derived verdicts.
//
// Inside a batch the warp's lanes own decode steps: lane l folds step k0+l's
// duration over the batch members in batch order (engine.hpp:358-365), then
// the absolute-time fold now_k = now_{k-1} + d_k runs through the lanes in
// order via shuffles -- every f64 operation is the reference's, in the
// reference's order, so all passes reproduce Simulation::run bit for bit.
// Reference paths are relative to /root/reference/proj/.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "colo_internal.h"
#include "colo_replay.cuh"

using namespace colo;

namespace {

constexpr int kWarps = 4;    // warps per CTA
constexpr int kStage = 256;  // batch members staged in shared memory per warp
constexpr int kRegen = 30;   // idle batch starts recorded per speculative segment
constexpr double kSpecGiveUp = 900.0;  // s of queueing after which a speculative run without idle starts stops
#ifndef COLO_SAT_HDR
#define COLO_SAT_HDR 4
#endif
constexpr int kSatHdr = COLO_SAT_HDR;  // per all-queued record: its chain sums in kSatHdr candidate binades (k_sat_durations)
#ifndef COLO_REPLAY_BLOCKS
#define COLO_REPLAY_BLOCKS 5
#endif
constexpr int kReplayBlocks = COLO_REPLAY_BLOCKS;
#ifndef COLO_SPEC_BLOCKS
#define COLO_SPEC_BLOCKS 6  // resident CTAs per SM k_speculate is compiled for
#endif  // resident CTAs per SM the replay pass is compiled for
constexpr int kTileBytes = kWarps * 32 * 33 * 8;   // k_replay_full's dynamic shared memory
constexpr unsigned FULL = 0xffffffffu;

struct DevProfile {
    colo_model m;
    uint64_t budget;  // capacity - reserve - weights, engine.hpp:278-280
    uint64_t fixed;   // weights + reserve, engine.hpp:141
};

struct Seg {
    uint32_t dev, pad;
    uint64_t start, end;  // device-local query range
};

// One all-queued batch record (k_sat_durations), dense in the order
// k_sat_partition's pass 2 forms them: within a partition segment record
// r + 1 starts where record r ends, so the resolve pass streams records
// instead of chasing sat_end.  R[c]: the decode chain's sum in units of the
// binade (binade of the last arrival) + c (~0 = not usable); the step
// durations are at sat_dk[doff], K of them.
struct alignas(16) SatRec {
    uint64_t R[kSatHdr];
    uint64_t doff;
    uint32_t start, end;  // device-local [start, end)
    uint32_t K, dev;
    double pre;           // prefill duration (engine.hpp:321-325)
    double alast;         // the batch's last arrival (the fast path needs alast <= T)
    uint64_t need;        // sum of the members' serving memory (engine.hpp:297-306)
};

// the record's chain sum for binade offset c (0 <= c < kSatHdr)
__device__ __forceinline__ uint64_t rec_R(const SatRec& x, int c) {
    uint64_t r = x.R[0];
#pragma unroll
    for (int i = 1; i < kSatHdr; ++i) r = c == i ? x.R[i] : r;
    return r;
}

struct SpecOut {
    uint64_t exit_head;
    double exit_T;
    uint32_t nregen;
    uint32_t regen[kRegen + 1];  // device-local offsets from the segment start
    // struct_out: batch count, peak need and largest batch of the speculative
    // run's interval i (batches from regen[i-1] up to regen[i]; interval 0 from
    // the segment start, interval kRegen to the segment end)
    uint32_t ib[kRegen + 1], imaxb[kRegen + 1];
    uint64_t ineed[kRegen + 1];
};

struct Entry {
    uint64_t head;
    double T;
};

struct Partial {
    uint64_t gen, slow_tok, slow_q, nbatch, max_need, maxb;
    uint64_t acc[3];
    uint64_t flags;
    double t_end;
    uint64_t pad;
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
    uint32_t ndev, nsegs;
    const Seg* segs;
    const uint32_t* dev_seg;  // [ndev+1] first segment of each device
    SpecOut* spec;
    Entry* entry;
    Partial* part;
    uint64_t* seg_base;       // device-local sample offset at each segment start
    double tau;
    double* samples;
    const uint64_t* sample_off;
    uint8_t* labels;
    colo_batch* bstage;       // batch record staged at its first query's global index
    uint8_t* bflag;
    uint64_t* vstage;         // compact stage for d_verdicts: (n << 32) | max_incoming at the first query, 0 elsewhere
    uint32_t* verdicts;
    colo_batch* batches;
    colo_device_summary* summary;
    uint64_t* hist;
    uint32_t nfilters, hist_shift, filter_shift;
    uint64_t prefix[3];
    int* err;
    // Saturated fast path of the resolve pass (see k_sat_partition): per
    // query q, the batch start_serving_batch forms at q when every query has
    // already arrived -- [q, sat_end[q]) -- and its record (SatRec: step count,
    // prefill, chain sums, per-step decode durations).  sat_end == 0: no record at q.
    uint32_t* sat_end;     // [dev_off[d] + q]
    uint32_t* sat_rec;     // [dev_off[d] + q] record index
    SatRec* sat_recs;
    uint64_t sat_nrec;     // records in sat_recs
    uint64_t* sat_recbase; // [pseg] record count, then its base (exclusive scan)
    const Seg* psegs;      // partition segments (longer than the replay segments: the greedy
    uint32_t npsegs;       // partition from a segment's start needs a few batches to meet the true one)
    uint64_t* sat_seg;     // [pseg] step durations of the segment's records, then their base (exclusive scan)
    uint64_t* sat_exit;    // [pseg] pass 1: where the segment's own partition leaves it
    uint32_t sat_pass;     // k_sat_partition pass (1 or 2)
    uint64_t* sat_seg_start;  // [pseg] first recorded batch (pass 2)
    double* sat_dk;
    uint32_t sat_on;
    uint32_t singles;  // idle starts 32 at a time (run_batches); COLO_SINGLES=0 turns it off
    // Sparse stats passes (serving_stats): the first pass records, at each
    // batch's first query, its start time and the range of its samples' top
    // 21-bit bins (bmeta_bins: valid<<63 | idle<<62 | max<<21 | min); the
    // narrowing passes then replay only batches whose range covers a filter bin
    double* bmeta_start;
    uint64_t* bmeta_bins;
    const double* sparse_start;  // the same records, read by k_sparse_hist
    const uint64_t* sparse_bins;
    unsigned long long* dbg;  // COLO_REPLAY_TIMING: [0] fast-path batches, [1] other batches of the resolve pass
    // decode-step latency table per profile: dtab[pi][x] = gamma + delta * x for
    // every context x < dtab_n (cost_model.hpp:28-35 with batch 1, the same f64
    // ops); k_sat_durations' folds load a term instead of computing it (in the
    // replay passes computing it is as fast: B200's f64 pipe keeps up with L1)
    const double* dtab[kMaxSets];
    uint64_t dtab_n;        // 0 = no table
    unsigned long long* maxctx;  // k_validate: max p + o over the trace
    // first stats pass: the speculative and resolve passes also write every
    // batch's start to bmeta (member positions cleared, within the segment)
    // and its counts (SpecOut intervals / Partial), so no separate structure
    // pass runs before k_batch_stats
    uint32_t struct_out;
    // k_batch_stats, first stats pass: the histogram bins [hwin_base, hwin_base +
    // kHistWin) are counted in shared memory per CTA (u32; hwin = 0: off)
    uint32_t hwin_base, hwin;
};

enum { RUN_SPEC = 0, RUN_RESOLVE = 1, RUN_FULL = 2 };

struct Acc {  // per-warp outputs of RUN_FULL (every lane holds its own partials)
    uint64_t gen = 0, slow_tok = 0, slow_q = 0, nbatch = 0, max_need = 0, maxb = 0;
    uint64_t acc[3] = {0, 0, 0};
    uint32_t flags = 0;
    uint64_t sample_pos = 0;
};

// Replays whole batches from (head, T) while head < stop (engine.hpp:270-387).
// SPEC records idle batch starts into *sp; RESOLVE stops (synced = true) at
// the first idle start that the speculative run *sp also had; FULL writes all
// outputs.  head/T are updated in place.
template <int MODE>
__device__ void run_batches(const ReplayParams& P, uint32_t d, uint64_t& head, double& T, uint64_t stop,
                            uint64_t seg_start, SpecOut* sp, bool& synced, Acc& A, uint2* sPO, double* sPD,
                            double* sDK, double* sT) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t pi = P.dev_prof[d];
    const colo_model& m = P.prof[pi].m;
    const uint64_t budget = P.prof[pi].budget;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const double* __restrict__ arr = P.arr + lo;
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;
    const bool want_hist = MODE == RUN_FULL && P.hist != nullptr;
    // every decode step duration >= the step constant (positive coefficients, validate_profile_pair)
    const bool dpos = m.decode_coef_const >= 0x1p-700 && m.decode_coef_context >= 0.0;
    uint64_t tail_ptr = head;
    uint32_t ridx = 0;
    const uint32_t nreg = MODE == RUN_RESOLVE ? min(sp->nregen, static_cast<uint32_t>(kRegen)) : 0u;
    synced = false;
    // batch structure out (bmeta starts + counts): the speculative and
    // resolve passes with struct_out
    const bool so = (MODE == RUN_SPEC || MODE == RUN_RESOLVE) && P.struct_out;
    uint32_t ib = 0, imaxb = 0;  // SPEC with struct_out: lane i holds interval i
    uint64_t ineed = 0;
    auto mark = [&](uint64_t h, uint64_t e, double st, bool idl) {  // warp-uniform; [h, e) one batch
        const uint64_t ce = min(e, stop);
        for (uint64_t j = h + 1 + lane; j < ce; j += 32) P.bmeta_bins[lo + j] = 0;
        if (lane == 0) {
            P.bmeta_start[lo + h] = st;
            P.bmeta_bins[lo + h] = (1ull << 63) | (idl ? 1ull << 62 : 0ull);
        }
    };
    auto count_batch = [&](uint64_t need, uint64_t nb) {  // warp-uniform, one batch
        if (MODE == RUN_SPEC) {
            if (lane == min(ridx, static_cast<uint32_t>(kRegen))) {
                ++ib;
                ineed = max(ineed, need);
                imaxb = max(imaxb, static_cast<uint32_t>(min(nb, static_cast<uint64_t>(0xffffffffu))));
            }
        } else {
            ++A.nbatch;
            A.max_need = max(A.max_need, need);
            A.maxb = max(A.maxb, nb);
        }
    };
    while (head < stop && head < N) {
        // ---- batch window: engine.hpp:146-147,178-188,270-276 -------------------
        uint64_t tail;
        const SatRec* rrec_head = nullptr;  // FULL: the all-queued record that is this batch
        bool idle_b = false;
        uint32_t bmin = 0xffffffffu, bmax = 0;  // bins (bits >> 42) of this batch's samples
        const double ah = arr[head];
        if (ah > T && P.singles && m.decode_coef_const >= 0.0 && m.decode_coef_context >= 0.0) {
            // ---- idle starts, up to 32 at a time -------------------------------
            // An idle start is a batch of one query that starts at its arrival
            // (T = arr[q]), so its whole timeline depends on q alone.  Lane l
            // takes query head+l.  It is the next batch iff every lane before
            // it is and arr[head+l] > T_end(l-1); the exact-arithmetic decode
            // time S = o*gamma + delta*(o*p + o(o-1)/2) bounds T_end to within
            // o rounding steps, so lanes whose arrival clears the bound by that
            // margin are certain, and the block stops before the first lane
            // that is not (the sequential loop below takes it).  The batches'
            // step chains then run one per lane in 32-step windows through a
            // shared-memory tile, and each batch's samples are post-processed
            // with lanes = steps, exactly as the per-batch path does.
            const uint64_t q = head + lane;
            const bool inr = q < stop && q < N;
            const uint32_t pq = inr ? pp[q] : 0u, oq = inr ? po[q] : 0u;
            const double aq = inr ? arr[q] : 0.0;
            const double tq = static_cast<double>(pq), od = static_cast<double>(oq);
            const double gam = m.decode_coef_const, del = m.decode_coef_context;
            // prefill of one member: 0.0 + (lin*t + (quad*t)*t) (cost_model.hpp:18-25)
            const double t_pre = (aq + 0.0) + (0.0 + (m.prefill_coef_linear * tq + m.prefill_coef_quad * tq * tq));
            const double S = od * gam + del * (od * tq + 0.5 * od * (od - 1.0));
            const double est = t_pre + S;
            const double hi_end = est + (8.0 * od * fabs(est) * 0x1p-52 + 1e-9 * S);
            const double prev_hi = __shfl_up_sync(FULL, hi_end, 1);
            const bool fits = inr && (lane == 0 || aq > prev_hi);
            const uint32_t bad = __ballot_sync(FULL, !fits);
            const uint32_t nv = bad ? static_cast<uint32_t>(__ffs(bad) - 1) : 32u;  // lanes [0, nv): batches
            uint32_t hb = 0;
            if constexpr (MODE == RUN_RESOLVE) {  // stop at the first idle start the speculative run also had
                const uint32_t rel = static_cast<uint32_t>(q - seg_start);
                bool hit = false;
                for (uint32_t i = 0; i < nreg; ++i) hit |= sp->regen[i] == rel;
                hb = __ballot_sync(FULL, hit && lane < nv);
            }
            if (so && MODE != RUN_FULL) {  // the window's batches (up to a sync point) into bmeta and the counts
                const uint32_t nw = hb ? static_cast<uint32_t>(__ffs(hb) - 1) : nv;
                const bool vw = lane < nw;
                if (vw) {
                    P.bmeta_start[lo + q] = aq + 0.0;
                    P.bmeta_bins[lo + q] = (1ull << 63) | (1ull << 62);
                }
                const uint64_t need = vw ? serving_memory(m, static_cast<uint64_t>(pq) + oq, 1) : 0ull;
                if (MODE == RUN_SPEC) {  // lane l's batch is regen point ridx + l: it opens interval ridx + l + 1
                    const int src = static_cast<int>(lane) - static_cast<int>(ridx) - 1;
                    const uint64_t nd = __shfl_sync(FULL, need, static_cast<uint32_t>(src) & 31u);
                    if (src >= 0 && src < static_cast<int>(nw) && lane < static_cast<uint32_t>(kRegen)) {
                        ++ib;
                        ineed = max(ineed, nd);
                        imaxb = max(imaxb, 1u);
                    }
                    const bool capped = vw && ridx + lane + 1 >= static_cast<uint32_t>(kRegen);
                    const uint32_t nc = __popc(__ballot_sync(FULL, capped));
                    const uint64_t mc = warp_max_u64(capped ? need : 0ull);
                    if (lane == static_cast<uint32_t>(kRegen) && nc) {
                        ib += nc;
                        ineed = max(ineed, mc);
                        imaxb = max(imaxb, 1u);
                    }
                } else {
                    A.nbatch += nw;
                    A.max_need = max(A.max_need, warp_max_u64(need));
                    if (nw) A.maxb = max(A.maxb, static_cast<uint64_t>(1));
                }
            }
            if (hb) {
                head += __ffs(hb) - 1;
                synced = true;
                return;
            }
            if (MODE == RUN_SPEC) {
                if (lane < nv && ridx + lane < kRegen) sp->regen[ridx + lane] = static_cast<uint32_t>(q - seg_start);
                ridx += nv;
            }
            const bool v = lane < nv;
            const uint32_t ov = v ? oq : 0u;
            double now = t_pre, kd = 0.0;
            if (MODE != RUN_FULL) {
                // only the block's last batch's end is used here (T for the next
                // query), so its chain alone runs, 128 steps at a time across the
                // warp: a scan while it stays in one binade, else sequentially
                const uint32_t L = nv - 1;
                double t = __shfl_sync(FULL, t_pre, L);
                const double tqL = __shfl_sync(FULL, tq, L);
                const uint32_t oL = __shfl_sync(FULL, ov, L);
                for (uint32_t k0 = 0; k0 < oL; k0 += 128) {
                    const uint32_t K = min(128u, oL - k0);
                    double dk[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        const uint32_t i = 32 * r + lane;
                        dk[r] = i < K ? 0.0 + (gam + del * (tqL + static_cast<double>(k0 + i))) : 0.0;
                    }
                    double te;
                    if (dpos ? chain_fast_end<true>(t, dk, K, te) : chain_fast_end(t, dk, K, te)) {
                        t = te;
                    } else {
                        for (uint32_t i = 0; i < K; ++i) t = t + (0.0 + (gam + del * (tqL + static_cast<double>(k0 + i))));
                    }
                }
                now = t;
            } else {
                uint32_t kmax = ov;
#pragma unroll
                for (int s = 16; s > 0; s >>= 1) kmax = max(kmax, __shfl_xor_sync(FULL, kmax, s));
                uint32_t ex = ov;  // sample slots: the batches' samples in batch order
#pragma unroll
                for (int s = 1; s < 32; s <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, ex, s);
                    if (lane >= static_cast<uint32_t>(s)) ex += y;
                }
                const uint64_t spos = A.sample_pos + ex - ov;
                A.sample_pos += __shfl_sync(FULL, ex, 31);
                // exact TPT sum by telescoping when every step time lies in [t_pre, 2 t_pre]
                // (each sample T_k - T_{k-1} is then exact, Sterbenz)
                const bool tl = v && t_pre >= 0x1p-44 && hi_end <= 2.0 * t_pre;
                if (tl) acc_fixed_sub(A.acc, A.flags, t_pre, 1u);
                const uint32_t tlm = __ballot_sync(FULL, tl);
                uint32_t slowm = 0;
                double* row = sT + lane * 33;
                for (uint32_t k0 = 0; k0 < kmax; k0 += 32) {
                    row[0] = now;  // T_{k0-1}
#pragma unroll 8
                    for (uint32_t i = 0; i < 32; ++i) {
                        if (k0 + i < ov) {
                            now = now + (0.0 + (gam + del * (tq + kd)));
                            kd += 1.0;
                        }
                        row[1 + i] = now;
                    }
                    __syncwarp();
                    for (uint32_t b = 0; b < nv; ++b) {  // batch b's window, lanes = steps
                        const uint32_t ob = __shfl_sync(FULL, ov, b);
                        if (k0 >= ob) continue;
                        const uint32_t k = k0 + lane;
                        const bool live = k < ob;
                        const double s = sT[b * 33 + 1 + lane] - sT[b * 33 + lane];
                        const bool slow = live && s > P.tau;
                        if (__ballot_sync(FULL, slow)) slowm |= 1u << b;
                        A.slow_tok += slow;
                        if (want_hist) {
                            const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
                            const uint64_t hb = bits >> P.filter_shift;
                            const uint32_t nf = P.nfilters;
                            const bool any = live && (hb == P.prefix[0] || (nf > 1 && hb == P.prefix[1]) ||
                                                      (nf > 2 && hb == P.prefix[2]));
                            if (__any_sync(FULL, any))
                                for (uint32_t f = 0; f < nf; ++f)
                                    hist_add1(P.hist,
                                              f * COLO_HIST_BINS +
                                                  static_cast<uint32_t>((bits >> P.hist_shift) & (COLO_HIST_BINS - 1)),
                                              live && hb == P.prefix[f]);
                        }
                        if (live && !((tlm >> b) & 1u)) acc_fixed(A.acc, A.flags, s, 1u);
                        const uint64_t sb = __shfl_sync(FULL, spos, b);
                        if (live && P.samples) P.samples[sb + k] = s;
                    }
                    __syncwarp();
                }
                if (tl) acc_fixed(A.acc, A.flags, now, 1u);
                const uint64_t need = v ? serving_memory(m, static_cast<uint64_t>(pq) + oq, 1) : 0ull;
                if (MODE == RUN_FULL && v && P.bmeta_bins) {
                    // a conservative bin range without looking at the samples: d_k grows with k
                    // (delta >= 0) and each sample is d_k within one rounding of the time (<= ulp(T_end))
                    const double d_first = 0.0 + (gam + del * tq);
                    const double d_last = 0.0 + (gam + del * (tq + static_cast<double>(oq - 1)));
                    const double ue = fabs(now) * 0x1p-51 + 0x1p-1000;
                    const double slo = d_first - ue - d_first * 0x1p-40, shi = d_last + ue + d_last * 0x1p-40;
                    const uint32_t blo = slo > 0.0 ? static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(slo)) >> 42) : 0u;
                    const uint32_t bhi = static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(shi)) >> 42);
                    P.bmeta_start[lo + q] = aq + 0.0;
                    P.bmeta_bins[lo + q] = (1ull << 63) | (1ull << 62) | (static_cast<uint64_t>(bhi) << 21) | blo;
                }
                if (MODE == RUN_FULL && v) {  // (the speculative passes write no outputs)
                    const bool slowq = (slowm >> lane) & 1u;  // a lone query's tokens are every step
                    A.gen += ov;
                    A.slow_q += slowq;
                    if (P.labels) P.labels[lo + q] = slowq ? 1 : 0;
                    if (P.bstage) {
                        colo_batch b;
                        b.start = aq + 0.0;
                        b.end = now;
                        b.first = static_cast<uint32_t>(q);
                        b.n = 1;
                        b.need_total = need;
                        const uint64_t inc = static_cast<uint64_t>(pq) + oq;
                        b.max_incoming = inc < 0xffffffffull ? static_cast<uint32_t>(inc) : 0xffffffffu;
                        b.verdict = 0;
                        P.bstage[lo + q] = b;
                        P.bflag[lo + q] = 1;
                    }
                    if (P.vstage) {
                        const uint64_t inc = static_cast<uint64_t>(pq) + oq;
                        P.vstage[lo + q] = (1ull << 32) | (inc < 0xffffffffull ? inc : 0xffffffffull);
                    }
                }
                A.max_need = max(A.max_need, warp_max_u64(need));
                A.maxb = max(A.maxb, static_cast<uint64_t>(1));
                A.nbatch += nv;
            }
            if (MODE == RUN_FULL && P.dbg && lane == 0) {
                atomicAdd(P.dbg + 4, static_cast<unsigned long long>(nv));
                atomicAdd(P.dbg + 5, 1ull);
            }
            T = __shfl_sync(FULL, now, nv - 1);
            head += nv;
            tail_ptr = head;
            __syncwarp();
            continue;
        }
        if (ah > T) {  // idle: the first popped arrival starts a batch alone
            if (MODE == RUN_SPEC) {
                if (lane == 0 && ridx < kRegen) sp->regen[ridx] = static_cast<uint32_t>(head - seg_start);
                ++ridx;
            }
            if constexpr (MODE == RUN_RESOLVE) {
                const uint32_t rel = static_cast<uint32_t>(head - seg_start);
                while (ridx < nreg && sp->regen[ridx] < rel) ++ridx;
                if (ridx < nreg && sp->regen[ridx] == rel) {
                    synced = true;  // both runs restart identically from this idle start
                    return;
                }
            }
            T = ah;
            tail = head + 1;
            tail_ptr = head + 1;
            idle_b = true;
        } else {  // queued: every arrival with time <= T has been popped
            if (MODE == RUN_RESOLVE && P.sat_on) {
                // Saturated fast path: a record at head whose last member has
                // already arrived is exactly the batch start_serving_batch forms
                // (engine.hpp:292-306 never reaches the queue's end), so only the
                // absolute-time chain remains: now = (T + 0.0) + prefill, then
                // now += d_k for every step, in order.  While now stays in its
                // binade that chain is now + u * R with the record's precomputed
                // R (exact, see chain_fast_end), so a record costs a few integer
                // operations.  The records of a partition come dense in chain
                // order: the warp loads 32 at a time (lane l: record r + l) and
                // walks them on broadcasts, re-entering through sat_rec where a
                // partition segment's chain does not continue.
                const uint32_t* __restrict__ se = P.sat_end + lo;
                const uint32_t* __restrict__ srec = P.sat_rec + lo;
                const double* __restrict__ pool = P.sat_dk;
                bool progressed = false;
                bool more = se[head] != 0;
                uint64_t r = more ? srec[head] : 0;
                auto load_rec = [&](uint64_t i) {
                    SatRec y;
                    if (i < P.sat_nrec) {
                        y = P.sat_recs[i];
                    } else {
                        y.dev = 0xffffffffu;
                        y.start = y.end = 0;
                    }
                    return y;
                };
                // window r in x; window r + 32 is loaded while x is walked
                SatRec x = more ? load_rec(r + lane) : SatRec{};
                while (more) {
                    const uint64_t rl = r + lane;
                    const SatRec xn = load_rec(r + 32 + lane);
                    const double al = x.dev == d ? x.alast : 0.0;
                    if (P.dbg && lane == 0) atomicAdd(P.dbg + 3, 1ull);
                    {  // the windows after that: into L2
                        const char* q = reinterpret_cast<const char*>(P.sat_recs + r + 64) + lane * 2 * sizeof(SatRec);
                        if (r + 128 < P.sat_nrec) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
                    }
                    // The window in one step: while T stays in its binade e every
                    // addend is an integer number of units u = 2^(e-52) (fl(T + x)
                    // = T + RN_u(x), no ties), so record l moves T's bit pattern by
                    // RN_u(pre_l)/u + R_l[e] and the T at every record boundary is an
                    // exclusive warp scan.  Lanes up to the first one whose record
                    // does not continue the chain, has not fully arrived, needs
                    // another binade or has a tie are applied at once; that record
                    // then goes through the per-record loop below.
                    uint32_t l = 0;
                    if (T >= 0x1p-190 && T <= 0x1p190) {
                        const uint64_t t0 = static_cast<uint64_t>(__double_as_longlong(T));
                        const int eT = binade_of(T);
                        const double sc = pow2i(52 - eT);
                        const uint32_t pend = __shfl_up_sync(FULL, x.end, 1);
                        bool v = rl < P.sat_nrec && x.dev == d && x.K <= 128 && al >= 0x1p-190 &&
                                 static_cast<uint64_t>(x.start) == (lane == 0 ? head : static_cast<uint64_t>(pend)) &&
                                 x.start < stop && x.start < N;
                        const int c = eT - binade_of(al);
                        const uint64_t Rc = rec_R(x, c);
                        v = v && c >= 0 && c < kSatHdr && Rc != ~0ull;
                        uint64_t rp = 0;
                        v = v && rn_units(x.pre, sc, rp);
                        const uint64_t a = v ? rp + Rc : 0ull;
                        uint64_t incl = a;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint64_t y = __shfl_up_sync(FULL, incl, o);
                            if (lane >= static_cast<uint32_t>(o)) incl += y;
                        }
                        v = v && (t0 & ((1ull << 52) - 1)) + incl < (1ull << 52);
                        const double tl = __longlong_as_double(static_cast<long long>(t0 + (incl - a)));
                        v = v && al <= tl;
                        const uint32_t bad = __ballot_sync(FULL, !v);
                        l = bad ? static_cast<uint32_t>(__ffs(bad) - 1) : 32u;
                        if (so && l > 0) {
                            const bool tk = lane < l;
                            // members of the l records (within the segment), then their starts
                            const uint64_t ce = min(static_cast<uint64_t>(__shfl_sync(FULL, x.end, l - 1)), stop);
                            for (uint64_t j = head + lane; j < ce; j += 32) P.bmeta_bins[lo + j] = 0;
                            __syncwarp();
                            if (tk) {  // start = T + 0.0 (engine.hpp:319) = T here (T > 0)
                                P.bmeta_start[lo + x.start] = tl;
                                P.bmeta_bins[lo + x.start] = 1ull << 63;
                            }
                            A.nbatch += l;
                            A.max_need = max(A.max_need, warp_max_u64(tk ? x.need : 0ull));
                            A.maxb = max(A.maxb, warp_max_u64(tk ? static_cast<uint64_t>(x.end - x.start) : 0ull));
                        }
                        if (l > 0) {
                            T = __longlong_as_double(static_cast<long long>(t0 + __shfl_sync(FULL, incl, l - 1)));
                            head = __shfl_sync(FULL, x.end, l - 1);
                            progressed = true;
                            if (P.dbg && lane == 0) {
                                atomicAdd(P.dbg, static_cast<unsigned long long>(l));
                                atomicAdd(P.dbg + 2, static_cast<unsigned long long>(l));
                            }
                        }
                    }
                    bool chain_break = false;  // else: the window is done, or the fast path ends here
                    const uint32_t l1 = l < 32 ? l + 1 : 32u;  // one record past the scanned ones, then rescan
                    for (; l < l1; ++l) {
                        const uint32_t xs = __shfl_sync(FULL, x.start, l), xe = __shfl_sync(FULL, x.end, l);
                        const uint32_t xd = __shfl_sync(FULL, x.dev, l);
                        if (head >= stop || head >= N) break;
                        if (xd != d || xs != head) {
                            chain_break = true;
                            break;
                        }
                        const double alast = __shfl_sync(FULL, al, l);
                        if (!(alast <= T)) break;  // a member has not arrived: form it the slow way
                        const double pre = __shfl_sync(FULL, x.pre, l);
                        const uint32_t K = __shfl_sync(FULL, x.K, l);
                        double now = (T + 0.0) + pre;
                        const bool rng = K <= 128 && now >= 0x1p-190 && now <= 0x1p190 && alast >= 0x1p-190;
                        const int c = rng ? binade_of(now) - binade_of(alast) : -1;
                        const uint64_t Rc = rec_R(x, c);
                        const uint64_t R = __shfl_sync(FULL, Rc, l);
                        const uint64_t nbits = static_cast<uint64_t>(__double_as_longlong(now));
                        const uint64_t mnow = (nbits & ((1ull << 52) - 1)) | (1ull << 52);
                        if (c >= 0 && c < kSatHdr && R != ~0ull && R < (1ull << 53) - mnow) {
                            if (P.dbg && lane == 0) atomicAdd(P.dbg + 2, 1ull);
                            now = __longlong_as_double(
                                static_cast<long long>((nbits & ~((1ull << 52) - 1)) | ((mnow + R) & ((1ull << 52) - 1))));
                        } else {
                            const uint64_t dof = __shfl_sync(FULL, x.doff, l);
                            if (K <= 128) {
                                double cur[4];
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const uint32_t i = 32 * q + lane;
                                    cur[q] = i < K ? pool[dof + i] : 0.0;
                                }
                                double fast_end;
                                if (chain_fast_end(now, cur, K, fast_end)) {
                                    now = fast_end;
                                } else {
#pragma unroll
                                    for (int q = 0; q < 4; ++q) sDK[32 * q + lane] = cur[q];
                                    __syncwarp();
                                    if (lane == 0) sDK[0] = chain_fold(now, sDK, K);
                                    __syncwarp();
                                    now = sDK[0];
                                    __syncwarp();
                                }
                            } else {
                                for (uint32_t k0 = 0; k0 < K; k0 += 128) {
                                    const uint32_t cc = min(128u, K - k0);
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        const uint32_t i = 32 * q + lane;
                                        if (i < cc) sDK[i] = pool[dof + k0 + i];
                                    }
                                    __syncwarp();
                                    if (lane == 0) sDK[0] = chain_fold(now, sDK, cc);
                                    __syncwarp();
                                    now = sDK[0];
                                    __syncwarp();
                                }
                            }
                        }
                        if (so) {
                            mark(head, xe, T + 0.0, false);
                            ++A.nbatch;
                            A.max_need = max(A.max_need, __shfl_sync(FULL, x.need, l));
                            A.maxb = max(A.maxb, static_cast<uint64_t>(xe - xs));
                        }
                        T = now;
                        head = xe;
                        progressed = true;
                        if (P.dbg && lane == 0) atomicAdd(P.dbg, 1ull);
                    }
                    if (l == l1) {
                        r += l;
                        x = l == 32 ? xn : load_rec(r + lane);
                    } else if (chain_break && se[head] != 0) {
                        r = srec[head];  // the chain continues in another partition segment's records
                        x = load_rec(r + lane);
                    } else {
                        more = false;
                    }
                }
                if (progressed) continue;
            }
            if (MODE == RUN_SPEC && ridx <= 1 && T - ah > kSpecGiveUp) {
                // A deep backlog and no idle start since the segment's first query:
                // the speculative run stops and drops its regeneration points, so
                // the resolve pass replays this segment itself (at saturation
                // through the all-queued records) instead of waiting for the
                // queue to drain here
                ridx = 0;
                head = stop;
                break;
            }
            if (MODE == RUN_RESOLVE && P.dbg && lane == 0) atomicAdd(P.dbg + 1, 1ull);
            if (MODE == RUN_FULL && P.sat_on && P.sat_end[lo + head] != 0) {
                // an all-queued record at head whose last member has arrived is
                // the batch formation would build (see the resolve fast path):
                // no queue-tail search and no need scan
                const SatRec* __restrict__ q = P.sat_recs + P.sat_rec[lo + head];
                if (q->dev == d && q->start == head && q->alast <= T) rrec_head = q;
            }
            if (rrec_head == nullptr) {
                tail_ptr = find_tail(arr, N, tail_ptr < head ? head : tail_ptr, T);
                tail = tail_ptr;
            }
        }
        // ---- batch formation: FIFO, at least one, sum(need) <= budget (engine.hpp:292-306)
        uint64_t end = head, need_total = 0, max_inc = 0;
        uint32_t maxo = 0, mino = 0xffffffffu;
        if (MODE == RUN_FULL && rrec_head != nullptr) {
            end = rrec_head->end;
            need_total = rrec_head->need;
            for (uint64_t j0 = head; j0 < end; j0 += 32) {  // stage the members
                const uint64_t j = j0 + lane;
                const bool valid = j < end;
                const uint32_t pj = valid ? pp[j] : 0u, oj = valid ? po[j] : 0u;
                if (valid && j - head < kStage) {
                    sPO[j - head] = make_uint2(pj, oj);
                    sPD[j - head] = static_cast<double>(pj);
                }
                maxo = max(maxo, __reduce_max_sync(FULL, oj));
                max_inc = max(max_inc, warp_max_u64(static_cast<uint64_t>(pj) + oj));
                mino = min(mino, __reduce_min_sync(FULL, valid ? oj : 0xffffffffu));
            }
            tail = end;
        } else if (tail == head + 1) {  // one query in the queue: the batch is that query
            const uint32_t pj = pp[head], oj = po[head];
            need_total = serving_memory(m, static_cast<uint64_t>(pj) + oj, 1);
            if (lane == 0) {
                sPO[0] = make_uint2(pj, oj);
                sPD[0] = static_cast<double>(pj);
            }
            maxo = oj;
            if (MODE == RUN_FULL) {
                max_inc = static_cast<uint64_t>(pj) + oj;
                mino = oj;
            }
            end = tail;
        }
        while (end < tail) {
            const uint64_t j = end + lane;
            const bool valid = j < tail;
            const uint32_t pj = valid ? pp[j] : 0u, oj = valid ? po[j] : 0u;
            const uint64_t nd = valid ? serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) : 0ull;
            uint64_t incl = nd;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint64_t y = __shfl_up_sync(FULL, incl, s);
                if (lane >= static_cast<uint32_t>(s)) incl += y;
            }
            incl += need_total;
            const bool ok = valid && (j == head || incl <= budget);
            const uint32_t cnt = __popc(__ballot_sync(FULL, ok));
            if (ok && j - head < kStage) {
                sPO[j - head] = make_uint2(pj, oj);
                sPD[j - head] = static_cast<double>(pj);
            }
            maxo = max(maxo, __reduce_max_sync(FULL, ok ? oj : 0u));
            if (MODE == RUN_FULL) {  // (the other passes only need the batch's extent and step count)
                max_inc = max(max_inc, warp_max_u64(ok ? static_cast<uint64_t>(pj) + oj : 0ull));
                mino = min(mino, __reduce_min_sync(FULL, ok ? oj : 0xffffffffu));
            }
            if (cnt) need_total = __shfl_sync(FULL, incl, cnt - 1);
            end += cnt;
            if (cnt < 32) break;
        }
        __syncwarp();
        const uint64_t nb = end - head;
        // FULL pass: a batch the all-queued records describe exactly takes its
        // prefill and step durations from them (the same folds, done once)
        const bool recd = rrec_head != nullptr ||
                          ((MODE == RUN_FULL || (MODE == RUN_RESOLVE && P.struct_out)) && P.sat_on && P.sat_end[lo + head] == end);
        const SatRec* __restrict__ rrec = rrec_head != nullptr ? rrec_head : recd ? P.sat_recs + P.sat_rec[lo + head] : nullptr;
        const double* __restrict__ rdk = recd ? P.sat_dk + rrec->doff : nullptr;
        // The replay walks each array sequentially: keep the next ~1K queries of
        // prompt/output and the arrivals around the queue tail warm in L2 so the
        // dependent loads of later batches hit L2 instead of DRAM (issued when the
        // head crosses a 256-query line, not for every batch).
        if ((end ^ head) >> 8) {
            const uint64_t q = end + 512 + lane * 32;
            if (q < N) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + q));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(po + q));
            }
            const uint64_t a0 = (tail_ptr > end ? tail_ptr : end) + lane * 16;
            if (a0 < N) asm volatile("prefetch.global.L2 [%0];" ::"l"(arr + a0));
        }
        const bool staged = nb <= kStage;  // every member in shared memory (else read from L1/L2)
        auto member = [&](uint64_t j) -> uint2 { return staged ? sPO[j] : make_uint2(pp[head + j], po[head + j]); };
        // exact (double)p_j: p < 2^32 and k < 2^32, so (double)p + (double)k == (double)(p + k)
        auto member_pd = [&](uint64_t j) -> double { return staged ? sPD[j] : static_cast<double>(pp[head + j]); };

        // ---- prefill: left fold in batch order (engine.hpp:321-325) -------------
        // cost_model.hpp:18-25 with batch 1: 1.0 * (lin*t + (quad*t)*t) == lin*t + (quad*t)*t
        double dur = 0.0;
        if (recd) {
            dur = rrec->pre;
        } else {
#pragma unroll 4
            for (uint64_t j = 0; j < nb; ++j) {
                const double t = member_pd(j);
                dur += m.prefill_coef_linear * t + m.prefill_coef_quad * t * t;
            }
        }
        const double start = T + 0.0;  // prefill_start = now_ + stall, stall = 0
        double now = start + dur;      // PrefillDone time = every member's last_token_time
        // Exact TPT sum by telescoping: when every step time of the batch lies
        // in [now, 2 now], each sample T_k - T_{k-1} is exact (Sterbenz), so
        // sum_k alive_k * s_k = sum_j T_{o_j - 1} - n * now: one fixed-point
        // add per member instead of one per sample.  span bounds the batch's
        // decode time from above (n members, <= maxo steps of at most
        // n * (gamma + delta * (max_incoming + maxo)) each).
        bool tele = false;
        if (MODE == RUN_FULL) {
            const double span = static_cast<double>(maxo) *
                                (static_cast<double>(nb) * (m.decode_coef_const +
                                                            m.decode_coef_context * static_cast<double>(max_inc + maxo))) *
                                1.001;
            tele = now >= 0x1p-44 && span <= now && m.decode_coef_const >= 0.0 && m.decode_coef_context >= 0.0;
            if (tele && lane == 0) acc_fixed_sub(A.acc, A.flags, now, static_cast<uint32_t>(nb));
        }

        // ---- decode steps (engine.hpp:358-387) ---------------------------------
        // Lane l owns steps k0+l, k0+32+l, k0+64+l, k0+96+l: four independent
        // left folds over the members in batch order (cost_model.hpp:28-35,
        // batch 1: 1.0 * (gamma + delta*ctx)), unrolled so member loads and
        // multiplies overlap the accumulate chains; the step durations go to
        // shared memory and the absolute-time chain reads them back in order.
        uint32_t first_slow = 0xffffffffu;
        const double gam = m.decode_coef_const, del = m.decode_coef_context;
        for (uint32_t k0 = 0; k0 < maxo; k0 += 128) {
            double dk[4] = {0.0, 0.0, 0.0, 0.0};
            uint32_t alive[4] = {0, 0, 0, 0};
            const uint32_t kb = k0 + lane;
            double kd[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) kd[r] = static_cast<double>(kb + 32 * r);
            if (recd) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t k = kb + 32 * r;
                    if (k < maxo) dk[r] = rdk[k];
                }
                if (MODE != RUN_FULL) {
                } else if (mino == maxo) {  // every member alive at every step
#pragma unroll
                    for (int r = 0; r < 4; ++r) alive[r] = kb + 32 * r < maxo ? static_cast<uint32_t>(nb) : 0u;
                } else {
                    for (uint64_t j = 0; j < nb; ++j) {
                        const uint32_t oj = member(j).y;
#pragma unroll
                        for (int r = 0; r < 4; ++r) alive[r] += kb + 32 * r < oj;
                    }
                }
            } else if (staged) {
#pragma unroll 4
                for (uint64_t j = 0; j < nb; ++j) {
                    const uint32_t oj = sPO[j].y;
                    const double pj = sPD[j];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (kb + 32 * r < oj) {
                            dk[r] += gam + del * (pj + kd[r]);
                            ++alive[r];
                        }
                    }
                }
            } else {
                for (uint64_t j = 0; j < nb; ++j) {
                    const uint32_t oj = po[head + j];
                    const double pj = static_cast<double>(pp[head + j]);
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        if (kb + 32 * r < oj) {
                            dk[r] += gam + del * (pj + kd[r]);
                            ++alive[r];
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) sDK[32 * r + lane] = dk[r];
            const uint32_t cnt = min(128u, maxo - k0);
            if (MODE != RUN_FULL) {
                // only the batch's end is needed: the chain as one warp scan while
                // it stays in its binade, else one lane's sequential fold
                double te;
                if (dpos ? chain_fast_end<true>(now, dk, cnt, te) : chain_fast_end(now, dk, cnt, te)) {
                    now = te;
                } else {
                    __syncwarp();
                    if (lane == 0) sDK[0] = chain_fold(now, sDK, cnt);
                    __syncwarp();
                    now = sDK[0];
                }
                __syncwarp();
                continue;
            }
            __syncwarp();
            // absolute-time chain now_k = now_{k-1} + d_k, sequential on one
            // lane; the durations are overwritten by the absolute times
            if (!chain_fast_store(now, sDK, cnt) && lane == 0) chain_fold_store(now, sDK, cnt);
            __syncwarp();
            // the four 32-step rows are post-processed by one (not unrolled)
            // body, which reads its samples and alive counts back from shared
            // memory: a smaller kernel for the instruction cache
            const double now0 = now;
            uint32_t* const sAL = reinterpret_cast<uint32_t*>(sDK + 128);  // FULL: inside the warp's tile region
            if (MODE == RUN_FULL) {
#pragma unroll
                for (int r = 0; r < 4; ++r) sAL[32 * r + lane] = alive[r];
            }
            if (MODE == RUN_FULL && tele) {  // members whose last step is in this window: + T_{o_j - 1}
                for (uint64_t j = lane; j < nb; j += 32) {
                    const uint32_t last = member(j).y - 1;
                    if (last >= k0 && last < k0 + cnt) acc_fixed(A.acc, A.flags, sDK[last - k0], 1u);
                }
            }
            now = sDK[cnt - 1];
            __syncwarp();
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
            const uint32_t kr0 = k0 + 32 * r;
            if (kr0 >= maxo) break;
            const uint32_t k = kr0 + lane;
            if (MODE == RUN_FULL) {
                const uint32_t i = 32 * r + lane;  // sample = now - last_token_time
                const double s = i < cnt ? sDK[i] - (i ? sDK[i - 1] : now0) : 0.0;
                const uint32_t alv = sAL[i];
                const bool live = k < maxo;
                if (P.bmeta_bins && live && !(s < 0.0)) {  // (negative samples never match a filter)
                    const uint32_t bn = static_cast<uint32_t>(static_cast<uint64_t>(__double_as_longlong(s)) >> 42);
                    bmin = min(bmin, bn);
                    bmax = max(bmax, bn);
                }
                const bool slow = live && s > P.tau;
                const uint32_t sb = __ballot_sync(FULL, slow);
                if (sb && first_slow == 0xffffffffu) first_slow = kr0 + __ffs(sb) - 1;
                A.gen += alv;
                if (slow) A.slow_tok += alv;
                if (want_hist) {  // warp-aggregated: lanes with the same bin add once
                    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
                    const uint64_t hb = bits >> P.filter_shift;
                    const uint32_t nf = P.nfilters;
                    const bool any = live && (hb == P.prefix[0] || (nf > 1 && hb == P.prefix[1]) ||
                                              (nf > 2 && hb == P.prefix[2]));
                    if (__any_sync(FULL, any))  // most samples of a narrowing pass match no filter
                        for (uint32_t f = 0; f < nf; ++f)
                            hist_add(P.hist, f * COLO_HIST_BINS + static_cast<uint32_t>((bits >> P.hist_shift) & (COLO_HIST_BINS - 1)),
                                     alv, live && hb == P.prefix[f]);
                }
                if (live && !tele) {
                    acc_fixed(A.acc, A.flags, s, alv);
                }
                if (P.samples) {
                    // samples of step k occupy alive_k consecutive slots, steps in order
                    uint32_t ex = alv;
#pragma unroll
                    for (int sft = 1; sft < 32; sft <<= 1) {
                        const uint32_t y = __shfl_up_sync(FULL, ex, sft);
                        if (lane >= static_cast<uint32_t>(sft)) ex += y;
                    }
                    const uint32_t total = __shfl_sync(FULL, ex, 31);
                    const uint64_t pos = A.sample_pos + ex - alv;
                    for (uint32_t a = 0; a < alv; ++a) P.samples[pos + a] = s;
                    A.sample_pos += total;
                }
            }
            }
            __syncwarp();  // the rows' reads of sDK / sAL before the next window writes them
        }
        if (MODE == RUN_FULL) {
            // labels: a query is slow iff one of its tokens is (o_j > first slow step)
            for (uint64_t j = lane; j < nb; j += 32) {
                const bool slowq = member(j).y > first_slow;
                A.slow_q += slowq;
                if (P.labels) P.labels[lo + head + j] = slowq ? 1 : 0;
            }
            if (P.bmeta_bins) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    bmin = min(bmin, __shfl_xor_sync(FULL, bmin, o));
                    bmax = max(bmax, __shfl_xor_sync(FULL, bmax, o));
                }
                if (lane == 0) {
                    P.bmeta_start[lo + head] = start;
                    P.bmeta_bins[lo + head] = (1ull << 63) | (idle_b ? 1ull << 62 : 0ull) |
                                              (static_cast<uint64_t>(bmax) << 21) | bmin;
                }
            }
            if (lane == 0 && P.bstage) {
                colo_batch b;
                b.start = start;
                b.end = now;
                b.first = static_cast<uint32_t>(head);
                b.n = static_cast<uint32_t>(nb);
                b.need_total = need_total;
                b.max_incoming = max_inc < 0xffffffffull ? static_cast<uint32_t>(max_inc) : 0xffffffffu;
                b.verdict = 0;
                P.bstage[lo + head] = b;
                P.bflag[lo + head] = 1;
            }
            if (lane == 0 && P.vstage)
                P.vstage[lo + head] = (static_cast<uint64_t>(nb) << 32) | (max_inc < 0xffffffffull ? max_inc : 0xffffffffull);
            A.max_need = max(A.max_need, need_total);
            A.maxb = max(A.maxb, nb);
            ++A.nbatch;
            if (P.dbg && lane == 0) {
                atomicAdd(P.dbg + 6, 1ull);
                atomicAdd(P.dbg + 7, static_cast<unsigned long long>(nb));
            }
        }
        if (so && MODE != RUN_FULL) {
            mark(head, end, start, idle_b);
            count_batch(need_total, nb);
        }
        T = now;
        head = end;
        __syncwarp();
    }
    if (MODE == RUN_SPEC && lane == 0) sp->nregen = ridx;
    if (MODE == RUN_SPEC && so && lane <= static_cast<uint32_t>(kRegen)) {
        sp->ib[lane] = ib;
        sp->imaxb[lane] = imaxb;
        sp->ineed[lane] = ineed;
    }
}

// dtab[pi][x] = gamma + delta * (double)x: decode_step_latency(x, 1, false)
// (cost_model.hpp:28-35; 1.0 * v == v), the same f64 ops as the folds.
__global__ void k_fill_dtab(double* tab, uint64_t n, double gam, double del) {
    for (uint64_t x = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; x < n;
         x += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        tab[x] = gam + del * static_cast<double>(x);
}

// All-queued ("saturated") batch records.  The batch start_serving_batch
// forms at head q when every query up to its end has arrived depends on q
// alone (FIFO, at least one, sum(need) <= budget: engine.hpp:292-306 without
// reaching the queue's end), so any greedy partition yields valid records.
// One warp per partition segment walks a greedy partition in 256-query
// windows (lane l holds queries base+8l..+7, a warp scan gives the need
// prefix, one ballot cuts each batch).  Pass 1 starts at the segment's first
// query and only notes where its partition leaves the segment; pass 2 starts
// at the previous segment's pass-1 exit and records every batch that starts
// inside the segment.  Greedy partitions from different starts meet after
// some batches (and then coincide), so pass 2 continues, segment after
// segment, the partition the true run follows while the queue stays full.
__global__ void __launch_bounds__(kWarps * 32) k_sat_partition(const __grid_constant__ ReplayParams P) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w >= P.npsegs) return;
    const Seg sg = P.psegs[w];
    const uint32_t d = sg.dev;
    const uint32_t pi = P.dev_prof[d];
    const colo_model& m = P.prof[pi].m;
    const uint64_t budget = P.prof[pi].budget;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;
    const bool rec = P.sat_pass == 2;
    uint64_t h = sg.start, steps = 0;
    if (rec && sg.start > 0) h = P.sat_exit[w - 1];  // the previous segment of this device (same device: start > 0)
    if (lane == 0 && rec) P.sat_seg_start[w] = h;
    uint64_t nrec = 0;
    auto record = [&](uint64_t start, uint64_t end, uint32_t mo) {
        if (rec && lane == 0) P.sat_end[lo + start] = static_cast<uint32_t>(end);
        steps += mo;
        ++nrec;
    };
    while (h < sg.end) {
        const uint64_t base = h;
        uint64_t pre[8];
        uint32_t oo[8];
        uint64_t s = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint64_t j = base + lane * 8 + r;
            const bool v = j < N;
            const uint32_t pj = v ? pp[j] : 0u, oj = v ? po[j] : 0u;
            s += v ? serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) : 0ull;
            pre[r] = s;
            oo[r] = oj;
        }
        uint64_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint64_t excl = incl - s;
#pragma unroll
        for (int r = 0; r < 8; ++r) pre[r] += excl;  // need over [base, base + 8 lane + r]
        const uint64_t wend = min(base + 256, N);
        uint64_t hoff = 0;  // need over [base, h)
        while (h < wend && h < sg.end) {
            const uint64_t thr = hoff + budget;
            uint32_t fr = 8;
#pragma unroll
            for (int r = 7; r >= 0; --r) {
                const uint64_t j = base + lane * 8 + r;
                if (j > h && j < wend && pre[r] > thr) fr = r;
            }
            const uint32_t bal = __ballot_sync(FULL, fr < 8);
            uint64_t e;
            if (bal) {
                const uint32_t fl = __ffs(bal) - 1;
                e = base + fl * 8 + __shfl_sync(FULL, fr, fl);
            } else if (wend == N) {
                e = N;
            } else {
                break;  // the batch runs past the window: reload from h
            }
            uint32_t mo = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const uint64_t j = base + lane * 8 + r;
                if (j >= h && j < e) mo = max(mo, oo[r]);
            }
            mo = static_cast<uint32_t>(warp_max_u64(mo));
            record(h, e, mo);
            const uint64_t idx = e - 1 - base;
            uint64_t v = 0;
#pragma unroll
            for (int r = 0; r < 8; ++r) v = (idx & 7) == static_cast<uint64_t>(r) ? pre[r] : v;
            hoff = __shfl_sync(FULL, v, static_cast<int>(idx >> 3));
            h = e;
        }
        if (h == base) {  // one batch longer than the window: form it chunk by chunk
            uint64_t end = h, need_total = 0;
            uint32_t mo = 0;
            while (end < N) {
                const uint64_t j = end + lane;
                const bool valid = j < N;
                const uint32_t pj = valid ? pp[j] : 0u, oj = valid ? po[j] : 0u;
                const uint64_t nd = valid ? serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) : 0ull;
                uint64_t in2 = nd;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t y = __shfl_up_sync(FULL, in2, o);
                    if (lane >= static_cast<uint32_t>(o)) in2 += y;
                }
                in2 += need_total;
                const bool ok = valid && (j == h || in2 <= budget);
                const uint32_t c = __popc(__ballot_sync(FULL, ok));
                mo = max(mo, static_cast<uint32_t>(warp_max_u64(ok ? oj : 0u)));
                if (c) need_total = __shfl_sync(FULL, in2, c - 1);
                end += c;
                if (c < 32) break;
            }
            record(h, end, mo);
            h = end;
        }
    }
    if (lane == 0) {
        if (rec) {
            P.sat_seg[w] = steps;
            P.sat_recbase[w] = nrec;
        } else {
            P.sat_exit[w] = h;
        }
    }
}

// Prefill and per-step decode durations of every record, one warp per
// segment walking its records (the same folds, in the same order, as
// run_batches); the segment's step durations start at sat_seg[w].
__global__ void __launch_bounds__(kWarps * 32) k_sat_durations(const __grid_constant__ ReplayParams P) {
    __shared__ uint2 spo[kWarps][kStage];
    __shared__ double spd[kWarps][kStage];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w >= P.npsegs) return;
    const Seg sg = P.psegs[w];
    const uint32_t d = sg.dev;
    const uint32_t pi = P.dev_prof[d];
    const colo_model& m = P.prof[pi].m;
    const uint64_t lo = P.dev_off[d];
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;
    const double gam = m.decode_coef_const, del = m.decode_coef_context;
    uint2* sPO = spo[warp];
    double* sPD = spd[warp];
    uint64_t doff = P.sat_seg[w];
    uint64_t ridx = P.sat_recbase[w];
    uint64_t head = P.sat_seg_start[w];
    while (head < sg.end) {
        const uint64_t end = P.sat_end[lo + head];
        const uint64_t nb = end - head;
        const bool staged = nb <= kStage;
        uint64_t mi = 0;  // max p + o of the members (table coverage)
        if (staged)
            for (uint64_t j = lane; j < nb; j += 32) {
                const uint32_t pj = pp[head + j], oj = po[head + j];
                sPO[j] = make_uint2(pj, oj);
                sPD[j] = static_cast<double>(pj);
                mi = max(mi, static_cast<uint64_t>(pj) + oj);
            }
        const bool tab_ok = warp_max_u64(mi) < P.dtab_n;
        __syncwarp();
        auto member_pd = [&](uint64_t j) -> double { return staged ? sPD[j] : static_cast<double>(pp[head + j]); };
        uint32_t maxo = 0, mino = 0xffffffffu;
        uint64_t needs = 0;
        for (uint64_t j = lane; j < nb; j += 32) {
            const uint32_t pj = staged ? sPO[j].x : pp[head + j], oj = staged ? sPO[j].y : po[head + j];
            maxo = max(maxo, oj);
            mino = min(mino, oj);
            needs += serving_memory(m, static_cast<uint64_t>(pj) + oj, 1);
        }
        maxo = __reduce_max_sync(FULL, maxo);
        mino = __reduce_min_sync(FULL, mino);
        needs = warp_sum_u64(needs);
        // engine.hpp:321-325 (cost_model.hpp:18-25, batch 1, unrecorded): folded with
        // the decode steps below when one all-alive window covers the batch
        const bool fused_pre = staged && tab_ok && maxo <= 128 && mino >= 128;
        double dur = 0.0;
        if (!fused_pre) {
#pragma unroll 4
            for (uint64_t j = 0; j < nb; ++j) {
                const double t = member_pd(j);
                dur += m.prefill_coef_linear * t + m.prefill_coef_quad * t * t;
            }
        }
        double* dk = P.sat_dk + doff;
        double first[4] = {0.0, 0.0, 0.0, 0.0};  // steps 0..127 (lane = step mod 32)
        for (uint32_t k0 = 0; k0 < maxo; k0 += 128) {  // engine.hpp:358-365 per step
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            const uint32_t kb = k0 + lane;
            double kd[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) kd[r] = static_cast<double>(kb + 32 * r);
            if (staged && tab_ok && k0 + 128 <= mino) {  // every member alive at every step of the window
                // two steps from the table, two computed (the same f64 value: dtab[x] =
                // gamma + delta * (double)x and (double)p + (double)k == (double)(p + k)),
                // so L1 and the f64 pipe share the fold
                const double* __restrict__ dt = P.dtab[pi] + kb;
                if (fused_pre) {
#pragma unroll 4
                    for (uint64_t j = 0; j < nb; ++j) {
                        const uint32_t pj = sPO[j].x;
                        const double pdj = sPD[j];
                        dur += m.prefill_coef_linear * pdj + m.prefill_coef_quad * pdj * pdj;
                        acc[0] += dt[pj];
                        acc[1] += dt[pj + 32];
                        acc[2] += gam + del * (pdj + kd[2]);
                        acc[3] += gam + del * (pdj + kd[3]);
                    }
                } else {
#pragma unroll 4
                    for (uint64_t j = 0; j < nb; ++j) {
                        const uint32_t pj = sPO[j].x;
                        const double pdj = sPD[j];
                        acc[0] += dt[pj];
                        acc[1] += dt[pj + 32];
                        acc[2] += gam + del * (pdj + kd[2]);
                        acc[3] += gam + del * (pdj + kd[3]);
                    }
                }
            } else if (staged && tab_ok) {
                const double* __restrict__ dt = P.dtab[pi] + kb;
#pragma unroll 4
                for (uint64_t j = 0; j < nb; ++j) {
                    const uint2 po_j = sPO[j];
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (kb + 32 * r < po_j.y) acc[r] += dt[po_j.x + 32 * r];
                }
            } else {
#pragma unroll 4
                for (uint64_t j = 0; j < nb; ++j) {
                    const uint32_t oj = staged ? sPO[j].y : po[head + j];
                    const double pj = member_pd(j);
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (kb + 32 * r < oj) acc[r] += gam + del * (pj + kd[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (kb + 32 * r < maxo) dk[kb + 32 * r] = acc[r];
                if (k0 == 0) first[r] = acc[r];
            }
        }
        // Chain sums for the resolve pass: the batch's decode chain from now
        // (after its prefill) is now + u * R with R = sum_k RN_u(d_k) / u
        // while now stays in its binade e (u = 2^(e-52); see chain_fast_end).
        // now >= the batch's last arrival whenever the record is used, so
        // R is kept for the binades of that arrival and the three above;
        // ~0 = not usable (a tie, a step count above 128, or out of range).
        {
            const double alast = P.arr[lo + end - 1];
            const bool ok0 = maxo <= 128 && alast >= 0x1p-190 && alast <= 0x1p190;
            const int eb = ok0 ? binade_of(alast) : 0;
            uint64_t Rmine = ~0ull;
#pragma unroll
            for (int c = 0; c < kSatHdr; ++c) {
                const double sc = pow2i(52 - (eb + c));
                bool ok = ok0;
                uint64_t sum = 0;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    uint64_t rk = 0;
                    if (ok0 && static_cast<uint32_t>(32 * r) + lane < maxo) ok &= rn_units(first[r], sc, rk);
                    sum += rk;
                }
                const bool all = __all_sync(FULL, ok);
                const uint64_t R = warp_sum_small(sum);
                if (lane == static_cast<uint32_t>(c)) Rmine = all ? R : ~0ull;
            }
            SatRec& rr = P.sat_recs[ridx];
            if (lane < static_cast<uint32_t>(kSatHdr)) rr.R[lane] = Rmine;
            if (lane == 0) {
                rr.doff = doff;
                rr.start = static_cast<uint32_t>(head);
                rr.end = static_cast<uint32_t>(end);
                rr.K = maxo;
                rr.dev = d;
                rr.pre = dur;
                rr.alast = alast;
                rr.need = needs;
                P.sat_rec[lo + head] = static_cast<uint32_t>(ridx);
            }
        }
        ++ridx;
        doff += maxo;
        head = end;
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kWarps * 32) k_validate(const __grid_constant__ ReplayParams P) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const uint32_t pi = P.dev_prof[sg.dev];
    const colo_model& m = P.prof[pi].m;
    const uint64_t lo = P.dev_off[sg.dev];
    bool bad = false;
    unsigned long long mx = 0;
    for (uint64_t j = sg.start + lane; j < sg.end; j += 32) {
        const uint32_t pj = P.p[lo + j], oj = P.o[lo + j];
        if (pj == 0 || oj == 0) bad = true;  // workload.hpp:176-181
        else if (serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) > P.prof[pi].budget) bad = true;  // engine.hpp:70-74
        if (j > 0 && P.arr[lo + j] < P.arr[lo + j - 1]) bad = true;  // sorted by arrival (workload.hpp:165-169)
        mx = max(mx, static_cast<unsigned long long>(pj) + oj);
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(P.err, 1);
    mx = warp_max_u64(mx);
    if (lane == 0 && P.maxctx && mx) atomicMax(P.maxctx, mx);
}

// samples: device-local output-token prefix at each segment start
__global__ void __launch_bounds__(kWarps * 32) k_seg_sums(const __grid_constant__ ReplayParams P) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const uint64_t lo = P.dev_off[sg.dev];
    uint64_t s = 0;
    for (uint64_t j = sg.start + lane; j < sg.end; j += 32) s += P.o[lo + j];
    s = warp_sum_u64(s);
    if (lane == 0) P.seg_base[w] = s;
}

__global__ void k_seg_scan(const __grid_constant__ ReplayParams P) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= P.ndev) return;
    uint64_t run = 0;
    for (uint32_t k = P.dev_seg[d]; k < P.dev_seg[d + 1]; ++k) {
        const uint64_t s = P.seg_base[k];
        P.seg_base[k] = run;
        run += s;
    }
}

__global__ void __launch_bounds__(kWarps * 32, COLO_SPEC_BLOCKS) k_speculate(const __grid_constant__ ReplayParams P) {
    __shared__ uint2 spo[kWarps][kStage];
    __shared__ double spd[kWarps][kStage];
    __shared__ __align__(16) double sdk[kWarps][128];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    uint64_t head = sg.start;
    double T = -INFINITY;
    bool synced;
    Acc A;
    run_batches<RUN_SPEC>(P, sg.dev, head, T, sg.end, sg.start, &P.spec[w], synced, A, spo[warp], spd[warp], sdk[warp],
                          nullptr);
    if ((threadIdx.x & 31) == 0) {
        P.spec[w].exit_head = head;
        P.spec[w].exit_T = T;
    }
}

// One warp per CTA: resolve is a sequential chain per device, so each device
// gets an SM of its own (no issue-slot or FP64-pipe sharing between devices).
__global__ void __launch_bounds__(32) k_resolve(const __grid_constant__ ReplayParams P) {
    __shared__ uint2 spo[1][kStage];
    __shared__ double spd[1][kStage];
    __shared__ __align__(16) double sdk[1][128];
    const uint32_t warp = 0, lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x;
    if (d >= P.ndev) return;
    const uint64_t lo = P.dev_off[d];
    uint64_t head = 0;
    double T = -INFINITY;  // server idle before the first arrival (probe B4b)
    for (uint32_t k = P.dev_seg[d]; k < P.dev_seg[d + 1]; ++k) {
        const Seg sg = P.segs[k];
        if (lane == 0) P.entry[k] = Entry{head, T};
        Acc A;
        if (P.struct_out)  // [start, head): members of an earlier segment's batch
            for (uint64_t j = sg.start + lane; j < min(head, sg.end); j += 32) P.bmeta_bins[lo + j] = 0;
        if (head < sg.end) {  // (else an earlier batch already covers this segment)
            bool synced;
            run_batches<RUN_RESOLVE>(P, d, head, T, sg.end, sg.start, &P.spec[k], synced, A, spo[warp], spd[warp],
                                     sdk[warp], nullptr);
            if (synced) {
                if (P.struct_out) {  // from the sync point on, the speculative run's batches and counts
                    const SpecOut& so = P.spec[k];
                    const uint32_t rel = static_cast<uint32_t>(head - sg.start);
                    const uint32_t nreg = min(so.nregen, static_cast<uint32_t>(kRegen));
                    const uint32_t hit = __ballot_sync(FULL, lane < nreg && so.regen[lane] == rel);
                    const uint32_t j = __ffs(hit) - 1;  // synced: the head is regen point j
                    const bool suf = lane > j && lane <= static_cast<uint32_t>(kRegen);
                    A.nbatch += warp_sum_u64(suf ? so.ib[lane] : 0u);
                    A.max_need = max(A.max_need, warp_max_u64(suf ? so.ineed[lane] : 0ull));
                    A.maxb = max(A.maxb, warp_max_u64(suf ? so.imaxb[lane] : 0u));
                }
                head = P.spec[k].exit_head;
                T = P.spec[k].exit_T;
            }
        }
        if (P.struct_out && lane == 0) {
            Partial& q = P.part[k];
            q.nbatch = A.nbatch;
            q.max_need = A.max_need;
            q.maxb = A.maxb;
            q.t_end = T;
        }
    }
}

__global__ void __launch_bounds__(kWarps * 32, kReplayBlocks) k_replay_full(const __grid_constant__ ReplayParams P) {
    // one region per warp: the idle-start tile (32 rows of 33 step times), which
    // the per-batch path's member stage and step durations alias (never live
    // at the same time)
    extern __shared__ double stile[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* const wreg = stile + warp * (32 * 33);
    uint2* const spo_w = reinterpret_cast<uint2*>(wreg);
    double* const spd_w = wreg + kStage;
    double* const sdk_w = wreg + 2 * kStage;
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const Entry e = P.entry[w];
    uint64_t head = e.head;
    double T = e.T;
    Acc A;
    if (P.samples) {
        const uint64_t lo = P.dev_off[sg.dev];
        uint64_t s = 0;  // output tokens of the queries before the entry head inside this segment
        for (uint64_t j = sg.start + lane; j < min(head, sg.end); j += 32) s += P.o[lo + j];
        A.sample_pos = P.sample_off[sg.dev] + P.seg_base[w] + warp_sum_u64(s);
    }
    bool synced;
    if (head < sg.end)
        run_batches<RUN_FULL>(P, sg.dev, head, T, sg.end, sg.start, nullptr, synced, A, spo_w, spd_w, sdk_w, wreg);
    const uint64_t gen = warp_sum_u64(A.gen), slow_tok = warp_sum_u64(A.slow_tok), slow_q = warp_sum_u64(A.slow_q);
    const uint32_t fl = __reduce_or_sync(FULL, A.flags);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint64_t b0 = __shfl_xor_sync(FULL, A.acc[0], s);
        const uint64_t b1 = __shfl_xor_sync(FULL, A.acc[1], s);
        const uint64_t b2 = __shfl_xor_sync(FULL, A.acc[2], s);
        add3(A.acc, b0, b1, b2);
    }
    if (lane == 0) {
        Partial& q = P.part[w];
        q.gen = gen;
        q.slow_tok = slow_tok;
        q.slow_q = slow_q;
        q.nbatch = A.nbatch;
        q.max_need = A.max_need;
        q.maxb = A.maxb;
        q.acc[0] = A.acc[0];
        q.acc[1] = A.acc[1];
        q.acc[2] = A.acc[2];
        q.flags = fl;
        q.t_end = T;
    }
}

constexpr uint32_t kLaneMax = 4;     // members a lane replays by itself in k_batch_stats
constexpr uint32_t kHistWin = 1024;  // first-pass histogram bins per CTA in shared memory (from just below the step constant)
// k_batch_stats' per-warp region for run_batches on a queued batch (member
// stage, step durations, alive counts; never the idle-start tile: a queued
// batch starts at or after every member's arrival)
constexpr int kBsWarpBytes = (2 * kStage + 128) * 8 + 128 * 4;

// The decode steps of up to 32 batches at once, one per lane, from their
// recorded starts: a batch's timeline depends only on its members and its
// start (engine.hpp:319-387), so batches replay independently.  Per step the
// lane folds the alive members' durations in batch order, advances the
// absolute time (now + d, the reference's f64 add) and post-processes the
// sample: slow count and first slow step, the sample-bin range, histogram
// runs (a lane adds a run's weight when its key changes), the exact sum
// (telescoped when every step time lies in [now, 2 now], as the full pass).
// Batches of more than kLaneMax members go through run_batches one at a time.
// A histogram run of cnt samples into bin key: the CTA's shared-memory window
// (u32: the host enables it only when a CTA's samples stay below 2^31) or the
// global histogram.
__device__ __forceinline__ void hist_flush(const ReplayParams& P, uint32_t* shist, uint32_t key, uint64_t cnt) {
    const uint32_t r = key - P.hwin_base;
    if (r < P.hwin) atomicAdd(shist + r, static_cast<uint32_t>(cnt));
    else atomicAdd(reinterpret_cast<unsigned long long*>(P.hist + key), static_cast<unsigned long long>(cnt));
}

template <bool SINGLE, bool ONEF>
__device__ __noinline__ void lane_batch(const ReplayParams& P, const colo_model& m, uint64_t lo, uint64_t qb,
                                           uint32_t n, double start, bool idle, bool first_pass, Acc& A,
                                           uint64_t* bins_rw, uint32_t* shist) {
    // SINGLE: n == 1 (the loops over members and over the member ends drop
    // out); ONEF: one histogram filter (the first pass)
    constexpr uint32_t J = SINGLE ? 1u : kLaneMax;
    const double gam = m.decode_coef_const, del = m.decode_coef_context;
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;
    uint32_t oj[J];
    double pd[J];
    double dur = 0.0;
    uint32_t maxo = 0;
    uint64_t max_inc = 0;
#pragma unroll
    for (uint32_t j = 0; j < J; ++j) {
        const uint32_t pj = j < n ? pp[qb + j] : 0u;
        oj[j] = j < n ? po[qb + j] : 0u;
        pd[j] = static_cast<double>(pj);
        if (j < n) {
            dur += m.prefill_coef_linear * pd[j] + m.prefill_coef_quad * pd[j] * pd[j];  // engine.hpp:321-325
            maxo = max(maxo, oj[j]);
            max_inc = max(max_inc, static_cast<uint64_t>(pj) + oj[j]);
        }
    }
    double now = start + dur;
    const double span = static_cast<double>(maxo) *
                        (static_cast<double>(n) * (gam + del * static_cast<double>(max_inc + maxo))) * 1.001;
    const bool tele = now >= 0x1p-44 && span <= now && gam >= 0.0 && del >= 0.0;
    if (tele) acc_fixed_sub(A.acc, A.flags, now, n);
    const uint32_t nf = ONEF ? 1u : (P.hist ? P.nfilters : 0u);
    constexpr uint32_t F = ONEF ? 1u : 3u;
    uint32_t rkey[F];
    uint32_t rcnt[F];
#pragma unroll
    for (uint32_t f = 0; f < F; ++f) {
        rkey[f] = 0xffffffffu;
        rcnt[f] = 0;
    }
    uint32_t first_slow = 0xffffffffu, bmin = 0xffffffffu, bmax = 0, nslow = 0;
    uint64_t gen = 0;
    double kd = 0.0;
    for (uint32_t k = 0; k < maxo; ++k) {
        double d = 0.0;
        uint32_t alive = 0;
#pragma unroll
        for (uint32_t j = 0; j < J; ++j)
            if (SINGLE || (j < n && k < oj[j])) {
                d += gam + del * (pd[j] + kd);  // cost_model.hpp:28-35, batch 1, in batch order
                ++alive;
            }
        kd += 1.0;
        const double nn = now + d;
        const double s = nn - now;  // TPT sample of every alive member (engine.hpp:370-375)
        now = nn;
        gen += alive;
        const bool sl = s > P.tau;
        nslow += sl ? alive : 0u;
        first_slow = sl ? min(first_slow, k) : first_slow;
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
        if (!(s < 0.0)) {
            const uint32_t bn = static_cast<uint32_t>(bits >> 42);
            bmin = min(bmin, bn);
            bmax = max(bmax, bn);
        }
        if (nf) {
            const uint64_t hb = bits >> P.filter_shift;
            const uint32_t bin = static_cast<uint32_t>((bits >> P.hist_shift) & (COLO_HIST_BINS - 1));
#pragma unroll
            for (uint32_t f = 0; f < F; ++f) {
                const bool match = f < nf && hb == P.prefix[f];
                const uint32_t key = f * COLO_HIST_BINS + bin;
                const bool chg = match && key != rkey[f];
                if (chg && rcnt[f]) hist_flush(P, shist, rkey[f], rcnt[f]);
                rcnt[f] = chg ? alive : rcnt[f] + (match ? alive : 0u);
                rkey[f] = chg ? key : rkey[f];
            }
        }
        if (!tele) {
            acc_fixed(A.acc, A.flags, s, alive);
        } else if (!SINGLE) {
#pragma unroll
            for (uint32_t j = 0; j < J; ++j)
                if (j < n && k + 1 == oj[j]) acc_fixed(A.acc, A.flags, now, 1u);  // + T_{o_j - 1}
        }
    }
    if (SINGLE && tele) acc_fixed(A.acc, A.flags, now, 1u);  // + T_{o - 1}
    A.gen += gen;
    A.slow_tok += nslow;
#pragma unroll
    for (uint32_t f = 0; f < F; ++f)
        if (rcnt[f]) hist_flush(P, shist, rkey[f], rcnt[f]);
#pragma unroll
    for (uint32_t j = 0; j < J; ++j)
        if (j < n) {  // a query is slow iff one of its tokens is
            const bool slowq = oj[j] > first_slow;
            A.slow_q += slowq;
            if (P.labels) P.labels[lo + qb + j] = slowq ? 1 : 0;
        }
    if (first_pass)
        bins_rw[lo + qb] = (1ull << 63) | (idle ? 1ull << 62 : 0ull) | (static_cast<uint64_t>(bmax) << 21) | bmin;
}

// lane_batch for a single-member batch in the first stats pass (histogram
// key = the sample's top 21 bits = its bmeta bin) when the step constant is
// positive (validate_profile_pair), so every step duration is positive:
// 0.0 + x == x, every sample is >= 0 and matches the first pass's filter.
// Telescoping sums only; other batches take lane_batch.
__device__ __forceinline__ bool lane_single_p1(const ReplayParams& P, const colo_model& m, uint64_t lo, uint64_t qb,
                                               double start, bool idle, Acc& A, uint64_t* bins_rw, uint32_t* shist) {
    const double gam = m.decode_coef_const, del = m.decode_coef_context;
    const uint32_t pj = P.p[lo + qb], o = P.o[lo + qb];
    const double pd = static_cast<double>(pj);
    double now = start + (0.0 + (m.prefill_coef_linear * pd + m.prefill_coef_quad * pd * pd));  // engine.hpp:321-325
    const double span = static_cast<double>(o) * (gam + del * static_cast<double>(static_cast<uint64_t>(pj) + o + o)) * 1.001;
    if (!(now >= 0x1p-44 && span <= now)) return false;  // the sum would not telescope
    acc_fixed_sub(A.acc, A.flags, now, 1u);
    uint32_t first_slow = 0xffffffffu, bmin = 0xffffffffu, bmax = 0, nslow = 0, rkey = 0xffffffffu, rcnt = 0;
    // A finished run waits in (pkey, pcnt) and is flushed at the end of its
    // 4-step group: the lanes' runs end at different steps, so flushing at
    // the step would issue the (divergent) flush at almost every step
    uint32_t pkey = 0, pcnt = 0;
    double x = pd;  // pd + k, exact
    auto step = [&](uint32_t k) {
        const double d = gam + del * x;  // cost_model.hpp:28-35 (batch 1) = 0.0 + d
        x += 1.0;
        const double nn = now + d;
        const double s = nn - now;  // >= 0: TPT sample (engine.hpp:370-375)
        now = nn;
        const bool sl = s > P.tau;
        nslow += sl;
        first_slow = (sl && first_slow == 0xffffffffu) ? k : first_slow;
        const uint32_t bn = static_cast<uint32_t>(__double2hiint(s)) >> 10;  // bits >> 42
        bmin = min(bmin, bn);
        bmax = max(bmax, bn);
        const bool chg = bn != rkey;
        const bool ends = chg && rcnt != 0;
        if (ends && pcnt) hist_flush(P, shist, pkey, pcnt);  // a second run ends in the group (rare)
        pkey = ends ? rkey : pkey;
        pcnt = ends ? rcnt : pcnt;
        rkey = chg ? bn : rkey;
        rcnt = chg ? 1u : rcnt + 1;
    };
    uint32_t k = 0;
    for (; k + 4 <= o; k += 4) {
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i) step(k + i);
        if (pcnt) {
            hist_flush(P, shist, pkey, pcnt);
            pcnt = 0;
        }
    }
    for (; k < o; ++k) step(k);
    if (pcnt) hist_flush(P, shist, pkey, pcnt);
    if (rcnt) hist_flush(P, shist, rkey, rcnt);
    acc_fixed(A.acc, A.flags, now, 1u);  // + T_{o - 1}
    A.gen += o;
    A.slow_tok += nslow;
    const bool slowq = o > first_slow;
    A.slow_q += slowq;
    if (P.labels) P.labels[lo + qb] = slowq ? 1 : 0;
    bins_rw[lo + qb] = (1ull << 63) | (idle ? 1ull << 62 : 0ull) | (static_cast<uint64_t>(bmax) << 21) | bmin;
    return true;
}

// lane_batch for a single-member batch in a narrowing pass (only its
// samples whose high bits match a filter prefix feed the histogram; no other
// output), under the same positive-step-constant condition as lane_single_p1.
__device__ __forceinline__ void lane_single_narrow(const ReplayParams& P, const colo_model& m, uint64_t lo,
                                                   uint64_t qb, double start) {
    const double gam = m.decode_coef_const, del = m.decode_coef_context;
    const uint32_t pj = P.p[lo + qb], o = P.o[lo + qb];
    const double pd = static_cast<double>(pj);
    double now = start + (0.0 + (m.prefill_coef_linear * pd + m.prefill_coef_quad * pd * pd));  // engine.hpp:321-325
    const uint32_t nf = P.nfilters;
    const uint64_t pre0 = P.prefix[0], pre1 = nf > 1 ? P.prefix[1] : ~0ull, pre2 = nf > 2 ? P.prefix[2] : ~0ull;
    uint32_t rkey = 0xffffffffu, rcnt = 0;
    double x = pd;
#pragma unroll 2
    for (uint32_t k = 0; k < o; ++k) {
        const double d = gam + del * x;  // = 0.0 + d (d > 0)
        x += 1.0;
        const double nn = now + d;
        const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(nn - now));
        now = nn;
        const uint64_t top = bits >> P.filter_shift;
        if (top == pre0 || top == pre1 || top == pre2) {
            const uint32_t bin = static_cast<uint32_t>((bits >> P.hist_shift) & (COLO_HIST_BINS - 1));
#pragma unroll
            for (uint32_t f = 0; f < 3; ++f) {
                if (f < nf && top == P.prefix[f]) {
                    const uint32_t key = f * COLO_HIST_BINS + bin;
                    if (key != rkey) {
                        if (rcnt) atomicAdd(reinterpret_cast<unsigned long long*>(P.hist + rkey), static_cast<unsigned long long>(rcnt));
                        rkey = key;
                        rcnt = 0;
                    }
                    ++rcnt;
                }
            }
        }
    }
    if (rcnt) atomicAdd(reinterpret_cast<unsigned long long*>(P.hist + rkey), static_cast<unsigned long long>(rcnt));
}

// A batch of more than kLaneMax members: the warp replays it alone from its
// start with run_batches (out of line: rare, and it keeps k_batch_stats'
// register count to the lane path's)
__device__ __noinline__ void big_batch(const ReplayParams& P, uint32_t d, uint64_t head, double T, uint64_t seg_start,
                                       Acc& A, uint2* spo_w, double* spd_w, double* sdk_w, double* wreg) {
    if (!(P.arr[P.dev_off[d] + head] <= T)) {  // (cannot happen: the region has no idle-start tile)
        if ((threadIdx.x & 31) == 0) atomicOr(P.err, 2);
        return;
    }
    Acc B;
    bool synced;
    run_batches<RUN_FULL>(P, d, head, T, head + 1, seg_start, nullptr, synced, B, spo_w, spd_w, sdk_w, wreg);
    A.gen += B.gen;
    A.slow_tok += B.slow_tok;
    A.slow_q += B.slow_q;
    add3(A.acc, B.acc[0], B.acc[1], B.acc[2]);
    A.flags |= B.flags;
}

// Post-processing of the first stats pass over the batches the speculative
// and resolve passes recorded
// (first_pass: every batch; bmeta gets each batch's sample-bin range), or of
// a narrowing pass over the batches whose recorded range covers a filter bin.
// One warp per replay segment takes the batches that start in it, queues them
// in shared memory and replays them 32 at a time (lane_batch).
__device__ __forceinline__ void batch_stats_segment(const ReplayParams& P, uint32_t w, uint32_t warp, uint32_t lane,
                                                    double* wreg, uint32_t* shist) {
    // two queues per warp: single-member batches (the common case, replayed
    // by a loop without the member loops) and the rest
    __shared__ uint64_t qq[kWarps][2][64];
    __shared__ double qs[kWarps][2][64];
    __shared__ uint32_t qn[kWarps][2][64];
    uint2* const spo_w = reinterpret_cast<uint2*>(wreg);
    double* const spd_w = wreg + kStage;
    double* const sdk_w = wreg + 2 * kStage;
    const Seg sg = P.segs[w];
    const uint32_t d = sg.dev;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const colo_model& m = P.prof[P.dev_prof[d]].m;
    const bool first_pass = P.sparse_bins == nullptr;
    const bool onef = P.hist != nullptr && P.nfilters == 1;
    // the first pass's shape: one filter on the sign bit, bins = top 21 bits
    const bool p1 = first_pass && onef && P.filter_shift == 63 && P.prefix[0] == 0 && P.hist_shift == 42 &&
                    m.decode_coef_const > 0.0 && m.decode_coef_context >= 0.0;
    // a narrowing pass: only the histogram (no labels, counts or records)
    const bool pn = !first_pass && P.hist && !P.labels && m.decode_coef_const > 0.0 && m.decode_coef_context >= 0.0;
    const uint64_t* bins = first_pass ? P.bmeta_bins : P.sparse_bins;
    const double* starts = first_pass ? P.bmeta_start : P.sparse_start;
    uint64_t* const bins_rw = first_pass ? P.bmeta_bins : nullptr;
    const uint32_t sh = 42 - P.filter_shift;  // filter prefix -> its top-21-bit bin
    uint32_t fb[3];
#pragma unroll
    for (int f = 0; f < 3; ++f)
        fb[f] = f < static_cast<int>(P.nfilters) ? static_cast<uint32_t>(P.prefix[f] >> sh) : 0xffffffffu;
    Acc A;
    uint32_t nq[2] = {0, 0};
    auto process = [&](uint32_t qi, uint32_t cnt) {
        const bool has = lane < cnt;
        const uint64_t qb = has ? qq[warp][qi][lane] : 0ull;
        const uint32_t n = has ? qn[warp][qi][lane] & 0x7fffffffu : 0u;
        const bool idle = has && (qn[warp][qi][lane] >> 31);
        const double st = has ? qs[warp][qi][lane] : 0.0;
        if (qi == 0) {
            if (has) {
                if (pn) {
                    lane_single_narrow(P, m, lo, qb, st);
                } else if (p1 && lane_single_p1(P, m, lo, qb, st, idle, A, bins_rw, shist)) {
                } else if (onef) {  // (the general loop with n = 1: a smaller kernel than a third variant)
                    lane_batch<false, true>(P, m, lo, qb, 1u, st, idle, first_pass, A, bins_rw, shist);
                } else {
                    lane_batch<false, false>(P, m, lo, qb, 1u, st, idle, first_pass, A, bins_rw, shist);
                }
            }
        } else {
            if (has && n <= kLaneMax) {
                if (onef) lane_batch<false, true>(P, m, lo, qb, n, st, idle, first_pass, A, bins_rw, shist);
                else lane_batch<false, false>(P, m, lo, qb, n, st, idle, first_pass, A, bins_rw, shist);
            }
            uint32_t big = __ballot_sync(FULL, has && n > kLaneMax);
            while (big) {  // the warp together, one batch at a time (run_batches from its start)
                const uint32_t l = __ffs(big) - 1;
                big &= big - 1;
                const uint64_t head = __shfl_sync(FULL, qb, l);
                const bool idl = __shfl_sync(FULL, idle, l);
                const double T = idl ? -INFINITY : __shfl_sync(FULL, st, l);
                big_batch(P, d, head, T, sg.start, A, spo_w, spd_w, sdk_w, wreg);
            }
        }
        __syncwarp();
    };
    for (uint64_t j0 = sg.start; j0 < sg.end; j0 += 32) {
        const uint64_t q = j0 + lane;
        const uint64_t bb = q < N ? bins[lo + q] : 0ull;
        const bool stq = q >= N || (bb >> 63);  // a batch starts here (or the device ends)
        const uint32_t smask = __ballot_sync(FULL, stq);
        const bool mine = q < sg.end && q < N && (bb >> 63);
        const uint32_t above = lane == 31 ? 0u : smask & (~0u << (lane + 1));
        uint64_t far = 0;  // the first batch start past this chunk (for the batch that runs into it)
        if (__any_sync(FULL, mine && above == 0)) {
            for (uint64_t k0 = j0 + 32;; k0 += 32) {
                const uint64_t qk = k0 + lane;
                const uint32_t m2 = __ballot_sync(FULL, qk >= N || (bins[lo + qk] >> 63));
                if (m2) {
                    far = k0 + __ffs(m2) - 1;
                    break;
                }
            }
        }
        const uint64_t end = above ? j0 + __ffs(above) - 1 : far;
        bool sel = mine;
        if (!first_pass && sel) {  // narrowing pass: only batches whose sample-bin range covers a filter bin
            const uint32_t mn = static_cast<uint32_t>(bb & 0x1fffff), mx = static_cast<uint32_t>((bb >> 21) & 0x1fffff);
            bool hit = false;
#pragma unroll
            for (int f = 0; f < 3; ++f) hit |= mn <= fb[f] && fb[f] <= mx;
            sel = hit;
        }
#pragma unroll
        for (uint32_t qi = 0; qi < 2; ++qi) {
            const bool in = sel && ((end - q == 1) == (qi == 0));
            const uint32_t sm = __ballot_sync(FULL, in);
            if (in) {
                const uint32_t pos = nq[qi] + __popc(sm & ((1u << lane) - 1));
                qq[warp][qi][pos] = q;
                qn[warp][qi][pos] = static_cast<uint32_t>(end - q) | (((bb >> 62) & 1ull) ? 0x80000000u : 0u);
                qs[warp][qi][pos] = starts[lo + q];
            }
            nq[qi] += __popc(sm);
            __syncwarp();
            if (nq[qi] >= 32) {
                process(qi, 32);
                if (lane < nq[qi] - 32) {  // (reads [32, nq), writes [0, nq - 32): disjoint)
                    const uint64_t a = qq[warp][qi][32 + lane];
                    const uint32_t b = qn[warp][qi][32 + lane];
                    const double c = qs[warp][qi][32 + lane];
                    qq[warp][qi][lane] = a;
                    qn[warp][qi][lane] = b;
                    qs[warp][qi][lane] = c;
                }
                nq[qi] -= 32;
                __syncwarp();
            }
        }
    }
    if (nq[0]) process(0, nq[0]);
    if (nq[1]) process(1, nq[1]);
    if (first_pass) {
        const uint64_t gen = warp_sum_u64(A.gen), slow_tok = warp_sum_u64(A.slow_tok), slow_q = warp_sum_u64(A.slow_q);
        const uint32_t fl = __reduce_or_sync(FULL, A.flags);
#pragma unroll
        for (int s2 = 16; s2 > 0; s2 >>= 1) {
            const uint64_t b0 = __shfl_xor_sync(FULL, A.acc[0], s2);
            const uint64_t b1 = __shfl_xor_sync(FULL, A.acc[1], s2);
            const uint64_t b2 = __shfl_xor_sync(FULL, A.acc[2], s2);
            add3(A.acc, b0, b1, b2);
        }
        if (lane == 0) {
            Partial& q = P.part[w];
            q.gen = gen;
            q.slow_tok = slow_tok;
            q.slow_q = slow_q;
            q.acc[0] = A.acc[0];
            q.acc[1] = A.acc[1];
            q.acc[2] = A.acc[2];
            q.flags = fl;
        }
    }
}

__global__ void __launch_bounds__(kWarps * 32, 6) k_batch_stats(const __grid_constant__ ReplayParams P) {
    extern __shared__ double stile[];  // per warp the run_batches region, then the CTA's histogram window
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* const shist = reinterpret_cast<uint32_t*>(stile + kWarps * kBsWarpBytes / 8);
    for (uint32_t i = threadIdx.x; i < P.hwin; i += blockDim.x) shist[i] = 0;
    __syncthreads();
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w < P.nsegs) batch_stats_segment(P, w, warp, lane, stile + warp * (kBsWarpBytes / 8), shist);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P.hwin; i += blockDim.x)
        if (shist[i])
            atomicAdd(reinterpret_cast<unsigned long long*>(P.hist + P.hwin_base + i),
                      static_cast<unsigned long long>(shist[i]));
}

// Narrowing stats passes over the batches of the first pass whose sample-bin
// range covers a filter bin: each is replayed alone from its recorded start
// (an idle start forms the same one-query batch from T = -inf; a queued batch
// starts at the previous end, T = start).  One warp per replay segment.
__global__ void __launch_bounds__(kWarps * 32, kReplayBlocks) k_sparse_hist(const __grid_constant__ ReplayParams P) {
    extern __shared__ double stile[];  // as k_replay_full: the tile with the member stage aliased
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* const wreg = stile + warp * (32 * 33);
    uint2* const spo_w = reinterpret_cast<uint2*>(wreg);
    double* const spd_w = wreg + kStage;
    double* const sdk_w = wreg + 2 * kStage;
    const uint32_t w = blockIdx.x * kWarps + warp;
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const uint64_t lo = P.dev_off[sg.dev];
    const uint32_t sh = 42 - P.filter_shift;  // filter prefix -> its top-21-bit bin
    uint32_t fb[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) fb[f] = f < static_cast<int>(P.nfilters) ? static_cast<uint32_t>(P.prefix[f] >> sh) : 0xffffffffu;
    Acc A;
    for (uint64_t j0 = sg.start; j0 < sg.end; j0 += 32) {
        const uint64_t q = j0 + lane;
        const uint64_t bb = q < sg.end ? P.sparse_bins[lo + q] : 0ull;
        const uint32_t mn = static_cast<uint32_t>(bb & 0x1fffff), mx = static_cast<uint32_t>((bb >> 21) & 0x1fffff);
        bool hit = false;
#pragma unroll
        for (int f = 0; f < 3; ++f) hit |= mn <= fb[f] && fb[f] <= mx;
        uint32_t hits = __ballot_sync(FULL, (bb >> 63) && hit);
        while (hits) {
            const uint32_t l = __ffs(hits) - 1;
            hits &= hits - 1;
            const uint64_t b2 = __shfl_sync(FULL, bb, l);
            uint64_t head = j0 + l;
            double T = (b2 >> 62) & 1ull ? -INFINITY : P.sparse_start[lo + head];
            bool synced;
            run_batches<RUN_FULL>(P, sg.dev, head, T, j0 + l + 1, sg.start, nullptr, synced, A, spo_w, spd_w, sdk_w,
                                  wreg);
        }
    }
}

__global__ void __launch_bounds__(kWarps * 32) k_finalize(const __grid_constant__ ReplayParams P) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * kWarps + warp;
    if (d >= P.ndev) return;
    uint64_t gen = 0, slow_tok = 0, slow_q = 0, nbatch = 0, max_need = 0, maxb = 0, fl = 0;
    uint64_t acc[3] = {0, 0, 0};
    double t_end = 0.0;
    const uint64_t N = P.dev_off[d + 1] - P.dev_off[d];
    for (uint32_t k = P.dev_seg[d] + lane; k < P.dev_seg[d + 1]; k += 32) {
        const Partial& q = P.part[k];
        gen += q.gen;
        slow_tok += q.slow_tok;
        slow_q += q.slow_q;
        nbatch += q.nbatch;
        max_need = max(max_need, q.max_need);
        maxb = max(maxb, q.maxb);
        fl |= q.flags;
        add3(acc, q.acc[0], q.acc[1], q.acc[2]);
        t_end = fmax(t_end, q.t_end);
    }
    gen = warp_sum_u64(gen);
    slow_tok = warp_sum_u64(slow_tok);
    slow_q = warp_sum_u64(slow_q);
    nbatch = warp_sum_u64(nbatch);
    max_need = warp_max_u64(max_need);
    maxb = warp_max_u64(maxb);
    fl = warp_max_u64(fl);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint64_t b0 = __shfl_xor_sync(FULL, acc[0], s);
        const uint64_t b1 = __shfl_xor_sync(FULL, acc[1], s);
        const uint64_t b2 = __shfl_xor_sync(FULL, acc[2], s);
        add3(acc, b0, b1, b2);
        t_end = fmax(t_end, __shfl_xor_sync(FULL, t_end, s));
    }
    if (lane == 0) {
        colo_device_summary& S = P.summary[d];
        S.generated_tokens = gen;
        S.slow_tokens = slow_tok;
        S.slow_queries = slow_q;
        S.batches = nbatch;
        S.peak_device_bytes = P.prof[P.dev_prof[d]].fixed + max_need;  // memory.hpp:28-35 watermark
        S.max_batch_size = maxb;
        S.end_time = N ? t_end : 0.0;
        S.tpt_sum[0] = acc[0];
        S.tpt_sum[1] = acc[1];
        S.tpt_sum[2] = acc[2];
        S.flags = fl;
    }
}

// Dense batch list per device + the replay-derived verdicts (SURVEY §8(d) C3
// rule: cached = charged tokens of the last single-query batch before this
// one, incoming = max_incoming, batch = n, pending 0, dev_layers L,
// charged = charged(first query)).
__global__ void __launch_bounds__(kWarps * 32) k_batches(const __grid_constant__ ReplayParams P) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * kWarps + warp;
    if (d >= P.ndev) return;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const uint32_t pi = P.dev_prof[d];
    uint64_t pos = 0;
    uint64_t slot = 0;  // carry: charged tokens of the last single-query batch so far
    for (uint64_t j0 = 0; j0 < N; j0 += 32) {
        const uint64_t j = j0 + lane;
        const bool f = j < N && P.bflag[lo + j];
        const uint32_t bal = __ballot_sync(FULL, f);
        colo_batch b{};
        uint64_t ch = 0;
        bool single = false;
        if (f) {
            b = P.bstage[lo + j];
            if (P.has_sets) ch = charged_tokens(P.p[lo + j], P.o[lo + j], P.sets[pi].cpa);
            single = b.n == 1;
        }
        if (P.has_sets) {
            const uint32_t sm = __ballot_sync(FULL, single);
            const uint32_t below = sm & ((1u << lane) - 1u);
            const uint32_t src = below ? 31 - __clz(below) : 0;
            const uint64_t from = __shfl_sync(FULL, ch, src);
            const uint64_t my_slot = below ? from : slot;
            if (f) {
                const MapView& mv = P.sets[pi];
                b.verdict = compose(mv, mv.off, mv.hed, my_slot, b.max_incoming, b.n, 0, mv.L) | stream_bits(mv, mv.off, ch);
            }
            if (sm) slot = __shfl_sync(FULL, ch, 31 - __clz(sm));
        }
        if (f) P.batches[lo + pos + __popc(bal & ((1u << lane) - 1u))] = b;
        pos += __popc(bal);
    }
}

// The same verdicts from the compact 8 B stage (d_verdicts without batch
// records), segment-parallel.  The slot a batch sees is the charged tokens of
// the device's last single-query batch before it, and its output position is
// the number of batches before it: both are scans over the device's queries.
// k_vseg_count: per replay segment (one warp), its batch count and its last
// single-query batch's charged tokens (+1; 0 = none).  k_vseg_scan: per
// device (one warp), exclusive scans of both over its segments.
// k_vseg_emit: per segment, the verdicts from the scanned entry state.
struct VSeg {
    uint64_t count, last;
};

__device__ __forceinline__ uint64_t single_charged(const ReplayParams& P, uint64_t g, uint32_t pi) {
    return charged_tokens(P.p[g], P.o[g], P.sets[pi].cpa);
}

__global__ void __launch_bounds__(kWarps * 32) k_vseg_count(const __grid_constant__ ReplayParams P, VSeg* vs) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const uint64_t lo = P.dev_off[sg.dev];
    const uint32_t pi = P.dev_prof[sg.dev];
    uint64_t cnt = 0, last = 0;
    for (uint64_t j0 = sg.start; j0 < sg.end; j0 += 32) {
        const uint64_t j = j0 + lane;
        const uint64_t x = j < sg.end ? P.vstage[lo + j] : 0ull;
        const bool f = x != 0;
        cnt += __popc(__ballot_sync(FULL, f));
        const bool single = f && (x >> 32) == 1;
        const uint32_t sm = __ballot_sync(FULL, single);
        if (sm) {
            const uint32_t src = 31 - __clz(sm);
            const uint64_t ch = (lane == src) ? single_charged(P, lo + j, pi) : 0ull;
            last = __shfl_sync(FULL, ch, src) + 1;
        }
    }
    if (lane == 0) vs[w] = VSeg{cnt, last};
}

__global__ void __launch_bounds__(kWarps * 32) k_vseg_scan(const __grid_constant__ ReplayParams P, VSeg* vs) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (d >= P.ndev) return;
    uint64_t pos = 0, slot = 0;  // the device's slot starts empty (0 charged tokens)
    for (uint32_t s0 = P.dev_seg[d]; s0 < P.dev_seg[d + 1]; s0 += 32) {
        const uint32_t s = s0 + lane;
        const bool in = s < P.dev_seg[d + 1];
        const VSeg v = in ? vs[s] : VSeg{0, 0};
        uint64_t incl = v.count;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t m = __ballot_sync(FULL, v.last != 0);
        const uint32_t below = m & ((1u << lane) - 1u);
        const uint64_t from = __shfl_sync(FULL, v.last, below ? 31 - __clz(below) : 0);
        if (in) vs[s] = VSeg{pos + incl - v.count, below ? from - 1 : slot};
        pos += __shfl_sync(FULL, incl, 31);
        if (m) slot = __shfl_sync(FULL, v.last, 31 - __clz(m)) - 1;
    }
}

__global__ void __launch_bounds__(kWarps * 32) k_vseg_emit(const __grid_constant__ ReplayParams P, const VSeg* vs) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * kWarps + (threadIdx.x >> 5);
    if (w >= P.nsegs) return;
    const Seg sg = P.segs[w];
    const uint64_t lo = P.dev_off[sg.dev];
    const uint32_t pi = P.dev_prof[sg.dev];
    const MapView& mv = P.sets[pi];
    uint64_t pos = vs[w].count, slot = vs[w].last;
    for (uint64_t j0 = sg.start; j0 < sg.end; j0 += 32) {
        const uint64_t j = j0 + lane;
        const uint64_t x = j < sg.end ? P.vstage[lo + j] : 0ull;
        const bool f = x != 0;
        const uint32_t bal = __ballot_sync(FULL, f);
        if (!bal) continue;
        const uint32_t nb = static_cast<uint32_t>(x >> 32);
        const uint64_t ch = f ? charged_tokens(P.p[lo + j], P.o[lo + j], mv.cpa) : 0ull;
        const uint32_t sm = __ballot_sync(FULL, f && nb == 1);
        const uint32_t below = sm & ((1u << lane) - 1u);
        const uint64_t from = __shfl_sync(FULL, ch, below ? 31 - __clz(below) : 0);
        if (f) {
            const uint64_t my_slot = below ? from : slot;
            P.verdicts[lo + pos + __popc(bal & ((1u << lane) - 1u))] =
                compose(mv, mv.off, mv.hed, my_slot, static_cast<uint32_t>(x), nb, 0, mv.L) | stream_bits(mv, mv.off, ch);
        }
        if (sm) slot = __shfl_sync(FULL, ch, 31 - __clz(sm));
        pos += __popc(bal);
    }
}

// Grow-only context buffers (allocating tens of GB per call costs more than
// the passes themselves).
colo_status grow_buf(colo_ctx* ctx, void** buf, size_t* have, size_t bytes) {
    if (*have >= bytes) return COLO_OK;
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
    COLO_CK(ctx, cudaMalloc(buf, bytes));
    *have = bytes;
    return COLO_OK;
}

// Segments whose speculative run never went idle after its first batch: the
// queue stayed non-empty, which is where the all-queued fast path pays.
__global__ void k_count_saturated(const SpecOut* __restrict__ spec, uint32_t nsegs, unsigned long long* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool sat = i < nsegs && spec[i].nregen <= 1;
    const uint32_t b = __ballot_sync(0xffffffffu, sat);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, static_cast<unsigned long long>(__popc(b)));
}

struct SatBuffers {  // per-call scratch of sat_prepare
    void* tmp = nullptr;
    ~SatBuffers() {
        if (tmp) cudaFree(tmp);
    }
};

constexpr uint64_t kPSeg = 131072;  // queries per partition segment

colo_status sat_prepare(colo_ctx* ctx, ReplayParams& P, const std::vector<uint64_t>& off, SatBuffers& sb,
                        cudaStream_t st) {
    P.sat_on = 0;
    colo_ctx* sc = ctx->temps ? ctx->temps : ctx;  // owner of the per-call temporaries (colo_ctx_share_temps)
    const size_t ndev = P.ndev, n = off[ndev];
    const char* env = std::getenv("COLO_SAT");
    if ((env && env[0] == '0') || n >= (1ull << 32) || n == 0) return COLO_OK;
    std::vector<Seg> ps;
    for (size_t d = 0; d < ndev; ++d) {
        const uint64_t N = off[d + 1] - off[d];
        for (uint64_t s0 = 0; s0 < N; s0 += kPSeg) ps.push_back(Seg{static_cast<uint32_t>(d), 0, s0, std::min(N, s0 + kPSeg)});
    }
    const size_t ns = ps.size();
    // only when a noticeable share of segments stayed saturated (k_speculate ran first)
    {
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ctx->d_counters);
        COLO_CK(ctx, cudaMemsetAsync(cnt, 0, 8, st));
        COLO_LAUNCHED(ctx);
        k_count_saturated<<<(P.nsegs + 255) / 256, 256, 0, st>>>(P.spec, P.nsegs, cnt);
        unsigned long long nsat = 0;
        COLO_CK(ctx, cudaMemcpyAsync(&nsat, cnt, 8, cudaMemcpyDeviceToHost, st));
        COLO_CK(ctx, cudaStreamSynchronize(st));
        if (nsat * 50 < P.nsegs || nsat < 2) return COLO_OK;
    }
    const size_t need_rec = n * 8 + ns * 72 + 1024;
    if (sc->sat_bytes < need_rec) {
        size_t freeb = 0, totb = 0;
        COLO_CK(ctx, cudaMemGetInfo(&freeb, &totb));
        if (need_rec + (4ull << 30) > freeb + sc->sat_bytes) return COLO_OK;  // no room: replay every batch
    }
    {
        const colo_status g = grow_buf(ctx, &sc->d_sat, &sc->sat_bytes, need_rec);
        if (g != COLO_OK) return g;
    }
    auto* bp = static_cast<uint8_t*>(sc->d_sat);
    P.sat_end = reinterpret_cast<uint32_t*>(bp);
    P.sat_rec = reinterpret_cast<uint32_t*>(bp + n * 4);
    const size_t s8 = (ns * 8 + 127) & ~size_t(127);
    P.sat_seg = reinterpret_cast<uint64_t*>(bp + n * 8 + 128);
    P.sat_recbase = reinterpret_cast<uint64_t*>(bp + n * 8 + 128 + s8);
    Seg* dps = reinterpret_cast<Seg*>(bp + n * 8 + 128 + 2 * s8);
    P.sat_exit = reinterpret_cast<uint64_t*>(bp + n * 8 + 128 + 2 * s8 + ((ns * sizeof(Seg) + 127) & ~size_t(127)));
    P.sat_seg_start = P.sat_exit + ((ns + 15) & ~size_t(15));
    COLO_CK(ctx, cudaMemcpyAsync(dps, ps.data(), ns * sizeof(Seg), cudaMemcpyHostToDevice, st));
    P.psegs = dps;
    P.npsegs = static_cast<uint32_t>(ns);
    const bool timing = std::getenv("COLO_REPLAY_TIMING") != nullptr;
    cudaEvent_t ev[3];
    if (timing) {
        for (auto& e : ev) cudaEventCreate(&e);
        cudaEventRecord(ev[0], st);
    }
    COLO_CK(ctx, cudaMemsetAsync(P.sat_end, 0, n * 4, st));
    const uint32_t blocks = static_cast<uint32_t>((ns + kWarps - 1) / kWarps);
    P.sat_pass = 1;
    COLO_LAUNCHED(ctx);
    k_sat_partition<<<blocks, kWarps * 32, 0, st>>>(P);
    P.sat_pass = 2;
    COLO_LAUNCHED(ctx);
    k_sat_partition<<<blocks, kWarps * 32, 0, st>>>(P);
    // segment step counts -> exclusive bases (in place) and the pool size
    size_t tb = 0;
    COLO_CK(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tb, P.sat_seg, P.sat_seg, static_cast<int>(ns), st));
    {
        const colo_status gs = grow_buf(ctx, &sc->d_tmp, &sc->tmp_bytes, tb + 16);
        if (gs != COLO_OK) return gs;
    }
    // (the same scan for the record counts; both totals come back to size the pool)
    uint64_t last[4] = {0, 0, 0, 0};
    COLO_CK(ctx, cudaMemcpyAsync(&last[0], P.sat_seg + ns - 1, 8, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cudaMemcpyAsync(&last[2], P.sat_recbase + ns - 1, 8, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cub::DeviceScan::ExclusiveSum(sc->d_tmp, tb, P.sat_seg, P.sat_seg, static_cast<int>(ns), st));
    COLO_CK(ctx, cub::DeviceScan::ExclusiveSum(sc->d_tmp, tb, P.sat_recbase, P.sat_recbase, static_cast<int>(ns), st));
    COLO_CK(ctx, cudaMemcpyAsync(&last[1], P.sat_seg + ns - 1, 8, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cudaMemcpyAsync(&last[3], P.sat_recbase + ns - 1, 8, cudaMemcpyDeviceToHost, st));
    COLO_CK(ctx, cudaStreamSynchronize(st));
    const uint64_t np = last[1] + last[0], nr = last[3] + last[2];
    const size_t pool_bytes = ((np * 8 + 255) & ~size_t(255)) + nr * sizeof(SatRec) + 256;
    if (sc->satpool_bytes < pool_bytes) {
        size_t freeb = 0, totb = 0;
        COLO_CK(ctx, cudaMemGetInfo(&freeb, &totb));
        if (pool_bytes + (2ull << 30) > freeb + sc->satpool_bytes) return COLO_OK;  // no room for the step durations
    }
    if (timing) cudaEventRecord(ev[1], st);
    {
        const colo_status g = grow_buf(ctx, &sc->d_satpool, &sc->satpool_bytes, pool_bytes);
        if (g != COLO_OK) return g;
    }
    P.sat_dk = static_cast<double*>(sc->d_satpool);
    P.sat_recs = reinterpret_cast<SatRec*>(static_cast<uint8_t*>(sc->d_satpool) + ((np * 8 + 255) & ~size_t(255)));
    P.sat_nrec = nr;
    COLO_LAUNCHED(ctx);
    k_sat_durations<<<blocks, kWarps * 32, 0, st>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    P.sat_on = 1;
    if (timing) {
        cudaEventRecord(ev[2], st);
        cudaEventSynchronize(ev[2]);
        float a, b;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        std::fprintf(stderr, "colo sat: %llu step durations; records %.3f ms, durations %.3f ms\n",
                     static_cast<unsigned long long>(np), a, b);
        for (auto& x : ev) cudaEventDestroy(x);
    }
    return COLO_OK;
}

colo_status grow_rscratch(colo_ctx* ctx, size_t bytes) {
    if (ctx->rscratch_bytes >= bytes) return COLO_OK;
    if (ctx->d_rscratch) cudaFree(ctx->d_rscratch);
    ctx->d_rscratch = nullptr;
    ctx->rscratch_bytes = 0;
    COLO_CK(ctx, cudaMalloc(&ctx->d_rscratch, bytes));
    ctx->rscratch_bytes = bytes;
    return COLO_OK;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Cross-rank totals of the first stats pass (colo_serving_stats_nccl): sums
// of the counters and of the exact 192-bit TPT sum, the latter as six 32-bit
// chunks so no carry is lost in the u64 reduction; max of the peaks; the
// flag words OR-ed (NCCL has no bitwise reduction: each of the 8 flag bits is
// summed as a count, and a bit is set when any rank had it).
constexpr int kFlagBits = 8;
colo_status dist_totals(colo_ctx* ctx, void* comm, colo_device_summary* t) {
    constexpr int NS = 10 + kFlagBits;
    uint64_t hs[NS] = {t->generated_tokens, t->slow_tokens, t->slow_queries, t->batches};
    for (int i = 0; i < 6; ++i) hs[4 + i] = (t->tpt_sum[i / 2] >> (32 * (i & 1))) & 0xffffffffull;
    for (int b = 0; b < kFlagBits; ++b) hs[10 + b] = (t->flags >> b) & 1ull;
    uint64_t hm[2] = {t->peak_device_bytes, t->max_batch_size};
    double he = t->end_time;
    uint64_t* d = nullptr;
    COLO_CK(ctx, cudaMalloc(&d, (NS + 3) * 8));
    colo_status st = COLO_OK;
    do {
        if (cudaMemcpy(d, hs, NS * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(d + NS, hm, 2 * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(d + NS + 2, &he, 8, cudaMemcpyHostToDevice) != cudaSuccess) {
            st = set_err(ctx, COLO_ECUDA, "dist_totals staging");
            break;
        }
        if ((st = colo_stats_allreduce(ctx, comm, d, NS)) != COLO_OK) break;
        if ((st = nccl_allreduce_raw(ctx, comm, d + NS, 2, /*ncclUint64*/ 5, /*ncclMax*/ 2)) != COLO_OK) break;
        if ((st = nccl_allreduce_raw(ctx, comm, d + NS + 2, 1, /*ncclFloat64*/ 8, /*ncclMax*/ 2)) != COLO_OK) break;
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess || cudaMemcpy(hs, d, NS * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(hm, d + NS, 2 * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(&he, d + NS + 2, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
            st = set_err(ctx, COLO_ECUDA, "dist_totals readback");
            break;
        }
        t->generated_tokens = hs[0];
        t->slow_tokens = hs[1];
        t->slow_queries = hs[2];
        t->batches = hs[3];
        uint64_t acc[3] = {0, 0, 0};
        for (int i = 0; i < 6; ++i) {  // chunk i weighs 2^(32 i); each chunk sum < 2^64
            const uint64_t v = hs[4 + i];
            uint64_t add[3] = {0, 0, 0};
            const int limb = i / 2, sh = 32 * (i & 1);
            add[limb] = v << sh;
            if (sh && limb + 1 < 3) add[limb + 1] = v >> (64 - sh);
            fixed_add(acc, add);
        }
        t->tpt_sum[0] = acc[0];
        t->tpt_sum[1] = acc[1];
        t->tpt_sum[2] = acc[2];
        t->peak_device_bytes = hm[0];
        t->max_batch_size = hm[1];
        uint64_t fl = t->flags & ~((1ull << kFlagBits) - 1);
        for (int b = 0; b < kFlagBits; ++b)
            if (hs[10 + b]) fl |= 1ull << b;
        t->flags = fl;
        t->end_time = he;
    } while (false);
    cudaFree(d);
    return st;
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
    {
        const char* e = std::getenv("COLO_SINGLES");
        P.singles = (e && e[0] == '0') ? 0u : 1u;
    }
    for (size_t i = 0; i < nprofiles; ++i) {
        const colo_status st = colo_validate_profile_pair(&models[i], &gpus[i]);
        if (st != COLO_OK) return set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
        P.prof[i].m = models[i];
        P.prof[i].budget = gpus[i].capacity_bytes - gpus[i].runtime_reserve_bytes - models[i].weights_bytes;
        P.prof[i].fixed = models[i].weights_bytes + gpus[i].runtime_reserve_bytes;
        if (opts->sets) {
            if (!opts->sets[i]) return set_err(ctx, COLO_EINVAL, "null map set");
            P.sets[i] = make_view(opts->sets[i]);
        }
    }
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    // segments (host): device offsets come back once per call
    std::vector<uint64_t> off(ndev + 1);
    std::vector<uint16_t> prof(ndev);
    COLO_CK(ctx, cudaMemcpyAsync(off.data(), d_dev_offsets, (ndev + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaMemcpyAsync(prof.data(), d_dev_profile, ndev * 2, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (off[0] != 0 || off[ndev] != n) return set_err(ctx, COLO_EINVAL, "device offsets must span [0, n]");
    for (size_t d = 0; d < ndev; ++d) {
        if (off[d + 1] < off[d]) return set_err(ctx, COLO_EINVAL, "device offsets not monotone");
        if (prof[d] >= nprofiles) return set_err(ctx, COLO_EINVAL, "device profile index out of range");
    }
    uint64_t seg = opts->segment_len;
    if (seg == 0) {  // enough segments to fill the GPU several times over, 256..16384 queries each
        const uint64_t target = static_cast<uint64_t>(ctx->sm_count) * 64;
        seg = std::min<uint64_t>(16384, std::max<uint64_t>(256, n / std::max<uint64_t>(target, 1)));
    }
    std::vector<Seg> segs;
    std::vector<uint32_t> dev_seg(ndev + 1);
    for (size_t d = 0; d < ndev; ++d) {
        dev_seg[d] = static_cast<uint32_t>(segs.size());
        const uint64_t N = off[d + 1] - off[d];
        for (uint64_t s = 0; s < N; s += seg) segs.push_back(Seg{static_cast<uint32_t>(d), 0, s, std::min(N, s + seg)});
    }
    dev_seg[ndev] = static_cast<uint32_t>(segs.size());
    const size_t ns = segs.size();
    const bool want_batches = opts->d_batches != nullptr;
    size_t bytes = 0;
    const size_t o_segs = bytes;
    bytes += align256(ns * sizeof(Seg) + 8);
    const size_t o_dseg = bytes;
    bytes += align256((ndev + 1) * 4);
    const size_t o_spec = bytes;
    bytes += align256(ns * sizeof(SpecOut) + 8);
    const size_t o_entry = bytes;
    bytes += align256(ns * sizeof(Entry) + 8);
    const size_t o_part = bytes;
    bytes += align256(ns * sizeof(Partial) + 8);
    const size_t o_base = bytes;
    bytes += align256(ns * 8 + 8);
    const size_t o_bstage = bytes;
    bytes += want_batches ? align256(n * sizeof(colo_batch) + 8) : 0;
    const size_t o_bflag = bytes;
    bytes += want_batches ? align256(n + 8) : 0;
    const bool want_verdicts = opts->d_verdicts != nullptr;
    if (want_verdicts && !opts->sets) return set_err(ctx, COLO_EINVAL, "d_verdicts needs map sets");
    const size_t o_vstage = bytes;
    bytes += want_verdicts ? align256(n * 8 + 8) : 0;
    const size_t o_vseg = bytes;
    bytes += want_verdicts ? align256(ns * sizeof(VSeg) + 8) : 0;
    uint64_t prof_hash = 14695981039346656037ull;  // FNV-1a over the profile structs' bytes
    for (size_t i = 0; i < nprofiles; ++i) {
        const auto* mb = reinterpret_cast<const uint8_t*>(&models[i]);
        const auto* gb = reinterpret_cast<const uint8_t*>(&gpus[i]);
        for (size_t b = 0; b < sizeof(colo_model); ++b) prof_hash = (prof_hash ^ mb[b]) * 1099511628211ull;
        for (size_t b = 0; b < sizeof(colo_gpu); ++b) prof_hash = (prof_hash ^ gb[b]) * 1099511628211ull;
    }
    const uint64_t sig[11] = {n, ndev, seg, nprofiles, reinterpret_cast<uintptr_t>(d_arrival),
                              reinterpret_cast<uintptr_t>(d_prompt), reinterpret_cast<uintptr_t>(d_output),
                              reinterpret_cast<uintptr_t>(d_dev_offsets), reinterpret_cast<uintptr_t>(d_dev_profile),
                              ns, prof_hash};
    const bool reuse = opts->reuse_entries && ctx->rs_valid && ctx->rscratch_bytes >= bytes &&
                       std::memcmp(sig, ctx->rs_sig, sizeof sig) == 0;
    if (!reuse) ctx->rs_valid = false;
    colo_status st = grow_rscratch(ctx, bytes);
    if (st != COLO_OK) return st;
    auto* base = static_cast<uint8_t*>(ctx->d_rscratch);
    P.segs = reinterpret_cast<const Seg*>(base + o_segs);
    P.dev_seg = reinterpret_cast<const uint32_t*>(base + o_dseg);
    P.spec = reinterpret_cast<SpecOut*>(base + o_spec);
    P.entry = reinterpret_cast<Entry*>(base + o_entry);
    P.part = reinterpret_cast<Partial*>(base + o_part);
    P.seg_base = reinterpret_cast<uint64_t*>(base + o_base);
    if (!reuse) {  // (a reuse pass has exactly these segments in place)
        if (ns)
            COLO_CK(ctx, cudaMemcpyAsync(base + o_segs, segs.data(), ns * sizeof(Seg), cudaMemcpyHostToDevice, ctx->stream));
        COLO_CK(ctx, cudaMemcpyAsync(base + o_dseg, dev_seg.data(), (ndev + 1) * 4, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (want_batches) {
        P.bstage = reinterpret_cast<colo_batch*>(base + o_bstage);
        P.bflag = base + o_bflag;
        COLO_CK(ctx, cudaMemsetAsync(P.bflag, 0, n + 8, ctx->stream));
    }
    if (want_verdicts) {
        P.vstage = reinterpret_cast<uint64_t*>(base + o_vstage);
        P.verdicts = opts->d_verdicts;
        COLO_CK(ctx, cudaMemsetAsync(P.vstage, 0, n * 8 + 8, ctx->stream));
    }
    P.nprof = static_cast<uint32_t>(nprofiles);
    P.has_sets = opts->sets ? 1u : 0u;
    P.arr = d_arrival;
    P.p = d_prompt;
    P.o = d_output;
    P.dev_off = d_dev_offsets;
    P.dev_prof = d_dev_profile;
    P.ndev = static_cast<uint32_t>(ndev);
    P.nsegs = static_cast<uint32_t>(ns);
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
    if (opts->stats_mode == 1 && n) {  // first stats pass: record every batch's start and sample-bin range
        ctx->bmeta_valid = false;
        size_t freeb = 0, totb = 0;
        bool room = ctx->bmeta_bytes >= n * 16;
        if (!room && cudaMemGetInfo(&freeb, &totb) == cudaSuccess)
            room = n * 16 + (8ull << 30) < freeb + ctx->bmeta_bytes;
        if (room && grow_buf(ctx, &ctx->d_bmeta, &ctx->bmeta_bytes, n * 16) == COLO_OK) {
            P.bmeta_start = static_cast<double*>(ctx->d_bmeta);
            P.bmeta_bins = reinterpret_cast<uint64_t*>(static_cast<double*>(ctx->d_bmeta) + n);
            COLO_CK(ctx, cudaMemsetAsync(P.bmeta_bins, 0, n * 8, ctx->stream));
        }
    }
    COLO_CK(ctx, cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
    P.maxctx = reinterpret_cast<unsigned long long*>(ctx->d_counters) + 2;
    COLO_CK(ctx, cudaMemsetAsync(P.maxctx, 0, 8, ctx->stream));
    const uint32_t seg_blocks = static_cast<uint32_t>((ns + kWarps - 1) / kWarps);
    COLO_CK(ctx, cudaFuncSetAttribute(k_replay_full, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
    const uint32_t dev_blocks = static_cast<uint32_t>((ndev + kWarps - 1) / kWarps);
    if (ns && reuse) {  // histogram passes 2-3: the entry states of the previous full replay
        if (P.samples) {
            COLO_LAUNCHED(ctx);
            k_seg_sums<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P);
            COLO_LAUNCHED(ctx);
            k_seg_scan<<<static_cast<uint32_t>((ndev + 127) / 128), 128, 0, ctx->stream>>>(P);
        }
        if (opts->stats_mode == 2 && ctx->bmeta_valid && P.hist && !P.vstage && !P.bstage) {  // narrowing pass: only batches that can hit a filter bin
            P.sparse_start = static_cast<const double*>(ctx->d_bmeta);
            P.sparse_bins = reinterpret_cast<const uint64_t*>(static_cast<const double*>(ctx->d_bmeta) + n);
            const char* bse = std::getenv("COLO_BATCH_STATS");
            if (!(bse && bse[0] == '0')) {
                COLO_CK(ctx, cudaFuncSetAttribute(k_batch_stats, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  kWarps * kBsWarpBytes));
                COLO_LAUNCHED(ctx);
                k_batch_stats<<<seg_blocks, kWarps * 32, kWarps * kBsWarpBytes, ctx->stream>>>(P);
            } else {
                COLO_CK(ctx, cudaFuncSetAttribute(k_sparse_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileBytes));
                COLO_LAUNCHED(ctx);
                k_sparse_hist<<<seg_blocks, kWarps * 32, kTileBytes, ctx->stream>>>(P);
            }
        } else {
            COLO_LAUNCHED(ctx);
            k_replay_full<<<seg_blocks, kWarps * 32, kTileBytes, ctx->stream>>>(P);
        }
    } else if (ns) {
        COLO_LAUNCHED(ctx);
        k_validate<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P);
        int flag = 0;
        COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
        if (flag)
            return set_err(ctx, COLO_EVALIDATION,
                           "trace rejected: unsorted arrivals, zero tokens, or a query that cannot fit the device alone");
        unsigned long long mctx_seen = 0;  // max p + o over the trace (k_validate)
        {  // decode-latency tables up to the trace's largest context
            unsigned long long mctx = 0;
            COLO_CK(ctx, cudaMemcpy(&mctx, P.maxctx, 8, cudaMemcpyDeviceToHost));
            mctx_seen = mctx;
            P.dtab_n = 0;
            if (mctx > 0 && mctx < (1ull << 20)) {
                const uint64_t tn = mctx + 1;
                const size_t tb = ((tn * 8 + 255) & ~size_t(255)) * nprofiles;
                if (ctx->dtab_bytes < tb) {
                    if (ctx->d_dtab) cudaFree(ctx->d_dtab);
                    ctx->d_dtab = nullptr;
                    ctx->dtab_bytes = 0;
                    COLO_CK(ctx, cudaMalloc(&ctx->d_dtab, tb));
                    ctx->dtab_bytes = tb;
                }
                for (size_t i = 0; i < nprofiles; ++i) {
                    double* t = reinterpret_cast<double*>(static_cast<uint8_t*>(ctx->d_dtab) +
                                                          i * ((tn * 8 + 255) & ~size_t(255)));
                    COLO_LAUNCHED(ctx);
                    k_fill_dtab<<<256, 256, 0, ctx->stream>>>(t, tn, models[i].decode_coef_const,
                                                              models[i].decode_coef_context);
                    P.dtab[i] = t;
                }
                P.dtab_n = tn;
            }
        }
        if (P.samples) {
            COLO_LAUNCHED(ctx);
            k_seg_sums<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P);
            COLO_LAUNCHED(ctx);
            k_seg_scan<<<static_cast<uint32_t>((ndev + 127) / 128), 128, 0, ctx->stream>>>(P);
        }
        const bool timing = std::getenv("COLO_REPLAY_TIMING") != nullptr;  // per-pass device times to stderr
        cudaEvent_t ev[4];
        if (timing)
            for (auto& e : ev) cudaEventCreate(&e);
        const char* bse = std::getenv("COLO_BATCH_STATS");
        // first stats pass: the speculative and resolve passes also lay down the
        // batch structure, and k_batch_stats replays every batch's decode steps
        // from its start, many batches at once (no full replay pass)
        const bool bstats = opts->stats_mode == 1 && P.bmeta_bins && !P.samples && !P.bstage && !P.vstage &&
                            !(bse && bse[0] == '0');
        P.struct_out = bstats ? 1u : 0u;
        if (timing) cudaEventRecord(ev[0], ctx->stream);
        COLO_LAUNCHED(ctx);
        k_speculate<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P);
        SatBuffers sat;  // all-queued batch records for the resolve pass's fast path
        const colo_status sst = sat_prepare(ctx, P, off, sat, ctx->stream);
        if (sst != COLO_OK) return sst;
        if (timing) cudaEventRecord(ev[1], ctx->stream);
        if (timing) {
            P.dbg = reinterpret_cast<unsigned long long*>(ctx->d_counters);
            cudaMemsetAsync(ctx->d_counters, 0, 64, ctx->stream);
        }
        COLO_LAUNCHED(ctx);
        k_resolve<<<static_cast<uint32_t>(ndev), 32, 0, ctx->stream>>>(P);
        if (timing) cudaEventRecord(ev[2], ctx->stream);
        if (bstats) {
            P.dbg = nullptr;
            cudaEvent_t es = nullptr;
            if (timing) {
                cudaEventCreate(&es);
                cudaEventRecord(es, ctx->stream);
            }
            // the first pass's histogram (bins = top 21 bits) gets a per-CTA window
            // in shared memory from half the smallest decode-step constant up 4
            // binades (TPT samples are at least about one step).  Its u32 counts
            // cannot wrap: a CTA replays the batches that start in its kWarps
            // segments, whose members are those queries plus at most one batch
            // past the last segment (at most budget / kv_bytes_per_token
            // members: every query needs more than one token's KV), each with
            // fewer than max(p + o) samples.
            uint64_t bmax = 0;
            for (size_t i = 0; i < nprofiles; ++i)
                bmax = std::max<uint64_t>(bmax, (gpus[i].capacity_bytes - gpus[i].runtime_reserve_bytes -
                                                 models[i].weights_bytes) / models[i].kv_bytes_per_token);
            const double per_cta = (static_cast<double>(kWarps) * static_cast<double>(seg) + static_cast<double>(bmax)) *
                                   static_cast<double>(mctx_seen);
            P.hwin = 0;
            if (P.hist && P.nfilters == 1 && P.filter_shift == 63 && P.prefix[0] == 0 && P.hist_shift == 42 &&
                mctx_seen > 0 && per_cta < 2147483648.0) {
                double g = models[0].decode_coef_const;
                for (size_t i = 1; i < nprofiles; ++i) g = std::min(g, models[i].decode_coef_const);
                const double lo_s = g * (1.0 - 0x1p-20);  // every single-query sample is >= g within rounding
                uint64_t b = 0;
                std::memcpy(&b, &lo_s, 8);
                if (lo_s > 0.0 && std::isfinite(lo_s)) {
                    P.hwin_base = static_cast<uint32_t>(b >> 42);
                    P.hwin = kHistWin;
                }
            }
            const size_t bs_smem = kWarps * kBsWarpBytes + P.hwin * 4u;
            COLO_CK(ctx, cudaFuncSetAttribute(k_batch_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bs_smem));
            COLO_LAUNCHED(ctx);
            k_batch_stats<<<seg_blocks, kWarps * 32, bs_smem, ctx->stream>>>(P);
            P.hwin = 0;
            if (timing) {
                cudaEvent_t ee;
                cudaEventCreate(&ee);
                cudaEventRecord(ee, ctx->stream);
                cudaEventSynchronize(ee);
                float x = 0, y = 0;
                cudaEventElapsedTime(&x, ev[2], es);
                cudaEventElapsedTime(&y, es, ee);
                std::fprintf(stderr, "colo replay: (setup %.3f ms) batch stats %.3f ms\n", x, y);
                cudaEventDestroy(es);
                cudaEventDestroy(ee);
            }
        } else {
            COLO_LAUNCHED(ctx);
            k_replay_full<<<seg_blocks, kWarps * 32, kTileBytes, ctx->stream>>>(P);
        }
        P.dbg = nullptr;
        if (timing) {
            cudaEventRecord(ev[3], ctx->stream);
            cudaEventSynchronize(ev[3]);
            float a, b, c;
            cudaEventElapsedTime(&a, ev[0], ev[1]);
            cudaEventElapsedTime(&b, ev[1], ev[2]);
            cudaEventElapsedTime(&c, ev[2], ev[3]);
            unsigned long long hits[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            cudaMemcpy(hits, ctx->d_counters, 64, cudaMemcpyDeviceToHost);
            std::fprintf(stderr, "colo replay full pass: %llu idle-start queries in %llu windows, %llu other batches "
                                 "(%llu queries)\n", hits[4], hits[5], hits[6], hits[7]);
            std::fprintf(stderr, "colo replay: %zu segments (len %llu), speculate %.3f ms, resolve %.3f ms (%llu fast "
                                 "[%llu by chain sums, %llu record windows] / %llu formed batches), replay %.3f ms\n",
                         ns, static_cast<unsigned long long>(seg), a, b, hits[0], hits[2], hits[3], hits[1], c);
            for (auto& e : ev) cudaEventDestroy(e);
        }
    }
    if (P.summary) {
        COLO_LAUNCHED(ctx);
        k_finalize<<<dev_blocks, kWarps * 32, 0, ctx->stream>>>(P);
    }
    if (want_batches && ns) {
        COLO_LAUNCHED(ctx);
        k_batches<<<dev_blocks, kWarps * 32, 0, ctx->stream>>>(P);
    }
    if (want_verdicts && ns) {
        VSeg* vs = reinterpret_cast<VSeg*>(base + o_vseg);
        COLO_LAUNCHED(ctx);
        k_vseg_count<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P, vs);
        COLO_LAUNCHED(ctx);
        k_vseg_scan<<<dev_blocks, kWarps * 32, 0, ctx->stream>>>(P, vs);
        COLO_LAUNCHED(ctx);
        k_vseg_emit<<<seg_blocks, kWarps * 32, 0, ctx->stream>>>(P, vs);
    }
    COLO_CK(ctx, cudaGetLastError());
    int late = 0;
    COLO_CK(ctx, cudaMemcpyAsync(&late, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (late) return set_err(ctx, COLO_EBREACH, "replay: internal consistency check failed");
    std::memcpy(ctx->rs_sig, sig, sizeof sig);
    ctx->rs_valid = true;
    if (!reuse) ctx->bmeta_valid = P.bmeta_bins != nullptr;  // records of exactly this replay
    return COLO_OK;
}

static colo_status serving_stats_impl(colo_ctx* ctx, void* comm, const colo_model* models, const colo_gpu* gpus,
                                      size_t nprofiles, const double* d_arrival, const uint32_t* d_prompt,
                                      const uint32_t* d_output, size_t n, const uint64_t* d_dev_offsets,
                                      const uint16_t* d_dev_profile, size_t ndev, double tau, double* pctl,
                                      colo_device_summary* totals) {
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
    for (int i = 0; i < 4; ++i) pctl[i] = std::nan("");
    const char* sparse_env = std::getenv("COLO_SPARSE_STATS");
    const bool sparse = !(sparse_env && sparse_env[0] == '0');
    for (int pass = 0; pass < 3 && st == COLO_OK; ++pass) {
        colo_replay_opts o{};
        o.stats_mode = sparse ? (pass == 0 ? 1u : 2u) : 0u;
        o.tau = tau;
        o.d_hist = d_hist;
        o.d_summary = pass == 0 ? d_sum : nullptr;
        o.reuse_entries = pass > 0 ? 1u : 0u;
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
        const bool timing = std::getenv("COLO_REPLAY_TIMING") != nullptr;
        cudaEvent_t pe[2];
        if (timing) {
            cudaEventCreate(&pe[0]);
            cudaEventCreate(&pe[1]);
            cudaEventRecord(pe[0], ctx->stream);
        }
        st = colo_replay_serving(ctx, models, gpus, nprofiles, d_arrival, d_prompt, d_output, n, d_dev_offsets,
                                 d_dev_profile, ndev, &o);
        if (timing) {
            cudaEventRecord(pe[1], ctx->stream);
            cudaEventSynchronize(pe[1]);
            float ms = 0;
            cudaEventElapsedTime(&ms, pe[0], pe[1]);
            std::fprintf(stderr, "colo stats pass %d (mode %u): %.3f ms\n", pass, o.stats_mode, ms);
            cudaEventDestroy(pe[0]);
            cudaEventDestroy(pe[1]);
        }
        if (st != COLO_OK) break;
        if (comm) {  // every rank holds its own device shard: sum the histograms
            st = colo_stats_allreduce(ctx, comm, d_hist, static_cast<size_t>(o.nfilters) * COLO_HIST_BINS);
            if (st != COLO_OK) break;
        }
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
            if (comm) {  // counters and the exact sum (as 32-bit chunks) summed; peaks and end time maxed
                st = dist_totals(ctx, comm, totals);
                if (st != COLO_OK) break;
            }
            ntot = totals->generated_tokens;
            if (ntot == 0) break;
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
                const uint64_t bits = (b1[f] << 42) | (b2[f] << 21) | bin;
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


colo_status colo_serving_stats(colo_ctx* ctx, const colo_model* models, const colo_gpu* gpus, size_t nprofiles,
                               const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                               const uint64_t* d_dev_offsets, const uint16_t* d_dev_profile, size_t ndev, double tau,
                               double* pctl, colo_device_summary* totals) {
    return serving_stats_impl(ctx, nullptr, models, gpus, nprofiles, d_arrival, d_prompt, d_output, n, d_dev_offsets,
                              d_dev_profile, ndev, tau, pctl, totals);
}

colo_status colo_serving_stats_nccl(colo_ctx* ctx, void* nccl_comm, const colo_model* models, const colo_gpu* gpus,
                                    size_t nprofiles, const double* d_arrival, const uint32_t* d_prompt,
                                    const uint32_t* d_output, size_t n, const uint64_t* d_dev_offsets,
                                    const uint16_t* d_dev_profile, size_t ndev, double tau, double* pctl,
                                    colo_device_summary* totals) {
    if (!nccl_comm) return COLO_EINVAL;
    return serving_stats_impl(ctx, nccl_comm, models, gpus, nprofiles, d_arrival, d_prompt, d_output, n, d_dev_offsets,
                              d_dev_profile, ndev, tau, pctl, totals);
}

}  // extern "C"
