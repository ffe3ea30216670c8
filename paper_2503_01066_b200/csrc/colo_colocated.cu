// colo_colocated.cu -- colocated replay: Simulation::run
// in SimMode::Colocated, the full admission loop -- serving batches, the
// single activation slot, the offloading/hedging decision and its side
// effects, forward-order freeing, prefetch plans, per-layer preemption and the
// cache timeout (include/colosim/engine.hpp:140-822, memory.hpp:19-211).
//
// One warp per device (devices share no state).  The event
// loop is warp-uniform scalar code; the data-parallel parts run across the
// lanes:
//   * batch formation (prefix sums of serving_memory over the queue),
//   * a batch's decode: lane l folds the durations of steps k0+l, k0+32+l, ...
//     over the members in batch order, the absolute-time chain then runs
//     through the lanes in order (the same scheme as colo_serving.cu),
//   * per-layer slot state (lane l owns layers l, l+32, ...): footprints,
//     forward-order freeing, prefetch-plan construction, peaks.
//
// Event order.  The reference pushes all arrivals first (seq 0..N-1,
// engine.hpp:146-147) and pops by (time, seq) (:184-187): arrivals are a
// sorted stream that wins every tie.  Every other event takes the next
// sequence number at schedule() time.  Pending non-arrival events are few and
// kept in registers:
//   serving   one event per batch: its last decode step.  Nothing that can
//             interleave with a batch (arrivals, labels, timeouts -- prefetch
//             loads are always stale while serving runs, training never is in
//             flight) reads what the intermediate steps change, and their
//             ledger frees commute, so the whole batch is computed when it
//             starts and handled at its end.  Its PrefillDone / step events'
//             sequence numbers are still consumed (s_end = s_0 + K - 1).
//   training  at most one forward/backward layer (training_inflight_).
//   label     at most one live: a second label can only be scheduled after the
//             first one's generation was torn down, and a stale label only
//             counts labels_dropped when popped (engine.hpp:493-495) -- it is
//             counted when superseded.
//   timeout   at most one live: older generations' timeouts are no-ops.
//   loads     the current prefetch plan (shared memory), a sorted stream;
//             a bumped plan_generation_ makes all of it no-ops.
// CopyDone events only update host_bytes, which no report field reads; they
// consume their sequence numbers and are not materialised (the event log
// records them with their time and sequence number instead).
//
// Instantiations: k_colocated<false> runs device w on warp w over its whole
// trace; k_colocated<true> runs P.tasks[w] -- a whole trace, a speculative
// segment or an output segment of one long device (see SegTask); and
// k_colocated<false, true> additionally appends every event the reference
// logs (see EvRec; colo_colocated_events).  SeparateCluster devices serve as
// ServingOnly and emit their trainer jobs (k_trainer_fold folds them).
//
// Every f64 operation is the reference's, in the reference's order
// (-fmad=false), so each device's MetricsReport fields and TPT samples equal
// Simulation::run's bit for bit.  Reference paths are relative to
// /root/reference/proj/.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "colo_internal.h"
#include "colo_replay.cuh"

using namespace colo;

namespace {

constexpr int kWarpsC = 4;     // warps (devices) per CTA
constexpr int kStageC = 256;   // batch members staged in shared memory
constexpr int kLayerCap = 256; // >= kMaxLayers

enum { PH_WAIT = 0, PH_READY = 1, PH_FWD = 2, PH_BWD = 3 };  // engine.hpp:203
enum { LF_DEV = 1, LF_CONS = 2, LF_DROP = 4 };               // memory.hpp:49-51
enum { EK_NONE = 0, EK_SERVE, EK_TRAIN, EK_LABEL, EK_TIMEOUT, EK_LOAD };

struct CoProfile {
    colo_model m;
    uint64_t cap, budget, fixed, h2d, d2h;
    uint32_t cpa, L;
};

// ---- one device's trace in parallel segments ----------------------------------
// At an arrival popped while no batch is serving, no training layer is in
// flight, the queue is empty (arrivals queued behind a training layer wait for
// the next arrival, engine.hpp:273), there is no slot / job (has_store_
// false), no label pending and the d2h channel is free (busy_until <= now),
// the state is *fresh-equivalent*:
// the rest of the run equals a run started fresh at that arrival.  Pending
// cache timeouts are stale (generation mismatch) and prefetch plans cancelled,
// so both are no-ops; sequence numbers only order events relative to each
// other; the ledger's live bytes are the fixed footprint, and allocated_ =
// max(allocated_ before, live) makes peak_allocated the max over segments.
// So (speculate) every segment j runs fresh from s_j and records the idle
// arrivals it meets in [s_j, s_{j+1}) (head) and past s_{j+1} (tail); (resolve)
// the true run enters segment j at b_j = the first arrival idle in both
// segment j-1's tail and segment j's head (b_0 = 0, by induction the truth is
// idle there and equals segment j's run); (out) every segment replays
// [b_j, b_{j+1}) with all outputs at offsets from the recorded counters.  The
// three f64 sums of the report are sequential folds; the segments log their
// addends and k_fold_* fold the logs exactly in the reference's order.
constexpr int kSegPts = 32;  // idle arrivals kept per head / tail list
enum { TM_DIRECT = 0, TM_SPEC = 1, TM_OUT = 2 };

struct SegTask {
    uint32_t dev, mode;
    uint64_t start;  // first query (device-local)
    uint64_t next;   // SPEC: the next segment's start; OUT: the stop arrival (b_{j+1}, or N)
    uint64_t xend;   // SPEC: give up past this query
    uint64_t batch_base, job_base, sample_base;
    uint64_t log_base[3];  // absolute positions in P.log[k]
    uint64_t expect[5];    // OUT: batches, jobs, log entries the speculation counted (a mismatch is an error)
};

struct SegPoint {  // counters at an idle arrival (relative to the segment start)
    uint64_t idx, samples, batches, jobs, nlog[3];
};

struct SegSpec {
    uint32_t nhead, ntail, err, pad;
    SegPoint end;  // counters at the end of the trace (idx = ~0: not reached)
    SegPoint head[kSegPts];
    SegPoint tail[kSegPts];
};

struct SegOut {
    colo_colocated_summary s;
    uint64_t jobs;
    uint64_t err;     // 0, or why the segment disagreed with its speculation (1 busy / 2 not idle at the stop, 3 counts)
    uint64_t nlog[3];
};

// Event log (tools/colosim.cpp --emit-events, engine.hpp:109-129, 241-244):
// the kernel appends one record per logged event; the dispatch order is the
// (time, sequence) order of the handled events, so the host sorts records by
// (t, seq, sub) -- sub orders several records logged inside one handler --
// and a store-teardown marker drops CopyDone records of torn-down stores
// (engine.hpp:798-805).  Kinds follow EventKind (engine.hpp:78-90).
enum { EV_ARRIVAL = 0, EV_PREFILL, EV_STEP, EV_QDONE, EV_LABEL, EV_TIMEOUT, EV_RESUME, EV_BWD, EV_FWD, EV_LOAD,
       EV_COPY, EV_TEARDOWN = 100 };
struct EvRec {
    double t, start, dur;
    uint64_t key;  // seq << 16 | sub
    int64_t a, b;
    uint32_t kind, gen;
};

struct CoParams {
    CoProfile prof[kMaxSets];
    MapView sets[kMaxSets];
    const double* arr;
    const uint32_t* p;
    const uint32_t* o;
    const double* ld;
    double ld_default;
    const uint64_t* dev_off;
    const uint16_t* dev_set;
    uint32_t ndev;
    double timeout, tau;
    double* samples;
    const uint64_t* sample_off;
    uint8_t* labels;
    colo_batch* batches;
    colo_colocated_summary* summary;
    uint64_t* hist;
    uint32_t nfilters, hist_shift, filter_shift;
    uint64_t prefix[3];
    int* err;      // bit0 validation, bit1 breach, bit2 a SeparateCluster job stream needs sorting
    const uint8_t* sim_mode;
    double* job_t;     // SeparateCluster job stream (enqueue time), at dev_off[d] + i
    uint32_t* job_q;   // ... and its query (device-local index)
    uint64_t* job_cnt; // [ndev]
    // segmented runs (NULL tasks: warp w = device w, whole trace)
    const SegTask* tasks;
    uint32_t ntasks;
    EvRec* evlog;      // event log (LOG instantiation): records, their count and capacity
    unsigned long long* evcnt;
    uint64_t evcap;
    const uint64_t* qid;  // query ids (device-local index -> id) for the log
    double* lstart;       // LOG: [device][kLayerCap] start times of the current prefetch plan's loads
    SegSpec* spec;     // [task] (SPEC)
    SegOut* segout;    // [task] (OUT)
    double* log[3];    // addends of training_busy_time, copy_stall_seconds, prefetch_wait_seconds (OUT)
};

struct WarpSmem {
    uint64_t rec[kLayerCap];     // LayerActivation::recorded_bytes
    double lcd[kLayerCap];       // LayerActivation::last_copy_done
    double ldone[kLayerCap];     // current prefetch plan: completion times, channel order
    uint16_t llayer[kLayerCap];  // current prefetch plan: layer per load
    uint8_t flg[kLayerCap];      // LF_* (on_device, consumed, dropped)
    uint2 po[kStageC];           // batch members (prompt, output)
    double pd[kStageC];          // (double)prompt
    alignas(16) double dk[128];  // step durations of the current 128-step window
};

__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v = min(v, __shfl_xor_sync(kFullMask, v, s));
    return v;
}

__device__ __forceinline__ double warp_max_f64(double v) {
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v = dmax(v, __shfl_xor_sync(kFullMask, v, s));
    return v;
}

// SEG = false: warp w is device w over its whole trace (no segment code at all);
// SEG = true: warp w runs P.tasks[w] (whole-trace, speculative or output segment)
template <bool SEG, bool LOG = false>
__global__ void __launch_bounds__(kWarpsC * 32) k_colocated(const __grid_constant__ CoParams P) {
    __shared__ WarpSmem SM[kWarpsC];
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * kWarpsC + wib;
    if (SEG ? w >= P.ntasks : w >= P.ndev) return;
    const uint32_t d = SEG ? P.tasks[w].dev : w;
    const int tmode = SEG ? static_cast<int>(P.tasks[w].mode) : static_cast<int>(TM_DIRECT);
    const uint64_t q0 = SEG ? P.tasks[w].start : 0;
    const bool spec = tmode == TM_SPEC;
    WarpSmem& S = SM[wib];
    const uint32_t pi = P.dev_set[d];
    const CoProfile& pf = P.prof[pi];
    const MapView& mv = P.sets[pi];
    const colo_model& m = pf.m;
    const uint32_t L = pf.L;
    const bool cpa = pf.cpa != 0;
    const uint64_t cap = pf.cap, budget = pf.budget;
    const uint64_t lo = P.dev_off[d], N = P.dev_off[d + 1] - lo;
    const double* __restrict__ arr = P.arr + lo;
    const uint32_t* __restrict__ pp = P.p + lo;
    const uint32_t* __restrict__ po = P.o + lo;
    const double dL = static_cast<double>(L);
    const double gam = m.decode_coef_const, del = m.decode_coef_context;
    const int smode = P.sim_mode ? P.sim_mode[d] : COLO_SIM_COLOCATED;
    const bool colocated = smode == COLO_SIM_COLOCATED;  // the slot and the offloader exist only here
    const bool separate = smode == COLO_SIM_SEPARATE;    // jobs go to the trainer stream
    uint64_t jc = 0;        // SeparateCluster jobs emitted
    double last_t = -1.0;   // enqueue time of the last emitted job
    bool unsorted = false;  // an emitted enqueue time went backwards (label delays vary)

    for (uint32_t l = lane; l < kLayerCap; l += 32) {
        S.rec[l] = 0;
        S.lcd[l] = 0.0;
        S.flg[l] = 0;
    }
    __syncwarp();

    // ---- state (warp-uniform) ----------------------------------------------
    double now = 0.0;
    uint64_t seq = N;          // arrivals own 0..N-1
    uint64_t ai = q0, qhead = q0;  // queue_ = [qhead, ai)
    uint64_t alloc = 0, resv = 0, peak = 0;  // MemoryLedger device_
    double d2h_busy = 0.0;                   // TransferChannel d2h_
    bool breach = false;
    // serving
    bool sbusy = false;
    double s_t = 0.0;
    uint64_t s_seq = 0, bfirst = 0, bn = 0, bneed = 0;
    uint32_t s_nlast = 0;  // LOG: members that finish at the batch's last step
    // slot
    bool has_store = false, qcompleted = false, stream = false;
    uint64_t src = 0, prompt_kv = 0, kv_held = 0, cached_tokens = 0, gen = 0, store_gen = 0, plan_gen = 0;
    // job
    bool has_job = false, incl_prompt = false, waiting = false, tinf = false;
    int phase = PH_WAIT;
    uint64_t jp = 0, jo = 0, pass0 = 0, pass1 = 0, pass2 = 0, npasses = 0, pass_index = 0, cursor = 0;
    int64_t kv_charged = -1;
    double wait_since = 0.0, plb = 0.0, tbusy = 0.0;  // plb = per_layer_backward(job) (engine.hpp:614-618)
    double t_t = 0.0, t_dur = 0.0, t_st = 0.0;  // t_st: when the in-flight layer was scheduled (LOG)
    uint32_t t_pb = 0;                          // ... and its pass index (ForwardLayerDone b)
    double h_t = 0.0;  // LOG: the handled event's time and sequence, and the next sub-position in it
    uint64_t h_seq = 0;
    uint32_t h_sub = 0;
    uint64_t t_seq = 0;
    bool t_fwd = false;
    uint32_t t_a = 0;
    // label / timeout slots, prefetch plan
    bool l_on = false, to_on = false;
    double l_t = 0.0, to_t = 0.0;
    uint64_t l_seq = 0, l_gen = 0, to_seq = 0, to_gen = 0;
    uint32_t ld_n = 0, ld_cur = 0;
    uint64_t ld_gen = 0, ld_seq0 = 0;
    // slot aggregates kept incrementally (recomputed after bulk updates):
    //   ag_dev  device_act_bytes()       (memory.hpp:91-96)
    //   ag_cnt  device_resident_layers() (memory.hpp:108-113)
    //   ag_pend host_only_pending()      (memory.hpp:101-106)
    //   ag_t    sum of recorded bytes of not consumed / dropped layers (engine.hpp:817-819)
    uint64_t ag_dev = 0, ag_t = 0;
    uint32_t ag_cnt = 0, ag_pend = 0;
    // per-pass constants (recomputed bit-identically when the key changes)
    uint64_t fwd_tok = ~0ull, cp_bytes = ~0ull;
    double fwd_val = 0.0, cp_val = 0.0;
    double na = q0 < N ? arr[q0] : 0.0;  // arrival time of query ai
    // report (uniform) + per-lane sample partials
    uint64_t r_trained = 0, r_ptab = 0, r_pre = 0, r_freed = 0, r_loads = 0, r_recomp = 0, r_dropped = 0, r_jobs = 0,
             r_fb = 0, r_batches = 0, r_maxb = 0, r_offd = 0, r_adm = 0;
    double r_stall = 0.0, r_wait = 0.0, r_end = 0.0;
    uint64_t a_gen = 0, a_slow = 0, a_slowq = 0, a_acc[3] = {0, 0, 0};
    uint32_t a_flags = 0;
    // outputs (a speculative segment writes none; an OUT segment at its offsets)
    double* const samples_out = spec ? nullptr : P.samples;
    uint8_t* const labels_out = spec ? nullptr : P.labels;
    colo_batch* const batches_out =
        spec || !P.batches ? nullptr : P.batches + lo + (tmode == TM_OUT ? P.tasks[w].batch_base : 0);
    const uint64_t job_base = lo + (tmode == TM_OUT ? P.tasks[w].job_base : 0);
    uint64_t sample_pos = samples_out ? P.sample_off[d] + (tmode == TM_OUT ? P.tasks[w].sample_base : 0) : 0;
    const bool want_hist = !spec && P.hist != nullptr;
    // addends of the three f64 sums (counted by SPEC, logged by OUT)
    uint64_t nl0 = 0, nl1 = 0, nl2 = 0;
    bool seg_err = false, stopped = false;
    uint32_t seg_why = 0;
    uint32_t nhead = 0, ntail = 0;

    auto live = [&]() -> uint64_t { return alloc - resv; };
    auto led_alloc = [&](uint64_t bytes) -> bool {  // memory.hpp:28-35
        if (alloc - resv + bytes > cap) return false;
        const uint64_t reuse = resv < bytes ? resv : bytes;
        resv -= reuse;
        alloc += bytes - reuse;
        if (alloc > peak) peak = alloc;
        return true;
    };
    auto led_free = [&](uint64_t bytes) {  // memory.hpp:37-40
        if (bytes > alloc - resv) breach = true;  // std::logic_error
        resv += bytes;
    };
    // training_busy_time / copy_stall_seconds / prefetch_wait_seconds += x
    auto add_busy = [&](double x) {
        tbusy += x;
        if (tmode == TM_OUT && lane == 0 && nl0 < P.tasks[w].expect[2]) P.log[0][P.tasks[w].log_base[0] + nl0] = x;
        ++nl0;
    };
    auto add_stall = [&](double x) {
        r_stall += x;
        if (tmode == TM_OUT && lane == 0 && nl1 < P.tasks[w].expect[3]) P.log[1][P.tasks[w].log_base[1] + nl1] = x;
        ++nl1;
    };
    auto add_wait = [&](double x) {
        r_wait += x;
        if (tmode == TM_OUT && lane == 0 && nl2 < P.tasks[w].expect[4]) P.log[2][P.tasks[w].log_base[2] + nl2] = x;
        ++nl2;
    };
    // LOG: append one record from this lane (callers pick the lane)
    auto emit_from = [&](bool me, uint32_t kind, double t, uint64_t sq, uint32_t sub, int64_t a, int64_t b, double st,
                         double du, uint32_t g) {
        if (!LOG || !me) return;
        const unsigned long long i = atomicAdd(P.evcnt, 1ull);
        if (i < P.evcap) {
            EvRec r;
            r.t = t;
            r.start = st;
            r.dur = du;
            r.key = (sq << 16) | sub;
            r.a = a;
            r.b = b;
            r.kind = kind;
            r.gen = g;
            P.evlog[i] = r;
        }
    };
    auto emit = [&](uint32_t kind, double t, uint64_t sq, uint32_t sub, int64_t a, int64_t b, double st, double du,
                    uint32_t g) { emit_from(lane == 0, kind, t, sq, sub, a, b, st, du, g); };
    auto qid_of = [&](uint64_t j) -> int64_t { return static_cast<int64_t>(P.qid ? P.qid[lo + j] : j); };
    auto pass_tok = [&](uint64_t i) -> uint64_t { return i == 0 ? pass0 : (i == 1 ? pass1 : pass2); };
    uint64_t cur_tok = 0;  // passes[pass_index] of the running forward pass (set by begin_pass)
    auto fwd_layer = [&](uint64_t t) -> double {  // cost_model.hpp:39-41
        return prefill_latency(m, t, 1, false) / dL;
    };
    auto bwd_layer = [&](uint64_t t) -> double {  // cost_model.hpp:43-45
        return m.backward_to_forward_ratio * fwd_layer(t);
    };

    // ---- per-layer slot state ------------------------------------------------
    auto contrib = [&](uint8_t f, uint64_t r, bool add) {  // one layer's share of the aggregates
        const bool dv = f & LF_DEV, lv = !(f & (LF_CONS | LF_DROP));
        const uint64_t db = dv ? r : 0, tb = lv ? r : 0;
        const uint32_t dc = dv ? 1u : 0u, pc = (!dv && lv && r > 0) ? 1u : 0u;
        if (add) {
            ag_dev += db;
            ag_t += tb;
            ag_cnt += dc;
            ag_pend += pc;
        } else {
            ag_dev -= db;
            ag_t -= tb;
            ag_cnt -= dc;
            ag_pend -= pc;
        }
    };
    auto recount = [&]() {  // lane-parallel recomputation after a bulk update
        uint64_t db = 0, tb = 0;
        uint32_t dc = 0, pc = 0;
        for (uint32_t l = lane; l < L; l += 32) {
            const uint8_t f = S.flg[l];
            const uint64_t r = S.rec[l];
            const bool dv = f & LF_DEV, lv = !(f & (LF_CONS | LF_DROP));
            db += dv ? r : 0;
            tb += lv ? r : 0;
            dc += dv;
            pc += !dv && lv && r > 0;
        }
        ag_dev = warp_sum_u64(db);
        ag_t = warp_sum_u64(tb);
        ag_cnt = static_cast<uint32_t>(warp_sum_u64(dc));
        ag_pend = static_cast<uint32_t>(warp_sum_u64(pc));
    };
    auto set_layer = [&](uint32_t l, uint8_t f, uint64_t r) {  // single-layer update (owner lane writes)
        contrib(S.flg[l], S.rec[l], false);
        contrib(f, r, true);
        __syncwarp();
        if (lane == (l & 31)) {
            S.flg[l] = f;
            S.rec[l] = r;
        }
        __syncwarp();
    };
    auto training_peak = [&]() {  // engine.hpp:815-822
        if (!has_store) return;
        const uint64_t cur = kv_held + ag_t;
        if (cur > r_ptab) r_ptab = cur;
    };
    auto teardown = [&]() {  // engine.hpp:468-479
        if (!has_store) return;
        emit(EV_TEARDOWN, h_t, h_seq, 0xff00u, 0, 0, 0.0, 0.0, static_cast<uint32_t>(gen));
        uint64_t s = 0;
        for (uint32_t l = lane; l < L; l += 32)
            if (S.flg[l] & LF_DEV) {
                s += S.rec[l];
                S.flg[l] &= ~LF_DEV;
            }
        __syncwarp();
        led_free(warp_sum_u64(s));
        recount();
        if (kv_held) led_free(kv_held);
        has_store = false;
        has_job = false;
        ++plan_gen;
    };
    // memory.hpp:121-139 for one layer (+ its CopyDone sequence number)
    auto record = [&](uint32_t l, uint64_t bytes, double t) {
        uint8_t f = S.flg[l];
        uint64_t r = S.rec[l];
        f &= ~LF_DROP;
        const bool to_host = stream || (r > 0 && !(f & LF_DEV));
        if (!to_host) {
            if (!led_alloc(bytes)) breach = true;
            f |= LF_DEV;
        }
        r += bytes;
        if (bytes != cp_bytes) {  // transfer_time (cost_model.hpp:68-71)
            cp_bytes = bytes;
            cp_val = static_cast<double>(bytes) / static_cast<double>(pf.d2h);
        }
        const double start = dmax(t, d2h_busy);
        d2h_busy = start + cp_val;
        if (lane == (l & 31)) S.lcd[l] = d2h_busy;
        set_layer(l, f, r);
        emit(EV_COPY, d2h_busy, seq, 0, l, static_cast<int64_t>(bytes), t, d2h_busy - t, static_cast<uint32_t>(gen));
        ++seq;
    };
    // engine.hpp:563-610
    auto drop_for_recompute = [&](uint64_t need_total) {
        ++r_recomp;
        ++plan_gen;
        uint64_t s = 0;
        for (uint32_t l = lane; l < L; l += 32) {
            if (S.flg[l] & LF_DEV) s += S.rec[l];
            S.flg[l] = LF_DROP;
            S.rec[l] = 0;
            S.lcd[l] = 0.0;
        }
        __syncwarp();
        led_free(warp_sum_u64(s));
        ag_dev = ag_t = 0;
        ag_cnt = ag_pend = 0;
        const uint64_t response_kv = kv_held - prompt_kv;
        if (response_kv) led_free(response_kv);
        kv_held = prompt_kv;
        if (has_job) {
            pass_index = 0;
            cursor = 0;
            kv_charged = -1;
            waiting = false;
            if (phase != PH_WAIT) phase = PH_READY;
            if (!cpa) {
                pass0 = jp;
                npasses = 1;
                plb = 0.0 + bwd_layer(jp);
            } else {
                incl_prompt = true;
                pass0 = jp;
                pass1 = pass2 = jo;
                npasses = 3;
                double b = 0.0;
                b += bwd_layer(jp);
                b += bwd_layer(jo);
                b += bwd_layer(jo);
                plb = b;
            }
        }
        if (kv_held > 0 && live() + need_total > cap) {
            led_free(kv_held);
            kv_held = 0;
            prompt_kv = 0;
        }
        training_peak();
    };

    // ---- training path --------------------------------------------------------
    auto schedule_forward = [&]() {  // engine.hpp:685-691
        const uint64_t tok = cur_tok;
        if (tok != fwd_tok) {
            fwd_tok = tok;
            fwd_val = fwd_layer(tok);
        }
        t_dur = fwd_val;
        tinf = true;
        t_fwd = true;
        t_a = static_cast<uint32_t>(cursor);
        t_st = now;
        t_pb = static_cast<uint32_t>(pass_index);
        t_t = now + t_dur;
        t_seq = seq++;
    };
    auto begin_pass = [&]() {  // engine.hpp:662-683
        cur_tok = pass_tok(pass_index);
        if (kv_charged != static_cast<int64_t>(pass_index)) {
            kv_charged = static_cast<int64_t>(pass_index);
            if (cpa) {
                const bool is_prompt = incl_prompt && pass_index == 0;
                if (!(is_prompt && prompt_kv > 0)) {
                    const uint64_t kv = kv_bytes(m, cur_tok, 1);
                    if (!led_alloc(kv)) breach = true;
                    kv_held += kv;
                    if (is_prompt) prompt_kv += kv;
                    training_peak();
                }
            }
        }
        schedule_forward();
    };
    auto schedule_backward = [&]() {  // engine.hpp:749-759
        if (!(S.flg[cursor] & LF_DEV)) {
            waiting = true;
            wait_since = now;
            return;
        }
        t_dur = plb;
        tinf = true;
        t_fwd = false;
        t_a = static_cast<uint32_t>(cursor);
        t_st = now;
        t_t = now + t_dur;
        t_seq = seq++;
    };
    // engine.hpp:733-747 + plan_prefetch (memory.hpp:183-211; only the loads are consumed)
    auto start_backward = [&]() {
        ++plan_gen;
        double channel = now;
        uint32_t cnt = 0;
        for (int top = static_cast<int>(L) - 1; top >= 0; top -= 32) {
            const int l = top - static_cast<int>(lane);  // lane 0 = highest layer of the chunk
            bool el = false;
            double dur = 0.0;
            if (l >= 0) {
                const uint8_t f = S.flg[l];
                const uint64_t r = S.rec[l];
                el = !(f & (LF_DEV | LF_CONS | LF_DROP)) && r > 0;
                dur = static_cast<double>(r) / static_cast<double>(pf.h2d);
            }
            const uint32_t bal = __ballot_sync(kFullMask, el);
            double mine = 0.0, mine0 = 0.0;
            for (uint32_t b = bal; b; b &= b - 1) {  // channel += dur, descending layer order
                const int j = __ffs(b) - 1;
                const double before = channel;
                channel += __shfl_sync(kFullMask, dur, j);
                if (lane == static_cast<uint32_t>(j)) {
                    mine0 = before;
                    mine = channel;
                }
            }
            if (el) {
                const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                S.llayer[pos] = static_cast<uint16_t>(l);
                S.ldone[pos] = mine;
                if (LOG) P.lstart[static_cast<uint64_t>(d) * kLayerCap + pos] = mine0;  // LoadDone start
            }
            cnt += __popc(bal);
        }
        __syncwarp();
        ld_n = cnt;
        ld_cur = 0;
        ld_gen = plan_gen;
        ld_seq0 = seq;
        seq += cnt;
        schedule_backward();
    };
    auto try_start_training = [&]() {  // engine.hpp:633-660
        if (!has_job || sbusy || qhead != ai || tinf) return;
        if (phase != PH_WAIT) emit(EV_RESUME, h_t, h_seq, h_sub++, qid_of(src), 0, h_t, 0.0, 0u);
        switch (phase) {
            case PH_WAIT: return;
            case PH_READY:
                if (pass_index < npasses) {
                    phase = PH_FWD;
                    cursor = 0;
                    begin_pass();
                } else {
                    phase = PH_BWD;
                    cursor = L - 1;
                    start_backward();
                }
                return;
            case PH_FWD: begin_pass(); return;
            default: start_backward(); return;
        }
    };

    // ---- offloader ------------------------------------------------------------
    // engine.hpp:513-557 (+ free_layers_forward_order, memory.hpp:150-165)
    auto apply_offload = [&](uint64_t incoming, uint64_t batch_n, uint64_t need_total, uint32_t& vbits) -> double {
        ++r_offd;
        const uint64_t cached = cached_tokens;
        uint32_t code = offload_lookup(mv, mv.off, cached, incoming, batch_n);
        const uint32_t fallback = code == 0xffu;
        if (fallback) {
            ++r_fb;
            code = 1;
        }
        if (code == 0) {
            vbits = COLO_V_EVALUATED | pack_verdict(0, 0, 0, 0, 0, 0, COLO_VD_ADMIT);
            return 0.0;
        }
        const uint32_t dev_layers = ag_cnt, pending = ag_pend;
        const uint32_t action = code == 1 ? COLO_ACT_ALLTOHOST : COLO_ACT_FREELAYERS;
        const uint32_t layers = code >= 2 ? code - 2 : 0;
        const uint32_t free_now = code == 1 ? dev_layers : min(layers, dev_layers);
        const uint32_t ltf = code == 1 ? L : layers;
        const uint32_t total = min(pending + ltf, L);
        uint32_t recompute = 1, hedge_oor = 0;
        if (!fallback) {
            if (cached == 0 || cached > mv.hmax) {  // HedgingMap::lookup nullopt (maps.hpp:278)
                hedge_oor = 1;
                ++r_fb;
            } else {
                const uint32_t hi = ceil_div(mv.fh, static_cast<uint32_t>(cached)) - 1;
                recompute = mv.hed[hi * (L + 1) + total];
            }
        }
        if (recompute) {
            drop_for_recompute(need_total);
            vbits = COLO_V_EVALUATED |
                    pack_verdict(action, layers, free_now, 1, fallback, hedge_oor, COLO_VD_RECOMPUTE_DROP);
            return 0.0;
        }
        ++plan_gen;
        // free the free_now lowest device-resident layers
        uint32_t left = free_now, freed = 0;
        double ready = now;
        uint64_t fb = 0;
        for (uint32_t l0 = 0; l0 < L && left; l0 += 32) {
            const uint32_t l = l0 + lane;
            const bool dv = l < L && (S.flg[l] & LF_DEV);
            const uint32_t bal = __ballot_sync(kFullMask, dv);
            const bool take = dv && static_cast<uint32_t>(__popc(bal & ((1u << lane) - 1u))) < left;
            if (take) {
                ready = dmax(ready, S.lcd[l]);
                fb += S.rec[l];
                S.flg[l] &= ~LF_DEV;
            }
            const uint32_t t = min(static_cast<uint32_t>(__popc(bal)), left);
            left -= t;
            freed += t;
        }
        __syncwarp();
        ready = warp_max_f64(ready);
        led_free(warp_sum_u64(fb));
        recount();
        r_freed += freed;
        if (live() + need_total > cap) {  // KV corner (engine.hpp:549-552)
            drop_for_recompute(need_total);
            vbits = COLO_V_EVALUATED |
                    pack_verdict(action, layers, free_now, 0, fallback, hedge_oor, COLO_VD_RECOMPUTE_DROP);
            return 0.0;
        }
        const double stall = dmax(0.0, ready - now);
        add_stall(stall);
        add_busy(stall);
        vbits = COLO_V_EVALUATED | pack_verdict(action, layers, free_now, 0, fallback, hedge_oor, COLO_VD_FREE_LOADBACK);
        return stall;
    };

    // engine.hpp:421-466
    auto admit = [&](uint64_t j, uint32_t& vbits) {
        const uint32_t pj = pp[j], oj = po[j];
        const uint64_t charged = charged_tokens(pj, oj, cpa ? 1u : 0u);
        has_store = true;
        for (uint32_t l = lane; l < L; l += 32) {
            S.rec[l] = 0;
            S.lcd[l] = 0.0;
            S.flg[l] = 0;
        }
        __syncwarp();
        ag_dev = ag_t = 0;
        ag_cnt = ag_pend = 0;
        src = j;
        prompt_kv = 0;
        kv_held = 0;
        qcompleted = false;
        cached_tokens = charged;
        gen = ++store_gen;
        bool st = false;
        const uint32_t code = offload_lookup(mv, mv.off, charged, 1, 1);
        if (code == 0xffu) {
            st = true;
            ++r_fb;
            vbits |= COLO_V_STREAM_OOR;
        } else if (code == 1) {
            st = true;
        }
        const uint64_t prompt_acts = static_cast<uint64_t>(pj) * L * m.act_bytes_per_token_per_layer;
        if (live() + prompt_acts > cap) st = true;
        stream = st;
        vbits |= COLO_V_ADMITTED | (st ? COLO_V_STREAM : 0u);
        ++r_adm;
        has_job = true;
        jp = pj;
        jo = oj;
        pass_index = 0;
        cursor = 0;
        incl_prompt = false;
        kv_charged = -1;
        waiting = false;
        if (!cpa) {
            phase = PH_READY;
            npasses = 0;
            plb = 0.0 + bwd_layer(jp);
        } else {
            phase = PH_WAIT;
            pass0 = pass1 = oj;
            npasses = 2;
            double b = 0.0;
            b += bwd_layer(jp);
            b += bwd_layer(jo);
            b += bwd_layer(jo);
            plb = b;
            to_on = true;  // an older generation's timeout is a no-op when popped
            to_t = now + P.timeout;
            to_seq = seq++;
            to_gen = gen;
        }
    };

    // ---- serving path -----------------------------------------------------------
    // engine.hpp:282-328 + the whole batch (prefill, decode steps, samples)
    auto start_serving = [&]() {
        if (qhead == ai) {
            sbusy = false;
            try_start_training();
            return;
        }
        sbusy = true;
        const uint64_t head = qhead, tail = ai;
        // batch formation: FIFO, at least one, sum(need) <= budget (engine.hpp:292-306)
        uint64_t end = head, need_total = 0, max_inc = 0;
        uint32_t maxo = 0;
        while (end < tail) {
            const uint64_t j = end + lane;
            const bool valid = j < tail;
            const uint32_t pj = valid ? pp[j] : 0u, oj = valid ? po[j] : 0u;
            const uint64_t nd = valid ? serving_memory(m, static_cast<uint64_t>(pj) + oj, 1) : 0ull;
            uint64_t incl = nd;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint64_t y = __shfl_up_sync(kFullMask, incl, s);
                if (lane >= static_cast<uint32_t>(s)) incl += y;
            }
            incl += need_total;
            const bool ok = valid && (j == head || incl <= budget);
            const uint32_t cnt = __popc(__ballot_sync(kFullMask, ok));
            if (ok && j - head < kStageC) {
                S.po[j - head] = make_uint2(pj, oj);
                S.pd[j - head] = static_cast<double>(pj);
            }
            max_inc = max(max_inc, warp_max_u64(ok ? static_cast<uint64_t>(pj) + oj : 0ull));
            maxo = max(maxo, static_cast<uint32_t>(warp_max_u64(ok ? oj : 0u)));
            if (cnt) need_total = __shfl_sync(kFullMask, incl, cnt - 1);
            end += cnt;
            if (cnt < 32) break;
        }
        __syncwarp();
        const uint64_t nb = end - head;
        bfirst = head;
        bn = nb;
        bneed = need_total;
        qhead = end;
        uint32_t vbits = 0;
        double stall = 0.0;
        if (colocated && has_store && kv_held + ag_dev > 0) stall = apply_offload(max_inc, nb, need_total, vbits);
        if (!led_alloc(need_total)) breach = true;  // engine.hpp:312-313
        bool rec = false;
        if (colocated && nb == 1 && !has_store) {
            admit(head, vbits);
            rec = true;
        }
        const bool staged = nb <= kStageC;
        auto member_pd = [&](uint64_t j) -> double { return staged ? S.pd[j] : static_cast<double>(pp[head + j]); };
        // prefill: left fold in batch order (engine.hpp:321-325); member 0 may be recording
        double dur = 0.0;
        if (staged) {
#pragma unroll 4
            for (uint64_t j = 0; j < nb; ++j) {
                const double t = S.pd[j];
                double base = 1.0 * (m.prefill_coef_linear * t + m.prefill_coef_quad * t * t);
                if (j == 0 && rec) base = base * m.record_prefill_multiplier;
                dur += base;
            }
        } else {
            for (uint64_t j = 0; j < nb; ++j) {
                const double t = member_pd(j);
                double base = 1.0 * (m.prefill_coef_linear * t + m.prefill_coef_quad * t * t);
                if (j == 0 && rec) base = base * m.record_prefill_multiplier;
                dur += base;
            }
        }
        const double start = now + stall;
        const uint64_t pf_seq = seq;
        ++seq;  // PrefillDone
        if (rec) {  // engine.hpp:332-350
            const uint64_t per_layer = static_cast<uint64_t>(pp[head]) * m.act_bytes_per_token_per_layer;
            const double layer_dur = dur / dL;
            for (uint32_t l = 0; l < L; ++l) {
                const double seg_ready = start + static_cast<double>(l + 1) * layer_dur;
                if (stream && S.rec[l] == 0) ++r_freed;
                record(l, per_layer, seg_ready);
            }
            training_peak();
        }
        const uint64_t step_seq0 = seq;  // DecodeStepDone k takes step_seq0 + k (see the header)
        emit(EV_PREFILL, start + dur, pf_seq, 0, static_cast<int64_t>(nb), 0, start, dur, 0u);
        if (LOG) {  // QueryDone records: each member at its last step, in batch order among that step's finishers
            uint32_t nl = 0;
            for (uint64_t j = lane; j < nb; j += 32) nl += (staged ? S.po[j].y : po[head + j]) == maxo;
            s_nlast = static_cast<uint32_t>(warp_sum_u64(nl));
        }
        double tnow = start + dur;  // PrefillDone time: every member's last_token_time
        // decode steps (engine.hpp:358-387), four 32-step windows per pass
        uint32_t first_slow = 0xffffffffu;
        for (uint32_t k0 = 0; k0 < maxo; k0 += 128) {
            double dk[4] = {0.0, 0.0, 0.0, 0.0};
            uint32_t alive[4] = {0, 0, 0, 0};
            const uint32_t kb = k0 + lane;
            double kd[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) kd[r] = static_cast<double>(kb + 32 * r);
            if (staged) {  // members from shared memory, unrolled so loads overlap the accumulate chains
#pragma unroll 4
                for (uint64_t j = 0; j < nb; ++j) {
                    const uint32_t oj = S.po[j].y;
                    const double pj = S.pd[j];
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
            for (int r = 0; r < 4; ++r) S.dk[32 * r + lane] = dk[r];
            __syncwarp();
            // absolute-time chain now_k = now_{k-1} + d_k (sequential, one lane),
            // the durations are overwritten by the absolute times
            const uint32_t cnt = min(128u, maxo - k0);
            if (lane == 0) chain_fold_store(tnow, S.dk, cnt);  // (a warp scan is slower here: other warps hide this)
            __syncwarp();
            const double tnow0 = tnow;  // the rows below read their samples back (one rolled body)
            if (LOG) {
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint32_t i = 32 * r + lane;
                    emit_from(i < cnt, EV_STEP, i < cnt ? S.dk[i] : 0.0, step_seq0 + k0 + i, 0, 0, 0,
                              i < cnt ? (i ? S.dk[i - 1] : tnow) : 0.0, dk[r], 0u);
                }
                for (uint64_t j = lane; j < nb; j += 32) {
                    const uint32_t oj = staged ? S.po[j].y : po[head + j];
                    if (oj - 1 < k0 || oj - 1 >= k0 + cnt) continue;
                    uint32_t rank = 0;
                    for (uint64_t jj = 0; jj < j; ++jj) rank += (staged ? S.po[jj].y : po[head + jj]) == oj;
                    const double tf = S.dk[oj - 1 - k0];
                    emit_from(true, EV_QDONE, tf, step_seq0 + oj - 1, 1 + rank, qid_of(head + j), 0, tf, 0.0, 0u);
                }
            }
            tnow = S.dk[cnt - 1];
            if (separate) {
                // finish_query of the members that finish in this window, in the
                // reference's order (step, then batch order): CPT enqueues the
                // job at the finish time, CPA schedules its label at finish +
                // delay (engine.hpp:410-416)
                auto member_o = [&](uint64_t j) -> uint32_t { return staged ? S.po[j].y : po[head + j]; };
                const uint32_t wend = k0 + cnt;
                uint32_t cur = k0;
                for (;;) {
                    uint32_t mn = 0xffffffffu;
                    for (uint64_t j = lane; j < nb; j += 32) {
                        const uint32_t f = member_o(j) - 1;
                        if (f >= cur && f < wend) mn = min(mn, f);
                    }
                    mn = warp_min_u32(mn);
                    if (mn == 0xffffffffu) break;
                    const double tf = S.dk[mn - k0];
                    for (uint64_t j0 = 0; j0 < nb; j0 += 32) {
                        const uint64_t j = j0 + lane;
                        bool em = false;
                        double te = tf;
                        if (j < nb && member_o(j) - 1 == mn) {
                            if (!cpa) {
                                em = true;
                            } else {
                                const double ldl = P.ld ? P.ld[lo + head + j] : P.ld_default;
                                if (ldl >= 0.0) {
                                    em = true;
                                    te = tf + ldl;
                                }
                            }
                        }
                        const uint32_t bal = __ballot_sync(kFullMask, em);
                        if (bal) {
                            const uint32_t below = bal & ((1u << lane) - 1u);
                            const double prev_lane = __shfl_sync(kFullMask, te, below ? 31 - __clz(below) : 0);
                            if (LOG && em && cpa)  // LabelArrival (-1, query) popped at te (engine.hpp:414-416, 481-486)
                                emit_from(true, EV_LABEL, te, step_seq0 + mn, 0x4000u + static_cast<uint32_t>(j0 + lane),
                                          -1, qid_of(head + j), te, 0.0, 0u);
                            if (em) {
                                if (te < (below ? prev_lane : last_t)) unsorted = true;
                                if (!spec && (tmode != TM_OUT || jc + __popc(below) < P.tasks[w].expect[1])) {
                                    const uint64_t pos = job_base + jc + __popc(below);
                                    P.job_t[pos] = te;
                                    P.job_q[pos] = static_cast<uint32_t>(head + j);
                                }
                            }
                            last_t = __shfl_sync(kFullMask, te, 31 - __clz(bal));
                            jc += __popc(bal);
                        }
                    }
                    cur = mn + 1;
                }
            }
            __syncwarp();
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
                const uint32_t kr0 = k0 + 32 * r;
                if (kr0 >= maxo) break;
                const uint32_t k = kr0 + lane;
                const uint32_t i = 32 * r + lane;  // sample = now - last_token_time
                const double s = i < cnt ? S.dk[i] - (i ? S.dk[i - 1] : tnow0) : 0.0;
                const uint32_t alv = r == 0 ? alive[0] : r == 1 ? alive[1] : r == 2 ? alive[2] : alive[3];
                const bool lv = k < maxo;
                const bool slow = lv && s > P.tau;
                const uint32_t sb = __ballot_sync(kFullMask, slow);
                if (sb && first_slow == 0xffffffffu) first_slow = kr0 + __ffs(sb) - 1;
                a_gen += alv;
                if (slow) a_slow += alv;
                if (want_hist) {  // warp-aggregated: lanes with the same bin add once
                    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(s));
                    for (uint32_t f = 0; f < P.nfilters; ++f)
                        hist_add(P.hist, f * COLO_HIST_BINS + static_cast<uint32_t>((bits >> P.hist_shift) & (COLO_HIST_BINS - 1)),
                                 alv, lv && (bits >> P.filter_shift) == P.prefix[f]);
                }
                if (lv) {
                    acc_fixed(a_acc, a_flags, s, alv);
                }
                if (samples_out) {  // step k's samples: alive_k consecutive slots, steps in order
                    uint32_t ex = alv;
#pragma unroll
                    for (int sft = 1; sft < 32; sft <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFullMask, ex, sft);
                        if (lane >= static_cast<uint32_t>(sft)) ex += y;
                    }
                    const uint32_t tot = __shfl_sync(kFullMask, ex, 31);
                    const uint64_t pos = sample_pos + ex - alv;
                    for (uint32_t a = 0; a < alv; ++a) samples_out[pos + a] = s;
                    sample_pos += tot;
                }
            }
            __syncwarp();  // the rows' reads of dk before the next window writes them
        }
        for (uint64_t j = lane; j < nb; j += 32) {  // a query is slow iff one of its tokens is
            const uint32_t oj = staged ? S.po[j].y : po[head + j];
            const bool slowq = oj > first_slow;
            a_slowq += slowq;
            if (labels_out) labels_out[lo + head + j] = slowq ? 1 : 0;
        }
        if (lane == 0 && batches_out && (tmode != TM_OUT || r_batches < P.tasks[w].expect[0])) {
            colo_batch b;
            b.start = start;
            b.end = tnow;
            b.first = static_cast<uint32_t>(head);
            b.n = static_cast<uint32_t>(nb);
            b.need_total = need_total;
            b.max_incoming = max_inc < 0xffffffffull ? static_cast<uint32_t>(max_inc) : 0xffffffffu;
            b.verdict = vbits;
            batches_out[r_batches] = b;
        }
        ++r_batches;
        if (nb > r_maxb) r_maxb = nb;
        seq += maxo;  // DecodeStepDone 0..K-1
        s_t = tnow;
        s_seq = seq - 1;
        __syncwarp();
    };
    // start_serving_batch is always the tail action of the handler that calls
    // it, so it runs once at the bottom of the event loop (one inlined copy).
    bool want_serve = false;
    auto preempt = [&]() -> bool {  // engine.hpp:725-731
        if (qhead == ai) return false;
        ++r_pre;
        ++plan_gen;
        want_serve = true;
        return true;
    };

    if (!led_alloc(pf.fixed)) breach = true;  // engine.hpp:141-142

    // ---- event loop ---------------------------------------------------------------
    while (!breach) {
        double bt = 0.0;
        uint64_t bs = ~0ull;
        int bk = EK_NONE;
        auto consider = [&](bool on, double t, uint64_t s, int k) {
            if (on && (bk == EK_NONE || t < bt || (t == bt && s < bs))) {
                bt = t;
                bs = s;
                bk = k;
            }
        };
        consider(sbusy, s_t, s_seq, EK_SERVE);
        consider(tinf, t_t, t_seq, EK_TRAIN);
        consider(l_on, l_t, l_seq, EK_LABEL);
        consider(to_on, to_t, to_seq, EK_TIMEOUT);
        if (ld_cur < ld_n && ld_gen != plan_gen) ld_cur = ld_n;  // cancelled plan: every load is a no-op
        if (ld_cur < ld_n) consider(true, S.ldone[ld_cur], ld_seq0 + ld_cur, EK_LOAD);
        if (ai < N && (bk == EK_NONE || na <= bt)) {  // arrivals win time ties
            if (sbusy || tinf) {  // engine.hpp:273: queued only; take every arrival up to the next event
                ai = bk == EK_NONE ? N : find_tail(arr, N, ai, bt);
                na = ai < N ? arr[ai] : 0.0;
                if (tmode != TM_DIRECT) {
                    if (tmode == TM_OUT && ai > P.tasks[w].next) {  // the stop arrival came while busy
                        seg_err = stopped = true;
                        seg_why = 1;
                        break;
                    }
                    if (spec && ai < N && ai >= P.tasks[w].xend) {
                        stopped = true;
                        break;
                    }
                }
                continue;
            }
            if (tmode != TM_DIRECT) {  // a fresh-equivalent state (see SegTask)?
                const bool idle = qhead == ai && !has_store && !has_job && !l_on && d2h_busy <= na;
                const uint64_t nx = P.tasks[w].next;
                if (tmode == TM_OUT) {
                    if (ai == nx) {
                        seg_err = !idle;
                        if (!idle) seg_why = 2;
                        stopped = true;
                        break;
                    }
                } else {
                    if (idle && (ai < nx ? nhead : ntail) < kSegPts) {
                        const uint64_t gen_tot = warp_sum_u64(a_gen);
                        if (lane == 0) {
                            SegPoint& sp = ai < nx ? P.spec[w].head[nhead] : P.spec[w].tail[ntail];
                            sp.idx = ai;
                            sp.samples = gen_tot;
                            sp.batches = r_batches;
                            sp.jobs = jc;
                            sp.nlog[0] = nl0;
                            sp.nlog[1] = nl1;
                            sp.nlog[2] = nl2;
                        }
                        if (ai < nx) ++nhead;
                        else ++ntail;
                    }
                    if (ntail == kSegPts || (ai >= P.tasks[w].xend && P.tasks[w].xend < N)) {
                        stopped = true;
                        break;
                    }
                }
            }
            h_t = na;  // LOG: this arrival's handler (its QueryArrival record comes from k_log_arrivals)
            h_seq = ai;
            h_sub = 1;
            now = na;
            ++ai;
            na = ai < N ? arr[ai] : 0.0;
            if (has_job && waiting) {  // interrupt_training_wait(true), engine.hpp:622-631
                const double waited = now - wait_since;
                add_wait(waited);
                add_busy(waited);
                waiting = false;
                ++r_pre;
                ++plan_gen;
            }
            want_serve = true;
        } else {
        if (bk == EK_NONE) break;
        now = bt;
        h_t = bt;  // LOG: the handled event; sub 0 is its own record
        h_seq = bs;
        h_sub = 1;
        if (bk == EK_SERVE) {  // the batch's last DecodeStepDone (engine.hpp:367-408)
            h_sub = 1 + s_nlast;  // after the QueryDone records of the last step
            uint64_t release = bneed;
            if (has_store && !qcompleted && src >= bfirst && src < bfirst + bn) {
                qcompleted = true;
                if (cpa) {  // prompt KV ownership moves to the slot
                    const uint32_t ps = pp[src];
                    const uint64_t keep = kv_bytes(m, ps, 1);
                    const uint64_t need_s = serving_memory(m, static_cast<uint64_t>(ps) + po[src], 1);
                    kv_held += keep;
                    prompt_kv += keep;
                    release -= need_s < keep ? need_s : keep;
                    training_peak();
                    const double ldl = P.ld ? P.ld[lo + src] : P.ld_default;
                    if (ldl >= 0.0) {
                        if (l_on) ++r_dropped;  // the superseded label is stale (see header)
                        l_on = true;
                        l_t = now + ldl;
                        l_seq = seq++;
                        l_gen = gen;
                        emit(EV_LABEL, l_t, l_seq, 0, static_cast<int64_t>(gen), qid_of(src), l_t, 0.0, 0u);
                    }
                }
            }
            led_free(release);
            r_end = now;
            want_serve = true;
        } else if (bk == EK_TRAIN) {
            tinf = false;
            add_busy(t_dur);
            emit(t_fwd ? EV_FWD : EV_BWD, t_t, t_seq, 0, t_a, t_fwd ? static_cast<int64_t>(t_pb) : 0, t_st, t_dur, 0u);
            if (t_fwd) {  // engine.hpp:693-722
                const uint64_t bytes = cur_tok * m.act_bytes_per_token_per_layer;
                if (stream && S.rec[cursor] == 0) ++r_freed;
                record(static_cast<uint32_t>(cursor), bytes, now);
                training_peak();
                ++cursor;
                if (cursor == L) {
                    ++pass_index;
                    cursor = 0;
                    if (pass_index >= npasses) {
                        phase = PH_BWD;
                        cursor = L - 1;
                        if (!preempt()) start_backward();
                    } else if (!preempt()) {
                        begin_pass();
                    }
                } else if (!preempt()) {
                    schedule_forward();
                }
            } else {  // engine.hpp:761-779, complete_job :807-813
                const uint32_t a = t_a;
                const uint8_t f = S.flg[a];
                const uint64_t r = S.rec[a];
                if (f & LF_DEV) led_free(r);
                set_layer(a, static_cast<uint8_t>((f & ~LF_DEV) | LF_CONS), r);
                if (a == 0) {
                    r_trained += jp + (cpa ? 2 * jo : 0);
                    ++r_jobs;
                    teardown();
                } else {
                    cursor = a - 1;
                    if (!preempt()) schedule_backward();
                }
            }
        } else if (bk == EK_LABEL) {  // engine.hpp:481-496
            l_on = false;
            if (has_store && gen == l_gen && has_job && phase == PH_WAIT) {
                phase = PH_READY;
                try_start_training();
            } else {
                ++r_dropped;
            }
        } else if (bk == EK_TIMEOUT) {  // engine.hpp:498-505
            to_on = false;
            if (has_store && gen == to_gen && has_job && phase == PH_WAIT) {
                emit(EV_TIMEOUT, bt, bs, 0, static_cast<int64_t>(to_gen), 0, bt, 0.0, 0u);
                ++r_dropped;
                teardown();
            }
        } else {  // EK_LOAD, engine.hpp:781-797
            const uint32_t a = S.llayer[ld_cur];
            if (LOG) {
                const double ls = P.lstart[static_cast<uint64_t>(d) * kLayerCap + ld_cur];
                emit(EV_LOAD, bt, bs, 0, a, 0, ls, bt - ls, 0u);
            }
            ++ld_cur;
            const uint64_t r = S.rec[a];
            if (!led_alloc(r)) breach = true;
            set_layer(a, static_cast<uint8_t>(S.flg[a] | LF_DEV), r);
            ++r_loads;
            if (has_job && waiting && phase == PH_BWD && cursor == a && !sbusy && qhead == ai) {
                const double waited = now - wait_since;
                add_wait(waited);
                add_busy(waited);
                waiting = false;
                schedule_backward();
            }
        }
        }
        if (want_serve) {
            want_serve = false;
            start_serving();
        }
    }

    // ---- per-device report --------------------------------------------------------
    const uint64_t g_gen = warp_sum_u64(a_gen), g_slow = warp_sum_u64(a_slow), g_slowq = warp_sum_u64(a_slowq);
    uint64_t acc[3];
    uint32_t flags = a_flags;
    {  // lane partial fixed-point sums -> one (exact)
        uint64_t a0 = a_acc[0], a1 = a_acc[1], a2 = a_acc[2];
        for (int s = 16; s > 0; s >>= 1) {
            const uint64_t b0 = __shfl_xor_sync(kFullMask, a0, s), b1 = __shfl_xor_sync(kFullMask, a1, s),
                           b2 = __shfl_xor_sync(kFullMask, a2, s);
            uint64_t t[3] = {a0, a1, a2};
            add3(t, b0, b1, b2);
            a0 = t[0];
            a1 = t[1];
            a2 = t[2];
        }
        acc[0] = a0;
        acc[1] = a1;
        acc[2] = a2;
        for (int s = 16; s > 0; s >>= 1) flags |= __shfl_xor_sync(kFullMask, flags, s);
    }
    if (spec) {
        if (lane == 0) {
            SegSpec& sp = P.spec[w];
            sp.nhead = nhead;
            sp.ntail = ntail;
            sp.err = breach || seg_err;
            sp.end.idx = stopped || breach ? ~0ull : N;
            sp.end.samples = g_gen;
            sp.end.batches = r_batches;
            sp.end.jobs = jc;
            sp.end.nlog[0] = nl0;
            sp.end.nlog[1] = nl1;
            sp.end.nlog[2] = nl2;
        }
        return;
    }
    if (tmode == TM_OUT) {  // a breach is re-run on the whole trace (its report stops there)
        const uint64_t* ex = P.tasks[w].expect;
        if (!breach && !seg_err && (r_batches != ex[0] || jc != ex[1] || nl0 != ex[2] || nl1 != ex[3] || nl2 != ex[4])) {
            seg_err = true;
            seg_why = 3;
        }
        if (breach && lane == 0) atomicOr(P.err, 8);
        if (seg_err && lane == 0) atomicOr(P.err, 16);
    } else if (breach && lane == 0) {
        atomicOr(P.err, 2);
    }
    if (__any_sync(kFullMask, unsorted) && lane == 0) atomicOr(P.err, 4);
    if (tmode == TM_DIRECT && P.job_cnt && lane == 0) P.job_cnt[d] = jc;  // every device (0 unless SeparateCluster)
    if (lane == 0 && (P.summary || tmode == TM_OUT)) {
        colo_colocated_summary r;
        r.generated_tokens = g_gen;
        r.trained_tokens = r_trained;
        r.training_busy_time = tbusy;
        r.peak_device_bytes = peak;
        r.peak_training_activation_bytes = r_ptab;
        r.preemptions = r_pre;
        r.layers_freed = r_freed;
        r.loads = r_loads;
        r.recomputes = r_recomp;
        r.copy_stall_seconds = r_stall;
        r.labels_dropped = r_dropped;
        r.prefetch_wait_seconds = r_wait;
        r.completed_jobs = r_jobs;
        r.map_fallbacks = r_fb;
        r.oom_jobs = 0;
        r.batches = r_batches;
        r.max_batch_size = r_maxb;
        r.offload_decisions = r_offd;
        r.admissions = r_adm;
        r.slow_tokens = g_slow;
        r.slow_queries = g_slowq;
        r.end_time = r_end;
        r.status = breach ? COLO_EBREACH : COLO_OK;
        r.tpt_sum[0] = acc[0];
        r.tpt_sum[1] = acc[1];
        r.tpt_sum[2] = acc[2];
        r.flags = flags;
        if (tmode == TM_OUT) {
            P.segout[w].s = r;
            P.segout[w].jobs = jc;
            P.segout[w].err = seg_why;
            P.segout[w].nlog[0] = nl0;
            P.segout[w].nlog[1] = nl1;
            P.segout[w].nlog[2] = nl2;
        } else {
            P.summary[d] = r;
        }
    }
}

// SeparateCluster trainer (engine.hpp:824-903), one thread per device, folded
// over the job stream in enqueue order.  Jobs run FIFO one at a time: a job
// starts at max(enqueue, previous job's last layer) (schedule_baseline_layer
// with trainer_free_at_, :850-858), each layer completes at the previous one's
// time + its duration (:860-872, 888, 902), and training_busy_time adds every
// layer's duration in that order (:875).  The trainer ledger peaks at the
// fixed footprint plus the largest job it ran (memory.hpp:28-35 reuse).
// SeparateCluster trainer layer events for the event log (lane 'r', b = -1,
// engine.hpp:860-877).  Their sequence numbers are not tracked (the trainer is
// folded after the serving run), so at an exactly equal time they sort after
// the serving events; times of the two timelines practically never tie.
__device__ __forceinline__ void trainer_log(const CoParams& P, uint32_t kind, double t, double t0, double dur,
                                            int64_t layer) {
    const unsigned long long i = atomicAdd(P.evcnt, 1ull);
    if (i < P.evcap) {
        EvRec r;
        r.t = t;
        r.start = t0;
        r.dur = dur;
        r.key = ((1ull << 48) - 1) << 16;
        r.a = layer;
        r.b = -1;
        r.kind = kind;
        r.gen = 1;  // trainer lane
        P.evlog[i] = r;
    }
}

__global__ void __launch_bounds__(128) k_trainer_fold(const __grid_constant__ CoParams P, const double* __restrict__ jt,
                                                      const uint32_t* __restrict__ jq) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= P.ndev) return;
    if ((P.sim_mode ? P.sim_mode[d] : COLO_SIM_COLOCATED) != COLO_SIM_SEPARATE) return;
    const CoProfile& pf = P.prof[P.dev_set[d]];
    const colo_model& m = pf.m;
    const uint64_t L = pf.L;
    const bool cpa = pf.cpa != 0;
    const uint64_t lo = P.dev_off[d], cnt = P.job_cnt[d];
    const uint64_t per_token = L * m.act_bytes_per_token_per_layer + m.kv_bytes_per_token;  // :834-835
    const uint32_t np = cpa ? 2u : 1u;  // passes: {p} (CPT) or {p+o, p+o} (CPA), :830-833
    double prev_end = 0.0, busy = 0.0;
    uint64_t trained = 0, done = 0, ptab = 0, oom = 0, maxfp = 0;
    uint64_t fd_tok = ~0ull;
    double fd = 0.0, bd = 0.0;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint32_t q = jq[lo + i];
        const double te = jt[lo + i];
        const uint64_t p = P.p[lo + q], o = P.o[lo + q];
        const uint64_t tok = cpa ? p + o : p;
        uint64_t fp = 0;
        for (uint32_t k = 0; k < np; ++k) fp += tok * per_token;
        if (fp > ptab) ptab = fp;
        if (fp > pf.budget) {  // :841-845 OOM datapoint
            ++oom;
            continue;
        }
        if (fp > maxfp) maxfp = fp;
        if (tok != fd_tok) {  // forward_layer_latency / backward sum (:864, 867-868)
            fd_tok = tok;
            fd = prefill_latency(m, tok, 1, false) / static_cast<double>(L);
            bd = 0.0;
            for (uint32_t k = 0; k < np; ++k) bd += m.backward_to_forward_ratio * fd;
        }
        double t = te < prev_end ? prev_end : te;  // std::max(now_, trainer_free_at_)
        for (uint32_t k = 0; k < np; ++k)
            for (uint64_t l = 0; l < L; ++l) {
                const double t0 = t;
                t = t + fd;
                busy += fd;
                if (P.evlog) trainer_log(P, EV_FWD, t, t0, fd, static_cast<int64_t>(l));
            }
        for (uint64_t l = 0; l < L; ++l) {
            const double t0 = t;
            t = t + bd;
            busy += bd;
            if (P.evlog) trainer_log(P, EV_BWD, t, t0, bd, static_cast<int64_t>(L - 1 - l));
        }
        prev_end = t;
        trained += cpa ? p + 2 * o : p;
        ++done;
    }
    colo_colocated_summary& r = P.summary[d];
    r.trained_tokens = trained;
    r.completed_jobs = done;
    r.training_busy_time = busy;
    r.peak_device_bytes = pf.fixed + maxfp;  // trainer_device_.peak_allocated (engine.hpp:159-161)
    r.peak_training_activation_bytes = ptab;
    r.oom_jobs = oom;
}

// Trace checks of colo_replay_serving's k_validate (workload.hpp:165-181,
// engine.hpp:70-74), one warp per device.
__global__ void __launch_bounds__(128) k_co_validate(const __grid_constant__ CoParams P) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= P.ndev) return;
    const CoProfile& pf = P.prof[P.dev_set[w]];
    const uint64_t lo = P.dev_off[w], hi = P.dev_off[w + 1];
    bool bad = false;
    for (uint64_t j = lo + lane; j < hi; j += 32) {
        const uint32_t pj = P.p[j], oj = P.o[j];
        if (pj == 0 || oj == 0) bad = true;
        else if (serving_memory(pf.m, static_cast<uint64_t>(pj) + oj, 1) > pf.budget) bad = true;
        if (j > lo && P.arr[j] < P.arr[j - 1]) bad = true;
    }
    if (__any_sync(kFullMask, bad) && lane == 0) atomicOr(P.err, 1);
}

// ---- exact sequential f64 folds of the segments' addend logs ------------------
// S_{i+1} = fl(S_i + a_i), a_i >= 0, in log order, without a sequential pass
// over every addend.  While S stays in one binade [2^e, 2^(e+1)) the grid is
// u = 2^(e-52), S is a multiple of u, and fl(S + a) = S + RN_u(a) unless
// S + a is exactly halfway between two grid points (ties-to-even then depends
// on S's last bit).  So per chunk of kFoldCh addends and per candidate binade
// e, k_fold_cand sums the integers RN_u(a)/u (a tie, a negative / NaN addend
// or a term >= 2^53 marks the candidate unusable), and k_fold_walk advances S
// over whole chunks as long as it provably stays in its binade; a chunk where
// S crosses into the next binade (a few per log), a tie, or S = 0 is folded
// addend by addend.  The logs are zero-padded to whole chunks (S + 0 = S).
constexpr int kFoldCh = 2048;
constexpr int kFoldE0 = -30;  // candidate binades e = kFoldE0 .. kFoldE0 + 63
constexpr uint64_t kFoldBad = ~0ull;

struct SegDev {  // a segmented device: its OUT tasks and its three log ranges
    uint32_t dev, t0, t1, pad;
    uint64_t lbase[3], lcnt[3];  // lcnt padded to kFoldCh
};

__global__ void __launch_bounds__(128) k_fold_cand(const double* __restrict__ log, uint64_t nchunks,
                                                   uint64_t* __restrict__ cand) {
    const uint64_t c = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (c >= nchunks) return;
    const double sc0 = ldexp(1.0, 52 - (kFoldE0 + static_cast<int>(lane)));
    const double sc1 = ldexp(1.0, 52 - (kFoldE0 + 32 + static_cast<int>(lane)));
    uint64_t acc0 = 0, acc1 = 0;
    bool bad0 = false, bad1 = false;
    const double* p = log + c * kFoldCh;
    auto term = [](double x, double sc, uint64_t& acc, bool& bad) {
        if (!(x >= 0.0)) {
            bad = true;
            return;
        }
        const double xs = x * sc;  // exact (power-of-two scaling, no overflow in range)
        if (xs >= 9007199254740992.0) {
            bad = true;
            return;
        }
        const double fl = floor(xs), fr = xs - fl;  // both exact below 2^53
        if (fr == 0.5) bad = true;
        acc += static_cast<uint64_t>(fl) + (fr > 0.5 ? 1u : 0u);
    };
    for (int i = 0; i < kFoldCh; i += 32) {
        const double v = p[i + lane];
#pragma unroll 8
        for (int t = 0; t < 32; ++t) {
            const double x = __shfl_sync(kFullMask, v, t);
            term(x, sc0, acc0, bad0);
            term(x, sc1, acc1, bad1);
        }
    }
    cand[c * 64 + lane] = bad0 ? kFoldBad : acc0;
    cand[c * 64 + 32 + lane] = bad1 ? kFoldBad : acc1;
}

// one warp per (segmented device, log): S over its chunks (see above)
__global__ void __launch_bounds__(32) k_fold_walk(const SegDev* __restrict__ devs, const double* const* logs,
                                                  const uint64_t* const* cands, double* __restrict__ out) {
    __shared__ alignas(16) double buf[128];
    const uint32_t r = blockIdx.x, lane = threadIdx.x;
    const SegDev& sd = devs[r / 3];
    const int k = static_cast<int>(r % 3);
    const double* lg = logs[k];
    const uint64_t* cd = cands[k];
    const uint64_t c0 = sd.lbase[k] / kFoldCh, c1 = c0 + sd.lcnt[k] / kFoldCh;
    double S = 0.0;
    uint64_t c = c0;
    while (c < c1) {
        int e = 0;
        bool whole = false;
        if (S > 0.0) {
            e = ilogb(S);
            whole = e >= kFoldE0 && e < kFoldE0 + 64;
        }
        uint32_t took = 0;
        if (whole) {  // as many whole chunks as stay in S's binade
            const uint32_t idx = static_cast<uint32_t>(e - kFoldE0);
            const double u = ldexp(1.0, e - 52);
            const uint64_t m = static_cast<uint64_t>(S / u);  // S's significand, in [2^52, 2^53)
            const uint64_t room = (1ull << 53) - m;          // S + T*u < 2^(e+1)  <=>  T < room
            const uint64_t cc = c + lane;
            uint64_t t = cc < c1 ? cd[cc * 64 + idx] : kFoldBad;
            bool ok = t != kFoldBad;
            uint64_t pre = ok ? t : 0;  // inclusive prefix, saturating at 2^53
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const uint64_t y = __shfl_up_sync(kFullMask, pre, s);
                const bool yo = __shfl_up_sync(kFullMask, ok, s);
                if (lane >= static_cast<uint32_t>(s)) {
                    pre = min(pre + y, static_cast<uint64_t>(1ull << 53));
                    ok = ok && yo;
                }
            }
            ok = ok && pre < room;
            took = __popc(__ballot_sync(kFullMask, ok));  // leading lanes (ok is monotone)
            if (took) {
                const uint64_t T = __shfl_sync(kFullMask, pre, took - 1);
                S = S + static_cast<double>(T) * u;  // exact: a multiple of u below 2^(e+1)
                c += took;
            }
        }
        if (!took) {  // addend by addend
            const double* p = lg + c * kFoldCh;
            for (int i = 0; i < kFoldCh; i += 128) {
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 4; ++q) buf[q * 32 + lane] = p[i + q * 32 + lane];
                __syncwarp();
                if (lane == 0) S = chain_fold(S, buf, 128);
                S = __shfl_sync(kFullMask, S, 0);
            }
            ++c;
        }
    }
    if (lane == 0) out[r] = S;
}

// one warp per segmented device: its OUT segments' partial reports -> the report
__global__ void __launch_bounds__(32) k_seg_combine(const __grid_constant__ CoParams P, const SegDev* __restrict__ devs,
                                                    const double* __restrict__ folds) {
    const SegDev& sd = devs[blockIdx.x];
    const uint32_t lane = threadIdx.x;
    uint64_t gen = 0, trained = 0, peak = 0, ptab = 0, pre = 0, freed = 0, loads = 0, recomp = 0, dropped = 0, jobs = 0,
             fb = 0, oom = 0, batches = 0, maxb = 0, offd = 0, adm = 0, slow = 0, slowq = 0, njobs = 0;
    uint64_t acc[3] = {0, 0, 0};
    uint64_t flags = 0;
    double end = 0.0;
    for (uint32_t t = sd.t0 + lane; t < sd.t1; t += 32) {
        const colo_colocated_summary& s = P.segout[t].s;
        gen += s.generated_tokens;
        trained += s.trained_tokens;
        peak = max(peak, s.peak_device_bytes);
        ptab = max(ptab, s.peak_training_activation_bytes);
        pre += s.preemptions;
        freed += s.layers_freed;
        loads += s.loads;
        recomp += s.recomputes;
        dropped += s.labels_dropped;
        jobs += s.completed_jobs;
        fb += s.map_fallbacks;
        oom += s.oom_jobs;
        batches += s.batches;
        maxb = max(maxb, s.max_batch_size);
        offd += s.offload_decisions;
        adm += s.admissions;
        slow += s.slow_tokens;
        slowq += s.slow_queries;
        end = dmax(end, s.end_time);
        add3(acc, s.tpt_sum[0], s.tpt_sum[1], s.tpt_sum[2]);
        flags |= s.flags;
        njobs += P.segout[t].jobs;
    }
    gen = warp_sum_u64(gen);
    trained = warp_sum_u64(trained);
    peak = warp_max_u64(peak);
    ptab = warp_max_u64(ptab);
    pre = warp_sum_u64(pre);
    freed = warp_sum_u64(freed);
    loads = warp_sum_u64(loads);
    recomp = warp_sum_u64(recomp);
    dropped = warp_sum_u64(dropped);
    jobs = warp_sum_u64(jobs);
    fb = warp_sum_u64(fb);
    oom = warp_sum_u64(oom);
    batches = warp_sum_u64(batches);
    maxb = warp_max_u64(maxb);
    offd = warp_sum_u64(offd);
    adm = warp_sum_u64(adm);
    slow = warp_sum_u64(slow);
    slowq = warp_sum_u64(slowq);
    njobs = warp_sum_u64(njobs);
    end = warp_max_f64(end);
    for (int s = 16; s > 0; s >>= 1) {
        const uint64_t b0 = __shfl_xor_sync(kFullMask, acc[0], s), b1 = __shfl_xor_sync(kFullMask, acc[1], s),
                       b2 = __shfl_xor_sync(kFullMask, acc[2], s);
        add3(acc, b0, b1, b2);
        flags |= __shfl_xor_sync(kFullMask, flags, s);
    }
    if (lane) return;
    if (P.job_cnt) P.job_cnt[sd.dev] = njobs;
    if (!P.summary) return;
    colo_colocated_summary r;
    r.generated_tokens = gen;
    r.trained_tokens = trained;
    r.training_busy_time = folds[blockIdx.x * 3 + 0];
    r.peak_device_bytes = peak;
    r.peak_training_activation_bytes = ptab;
    r.preemptions = pre;
    r.layers_freed = freed;
    r.loads = loads;
    r.recomputes = recomp;
    r.copy_stall_seconds = folds[blockIdx.x * 3 + 1];
    r.labels_dropped = dropped;
    r.prefetch_wait_seconds = folds[blockIdx.x * 3 + 2];
    r.completed_jobs = jobs;
    r.map_fallbacks = fb;
    r.oom_jobs = oom;
    r.batches = batches;
    r.max_batch_size = maxb;
    r.offload_decisions = offd;
    r.admissions = adm;
    r.slow_tokens = slow;
    r.slow_queries = slowq;
    r.end_time = end;
    r.status = COLO_OK;
    r.tpt_sum[0] = acc[0];
    r.tpt_sum[1] = acc[1];
    r.tpt_sum[2] = acc[2];
    r.flags = flags;
    P.summary[sd.dev] = r;
}

// QueryArrival records (engine.hpp:270-276): state-independent, one per query
__global__ void k_log_arrivals(const double* __restrict__ arr, const uint64_t* __restrict__ qid, uint64_t n,
                               EvRec* __restrict__ out) {
    for (uint64_t q = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        EvRec r;
        r.t = arr[q];
        r.start = arr[q];
        r.dur = 0.0;
        r.key = q << 16;
        r.a = static_cast<int64_t>(qid ? qid[q] : q);
        r.b = 0;
        r.kind = EV_ARRIVAL;
        r.gen = 0;
        out[q] = r;
    }
}

size_t align256c(size_t x) { return (x + 255) & ~size_t(255); }

colo_status grow_scratch(colo_ctx* ctx, size_t bytes) {
    ctx->rs_valid = false;  // the serving replay's entry states share this buffer
    if (ctx->rscratch_bytes >= bytes) return COLO_OK;
    if (ctx->d_rscratch) cudaFree(ctx->d_rscratch);
    ctx->d_rscratch = nullptr;
    ctx->rscratch_bytes = 0;
    COLO_CK(ctx, cudaMalloc(&ctx->d_rscratch, bytes));
    ctx->rscratch_bytes = bytes;
    return COLO_OK;
}

colo_status grow_buf(colo_ctx* ctx, void*& p, size_t& cap, size_t bytes) {
    if (cap >= bytes) return COLO_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    COLO_CK(ctx, cudaMalloc(&p, bytes));
    cap = bytes;
    return COLO_OK;
}

colo_status launch_co(colo_ctx* ctx, const CoParams& Q, size_t nwarps, int& flag) {
    COLO_CK(ctx, cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
    const uint32_t blocks = static_cast<uint32_t>((nwarps + kWarpsC - 1) / kWarpsC);
    COLO_LAUNCHED(ctx);
    if (Q.tasks) k_colocated<true><<<blocks, kWarpsC * 32, 0, ctx->stream>>>(Q);
    else k_colocated<false><<<blocks, kWarpsC * 32, 0, ctx->stream>>>(Q);
    COLO_CK(ctx, cudaGetLastError());
    COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

// Every device's run: one warp per device, or -- when there are too few
// devices to fill the GPU -- long devices in parallel segments (see SegTask):
// speculate, resolve the entry arrivals here, replay the segments with their
// outputs, fold the f64 sums, combine the partial reports.  A device whose
// segments do not resolve (no common idle arrival, e.g. a server that never
// drains) or whose replay breaches runs whole.  seg_len: 0 = automatic,
// 0xffffffff = never, else the segment length in queries.
colo_status run_devices(colo_ctx* ctx, CoParams P, const std::vector<uint64_t>& off,
                        const std::vector<uint8_t>& smode, size_t n, uint32_t seg_len, int& flag) {
    const size_t ndev = P.ndev;
    flag = 0;
    const size_t W = static_cast<size_t>(std::max(ctx->sm_count, 1)) * 8;  // resident warps
    uint64_t L = 0;
    if (seg_len == 0) {
        if (ndev < W) L = std::max<uint64_t>(512, (n + 4 * W - 1) / (4 * W));
    } else if (seg_len != 0xffffffffu) {
        L = seg_len;
    }
    std::vector<uint32_t> sdevs;
    for (size_t d = 0; L && d < ndev; ++d) {
        const uint64_t nd = off[d + 1] - off[d];
        if (seg_len == 0 ? nd >= 4 * L : nd > L) sdevs.push_back(static_cast<uint32_t>(d));
    }
    if (sdevs.empty()) return launch_co(ctx, P, ndev, flag);

    // ---- speculate ----
    const uint64_t ext = std::max<uint64_t>(L, 2048);
    std::vector<SegTask> t1;
    std::vector<size_t> sfirst(sdevs.size());
    std::vector<char> isseg(ndev, 0);
    bool seg_separate = false;
    for (size_t i = 0; i < sdevs.size(); ++i) {
        const uint32_t d = sdevs[i];
        const uint64_t nd = off[d + 1] - off[d];
        isseg[d] = 1;
        seg_separate |= smode[d] == COLO_SIM_SEPARATE;
        sfirst[i] = t1.size();
        for (uint64_t s0 = 0; s0 < nd; s0 += L) {
            SegTask t{};
            t.dev = d;
            t.mode = TM_SPEC;
            t.start = s0;
            t.next = std::min(nd, s0 + L);
            t.xend = t.next < nd ? std::min(nd, t.next + ext) : nd;
            t1.push_back(t);
        }
    }
    const size_t nspec = t1.size();
    for (size_t d = 0; d < ndev; ++d)
        if (!isseg[d]) {
            SegTask t{};
            t.dev = static_cast<uint32_t>(d);
            t.mode = TM_DIRECT;
            t1.push_back(t);
        }
    const size_t nsd = sdevs.size();
    const size_t maxt = nspec + ndev;
    size_t b = 0;
    const size_t o_task = b;
    b += align256c(maxt * sizeof(SegTask));
    const size_t o_spec = b;
    b += align256c(nspec * sizeof(SegSpec));
    const size_t o_out = b;
    b += align256c(nspec * sizeof(SegOut));
    const size_t o_sdv = b;
    b += align256c(nsd * sizeof(SegDev));
    const size_t o_fold = b;
    b += align256c(nsd * 3 * sizeof(double));
    const size_t o_ptr = b;
    b += align256c(6 * sizeof(void*));
    {
        const colo_status st = grow_buf(ctx, ctx->d_seg, ctx->seg_bytes, b);
        if (st != COLO_OK) return st;
    }
    auto* base = static_cast<uint8_t*>(ctx->d_seg);
    auto* d_task = reinterpret_cast<SegTask*>(base + o_task);
    auto* d_spec = reinterpret_cast<SegSpec*>(base + o_spec);
    auto* d_out = reinterpret_cast<SegOut*>(base + o_out);
    auto* d_sdv = reinterpret_cast<SegDev*>(base + o_sdv);
    auto* d_fold = reinterpret_cast<double*>(base + o_fold);
    auto* d_ptr = reinterpret_cast<void**>(base + o_ptr);
    COLO_CK(ctx, cudaMemcpyAsync(d_task, t1.data(), t1.size() * sizeof(SegTask), cudaMemcpyHostToDevice, ctx->stream));
    CoParams P1 = P;
    P1.tasks = d_task;
    P1.ntasks = static_cast<uint32_t>(t1.size());
    P1.spec = d_spec;
    int f1 = 0;
    {
        const colo_status st = launch_co(ctx, P1, t1.size(), f1);
        if (st != COLO_OK) return st;
    }
    std::vector<SegSpec> sp(nspec);
    COLO_CK(ctx, cudaMemcpyAsync(sp.data(), d_spec, nspec * sizeof(SegSpec), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));

    // ---- resolve: b_0 = 0, b_j = first arrival idle in tail(j-1) and head(j) ----
    std::vector<SegTask> t2;
    std::vector<SegDev> sdv;
    std::vector<uint32_t> whole;
    uint64_t LB[3] = {0, 0, 0};
    for (size_t i = 0; i < nsd; ++i) {
        const uint32_t d = sdevs[i];
        const uint64_t nd = off[d + 1] - off[d];
        const SegSpec* S = sp.data() + sfirst[i];
        const size_t ns = static_cast<size_t>((nd + L - 1) / L);
        std::vector<uint64_t> bj(ns, 0);
        std::vector<SegPoint> ph(ns), pt(ns);
        bool ok = !S[0].err && S[0].nhead > 0 && S[0].head[0].idx == 0;
        if (ok) ph[0] = S[0].head[0];
        size_t used = ns;  // segments that replay (the last one may run to the end of the trace)
        for (size_t j = 1; ok && j < ns; ++j) {
            const SegSpec &A = S[j - 1], &B = S[j];
            if (A.end.idx == nd && !A.err) {
                // segment j-1's own run reached the end of the trace: it is the truth up to there
                used = j;
                break;
            }
            if (B.err) {
                ok = false;
                break;
            }
            uint32_t ia = 0, ib = 0;
            bool found = false;
            while (ia < A.ntail && ib < B.nhead) {
                if (A.tail[ia].idx == B.head[ib].idx) {
                    found = true;
                    break;
                }
                if (A.tail[ia].idx < B.head[ib].idx) ++ia;
                else ++ib;
            }
            if (!found) {
                ok = false;
                break;
            }
            bj[j] = B.head[ib].idx;
            pt[j - 1] = A.tail[ia];
            ph[j] = B.head[ib];
        }
        if (ok) {
            const SegPoint& E = S[used - 1].end;
            if (E.idx != nd) ok = false;
            else pt[used - 1] = E;
        }
        if (!ok) {
            if (std::getenv("COLO_SEG_DEBUG")) {
                size_t j = 0;
                while (j < ns && !S[j].err) ++j;
                std::fprintf(stderr, "seg dev %u: %zu segments, unresolved; first err seg %zu\n", d, ns, j);
                for (size_t q = ns > 4 ? ns - 3 : 0; q < ns; ++q) {
                    std::fprintf(stderr, "  seg %zu err %u nhead %u ntail %u end %llu head:", q, S[q].err, S[q].nhead,
                                 S[q].ntail, static_cast<unsigned long long>(S[q].end.idx));
                    for (uint32_t h = 0; h < std::min<uint32_t>(S[q].nhead, 8); ++h)
                        std::fprintf(stderr, " %llu", static_cast<unsigned long long>(S[q].head[h].idx));
                    std::fprintf(stderr, " tail:");
                    for (uint32_t h = 0; h < std::min<uint32_t>(S[q].ntail, 8); ++h)
                        std::fprintf(stderr, " %llu", static_cast<unsigned long long>(S[q].tail[h].idx));
                    std::fprintf(stderr, "\n");
                }
            }
            whole.push_back(d);
            continue;
        }
        SegDev sd{};
        sd.dev = d;
        sd.t0 = static_cast<uint32_t>(t2.size());
        uint64_t bb = 0, jb = 0, sb = 0, lb[3] = {LB[0], LB[1], LB[2]};
        for (size_t j = 0; j < used; ++j) {
            SegTask t{};
            t.dev = d;
            t.mode = TM_OUT;
            t.start = bj[j];
            t.next = j + 1 < used ? bj[j + 1] : nd;
            t.batch_base = bb;
            t.job_base = jb;
            t.sample_base = sb;
            t.expect[0] = pt[j].batches - ph[j].batches;
            t.expect[1] = pt[j].jobs - ph[j].jobs;
            for (int k = 0; k < 3; ++k) {
                t.log_base[k] = lb[k];
                t.expect[2 + k] = pt[j].nlog[k] - ph[j].nlog[k];
                lb[k] += t.expect[2 + k];
            }
            bb += t.expect[0];
            jb += t.expect[1];
            sb += pt[j].samples - ph[j].samples;
            t2.push_back(t);
        }
        sd.t1 = static_cast<uint32_t>(t2.size());
        for (int k = 0; k < 3; ++k) {
            sd.lbase[k] = LB[k];
            sd.lcnt[k] = (lb[k] - LB[k] + kFoldCh - 1) / kFoldCh * kFoldCh;
            LB[k] += sd.lcnt[k];
        }
        sdv.push_back(sd);
    }
    for (uint32_t d : whole) {
        SegTask t{};
        t.dev = d;
        t.mode = TM_DIRECT;
        t2.push_back(t);
    }

    // ---- replay the segments with outputs ----
    const size_t nlog = LB[0] + LB[1] + LB[2], nch = nlog / kFoldCh;
    {
        const colo_status st =
            grow_buf(ctx, ctx->d_seglog, ctx->seglog_bytes, std::max<size_t>(nlog * 8 + nch * 64 * 8, 256));
        if (st != COLO_OK) return st;
    }
    auto* logs = static_cast<double*>(ctx->d_seglog);
    auto* cands = reinterpret_cast<uint64_t*>(logs + nlog);
    if (nlog) COLO_CK(ctx, cudaMemsetAsync(logs, 0, nlog * 8, ctx->stream));
    const double* lp[3] = {logs, logs + LB[0], logs + LB[0] + LB[1]};
    const uint64_t* cp[3] = {cands, cands + LB[0] / kFoldCh * 64, cands + (LB[0] + LB[1]) / kFoldCh * 64};
    const void* ptrs[6] = {lp[0], lp[1], lp[2], cp[0], cp[1], cp[2]};
    COLO_CK(ctx, cudaMemcpyAsync(d_ptr, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, ctx->stream));
    if (!sdv.empty())
        COLO_CK(ctx, cudaMemcpyAsync(d_sdv, sdv.data(), sdv.size() * sizeof(SegDev), cudaMemcpyHostToDevice, ctx->stream));
    int f2 = 0;
    CoParams P2 = P;
    if (!t2.empty()) {
        COLO_CK(ctx, cudaMemcpyAsync(d_task, t2.data(), t2.size() * sizeof(SegTask), cudaMemcpyHostToDevice, ctx->stream));
        P2.tasks = d_task;
        P2.ntasks = static_cast<uint32_t>(t2.size());
        P2.segout = d_out;
        for (int k = 0; k < 3; ++k) P2.log[k] = const_cast<double*>(lp[k]);
        const colo_status st = launch_co(ctx, P2, t2.size(), f2);
        if (st != COLO_OK) return st;
    }
    if (f2 & 16) {
        if (std::getenv("COLO_SEG_DEBUG")) {
            std::vector<SegOut> so(t2.size());
            cudaMemcpy(so.data(), d_out, t2.size() * sizeof(SegOut), cudaMemcpyDeviceToHost);
            int shown = 0;
            for (size_t t = 0; t < t2.size() && shown < 6; ++t) {
                if (t2[t].mode != TM_OUT || !so[t].err) continue;
                ++shown;
                const SegTask& k = t2[t];
                std::fprintf(stderr,
                             "out task %zu dev %u [%llu, %llu) err %llu: batches %llu/%llu jobs %llu/%llu log %llu/%llu "
                             "%llu/%llu %llu/%llu\n",
                             t, k.dev, (unsigned long long)k.start, (unsigned long long)k.next,
                             (unsigned long long)so[t].err, (unsigned long long)so[t].s.batches,
                             (unsigned long long)k.expect[0], (unsigned long long)so[t].jobs,
                             (unsigned long long)k.expect[1], (unsigned long long)so[t].nlog[0],
                             (unsigned long long)k.expect[2], (unsigned long long)so[t].nlog[1],
                             (unsigned long long)k.expect[3], (unsigned long long)so[t].nlog[2],
                             (unsigned long long)k.expect[4]);
            }
        }
        return set_err(ctx, COLO_ECUDA, "colocated replay: a segment disagreed with its speculation (internal)");
    }
    if (!sdv.empty()) {
        for (int k = 0; k < 3; ++k) {
            const uint64_t c = LB[k] / kFoldCh;
            if (c) COLO_LAUNCHED(ctx);
            if (c) k_fold_cand<<<static_cast<uint32_t>((c * 32 + 127) / 128), 128, 0, ctx->stream>>>(lp[k], c,
                                                                                                   const_cast<uint64_t*>(cp[k]));
        }
        COLO_LAUNCHED(ctx);
        k_fold_walk<<<static_cast<uint32_t>(sdv.size() * 3), 32, 0, ctx->stream>>>(
            d_sdv, reinterpret_cast<const double* const*>(d_ptr), reinterpret_cast<const uint64_t* const*>(d_ptr + 3),
            d_fold);
        COLO_LAUNCHED(ctx);
        k_seg_combine<<<static_cast<uint32_t>(sdv.size()), 32, 0, ctx->stream>>>(P2, d_sdv, d_fold);
        COLO_CK(ctx, cudaGetLastError());
    }
    int f3 = 0;
    if (f2 & 8) {  // a segment breached: those devices run whole (the report stops at the breach)
        std::vector<SegOut> so(t2.size());
        COLO_CK(ctx, cudaMemcpyAsync(so.data(), d_out, t2.size() * sizeof(SegOut), cudaMemcpyDeviceToHost, ctx->stream));
        COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<SegTask> t3;
        for (const SegDev& sd : sdv) {
            bool br = false;
            for (uint32_t t = sd.t0; t < sd.t1; ++t) br |= so[t].s.status == COLO_EBREACH;
            if (br) {
                SegTask t{};
                t.dev = sd.dev;
                t.mode = TM_DIRECT;
                t3.push_back(t);
            }
        }
        COLO_CK(ctx, cudaMemcpyAsync(d_task, t3.data(), t3.size() * sizeof(SegTask), cudaMemcpyHostToDevice, ctx->stream));
        CoParams P3 = P;
        P3.tasks = d_task;
        P3.ntasks = static_cast<uint32_t>(t3.size());
        const colo_status st = launch_co(ctx, P3, t3.size(), f3);
        if (st != COLO_OK) return st;
    }
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    flag = f1 | (f2 & ~8) | f3;
    if (seg_separate) flag |= 4;  // enqueue order across segments is not checked: sort (stable, so exact)
    return COLO_OK;
}

}  // namespace

extern "C" {

colo_status colo_replay_colocated(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const double* d_arrival,
                                  const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                  const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev,
                                  const colo_colocated_opts* opts) {
    if (!ctx || !sets || !opts || nsets == 0 || nsets > kMaxSets || !d_dev_offsets || !d_dev_set) return COLO_EINVAL;
    if (ndev == 0) return COLO_OK;
    if (n && (!d_arrival || !d_prompt || !d_output)) return COLO_EINVAL;
    if (opts->d_samples && !opts->d_sample_offsets) return set_err(ctx, COLO_EINVAL, "samples need d_sample_offsets");
    if (opts->d_hist && (opts->nfilters == 0 || opts->nfilters > 3)) return set_err(ctx, COLO_EINVAL, "nfilters 1..3");
    if (!(opts->cache_timeout == opts->cache_timeout)) return set_err(ctx, COLO_EINVAL, "cache_timeout is NaN");
    CoParams P{};
    for (size_t i = 0; i < nsets; ++i) {
        const colo_mapset* ms = sets[i];
        if (!ms) return set_err(ctx, COLO_EINVAL, "null map set");
        const colo_status st = colo_validate_profile_pair(&ms->m, &ms->g);
        if (st != COLO_OK) return set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
        if (ms->hash != colo_profile_hash(&ms->m, &ms->g))
            return set_err(ctx, COLO_EVALIDATION, "sim config: map profile hash does not match the profiles");
        if (ms->m.num_layers > kMaxLayers) return set_err(ctx, COLO_EINVAL, "num_layers > 253");
        CoProfile& pf = P.prof[i];
        pf.m = ms->m;
        pf.cap = ms->g.capacity_bytes;
        pf.budget = ms->g.capacity_bytes - ms->g.runtime_reserve_bytes - ms->m.weights_bytes;
        pf.fixed = ms->m.weights_bytes + ms->g.runtime_reserve_bytes;
        pf.h2d = ms->g.h2d_bandwidth;
        pf.d2h = ms->g.d2h_bandwidth;
        pf.cpa = ms->mode == COLO_CPA ? 1u : 0u;
        pf.L = static_cast<uint32_t>(ms->m.num_layers);
        P.sets[i] = make_view(ms);
    }
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    std::vector<uint64_t> off(ndev + 1);
    std::vector<uint16_t> dset(ndev);
    COLO_CK(ctx, cudaMemcpyAsync(off.data(), d_dev_offsets, (ndev + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaMemcpyAsync(dset.data(), d_dev_set, ndev * 2, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (off[0] != 0 || off[ndev] != n) return set_err(ctx, COLO_EINVAL, "device offsets must span [0, n]");
    std::vector<uint8_t> smode(ndev, COLO_SIM_COLOCATED);
    if (opts->d_dev_sim_mode) {
        COLO_CK(ctx, cudaMemcpyAsync(smode.data(), opts->d_dev_sim_mode, ndev, cudaMemcpyDeviceToHost, ctx->stream));
        COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    bool any_separate = false;
    for (size_t d = 0; d < ndev; ++d) {
        if (off[d + 1] < off[d]) return set_err(ctx, COLO_EINVAL, "device offsets not monotone");
        if (dset[d] >= nsets) return set_err(ctx, COLO_EINVAL, "device map-set index out of range");
        if (off[d + 1] - off[d] >= (1ull << 31)) return set_err(ctx, COLO_EINVAL, "2^31 or more queries on a device");
        if (smode[d] > COLO_SIM_SEPARATE) return set_err(ctx, COLO_EINVAL, "sim mode must be 0, 1 or 2");
        any_separate |= smode[d] == COLO_SIM_SEPARATE;
    }
    P.arr = d_arrival;
    P.p = d_prompt;
    P.o = d_output;
    P.ld = opts->d_label_delay;
    P.ld_default = opts->default_label_delay;
    P.dev_off = d_dev_offsets;
    P.dev_set = d_dev_set;
    P.ndev = static_cast<uint32_t>(ndev);
    P.timeout = opts->cache_timeout;
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
    P.sim_mode = opts->d_dev_sim_mode;
    // SeparateCluster job streams: (enqueue time, query) per device + sort buffers
    size_t o_jt = 0, o_jq = 0, o_jc = 0, o_jt2 = 0, o_jq2 = 0, o_beg = 0, o_end = 0, o_tmp = 0, tmp_bytes = 0;
    if (any_separate) {
        size_t b = 0;
        o_jt = b;
        b += align256c(n * 8 + 8);
        o_jq = b;
        b += align256c(n * 4 + 8);
        o_jc = b;
        b += align256c(ndev * 8 + 8);
        o_jt2 = b;
        b += align256c(n * 8 + 8);
        o_jq2 = b;
        b += align256c(n * 4 + 8);
        o_beg = b;
        b += align256c(ndev * 8 + 8);
        o_end = b;
        b += align256c(ndev * 8 + 8);
        // cub temp storage for a segmented stable sort of up to n items
        int ni = static_cast<int>(std::min<size_t>(n, (1u << 31) - 1));
        cub::DeviceSegmentedSort::StableSortPairs(nullptr, tmp_bytes, static_cast<const double*>(nullptr),
                                                  static_cast<double*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                                  static_cast<uint32_t*>(nullptr), ni, static_cast<int>(ndev),
                                                  static_cast<const uint64_t*>(nullptr),
                                                  static_cast<const uint64_t*>(nullptr), ctx->stream);
        o_tmp = b;
        b += align256c(tmp_bytes + 8);
        const colo_status st = grow_scratch(ctx, b);
        if (st != COLO_OK) return st;
        auto* base = static_cast<uint8_t*>(ctx->d_rscratch);
        P.job_t = reinterpret_cast<double*>(base + o_jt);
        P.job_q = reinterpret_cast<uint32_t*>(base + o_jq);
        P.job_cnt = reinterpret_cast<uint64_t*>(base + o_jc);
    }
    COLO_CK(ctx, cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream));
    const uint32_t vblocks = static_cast<uint32_t>((ndev + 3) / 4);
    COLO_LAUNCHED(ctx);
    k_co_validate<<<vblocks, 128, 0, ctx->stream>>>(P);
    int flag = 0;
    COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (flag)
        return set_err(ctx, COLO_EVALIDATION,
                       "trace rejected: unsorted arrivals, zero tokens, or a query that cannot fit the device alone");
    {
        const colo_status st = run_devices(ctx, P, off, smode, n, opts->seg_len, flag);
        if (st != COLO_OK) return st;
    }
    if (any_separate && P.summary) {
        const double* jt = P.job_t;
        const uint32_t* jq = P.job_q;
        if (flag & 4) {  // label delays vary: stable sort of each device's jobs by enqueue time (ties keep finish order)
            auto* base = static_cast<uint8_t*>(ctx->d_rscratch);
            std::vector<uint64_t> cnt(ndev), beg(ndev), end(ndev);
            COLO_CK(ctx, cudaMemcpyAsync(cnt.data(), P.job_cnt, ndev * 8, cudaMemcpyDeviceToHost, ctx->stream));
            COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
            for (size_t d = 0; d < ndev; ++d) {
                beg[d] = off[d];
                end[d] = off[d] + cnt[d];
            }
            COLO_CK(ctx, cudaMemcpyAsync(base + o_beg, beg.data(), ndev * 8, cudaMemcpyHostToDevice, ctx->stream));
            COLO_CK(ctx, cudaMemcpyAsync(base + o_end, end.data(), ndev * 8, cudaMemcpyHostToDevice, ctx->stream));
            // device groups below 2^31 items (cub's int item count)
            size_t d0 = 0;
            while (d0 < ndev) {
                size_t d1 = d0 + 1;
                while (d1 < ndev && off[d1 + 1] - off[d0] < (1ull << 31)) ++d1;
                const uint64_t gb = off[d0];
                std::vector<uint64_t> gbeg(d1 - d0), gend(d1 - d0);
                for (size_t d = d0; d < d1; ++d) {
                    gbeg[d - d0] = beg[d] - gb;
                    gend[d - d0] = end[d] - gb;
                }
                COLO_CK(ctx, cudaMemcpyAsync(base + o_beg, gbeg.data(), gbeg.size() * 8, cudaMemcpyHostToDevice,
                                             ctx->stream));
                COLO_CK(ctx, cudaMemcpyAsync(base + o_end, gend.data(), gend.size() * 8, cudaMemcpyHostToDevice,
                                             ctx->stream));
                size_t tb = tmp_bytes;
                COLO_CK(ctx, cub::DeviceSegmentedSort::StableSortPairs(
                                 base + o_tmp, tb, P.job_t + gb, reinterpret_cast<double*>(base + o_jt2) + gb,
                                 P.job_q + gb, reinterpret_cast<uint32_t*>(base + o_jq2) + gb,
                                 static_cast<int>(off[d1] - gb), static_cast<int>(d1 - d0),
                                 reinterpret_cast<const uint64_t*>(base + o_beg),
                                 reinterpret_cast<const uint64_t*>(base + o_end), ctx->stream));
                COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));  // the offset arrays are reused per group
                d0 = d1;
            }
            jt = reinterpret_cast<const double*>(base + o_jt2);
            jq = reinterpret_cast<const uint32_t*>(base + o_jq2);
        }
        COLO_LAUNCHED(ctx);
        k_trainer_fold<<<static_cast<uint32_t>((ndev + 127) / 128), 128, 0, ctx->stream>>>(P, jt, jq);
        COLO_CK(ctx, cudaGetLastError());
        COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    if (flag & 2) return set_err(ctx, COLO_EBREACH, "colocated replay: invariant breach on at least one device");
    return COLO_OK;
}

int64_t colo_colocated_events(colo_ctx* ctx, const colo_mapset* set, int sim_mode, double cache_timeout,
                              const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output,
                              const double* d_label_delay, double default_label_delay, const uint64_t* d_query_id,
                              size_t n, double tau) {
    if (!ctx || !set || (n && (!d_arrival || !d_prompt || !d_output))) return -COLO_EINVAL;
    if (sim_mode < COLO_SIM_SERVING_ONLY || sim_mode > COLO_SIM_SEPARATE)
        return -set_err(ctx, COLO_EINVAL, "event log: sim mode must be 0, 1 or 2");
    if (n >= (1ull << 40)) return -set_err(ctx, COLO_EINVAL, "event log: trace too long");
    ctx->evtext.clear();
    {
        const colo_status st = colo_validate_profile_pair(&set->m, &set->g);
        if (st != COLO_OK) return -set_err(ctx, st, "profile pair rejected (profiles.hpp:129-134)");
    }
    if (set->hash != colo_profile_hash(&set->m, &set->g))
        return -set_err(ctx, COLO_EVALIDATION, "sim config: map profile hash does not match the profiles");
    if (set->m.num_layers > kMaxLayers) return -set_err(ctx, COLO_EINVAL, "num_layers > 253");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return -cuda_err(ctx, cudaGetLastError(), "cudaSetDevice");
    CoParams P{};
    CoProfile& pf = P.prof[0];
    pf.m = set->m;
    pf.cap = set->g.capacity_bytes;
    pf.budget = set->g.capacity_bytes - set->g.runtime_reserve_bytes - set->m.weights_bytes;
    pf.fixed = set->m.weights_bytes + set->g.runtime_reserve_bytes;
    pf.h2d = set->g.h2d_bandwidth;
    pf.d2h = set->g.d2h_bandwidth;
    pf.cpa = set->mode == COLO_CPA ? 1u : 0u;
    pf.L = static_cast<uint32_t>(set->m.num_layers);
    P.sets[0] = make_view(set);
    // device scratch: offsets, set index, mode, lstart, then the records
    size_t cap = n * 8 + 65536;  // records (grown and re-run when the run logs more)
    for (int attempt = 0; attempt < 4; ++attempt) {
        const size_t o_off = 0, o_set = 64, o_mode = 128, o_ls = 256, o_sum = o_ls + align256c(kLayerCap * 8),
                     o_jc = o_sum + align256c(sizeof(colo_colocated_summary)), o_jt = o_jc + 256,
                     o_jq = o_jt + align256c(n * 8 + 8), o_jt2 = o_jq + align256c(n * 4 + 8),
                     o_jq2 = o_jt2 + align256c(n * 8 + 8), o_tmp = o_jq2 + align256c(n * 4 + 8);
        size_t tb = 0;
        if (sim_mode == COLO_SIM_SEPARATE && n)
            cub::DeviceRadixSort::SortPairs(nullptr, tb, static_cast<const double*>(nullptr), static_cast<double*>(nullptr),
                                            static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                            static_cast<int>(n), 0, 64, ctx->stream);
        const size_t o_ev = o_tmp + align256c(tb + 8);
        const size_t bytes = o_ev + (n + cap) * sizeof(EvRec);
        {
            const colo_status st = grow_buf(ctx, ctx->d_seglog, ctx->seglog_bytes, bytes);
            if (st != COLO_OK) return -st;
        }
        auto* base = static_cast<uint8_t*>(ctx->d_seglog);
        const uint64_t off[2] = {0, n};
        const uint16_t dset = 0;
        const uint8_t md = static_cast<uint8_t>(sim_mode);
        if (cudaMemcpyAsync(base + o_off, off, 16, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaMemcpyAsync(base + o_set, &dset, 2, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaMemcpyAsync(base + o_mode, &md, 1, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
            return -cuda_err(ctx, cudaGetLastError(), "event log setup");
        P.arr = d_arrival;
        P.p = d_prompt;
        P.o = d_output;
        P.ld = d_label_delay;
        P.ld_default = default_label_delay;
        P.dev_off = reinterpret_cast<const uint64_t*>(base + o_off);
        P.dev_set = reinterpret_cast<const uint16_t*>(base + o_set);
        P.sim_mode = base + o_mode;
        P.ndev = 1;
        P.timeout = cache_timeout;
        P.tau = tau;
        P.err = ctx->d_flag;
        P.qid = d_query_id;
        P.lstart = reinterpret_cast<double*>(base + o_ls);
        P.evlog = reinterpret_cast<EvRec*>(base + o_ev);
        P.evcap = n + cap;
        if (sim_mode == COLO_SIM_SEPARATE) {  // the job stream and the trainer's report slot
            P.job_t = reinterpret_cast<double*>(base + o_jt);
            P.job_q = reinterpret_cast<uint32_t*>(base + o_jq);
            P.job_cnt = reinterpret_cast<uint64_t*>(base + o_jc);
            P.summary = reinterpret_cast<colo_colocated_summary*>(base + o_sum);
        }
        P.evcnt = reinterpret_cast<unsigned long long*>(ctx->d_counters);
        const unsigned long long start_cnt = n;  // the arrival records come first
        if (cudaMemcpyAsync(P.evcnt, &start_cnt, 8, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaMemsetAsync(ctx->d_flag, 0, sizeof(int), ctx->stream) != cudaSuccess)
            return -cuda_err(ctx, cudaGetLastError(), "event log setup");
        COLO_LAUNCHED(ctx);
        k_co_validate<<<1, 128, 0, ctx->stream>>>(P);
        int flag = 0;
        cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -cuda_err(ctx, cudaGetLastError(), "validate");
        if (flag)
            return -set_err(ctx, COLO_EVALIDATION,
                            "trace rejected: unsorted arrivals, zero tokens, or a query that cannot fit the device alone");
        if (n) {
            COLO_LAUNCHED(ctx);
            k_log_arrivals<<<static_cast<uint32_t>(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0, ctx->stream>>>(
                d_arrival, d_query_id, n, P.evlog);
        }
        COLO_LAUNCHED(ctx);
        k_colocated<false, true><<<1, kWarpsC * 32, 0, ctx->stream>>>(P);
        if (sim_mode == COLO_SIM_SEPARATE) {  // the trainer over the job stream in enqueue order (stable sort)
            int f2 = 0;
            uint64_t jn = 0;
            cudaMemcpyAsync(&f2, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
            cudaMemcpyAsync(&jn, P.job_cnt, 8, cudaMemcpyDeviceToHost, ctx->stream);
            if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -cuda_err(ctx, cudaGetLastError(), "jobs");
            const double* jt = P.job_t;
            const uint32_t* jq = P.job_q;
            if ((f2 & 4) && jn > 1) {
                size_t tb2 = tb;
                if (cub::DeviceRadixSort::SortPairs(base + o_tmp, tb2, P.job_t, reinterpret_cast<double*>(base + o_jt2),
                                                    P.job_q, reinterpret_cast<uint32_t*>(base + o_jq2),
                                                    static_cast<int>(jn), 0, 64, ctx->stream) != cudaSuccess)
                    return -cuda_err(ctx, cudaGetLastError(), "job sort");
                jt = reinterpret_cast<const double*>(base + o_jt2);
                jq = reinterpret_cast<const uint32_t*>(base + o_jq2);
            }
            COLO_LAUNCHED(ctx);
            k_trainer_fold<<<1, 128, 0, ctx->stream>>>(P, jt, jq);
        }
        unsigned long long cnt = 0;
        cudaMemcpyAsync(&cnt, P.evcnt, 8, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -cuda_err(ctx, cudaGetLastError(), "event log");
        if (flag & 2) return -set_err(ctx, COLO_EBREACH, "event log: the run breached an invariant (no log)");
        if (cnt > n + cap) {  // more records than room: grow and run again
            cap = static_cast<size_t>(cnt) * 5 / 4 + 65536;
            continue;
        }
        std::vector<EvRec> ev(cnt);
        if (cnt && cudaMemcpy(ev.data(), P.evlog, cnt * sizeof(EvRec), cudaMemcpyDeviceToHost) != cudaSuccess)
            return -cuda_err(ctx, cudaGetLastError(), "event log D2H");
        // dispatch order: (time, sequence, position inside the handler); times are >= 0 here
        std::stable_sort(ev.begin(), ev.end(), [](const EvRec& x, const EvRec& y) {
            return x.t < y.t || (x.t == y.t && x.key < y.key);
        });
        std::vector<uint32_t> dead;  // torn-down store generations: their later CopyDone events are no-ops
        std::string out;
        out.reserve(ev.size() * 120);
        static const char* const kNames[] = {"QueryArrival", "PrefillDone", "DecodeStepDone", "QueryDone",
                                             "LabelArrival", "CacheTimeout", "TrainingResume", "BackwardLayerDone",
                                             "ForwardLayerDone", "LoadDone", "CopyDone"};
        static const char kLane[] = {'-', 's', 's', '-', '-', '-', '-', 't', 't', 'x', 'x'};
        unsigned long long lseq = 0;
        char buf[320];
        for (const EvRec& r : ev) {
            if (r.kind == EV_TEARDOWN) {
                dead.push_back(r.gen);
                continue;
            }
            if (r.kind == EV_COPY && std::find(dead.begin(), dead.end(), r.gen) != dead.end()) continue;
            if (r.kind > EV_COPY) continue;
            const char lane_c = (r.kind == EV_FWD || r.kind == EV_BWD) && r.gen == 1 ? 'r' : kLane[r.kind];
            const int k = std::snprintf(buf, sizeof buf,
                                        "{\"t\":%.9f,\"seq\":%llu,\"kind\":\"%s\",\"a\":%lld,\"b\":%lld,"
                                        "\"start\":%.9f,\"dur\":%.9f,\"lane\":\"%c\"}\n",
                                        r.t, lseq++, kNames[r.kind], static_cast<long long>(r.a),
                                        static_cast<long long>(r.b), r.start, r.dur, lane_c);
            out.append(buf, static_cast<size_t>(k));
        }
        ctx->evtext.swap(out);
        return static_cast<int64_t>(ctx->evtext.size());
    }
    return -set_err(ctx, COLO_EINVAL, "event log: could not size the record buffer");
}

int64_t colo_events_text(colo_ctx* ctx, char* out, size_t cap) {
    if (!ctx) return -COLO_EINVAL;
    const size_t len = ctx->evtext.size();
    if (out && cap > len) {
        std::memcpy(out, ctx->evtext.data(), len);
        out[len] = '\0';
    }
    return static_cast<int64_t>(len);
}

colo_status colo_sort_f64(colo_ctx* ctx, const double* d_in, double* d_out, size_t n) {
    if (!ctx || (n && (!d_in || !d_out)) || d_in == d_out) return COLO_EINVAL;
    if (n == 0) return COLO_OK;
    if (n >= (1ull << 31)) return set_err(ctx, COLO_EINVAL, "colo_sort_f64: at most 2^31-1 values");
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    size_t tb = 0;
    COLO_CK(ctx, cub::DeviceRadixSort::SortKeys(nullptr, tb, d_in, d_out, static_cast<int>(n), 0, 64, ctx->stream));
    const colo_status st = grow_scratch(ctx, tb + 256);
    if (st != COLO_OK) return st;
    COLO_CK(ctx, cub::DeviceRadixSort::SortKeys(ctx->d_rscratch, tb, d_in, d_out, static_cast<int>(n), 0, 64,
                                                ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

colo_status colo_finalize(colo_ctx* ctx, const double* d_samples, size_t n, double* d_sorted, double* out) {
    if (!ctx || !out || (n && !d_samples) || (d_sorted && d_sorted == d_samples)) return COLO_EINVAL;
    for (int i = 0; i < 4; ++i) out[i] = std::nan("");
    if (n == 0) return COLO_OK;
    if (n >= (1ull << 31)) return set_err(ctx, COLO_EINVAL, "colo_finalize: at most 2^31-1 samples");
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    // sorted values zero-padded to whole fold chunks (S + 0 = S), the fold's
    // chunk candidates, one SegDev range, the pointer table and the result
    const size_t nch = (n + kFoldCh - 1) / kFoldCh, npad = nch * kFoldCh;
    size_t tb = 0;
    COLO_CK(ctx, cub::DeviceRadixSort::SortKeys(nullptr, tb, d_samples, static_cast<double*>(nullptr),
                                                static_cast<int>(n), 0, 64, ctx->stream));
    const size_t o_srt = 0, o_cand = align256c(npad * 8), o_sd = o_cand + align256c(nch * 64 * 8),
                 o_ptr = o_sd + align256c(sizeof(SegDev)), o_res = o_ptr + 256, o_tmp = o_res + 256;
    {
        const colo_status st = grow_buf(ctx, ctx->d_seglog, ctx->seglog_bytes, o_tmp + tb + 256);
        if (st != COLO_OK) return st;
    }
    auto* base = static_cast<uint8_t*>(ctx->d_seglog);
    auto* srt = reinterpret_cast<double*>(base + o_srt);
    auto* cand = reinterpret_cast<uint64_t*>(base + o_cand);
    COLO_CK(ctx, cub::DeviceRadixSort::SortKeys(base + o_tmp, tb, d_samples, srt, static_cast<int>(n), 0, 64,
                                                ctx->stream));
    if (npad > n) COLO_CK(ctx, cudaMemsetAsync(srt + n, 0, (npad - n) * 8, ctx->stream));
    SegDev sd{};
    sd.lcnt[0] = npad;
    const void* ptrs[6] = {srt, srt, srt, cand, cand, cand};
    COLO_CK(ctx, cudaMemcpyAsync(base + o_sd, &sd, sizeof sd, cudaMemcpyHostToDevice, ctx->stream));
    COLO_CK(ctx, cudaMemcpyAsync(base + o_ptr, ptrs, sizeof ptrs, cudaMemcpyHostToDevice, ctx->stream));
    COLO_LAUNCHED(ctx);
    k_fold_cand<<<static_cast<uint32_t>((nch * 32 + 127) / 128), 128, 0, ctx->stream>>>(srt, nch, cand);
    COLO_LAUNCHED(ctx);
    k_fold_walk<<<1, 32, 0, ctx->stream>>>(reinterpret_cast<const SegDev*>(base + o_sd),
                                          reinterpret_cast<const double* const*>(base + o_ptr),
                                          reinterpret_cast<const uint64_t* const*>(base + o_ptr + 3 * sizeof(void*)),
                                          reinterpret_cast<double*>(base + o_res));
    COLO_CK(ctx, cudaGetLastError());
    double sum = 0.0, q[3];
    const double qs[3] = {0.50, 0.90, 0.99};
    COLO_CK(ctx, cudaMemcpyAsync(&sum, base + o_res, 8, cudaMemcpyDeviceToHost, ctx->stream));
    for (int i = 0; i < 3; ++i)  // nearest_rank (metrics.hpp:48-53)
        COLO_CK(ctx, cudaMemcpyAsync(&q[i], srt + colo_nearest_rank_index(qs[i], n) - 1, 8, cudaMemcpyDeviceToHost,
                                     ctx->stream));
    if (d_sorted) COLO_CK(ctx, cudaMemcpyAsync(d_sorted, srt, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    out[0] = q[0];
    out[1] = q[1];
    out[2] = q[2];
    out[3] = sum / static_cast<double>(n);  // metrics.hpp:63-65
    return COLO_OK;
}

colo_status colo_colocated_stats(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const double* d_arrival,
                                 const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                 const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev,
                                 const colo_colocated_opts* opts, double* pctl, colo_colocated_summary* totals) {
    if (!ctx || !opts || !pctl || !totals) return COLO_EINVAL;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    const size_t hbytes = sizeof(uint64_t) * 3 * COLO_HIST_BINS;
    uint64_t* d_hist = nullptr;
    colo_colocated_summary* d_sum = opts->d_summary;
    const bool own_sum = d_sum == nullptr;
    COLO_CK(ctx, cudaMalloc(&d_hist, hbytes));
    if (own_sum) {
        const cudaError_t e = cudaMalloc(&d_sum, sizeof(colo_colocated_summary) * std::max<size_t>(ndev, 1));
        if (e != cudaSuccess) {
            cudaFree(d_hist);
            return cuda_err(ctx, e, "cudaMalloc(summary)");
        }
    }
    std::vector<uint64_t> h(3 * static_cast<size_t>(COLO_HIST_BINS));
    std::vector<colo_colocated_summary> sums(ndev);
    colo_status st = COLO_OK;
    const double qs[3] = {0.50, 0.90, 0.99};
    uint64_t rank[3] = {0, 0, 0}, b1[3] = {0, 0, 0}, b2[3] = {0, 0, 0};
    uint64_t ntot = 0;
    *totals = colo_colocated_summary{};
    for (int i = 0; i < 4; ++i) pctl[i] = std::nan("");
    for (int pass = 0; pass < 3 && st == COLO_OK; ++pass) {
        colo_colocated_opts o = *opts;
        o.d_hist = d_hist;
        o.d_summary = pass == 0 ? d_sum : nullptr;
        if (pass > 0) {  // outputs are written by the first pass only
            o.d_samples = nullptr;
            o.d_labels = nullptr;
            o.d_batches = nullptr;
        }
        if (pass == 0) {
            o.nfilters = 1;
            o.filter_shift = 63;
            o.hist_shift = 42;
            o.filter_prefix[0] = 0;
        } else {
            o.nfilters = 3;
            o.filter_shift = pass == 1 ? 42 : 21;
            o.hist_shift = pass == 1 ? 21 : 0;
            for (int f = 0; f < 3; ++f) o.filter_prefix[f] = pass == 1 ? b1[f] : ((b1[f] << 21) | b2[f]);
        }
        cudaError_t e = cudaMemsetAsync(d_hist, 0, hbytes, ctx->stream);
        if (e != cudaSuccess) {
            st = cuda_err(ctx, e, "cudaMemset(hist)");
            break;
        }
        st = colo_replay_colocated(ctx, sets, nsets, d_arrival, d_prompt, d_output, n, d_dev_offsets, d_dev_set, ndev,
                                   &o);
        if (st != COLO_OK) break;
        e = cudaMemcpy(h.data(), d_hist, sizeof(uint64_t) * o.nfilters * COLO_HIST_BINS, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            st = cuda_err(ctx, e, "hist D2H");
            break;
        }
        if (pass == 0) {
            e = cudaMemcpy(sums.data(), d_sum, sizeof(colo_colocated_summary) * ndev, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) {
                st = cuda_err(ctx, e, "summary D2H");
                break;
            }
            colo_colocated_summary& t = *totals;
            for (const auto& s : sums) {
                t.generated_tokens += s.generated_tokens;
                t.trained_tokens += s.trained_tokens;
                t.training_busy_time += s.training_busy_time;
                t.peak_device_bytes = std::max(t.peak_device_bytes, s.peak_device_bytes);
                t.peak_training_activation_bytes =
                    std::max(t.peak_training_activation_bytes, s.peak_training_activation_bytes);
                t.preemptions += s.preemptions;
                t.layers_freed += s.layers_freed;
                t.loads += s.loads;
                t.recomputes += s.recomputes;
                t.copy_stall_seconds += s.copy_stall_seconds;
                t.labels_dropped += s.labels_dropped;
                t.prefetch_wait_seconds += s.prefetch_wait_seconds;
                t.completed_jobs += s.completed_jobs;
                t.map_fallbacks += s.map_fallbacks;
                t.oom_jobs += s.oom_jobs;
                t.batches += s.batches;
                t.max_batch_size = std::max(t.max_batch_size, s.max_batch_size);
                t.offload_decisions += s.offload_decisions;
                t.admissions += s.admissions;
                t.slow_tokens += s.slow_tokens;
                t.slow_queries += s.slow_queries;
                t.end_time = std::max(t.end_time, s.end_time);
                t.status = std::max(t.status, s.status);
                fixed_add(t.tpt_sum, s.tpt_sum);
                t.flags |= s.flags;
            }
            ntot = t.generated_tokens;
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
    if (own_sum) cudaFree(d_sum);
    return st;
}

}  // extern "C"
