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
// consume their sequence numbers and are not materialised.
//
// Every f64 operation is the reference's, in the reference's order
// (-fmad=false), so each device's MetricsReport fields and TPT samples equal
// Simulation::run's bit for bit.  Reference paths are relative to
// /root/reference/proj/.
#include <algorithm>
#include <cmath>
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

__global__ void __launch_bounds__(kWarpsC * 32) k_colocated(const __grid_constant__ CoParams P) {
    __shared__ WarpSmem SM[kWarpsC];
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t d = blockIdx.x * kWarpsC + wib;
    if (d >= P.ndev) return;
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
    uint64_t ai = 0, qhead = 0;  // queue_ = [qhead, ai)
    uint64_t alloc = 0, resv = 0, peak = 0;  // MemoryLedger device_
    double d2h_busy = 0.0;                   // TransferChannel d2h_
    bool breach = false;
    // serving
    bool sbusy = false;
    double s_t = 0.0;
    uint64_t s_seq = 0, bfirst = 0, bn = 0, bneed = 0;
    // slot
    bool has_store = false, qcompleted = false, stream = false;
    uint64_t src = 0, prompt_kv = 0, kv_held = 0, cached_tokens = 0, gen = 0, store_gen = 0, plan_gen = 0;
    // job
    bool has_job = false, incl_prompt = false, waiting = false, tinf = false;
    int phase = PH_WAIT;
    uint64_t jp = 0, jo = 0, pass0 = 0, pass1 = 0, pass2 = 0, npasses = 0, pass_index = 0, cursor = 0;
    int64_t kv_charged = -1;
    double wait_since = 0.0, plb = 0.0, tbusy = 0.0;  // plb = per_layer_backward(job) (engine.hpp:614-618)
    double t_t = 0.0, t_dur = 0.0;
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
    double na = N ? arr[0] : 0.0;  // arrival time of query ai
    // report (uniform) + per-lane sample partials
    uint64_t r_trained = 0, r_ptab = 0, r_pre = 0, r_freed = 0, r_loads = 0, r_recomp = 0, r_dropped = 0, r_jobs = 0,
             r_fb = 0, r_batches = 0, r_maxb = 0, r_offd = 0, r_adm = 0;
    double r_stall = 0.0, r_wait = 0.0, r_end = 0.0;
    uint64_t a_gen = 0, a_slow = 0, a_slowq = 0, a_acc[3] = {0, 0, 0};
    uint32_t a_flags = 0;
    uint64_t sample_pos = P.samples ? P.sample_off[d] : 0;
    const bool want_hist = P.hist != nullptr;

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
            double mine = 0.0;
            for (uint32_t b = bal; b; b &= b - 1) {  // channel += dur, descending layer order
                const int j = __ffs(b) - 1;
                channel += __shfl_sync(kFullMask, dur, j);
                if (lane == static_cast<uint32_t>(j)) mine = channel;
            }
            if (el) {
                const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                S.llayer[pos] = static_cast<uint16_t>(l);
                S.ldone[pos] = mine;
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
        r_stall += stall;
        tbusy += stall;
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
        for (uint64_t j = 0; j < nb; ++j) {
            const double t = member_pd(j);
            double base = 1.0 * (m.prefill_coef_linear * t + m.prefill_coef_quad * t * t);
            if (j == 0 && rec) base = base * m.record_prefill_multiplier;
            dur += base;
        }
        const double start = now + stall;
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
            for (uint64_t j = 0; j < nb; ++j) {
                const uint32_t oj = staged ? S.po[j].y : po[head + j];
                const double pj = member_pd(j);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (kb + 32 * r < oj) {
                        dk[r] += gam + del * (pj + kd[r]);
                        ++alive[r];
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) S.dk[32 * r + lane] = dk[r];
            __syncwarp();
            // absolute-time chain now_k = now_{k-1} + d_k (sequential, one lane),
            // the durations are overwritten by the absolute times
            const uint32_t cnt = min(128u, maxo - k0);
            if (lane == 0) chain_fold_store(tnow, S.dk, cnt);
            __syncwarp();
            double sv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int r = 0; r < 4; ++r) {  // sample = now - last_token_time
                const uint32_t i = 32 * r + lane;
                if (i < cnt) sv[r] = S.dk[i] - (i ? S.dk[i - 1] : tnow);
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
                            if (em) {
                                if (te < (below ? prev_lane : last_t)) unsorted = true;
                                const uint64_t pos = lo + jc + __popc(below);
                                P.job_t[pos] = te;
                                P.job_q[pos] = static_cast<uint32_t>(head + j);
                            }
                            last_t = __shfl_sync(kFullMask, te, 31 - __clz(bal));
                            jc += __popc(bal);
                        }
                    }
                    cur = mn + 1;
                }
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t kr0 = k0 + 32 * r;
                if (kr0 >= maxo) break;
                const uint32_t k = kr0 + lane;
                const double s = sv[r];
                const uint32_t alv = alive[r];
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
                if (P.samples) {  // step k's samples: alive_k consecutive slots, steps in order
                    uint32_t ex = alv;
#pragma unroll
                    for (int sft = 1; sft < 32; sft <<= 1) {
                        const uint32_t y = __shfl_up_sync(kFullMask, ex, sft);
                        if (lane >= static_cast<uint32_t>(sft)) ex += y;
                    }
                    const uint32_t tot = __shfl_sync(kFullMask, ex, 31);
                    const uint64_t pos = sample_pos + ex - alv;
                    for (uint32_t a = 0; a < alv; ++a) P.samples[pos + a] = s;
                    sample_pos += tot;
                }
            }
        }
        for (uint64_t j = lane; j < nb; j += 32) {  // a query is slow iff one of its tokens is
            const uint32_t oj = staged ? S.po[j].y : po[head + j];
            const bool slowq = oj > first_slow;
            a_slowq += slowq;
            if (P.labels) P.labels[lo + head + j] = slowq ? 1 : 0;
        }
        if (lane == 0 && P.batches) {
            colo_batch b;
            b.start = start;
            b.end = tnow;
            b.first = static_cast<uint32_t>(head);
            b.n = static_cast<uint32_t>(nb);
            b.need_total = need_total;
            b.max_incoming = max_inc < 0xffffffffull ? static_cast<uint32_t>(max_inc) : 0xffffffffu;
            b.verdict = vbits;
            P.batches[lo + r_batches] = b;
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
                continue;
            }
            now = na;
            ++ai;
            na = ai < N ? arr[ai] : 0.0;
            if (has_job && waiting) {  // interrupt_training_wait(true), engine.hpp:622-631
                const double waited = now - wait_since;
                r_wait += waited;
                tbusy += waited;
                waiting = false;
                ++r_pre;
                ++plan_gen;
            }
            want_serve = true;
        } else {
        if (bk == EK_NONE) break;
        now = bt;
        if (bk == EK_SERVE) {  // the batch's last DecodeStepDone (engine.hpp:367-408)
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
                    }
                }
            }
            led_free(release);
            r_end = now;
            want_serve = true;
        } else if (bk == EK_TRAIN) {
            tinf = false;
            tbusy += t_dur;
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
                ++r_dropped;
                teardown();
            }
        } else {  // EK_LOAD, engine.hpp:781-797
            const uint32_t a = S.llayer[ld_cur];
            ++ld_cur;
            const uint64_t r = S.rec[a];
            if (!led_alloc(r)) breach = true;
            set_layer(a, static_cast<uint8_t>(S.flg[a] | LF_DEV), r);
            ++r_loads;
            if (has_job && waiting && phase == PH_BWD && cursor == a && !sbusy && qhead == ai) {
                const double waited = now - wait_since;
                r_wait += waited;
                tbusy += waited;
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
    if (breach && lane == 0) atomicOr(P.err, 2);
    if (__any_sync(kFullMask, unsorted) && lane == 0) atomicOr(P.err, 4);
    if (P.job_cnt && lane == 0) P.job_cnt[d] = jc;  // every device (0 unless SeparateCluster): sort segments
    if (lane == 0 && P.summary) {
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
        P.summary[d] = r;
    }
}

// SeparateCluster trainer (engine.hpp:824-903), one thread per device, folded
// over the job stream in enqueue order.  Jobs run FIFO one at a time: a job
// starts at max(enqueue, previous job's last layer) (schedule_baseline_layer
// with trainer_free_at_, :850-858), each layer completes at the previous one's
// time + its duration (:860-872, 888, 902), and training_busy_time adds every
// layer's duration in that order (:875).  The trainer ledger peaks at the
// fixed footprint plus the largest job it ran (memory.hpp:28-35 reuse).
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
                t = t + fd;
                busy += fd;
            }
        for (uint64_t l = 0; l < L; ++l) {
            t = t + bd;
            busy += bd;
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
    k_co_validate<<<vblocks, 128, 0, ctx->stream>>>(P);
    int flag = 0;
    COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (flag)
        return set_err(ctx, COLO_EVALIDATION,
                       "trace rejected: unsorted arrivals, zero tokens, or a query that cannot fit the device alone");
    const uint32_t blocks = static_cast<uint32_t>((ndev + kWarpsC - 1) / kWarpsC);
    k_colocated<<<blocks, kWarpsC * 32, 0, ctx->stream>>>(P);
    COLO_CK(ctx, cudaGetLastError());
    COLO_CK(ctx, cudaMemcpyAsync(&flag, ctx->d_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
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
        k_trainer_fold<<<static_cast<uint32_t>((ndev + 127) / 128), 128, 0, ctx->stream>>>(P, jt, jq);
        COLO_CK(ctx, cudaGetLastError());
        COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    }
    if (flag & 2) return set_err(ctx, COLO_EBREACH, "colocated replay: invariant breach on at least one device");
    return COLO_OK;
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
