/*
 * colo_colocated.c -- TEST INFRASTRUCTURE ONLY (see colo_oracle.h).
 *
 * Plain-C restatement of colosim's colocated replay: Simulation::run in
 * SimMode::Colocated (include/colosim/engine.hpp:140-822) with the memory
 * model of include/colosim/memory.hpp:19-211.  It is the parity checker for
 * the sm_100a colocated-replay kernel (colo_colocated.cu); it is itself
 * checked against the unchanged reference (oracle/_ref, ref_replay_colocated)
 * in tests/test_oracle_golden.py and against golden fixtures.
 *
 * Event order.  The reference pushes every arrival first (seq 0..N-1,
 * engine.hpp:146-147) and pops by (time, seq) (:184-187).  Arrivals are
 * therefore a sorted stream that wins every time tie; every other event
 * gets the next sequence number at schedule() time and is kept in a small
 * unsorted list here (pop = linear min scan).  CopyDone events only update
 * host_bytes, which no MetricsReport field reads (engine.hpp:799-805), so
 * they consume their sequence number and are otherwise not materialised.
 * Paths are relative to /root/reference/proj/.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "colo_oracle.h"

enum { EV_PREFILL, EV_DECODE, EV_LABEL, EV_TIMEOUT, EV_FWD, EV_BWD, EV_LOAD, EV_BLAYER };
enum { PH_WAITING_LABEL, PH_READY, PH_FORWARD, PH_BACKWARD }; /* engine.hpp:203 */

typedef struct {
    double t;
    uint64_t seq;
    int kind;
    int64_t a, b;
    double dur;
} co_ev;

typedef struct { /* memory.hpp:45-52 (host_bytes is write-only for the metrics) */
    uint64_t recorded;
    double last_copy_done;
    int on_device, consumed, dropped;
} co_layer;

typedef struct {
    uint64_t p, o, fp;
} co_bjob; /* engine.hpp:225-232 (passes derived from p, o and the mode) */

typedef struct {
    const orc_model* m;
    const orc_gpu* g;
    const orc_maps* maps;
    int cpa;
    int sim_mode; /* ORC_SIM_* */
    double cache_timeout;
    const double* arr;
    const uint32_t* p;
    const uint32_t* o;
    const double* label_delay;
    uint64_t n, L, budget;

    double now;
    uint64_t next_seq;
    uint64_t ai;    /* next arrival to pop */
    uint64_t qhead; /* queue_ = [qhead, ai) (engine.hpp:918) */

    /* MemoryLedger device_ (memory.hpp:19-41) */
    uint64_t cap, allocated, reserved, peak;
    double d2h_busy; /* TransferChannel d2h_ (memory.hpp:61-70) */

    co_ev* ev;
    size_t nev, capev;

    /* serving batch */
    int serving_busy;
    uint64_t bfirst, bn;
    uint32_t bstep; /* decode steps completed */
    uint32_t bfirst_slow; /* first decode step whose sample exceeds tau */
    double last_token_time;
    int brec;

    /* Slot + ActivationStore (engine.hpp:215-223, memory.hpp:75-114) */
    int has_store;
    uint64_t src, src_p, src_o, prompt_kv, kv_held, cached_tokens, generation;
    int query_completed, stream;
    co_layer* layers;
    uint64_t store_gen, plan_gen;

    /* TrainingJob (engine.hpp:199-212) */
    int has_job, phase;
    uint64_t jp, jo;
    uint64_t passes[3], npasses, pass_index, cursor;
    uint64_t basis[3], nbasis;
    int include_prompt;
    int64_t kv_charged_pass;
    int waiting;
    double wait_since;
    int training_inflight;
    double train_busy;

    /* separate-cluster trainer (engine.hpp:824-903) */
    uint64_t t_alloc, t_resv, t_peak; /* MemoryLedger trainer_device_ */
    co_bjob* bq;
    size_t bq_head, bq_tail;
    co_bjob bjob;
    uint64_t b_pass, b_cursor;
    int b_backward, b_busy;
    double b_free_at;

    orc_colo_report* r;
    double tau;
    double* samples;
    uint64_t sample_pos;
    uint8_t* labels;
    orc_batch* batches;
    int breach;
} co_sim;

static void co_push(co_sim* s, double t, int kind, int64_t a, int64_t b, double dur) {
    if (s->nev == s->capev) {
        s->capev = s->capev ? 2 * s->capev : 64;
        s->ev = (co_ev*)realloc(s->ev, s->capev * sizeof(co_ev));
    }
    co_ev e = {t, s->next_seq++, kind, a, b, dur};
    s->ev[s->nev++] = e;
}

/* memory.hpp:28-35 */
static int co_alloc(co_sim* s, uint64_t bytes) {
    if (s->allocated - s->reserved + bytes > s->cap) return 0;
    uint64_t reuse = s->reserved < bytes ? s->reserved : bytes;
    s->reserved -= reuse;
    s->allocated += bytes - reuse;
    if (s->allocated > s->peak) s->peak = s->allocated;
    return 1;
}
/* memory.hpp:37-40 */
static void co_free(co_sim* s, uint64_t bytes) {
    if (bytes > s->allocated - s->reserved) s->breach = 1; /* std::logic_error */
    s->reserved += bytes;
}
static uint64_t co_live(const co_sim* s) { return s->allocated - s->reserved; }
static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */

static uint64_t co_need(const co_sim* s, uint64_t j) {
    return orc_serving_memory(s->m, (uint64_t)s->p[j] + s->o[j], 1, NULL);
}

/* engine.hpp:815-822 */
static void co_training_peak(co_sim* s) {
    if (!s->has_store) return;
    uint64_t cur = s->kv_held;
    for (uint64_t l = 0; l < s->L; ++l)
        if (!s->layers[l].consumed && !s->layers[l].dropped) cur += s->layers[l].recorded;
    if (cur > s->r->peak_training_activation_bytes) s->r->peak_training_activation_bytes = cur;
}

/* memory.hpp:121-139 (+ the CopyDone schedule of engine.hpp:344-347, 704-705) */
static void co_record(co_sim* s, uint64_t l, uint64_t bytes, double now) {
    co_layer* e = &s->layers[l];
    e->dropped = 0;
    int to_host = s->stream || (e->recorded > 0 && !e->on_device);
    if (!to_host) {
        if (!co_alloc(s, bytes)) s->breach = 1;
        e->on_device = 1;
    }
    e->recorded += bytes;
    double start = dmax(now, s->d2h_busy);
    s->d2h_busy = start + orc_transfer_time(s->g, bytes, 0);
    e->last_copy_done = s->d2h_busy;
    s->next_seq++; /* CopyDone */
}

/* engine.hpp:468-479 */
static void co_teardown(co_sim* s) {
    if (!s->has_store) return;
    for (uint64_t l = 0; l < s->L; ++l)
        if (s->layers[l].on_device) {
            co_free(s, s->layers[l].recorded);
            s->layers[l].on_device = 0;
        }
    if (s->kv_held) co_free(s, s->kv_held);
    s->has_store = 0;
    s->has_job = 0;
    ++s->plan_gen;
}

static void co_start_serving(co_sim* s);
static void co_try_start_training(co_sim* s);

/* engine.hpp:614-618 */
static double co_per_layer_backward(const co_sim* s) {
    double d = 0;
    for (uint64_t i = 0; i < s->nbasis; ++i) d += orc_backward_layer_latency(s->m, s->basis[i], NULL);
    return d;
}

/* engine.hpp:622-631 */
static void co_interrupt_wait(co_sim* s, int count) {
    if (s->has_job && s->waiting) {
        double waited = s->now - s->wait_since;
        s->r->prefetch_wait_seconds += waited;
        s->train_busy += waited;
        s->waiting = 0;
        if (count) ++s->r->preemptions;
        ++s->plan_gen;
    }
}

/* engine.hpp:725-731 */
static int co_preempt(co_sim* s) {
    if (s->qhead == s->ai) return 0;
    ++s->r->preemptions;
    ++s->plan_gen;
    co_start_serving(s);
    return 1;
}

/* engine.hpp:669-683 */
static void co_charge_pass_kv(co_sim* s) {
    if (s->kv_charged_pass == (int64_t)s->pass_index) return;
    s->kv_charged_pass = (int64_t)s->pass_index;
    if (!s->cpa) return;
    int is_prompt = s->include_prompt && s->pass_index == 0;
    if (is_prompt && s->prompt_kv > 0) return;
    uint64_t kv = orc_kv_bytes(s->m, s->passes[s->pass_index], 1);
    if (!co_alloc(s, kv)) s->breach = 1;
    s->kv_held += kv;
    if (is_prompt) s->prompt_kv += kv;
    co_training_peak(s);
}

/* engine.hpp:685-691 */
static void co_schedule_forward(co_sim* s) {
    double dur = orc_forward_layer_latency(s->m, s->passes[s->pass_index], NULL);
    s->training_inflight = 1;
    co_push(s, s->now + dur, EV_FWD, (int64_t)s->cursor, (int64_t)s->pass_index, dur);
}

static void co_begin_pass(co_sim* s) { /* engine.hpp:662-665 */
    co_charge_pass_kv(s);
    co_schedule_forward(s);
}

/* engine.hpp:749-759 */
static void co_schedule_backward(co_sim* s) {
    if (!s->layers[s->cursor].on_device) {
        s->waiting = 1;
        s->wait_since = s->now;
        return;
    }
    double dur = co_per_layer_backward(s);
    s->training_inflight = 1;
    co_push(s, s->now + dur, EV_BWD, (int64_t)s->cursor, 0, dur);
}

/* engine.hpp:733-747 + plan_prefetch (memory.hpp:183-211; only the loads are used) */
static void co_start_backward(co_sim* s) {
    ++s->plan_gen;
    double channel = s->now;
    for (uint64_t i = s->L; i-- > 0;) {
        const co_layer* l = &s->layers[i];
        if (l->on_device || l->consumed || l->dropped || l->recorded == 0) continue;
        double start = channel;
        channel += orc_transfer_time(s->g, l->recorded, 1);
        co_push(s, channel, EV_LOAD, (int64_t)i, (int64_t)s->plan_gen, channel - start);
    }
    co_schedule_backward(s);
}

/* engine.hpp:633-660 */
static void co_try_start_training(co_sim* s) {
    if (!s->has_job || s->serving_busy || s->qhead != s->ai || s->training_inflight) return;
    switch (s->phase) {
        case PH_WAITING_LABEL: return;
        case PH_READY:
            if (s->pass_index < s->npasses) {
                s->phase = PH_FORWARD;
                s->cursor = 0;
                co_begin_pass(s);
            } else {
                s->phase = PH_BACKWARD;
                s->cursor = s->L - 1;
                co_start_backward(s);
            }
            return;
        case PH_FORWARD: co_begin_pass(s); return;
        case PH_BACKWARD: co_start_backward(s); return;
    }
}

/* engine.hpp:421-466 */
static int co_admit(co_sim* s, uint64_t j) {
    uint64_t charged = s->p[j];
    if (s->cpa) charged += 2ull * s->o[j];
    s->has_store = 1;
    memset(s->layers, 0, s->L * sizeof(co_layer));
    s->src = j;
    s->src_p = s->p[j];
    s->src_o = s->o[j];
    s->prompt_kv = 0;
    s->kv_held = 0;
    s->query_completed = 0;
    s->cached_tokens = charged;
    s->generation = ++s->store_gen;
    int stream = 0, action;
    uint64_t layers;
    if (!orc_offload_lookup(&s->maps->grid, s->maps->offload_cells, charged, 1, 1, &action, &layers)) {
        stream = 1;
        ++s->r->map_fallbacks;
    } else if (action == 2 /* AllToHost */) {
        stream = 1;
    }
    uint64_t prompt_acts = orc_activation_bytes(s->m, s->p[j], s->L, NULL);
    if (co_live(s) + prompt_acts > s->cap) stream = 1;
    s->stream = stream;
    ++s->r->admissions;

    s->has_job = 1;
    s->jp = s->p[j];
    s->jo = s->o[j];
    s->pass_index = 0;
    s->cursor = 0;
    s->include_prompt = 0;
    s->kv_charged_pass = -1;
    s->waiting = 0;
    if (!s->cpa) {
        s->phase = PH_READY;
        s->npasses = 0;
        s->basis[0] = s->jp;
        s->nbasis = 1;
    } else {
        s->phase = PH_WAITING_LABEL;
        s->passes[0] = s->passes[1] = s->jo;
        s->npasses = 2;
        s->basis[0] = s->jp;
        s->basis[1] = s->basis[2] = s->jo;
        s->nbasis = 3;
        co_push(s, s->now + s->cache_timeout, EV_TIMEOUT, (int64_t)s->generation, 0, 0);
    }
    return 1;
}

/* engine.hpp:563-610 */
static void co_drop_for_recompute(co_sim* s, uint64_t need_total) {
    ++s->r->recomputes;
    ++s->plan_gen;
    for (uint64_t l = 0; l < s->L; ++l) {
        co_layer* e = &s->layers[l];
        if (e->on_device) {
            co_free(s, e->recorded);
            e->on_device = 0;
        }
        e->dropped = 1;
        e->recorded = 0;
        e->consumed = 0;
        e->last_copy_done = 0;
    }
    uint64_t response_kv = s->kv_held - s->prompt_kv;
    if (response_kv) co_free(s, response_kv);
    s->kv_held = s->prompt_kv;
    if (s->has_job) {
        s->pass_index = 0;
        s->cursor = 0;
        s->kv_charged_pass = -1;
        s->waiting = 0;
        if (s->phase != PH_WAITING_LABEL) s->phase = PH_READY;
        if (!s->cpa) {
            s->passes[0] = s->jp;
            s->npasses = 1;
            s->basis[0] = s->jp;
            s->nbasis = 1;
        } else {
            s->include_prompt = 1;
            s->passes[0] = s->jp;
            s->passes[1] = s->passes[2] = s->jo;
            s->npasses = 3;
            memcpy(s->basis, s->passes, sizeof s->basis);
            s->nbasis = 3;
        }
    }
    if (s->kv_held > 0 && co_live(s) + need_total > s->cap) {
        co_free(s, s->kv_held);
        s->kv_held = 0;
        s->prompt_kv = 0;
    }
    co_training_peak(s);
}

/* engine.hpp:513-557 (free_layers_forward_order: memory.hpp:150-165) */
static double co_apply_offload(co_sim* s, uint64_t incoming, uint64_t batch_n, uint64_t need_total) {
    ++s->r->offload_decisions;
    const uint64_t L = s->L;
    uint64_t cached = s->cached_tokens;
    int action;
    uint64_t layers;
    int fallback = !orc_offload_lookup(&s->maps->grid, s->maps->offload_cells, cached, incoming, batch_n, &action,
                                       &layers);
    if (fallback) {
        ++s->r->map_fallbacks;
        action = 2;
        layers = 0;
    }
    if (action == 0) return 0;
    uint64_t dev_layers = 0, pending = 0;
    for (uint64_t l = 0; l < L; ++l) {
        const co_layer* e = &s->layers[l];
        dev_layers += e->on_device != 0;
        pending += !e->on_device && !e->consumed && !e->dropped && e->recorded > 0;
    }
    uint64_t free_now = action == 2 ? dev_layers : (layers < dev_layers ? layers : dev_layers);
    uint64_t ltf = action == 2 ? L : layers;
    uint64_t total_freed = pending + ltf < L ? pending + ltf : L;
    int recompute = 1;
    if (!fallback) {
        int rc;
        if (orc_hedge_lookup(s->maps->hedge_step, s->maps->hedge_max, L, s->maps->hedge_cells, cached, total_freed,
                             &rc))
            recompute = rc;
        else
            ++s->r->map_fallbacks;
    }
    if (recompute) {
        co_drop_for_recompute(s, need_total);
        return 0;
    }
    ++s->plan_gen;
    double ready = s->now;
    uint64_t freed = 0;
    for (uint64_t l = 0; l < L && freed < free_now; ++l) {
        co_layer* e = &s->layers[l];
        if (!e->on_device) continue;
        ready = dmax(ready, e->last_copy_done);
        co_free(s, e->recorded);
        e->on_device = 0;
        ++freed;
    }
    s->r->layers_freed += freed;
    if (co_live(s) + need_total > s->cap) {
        co_drop_for_recompute(s, need_total);
        return 0;
    }
    double stall = dmax(0.0, ready - s->now);
    s->r->copy_stall_seconds += stall;
    s->train_busy += stall;
    return stall;
}

/* engine.hpp:282-328 */
static void co_start_serving(co_sim* s) {
    if (s->qhead == s->ai) {
        s->serving_busy = 0;
        co_try_start_training(s);
        return;
    }
    s->serving_busy = 1;
    uint64_t n = 0, need_total = 0, max_inc = 0;
    while (s->qhead + n < s->ai) {
        uint64_t j = s->qhead + n;
        uint64_t need = co_need(s, j);
        if (n > 0 && need_total + need > s->budget) break;
        need_total += need;
        uint64_t inc = (uint64_t)s->p[j] + s->o[j];
        if (inc > max_inc) max_inc = inc;
        ++n;
    }
    s->bfirst = s->qhead;
    s->bn = n;
    s->qhead += n;
    double stall = 0;
    if (s->sim_mode == ORC_SIM_COLOCATED && s->has_store) {
        uint64_t fp = s->kv_held;
        for (uint64_t l = 0; l < s->L; ++l)
            if (s->layers[l].on_device) fp += s->layers[l].recorded;
        if (fp > 0) stall = co_apply_offload(s, max_inc, n, need_total);
    }
    if (!co_alloc(s, need_total)) s->breach = 1;
    int recording = 0;
    if (s->sim_mode == ORC_SIM_COLOCATED && n == 1 && !s->has_store) recording = co_admit(s, s->bfirst);
    s->brec = recording;
    double start = s->now + stall;
    double dur = 0;
    for (uint64_t j = 0; j < n; ++j)
        dur += orc_prefill_latency(s->m, s->p[s->bfirst + j], 1, j == 0 && recording, NULL);
    co_push(s, start + dur, EV_PREFILL, 0, 0, dur);
    if (s->batches) {
        orc_batch* b = &s->batches[s->r->batches];
        b->start = start;
        b->first = (uint32_t)s->bfirst;
        b->n = (uint32_t)n;
        b->need_total = need_total;
        b->max_incoming = max_inc > 0xffffffffull ? 0xffffffffu : (uint32_t)max_inc;
        b->verdict = 0;
    }
    ++s->r->batches;
    if (n > s->r->max_batch_size) s->r->max_batch_size = n;
    if (recording) { /* engine.hpp:332-350 */
        uint64_t per_layer = s->src_p * s->m->act_bytes_per_token_per_layer;
        double layer_dur = dur / (double)s->L;
        for (uint64_t l = 0; l < s->L; ++l) {
            double seg_ready = start + (double)(l + 1) * layer_dur;
            if (s->stream && s->layers[l].recorded == 0) ++s->r->layers_freed;
            co_record(s, l, per_layer, seg_ready);
        }
        co_training_peak(s);
    }
}

static void co_schedule_decode(co_sim* s) { /* engine.hpp:358-365 */
    double dur = 0;
    for (uint64_t j = 0; j < s->bn; ++j) {
        uint64_t q = s->bfirst + j;
        if (s->bstep >= s->o[q]) continue;
        dur += orc_decode_step_latency(s->m, (uint64_t)s->p[q] + s->bstep, 1, 0, NULL);
    }
    co_push(s, s->now + dur, EV_DECODE, 0, 0, dur);
}

/* ---- separate-cluster trainer, engine.hpp:824-903 ---------------------------- */
static void co_baseline_layer_schedule(co_sim* s, double at) { /* :860-872 */
    double dur;
    int64_t kind_bwd = s->b_backward;
    if (!s->b_backward) {
        uint64_t tok = s->cpa ? s->bjob.p + s->bjob.o : s->bjob.p;
        dur = orc_forward_layer_latency(s->m, tok, NULL);
    } else {
        dur = 0;
        uint64_t np = s->cpa ? 2 : 1;
        uint64_t tok = s->cpa ? s->bjob.p + s->bjob.o : s->bjob.p;
        for (uint64_t i = 0; i < np; ++i) dur += orc_backward_layer_latency(s->m, tok, NULL);
    }
    co_push(s, at + dur, EV_BLAYER, (int64_t)s->b_cursor, kind_bwd, dur);
}

static int t_alloc(co_sim* s, uint64_t bytes) { /* memory.hpp:28-35 on trainer_device_ */
    if (s->t_alloc - s->t_resv + bytes > s->cap) return 0;
    uint64_t reuse = s->t_resv < bytes ? s->t_resv : bytes;
    s->t_resv -= reuse;
    s->t_alloc += bytes - reuse;
    if (s->t_alloc > s->t_peak) s->t_peak = s->t_alloc;
    return 1;
}

static void co_baseline_try_start(co_sim* s) { /* :850-858 */
    if (s->b_busy || s->bq_head == s->bq_tail) return;
    s->b_busy = 1;
    s->bjob = s->bq[s->bq_head++];
    s->b_pass = 0;
    s->b_cursor = 0;
    s->b_backward = 0;
    if (!t_alloc(s, s->bjob.fp)) s->breach = 1;
    co_baseline_layer_schedule(s, dmax(s->now, s->b_free_at));
}

static void co_baseline_enqueue(co_sim* s, uint64_t p, uint64_t o) { /* :826-848 */
    co_bjob j = {p, o, 0};
    uint64_t per_token = s->L * s->m->act_bytes_per_token_per_layer + s->m->kv_bytes_per_token;
    if (!s->cpa) j.fp += p * per_token;
    else {
        j.fp += (p + o) * per_token;
        j.fp += (p + o) * per_token;
    }
    if (j.fp > s->r->peak_training_activation_bytes) s->r->peak_training_activation_bytes = j.fp;
    uint64_t budget = s->cap - s->m->weights_bytes - s->g->runtime_reserve_bytes;
    if (j.fp > budget) {
        s->r->oom_jobs++;
        return;
    }
    s->bq[s->bq_tail++] = j;
    co_baseline_try_start(s);
}

static void co_on_baseline_layer(co_sim* s, double dur) { /* :874-903 */
    s->train_busy += dur;
    s->b_free_at = s->now;
    if (!s->b_backward) {
        ++s->b_cursor;
        if (s->b_cursor == s->L) {
            s->b_cursor = 0;
            ++s->b_pass;
            if (s->b_pass >= (uint64_t)(s->cpa ? 2 : 1)) {
                s->b_backward = 1;
                s->b_cursor = s->L - 1;
            }
        }
        co_baseline_layer_schedule(s, s->now);
        return;
    }
    if (s->b_cursor == 0) {
        s->r->trained_tokens += s->bjob.p + (s->cpa ? 2 * s->bjob.o : 0);
        ++s->r->completed_jobs;
        s->t_resv += s->bjob.fp; /* trainer_device_.free_bytes */
        s->b_busy = 0;
        co_baseline_try_start(s);
        return;
    }
    --s->b_cursor;
    co_baseline_layer_schedule(s, s->now);
}

/* engine.hpp:389-408 */
static void co_finish_query(co_sim* s, uint64_t q) {
    uint64_t release = co_need(s, q);
    if (s->has_store && s->src == q && !s->query_completed) {
        s->query_completed = 1;
        if (s->cpa) {
            uint64_t keep = orc_kv_bytes(s->m, s->p[q], 1);
            s->kv_held += keep;
            s->prompt_kv += keep;
            release -= release < keep ? release : keep;
            co_training_peak(s);
            double ld = s->label_delay ? s->label_delay[q] : -1.0;
            if (ld >= 0) co_push(s, s->now + ld, EV_LABEL, (int64_t)s->generation, (int64_t)q, 0);
        }
    }
    co_free(s, release);
    if (s->sim_mode == ORC_SIM_SEPARATE) { /* engine.hpp:410-416 */
        if (!s->cpa) {
            co_baseline_enqueue(s, s->p[q], s->o[q]);
        } else {
            double ld = s->label_delay ? s->label_delay[q] : -1.0;
            if (ld >= 0) co_push(s, s->now + ld, EV_LABEL, -1, (int64_t)q, 0);
        }
    }
}

/* engine.hpp:367-387 (+ the slow label rule) */
static void co_on_decode(co_sim* s) {
    int any_alive = 0;
    double smp = s->now - s->last_token_time;
    for (uint64_t j = 0; j < s->bn; ++j) {
        uint64_t q = s->bfirst + j;
        if (s->bstep >= s->o[q]) continue;
        if (s->samples) s->samples[s->sample_pos] = smp;
        ++s->sample_pos;
        ++s->r->generated_tokens;
        if (smp > s->tau) {
            ++s->r->slow_tokens;
            if (s->bstep < s->bfirst_slow) s->bfirst_slow = s->bstep;
        }
        if (s->bstep + 1 == s->o[q]) co_finish_query(s, q);
        else any_alive = 1;
    }
    s->last_token_time = s->now;
    ++s->bstep;
    if (any_alive) {
        co_schedule_decode(s);
    } else {
        for (uint64_t j = 0; j < s->bn; ++j) { /* a query is slow iff one of its tokens is */
            int slow = s->o[s->bfirst + j] > s->bfirst_slow;
            if (s->labels) s->labels[s->bfirst + j] = (uint8_t)slow;
            s->r->slow_queries += (uint64_t)slow;
        }
        if (s->batches) s->batches[s->r->batches - 1].end = s->now;
        s->r->end_time = s->now;
        co_start_serving(s);
    }
}

/* engine.hpp:693-722 */
static void co_on_forward(co_sim* s, double dur) {
    s->training_inflight = 0;
    s->train_busy += dur;
    uint64_t bytes = s->passes[s->pass_index] * s->m->act_bytes_per_token_per_layer;
    if (s->stream && s->layers[s->cursor].recorded == 0) ++s->r->layers_freed;
    co_record(s, s->cursor, bytes, s->now);
    co_training_peak(s);
    ++s->cursor;
    if (s->cursor == s->L) {
        ++s->pass_index;
        s->cursor = 0;
        if (s->pass_index >= s->npasses) {
            s->phase = PH_BACKWARD;
            s->cursor = s->L - 1;
            if (!co_preempt(s)) co_start_backward(s);
            return;
        }
        if (!co_preempt(s)) co_begin_pass(s);
        return;
    }
    if (!co_preempt(s)) co_schedule_forward(s);
}

/* engine.hpp:761-779 + complete_job :807-813 */
static void co_on_backward(co_sim* s, int64_t a, double dur) {
    s->training_inflight = 0;
    s->train_busy += dur;
    co_layer* e = &s->layers[a];
    if (e->on_device) {
        co_free(s, e->recorded);
        e->on_device = 0;
    }
    e->consumed = 1;
    if (a == 0) {
        uint64_t tokens = s->jp + (s->cpa ? 2 * s->jo : 0);
        s->r->trained_tokens += tokens;
        ++s->r->completed_jobs;
        co_teardown(s);
        return;
    }
    s->cursor = (uint64_t)a - 1;
    if (!co_preempt(s)) co_schedule_backward(s);
}

/* engine.hpp:781-797 */
static void co_on_load(co_sim* s, int64_t a, int64_t gen) {
    if ((uint64_t)gen != s->plan_gen) return;
    co_layer* e = &s->layers[a];
    if (!co_alloc(s, e->recorded)) s->breach = 1;
    e->on_device = 1;
    ++s->r->loads;
    if (s->has_job && s->waiting && s->phase == PH_BACKWARD && s->cursor == (uint64_t)a && !s->serving_busy &&
        s->qhead == s->ai) {
        double waited = s->now - s->wait_since;
        s->r->prefetch_wait_seconds += waited;
        s->train_busy += waited;
        s->waiting = 0;
        co_schedule_backward(s);
    }
}

int orc_replay_sim(const orc_model* m, const orc_gpu* g, const orc_maps* maps, int sim_mode, int mode_cpa,
                   double cache_timeout, const double* arrival, const uint32_t* prompt, const uint32_t* output,
                         const double* label_delay, uint64_t n, double tau, double* samples, uint8_t* labels,
                   orc_batch* batches, orc_colo_report* out) {
    memset(out, 0, sizeof *out);
    if (sim_mode < 0 || sim_mode > 2) return ORC_EINVAL;
    if (orc_validate_profile_pair(m, g) != ORC_OK) return ORC_EVALIDATION; /* engine.hpp:61 */
    co_sim S;
    memset(&S, 0, sizeof S);
    co_sim* s = &S;
    s->m = m;
    s->g = g;
    s->maps = maps;
    s->cpa = mode_cpa;
    s->sim_mode = sim_mode;
    s->cache_timeout = cache_timeout;
    s->arr = arrival;
    s->p = prompt;
    s->o = output;
    s->label_delay = label_delay;
    s->n = n;
    s->L = m->num_layers;
    s->budget = g->capacity_bytes - g->runtime_reserve_bytes - m->weights_bytes;
    s->cap = g->capacity_bytes;
    s->tau = tau;
    s->samples = samples;
    s->labels = labels;
    s->batches = batches;
    s->r = out;
    for (uint64_t i = 0; i < n; ++i) { /* workload.hpp:164-188, engine.hpp:70-74 */
        if (prompt[i] == 0 || output[i] == 0) return ORC_EVALIDATION;
        if (i && arrival[i] < arrival[i - 1]) return ORC_EVALIDATION;
        if (co_need(s, i) > s->budget) return ORC_EVALIDATION;
    }
    s->layers = (co_layer*)calloc(s->L ? s->L : 1, sizeof(co_layer));
    s->bq = (co_bjob*)calloc(n ? n : 1, sizeof(co_bjob));
    s->next_seq = n;
    if (!co_alloc(s, m->weights_bytes + g->runtime_reserve_bytes)) s->breach = 1; /* engine.hpp:141-142 */
    if (sim_mode == ORC_SIM_SEPARATE && !t_alloc(s, m->weights_bytes + g->runtime_reserve_bytes)) s->breach = 1;
    while (!s->breach) {
        /* pop min (time, seq): the next arrival (seq = its index) or a listed event */
        size_t best = (size_t)-1;
        for (size_t i = 0; i < s->nev; ++i)
            if (best == (size_t)-1 || s->ev[i].t < s->ev[best].t ||
                (s->ev[i].t == s->ev[best].t && s->ev[i].seq < s->ev[best].seq))
                best = i;
        int arrival_first = s->ai < n && (best == (size_t)-1 || !(s->ev[best].t < s->arr[s->ai]));
        if (arrival_first) { /* engine.hpp:270-276 */
            s->now = s->arr[s->ai];
            ++s->ai;
            if (s->serving_busy || s->training_inflight) continue;
            co_interrupt_wait(s, 1);
            co_start_serving(s);
            continue;
        }
        if (best == (size_t)-1) break;
        co_ev e = s->ev[best];
        s->ev[best] = s->ev[--s->nev];
        s->now = e.t;
        switch (e.kind) {
            case EV_PREFILL: /* engine.hpp:352-356 */
                s->last_token_time = s->now;
                s->bstep = 0;
                s->bfirst_slow = 0xffffffffu;
                co_schedule_decode(s);
                break;
            case EV_DECODE: co_on_decode(s); break;
            case EV_LABEL: /* engine.hpp:481-496 */
                if (e.a < 0) {
                    co_baseline_enqueue(s, s->p[e.b], s->o[e.b]);
                    break;
                }
                if (s->has_store && s->generation == (uint64_t)e.a && s->has_job && s->phase == PH_WAITING_LABEL) {
                    s->phase = PH_READY;
                    co_try_start_training(s);
                } else {
                    ++s->r->labels_dropped;
                }
                break;
            case EV_TIMEOUT: /* engine.hpp:498-505 */
                if (s->has_store && s->generation == (uint64_t)e.a && s->has_job && s->phase == PH_WAITING_LABEL) {
                    ++s->r->labels_dropped;
                    co_teardown(s);
                }
                break;
            case EV_FWD: co_on_forward(s, e.dur); break;
            case EV_BWD: co_on_backward(s, e.a, e.dur); break;
            case EV_LOAD: co_on_load(s, e.a, e.b); break;
            case EV_BLAYER: co_on_baseline_layer(s, e.dur); break;
        }
    }
    out->training_busy_time = s->train_busy;
    out->peak_device_bytes = sim_mode == ORC_SIM_SEPARATE ? s->t_peak : s->peak; /* engine.hpp:159-161 */
    out->status = s->breach ? ORC_EBREACH : ORC_OK;
    free(s->layers);
    free(s->bq);
    free(s->ev);
    return s->breach ? ORC_EBREACH : ORC_OK;
}

int orc_replay_colocated(const orc_model* m, const orc_gpu* g, const orc_maps* maps, int mode_cpa,
                         double cache_timeout, const double* arrival, const uint32_t* prompt, const uint32_t* output,
                         const double* label_delay, uint64_t n, double tau, double* samples, uint8_t* labels,
                         orc_batch* batches, orc_colo_report* out) {
    return orc_replay_sim(m, g, maps, ORC_SIM_COLOCATED, mode_cpa, cache_timeout, arrival, prompt, output,
                          label_delay, n, tau, samples, labels, batches, out);
}
