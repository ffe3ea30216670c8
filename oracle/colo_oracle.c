/*
 * colo_oracle.c -- TEST INFRASTRUCTURE ONLY (see colo_oracle.h).
 *
 * Plain-C restatement of the colosim admission hot path.  Compiled with
 * -O2 -ffp-contract=off (the reference's Release build is
 * SSE2 without FMA; contraction changes latency bit patterns).  All byte
 * arithmetic is uint64_t with the reference's wrap-around semantics; all
 * latency arithmetic keeps the reference's association order.
 *
 * Reference paths are relative to /root/reference/proj/.
 */
#include "colo_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- verdict packing (the output format; mirrors include/colo_abi.h) ---- */
#define V_ACTION_SHIFT 0
#define V_LAYERS_SHIFT 2
#define V_FREENOW_SHIFT 10
#define V_HEDGE_BIT (1u << 18)
#define V_OFFLOAD_OOR_BIT (1u << 19)
#define V_HEDGE_OOR_BIT (1u << 20)
#define V_VERDICT_SHIFT 21
#define V_STREAM_BIT (1u << 23)
#define V_STREAM_OOR_BIT (1u << 24)

enum { A_NOACTION = 0, A_FREELAYERS = 1, A_ALLTOHOST = 2 };
enum { VD_ADMIT = 0, VD_FREE_LOADBACK = 1, VD_RECOMPUTE_DROP = 2 };

/* ---------------------------------------------------------------- cost model */

/* cost_model.hpp:18-25 */
double orc_prefill_latency(const orc_model* m, uint64_t tokens, uint64_t batch, int recording, int* err) {
    if (tokens == 0 || batch == 0) {
        if (err) *err = ORC_EINVAL;
        return 0.0;
    }
    double t = (double)tokens;
    double base = (double)batch * (m->prefill_coef_linear * t + m->prefill_coef_quad * t * t);
    return recording ? base * m->record_prefill_multiplier : base;
}

/* cost_model.hpp:28-35 */
double orc_decode_step_latency(const orc_model* m, uint64_t ctx, uint64_t batch, int recording, int* err) {
    if (ctx == 0 || batch == 0) {
        if (err) *err = ORC_EINVAL;
        return 0.0;
    }
    double base = (double)batch * (m->decode_coef_const + m->decode_coef_context * (double)ctx);
    return recording ? base * m->record_decode_multiplier : base;
}

/* cost_model.hpp:39-41 */
double orc_forward_layer_latency(const orc_model* m, uint64_t tokens, int* err) {
    return orc_prefill_latency(m, tokens, 1, 0, err) / (double)m->num_layers;
}

/* cost_model.hpp:43-45 */
double orc_backward_layer_latency(const orc_model* m, uint64_t tokens, int* err) {
    return m->backward_to_forward_ratio * orc_forward_layer_latency(m, tokens, err);
}

/* cost_model.hpp:47-52 */
uint64_t orc_activation_bytes(const orc_model* m, uint64_t tokens, uint64_t layers, int* err) {
    if (layers > m->num_layers) {
        if (err) *err = ORC_EINVAL;
        return 0;
    }
    return tokens * layers * m->act_bytes_per_token_per_layer;
}

/* cost_model.hpp:54-56 */
uint64_t orc_kv_bytes(const orc_model* m, uint64_t tokens, uint64_t batch) {
    return batch * tokens * m->kv_bytes_per_token;
}

/* cost_model.hpp:59-66 (std::llround == C llround) */
uint64_t orc_serving_memory(const orc_model* m, uint64_t tokens, uint64_t batch, int* err) {
    if (tokens == 0 || batch == 0) {
        if (err) *err = ORC_EINVAL;
        return 0;
    }
    uint64_t kv = orc_kv_bytes(m, tokens, batch);
    uint64_t workspace = (uint64_t)llround(m->workspace_factor * (double)kv);
    return kv + workspace;
}

/* cost_model.hpp:68-71 */
double orc_transfer_time(const orc_gpu* g, uint64_t bytes, int host_to_device) {
    uint64_t bw = host_to_device ? g->h2d_bandwidth : g->d2h_bandwidth;
    return (double)bytes / (double)bw;
}

/* ------------------------------------------------------------------ profiles */

/* profiles.hpp:37-57, 104-108, 129-134 */
int orc_validate_profile_pair(const orc_model* m, const orc_gpu* g) {
    if (m->num_layers == 0 || m->kv_bytes_per_token == 0 || m->act_bytes_per_token_per_layer == 0 ||
        m->weights_bytes == 0)
        return ORC_EVALIDATION;
    if (!(m->prefill_coef_linear > 0) || !(m->prefill_coef_quad > 0) || !(m->decode_coef_const > 0) ||
        !(m->decode_coef_context > 0) || !(m->backward_to_forward_ratio > 0))
        return ORC_EVALIDATION;
    if (m->record_prefill_multiplier < 1.0 || m->record_decode_multiplier < 1.0) return ORC_EVALIDATION;
    if (m->workspace_factor < 0.0) return ORC_EVALIDATION;
    if (g->capacity_bytes == 0 || g->h2d_bandwidth == 0 || g->d2h_bandwidth == 0) return ORC_EVALIDATION;
    if (m->weights_bytes + g->runtime_reserve_bytes >= g->capacity_bytes) return ORC_EVALIDATION;
    return ORC_OK;
}

/* profiles.hpp:137-152: FNV-1a over the '|'-joined canonical fields, doubles
 * printed as an ostream with precision(17) (== printf "%.17g"). */
uint64_t orc_profile_hash(const orc_model* m, const orc_gpu* g) {
    char buf[1024];
    int len = snprintf(buf, sizeof buf,
                       "%llu|%llu|%llu|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%llu|%llu|%llu|%llu|%llu",
                       (unsigned long long)m->num_layers, (unsigned long long)m->kv_bytes_per_token,
                       (unsigned long long)m->act_bytes_per_token_per_layer, m->prefill_coef_linear,
                       m->prefill_coef_quad, m->decode_coef_const, m->decode_coef_context,
                       m->backward_to_forward_ratio, m->record_prefill_multiplier,
                       m->record_decode_multiplier, m->workspace_factor, (unsigned long long)m->weights_bytes,
                       (unsigned long long)g->capacity_bytes, (unsigned long long)g->h2d_bandwidth,
                       (unsigned long long)g->d2h_bandwidth, (unsigned long long)g->runtime_reserve_bytes);
    uint64_t h = 14695981039346656037ull;
    for (int i = 0; i < len; ++i) {
        h ^= (unsigned char)buf[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* ---------------------------------------------------------------------- maps */

/* maps.hpp:28-30 */
uint64_t orc_round_up_bucket(uint64_t value, uint64_t step) { return (value + step - 1) / step * step; }

/* maps.hpp:54-61, 215-231 -- the exact order of the reference's checks. */
void orc_offload_cell_decision(const orc_model* m, const orc_gpu* g, int mode_cpa, uint64_t cached,
                               uint64_t incoming, uint64_t batch, int* action, uint64_t* layers) {
    uint64_t budget = g->capacity_bytes - g->runtime_reserve_bytes - m->weights_bytes;
    uint64_t acts = cached * m->num_layers * m->act_bytes_per_token_per_layer;
    uint64_t kv = mode_cpa ? orc_kv_bytes(m, cached, 1) : 0;
    *layers = 0;
    if (acts + kv > budget) { *action = A_ALLTOHOST; return; }
    uint64_t headroom = budget - acts - kv;
    uint64_t need = orc_serving_memory(m, incoming, batch, NULL);
    if (need <= headroom) { *action = A_NOACTION; return; }
    uint64_t deficit = need - headroom;
    uint64_t per_layer = cached * m->act_bytes_per_token_per_layer;
    if (per_layer == 0) { *action = A_ALLTOHOST; return; }
    uint64_t n = (deficit + per_layer - 1) / per_layer;
    if (n > m->num_layers) { *action = A_ALLTOHOST; return; }
    *action = A_FREELAYERS;
    *layers = n;
}

/* maps.hpp:197-208 */
int orc_validate_grid(const orc_grid* s) {
    if (s->cached_step == 0 || s->incoming_step == 0 || s->batch_step == 0) return ORC_EVALIDATION;
    if (s->max_cached == 0 || s->max_incoming == 0 || s->max_batch == 0) return ORC_EVALIDATION;
    if (s->max_cached % s->cached_step || s->max_incoming % s->incoming_step || s->max_batch % s->batch_step)
        return ORC_EVALIDATION;
    return ORC_OK;
}

static uint8_t encode_cell(int action, uint64_t layers) {
    if (action == A_NOACTION) return 0;
    if (action == A_ALLTOHOST) return 1;
    return (uint8_t)(2 + layers);
}

static void decode_cell(uint8_t c, int* action, uint64_t* layers) {
    if (c == 0) { *action = A_NOACTION; *layers = 0; }
    else if (c == 1) { *action = A_ALLTOHOST; *layers = 0; }
    else { *action = A_FREELAYERS; *layers = (uint64_t)(c - 2); }
}

/* maps.hpp:85-87: cached_count = max/step + 1, incoming_count = max/step, batch_count = max/step */
static size_t n_offload_cells(const orc_grid* g) {
    return (size_t)(g->max_cached / g->cached_step + 1) * (size_t)(g->max_incoming / g->incoming_step) *
           (size_t)(g->max_batch / g->batch_step);
}

/* maps.hpp:233-252; cell (ci,ii,bi) at (ci*sc, (ii+1)*si, (bi+1)*sb), row-major (maps.hpp:89-94) */
int orc_build_offloading_map(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int mode_cpa,
                             uint8_t* cells, size_t ncells) {
    if (orc_validate_profile_pair(m, g)) return ORC_EVALIDATION;
    if (orc_validate_grid(grid)) return ORC_EVALIDATION;
    if (m->num_layers > 253) return ORC_EINVAL; /* cell code width */
    if (ncells != n_offload_cells(grid)) return ORC_EINVAL;
    size_t C = grid->max_cached / grid->cached_step + 1, I = grid->max_incoming / grid->incoming_step,
           B = grid->max_batch / grid->batch_step;
    for (size_t ci = 0; ci < C; ++ci)
        for (size_t ii = 0; ii < I; ++ii)
            for (size_t bi = 0; bi < B; ++bi) {
                int a;
                uint64_t l;
                orc_offload_cell_decision(m, g, mode_cpa, ci * grid->cached_step, (ii + 1) * grid->incoming_step,
                                          (bi + 1) * grid->batch_step, &a, &l);
                cells[(ci * I + ii) * B + bi] = encode_cell(a, l);
            }
    return ORC_OK;
}

/* maps.hpp:100-110; returns 1 = has_value, 0 = nullopt */
int orc_offload_lookup(const orc_grid* grid, const uint8_t* cells, uint64_t cached, uint64_t incoming,
                       uint64_t batch, int* action, uint64_t* layers) {
    uint64_t cb = orc_round_up_bucket(cached, grid->cached_step);
    uint64_t ib = orc_round_up_bucket(incoming, grid->incoming_step);
    uint64_t bb = orc_round_up_bucket(batch, grid->batch_step);
    if (cb > grid->max_cached || ib > grid->max_incoming || bb > grid->max_batch) return 0;
    if (incoming == 0 || batch == 0) return 0;
    size_t I = grid->max_incoming / grid->incoming_step, B = grid->max_batch / grid->batch_step;
    size_t ci = cb / grid->cached_step, ii = ib / grid->incoming_step - 1, bi = bb / grid->batch_step - 1;
    decode_cell(cells[(ci * I + ii) * B + bi], action, layers);
    return 1;
}

/* maps.hpp:341-346 */
double orc_hedge_recompute_time(const orc_model* m, int mode_cpa, uint64_t cached, uint64_t assumed_out,
                                int* err) {
    if (mode_cpa) return 2.0 * orc_prefill_latency(m, assumed_out, 1, 0, err);
    return orc_prefill_latency(m, cached, 1, 0, err);
}

/* maps.hpp:349-356 (std::max(0.0, x) == (0.0 < x) ? x : 0.0) */
double orc_hedge_residual_load_time(const orc_model* m, const orc_gpu* g, uint64_t cached, uint64_t freed,
                                    int* err) {
    double load = orc_transfer_time(g, orc_activation_bytes(m, cached, freed, err), 1);
    double credit = (double)(m->num_layers - freed) * orc_backward_layer_latency(m, cached == 0 ? 1 : cached, err);
    double x = load - credit;
    return (0.0 < x) ? x : 0.0;
}

/* maps.hpp:358-384; cells row-major (ci, fi) with cached_count = max/step, freed_count = L+1 */
int orc_build_hedging_map(const orc_model* m, const orc_gpu* g, uint64_t cached_step, uint64_t max_cached,
                          int mode_cpa, uint64_t assumed_out, uint8_t* cells, size_t ncells) {
    if (orc_validate_profile_pair(m, g)) return ORC_EVALIDATION;
    if (cached_step == 0 || max_cached == 0 || max_cached % cached_step) return ORC_EVALIDATION;
    size_t C = max_cached / cached_step, F = m->num_layers + 1;
    if (ncells != C * F) return ORC_EINVAL;
    for (size_t ci = 0; ci < C; ++ci) {
        uint64_t cached = (ci + 1) * cached_step;
        int err = 0;
        double recompute = orc_hedge_recompute_time(m, mode_cpa, cached, assumed_out, &err);
        if (err) return ORC_EINVAL;
        for (size_t fi = 0; fi < F; ++fi) {
            double residual = orc_hedge_residual_load_time(m, g, cached, fi, &err);
            cells[ci * F + fi] = residual > recompute ? 1 : 0;
        }
    }
    return ORC_OK;
}

/* maps.hpp:276-280 */
int orc_hedge_lookup(uint64_t cached_step, uint64_t max_cached, uint64_t num_layers, const uint8_t* cells,
                     uint64_t cached, uint64_t freed, int* recompute) {
    uint64_t cb = orc_round_up_bucket(cached, cached_step);
    if (cb == 0 || cb > max_cached || freed > num_layers) return 0;
    *recompute = cells[(cb / cached_step - 1) * (num_layers + 1) + freed];
    return 1;
}

/* -------------------------------------------------------- decision composition */

static uint32_t pack(int action, uint64_t layers, uint64_t free_now, int recompute, int off_oor, int hedge_oor,
                     int verdict, int stream, int stream_oor) {
    uint32_t v = (uint32_t)action << V_ACTION_SHIFT;
    v |= (uint32_t)(layers & 0xff) << V_LAYERS_SHIFT;
    v |= (uint32_t)(free_now & 0xff) << V_FREENOW_SHIFT;
    if (recompute) v |= V_HEDGE_BIT;
    if (off_oor) v |= V_OFFLOAD_OOR_BIT;
    if (hedge_oor) v |= V_HEDGE_OOR_BIT;
    v |= (uint32_t)verdict << V_VERDICT_SHIFT;
    if (stream) v |= V_STREAM_BIT;
    if (stream_oor) v |= V_STREAM_OOR_BIT;
    return v;
}

/* engine.hpp:513-557 (apply_offload_decision, the decision half) and
 * engine.hpp:437-444 (admit_to_store's streaming pre-commitment for `charged`).
 * pending = store.host_only_pending(), dev_layers = store.device_resident_layers(). */
static uint32_t verdict64(const orc_maps* mp, uint64_t cached, uint64_t incoming, uint64_t batch, uint64_t pending,
                          uint64_t dev_layers, uint64_t charged) {
    const uint64_t L = mp->num_layers;
    int action;
    uint64_t layers;
    int fallback = !orc_offload_lookup(&mp->grid, mp->offload_cells, cached, incoming, batch, &action, &layers);
    if (fallback) { action = A_ALLTOHOST; layers = 0; }                                 /* :517-521 */
    int recompute = 0, hedge_oor = 0, verdict = VD_ADMIT;
    uint64_t free_now = 0;
    if (action != A_NOACTION) {                                                           /* :522 */
        free_now = action == A_ALLTOHOST ? dev_layers : (layers < dev_layers ? layers : dev_layers); /* :524-527 */
        uint64_t ltf = action == A_ALLTOHOST ? L : layers;                                /* maps.hpp:41-48 */
        uint64_t total = pending + ltf < L ? pending + ltf : L;                           /* :528-530 */
        recompute = 1;                                                                    /* :532 */
        if (!fallback) {
            int r;
            if (orc_hedge_lookup(mp->hedge_step, mp->hedge_max, L, mp->hedge_cells, cached, total, &r))
                recompute = r;
            else
                hedge_oor = 1;                                                            /* :537-538 */
        }
        verdict = recompute ? VD_RECOMPUTE_DROP : VD_FREE_LOADBACK;                       /* :541-548 */
    }
    int sa;
    uint64_t sl;
    int stream_oor = !orc_offload_lookup(&mp->grid, mp->offload_cells, charged, 1, 1, &sa, &sl);
    int stream = stream_oor || sa == A_ALLTOHOST;                                        /* :438-444 */
    return pack(action, layers, free_now, recompute, fallback, hedge_oor, verdict, stream, stream_oor);
}

uint32_t orc_verdict(const orc_maps* maps, const orc_tuple* t) {
    return verdict64(maps, t->cached, t->incoming, t->batch, t->pending, t->dev_layers, t->charged);
}

void orc_decide(const orc_maps* maps, const orc_tuple* in, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_verdict(maps, &in[i]);
}

/* Exact per-query variant: offload_cell_decision at the
 * un-quantised point + the hedge inequality evaluated directly
 * (maps.hpp:215-231, 341-356, 380).  Domain rules mirror the lookups:
 * incoming==0 || batch==0 -> offload out-of-range (serving_memory throws,
 * cost_model.hpp:60-61); cached==0 -> hedge out-of-range (lookup's cb==0,
 * maps.hpp:278; CPT prefill(0) throws, cost_model.hpp:20). */
uint32_t orc_verdict_exact(const orc_model* m, const orc_gpu* g, int mode_cpa, uint64_t assumed_out,
                           const orc_tuple* t) {
    const uint64_t L = m->num_layers;
    uint64_t cached = t->cached, incoming = t->incoming, batch = t->batch;
    int action;
    uint64_t layers = 0;
    int fallback = incoming == 0 || batch == 0;
    if (fallback) action = A_ALLTOHOST;
    else orc_offload_cell_decision(m, g, mode_cpa, cached, incoming, batch, &action, &layers);
    int recompute = 0, hedge_oor = 0, verdict = VD_ADMIT;
    uint64_t free_now = 0;
    if (action != A_NOACTION) {
        uint64_t dev = t->dev_layers;
        free_now = action == A_ALLTOHOST ? dev : (layers < dev ? layers : dev);
        uint64_t ltf = action == A_ALLTOHOST ? L : layers;
        uint64_t total = t->pending + ltf < L ? t->pending + ltf : L;
        recompute = 1;
        if (!fallback) {
            if (cached == 0) {
                hedge_oor = 1;
            } else {
                int err = 0;
                double rc = orc_hedge_recompute_time(m, mode_cpa, cached, assumed_out, &err);
                double res = orc_hedge_residual_load_time(m, g, cached, total, &err);
                recompute = res > rc;
            }
        }
        verdict = recompute ? VD_RECOMPUTE_DROP : VD_FREE_LOADBACK;
    }
    int sa;
    uint64_t sl;
    orc_offload_cell_decision(m, g, mode_cpa, t->charged, 1, 1, &sa, &sl);
    int stream = sa == A_ALLTOHOST;
    return pack(action, layers, free_now, recompute, fallback, hedge_oor, verdict, stream, 0);
}

void orc_decide_exact(const orc_model* m, const orc_gpu* g, int mode_cpa, uint64_t assumed_out,
                      const orc_tuple* in, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_verdict_exact(m, g, mode_cpa, assumed_out, &in[i]);
}

/* --------------------------------------------------------- trace-fused decide */

/* Charged tokens of a query: engine.hpp:422-423. */
static uint64_t charged_of(uint32_t p, uint32_t o, int cpa) {
    return cpa ? (uint64_t)p + 2ull * (uint64_t)o : (uint64_t)p;
}

/* SURVEY §8(d) C2 rule: query i of device d asks the slot question with
 * cached = charged(previous query of d) (0 for the first), incoming = p+o,
 * batch = 1, pending = 0, dev_layers = L, charged = charged(i). */
int orc_features_decide(const orc_maps* const* sets, const int* set_is_cpa, size_t nsets,
                        const uint32_t* prompt, const uint32_t* output, const uint64_t* dev_offsets,
                        const uint16_t* dev_set, size_t ndev, uint32_t* out) {
    for (size_t d = 0; d < ndev; ++d) {
        if (dev_set[d] >= nsets) return ORC_EINVAL;
        const orc_maps* mp = sets[dev_set[d]];
        int cpa = set_is_cpa[dev_set[d]];
        uint64_t prev = 0;
        for (uint64_t i = dev_offsets[d]; i < dev_offsets[d + 1]; ++i) {
            uint64_t ch = charged_of(prompt[i], output[i], cpa);
            out[i] = verdict64(mp, prev, (uint64_t)prompt[i] + output[i], 1, 0, mp->num_layers, ch);
            prev = ch;
        }
    }
    return ORC_OK;
}

/* Per-query cost-model features: need = serving_memory(p+o, 1)
 * (engine.hpp:297), charged (engine.hpp:422-423), unrecorded prefill latency
 * (engine.hpp:324). */
int orc_features(const orc_model* m, int mode_cpa, const uint32_t* prompt, const uint32_t* output, size_t n,
                 uint64_t* need, uint64_t* charged, double* prefill) {
    for (size_t i = 0; i < n; ++i) {
        int err = 0;
        need[i] = orc_serving_memory(m, (uint64_t)prompt[i] + output[i], 1, &err);
        charged[i] = charged_of(prompt[i], output[i], mode_cpa);
        prefill[i] = orc_prefill_latency(m, prompt[i], 1, 0, &err);
        if (err) return ORC_EINVAL;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------ serving replay */

/* ServingOnly Simulation::run restated as the batch recurrence (SURVEY
 * Appendix A.2, verified bit-exact against the event loop):
 *   event order engine.hpp:146-147,178-188 (arrivals carry the lowest seq);
 *   on_arrival :270-276 (an idle server starts a batch on the first pop);
 *   start_serving_batch :282-328 (FIFO, at least one, sum(need) <= budget,
 *   prefill left fold :322-325); schedule_decode_step :358-365 (left fold over
 *   alive queries in batch order); on_decode_step :367-387 (one TPT sample per
 *   alive query, now - last_token_time).
 * Labels (a rule new to this build): a token is slow iff its
 * TPT > tau; a query is slow iff any of its tokens is slow.
 * Replay-derived verdicts (SURVEY §8(d) C3 rule): each batch asks
 * (cached = charged of the last single-query batch, incoming = max_incoming,
 * batch = n, pending = 0, dev_layers = L, charged = charged(first query)). */
int orc_replay_serving(const orc_model* m, const orc_gpu* g, const double* arrival, const uint32_t* prompt,
                       const uint32_t* output, uint64_t n, double tau, const orc_maps* maps, int mode_cpa,
                       double* samples, uint8_t* labels, orc_batch* batches, orc_replay_summary* out) {
    const uint64_t budget = g->capacity_bytes - g->runtime_reserve_bytes - m->weights_bytes; /* :278-280 */
    memset(out, 0, sizeof *out);
    uint64_t* need = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        if (prompt[i] == 0 || output[i] == 0) { free(need); return ORC_EVALIDATION; } /* workload.hpp:176-181 */
        if (i && arrival[i] < arrival[i - 1]) { free(need); return ORC_EVALIDATION; }
        need[i] = orc_serving_memory(m, (uint64_t)prompt[i] + output[i], 1, NULL);
        if (need[i] > budget) { free(need); return ORC_EVALIDATION; }                     /* :70-74 */
    }
    uint64_t max_need_total = 0, sample_pos = 0, slot_charged = 0;
    double T = -INFINITY;
    uint64_t head = 0, tail = 0;
    while (head < n) {
        if (arrival[head] > T) {                 /* idle: first arrival starts a batch alone */
            T = arrival[head];
            tail = head + 1;
        } else {                                 /* queued: everything that arrived by T */
            if (tail < head) tail = head;        /* T never decreases: resume the scan (linear overall) */
            while (tail < n && arrival[tail] <= T) ++tail;
        }
        uint64_t end = head, need_total = 0;
        uint64_t max_inc = 0;
        uint32_t maxo = 0;
        while (end < tail && (end == head || need_total + need[end] <= budget)) {
            need_total += need[end];
            uint64_t inc = (uint64_t)prompt[end] + output[end];
            if (inc > max_inc) max_inc = inc;
            if (output[end] > maxo) maxo = output[end];
            ++end;
        }
        if (need_total > max_need_total) max_need_total = need_total;
        uint32_t verdict = 0;
        if (maps) {
            uint64_t ch_first = charged_of(prompt[head], output[head], mode_cpa);
            verdict = verdict64(maps, slot_charged, max_inc, end - head, 0, m->num_layers, ch_first);
            if (end - head == 1) slot_charged = ch_first;
        }
        double dur = 0.0;
        for (uint64_t j = head; j < end; ++j) dur += orc_prefill_latency(m, prompt[j], 1, 0, NULL);
        double start = T + 0.0;
        double now = start + dur;
        double last = now;
        uint32_t first_slow = maxo; /* first step whose sample exceeds tau */
        for (uint32_t k = 0; k < maxo; ++k) {
            double d = 0.0;
            uint64_t alive = 0;
            for (uint64_t j = head; j < end; ++j)
                if (k < output[j]) {
                    d += orc_decode_step_latency(m, (uint64_t)prompt[j] + k, 1, 0, NULL);
                    ++alive;
                }
            now = now + d;
            double s = now - last;
            last = now;
            if (samples)
                for (uint64_t a = 0; a < alive; ++a) samples[sample_pos + a] = s;
            sample_pos += alive;
            out->generated_tokens += alive;
            if (s > tau) {
                out->slow_tokens += alive;
                if (k < first_slow) first_slow = k;
            }
        }
        for (uint64_t j = head; j < end; ++j) {
            int slow = output[j] > first_slow;
            if (labels) labels[j] = (uint8_t)slow;
            out->slow_queries += (uint64_t)slow;
        }
        if (batches) {
            orc_batch* b = &batches[out->batches];
            b->start = start;
            b->end = now;
            b->first = (uint32_t)head;
            b->n = (uint32_t)(end - head);
            b->need_total = need_total;
            b->max_incoming = max_inc > 0xffffffffull ? 0xffffffffu : (uint32_t)max_inc;
            b->verdict = verdict;
        }
        if (end - head > out->max_batch_size) out->max_batch_size = end - head;
        out->batches++;
        T = now;
        head = end;
    }
    out->peak_device_bytes = m->weights_bytes + g->runtime_reserve_bytes + max_need_total; /* memory.hpp:28-35 */
    out->end_time = n ? T : 0.0;
    free(need);
    return ORC_OK;
}

/* ------------------------------------------------------------------- metrics */

/* metrics.hpp:48-53 */
double orc_nearest_rank(const double* sorted, size_t n, double q) {
    size_t rank = (size_t)ceil(q * (double)n);
    if (rank == 0) rank = 1;
    return sorted[rank - 1];
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* metrics.hpp:56-66 (sort, nearest-rank, sequential mean over the sorted samples) */
int orc_finalize(const double* samples, size_t n, double* p50, double* p90, double* p99, double* mean) {
    if (n == 0) return ORC_EINVAL;
    double* s = (double*)malloc(sizeof(double) * n);
    memcpy(s, samples, sizeof(double) * n);
    qsort(s, n, sizeof(double), cmp_double);
    *p50 = orc_nearest_rank(s, n, 0.50);
    *p90 = orc_nearest_rank(s, n, 0.90);
    *p99 = orc_nearest_rank(s, n, 0.99);
    double sum = 0;
    for (size_t i = 0; i < n; ++i) sum += s[i];
    *mean = sum / (double)n;
    free(s);
    return ORC_OK;
}

/* ------------------------------------------------------------------ workload */

/* std::mt19937_64 (the reference's Rng engine, workload.hpp:20-32) */
typedef struct { uint64_t mt[312]; int mti; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull, A = 0xB5026F5AA96619E9ull;
    if (s->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        }
        for (; i < 311; ++i) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        }
        uint64_t x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1ull) ? A : 0ull);
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= (x >> 43);
    return x;
}

/* workload.hpp:25 */
static double uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

/* workload.hpp:90-107 */
static double sample_raw(const orc_dist* d, mt64* s) {
    switch (d->kind) {
        case 0: return d->fixed_value;
        case 1: return d->lo + (d->hi - d->lo) * uniform01(s);
        default: {
            double u = uniform01(s), acc = 0;
            for (size_t i = 0; i < d->nbins; ++i) {
                acc += d->bin_probs[i];
                if (u < acc) return d->bin_values[i];
            }
            return d->bin_values[d->nbins - 1];
        }
    }
}

/* workload.hpp:193-220 (output_tokens fixed at 128, :214); returns the number
 * of queries, or -1 when `cap` is too small. */
int64_t orc_generate_trace(double qps, double duration, const orc_dist* lengths, const orc_dist* label_delay,
                           uint64_t seed, double* arrival, uint32_t* prompt, uint32_t* output, double* label_out,
                           size_t cap) {
    mt64 s;
    mt64_seed(&s, seed);
    double t = 0;
    size_t n = 0;
    for (;;) {
        t += -log(1.0 - uniform01(&s)) / qps; /* workload.hpp:28 */
        if (t > duration) break;
        if (n >= cap) return -1;
        double raw = sample_raw(lengths, &s);
        uint64_t tok = (uint64_t)llround(raw < 1.0 ? 1.0 : raw); /* workload.hpp:111-116 (std::max(raw,1.0)) */
        if (lengths->min_tokens && tok < lengths->min_tokens) tok = lengths->min_tokens;
        arrival[n] = t;
        prompt[n] = (uint32_t)tok;
        output[n] = 128;
        double ld = -1.0; /* nullopt (content_hash convention, workload.hpp:156) */
        if (label_delay) { /* sample_seconds, workload.hpp:118-120 */
            double raw = sample_raw(label_delay, &s);
            ld = 0.0 < raw ? raw : 0.0;
        }
        if (label_out) label_out[n] = ld;
        ++n;
    }
    return (int64_t)n;
}
