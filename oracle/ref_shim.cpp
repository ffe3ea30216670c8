// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNCHANGED reference headers (/root/reference/proj/include,
// read-only, never copied) into oracle/_ref/libcolo_ref.so and exposes the
// hot-path functions through the same C signatures as colo_oracle.h (prefix
// ref_).  It is used (a) to pin the plain-C restatement in colo_oracle.c and
// (b) by tests/golden/make_golden.py to write the committed golden fixtures,
// and (c) as bench.py's `--impl reference` CPU arm.  Built by oracle/Makefile.
//
// Where the reference has no free function for a step (the decision
// composition lives inside Simulation::apply_offload_decision,
// engine.hpp:513-557, and admit_to_store, engine.hpp:434-448) this shim calls
// the reference's own OffloadingMap::lookup / HedgingMap::lookup and composes
// them exactly as those engine lines do.  The serving replay is the
// reference's Simulation::run in ServingOnly mode; batch membership is read
// back from its own event log (PrefillDone carries the batch size,
// engine.hpp:353).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <vector>

#include "colosim/cost_model.hpp"
#include "colosim/engine.hpp"
#include "colosim/maps.hpp"
#include "colosim/metrics.hpp"
#include "colosim/profiles.hpp"
#include "colosim/workload.hpp"

#include "colo_oracle.h"

using namespace colosim;

namespace {

ModelProfile to_model(const orc_model* m) {
    ModelProfile r;
    r.num_layers = m->num_layers;
    r.kv_bytes_per_token = m->kv_bytes_per_token;
    r.act_bytes_per_token_per_layer = m->act_bytes_per_token_per_layer;
    r.prefill_coef_linear = m->prefill_coef_linear;
    r.prefill_coef_quad = m->prefill_coef_quad;
    r.decode_coef_const = m->decode_coef_const;
    r.decode_coef_context = m->decode_coef_context;
    r.backward_to_forward_ratio = m->backward_to_forward_ratio;
    r.record_prefill_multiplier = m->record_prefill_multiplier;
    r.record_decode_multiplier = m->record_decode_multiplier;
    r.workspace_factor = m->workspace_factor;
    r.weights_bytes = m->weights_bytes;
    return r;
}

GpuProfile to_gpu(const orc_gpu* g) {
    GpuProfile r;
    r.capacity_bytes = g->capacity_bytes;
    r.h2d_bandwidth = g->h2d_bandwidth;
    r.d2h_bandwidth = g->d2h_bandwidth;
    r.runtime_reserve_bytes = g->runtime_reserve_bytes;
    return r;
}

TrainingMode to_mode(int cpa) { return cpa ? TrainingMode::CPA : TrainingMode::CPT; }

uint8_t code_of(const OffloadDecision& d) {
    switch (d.action) {
        case OffloadAction::NoAction: return 0;
        case OffloadAction::AllToHost: return 1;
        case OffloadAction::FreeLayers: return static_cast<uint8_t>(2 + d.layers);
    }
    return 0;
}

uint32_t pack(int action, uint64_t layers, uint64_t free_now, bool recompute, bool off_oor, bool hedge_oor,
              int verdict, bool stream, bool stream_oor) {
    uint32_t v = static_cast<uint32_t>(action);
    v |= static_cast<uint32_t>(layers & 0xff) << 2;
    v |= static_cast<uint32_t>(free_now & 0xff) << 10;
    if (recompute) v |= 1u << 18;
    if (off_oor) v |= 1u << 19;
    if (hedge_oor) v |= 1u << 20;
    v |= static_cast<uint32_t>(verdict) << 21;
    if (stream) v |= 1u << 23;
    if (stream_oor) v |= 1u << 24;
    return v;
}

int action_id(OffloadAction a) {
    return a == OffloadAction::NoAction ? 0 : a == OffloadAction::FreeLayers ? 1 : 2;
}

struct Maps {
    OffloadingMap off;
    HedgingMap hedge;
};

// engine.hpp:513-557 (decision half) + engine.hpp:437-444, using the
// reference's own lookups.
uint32_t compose(const Maps& mp, uint64_t L, uint64_t cached, uint64_t incoming, uint64_t batch, uint64_t pending,
                 uint64_t dev_layers, uint64_t charged) {
    auto dec = mp.off.lookup(cached, incoming, batch);
    bool fallback = !dec;
    if (fallback) dec = OffloadDecision{OffloadAction::AllToHost, 0};
    bool recompute = false, hedge_oor = false;
    int verdict = 0;
    uint64_t free_now = 0;
    if (dec->action != OffloadAction::NoAction) {
        free_now = dec->action == OffloadAction::AllToHost ? dev_layers
                                                            : std::min<std::uint64_t>(dec->layers, dev_layers);
        uint64_t total_freed = std::min(pending + dec->layers_to_free(L), L);
        HedgeDecision hedge = HedgeDecision::Recompute;
        if (!fallback) {
            auto h = mp.hedge.lookup(cached, total_freed);
            if (h)
                hedge = *h;
            else
                hedge_oor = true;
        }
        recompute = hedge == HedgeDecision::Recompute;
        verdict = recompute ? 2 : 1;
    }
    bool stream = false, stream_oor = false;
    auto cell = mp.off.lookup(charged, 1, 1);
    if (!cell) {
        stream = true;
        stream_oor = true;
    } else if (cell->action == OffloadAction::AllToHost) {
        stream = true;
    }
    return pack(action_id(dec->action), dec->action == OffloadAction::FreeLayers ? dec->layers : 0, free_now,
                recompute, fallback, hedge_oor, verdict, stream, stream_oor);
}

Maps make_maps(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int cpa, uint64_t hedge_step,
               uint64_t hedge_max, uint64_t assumed) {
    ModelProfile mm = to_model(m);
    GpuProfile gg = to_gpu(g);
    GridSteps s{grid->cached_step, grid->incoming_step, grid->batch_step};
    GridBounds b{grid->max_cached, grid->max_incoming, grid->max_batch};
    Maps mp;
    mp.off = build_offloading_map(mm, gg, s, b, to_mode(cpa));
    mp.hedge = build_hedging_map(mm, gg, hedge_step, hedge_max, to_mode(cpa), assumed);
    return mp;
}

}  // namespace

extern "C" {

double ref_prefill_latency(const orc_model* m, uint64_t tokens, uint64_t batch, int rec, int* err) {
    try { return prefill_latency(to_model(m), tokens, batch, rec != 0); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}
double ref_decode_step_latency(const orc_model* m, uint64_t ctx, uint64_t batch, int rec, int* err) {
    try { return decode_step_latency(to_model(m), ctx, batch, rec != 0); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}
double ref_forward_layer_latency(const orc_model* m, uint64_t tokens, int* err) {
    try { return forward_layer_latency(to_model(m), tokens); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}
double ref_backward_layer_latency(const orc_model* m, uint64_t tokens, int* err) {
    try { return backward_layer_latency(to_model(m), tokens); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}
uint64_t ref_activation_bytes(const orc_model* m, uint64_t tokens, uint64_t layers, int* err) {
    try { return activation_bytes(to_model(m), tokens, layers); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0; }
}
uint64_t ref_kv_bytes(const orc_model* m, uint64_t tokens, uint64_t batch) { return kv_bytes(to_model(m), tokens, batch); }
uint64_t ref_serving_memory(const orc_model* m, uint64_t tokens, uint64_t batch, int* err) {
    try { return serving_memory(to_model(m), tokens, batch); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0; }
}
double ref_transfer_time(const orc_gpu* g, uint64_t bytes, int h2d) {
    return transfer_time(to_gpu(g), bytes, h2d ? CopyDirection::HostToDevice : CopyDirection::DeviceToHost);
}
int ref_validate_profile_pair(const orc_model* m, const orc_gpu* g) {
    try { validate_profile_pair(to_model(m), to_gpu(g)); return ORC_OK; } catch (const std::exception&) { return ORC_EVALIDATION; }
}
uint64_t ref_profile_hash(const orc_model* m, const orc_gpu* g) { return profile_hash(to_model(m), to_gpu(g)); }
uint64_t ref_round_up_bucket(uint64_t v, uint64_t s) { return round_up_bucket(v, s); }

void ref_offload_cell_decision(const orc_model* m, const orc_gpu* g, int cpa, uint64_t c, uint64_t i, uint64_t b,
                               int* action, uint64_t* layers) {
    OffloadDecision d = offload_cell_decision(to_model(m), to_gpu(g), to_mode(cpa), c, i, b);
    *action = action_id(d.action);
    *layers = d.layers;
}

int ref_build_offloading_map(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int cpa, uint8_t* cells,
                             size_t ncells) {
    try {
        OffloadingMap map = build_offloading_map(to_model(m), to_gpu(g),
                                                 GridSteps{grid->cached_step, grid->incoming_step, grid->batch_step},
                                                 GridBounds{grid->max_cached, grid->max_incoming, grid->max_batch},
                                                 to_mode(cpa));
        size_t C = map.cached_count(), I = map.incoming_count(), B = map.batch_count();
        if (C * I * B != ncells) return ORC_EINVAL;
        for (size_t ci = 0; ci < C; ++ci)
            for (size_t ii = 0; ii < I; ++ii)
                for (size_t bi = 0; bi < B; ++bi) cells[(ci * I + ii) * B + bi] = code_of(map.cell(ci, ii, bi));
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

int ref_build_hedging_map(const orc_model* m, const orc_gpu* g, uint64_t step, uint64_t maxc, int cpa,
                          uint64_t assumed, uint8_t* cells, size_t ncells) {
    try {
        HedgingMap map = build_hedging_map(to_model(m), to_gpu(g), step, maxc, to_mode(cpa), assumed);
        size_t C = map.cached_count(), F = map.freed_count();
        if (C * F != ncells) return ORC_EINVAL;
        for (size_t ci = 0; ci < C; ++ci)
            for (size_t fi = 0; fi < F; ++fi)
                cells[ci * F + fi] = map.cell(ci, fi) == HedgeDecision::Recompute ? 1 : 0;
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

double ref_hedge_recompute_time(const orc_model* m, int cpa, uint64_t cached, uint64_t assumed, int* err) {
    try { return hedge_recompute_time(to_model(m), to_mode(cpa), cached, assumed); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}
double ref_hedge_residual_load_time(const orc_model* m, const orc_gpu* g, uint64_t cached, uint64_t freed, int* err) {
    try { return hedge_residual_load_time(to_model(m), to_gpu(g), cached, freed); } catch (const std::exception&) { if (err) *err = ORC_EINVAL; return 0.0; }
}

/* Composed verdicts through the reference's own map objects. */
int ref_decide(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int cpa, uint64_t hedge_step,
               uint64_t hedge_max, uint64_t assumed, const orc_tuple* in, size_t n, uint32_t* out) {
    try {
        Maps mp = make_maps(m, g, grid, cpa, hedge_step, hedge_max, assumed);
        for (size_t i = 0; i < n; ++i)
            out[i] = compose(mp, m->num_layers, in[i].cached, in[i].incoming, in[i].batch, in[i].pending,
                             in[i].dev_layers, in[i].charged);
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

/* Exact per-query verdicts: offload_cell_decision (maps.hpp:215) at the raw
 * point and the hedge inequality of maps.hpp:376-380 evaluated directly. */
int ref_decide_exact(const orc_model* m, const orc_gpu* g, int cpa, uint64_t assumed, const orc_tuple* in, size_t n,
                     uint32_t* out) {
    ModelProfile mm = to_model(m);
    GpuProfile gg = to_gpu(g);
    TrainingMode mode = to_mode(cpa);
    const uint64_t L = mm.num_layers;
    for (size_t i = 0; i < n; ++i) {
        const orc_tuple& t = in[i];
        bool fallback = t.incoming == 0 || t.batch == 0;
        OffloadDecision dec{OffloadAction::AllToHost, 0};
        if (!fallback) dec = offload_cell_decision(mm, gg, mode, t.cached, t.incoming, t.batch);
        bool recompute = false, hedge_oor = false;
        int verdict = 0;
        uint64_t free_now = 0;
        if (dec.action != OffloadAction::NoAction) {
            free_now = dec.action == OffloadAction::AllToHost ? t.dev_layers
                                                               : std::min<std::uint64_t>(dec.layers, t.dev_layers);
            uint64_t total = std::min<std::uint64_t>(t.pending + dec.layers_to_free(L), L);
            recompute = true;
            if (!fallback) {
                if (t.cached == 0) {
                    hedge_oor = true;
                } else {
                    double rc = hedge_recompute_time(mm, mode, t.cached, assumed);
                    double res = hedge_residual_load_time(mm, gg, t.cached, total);
                    recompute = res > rc;
                }
            }
            verdict = recompute ? 2 : 1;
        }
        OffloadDecision s = offload_cell_decision(mm, gg, mode, t.charged, 1, 1);
        out[i] = pack(action_id(dec.action), dec.action == OffloadAction::FreeLayers ? dec.layers : 0, free_now,
                      recompute, fallback, hedge_oor, verdict, s.action == OffloadAction::AllToHost, false);
    }
    return ORC_OK;
}

/* Trace-fused verdicts (SURVEY §8(d) C2 rule) through the reference's maps.
 * Each map set k is (models[k], gpus[k], cpa[k]) on the shared grid. */
int ref_features_decide(const orc_model* models, const orc_gpu* gpus, const int* cpa, size_t nsets,
                        const orc_grid* grid, uint64_t assumed, const uint32_t* prompt, const uint32_t* output,
                        const uint64_t* dev_offsets, const uint16_t* dev_set, size_t ndev, uint32_t* out) {
    try {
        std::vector<Maps> sets;
        for (size_t k = 0; k < nsets; ++k)
            sets.push_back(make_maps(&models[k], &gpus[k], grid, cpa[k], grid->cached_step, grid->max_cached, assumed));
        for (size_t d = 0; d < ndev; ++d) {
            size_t k = dev_set[d];
            if (k >= nsets) return ORC_EINVAL;
            uint64_t prev = 0;
            for (uint64_t i = dev_offsets[d]; i < dev_offsets[d + 1]; ++i) {
                uint64_t ch = prompt[i];
                if (cpa[k]) ch += 2 * static_cast<uint64_t>(output[i]);  // engine.hpp:422-423
                out[i] = compose(sets[k], models[k].num_layers, prev, static_cast<uint64_t>(prompt[i]) + output[i], 1,
                                 0, models[k].num_layers, ch);
                prev = ch;
            }
        }
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

/* Serving-only replay through Simulation::run (engine.hpp:140-164).
 * pctl[0..3] = p50, p90, p99, mean from the reference's finalize
 * (metrics.hpp:56-66); NaN when there are no samples.  grid may be NULL (no
 * replay-derived verdicts). */
int ref_replay_serving(const orc_model* m, const orc_gpu* g, const double* arrival, const uint32_t* prompt,
                       const uint32_t* output, uint64_t n, double tau, const orc_grid* grid, int cpa,
                       double* samples, uint8_t* labels, orc_batch* batches, orc_replay_summary* out,
                       double* pctl) {
    try {
        SimConfig cfg;
        cfg.mode = SimMode::ServingOnly;
        cfg.training = to_mode(cpa);
        cfg.model = to_model(m);
        cfg.gpu = to_gpu(g);
        cfg.collect_events = true;
        for (uint64_t i = 0; i < n; ++i) {
            QueryRecord r;
            r.query_id = i;
            r.arrival_time = arrival[i];
            r.prompt_tokens = prompt[i];
            r.output_tokens = output[i];
            cfg.trace.records.push_back(r);
        }
        validate_trace(cfg.trace);
        Simulation sim(cfg);
        MetricsReport rep = sim.run();
        std::memset(out, 0, sizeof *out);
        out->generated_tokens = rep.generated_tokens;
        out->peak_device_bytes = rep.peak_device_bytes;
        const double nan = std::nan("");
        pctl[0] = rep.tpt_p50 ? *rep.tpt_p50 : nan;
        pctl[1] = rep.tpt_p90 ? *rep.tpt_p90 : nan;
        pctl[2] = rep.tpt_p99 ? *rep.tpt_p99 : nan;
        pctl[3] = rep.tpt_mean ? *rep.tpt_mean : nan;
        if (samples) std::memcpy(samples, rep.tpt_samples.data(), rep.tpt_samples.size() * sizeof(double));

        Maps mp;
        if (grid) mp = make_maps(m, g, grid, cpa, grid->cached_step, grid->max_cached, 128);

        // Batch membership from the reference's own event log.
        std::vector<std::pair<uint64_t, double>> prefills;  // (size, start)
        std::vector<double> step_times;
        std::vector<size_t> first_step;  // index into step_times per batch
        for (const auto& e : sim.events()) {
            if (e.kind == EventKind::PrefillDone) {
                prefills.emplace_back(static_cast<uint64_t>(e.a), e.start);
                first_step.push_back(step_times.size());
            } else if (e.kind == EventKind::DecodeStepDone) {
                step_times.push_back(e.time);
            }
        }
        first_step.push_back(step_times.size());
        uint64_t head = 0, pos = 0, slot = 0, maxb = 0;
        for (size_t b = 0; b < prefills.size(); ++b) {
            uint64_t nb = prefills[b].first;
            uint32_t maxo = 0;
            uint64_t need_total = 0, max_inc = 0;
            for (uint64_t j = head; j < head + nb; ++j) {
                maxo = std::max(maxo, output[j]);
                need_total += serving_memory(cfg.model, static_cast<uint64_t>(prompt[j]) + output[j], 1);
                max_inc = std::max<uint64_t>(max_inc, static_cast<uint64_t>(prompt[j]) + output[j]);
            }
            std::vector<uint8_t> slow(nb, 0);
            for (uint32_t k = 0; k < maxo; ++k)
                for (uint64_t j = head; j < head + nb; ++j)
                    if (k < output[j]) {
                        double s = rep.tpt_samples[pos++];
                        if (s > tau) {
                            slow[j - head] = 1;
                            ++out->slow_tokens;
                        }
                    }
            for (uint64_t j = 0; j < nb; ++j) {
                if (labels) labels[head + j] = slow[j];
                out->slow_queries += slow[j];
            }
            uint32_t verdict = 0;
            if (grid) {
                uint64_t ch = prompt[head];
                if (cpa) ch += 2 * static_cast<uint64_t>(output[head]);
                verdict = compose(mp, m->num_layers, slot, max_inc, nb, 0, m->num_layers, ch);
                if (nb == 1) slot = ch;
            }
            if (batches) {
                orc_batch& rb = batches[b];
                rb.start = prefills[b].second;
                rb.end = first_step[b + 1] > first_step[b] ? step_times[first_step[b + 1] - 1] : rb.start;
                rb.first = static_cast<uint32_t>(head);
                rb.n = static_cast<uint32_t>(nb);
                rb.need_total = need_total;
                rb.max_incoming = static_cast<uint32_t>(std::min<uint64_t>(max_inc, 0xffffffffull));
                rb.verdict = verdict;
            }
            maxb = std::max(maxb, nb);
            head += nb;
        }
        out->batches = prefills.size();
        out->max_batch_size = maxb;
        out->end_time = step_times.empty() ? 0.0 : step_times.back();
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

/* Serving-only Simulation::run without the event log (for BASELINE-size
 * devices, whose log would not fit in host memory): the reference's TPT
 * samples in its own order, generated_tokens, peak_device_bytes and its
 * finalize (pctl[0..3] = p50, p90, p99, mean; NaN without samples).
 * samples may be NULL. */
int ref_serving_samples(const orc_model* m, const orc_gpu* g, const double* arrival, const uint32_t* prompt,
                        const uint32_t* output, uint64_t n, double* samples, uint64_t* generated_tokens,
                        uint64_t* peak_device_bytes, double* pctl) {
    try {
        SimConfig cfg;
        cfg.mode = SimMode::ServingOnly;
        cfg.model = to_model(m);
        cfg.gpu = to_gpu(g);
        cfg.trace.records.reserve(n);
        for (uint64_t i = 0; i < n; ++i) {
            QueryRecord r;
            r.query_id = i;
            r.arrival_time = arrival[i];
            r.prompt_tokens = prompt[i];
            r.output_tokens = output[i];
            cfg.trace.records.push_back(r);
        }
        validate_trace(cfg.trace);
        MetricsReport rep = run_simulation(std::move(cfg));
        *generated_tokens = rep.generated_tokens;
        *peak_device_bytes = rep.peak_device_bytes;
        const double nan = std::nan("");
        pctl[0] = rep.tpt_p50 ? *rep.tpt_p50 : nan;
        pctl[1] = rep.tpt_p90 ? *rep.tpt_p90 : nan;
        pctl[2] = rep.tpt_p99 ? *rep.tpt_p99 : nan;
        pctl[3] = rep.tpt_mean ? *rep.tpt_mean : nan;
        if (samples) std::memcpy(samples, rep.tpt_samples.data(), rep.tpt_samples.size() * sizeof(double));
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

/* Colocated replay through the reference's own Simulation::run in
 * SimMode::Colocated (engine.hpp:140-822) with maps from build_maps
 * (experiment.hpp:144-152: hedge grid = the offload grid's cached axis,
 * assumed output 128).  label_delay[i] < 0 (or NULL) = nullopt.  Fills the
 * MetricsReport fields of orc_colo_report, pctl[0..3] (p50/p90/p99/mean, NaN
 * without samples) and the raw samples; returns ORC_EBREACH when the run
 * throws InvariantBreach / std::logic_error, ORC_EVALIDATION for a refused
 * configuration.  batches: (start, end, first, n) from the event log. */
int ref_replay_sim(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int sim_mode, int cpa,
                   double cache_timeout, const double* arrival, const uint32_t* prompt, const uint32_t* output,
                   const double* label_delay, uint64_t n, double* samples, orc_batch* batches,
                   orc_colo_report* out, double* pctl) {
    std::memset(out, 0, sizeof *out);
    try {
        SimConfig cfg;
        cfg.mode = sim_mode == 0 ? SimMode::ServingOnly : (sim_mode == 1 ? SimMode::Colocated : SimMode::SeparateCluster);
        cfg.training = to_mode(cpa);
        cfg.model = to_model(m);
        cfg.gpu = to_gpu(g);
        cfg.cache_timeout = cache_timeout;
        cfg.collect_events = batches != nullptr;
        Maps mp = make_maps(m, g, grid, cpa, grid->cached_step, grid->max_cached, 128);
        cfg.offload_map = mp.off;
        cfg.hedge_map = mp.hedge;
        for (uint64_t i = 0; i < n; ++i) {
            QueryRecord r;
            r.query_id = i;
            r.arrival_time = arrival[i];
            r.prompt_tokens = prompt[i];
            r.output_tokens = output[i];
            if (label_delay && label_delay[i] >= 0) r.label_delay = label_delay[i];
            cfg.trace.records.push_back(r);
        }
        validate_trace(cfg.trace);
        Simulation sim(cfg);
        MetricsReport rep;
        try {
            rep = sim.run();
        } catch (const InvariantBreach&) {
            out->status = ORC_EBREACH;
            return ORC_EBREACH;
        } catch (const std::logic_error&) {
            out->status = ORC_EBREACH;
            return ORC_EBREACH;
        }
        out->generated_tokens = rep.generated_tokens;
        out->trained_tokens = rep.trained_tokens;
        out->training_busy_time = rep.training_busy_time;
        out->peak_device_bytes = rep.peak_device_bytes;
        out->peak_training_activation_bytes = rep.peak_training_activation_bytes;
        out->preemptions = rep.preemptions;
        out->layers_freed = rep.layers_freed;
        out->loads = rep.loads;
        out->recomputes = rep.recomputes;
        out->copy_stall_seconds = rep.copy_stall_seconds;
        out->labels_dropped = rep.labels_dropped;
        out->prefetch_wait_seconds = rep.prefetch_wait_seconds;
        out->completed_jobs = rep.completed_jobs;
        out->map_fallbacks = rep.map_fallbacks;
        out->oom_jobs = rep.oom_jobs;
        if (rep.oom_flag != (rep.oom_jobs > 0)) return ORC_EINVAL;  // oom_flag is derivable
        const double nan = std::nan("");
        if (pctl) {
            pctl[0] = rep.tpt_p50 ? *rep.tpt_p50 : nan;
            pctl[1] = rep.tpt_p90 ? *rep.tpt_p90 : nan;
            pctl[2] = rep.tpt_p99 ? *rep.tpt_p99 : nan;
            pctl[3] = rep.tpt_mean ? *rep.tpt_mean : nan;
        }
        if (samples) std::memcpy(samples, rep.tpt_samples.data(), rep.tpt_samples.size() * sizeof(double));
        if (batches) {
            uint64_t head = 0, b = 0;
            double last_step = 0;
            for (const auto& e : sim.events()) {
                if (e.kind == EventKind::PrefillDone) {
                    if (b) batches[b - 1].end = last_step;
                    orc_batch& rb = batches[b++];
                    std::memset(&rb, 0, sizeof rb);
                    rb.start = e.start;
                    rb.first = static_cast<uint32_t>(head);
                    rb.n = static_cast<uint32_t>(e.a);
                    head += static_cast<uint64_t>(e.a);
                } else if (e.kind == EventKind::DecodeStepDone) {
                    last_step = e.time;
                }
            }
            if (b) batches[b - 1].end = last_step;
            out->batches = b;
        }
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

int ref_finalize(const double* samples, size_t n, double* p50, double* p90, double* p99, double* mean) {
    if (n == 0) return ORC_EINVAL;
    MetricsReport r;
    r.tpt_samples.assign(samples, samples + n);
    finalize(r);
    *p50 = *r.tpt_p50;
    *p90 = *r.tpt_p90;
    *p99 = *r.tpt_p99;
    *mean = *r.tpt_mean;
    return ORC_OK;
}

static LengthDistribution to_dist(const orc_dist* d) {
    LengthDistribution r;
    if (d->kind == 0) r = LengthDistribution::fixed(d->fixed_value);
    else if (d->kind == 1) r = LengthDistribution::uniform(d->lo, d->hi);
    else {
        std::vector<std::pair<double, double>> bins;
        for (size_t i = 0; i < d->nbins; ++i) bins.emplace_back(d->bin_values[i], d->bin_probs[i]);
        r = LengthDistribution::histogram(bins);
    }
    if (d->min_tokens) r.min_tokens = d->min_tokens;
    return r;
}

int64_t ref_generate_trace(double qps, double duration, const orc_dist* lengths, const orc_dist* label_delay,
                           uint64_t seed, double* arrival, uint32_t* prompt, uint32_t* output, double* label_out,
                           size_t cap) {
    try {
        std::optional<LengthDistribution> ld;
        if (label_delay) ld = to_dist(label_delay);
        Trace t = generate_trace(qps, duration, to_dist(lengths), ld, seed);
        if (t.records.size() > cap) return -1;
        for (size_t i = 0; i < t.records.size(); ++i) {
            arrival[i] = t.records[i].arrival_time;
            prompt[i] = static_cast<uint32_t>(t.records[i].prompt_tokens);
            output[i] = static_cast<uint32_t>(t.records[i].output_tokens);
            if (label_out) label_out[i] = t.records[i].label_delay ? *t.records[i].label_delay : -1.0;
        }
        return static_cast<int64_t>(t.records.size());
    } catch (const std::exception&) {
        return -2;
    }
}

/* File formats through the reference's own writers/readers (maps.hpp:118-191,
 * 284-332; workload.hpp:224-271). */
int ref_save_maps(const orc_model* m, const orc_gpu* g, const orc_grid* grid, int cpa, uint64_t assumed,
                  const char* offload_path, const char* hedge_path) {
    try {
        Maps mp = make_maps(m, g, grid, cpa, grid->cached_step, grid->max_cached, assumed);
        mp.off.save(offload_path);
        mp.hedge.save(hedge_path);
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

int ref_save_trace(const double* arrival, const uint32_t* prompt, const uint32_t* output, const double* label_delay,
                   size_t n, const char* path) {
    try {
        Trace t;
        for (size_t i = 0; i < n; ++i) {
            QueryRecord r;
            r.query_id = i;
            r.arrival_time = arrival[i];
            r.prompt_tokens = prompt[i];
            r.output_tokens = output[i];
            if (label_delay && !std::isnan(label_delay[i])) r.label_delay = label_delay[i];
            t.records.push_back(r);
        }
        save_trace(t, path);
        return ORC_OK;
    } catch (const std::exception&) {
        return ORC_EVALIDATION;
    }
}

int64_t ref_load_trace(const char* path, double* arrival, uint32_t* prompt, uint32_t* output, uint64_t* ids,
                       double* label_delay, size_t cap) {
    try {
        Trace t = load_trace(path);
        if (t.records.size() > cap) return -1;
        for (size_t i = 0; i < t.records.size(); ++i) {
            const auto& r = t.records[i];
            arrival[i] = r.arrival_time;
            prompt[i] = static_cast<uint32_t>(r.prompt_tokens);
            output[i] = static_cast<uint32_t>(r.output_tokens);
            ids[i] = r.query_id;
            label_delay[i] = r.label_delay ? *r.label_delay : std::nan("");
        }
        return static_cast<int64_t>(t.records.size());
    } catch (const std::exception&) {
        return -2;
    }
}

}  // extern "C"
