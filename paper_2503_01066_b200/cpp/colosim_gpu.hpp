// colosim_gpu.hpp -- header-only C++ drop-in over the colo-b200 C-ABI
// (include/colo_abi.h) for code written against the colosim headers.
//
// It keeps the reference's vocabulary and call shapes (paths relative to
// /root/reference/proj/include/colosim/):
//   colosim_gpu::build_maps(ctx, model, gpu, steps, bounds, mode)   experiment.hpp:144-152
//   GpuMaps::offload_lookup(cached, incoming, batch)                 maps.hpp:100-110 (std::optional)
//   GpuMaps::hedge_lookup(cached, freed)                             maps.hpp:276-280 (std::optional)
//   GpuMaps::decide(tuples) / decide_exact(...)                      engine.hpp:434-448, 513-557 in bulk
//   colosim_gpu::replay_serving(...)                                 engine.hpp:140-387 (ServingOnly)
//   colosim_gpu::run_simulation<MetricsReport>(ctx, cfg)             engine.hpp:938-941 (every SimMode)
//   colosim_gpu::run_simulations<MetricsReport>(ctx, cfgs)           many runs as one device fleet
// and throws the reference's exception types for the reference's error
// cases: std::runtime_error for validation (COLO_EVALIDATION),
// std::invalid_argument for contract violations (COLO_EINVAL).  Any struct
// with the ModelProfile / GpuProfile / GridSteps / GridBounds field names
// converts, so colosim's own profile objects can be passed unchanged.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "colo_abi.h"

namespace colosim_gpu {

inline void check(colo_status st, const colo_ctx* ctx, const char* what) {
    if (st == COLO_OK) return;
    std::string msg = std::string(what) + ": " + (ctx ? colo_last_error(ctx) : "");
    if (st == COLO_EVALIDATION) throw std::runtime_error(msg);
    if (st == COLO_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("colo-b200 " + msg);
}

template <class ModelProfile>
colo_model to_c_model(const ModelProfile& m) {
    return colo_model{m.num_layers, m.kv_bytes_per_token, m.act_bytes_per_token_per_layer, m.prefill_coef_linear,
                      m.prefill_coef_quad, m.decode_coef_const, m.decode_coef_context, m.backward_to_forward_ratio,
                      m.record_prefill_multiplier, m.record_decode_multiplier, m.workspace_factor, m.weights_bytes};
}

template <class GpuProfile>
colo_gpu to_c_gpu(const GpuProfile& g) {
    return colo_gpu{g.capacity_bytes, g.h2d_bandwidth, g.d2h_bandwidth, g.runtime_reserve_bytes};
}

template <class GridSteps, class GridBounds>
colo_grid to_c_grid(const GridSteps& s, const GridBounds& b) {
    return colo_grid{s.cached_token_step, s.incoming_token_step, s.batch_step,
                     b.max_cached_tokens, b.max_incoming_tokens, b.max_batch};
}

/// One GPU, one stream (colo_ctx).  Not copyable; one per host thread.
class Context {
  public:
    explicit Context(int device = 0) { check(colo_ctx_create(device, &ctx_), nullptr, "colo_ctx_create"); }
    ~Context() { colo_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    colo_ctx* get() const { return ctx_; }
    void sync() { check(colo_sync(ctx_), ctx_, "colo_sync"); }

  private:
    colo_ctx* ctx_ = nullptr;
};

enum class Action { NoAction = COLO_ACT_NOACTION, FreeLayers = COLO_ACT_FREELAYERS, AllToHost = COLO_ACT_ALLTOHOST };

struct Decision {  // maps.hpp:34-49
    Action action = Action::NoAction;
    std::uint64_t layers = 0;
    bool operator==(const Decision&) const = default;
};

/// Offloading + hedging map of one (model, gpu, grid, mode), built and held
/// on the device -- colosim's BuiltMaps.
class GpuMaps {
  public:
    GpuMaps(Context& ctx, const colo_model& m, const colo_gpu& g, const colo_grid& grid, colo_mode mode,
            std::uint64_t assumed_output_tokens = 128)
        : ctx_(&ctx), grid_(grid), L_(m.num_layers) {
        check(colo_mapset_build(ctx.get(), &m, &g, &grid, mode, grid.cached_step, grid.max_cached,
                                assumed_output_tokens, &ms_),
              ctx.get(), "build_maps");
        size_t a = 0, b = 0;
        colo_mapset_shape(ms_, &a, &b);
        off_.resize(a);
        hed_.resize(b);
        check(colo_mapset_cells(ctx.get(), ms_, off_.data(), a, hed_.data(), b), ctx.get(), "map cells");
    }
    ~GpuMaps() { colo_mapset_destroy(ms_); }
    GpuMaps(const GpuMaps&) = delete;
    GpuMaps& operator=(const GpuMaps&) = delete;

    const colo_mapset* get() const { return ms_; }
    std::uint64_t profile_hash_value() const { return colo_mapset_hash(ms_); }
    const std::vector<std::uint8_t>& offload_cells() const { return off_; }
    const std::vector<std::uint8_t>& hedge_cells() const { return hed_; }

    /// OffloadingMap::lookup on the device-built cells (maps.hpp:100-110).
    std::optional<Decision> offload_lookup(std::uint64_t cached, std::uint64_t incoming, std::uint64_t batch) const {
        auto up = [](std::uint64_t v, std::uint64_t s) { return (v + s - 1) / s * s; };
        std::uint64_t cb = up(cached, grid_.cached_step), ib = up(incoming, grid_.incoming_step),
                      bb = up(batch, grid_.batch_step);
        if (cb > grid_.max_cached || ib > grid_.max_incoming || bb > grid_.max_batch) return std::nullopt;
        if (incoming == 0 || batch == 0) return std::nullopt;
        std::uint64_t I = grid_.max_incoming / grid_.incoming_step, B = grid_.max_batch / grid_.batch_step;
        std::uint8_t c = off_[((cb / grid_.cached_step) * I + ib / grid_.incoming_step - 1) * B + bb / grid_.batch_step - 1];
        if (c == 0) return Decision{Action::NoAction, 0};
        if (c == 1) return Decision{Action::AllToHost, 0};
        return Decision{Action::FreeLayers, static_cast<std::uint64_t>(c - 2)};
    }

    /// HedgingMap::lookup (maps.hpp:276-280); true = Recompute.
    std::optional<bool> hedge_lookup(std::uint64_t cached, std::uint64_t freed) const {
        std::uint64_t s = grid_.cached_step;
        std::uint64_t cb = (cached + s - 1) / s * s;
        if (cb == 0 || cb > grid_.max_cached || freed > L_) return std::nullopt;
        return hed_[(cb / s - 1) * (L_ + 1) + freed] != 0;
    }

    /// Bulk verdicts through the sm_100a kernel (host buffers in and out).
    std::vector<std::uint32_t> decide(const std::vector<colo_tuple>& tuples, std::uint64_t* counters = nullptr) const {
        std::vector<std::uint32_t> out(tuples.size());
        check(colo_decide_host(ctx_->get(), ms_, tuples.data(), tuples.size(), out.data(), counters), ctx_->get(),
              "decide");
        return out;
    }

  private:
    Context* ctx_;
    colo_grid grid_;
    std::uint64_t L_;
    colo_mapset* ms_ = nullptr;
    std::vector<std::uint8_t> off_, hed_;
};

template <class ModelProfile, class GpuProfile, class GridSteps, class GridBounds>
GpuMaps* build_maps(Context& ctx, const ModelProfile& m, const GpuProfile& g, const GridSteps& steps,
                    const GridBounds& bounds, bool cpa, std::uint64_t assumed_output_tokens = 128) {
    return new GpuMaps(ctx, to_c_model(m), to_c_gpu(g), to_c_grid(steps, bounds), cpa ? COLO_CPA : COLO_CPT,
                       assumed_output_tokens);
}

/// Serving-only replay of one device trace (Simulation::run in
/// SimMode::ServingOnly) -> TPT samples in the reference's order, plus the
/// per-query slow labels for threshold tau.
struct ServingReplay {
    std::vector<double> tpt_samples;
    std::vector<std::uint8_t> labels;
    colo_device_summary summary{};
};

template <class ModelProfile, class GpuProfile>
ServingReplay replay_serving(Context& ctx, const ModelProfile& m, const GpuProfile& g,
                             const std::vector<double>& arrival, const std::vector<std::uint32_t>& prompt,
                             const std::vector<std::uint32_t>& output, double tau) {
    const size_t n = prompt.size();
    if (arrival.size() != n || output.size() != n) throw std::invalid_argument("replay_serving: ragged trace arrays");
    std::uint64_t ns = 0;
    for (auto o : output) ns += o;
    colo_ctx* c = ctx.get();
    void *d_a, *d_p, *d_o, *d_off, *d_prof, *d_s, *d_soff, *d_l, *d_sum;
    const std::uint64_t offs[2] = {0, n}, soffs[2] = {0, ns};
    const std::uint16_t prof = 0;
    check(colo_dev_alloc(c, n * 8 + 8, &d_a), c, "alloc");
    check(colo_dev_alloc(c, n * 4 + 4, &d_p), c, "alloc");
    check(colo_dev_alloc(c, n * 4 + 4, &d_o), c, "alloc");
    check(colo_dev_alloc(c, 16, &d_off), c, "alloc");
    check(colo_dev_alloc(c, 16, &d_soff), c, "alloc");
    check(colo_dev_alloc(c, 2, &d_prof), c, "alloc");
    check(colo_dev_alloc(c, ns * 8 + 8, &d_s), c, "alloc");
    check(colo_dev_alloc(c, n + 1, &d_l), c, "alloc");
    check(colo_dev_alloc(c, sizeof(colo_device_summary), &d_sum), c, "alloc");
    ServingReplay r;
    try {
        check(colo_memcpy_h2d(c, d_a, arrival.data(), n * 8), c, "h2d");
        check(colo_memcpy_h2d(c, d_p, prompt.data(), n * 4), c, "h2d");
        check(colo_memcpy_h2d(c, d_o, output.data(), n * 4), c, "h2d");
        check(colo_memcpy_h2d(c, d_off, offs, 16), c, "h2d");
        check(colo_memcpy_h2d(c, d_soff, soffs, 16), c, "h2d");
        check(colo_memcpy_h2d(c, d_prof, &prof, 2), c, "h2d");
        colo_replay_opts o{};
        o.tau = tau;
        o.d_samples = static_cast<double*>(d_s);
        o.d_sample_offsets = static_cast<const std::uint64_t*>(d_soff);
        o.d_labels = static_cast<std::uint8_t*>(d_l);
        o.d_summary = static_cast<colo_device_summary*>(d_sum);
        colo_model cm = to_c_model(m);
        colo_gpu cg = to_c_gpu(g);
        check(colo_replay_serving(c, &cm, &cg, 1, static_cast<double*>(d_a), static_cast<std::uint32_t*>(d_p),
                                  static_cast<std::uint32_t*>(d_o), n, static_cast<std::uint64_t*>(d_off),
                                  static_cast<std::uint16_t*>(d_prof), 1, &o),
              c, "replay_serving");
        r.tpt_samples.resize(ns);
        r.labels.resize(n);
        check(colo_memcpy_d2h(c, r.tpt_samples.data(), d_s, ns * 8), c, "d2h");
        check(colo_memcpy_d2h(c, r.labels.data(), d_l, n), c, "d2h");
        check(colo_memcpy_d2h(c, &r.summary, d_sum, sizeof r.summary), c, "d2h");
    } catch (...) {
        for (void* p : {d_a, d_p, d_o, d_off, d_soff, d_prof, d_s, d_l, d_sum}) colo_dev_free(c, p);
        throw;
    }
    for (void* p : {d_a, d_p, d_o, d_off, d_soff, d_prof, d_s, d_l, d_sum}) colo_dev_free(c, p);
    return r;
}

/// The reference throws InvariantBreach (engine.hpp:43-46), a std::runtime_error.
struct invariant_breach : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {

template <class SimConfig>
int sim_mode_of(const SimConfig& cfg) {
    using M = decltype(cfg.mode);
    if (cfg.mode == M::Colocated) return COLO_SIM_COLOCATED;
    if (cfg.mode == M::SeparateCluster) return COLO_SIM_SEPARATE;
    return COLO_SIM_SERVING_ONLY;
}

template <class SimConfig>
bool is_cpa(const SimConfig& cfg) {
    return cfg.training == decltype(cfg.training)::CPA;
}

// The config's own maps as device cells (OffloadingMap::cell / HedgingMap::cell,
// maps.hpp:89-94, 269-270).  Non-colocated runs never consult them
// (SimConfig::validate checks maps only in Colocated mode, engine.hpp:62-68):
// those get freshly built maps of their profile.
template <class SimConfig>
colo_mapset* mapset_of(Context& ctx, const SimConfig& cfg) {
    const colo_model m = to_c_model(cfg.model);
    const colo_gpu g = to_c_gpu(cfg.gpu);
    const colo_mode mode = is_cpa(cfg) ? COLO_CPA : COLO_CPT;
    colo_mapset* ms = nullptr;
    if (sim_mode_of(cfg) != COLO_SIM_COLOCATED) {
        const colo_grid grid{500, 500, 5, 8000, 8000, 50};
        check(colo_mapset_build(ctx.get(), &m, &g, &grid, mode, 500, 8000, 128, &ms), ctx.get(), "build_maps");
        return ms;
    }
    const auto& om = cfg.offload_map;
    const auto& hm = cfg.hedge_map;
    const colo_grid grid = to_c_grid(om.steps, om.bounds);
    if (om.mode != cfg.training || hm.mode != cfg.training)
        throw std::runtime_error("sim config: map training mode does not match sim.training");  // engine.hpp:66-67
    if (hm.profile_hash_value != om.profile_hash_value)
        throw std::runtime_error("sim config: map profile hash does not match the profiles");  // engine.hpp:63-65
    std::vector<std::uint8_t> off(om.cached_count() * om.incoming_count() * om.batch_count());
    for (std::size_t ci = 0; ci < om.cached_count(); ++ci)
        for (std::size_t ii = 0; ii < om.incoming_count(); ++ii)
            for (std::size_t bi = 0; bi < om.batch_count(); ++bi) {
                const auto& d = om.cell(ci, ii, bi);
                using A = decltype(d.action);
                off[(ci * om.incoming_count() + ii) * om.batch_count() + bi] =
                    d.action == A::NoAction ? 0 : (d.action == A::AllToHost ? 1 : static_cast<std::uint8_t>(2 + d.layers));
            }
    std::vector<std::uint8_t> hed(hm.cached_count() * hm.freed_count());
    for (std::size_t ci = 0; ci < hm.cached_count(); ++ci)
        for (std::size_t fi = 0; fi < hm.freed_count(); ++fi)
            hed[ci * hm.freed_count() + fi] = hm.cell(ci, fi) == decltype(hm.cell(ci, fi))::Recompute ? 1 : 0;
    // refuses a hash other than profile_hash(model, gpu) (engine.hpp:63-65)
    check(colo_mapset_from_cells(ctx.get(), &m, &g, &grid, mode, hm.cached_token_step, hm.max_cached_tokens,
                                 hm.assumed_output_tokens, om.profile_hash_value, off.data(), off.size(), hed.data(),
                                 hed.size(), &ms),
          ctx.get(), "sim config maps");
    return ms;
}

}  // namespace detail

/// Simulation::run (engine.hpp:131-164) for every config, as one fleet of
/// devices on the GPU (one launch per group of <= 16 distinct profiles and one
/// cache timeout).  Returns the reference's own report type, finalized as
/// metrics.hpp:56-69 does; equal (operator==) to run_simulation(cfg) on the
/// CPU.  Throws std::runtime_error where the reference's constructor does and
/// invariant_breach where its run() does.
template <class Report, class SimConfig>
std::vector<Report> run_simulations(Context& ctx, const std::vector<SimConfig>& cfgs) {
    colo_ctx* c = ctx.get();
    std::vector<Report> out(cfgs.size());
    std::vector<std::size_t> todo;
    for (std::size_t i = 0; i < cfgs.size(); ++i) {
        const colo_model m = to_c_model(cfgs[i].model);
        const colo_gpu g = to_c_gpu(cfgs[i].gpu);
        check(colo_validate_profile_pair(&m, &g), c, "sim config");  // engine.hpp:61
        todo.push_back(i);
    }
    while (!todo.empty()) {
        // one launch: a shared cache timeout, at most 16 map sets
        const double timeout = cfgs[todo[0]].cache_timeout;
        std::vector<std::size_t> batch, rest;
        std::vector<colo_mapset*> sets;
        std::vector<std::uint16_t> dset;
        for (std::size_t i : todo) {
            if (cfgs[i].cache_timeout != timeout || sets.size() == 16) {
                rest.push_back(i);
                continue;
            }
            sets.push_back(detail::mapset_of(ctx, cfgs[i]));
            dset.push_back(static_cast<std::uint16_t>(sets.size() - 1));
            batch.push_back(i);
        }
        todo.swap(rest);
        std::vector<double> a, ld;
        std::vector<std::uint32_t> p, o;
        std::vector<std::uint64_t> off{0}, soff{0};
        std::vector<std::uint8_t> sm;
        for (std::size_t i : batch) {
            for (const auto& r : cfgs[i].trace.records) {
                a.push_back(r.arrival_time);
                p.push_back(static_cast<std::uint32_t>(r.prompt_tokens));
                o.push_back(static_cast<std::uint32_t>(r.output_tokens));
                // the device keeps "no label" as a negative delay: a present negative delay is refused
                if (r.label_delay && !(*r.label_delay >= 0.0))
                    throw std::invalid_argument("colo-b200: negative or NaN label_delay is not supported");
                ld.push_back(r.label_delay ? *r.label_delay : -1.0);
            }
            std::uint64_t ns = soff.back();
            for (const auto& r : cfgs[i].trace.records) ns += r.output_tokens;
            off.push_back(a.size());
            soff.push_back(ns);
            sm.push_back(static_cast<std::uint8_t>(detail::sim_mode_of(cfgs[i])));
        }
        const std::size_t n = a.size(), nd = batch.size(), ns = soff.back();
        void *d_a, *d_p, *d_o, *d_ld, *d_off, *d_soff, *d_set, *d_sm, *d_s, *d_sum;
        check(colo_dev_alloc(c, n * 8 + 8, &d_a), c, "alloc");
        check(colo_dev_alloc(c, n * 4 + 4, &d_p), c, "alloc");
        check(colo_dev_alloc(c, n * 4 + 4, &d_o), c, "alloc");
        check(colo_dev_alloc(c, n * 8 + 8, &d_ld), c, "alloc");
        check(colo_dev_alloc(c, (nd + 1) * 8, &d_off), c, "alloc");
        check(colo_dev_alloc(c, (nd + 1) * 8, &d_soff), c, "alloc");
        check(colo_dev_alloc(c, nd * 2 + 2, &d_set), c, "alloc");
        check(colo_dev_alloc(c, nd + 1, &d_sm), c, "alloc");
        check(colo_dev_alloc(c, ns * 8 + 8, &d_s), c, "alloc");
        check(colo_dev_alloc(c, nd * sizeof(colo_colocated_summary), &d_sum), c, "alloc");
        std::vector<colo_colocated_summary> sum(nd);
        std::vector<double> smp(ns);
        std::vector<std::array<double, 4>> fin(nd);  // finalize per report, on the device
        colo_status st = COLO_OK;
        try {
            check(colo_memcpy_h2d(c, d_a, a.data(), n * 8), c, "h2d");
            check(colo_memcpy_h2d(c, d_p, p.data(), n * 4), c, "h2d");
            check(colo_memcpy_h2d(c, d_o, o.data(), n * 4), c, "h2d");
            check(colo_memcpy_h2d(c, d_ld, ld.data(), n * 8), c, "h2d");
            check(colo_memcpy_h2d(c, d_off, off.data(), (nd + 1) * 8), c, "h2d");
            check(colo_memcpy_h2d(c, d_soff, soff.data(), (nd + 1) * 8), c, "h2d");
            check(colo_memcpy_h2d(c, d_set, dset.data(), nd * 2), c, "h2d");
            check(colo_memcpy_h2d(c, d_sm, sm.data(), nd), c, "h2d");
            colo_colocated_opts opt{};
            opt.cache_timeout = timeout;
            opt.d_label_delay = static_cast<const double*>(d_ld);
            opt.tau = std::numeric_limits<double>::infinity();
            opt.d_samples = static_cast<double*>(d_s);
            opt.d_sample_offsets = static_cast<const std::uint64_t*>(d_soff);
            opt.d_summary = static_cast<colo_colocated_summary*>(d_sum);
            opt.d_dev_sim_mode = static_cast<const std::uint8_t*>(d_sm);
            st = colo_replay_colocated(c, sets.data(), sets.size(), static_cast<double*>(d_a),
                                       static_cast<std::uint32_t*>(d_p), static_cast<std::uint32_t*>(d_o), n,
                                       static_cast<std::uint64_t*>(d_off), static_cast<std::uint16_t*>(d_set), nd, &opt);
            if (st != COLO_OK && st != COLO_EBREACH) check(st, c, "run_simulation");
            check(colo_memcpy_d2h(c, sum.data(), d_sum, nd * sizeof(colo_colocated_summary)), c, "d2h");
            check(colo_memcpy_d2h(c, smp.data(), d_s, ns * 8), c, "d2h");
            for (std::size_t k = 0; k < nd; ++k)  // finalize (metrics.hpp:56-69), bit-exact: colo_finalize
                if (sum[k].status == COLO_OK && sum[k].generated_tokens)
                    check(colo_finalize(c, static_cast<const double*>(d_s) + soff[k], sum[k].generated_tokens, nullptr,
                                        fin[k].data()),
                          c, "finalize");
        } catch (...) {
            for (void* q : {d_a, d_p, d_o, d_ld, d_off, d_soff, d_set, d_sm, d_s, d_sum}) colo_dev_free(c, q);
            for (auto* ms : sets) colo_mapset_destroy(ms);
            throw;
        }
        for (void* q : {d_a, d_p, d_o, d_ld, d_off, d_soff, d_set, d_sm, d_s, d_sum}) colo_dev_free(c, q);
        for (auto* ms : sets) colo_mapset_destroy(ms);
        for (std::size_t k = 0; k < nd; ++k) {
            const colo_colocated_summary& s = sum[k];
            if (s.status == COLO_EBREACH) throw invariant_breach("colo-b200: invariant breach in run_simulation");
            const SimConfig& cfg = cfgs[batch[k]];
            Report& r = out[batch[k]];
            r.tpt_samples.assign(smp.begin() + soff[k], smp.begin() + soff[k] + s.generated_tokens);
            r.trained_tokens = s.trained_tokens;
            r.training_busy_time = s.training_busy_time;
            r.peak_device_bytes = s.peak_device_bytes;
            r.peak_training_activation_bytes = s.peak_training_activation_bytes;
            r.oom_flag = s.oom_jobs > 0;
            r.preemptions = s.preemptions;
            r.layers_freed = s.layers_freed;
            r.loads = s.loads;
            r.recomputes = s.recomputes;
            r.copy_stall_seconds = s.copy_stall_seconds;
            r.labels_dropped = s.labels_dropped;
            r.prefetch_wait_seconds = s.prefetch_wait_seconds;
            r.completed_jobs = s.completed_jobs;
            r.oom_jobs = s.oom_jobs;
            r.map_fallbacks = s.map_fallbacks;
            r.generated_tokens = s.generated_tokens;
            r.trace_hash = cfg.trace.content_hash();                                   // engine.hpp:157
            r.mode_tag = std::string(to_string(cfg.mode)) + "/" + to_string(cfg.training);  // :158
            // finalize (metrics.hpp:56-69): nearest ranks and the sorted sequential mean from colo_finalize
            if (!r.tpt_samples.empty()) {
                r.tpt_p50 = fin[k][0];
                r.tpt_p90 = fin[k][1];
                r.tpt_p99 = fin[k][2];
                r.tpt_mean = fin[k][3];
            }
            if (r.training_busy_time > 0)
                r.training_throughput = static_cast<double>(r.trained_tokens) / r.training_busy_time;
        }
    }
    return out;
}

template <class Report, class SimConfig>
Report run_simulation(Context& ctx, const SimConfig& cfg) {
    return run_simulations<Report>(ctx, std::vector<SimConfig>{cfg})[0];
}

/// Simulation::events_json() of the run (engine.hpp:166-175, with
/// SimConfig::collect_events): every logged event in dispatch order as
/// LoggedEvent::to_json lines, from the run on the GPU
/// (colo_colocated_events).  Throws invariant_breach where run() does.
template <class SimConfig>
std::string events_json(Context& ctx, const SimConfig& cfg) {
    colo_ctx* c = ctx.get();
    const colo_model m = to_c_model(cfg.model);
    const colo_gpu g = to_c_gpu(cfg.gpu);
    check(colo_validate_profile_pair(&m, &g), c, "sim config");
    colo_mapset* ms = detail::mapset_of(ctx, cfg);
    std::vector<double> a, ld;
    std::vector<std::uint32_t> p, o;
    std::vector<std::uint64_t> q;
    for (const auto& r : cfg.trace.records) {
        a.push_back(r.arrival_time);
        p.push_back(static_cast<std::uint32_t>(r.prompt_tokens));
        o.push_back(static_cast<std::uint32_t>(r.output_tokens));
        if (r.label_delay && !(*r.label_delay >= 0.0))
            throw std::invalid_argument("colo-b200: negative or NaN label_delay is not supported");
        ld.push_back(r.label_delay ? *r.label_delay : -1.0);
        q.push_back(static_cast<std::uint64_t>(r.query_id));
    }
    const std::size_t n = a.size();
    void *d_a = nullptr, *d_p = nullptr, *d_o = nullptr, *d_ld = nullptr, *d_q = nullptr;
    std::string text;
    try {
        check(colo_dev_alloc(c, n * 8 + 8, &d_a), c, "alloc");
        check(colo_dev_alloc(c, n * 4 + 4, &d_p), c, "alloc");
        check(colo_dev_alloc(c, n * 4 + 4, &d_o), c, "alloc");
        check(colo_dev_alloc(c, n * 8 + 8, &d_ld), c, "alloc");
        check(colo_dev_alloc(c, n * 8 + 8, &d_q), c, "alloc");
        check(colo_memcpy_h2d(c, d_a, a.data(), n * 8), c, "h2d");
        check(colo_memcpy_h2d(c, d_p, p.data(), n * 4), c, "h2d");
        check(colo_memcpy_h2d(c, d_o, o.data(), n * 4), c, "h2d");
        check(colo_memcpy_h2d(c, d_ld, ld.data(), n * 8), c, "h2d");
        check(colo_memcpy_h2d(c, d_q, q.data(), n * 8), c, "h2d");
        const std::int64_t len = colo_colocated_events(
            c, ms, detail::sim_mode_of(cfg), cfg.cache_timeout, static_cast<const double*>(d_a),
            static_cast<const std::uint32_t*>(d_p), static_cast<const std::uint32_t*>(d_o),
            static_cast<const double*>(d_ld), -1.0, static_cast<const std::uint64_t*>(d_q), n,
            std::numeric_limits<double>::infinity());
        if (len < 0) {
            if (-len == COLO_EBREACH) throw invariant_breach("colo-b200: invariant breach in run_simulation");
            check(static_cast<colo_status>(-len), c, "events_json");
        }
        text.resize(static_cast<std::size_t>(len) + 1);
        colo_events_text(c, text.data(), text.size());
        text.resize(static_cast<std::size_t>(len));
    } catch (...) {
        for (void* x : {d_a, d_p, d_o, d_ld, d_q}) colo_dev_free(c, x);
        colo_mapset_destroy(ms);
        throw;
    }
    for (void* x : {d_a, d_p, d_o, d_ld, d_q}) colo_dev_free(c, x);
    colo_mapset_destroy(ms);
    return text;
}

}  // namespace colosim_gpu
