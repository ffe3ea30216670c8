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
// and throws the reference's exception types for the reference's error
// cases: std::runtime_error for validation (COLO_EVALIDATION),
// std::invalid_argument for contract violations (COLO_EINVAL).  Any struct
// with the ModelProfile / GpuProfile / GridSteps / GridBounds field names
// converts, so colosim's own profile objects can be passed unchanged.
#pragma once

#include <cstdint>
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

}  // namespace colosim_gpu
