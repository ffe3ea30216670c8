// overlay/colosim/maps.hpp -- the reference's maps.hpp with the two map
// builders running on the GPU.
//
// Put paper_2503_01066_b200/cpp/overlay first on the include path of code
// written against the colosim headers (tools/colosim.cpp, unchanged): every
// `#include "colosim/maps.hpp"` then lands here.  The reference header is
// included next (#include_next) with its builders renamed by macro, and
// build_offloading_map / build_hedging_map (maps.hpp:233-252, 358-384) are
// defined again with the same signatures: the cells come from
// colo_mapset_build (k_build_offload / k_build_hedge on sm_100a) and are
// returned in the reference's own OffloadingMap / HedgingMap objects, so the
// lookups, save/load and everything downstream are unchanged.  Validation is
// the reference's own (validate_profile_pair, validate_grid and the hedging
// map's step checks), so error texts and CLI exit codes stay identical.
#pragma once

#include "colosim_gpu_context.hpp"  // before the renaming macros below

#define build_offloading_map build_offloading_map_cpu_reference
#define build_hedging_map build_hedging_map_cpu_reference
#include_next <colosim/maps.hpp>
#undef build_offloading_map
#undef build_hedging_map

#include <stdexcept>
#include <vector>


namespace colosim {

namespace gpu_overlay {

inline void build_cells(const ModelProfile& m, const GpuProfile& g, const colo_grid& grid, TrainingMode mode,
                                std::uint64_t hedge_step, std::uint64_t hedge_max, std::uint64_t assumed,
                                std::vector<std::uint8_t>* off, std::vector<std::uint8_t>* hed) {
    colosim_gpu::Context& ctx = colosim_gpu::process_context();
    const colo_model cm = colosim_gpu::to_c_model(m);
    const colo_gpu cg = colosim_gpu::to_c_gpu(g);
    colo_mapset* ms = nullptr;
    colosim_gpu::check(colo_mapset_build(ctx.get(), &cm, &cg, &grid, mode == TrainingMode::CPA ? COLO_CPA : COLO_CPT,
                                         hedge_step, hedge_max, assumed, &ms),
                       ctx.get(), "build_maps");
    std::size_t a = 0, b = 0;
    colo_mapset_shape(ms, &a, &b);
    if (off) off->resize(a);
    if (hed) hed->resize(b);
    const colo_status st = colo_mapset_cells(ctx.get(), ms, off ? off->data() : nullptr, a,
                                             hed ? hed->data() : nullptr, b);
    colo_mapset_destroy(ms);
    colosim_gpu::check(st, ctx.get(), "map cells");
}

}  // namespace gpu_overlay

/// build_offloading_map (maps.hpp:233-252), cells from the GPU.
inline OffloadingMap build_offloading_map(const ModelProfile& m, const GpuProfile& g, const GridSteps& steps,
                                          const GridBounds& bounds, TrainingMode mode) {
    validate_profile_pair(m, g);
    validate_grid(steps, bounds);
    OffloadingMap map;
    map.steps = steps;
    map.bounds = bounds;
    map.mode = mode;
    map.profile_hash_value = profile_hash(m, g);
    map.num_layers = m.num_layers;
    map.init_cells();
    std::vector<std::uint8_t> off;
    const colo_grid grid = colosim_gpu::to_c_grid(steps, bounds);
    gpu_overlay::build_cells(m, g, grid, mode, steps.cached_token_step, bounds.max_cached_tokens, 128, &off, nullptr);
    std::size_t k = 0;
    for (std::size_t ci = 0; ci < map.cached_count(); ++ci)
        for (std::size_t ii = 0; ii < map.incoming_count(); ++ii)
            for (std::size_t bi = 0; bi < map.batch_count(); ++bi, ++k) {
                const std::uint8_t c = off.at(k);  // 0 NoAction, 1 AllToHost, 2+n FreeLayers(n)
                map.cell(ci, ii, bi) = c == 0   ? OffloadDecision{OffloadAction::NoAction, 0}
                                       : c == 1 ? OffloadDecision{OffloadAction::AllToHost, 0}
                                                : OffloadDecision{OffloadAction::FreeLayers, static_cast<std::uint64_t>(c - 2)};
            }
    return map;
}

/// build_hedging_map (maps.hpp:358-384), cells from the GPU.
inline HedgingMap build_hedging_map(const ModelProfile& m, const GpuProfile& g, std::uint64_t cached_step,
                                    std::uint64_t max_cached, TrainingMode mode,
                                    std::uint64_t assumed_output_tokens = 128) {
    validate_profile_pair(m, g);
    if (cached_step == 0 || max_cached == 0) throw std::runtime_error("hedging map: step and bound must be positive");
    if (max_cached % cached_step != 0)
        throw std::runtime_error("hedging map: cached bound is not a multiple of its step");
    HedgingMap map;
    map.cached_token_step = cached_step;
    map.max_cached_tokens = max_cached;
    map.num_layers = m.num_layers;
    map.mode = mode;
    map.assumed_output_tokens = assumed_output_tokens;
    map.profile_hash_value = profile_hash(m, g);
    map.init_cells();
    std::vector<std::uint8_t> hed;
    const colo_grid grid{500, 500, 5, 8000, 8000, 50};  // the offload half is not read back
    gpu_overlay::build_cells(m, g, grid, mode, cached_step, max_cached, assumed_output_tokens, nullptr, &hed);
    std::size_t k = 0;
    for (std::size_t ci = 0; ci < map.cached_count(); ++ci)
        for (std::size_t fi = 0; fi < map.freed_count(); ++fi, ++k)
            map.cell(ci, fi) = hed.at(k) ? HedgeDecision::Recompute : HedgeDecision::LoadBack;
    return map;
}

}  // namespace colosim
