// overlay/colosim/engine.hpp -- the reference's engine.hpp with Simulation
// and run_simulation running on the GPU.
//
// With paper_2503_01066_b200/cpp/overlay first on the include path, code
// written against colosim (tools/colosim.cpp and experiment.hpp, unchanged)
// gets this header for `#include "colosim/engine.hpp"`.  The reference
// header is included next with its Simulation / run_simulation renamed by
// macro (they stay available as Simulation_cpu_reference /
// run_simulation_cpu_reference); everything else it declares -- SimConfig,
// SimMode, LoggedEvent, InvariantBreach, MetricsReport via metrics.hpp -- is
// the reference's own.  Simulation below keeps the reference's public API
// (engine.hpp:131-175, 938-941):
//   Simulation(SimConfig)  validates exactly as the reference (SimConfig::validate)
//   run()                  one device of colo_replay_colocated on sm_100a, in the
//                          config's SimMode; the report is finalized on the GPU
//                          (colo_finalize, bit-exact metrics.hpp:56-69)
//   events() / events_json()  the event log from the GPU run (colo_colocated_events)
//                          when cfg.collect_events, as the reference logs it
// and throws InvariantBreach where the reference's run() does.
#pragma once

#include "colosim_gpu_context.hpp"  // before the renaming macros below

#define Simulation Simulation_cpu_reference
#define run_simulation run_simulation_cpu_reference
#include_next <colosim/engine.hpp>
#undef Simulation
#undef run_simulation

#include <string>
#include <utility>


namespace colosim {

class Simulation {
  public:
    explicit Simulation(SimConfig cfg) : cfg_(std::move(cfg)) { cfg_.validate(); }  // engine.hpp:133-134

    MetricsReport run() {
        colosim_gpu::Context& ctx = colosim_gpu::process_context();
        try {
            MetricsReport r = colosim_gpu::run_simulation<MetricsReport>(ctx, cfg_);
            if (cfg_.collect_events) events_ = colosim_gpu::events_json(ctx, cfg_);
            return r;
        } catch (const colosim_gpu::invariant_breach& e) {
            throw InvariantBreach(e.what(), 0);
        }
    }

    /// engine.hpp:166-175: one LoggedEvent::to_json line per logged event.
    std::string events_json() const { return events_; }

  private:
    SimConfig cfg_;
    std::string events_;
};

inline MetricsReport run_simulation(SimConfig cfg) {  // engine.hpp:938-941
    Simulation sim(std::move(cfg));
    return sim.run();
}

}  // namespace colosim
