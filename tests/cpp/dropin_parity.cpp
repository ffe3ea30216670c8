// dropin_parity.cpp -- the drop-in, exercised from C++: code written against
// the unchanged colosim headers (/root/reference/proj/include) hands its own
// ModelProfile / GpuProfile / GridSteps / GridBounds objects to colosim_gpu
// (paper_2503_01066_b200/cpp/colosim_gpu.hpp) and must get the reference's
// answers back, bit for bit.  Built by `make dropin` (needs /root/reference at
// build time only); run by tests/test_gpu_dropin.py on the GPU box.
#include <cstdio>
#include <cstring>
#include <random>

#include <nccl.h>

#include "colosim/engine.hpp"
#include "colosim/experiment.hpp"
#include "colosim_gpu.hpp"

using namespace colosim;

static int failures = 0;
#define EXPECT(cond, ...)                      \
    do {                                       \
        if (!(cond)) {                         \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");                 \
            ++failures;                        \
        }                                      \
    } while (0)

// engine.hpp:513-557 + 437-444 with the reference's own lookups
static uint32_t reference_verdict(const BuiltMaps& mp, uint64_t L, const colo_tuple& t) {
    auto dec = mp.offload.lookup(t.cached, t.incoming, t.batch);
    bool fallback = !dec;
    if (fallback) dec = OffloadDecision{OffloadAction::AllToHost, 0};
    uint32_t v = 0;
    if (dec->action != OffloadAction::NoAction) {
        uint64_t free_now = dec->action == OffloadAction::AllToHost ? t.dev_layers
                                                                    : std::min<uint64_t>(dec->layers, t.dev_layers);
        uint64_t total = std::min<uint64_t>(t.pending + dec->layers_to_free(L), L);
        bool recompute = true, hoor = false;
        if (!fallback) {
            auto h = mp.hedge.lookup(t.cached, total);
            if (h) recompute = *h == HedgeDecision::Recompute;
            else hoor = true;
        }
        uint32_t action = dec->action == OffloadAction::AllToHost ? 2 : 1;
        v = action | uint32_t((dec->action == OffloadAction::FreeLayers ? dec->layers : 0) << 2) |
            uint32_t(free_now << 10) | (recompute ? 1u << 18 : 0) | (fallback ? 1u << 19 : 0) | (hoor ? 1u << 20 : 0) |
            ((recompute ? 2u : 1u) << 21);
    }
    auto s = mp.offload.lookup(t.charged, 1, 1);
    if (!s) v |= (1u << 23) | (1u << 24);
    else if (s->action == OffloadAction::AllToHost) v |= 1u << 23;
    return v;
}

int main() {
    colosim_gpu::Context ctx(0);
    const GpuProfile gpu;
    for (ModelProfile model : {ModelProfile{}, ModelProfile::phi14b_like()}) {
        for (TrainingMode mode : {TrainingMode::CPA, TrainingMode::CPT}) {
            BuiltMaps ref = build_maps(model, gpu, GridSteps{}, GridBounds{}, mode);
            std::unique_ptr<colosim_gpu::GpuMaps> g(
                colosim_gpu::build_maps(ctx, model, gpu, GridSteps{}, GridBounds{}, mode == TrainingMode::CPA));
            EXPECT(g->profile_hash_value() == profile_hash(model, gpu), "profile hash");
            // every lookup the reference grid can answer, plus out-of-range probes
            for (uint64_t c = 0; c <= 8600; c += 97)
                for (uint64_t i = 0; i <= 8600; i += 131)
                    for (uint64_t b = 0; b <= 55; b += 3) {
                        auto r = ref.offload.lookup(c, i, b);
                        auto q = g->offload_lookup(c, i, b);
                        EXPECT(r.has_value() == q.has_value(), "offload nullopt (%lu,%lu,%lu)", c, i, b);
                        if (r && q)
                            EXPECT(int(r->action) == int(q->action) && r->layers == q->layers,
                                   "offload cell (%lu,%lu,%lu)", c, i, b);
                    }
            for (uint64_t c = 0; c <= 8600; c += 50)
                for (uint64_t f = 0; f <= model.num_layers + 1; ++f) {
                    auto r = ref.hedge.lookup(c, f);
                    auto q = g->hedge_lookup(c, f);
                    EXPECT(r.has_value() == q.has_value(), "hedge nullopt");
                    if (r && q) EXPECT((*r == HedgeDecision::Recompute) == *q, "hedge cell (%lu,%lu)", c, f);
                }
            std::mt19937_64 rng(42);
            std::vector<colo_tuple> tuples(2000000);
            for (auto& t : tuples) {
                t.cached = uint32_t(rng() % 9000);
                t.incoming = uint32_t(rng() % 9000);
                t.charged = uint32_t(rng() % 9500);
                t.batch = uint16_t(rng() % 60);
                t.pending = uint8_t(rng() % (model.num_layers + 4));
                t.dev_layers = uint8_t(rng() % (model.num_layers + 4));
            }
            uint64_t cnt[COLO_NCOUNTERS] = {};
            std::vector<uint32_t> v = g->decide(tuples, cnt);
            size_t bad = 0;
            for (size_t k = 0; k < tuples.size(); ++k) bad += v[k] != reference_verdict(ref, model.num_layers, tuples[k]);
            EXPECT(bad == 0, "%zu of %zu verdicts differ", bad, tuples.size());
            EXPECT(cnt[COLO_CNT_TOTAL] == tuples.size(), "counter total");
        }
        // serving replay: Simulation::run(ServingOnly) vs the GPU replay, sample for sample
        LengthDistribution lengths = LengthDistribution::uniform(100, 4000);
        for (double qps : {0.05, 0.4, 1.7}) {
            Trace trace = generate_trace(qps, 1500.0, lengths, std::nullopt, 17);
            SimConfig cfg;
            cfg.mode = SimMode::ServingOnly;
            cfg.model = model;
            cfg.gpu = gpu;
            cfg.trace = trace;
            MetricsReport rep = run_simulation(cfg);
            std::vector<double> a;
            std::vector<uint32_t> p, o;
            for (const auto& r : trace.records) {
                a.push_back(r.arrival_time);
                p.push_back(uint32_t(r.prompt_tokens));
                o.push_back(uint32_t(r.output_tokens));
            }
            auto g = colosim_gpu::replay_serving(ctx, model, gpu, a, p, o, 0.05);
            EXPECT(g.tpt_samples.size() == rep.tpt_samples.size(), "sample count qps %.2f", qps);
            EXPECT(std::memcmp(g.tpt_samples.data(), rep.tpt_samples.data(), 8 * rep.tpt_samples.size()) == 0,
                   "TPT samples differ at qps %.2f", qps);
            EXPECT(g.summary.peak_device_bytes == rep.peak_device_bytes, "peak bytes");
            EXPECT(g.summary.generated_tokens == rep.generated_tokens, "generated tokens");
        }
    }
    // Simulation::run in every mode: the reference's MetricsReport, operator== (samples,
    // finalize results, counters, mode tag, trace hash), from one GPU fleet launch
    {
        const GpuProfile gpu;
        std::vector<SimConfig> cfgs;
        std::vector<BuiltMaps> keep;
        for (ModelProfile model : {ModelProfile{}, ModelProfile::phi14b_like()})
            for (TrainingMode tm : {TrainingMode::CPA, TrainingMode::CPT}) {
                BuiltMaps maps = build_maps(model, gpu, GridSteps{}, GridBounds{}, tm);
                int k = 0;
                for (double qps : {0.05, 0.3, 1.2})
                    for (SimMode sm : {SimMode::Colocated, SimMode::SeparateCluster, SimMode::ServingOnly}) {
                        std::optional<LengthDistribution> ld = LengthDistribution::fixed(0.01);
                        if (++k % 3 == 0) ld = LengthDistribution::uniform(0.0, 60.0);
                        Trace t = generate_trace(qps, 60.0 / qps + 200.0, LengthDistribution::uniform(300, 7000), ld,
                                                 100 + k);
                        cfgs.push_back(make_sim_config(model, gpu, sm, tm, maps, t, 60.0));
                    }
            }
        // the engine tests' offload / stream cases (tests/test_engine.cpp:213-248)
        BuiltMaps cpa = build_maps(ModelProfile{}, gpu, GridSteps{}, GridBounds{}, TrainingMode::CPA);
        Trace burst;
        burst.records = {QueryRecord{0, 0.0, 4000, 128, 0.01}};
        for (std::uint64_t i = 1; i <= 10; ++i)
            burst.records.push_back(QueryRecord{i, 4.6 + 0.001 * double(i), 2000, 128, std::nullopt});
        cfgs.push_back(make_sim_config(ModelProfile{}, gpu, SimMode::Colocated, TrainingMode::CPA, cpa, burst));
        cfgs.push_back(make_sim_config(ModelProfile{}, gpu, SimMode::Colocated, TrainingMode::CPA, cpa,
                                       uncontended_trace(6000, 2, 2000.0)));
        cfgs.push_back(make_sim_config(ModelProfile{}, gpu, SimMode::SeparateCluster, TrainingMode::CPA, cpa,
                                       uncontended_trace(4000, 2, 2000.0)));  // trainer OOM datapoint
        std::vector<MetricsReport> got = colosim_gpu::run_simulations<MetricsReport>(ctx, cfgs);
        size_t bad = 0;
        for (size_t i = 0; i < cfgs.size(); ++i) {
            MetricsReport want = run_simulation(cfgs[i]);
            if (!(got[i] == want)) {
                ++bad;
                std::printf("  run %zu (%s): generated %llu/%llu trained %llu/%llu jobs %llu/%llu\n", i,
                            want.mode_tag.c_str(), (unsigned long long)got[i].generated_tokens,
                            (unsigned long long)want.generated_tokens, (unsigned long long)got[i].trained_tokens,
                            (unsigned long long)want.trained_tokens, (unsigned long long)got[i].completed_jobs,
                            (unsigned long long)want.completed_jobs);
            }
        }
        EXPECT(bad == 0, "%zu of %zu MetricsReports differ from Simulation::run", bad, cfgs.size());
        EXPECT(got.back().oom_flag && got.back().oom_jobs == 2, "trainer OOM datapoint");
        // the event log (SimConfig::collect_events, Simulation::events_json, engine.hpp:166-175)
        size_t ev_bad = 0, ev_done = 0;
        for (size_t i = 0; i < cfgs.size() && ev_done < 8; i += 3) {
            SimConfig ec = cfgs[i];
            ec.collect_events = true;
            Simulation sim(ec);
            try {
                sim.run();
            } catch (const std::exception&) {
                continue;  // a breaching run has no log
            }
            ++ev_done;
            if (colosim_gpu::events_json(ctx, cfgs[i]) != sim.events_json()) {
                ++ev_bad;
                std::printf("  events of run %zu differ\n", i);
            }
        }
        EXPECT(ev_done >= 4 && ev_bad == 0, "%zu of %zu event logs differ from Simulation::events_json", ev_bad, ev_done);
        // the constructor's refusals (engine.hpp:60-75)
        SimConfig badhash = cfgs[0];
        badhash.offload_map.profile_hash_value ^= 1;
        badhash.hedge_map.profile_hash_value ^= 1;
        try {
            colosim_gpu::run_simulation<MetricsReport>(ctx, badhash);
            EXPECT(false, "map hash mismatch accepted");
        } catch (const std::runtime_error&) {
        }
    }
    // fleet statistics over an NCCL communicator (one rank here): the same
    // bits as the single-process colo_serving_stats
    {
        ncclUniqueId id;
        ncclComm_t comm;
        EXPECT(ncclGetUniqueId(&id) == ncclSuccess, "ncclGetUniqueId");
        EXPECT(ncclCommInitRank(&comm, 1, id, 0) == ncclSuccess, "ncclCommInitRank");
        Trace trace = generate_trace(0.9, 3000.0, LengthDistribution::uniform(100, 4000), std::nullopt, 23);
        std::vector<double> a;
        std::vector<uint32_t> p, o;
        for (const auto& r : trace.records) {
            a.push_back(r.arrival_time);
            p.push_back(uint32_t(r.prompt_tokens));
            o.push_back(uint32_t(r.output_tokens));
        }
        colo_ctx* c = ctx.get();
        const size_t n = a.size();
        void *d_a, *d_p, *d_o, *d_off, *d_prof;
        colosim_gpu::check(colo_dev_alloc(c, n * 8, &d_a), c, "alloc");
        colosim_gpu::check(colo_dev_alloc(c, n * 4, &d_p), c, "alloc");
        colosim_gpu::check(colo_dev_alloc(c, n * 4, &d_o), c, "alloc");
        colosim_gpu::check(colo_dev_alloc(c, 16, &d_off), c, "alloc");
        colosim_gpu::check(colo_dev_alloc(c, 2, &d_prof), c, "alloc");
        const uint64_t offs[2] = {0, n};
        const uint16_t prof = 0;
        colo_memcpy_h2d(c, d_a, a.data(), n * 8);
        colo_memcpy_h2d(c, d_p, p.data(), n * 4);
        colo_memcpy_h2d(c, d_o, o.data(), n * 4);
        colo_memcpy_h2d(c, d_off, offs, 16);
        colo_memcpy_h2d(c, d_prof, &prof, 2);
        colo_model cm = colosim_gpu::to_c_model(ModelProfile{});
        colo_gpu cg = colosim_gpu::to_c_gpu(GpuProfile{});
        double p1[4], p2[4];
        colo_device_summary t1{}, t2{};
        EXPECT(colo_serving_stats(c, &cm, &cg, 1, (double*)d_a, (uint32_t*)d_p, (uint32_t*)d_o, n, (uint64_t*)d_off,
                                  (uint16_t*)d_prof, 1, 0.05, p1, &t1) == COLO_OK, "serving_stats");
        EXPECT(colo_serving_stats_nccl(c, comm, &cm, &cg, 1, (double*)d_a, (uint32_t*)d_p, (uint32_t*)d_o, n,
                                       (uint64_t*)d_off, (uint16_t*)d_prof, 1, 0.05, p2, &t2) == COLO_OK,
               "serving_stats_nccl: %s", colo_last_error(c));
        EXPECT(std::memcmp(p1, p2, sizeof p1) == 0, "NCCL stats percentiles differ");
        EXPECT(std::memcmp(&t1, &t2, sizeof t1) == 0, "NCCL stats totals differ");
        MetricsReport rep = run_simulation([&] {
            SimConfig cfg;
            cfg.mode = SimMode::ServingOnly;
            cfg.trace = trace;
            return cfg;
        }());
        EXPECT(p2[0] == *rep.tpt_p50 && p2[1] == *rep.tpt_p90 && p2[2] == *rep.tpt_p99, "NCCL stats vs finalize");
        for (void* q : {d_a, d_p, d_o, d_off, d_prof}) colo_dev_free(c, q);
        ncclCommDestroy(comm);
    }
    // the reference's error contract through the shim
    try {
        GpuProfile tiny;
        tiny.capacity_bytes = kGiB;
        colosim_gpu::build_maps(ctx, ModelProfile{}, tiny, GridSteps{}, GridBounds{}, true);
        EXPECT(false, "tiny gpu accepted");
    } catch (const std::runtime_error&) {
    }
    std::printf("%s: dropin parity, %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
