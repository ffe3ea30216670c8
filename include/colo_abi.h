/*
 * colo_abi.h -- C-ABI of colo-b200, the sm_100a implementation of the colosim
 * (arXiv 2503.01066 artifact) admission hot path.
 *
 * Plain C: POD structs, raw pointers and sizes, status codes.  No exceptions,
 * no C++ or torch types cross this boundary.  Device-pointer entry points
 * (d_*) are asynchronous on the context's stream; *_host entry points take
 * host buffers and return after the results are back in host memory.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj/):
 *
 *   colo_model / colo_gpu           ModelProfile / GpuProfile        include/colosim/profiles.hpp:23-35, 98-102
 *   colo_validate_profile_pair      validate_profile_pair            include/colosim/profiles.hpp:129-134
 *   colo_profile_hash               profile_hash                     include/colosim/profiles.hpp:137-152
 *   colo_validate_grid              validate_grid                    include/colosim/maps.hpp:197-208
 *   colo_mapset_build               build_offloading_map +           include/colosim/maps.hpp:233-252
 *                                   build_hedging_map (build_maps)   include/colosim/maps.hpp:358-384,
 *                                                                    include/colosim/experiment.hpp:144-152
 *   colo_mapset_from_cells          OffloadingMap::load / HedgingMap::load (hash refusal)
 *                                                                    include/colosim/maps.hpp:142-191, 297-332
 *   colo_mapset_cells               OffloadingMap::cell / HedgingMap::cell (save path)
 *                                                                    include/colosim/maps.hpp:89-94, 269-270
 *   colo_decide                     OffloadingMap::lookup + HedgingMap::lookup composed as
 *                                   Simulation::apply_offload_decision (decision half) and
 *                                   admit_to_store's streaming flag  include/colosim/maps.hpp:100-110, 276-280;
 *                                                                    include/colosim/engine.hpp:434-448, 513-557
 *   colo_decide_exact               offload_cell_decision + hedge_residual_load_time /
 *                                   hedge_recompute_time (un-quantised)
 *                                                                    include/colosim/maps.hpp:215-231, 341-356
 *   colo_features                   serving_memory / prefill_latency / charged tokens
 *                                                                    include/colosim/cost_model.hpp:18-66;
 *                                                                    include/colosim/engine.hpp:297, 422-423
 *   colo_features_decide(_host)     per-query feature extraction fused with the decision
 *                                   (SURVEY.md §8(d) C2 rule)
 *   colo_validate_trace             validate_trace (stable sort by (arrival, id), checks)
 *                                                                    include/colosim/workload.hpp:164-188
 *   colo_replay_serving             Simulation::run in SimMode::ServingOnly
 *                                                                    include/colosim/engine.hpp:140-164, 270-387
 *   colo_replay_colocated           Simulation::run in SimMode::Colocated (the admission loop:
 *                                   slot, offloader, hedge, prefetch, preemption, cache timeout)
 *                                                                    include/colosim/engine.hpp:140-822,
 *                                                                    include/colosim/memory.hpp:19-211
 *   colo_colocated_stats            run_simulation(Colocated) + finalize over a device set
 *                                                                    include/colosim/engine.hpp:938-941,
 *                                                                    include/colosim/metrics.hpp:56-69
 *   colo_hist_select / percentiles  finalize / nearest_rank          include/colosim/metrics.hpp:48-69
 *   colo_generate_trace             generate_trace (host, bit-exact) include/colosim/workload.hpp:193-220
 *   colo_stats_allreduce /          the fleet-wide statistics exchange (no reference
 *   colo_serving_stats_nccl         counterpart: the reference is single-process)
 */
#ifndef COLO_ABI_H
#define COLO_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COLO_ABI_VERSION 1

/* ------------------------------------------------------------------ status */
typedef enum colo_status {
    COLO_OK = 0,
    COLO_EINVAL = 1,      /* contract violation (reference: std::invalid_argument) or unsupported size */
    COLO_EVALIDATION = 2, /* validation failure (reference: std::runtime_error; CLI exit 2) */
    COLO_EBREACH = 3,     /* invariant breach (reference: InvariantBreach; CLI exit 3) */
    COLO_ECUDA = 4        /* CUDA runtime error; colo_last_error() has the text */
} colo_status;

/* ---------------------------------------------------------------- profiles */
/* ModelProfile, include/colosim/profiles.hpp:23-35 (same field order). */
typedef struct colo_model {
    uint64_t num_layers;
    uint64_t kv_bytes_per_token;
    uint64_t act_bytes_per_token_per_layer;
    double prefill_coef_linear;
    double prefill_coef_quad;
    double decode_coef_const;
    double decode_coef_context;
    double backward_to_forward_ratio;
    double record_prefill_multiplier;
    double record_decode_multiplier;
    double workspace_factor;
    uint64_t weights_bytes;
} colo_model;

/* GpuProfile, include/colosim/profiles.hpp:98-102. */
typedef struct colo_gpu {
    uint64_t capacity_bytes;
    uint64_t h2d_bandwidth;
    uint64_t d2h_bandwidth;
    uint64_t runtime_reserve_bytes;
} colo_gpu;

/* GridSteps + GridBounds, include/colosim/maps.hpp:63-73.  This build also
 * requires step <= 2^31 and max + step <= 2^32 on every axis (COLO_EINVAL). */
typedef struct colo_grid {
    uint64_t cached_step, incoming_step, batch_step;
    uint64_t max_cached, max_incoming, max_batch;
} colo_grid;

/* TrainingMode, include/colosim/maps.hpp:16. */
typedef enum colo_mode { COLO_CPT = 0, COLO_CPA = 1 } colo_mode;

/* --------------------------------------------------------- decision inputs */
/* One admission question, 16 B.  Field meaning at the engine call sites:
 *   cached     store.cached_tokens, the slot's charged tokens      engine.hpp:515
 *   incoming   max_incoming of the batch                           engine.hpp:304, 516
 *   charged    charged tokens of a query considered for the slot   engine.hpp:422-423, 438
 *   batch      batch size n                                        engine.hpp:516
 *   pending    store.host_only_pending()                           engine.hpp:529
 *   dev_layers store.device_resident_layers()                      engine.hpp:524 */
typedef struct colo_tuple {
    uint32_t cached;
    uint32_t incoming;
    uint32_t charged;
    uint16_t batch;
    uint8_t pending;
    uint8_t dev_layers;
} colo_tuple;

/* ------------------------------------------------------------ verdict word */
/* Packed 32-bit verdict.  action/layers are the offload decision after the
 * engine's nullopt->AllToHost substitution (engine.hpp:517-521); free_now is
 * engine.hpp:524-527; hedge bit is 1 for Recompute (engine.hpp:532-539);
 * verdict is the outcome (ADMIT = engine.hpp:522, FREE_LOADBACK = :546-548,
 * RECOMPUTE_DROP = :541-544); stream is admit_to_store's pre-commitment for
 * `charged` (engine.hpp:437-444).  *_OOR bits are the nullopt lookups the
 * engine counts as map_fallbacks (engine.hpp:519, 538, 441). */
#define COLO_V_ACTION(v) ((v) & 0x3u)            /* 0 NoAction, 1 FreeLayers, 2 AllToHost */
#define COLO_V_LAYERS(v) (((v) >> 2) & 0xffu)    /* FreeLayers(n), else 0 */
#define COLO_V_FREE_NOW(v) (((v) >> 10) & 0xffu)
#define COLO_V_HEDGE_RECOMPUTE (1u << 18)
#define COLO_V_OFFLOAD_OOR (1u << 19)
#define COLO_V_HEDGE_OOR (1u << 20)
#define COLO_V_VERDICT(v) (((v) >> 21) & 0x3u)   /* 0 ADMIT, 1 FREE_LOADBACK, 2 RECOMPUTE_DROP */
#define COLO_V_STREAM (1u << 23)
#define COLO_V_STREAM_OOR (1u << 24)

enum { COLO_ACT_NOACTION = 0, COLO_ACT_FREELAYERS = 1, COLO_ACT_ALLTOHOST = 2 };
enum { COLO_VD_ADMIT = 0, COLO_VD_FREE_LOADBACK = 1, COLO_VD_RECOMPUTE_DROP = 2 };

/* Decision counters (optional u64[COLO_NCOUNTERS] device array, accumulated). */
enum {
    COLO_CNT_ADMIT = 0,
    COLO_CNT_FREE_LOADBACK = 1,
    COLO_CNT_RECOMPUTE_DROP = 2,
    COLO_CNT_OFFLOAD_OOR = 3,
    COLO_CNT_HEDGE_OOR = 4,
    COLO_CNT_STREAM = 5,
    COLO_CNT_STREAM_OOR = 6,
    COLO_CNT_TOTAL = 7,
    COLO_NCOUNTERS = 8
};

/* Offload cell byte code (device map storage and colo_mapset_cells):
 * 0 NoAction, 1 AllToHost, 2+n FreeLayers(n).  Requires num_layers <= 253.
 * Hedge cell byte: 0 LoadBack, 1 Recompute. */

/* ----------------------------------------------------------------- context */
typedef struct colo_ctx colo_ctx;
typedef struct colo_mapset colo_mapset;

colo_status colo_ctx_create(int device, colo_ctx** out);
void colo_ctx_destroy(colo_ctx* ctx);
/* Launch on a caller-owned cudaStream_t (NULL = the legacy default stream).
 * A new context launches on its own non-blocking stream. */
colo_status colo_ctx_set_stream(colo_ctx* ctx, void* cuda_stream);
void* colo_ctx_stream(colo_ctx* ctx);
colo_status colo_sync(colo_ctx* ctx);
/* Frees the context's grow-only scratch (replay segment state, the serving
 * replay's all-queued records and step durations -- tens of GB after a
 * billion-query replay -- decode tables, host-pipeline buffers).  They are
 * re-created on demand; colo_ctx_destroy frees them too. */
colo_status colo_ctx_release_scratch(colo_ctx* ctx);
/* Let ctx use owner's per-call replay temporaries (the serving replay's
 * all-queued batch records and their step-duration pool, only live during one
 * colo_replay_serving call) instead of growing its own.  For several contexts
 * that each hold one chunk of a rank's devices across the three exact-stats
 * passes (their segment entry states and sparse-pass records stay per
 * context): calls on ctx and owner must not overlap (one host thread, one
 * stream).  owner = NULL or ctx restores ctx's own buffers. */
colo_status colo_ctx_share_temps(colo_ctx* ctx, colo_ctx* owner);
const char* colo_last_error(const colo_ctx* ctx);
int colo_ctx_sm_count(const colo_ctx* ctx);
/* Kernels this context has launched so far (the library's own kernels; the
 * sorts and scans it takes from CUB are not counted). */
uint64_t colo_ctx_launches(const colo_ctx* ctx);
int colo_abi_version(void);

/* Device memory helpers for C/C++ callers without another allocator. */
colo_status colo_dev_alloc(colo_ctx* ctx, size_t bytes, void** d_ptr);
colo_status colo_dev_free(colo_ctx* ctx, void* d_ptr);
colo_status colo_memcpy_h2d(colo_ctx* ctx, void* d_dst, const void* h_src, size_t bytes);
colo_status colo_memcpy_d2h(colo_ctx* ctx, void* h_dst, const void* d_src, size_t bytes);

/* ------------------------------------------------- profiles (host, no GPU) */
colo_status colo_validate_profile_pair(const colo_model* m, const colo_gpu* g);
uint64_t colo_profile_hash(const colo_model* m, const colo_gpu* g);
colo_status colo_validate_grid(const colo_grid* grid);

/* -------------------------------------------------------------- map sets */
/* Builds the offloading map (grid) and the hedging map (hedge_step,
 * hedge_max; build_maps passes grid.cached_step / grid.max_cached) on the
 * device, one thread per cell.  EVALIDATION exactly where build_* throw. */
colo_status colo_mapset_build(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const colo_grid* grid,
                              colo_mode mode, uint64_t hedge_step, uint64_t hedge_max,
                              uint64_t assumed_output_tokens, colo_mapset** out);
/* Load path: host cell arrays plus the hash they were built under; refuses a
 * hash different from profile_hash(m, g) with EVALIDATION (maps.hpp:155-157). */
colo_status colo_mapset_from_cells(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const colo_grid* grid,
                                   colo_mode mode, uint64_t hedge_step, uint64_t hedge_max,
                                   uint64_t assumed_output_tokens, uint64_t built_hash,
                                   const uint8_t* h_offload_cells, size_t n_offload, const uint8_t* h_hedge_cells,
                                   size_t n_hedge, colo_mapset** out);
colo_status colo_mapset_shape(const colo_mapset* ms, size_t* n_offload, size_t* n_hedge);
colo_status colo_mapset_cells(colo_ctx* ctx, const colo_mapset* ms, uint8_t* h_offload, size_t n_offload,
                              uint8_t* h_hedge, size_t n_hedge);
uint64_t colo_mapset_hash(const colo_mapset* ms);
void colo_mapset_destroy(colo_mapset* ms);

/* ----------------------------------------------------------------- decide */
/* Quantised (map) verdicts for n tuples.  d_counters: NULL or u64[COLO_NCOUNTERS]. */
colo_status colo_decide(colo_ctx* ctx, const colo_mapset* ms, const colo_tuple* d_in, size_t n, uint32_t* d_out,
                        uint64_t* d_counters);
/* Exact per-query verdicts (no quantisation).  Domain rules: incoming==0 or
 * batch==0 -> OFFLOAD_OOR; cached==0 with a non-NoAction offload -> HEDGE_OOR
 * (forced Recompute), mirroring the lookups' nullopt cases. */
colo_status colo_decide_exact(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, colo_mode mode,
                              uint64_t assumed_output_tokens, const colo_tuple* d_in, size_t n, uint32_t* d_out,
                              uint64_t* d_counters);

/* Trace-fused features -> verdict.  Trace SoA (prompt, output: n u32 each),
 * partitioned by device with CSR offsets d_dev_offsets[ndev+1]; device d uses
 * map set sets[d_dev_set[d]].  Query i of device d asks
 *   (cached = charged(previous query of d) or 0, incoming = p+o, batch = 1,
 *    pending = 0, dev_layers = L, charged = charged(i)),
 * charged = p + 2o (CPA) or p (CPT), engine.hpp:422-423. */
colo_status colo_features_decide(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets,
                                 const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                 const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev,
                                 uint32_t* d_out, uint64_t* d_counters);
/* Same over host buffers: chunked H2D / kernel / D2H pipeline on the context's
 * stream pair.  h_* may be pageable or pinned (pinned is faster); the
 * device-side offsets/sets are staged by the call. */
colo_status colo_features_decide_host(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets,
                                      const uint32_t* h_prompt, const uint32_t* h_output, size_t n,
                                      const uint64_t* h_dev_offsets, const uint16_t* h_dev_set, size_t ndev,
                                      uint32_t* h_out, uint64_t* h_counters);
/* Tuple-stream verdicts over host buffers. */
colo_status colo_decide_host(colo_ctx* ctx, const colo_mapset* ms, const colo_tuple* h_in, size_t n,
                             uint32_t* h_out, uint64_t* h_counters);

/* Per-query cost-model features (debug/parity outputs; any pointer may be NULL):
 * need = serving_memory(p+o, 1), charged, unrecorded prefill_latency(p, 1). */
colo_status colo_features(colo_ctx* ctx, const colo_model* m, colo_mode mode, const uint32_t* d_prompt,
                          const uint32_t* d_output, size_t n, uint64_t* d_need, uint64_t* d_charged,
                          double* d_prefill);

/* ---------------------------------------------------------- serving replay */
typedef struct colo_batch {
    double start;          /* prefill start (engine.hpp:321) */
    double end;            /* time of the batch's last decode step */
    uint32_t first;        /* first query, index within the device */
    uint32_t n;            /* batch size */
    uint64_t need_total;   /* engine.hpp:303 */
    uint32_t max_incoming; /* engine.hpp:304 (saturated at 2^32-1) */
    uint32_t verdict;      /* replay-derived verdict (SURVEY §8(d) C3 rule), 0 if no map sets */
} colo_batch;

typedef struct colo_device_summary {
    uint64_t generated_tokens;  /* MetricsReport::generated_tokens */
    uint64_t slow_tokens;       /* tokens with TPT > tau */
    uint64_t slow_queries;      /* queries with any token TPT > tau */
    uint64_t batches;
    uint64_t peak_device_bytes; /* MetricsReport::peak_device_bytes (ServingOnly) */
    uint64_t max_batch_size;
    double end_time;            /* time of the last decode step */
    uint64_t tpt_sum[3];        /* exact sum of TPT samples, fixed point, LSB 2^-96 (little-endian limbs) */
    uint64_t flags;             /* bit0: a sample fell outside the exact-sum range */
} colo_device_summary;

#define COLO_HIST_BITS 21
#define COLO_HIST_BINS (1u << COLO_HIST_BITS)

typedef struct colo_replay_opts {
    double tau;                       /* slow-token threshold (TPT > tau) */
    const colo_mapset* const* sets;   /* NULL, or per-profile map sets for replay-derived verdicts */
    /* output buffers (device pointers, each may be NULL) */
    double* d_samples;                /* TPT samples in reference order; needs d_sample_offsets */
    const uint64_t* d_sample_offsets; /* [ndev+1] prefix sums of output tokens per device */
    uint8_t* d_labels;                /* [n] 1 = slow query */
    colo_batch* d_batches;            /* batch b of device d at d_dev_offsets[d] + b */
    colo_device_summary* d_summary;   /* [ndev] */
    /* TPT histogram pass (radix select over f64 bit patterns): a sample with
     * bits x adds its multiplicity to d_hist[f * COLO_HIST_BINS + ((x >> hist_shift) & (BINS-1))]
     * for every filter f with (x >> filter_shift) == filter_prefix[f]. */
    uint64_t* d_hist;                 /* [nfilters * COLO_HIST_BINS] u64, accumulated; NULL = no pass */
    uint32_t nfilters;                /* 0..3 */
    uint32_t hist_shift;
    uint32_t filter_shift;            /* 63 with prefix 0 selects every sample */
    uint32_t segment_len;             /* queries per replay segment (0 = automatic), see below */
    uint64_t filter_prefix[3];
    uint32_t reuse_entries;           /* 1: the previous call on this context replayed the same trace:
                                         skip validation, speculation and resolution and reuse its segment
                                         entry states (histogram passes 2-3 of the exact-stats protocol).
                                         The context checks the buffers' addresses, the sizes, the profile
                                         contents and segment_len, and replays in full when they differ;
                                         it cannot see the buffers' contents, so the CALLER must guarantee
                                         the trace arrays were not rewritten in between. */
    uint32_t stats_mode;              /* sparse exact-stats passes: 1 = also record, per batch, its start
                                         and the range of its samples' top-21-bit bins (the first histogram
                                         pass); 2 (with reuse_entries, after a mode-1 call on the same
                                         trace) = replay only the batches whose range covers a filter bin
                                         (the narrowing passes; same histograms).  0 = off. */
    uint32_t* d_verdicts;             /* [n] replay-derived verdict of batch b of device d at
                                         d_dev_offsets[d] + b (needs sets; the same words d_batches'
                                         verdict field carries, without the 40 B records: SURVEY §8(d)
                                         C3, engine.hpp:513-557 composed per batch).  NULL = none. */
} colo_replay_opts;

/* validate_trace (workload.hpp:164-188) on the device, for every device of a
 * CSR trace: each device's rows [off[d], off[d+1]) are reordered in place by
 * (arrival, query_id) -- the reference's stable_sort -- across every given
 * column.  EVALIDATION (colo_last_error names the query, in the reference's
 * words) for a negative or NaN arrival, zero prompt or output tokens, or a
 * query_id repeated within one device.  d_query_id may be NULL (ids = the row
 * order, so equal arrivals keep their order); d_label_delay may be NULL.
 * n < 2^32.  Synchronous.  The replay entry points below take validated
 * traces (they reject unsorted input). */
colo_status colo_validate_trace(colo_ctx* ctx, uint64_t* d_query_id, double* d_arrival, uint32_t* d_prompt,
                                uint32_t* d_output, double* d_label_delay, size_t n, const uint64_t* d_dev_offsets,
                                size_t ndev);

/* Serving-only replay of every device's trace.  Each device is cut into
 * segments of segment_len queries; the replay runs in three passes:
 * speculate (every segment in parallel, from an idle server at its first
 * query), resolve (per device, in order: a segment whose true entry state is
 * not "idle at its first query" is replayed until it meets one of the
 * speculative run's idle batch starts, after which both runs coincide), and
 * replay (every segment in parallel from its true entry state, writing the
 * outputs).  Every f64 operation is the reference's, in the reference's
 * order, so the outputs are identical to a single sequential replay.
 * models/gpus: nprofiles profile pairs; d_dev_profile[ndev] picks one per
 * device.  Rejects (EVALIDATION) traces that are unsorted, have zero
 * prompt/output tokens, or hold a query that cannot fit the device alone
 * (engine.hpp:70-74). */
colo_status colo_replay_serving(colo_ctx* ctx, const colo_model* models, const colo_gpu* gpus, size_t nprofiles,
                                const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output,
                                size_t n, const uint64_t* d_dev_offsets, const uint16_t* d_dev_profile, size_t ndev,
                                const colo_replay_opts* opts);

/* Host: first bin whose running count reaches `rank` (1-based); returns the
 * bin and the rank within it.  EINVAL if the histogram holds fewer samples. */
colo_status colo_hist_select(const uint64_t* h_hist, size_t nbins, uint64_t rank, uint32_t* bin,
                             uint64_t* rank_in_bin);
/* nearest-rank index of metrics.hpp:48-53: max(1, ceil(q * n)). */
uint64_t colo_nearest_rank_index(double q, uint64_t n);

/* Single-GPU convenience: three replay passes, exact nearest-rank p50/p90/p99
 * (pctl[0..2]) and the mean (pctl[3], correctly rounded from the exact sum)
 * over all devices; also fills *totals (summed device summaries). */
colo_status colo_serving_stats(colo_ctx* ctx, const colo_model* models, const colo_gpu* gpus, size_t nprofiles,
                               const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                               const uint64_t* d_dev_offsets, const uint16_t* d_dev_profile, size_t ndev, double tau,
                               double* pctl, colo_device_summary* totals);

/* ------------------------------------------------------- colocated replay */
/* Per-device MetricsReport (metrics.hpp:17-44; the first 15 fields, same
 * meaning; oom_flag = oom_jobs > 0) plus replay extras.  training_throughput =
 * trained_tokens / training_busy_time when busy > 0 (metrics.hpp:67-68). */
typedef struct colo_colocated_summary {
    uint64_t generated_tokens;
    uint64_t trained_tokens;
    double training_busy_time;
    uint64_t peak_device_bytes;
    uint64_t peak_training_activation_bytes;
    uint64_t preemptions;
    uint64_t layers_freed;
    uint64_t loads;
    uint64_t recomputes;
    double copy_stall_seconds;
    uint64_t labels_dropped;
    double prefetch_wait_seconds;
    uint64_t completed_jobs;
    uint64_t map_fallbacks;
    uint64_t oom_jobs;          /* SeparateCluster: jobs the trainer could not fit (engine.hpp:841-845) */
    /* extras */
    uint64_t batches;
    uint64_t max_batch_size;
    uint64_t offload_decisions; /* apply_offload_decision calls (engine.hpp:309-310) */
    uint64_t admissions;        /* admit_to_store calls (engine.hpp:317-318) */
    uint64_t slow_tokens;       /* tokens with TPT > tau */
    uint64_t slow_queries;      /* queries with any token TPT > tau */
    double end_time;            /* time of the last decode step */
    uint64_t status;            /* COLO_OK, or COLO_EBREACH: the reference run throws (InvariantBreach /
                                   std::logic_error) and this device's other fields are partial */
    uint64_t tpt_sum[3];        /* exact sum of TPT samples, fixed point, LSB 2^-96 */
    uint64_t flags;             /* bit0: a sample fell outside the exact-sum range */
} colo_colocated_summary;

/* Extra verdict bits in colocated batch records (colo_batch.verdict): the
 * offload decision apply_offload_decision took for this batch (action,
 * layers, free_now, hedge, oor bits and the final outcome, including the KV
 * corner's drop, engine.hpp:549-552), and the slot admission. */
#define COLO_V_EVALUATED (1u << 25)  /* apply_offload_decision ran (engine.hpp:309-310) */
#define COLO_V_ADMITTED (1u << 26)   /* admit_to_store ran for this batch (engine.hpp:317-318);
                                        COLO_V_STREAM / _STREAM_OOR give its streaming flag */

/* SimMode (engine.hpp:23) per device in colo_colocated_opts.d_dev_sim_mode. */
enum { COLO_SIM_SERVING_ONLY = 0, COLO_SIM_COLOCATED = 1, COLO_SIM_SEPARATE = 2 };

typedef struct colo_colocated_opts {
    double cache_timeout;            /* SimConfig::cache_timeout (engine.hpp:55); the reference default is 60 */
    const double* d_label_delay;     /* [n] seconds; < 0 or NaN = the label never arrives; NULL = default_label_delay */
    double default_label_delay;      /* used when d_label_delay == NULL (< 0 = never) */
    double tau;                      /* slow-token threshold (TPT > tau) */
    double* d_samples;               /* TPT samples in reference order; needs d_sample_offsets */
    const uint64_t* d_sample_offsets;/* [ndev+1] prefix sums of output tokens per device */
    uint8_t* d_labels;               /* [n] 1 = slow query */
    colo_batch* d_batches;           /* batch b of device d at d_dev_offsets[d] + b */
    colo_colocated_summary* d_summary; /* [ndev] */
    uint64_t* d_hist;                /* TPT histogram pass, as colo_replay_opts */
    uint32_t nfilters;
    uint32_t hist_shift;
    uint32_t filter_shift;
    uint32_t seg_len;                /* 0: automatic -- with fewer devices than the GPU holds warps, long devices
                                        run in parallel segments split at idle arrivals (bit-identical results);
                                        0xffffffff: never; else the segment length in queries */
    uint64_t filter_prefix[3];
    const uint8_t* d_dev_sim_mode;   /* [ndev] COLO_SIM_*; NULL = every device Colocated */
} colo_colocated_opts;

/* Simulation::run of every device's trace, one warp per device, in the
 * device's SimMode (opts->d_dev_sim_mode; default Colocated).  Device d uses
 * map set sets[d_dev_set[d]], whose model, GPU profile and training mode are
 * the simulation's (SimConfig::validate requires the maps to match them,
 * engine.hpp:60-68).  SeparateCluster devices serve as ServingOnly and their
 * trainer (engine.hpp:824-903) is folded over the job stream afterwards, in
 * the reference's enqueue order (finish order for CPT; label arrival, ties in
 * finish order, for CPA -- a stable segmented sort when label delays vary).  Events are handled in the
 * reference's (time, sequence) order and every f64 operation is the
 * reference's in its order, so each device's report and samples equal
 * Simulation::run's.  EVALIDATION as colo_replay_serving; EBREACH when a
 * device's run breaches an invariant (its summary has status COLO_EBREACH).
 * Synchronous (returns after the replay finished). */
colo_status colo_replay_colocated(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const double* d_arrival,
                                  const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                  const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev,
                                  const colo_colocated_opts* opts);

/* Colocated replays of a device set plus exact TPT statistics over the union
 * of all devices' samples: pctl[0..2] nearest-rank p50/p90/p99, pctl[3] the
 * mean (correctly rounded from the exact sum); NaN without samples.  *totals:
 * counters summed, peaks maxed (d_summary may be NULL).  Three replay passes
 * (radix select over the f64 bit patterns). */
colo_status colo_colocated_stats(colo_ctx* ctx, const colo_mapset* const* sets, size_t nsets, const double* d_arrival,
                                 const uint32_t* d_prompt, const uint32_t* d_output, size_t n,
                                 const uint64_t* d_dev_offsets, const uint16_t* d_dev_set, size_t ndev,
                                 const colo_colocated_opts* opts, double* pctl, colo_colocated_summary* totals);

/* The event log of one device's Simulation::run (tools/colosim.cpp --emit-events;
 * LoggedEvent::to_json, engine.hpp:109-129, 241-244) in any SimMode: the run on the GPU records every logged event, which are put in
 * dispatch order ((time, sequence), engine.hpp:184-187) and formatted as the
 * reference formats them.  d_label_delay may be NULL (default_label_delay for
 * every query; < 0 = never); d_query_id may be NULL (ids 0..n-1).  Returns the
 * length of the JSON-lines text, kept in the context (colo_events_text), or
 * -status (EBREACH: the run breached, as the reference throws). */
int64_t colo_colocated_events(colo_ctx* ctx, const colo_mapset* set, int sim_mode, double cache_timeout,
                              const double* d_arrival, const uint32_t* d_prompt, const uint32_t* d_output,
                              const double* d_label_delay, double default_label_delay, const uint64_t* d_query_id,
                              size_t n, double tau);
/* Copies the last event log (NUL-terminated) when cap exceeds its length; returns the length. */
int64_t colo_events_text(colo_ctx* ctx, char* out, size_t cap);

/* ------------------------------------------------------------ report helpers */
/* Trace::content_hash (workload.hpp:140-161): FNV-1a over (query_id, arrival
 * bits, prompt, output, label_delay bits -- -1.0 for nullopt) per record.
 * label_delay may be NULL (all nullopt); a negative or NaN entry is nullopt. */
uint64_t colo_trace_hash(const uint64_t* query_id, const double* arrival, const uint32_t* prompt,
                         const uint32_t* output, const double* label_delay, size_t n);
/* Ascending sort of n f64 values on the device (the sorted TPT samples of
 * finalize / export_tpt_cdf, metrics.hpp:59-60, 280-288).  d_in and d_out may
 * not alias.  Synchronous. */
colo_status colo_sort_f64(colo_ctx* ctx, const double* d_in, double* d_out, size_t n);
/* finalize (metrics.hpp:56-69) of n TPT samples on the device, bit-exact:
 * out[0..2] nearest-rank p50/p90/p99 of the ascending sort, out[3] the mean as
 * the reference computes it -- the strictly sequential sum of the sorted
 * samples, divided by n (an exact parallel evaluation of that left fold;
 * NaN for n = 0).  d_sorted (may be NULL) receives the sorted samples.
 * Synchronous. */
colo_status colo_finalize(colo_ctx* ctx, const double* d_samples, size_t n, double* d_sorted, double* out);
/* n doubles formatted as nlohmann::json::dump() writes them (the reference's
 * report serializer, metrics.hpp:191-226), comma-separated, NUL-terminated
 * into out when cap exceeds the length.  Returns the length (without NUL). */
int64_t colo_json_doubles(const double* v, size_t n, char* out, size_t cap);

/* ------------------------------------------------------- multi-GPU stats */
/* The one cross-GPU exchange.  nccl_comm is the caller's
 * ncclComm_t (passed as void*; NCCL is resolved at run time, so this library
 * does not link it).  colo_stats_allreduce sums n u64 in place on the
 * context's stream.  colo_serving_stats_nccl is colo_serving_stats over a
 * device-sharded fleet: each rank replays its own devices and the histograms,
 * counters and exact sums are all-reduced between the passes, so every rank
 * returns the fleet-wide p50/p90/p99/mean and totals. */
colo_status colo_stats_allreduce(colo_ctx* ctx, void* nccl_comm, uint64_t* d_buf, size_t n);
colo_status colo_serving_stats_nccl(colo_ctx* ctx, void* nccl_comm, const colo_model* models, const colo_gpu* gpus,
                                    size_t nprofiles, const double* d_arrival, const uint32_t* d_prompt,
                                    const uint32_t* d_output, size_t n, const uint64_t* d_dev_offsets,
                                    const uint16_t* d_dev_profile, size_t ndev, double tau, double* pctl,
                                    colo_device_summary* totals);

/* --------------------------------------------------------- trace synthesis */
/* generate_trace (workload.hpp:193-220) on the host, bit-exact (mt19937_64 +
 * libm log).  dist kind: 0 fixed, 1 uniform, 2 histogram.  Returns the query
 * count, -1 if cap is too small, -2 on invalid input. */
typedef struct colo_dist {
    int kind;
    double fixed_value, lo, hi;
    const double* bin_values;
    const double* bin_probs;
    size_t nbins;
    uint64_t min_tokens; /* 0 = none */
} colo_dist;
int64_t colo_generate_trace(double qps, double duration, const colo_dist* lengths, const colo_dist* label_delay,
                            uint64_t seed, double* arrival, uint32_t* prompt, uint32_t* output, double* label_out,
                            size_t cap);
/* label_out (may be NULL): per-query label delay, sample_seconds of the
 * label-delay distribution (workload.hpp:118-120), -1.0 when label_delay is
 * NULL (QueryRecord::label_delay == nullopt). */

/* Bench-scale synthetic trace on the device (counter-based hash RNG, not
 * mt19937): per device d, queries [off[d], off[d+1]) get histogram-sampled
 * prompts (bin_values/bin_probs, <= 32 bins), output = 128, and arrivals
 * from the running sum of exponential gaps at qps[d].  Bursty traces: with
 * d_dev_qps_hi != NULL and burst_period > 0 the rate alternates between
 * qps[d] and qps_hi[d] every burst_period seconds (rate chosen per 32
 * arrivals).  The arrays are inputs only: parity is always checked by running
 * the oracle on the same arrays. */
colo_status colo_synth_trace(colo_ctx* ctx, const double* h_bin_values, const double* h_bin_probs, size_t nbins,
                             const uint64_t* d_dev_offsets, const double* d_dev_qps, const double* d_dev_qps_hi,
                             double burst_period, size_t ndev, uint64_t seed, double* d_arrival, uint32_t* d_prompt,
                             uint32_t* d_output);
/* The same with the RNG keyed on (d_dev_ids[d], query index within the
 * device) instead of the global query index, so fleet device g's trace is the
 * same whichever rank or array position holds it (C4: device g on rank
 * g % world at every world size).  Device ids < 2^28, devices < 2^36 queries. */
colo_status colo_synth_fleet_trace(colo_ctx* ctx, const double* h_bin_values, const double* h_bin_probs, size_t nbins,
                                   const uint64_t* d_dev_offsets, const double* d_dev_qps, const double* d_dev_qps_hi,
                                   double burst_period, size_t ndev, const uint32_t* d_dev_ids, uint64_t seed,
                                   double* d_arrival, uint32_t* d_prompt, uint32_t* d_output);

/* ------------------------------------------------------------ file formats */
/* Offloading / hedging map text files, byte-identical to OffloadingMap::save /
 * HedgingMap::save (maps.hpp:118-140, 284-295).  Loading refuses a profile
 * hash other than expected_hash with EVALIDATION (maps.hpp:155-157, 311-312);
 * cells == NULL queries the cell count.  err (optional) receives the
 * reference's message text. */
typedef struct colo_map_header {
    int kind;                 /* 0 offload, 1 hedge */
    colo_mode mode;
    uint64_t profile_hash;
    uint64_t num_layers;
    colo_grid grid;           /* hedge maps use cached_step and max_cached only */
    uint64_t assumed_output_tokens;
} colo_map_header;
colo_status colo_map_save(const char* path, const colo_map_header* h, const uint8_t* cells, size_t ncells);
colo_status colo_map_load(const char* path, uint64_t expected_hash, colo_map_header* h, uint8_t* cells, size_t cap,
                          size_t* ncells, char* err, size_t errlen);
colo_status colo_mapset_save(colo_ctx* ctx, const colo_mapset* ms, const char* offload_path, const char* hedge_path);
colo_status colo_mapset_load(colo_ctx* ctx, const colo_model* m, const colo_gpu* g, const char* offload_path,
                             const char* hedge_path, colo_mapset** out);
/* JSON-lines trace (load_trace, workload.hpp:224-254): one object per line
 * with query_id, arrival_time, prompt_tokens, output_tokens (default 128),
 * label_delay (null -> NaN); validated and ordered exactly as validate_trace
 * (stable sort by (arrival, id); negative arrival, zero tokens, duplicate ids
 * rejected).  Returns the record count, -1 if cap is too small, -2 on error. */
int64_t colo_load_trace_jsonl(const char* path, double* arrival, uint32_t* prompt, uint32_t* output,
                              uint64_t* query_id, double* label_delay, size_t cap, char* err, size_t errlen);
/* Histogram file of {tokens, probability} lines (load_histogram, workload.hpp:274-293). */
int64_t colo_load_histogram_jsonl(const char* path, double* values, double* probs, size_t cap, char* err,
                                  size_t errlen);

/* ------------------------------------------------------------ C5 sweep */
/* Synthetic admission questions on the device: cached
 * U[0,8000], incoming = p + 128 with p from the length histogram, batch
 * U[1,50], pending/dev_layers U[0,L], charged U[0,9000]; 1 % pushed out of the
 * default grid.  Counter-based RNG: input data only. */
colo_status colo_synth_tuples(colo_ctx* ctx, uint64_t seed, size_t n, uint32_t num_layers, const double* h_bin_values,
                              const double* h_bin_probs, size_t nbins, colo_tuple* d_out);
/* Map-vs-exact statistics over two verdict arrays on the same questions:
 * d_counts[0] += agree on (action, layers), [1] += map frees more layers,
 * [2] += map frees fewer, [3] += same outcome, [4] += total. */
colo_status colo_compare_verdicts(colo_ctx* ctx, const uint32_t* d_map, const uint32_t* d_exact, size_t n,
                                  uint32_t num_layers, uint64_t* d_counts);

#ifdef __cplusplus
}
#endif
#endif /* COLO_ABI_H */
