// colo_internal.h -- host-side internals shared by the colo-b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "colo_abi.h"
#include "colo_common.cuh"

struct colo_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own = nullptr;     // context-owned compute stream
    cudaStream_t stream = nullptr;  // current stream (own or caller's)
    cudaStream_t aux = nullptr;     // second stream for the host-buffer pipelines
    std::string err;
    std::string evtext;             // the last colo_colocated_events log (JSON lines)
    int* d_flag = nullptr;          // device error flag (replay validation)
    // host-pipeline scratch (lazily grown)
    void* d_pipe = nullptr;
    size_t pipe_bytes = 0;
    uint64_t* d_counters = nullptr; // COLO_NCOUNTERS scratch
    void* d_rscratch = nullptr;     // replay segment state (lazily grown)
    size_t rscratch_bytes = 0;
    void* d_sat = nullptr;          // serving replay: all-queued batch records (lazily grown)
    size_t sat_bytes = 0;
    void* d_satpool = nullptr;      // serving replay: their step durations (lazily grown)
    size_t satpool_bytes = 0;
    void* d_dtab = nullptr;         // serving replay: decode-latency tables (lazily grown)
    size_t dtab_bytes = 0;
    void* d_seg = nullptr;          // colocated replay: segment tasks / idle lists / partial reports (lazily grown)
    size_t seg_bytes = 0;
    void* d_seglog = nullptr;       // colocated replay: the segments' f64 addend logs (lazily grown)
    size_t seglog_bytes = 0;
    void* d_tmp = nullptr;          // small library temp storage (cub scans; lazily grown)
    size_t tmp_bytes = 0;
    void* d_bmeta = nullptr;        // serving stats: per-query batch start + sample-bin range (lazily grown)
    size_t bmeta_bytes = 0;
    bool bmeta_valid = false;       // d_bmeta holds the batch records of the replay rs_sig describes
    uint16_t* d_htab = nullptr;     // exact decide: per-value hedge thresholds + stream bits (k_exact_tab)
    unsigned char htab_key[sizeof(colo_model) + sizeof(colo_gpu) + 16] = {};  // what d_htab was built for
    bool htab_valid = false;
    // serving replay: identity of the last full replay whose segment entry
    // states are still in d_rscratch (reuse_entries); any other d_rscratch
    // user clears rs_valid
    uint64_t rs_sig[11] = {};
    bool rs_valid = false;
    uint64_t launches = 0;          // kernels this context launched (colo_ctx_launches)
    colo_ctx* temps = nullptr;      // colo_ctx_share_temps: the context whose per-call replay temporaries
                                    // (d_sat, d_satpool, d_tmp of the first pass) this one uses
};

#define COLO_LAUNCHED(ctx) (++(ctx)->launches)

struct colo_mapset {
    int device = 0;
    colo_model m{};
    colo_gpu g{};
    colo_grid grid{};
    colo_mode mode = COLO_CPA;
    uint64_t hedge_step = 0, hedge_max = 0, assumed = 128, hash = 0;
    uint32_t C = 0, I = 0, B = 0, Hc = 0, F = 0;
    uint8_t* d_off = nullptr;   // C*I*B offload codes
    uint8_t* d_hed = nullptr;   // Hc*F hedge bits
    uint32_t* d_tab = nullptr;  // (C+1)*(I+1) trace-fused verdict table (hedge_step == cached_step only)
    uint32_t* d_str = nullptr;  // C+1 stream bits per cached bucket
    uint8_t* d_img = nullptr;   // k_decide_packed's shared-memory image (packed cells, hedge bits, stream bytes)
    uint32_t img_bytes = 0;     // 0: the grid does not take the packed kernel
    bool fast = false;
};

namespace colo {

colo_status set_err(colo_ctx* ctx, colo_status st, const std::string& what);
colo_status cuda_err(colo_ctx* ctx, cudaError_t e, const char* where);
MapView make_view(const colo_mapset* ms);
colo_status check_grid_limits(const colo_grid* g);
colo_status check_model_limits(const colo_model* m);
// correctly rounded (sum * 2^-96) / n from a 192-bit little-endian fixed-point sum
double fixed_mean(const uint64_t sum[3], uint64_t n);
void fixed_add(uint64_t acc[3], const uint64_t v[3]);
// in-place ncclAllReduce on the context's stream (NCCL resolved at run time)
// k_decide_packed's shared-memory image of a map set (sweep-size grids only;
// a no-op otherwise), rebuilt whenever the cells change
colo_status build_pack_image(colo_ctx* ctx, colo_mapset* ms);
colo_status nccl_allreduce_raw(colo_ctx* ctx, void* comm, void* d_buf, size_t count, int dtype, int op);

}  // namespace colo

#define COLO_CK(ctx, call)                                          \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return colo::cuda_err(ctx, e_, #call); \
    } while (0)
