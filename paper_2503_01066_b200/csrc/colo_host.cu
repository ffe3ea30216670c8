// colo_host.cu -- host-side pieces of the C-ABI: context, validation, profile
// hash, trace synthesis (bit-exact generate_trace), histogram selection.
// Reference paths are relative to /root/reference/proj/.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "colo_internal.h"

namespace colo {

colo_status set_err(colo_ctx* ctx, colo_status st, const std::string& what) {
    if (ctx) ctx->err = what;
    return st;
}

colo_status cuda_err(colo_ctx* ctx, cudaError_t e, const char* where) {
    return set_err(ctx, COLO_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// validate_grid (maps.hpp:197-208) plus this build's 32-bit index limits.
colo_status check_grid_limits(const colo_grid* g) {
    colo_status st = colo_validate_grid(g);
    if (st != COLO_OK) return st;
    const uint64_t steps[3] = {g->cached_step, g->incoming_step, g->batch_step};
    const uint64_t maxs[3] = {g->max_cached, g->max_incoming, g->max_batch};
    for (int i = 0; i < 3; ++i)
        if (steps[i] > (1ull << 31) || maxs[i] + steps[i] > (1ull << 32)) return COLO_EINVAL;
    return COLO_OK;
}

colo_status check_model_limits(const colo_model* m) {
    return m->num_layers <= kMaxLayers ? COLO_OK : COLO_EINVAL;
}

MapView make_view(const colo_mapset* ms) {
    MapView v{};
    v.off = ms->d_off;
    v.hed = ms->d_hed;
    v.tab = ms->d_tab;
    v.str = ms->d_str;
    v.max_c = static_cast<uint32_t>(ms->grid.max_cached);
    v.max_i = static_cast<uint32_t>(ms->grid.max_incoming);
    v.max_b = static_cast<uint32_t>(ms->grid.max_batch);
    v.fc = make_fastdiv(static_cast<uint32_t>(ms->grid.cached_step));
    v.fi = make_fastdiv(static_cast<uint32_t>(ms->grid.incoming_step));
    v.fb = make_fastdiv(static_cast<uint32_t>(ms->grid.batch_step));
    v.fh = make_fastdiv(static_cast<uint32_t>(ms->hedge_step));
    v.C = ms->C;
    v.I = ms->I;
    v.B = ms->B;
    v.hmax = static_cast<uint32_t>(ms->hedge_max);
    v.hsame = ms->fast ? 1u : 0u;
    v.L = static_cast<uint32_t>(ms->m.num_layers);
    v.cpa = ms->mode == COLO_CPA ? 1u : 0u;
    v.off_bytes = ms->C * ms->I * ms->B;
    v.hed_bytes = ms->Hc * ms->F;
    return v;
}

void fixed_add(uint64_t acc[3], const uint64_t v[3]) {
    unsigned __int128 c = 0;
    for (int i = 0; i < 3; ++i) {
        c += static_cast<unsigned __int128>(acc[i]) + v[i];
        acc[i] = static_cast<uint64_t>(c);
        c >>= 64;
    }
}

// (S * 2^-96) / n, S a 192-bit little-endian integer: S is rounded to double
// once (top 64 bits with a sticky bit, then the RN u64->f64 conversion), the
// division rounds once more: within one ulp of the exact mean.
double fixed_mean(const uint64_t sum[3], uint64_t n) {
    if (n == 0) return std::nan("");
    int top = -1;
    for (int i = 2; i >= 0 && top < 0; --i)
        if (sum[i]) top = i * 64 + 63 - __builtin_clzll(sum[i]);
    if (top < 0) return 0.0;
    double s;
    if (top < 64) {
        s = static_cast<double>(sum[0]);
        return std::ldexp(s, -96) / static_cast<double>(n);
    }
    int shift = top - 63;  // bring bits [top..shift] into a u64
    uint64_t w = 0;
    bool sticky = false;
    for (int b = 0; b < 192; ++b) {
        uint64_t bit = (sum[b / 64] >> (b % 64)) & 1ull;
        if (b < shift) {
            sticky |= bit != 0;
        } else if (b <= top) {
            w |= bit << (b - shift);
        }
    }
    if (sticky) w |= 1ull;
    s = static_cast<double>(w);
    return std::ldexp(s, shift - 96) / static_cast<double>(n);
}

}  // namespace colo

using namespace colo;

extern "C" {

int colo_abi_version(void) { return COLO_ABI_VERSION; }

// profiles.hpp:37-57, 104-108, 129-134
colo_status colo_validate_profile_pair(const colo_model* m, const colo_gpu* g) {
    if (!m || !g) return COLO_EINVAL;
    if (m->num_layers == 0 || m->kv_bytes_per_token == 0 || m->act_bytes_per_token_per_layer == 0 ||
        m->weights_bytes == 0)
        return COLO_EVALIDATION;
    if (!(m->prefill_coef_linear > 0) || !(m->prefill_coef_quad > 0) || !(m->decode_coef_const > 0) ||
        !(m->decode_coef_context > 0) || !(m->backward_to_forward_ratio > 0))
        return COLO_EVALIDATION;
    if (m->record_prefill_multiplier < 1.0 || m->record_decode_multiplier < 1.0) return COLO_EVALIDATION;
    if (m->workspace_factor < 0.0) return COLO_EVALIDATION;
    if (g->capacity_bytes == 0 || g->h2d_bandwidth == 0 || g->d2h_bandwidth == 0) return COLO_EVALIDATION;
    if (m->weights_bytes + g->runtime_reserve_bytes >= g->capacity_bytes) return COLO_EVALIDATION;
    return COLO_OK;
}

// profiles.hpp:137-152: FNV-1a over the canonical '|'-joined field string;
// ostream precision(17) formats doubles exactly like printf("%.17g").
uint64_t colo_profile_hash(const colo_model* m, const colo_gpu* g) {
    char buf[1024];
    int len = std::snprintf(
        buf, sizeof buf, "%llu|%llu|%llu|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%.17g|%llu|%llu|%llu|%llu|%llu",
        (unsigned long long)m->num_layers, (unsigned long long)m->kv_bytes_per_token,
        (unsigned long long)m->act_bytes_per_token_per_layer, m->prefill_coef_linear, m->prefill_coef_quad,
        m->decode_coef_const, m->decode_coef_context, m->backward_to_forward_ratio, m->record_prefill_multiplier,
        m->record_decode_multiplier, m->workspace_factor, (unsigned long long)m->weights_bytes,
        (unsigned long long)g->capacity_bytes, (unsigned long long)g->h2d_bandwidth,
        (unsigned long long)g->d2h_bandwidth, (unsigned long long)g->runtime_reserve_bytes);
    uint64_t h = 14695981039346656037ull;
    for (int i = 0; i < len; ++i) {
        h ^= static_cast<unsigned char>(buf[i]);
        h *= 1099511628211ull;
    }
    return h;
}

// maps.hpp:197-208
colo_status colo_validate_grid(const colo_grid* s) {
    if (!s) return COLO_EINVAL;
    if (s->cached_step == 0 || s->incoming_step == 0 || s->batch_step == 0) return COLO_EVALIDATION;
    if (s->max_cached == 0 || s->max_incoming == 0 || s->max_batch == 0) return COLO_EVALIDATION;
    if (s->max_cached % s->cached_step || s->max_incoming % s->incoming_step || s->max_batch % s->batch_step)
        return COLO_EVALIDATION;
    return COLO_OK;
}

colo_status colo_ctx_create(int device, colo_ctx** out) {
    if (!out) return COLO_EINVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return COLO_ECUDA;
    colo_ctx* ctx = new colo_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_flag, sizeof(int) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_counters, sizeof(uint64_t) * COLO_NCOUNTERS);
    if (e != cudaSuccess) {
        colo_ctx_destroy(ctx);
        return COLO_ECUDA;
    }
    ctx->stream = ctx->own;
    *out = ctx;
    return COLO_OK;
}

void colo_ctx_destroy(colo_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->own) cudaStreamSynchronize(ctx->own);
    if (ctx->aux) cudaStreamSynchronize(ctx->aux);
    if (ctx->d_flag) cudaFree(ctx->d_flag);
    if (ctx->d_counters) cudaFree(ctx->d_counters);
    if (ctx->d_pipe) cudaFree(ctx->d_pipe);
    if (ctx->d_rscratch) cudaFree(ctx->d_rscratch);
    if (ctx->d_sat) cudaFree(ctx->d_sat);
    if (ctx->d_satpool) cudaFree(ctx->d_satpool);
    if (ctx->d_seg) cudaFree(ctx->d_seg);
    if (ctx->d_seglog) cudaFree(ctx->d_seglog);
    if (ctx->d_tmp) cudaFree(ctx->d_tmp);
    if (ctx->d_bmeta) cudaFree(ctx->d_bmeta);
    if (ctx->d_dtab) cudaFree(ctx->d_dtab);
    if (ctx->d_htab) cudaFree(ctx->d_htab);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->aux) cudaStreamDestroy(ctx->aux);
    delete ctx;
}

colo_status colo_ctx_release_scratch(colo_ctx* ctx) {
    if (!ctx) return COLO_EINVAL;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    if (ctx->aux) COLO_CK(ctx, cudaStreamSynchronize(ctx->aux));
    auto drop = [](void*& p, size_t& n) {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    };
    drop(ctx->d_pipe, ctx->pipe_bytes);
    drop(ctx->d_rscratch, ctx->rscratch_bytes);
    drop(ctx->d_sat, ctx->sat_bytes);
    drop(ctx->d_satpool, ctx->satpool_bytes);
    drop(ctx->d_seg, ctx->seg_bytes);
    drop(ctx->d_seglog, ctx->seglog_bytes);
    drop(ctx->d_tmp, ctx->tmp_bytes);
    drop(ctx->d_bmeta, ctx->bmeta_bytes);
    drop(ctx->d_dtab, ctx->dtab_bytes);
    ctx->rs_valid = false;
    ctx->bmeta_valid = false;
    return COLO_OK;
}

colo_status colo_ctx_share_temps(colo_ctx* ctx, colo_ctx* owner) {
    if (!ctx || (owner && owner->device != ctx->device)) return COLO_EINVAL;
    ctx->temps = (owner == ctx) ? nullptr : owner;
    return COLO_OK;
}

colo_status colo_ctx_set_stream(colo_ctx* ctx, void* s) {
    if (!ctx) return COLO_EINVAL;
    ctx->stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
    return COLO_OK;
}

void* colo_ctx_stream(colo_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

colo_status colo_sync(colo_ctx* ctx) {
    if (!ctx) return COLO_EINVAL;
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

const char* colo_last_error(const colo_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int colo_ctx_sm_count(const colo_ctx* ctx) { return ctx ? ctx->sm_count : 0; }

uint64_t colo_ctx_launches(const colo_ctx* ctx) { return ctx ? ctx->launches : 0; }

colo_status colo_dev_alloc(colo_ctx* ctx, size_t bytes, void** d_ptr) {
    if (!ctx || !d_ptr) return COLO_EINVAL;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    COLO_CK(ctx, cudaMalloc(d_ptr, bytes ? bytes : 1));
    return COLO_OK;
}

colo_status colo_dev_free(colo_ctx* ctx, void* p) {
    if (!ctx) return COLO_EINVAL;
    COLO_CK(ctx, cudaFree(p));
    return COLO_OK;
}

colo_status colo_memcpy_h2d(colo_ctx* ctx, void* d, const void* h, size_t bytes) {
    if (!ctx) return COLO_EINVAL;
    COLO_CK(ctx, cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

colo_status colo_memcpy_d2h(colo_ctx* ctx, void* h, const void* d, size_t bytes) {
    if (!ctx) return COLO_EINVAL;
    COLO_CK(ctx, cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    COLO_CK(ctx, cudaStreamSynchronize(ctx->stream));
    return COLO_OK;
}

colo_status colo_hist_select(const uint64_t* h, size_t nbins, uint64_t rank, uint32_t* bin, uint64_t* rank_in) {
    if (!h || !bin || !rank_in || rank == 0) return COLO_EINVAL;
    uint64_t cum = 0;
    for (size_t b = 0; b < nbins; ++b) {
        if (cum + h[b] >= rank) {
            *bin = static_cast<uint32_t>(b);
            *rank_in = rank - cum;
            return COLO_OK;
        }
        cum += h[b];
    }
    return COLO_EINVAL;
}

// metrics.hpp:48-53
uint64_t colo_nearest_rank_index(double q, uint64_t n) {
    uint64_t rank = static_cast<uint64_t>(std::ceil(q * static_cast<double>(n)));
    return rank == 0 ? 1 : rank;
}

}  // extern "C"

// ------------------------------------------------------------ trace synthesis
namespace {

bool dist_valid(const colo_dist* d) {
    if (!d) return true;
    switch (d->kind) {
        case 0: return d->fixed_value >= 0;
        case 1: return d->lo <= d->hi;
        case 2: {
            if (d->nbins == 0 || !d->bin_values || !d->bin_probs) return false;
            double sum = 0;
            for (size_t i = 0; i < d->nbins; ++i) {
                if (d->bin_probs[i] < 0) return false;
                sum += d->bin_probs[i];
            }
            return std::abs(sum - 1.0) <= 1e-9;  // workload.hpp:82
        }
        default: return false;
    }
}

// workload.hpp:25
double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// workload.hpp:90-107
double sample_raw(const colo_dist* d, std::mt19937_64& g) {
    switch (d->kind) {
        case 0: return d->fixed_value;
        case 1: return d->lo + (d->hi - d->lo) * uniform01(g);
        default: {
            double u = uniform01(g), acc = 0;
            for (size_t i = 0; i < d->nbins; ++i) {
                acc += d->bin_probs[i];
                if (u < acc) return d->bin_values[i];
            }
            return d->bin_values[d->nbins - 1];
        }
    }
}

}  // namespace

extern "C" int64_t colo_generate_trace(double qps, double duration, const colo_dist* lengths,
                                       const colo_dist* label_delay, uint64_t seed, double* arrival, uint32_t* prompt,
                                       uint32_t* output, double* label_out, size_t cap) {
    if (!(qps > 0) || !(duration > 0) || !lengths || !dist_valid(lengths) || !dist_valid(label_delay)) return -2;
    std::mt19937_64 gen(seed);
    double t = 0;
    size_t n = 0;
    for (;;) {
        t += -std::log(1.0 - uniform01(gen)) / qps;  // workload.hpp:28
        if (t > duration) break;
        if (n >= cap) return -1;
        double raw = sample_raw(lengths, gen);
        auto tok = static_cast<uint64_t>(std::llround(std::max(raw, 1.0)));  // workload.hpp:111-116
        if (lengths->min_tokens && tok < lengths->min_tokens) tok = lengths->min_tokens;
        arrival[n] = t;
        prompt[n] = static_cast<uint32_t>(tok);
        output[n] = 128;  // workload.hpp:214
        double ld = -1.0;  // nullopt
        if (label_delay) ld = std::max(0.0, sample_raw(label_delay, gen));  // sample_seconds, workload.hpp:118-120
        if (label_out) label_out[n] = ld;
        ++n;
    }
    return static_cast<int64_t>(n);
}

// Trace::content_hash, workload.hpp:140-161
extern "C" uint64_t colo_trace_hash(const uint64_t* query_id, const double* arrival, const uint32_t* prompt,
                                    const uint32_t* output, const double* label_delay, size_t n) {
    uint64_t h = 14695981039346656037ull;
    auto mix = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (i * 8)) & 0xff;
            h *= 1099511628211ull;
        }
    };
    for (size_t i = 0; i < n; ++i) {
        mix(query_id ? query_id[i] : static_cast<uint64_t>(i));
        uint64_t bits;
        std::memcpy(&bits, &arrival[i], 8);
        mix(bits);
        mix(prompt[i]);
        mix(output[i]);
        double d = label_delay ? label_delay[i] : -1.0;
        if (!(d >= 0.0)) d = -1.0;
        std::memcpy(&bits, &d, 8);
        mix(bits);
    }
    return h;
}
