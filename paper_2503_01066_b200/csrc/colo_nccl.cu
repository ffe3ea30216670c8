// colo_nccl.cu -- the one cross-GPU exchange: an NCCL
// all-reduce of statistics over a caller-owned communicator.
//
// NCCL is resolved at run time (dlsym in the process, else dlopen
// libnccl.so.2), so the library has no link-time NCCL dependency and uses
// the same NCCL as the caller that created the communicator (a C++ host
// with ncclCommInitRank, or a framework that already loaded one).
#include <dlfcn.h>

#include <cstdint>

#include "colo_internal.h"

using namespace colo;

namespace {

using AllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
using ErrStrFn = const char* (*)(int);

AllReduceFn nccl_allreduce_fn() {
    static AllReduceFn f = [] {
        void* sym = dlsym(RTLD_DEFAULT, "ncclAllReduce");
        if (!sym) {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (h) sym = dlsym(h, "ncclAllReduce");
        }
        return reinterpret_cast<AllReduceFn>(sym);
    }();
    return f;
}

}  // namespace

namespace colo {

colo_status nccl_allreduce_raw(colo_ctx* ctx, void* comm, void* d_buf, size_t count, int dtype, int op) {
    AllReduceFn f = nccl_allreduce_fn();
    if (!f) return set_err(ctx, COLO_ECUDA, "NCCL not found (ncclAllReduce / libnccl.so.2)");
    const int r = f(d_buf, d_buf, count, dtype, op, comm, ctx->stream);
    if (r != 0) {
        auto es = reinterpret_cast<ErrStrFn>(dlsym(RTLD_DEFAULT, "ncclGetErrorString"));
        return set_err(ctx, COLO_ECUDA, std::string("ncclAllReduce: ") + (es ? es(r) : std::to_string(r)));
    }
    return COLO_OK;
}

}  // namespace colo

extern "C" colo_status colo_stats_allreduce(colo_ctx* ctx, void* nccl_comm, uint64_t* d_buf, size_t count) {
    if (!ctx || !nccl_comm || (count && !d_buf)) return COLO_EINVAL;
    if (count == 0) return COLO_OK;
    COLO_CK(ctx, cudaSetDevice(ctx->device));
    return nccl_allreduce_raw(ctx, nccl_comm, d_buf, count, /*ncclUint64*/ 5, /*ncclSum*/ 0);
}
