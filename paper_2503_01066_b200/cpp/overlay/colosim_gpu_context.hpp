// colosim_gpu_context.hpp -- the process-wide GPU context the include overlay
// (overlay/colosim/maps.hpp, overlay/colosim/engine.hpp) runs on.
#pragma once

#include <cstdlib>

#include "colosim_gpu.hpp"

namespace colosim_gpu {

/// One colo_ctx per process, on COLOSIM_GPU_DEVICE (default 0), created on
/// first use.  The reference's driver is single-threaded, and so is this.
inline Context& process_context() {
    static Context ctx([] {
        const char* d = std::getenv("COLOSIM_GPU_DEVICE");
        return d ? std::atoi(d) : 0;
    }());
    return ctx;
}

}  // namespace colosim_gpu
