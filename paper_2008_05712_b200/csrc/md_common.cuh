// md_common.cuh -- float64 helpers shared by the MD kernels (md.cu, md_loop.cu).
#pragma once
#include <cuda_runtime.h>

namespace gc {

// numpy floor_divide / remainder for floats (npy_divmod)
__device__ __forceinline__ double np_floordiv(double a, double b)
{
    const double mod = fmod(a, b);
    double div = __ddiv_rn(__dsub_rn(a, mod), b);
    if (mod != 0.0 && ((b < 0) != (mod < 0))) div = __dsub_rn(div, 1.0);
    double fd;
    if (div != 0.0) {
        fd = floor(div);
        if (__dsub_rn(div, fd) > 0.5) fd = __dadd_rn(fd, 1.0);
    } else {
        fd = copysign(0.0, __ddiv_rn(a, b));
    }
    return fd;
}

__device__ __forceinline__ double np_remainder(double a, double b)
{
    double mod = fmod(a, b);
    if (mod != 0.0) {
        if ((b < 0) != (mod < 0)) mod = __dadd_rn(mod, b);
    } else {
        mod = copysign(0.0, b);
    }
    return mod;
}

}  // namespace gc
