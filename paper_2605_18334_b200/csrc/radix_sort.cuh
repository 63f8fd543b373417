// radix_sort.cuh -- small helpers shared by the binning kernels (the depth
// sort itself lives in depth_sort.cuh).
#pragma once

#include "ssg_common.cuh"

namespace ssg {
namespace radix {


inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace radix
}  // namespace ssg
