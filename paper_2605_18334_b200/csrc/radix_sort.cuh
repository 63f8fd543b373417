// radix_sort.cuh -- helpers shared by the radix sorts (depth_sort.cuh: the
// cooperative LSD sort; onesweep.cuh: the decoupled look-back sort;
// bucket_sort.cuh: the bucket depth sort) and the counting scatter: the
// 256-byte workspace carve-up and the lane mask used by warp-level ranking.
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
