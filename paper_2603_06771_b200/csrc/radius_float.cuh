// radius_float.cuh -- packed FP32 (f32x2) helpers shared by the filtered search kernels
// (radius_pt.cuh, radius_struct.cu, knn_float.cuh) and the warp geometry of the exact FP64
// fallback kernels.  sub / mul / fma.rn.f32x2 compile to FADD2 / FMUL2 / FFMA2 on sm_100a.
#pragma once

#include "search_common.cuh"

namespace lo {

__device__ __forceinline__ u64 pack2(float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(u64 v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ u64 fsub2(u64 a, u64 b) {
    u64 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b) {
    u64 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

constexpr int kRadiusWarps = 4;
constexpr int kRadiusThreads = 32 * kRadiusWarps;

}  // namespace lo
