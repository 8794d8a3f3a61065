// common.cuh -- device helpers shared by the sm_100a kernels (internal).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace st {

__device__ __forceinline__ uint32_t lowmask(int t1) { return (1u << t1) - 1u; }

// row index of (pixel bp, diff frame t1+1) in a diff tensor; 0 = zero row
__device__ __forceinline__ int row_of(const DView &v, int64_t bp, int t1) {
    const uint32_t a = __ldg(v.act + bp);
    if (!((a >> t1) & 1u)) return 0;
    return 1 + __ldg(v.pbase + bp) + __popc(__ldg(v.slot + bp) & lowmask(t1));
}

template <int G>
__device__ __forceinline__ float group_max(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o, G));
    return v;
}

// exact scalar functions, identical definitions to the oracle's (R10)
__device__ __forceinline__ float relu_f(float x) { return x > 0.0f ? x : 0.0f; }
__device__ __forceinline__ float exp_r(float v) { return (float)exp((double)v); }
__device__ __forceinline__ float silu_f(float x) { return __fdiv_rn(x, __fadd_rn(1.0f, exp_r(-x))); }
__device__ __forceinline__ float sigm_f(float x) { return __fdiv_rn(1.0f, __fadd_rn(1.0f, exp_r(-x))); }

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace st
