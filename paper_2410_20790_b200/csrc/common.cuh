// common.cuh -- device helpers shared by the sm_100a kernels (internal).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <unordered_map>
#include <algorithm>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.h"

// Checked build (python -m paper_2410_20790_b200.build --checked -> libsparsetem_checked.so,
// -DST_BOUNDS_CHECK): row indices of gathers / scatters against the tensor's
// row count, a trap with the failing condition on a violation.  The pool's
// compute-sanitizer is closed, so this build is the memory-safety check.
#ifdef ST_BOUNDS_CHECK
#include <cstdio>
#define ST_CHECK(cond)                                                                   \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("ST_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                   \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define ST_CHECK(cond) \
    do {               \
    } while (0)
#endif

namespace st {

// Programmatic dependent launch: inside the captured step graph the edges
// between consecutive kernels are programmatic (encoder.cu), so a kernel's
// CTAs may be scheduled while its predecessor drains.  Every kernel calls
// this first: wait until the prerequisite grids have completed and their
// writes are visible (no global access precedes it), then allow our own
// dependents to be scheduled.  Both are no-ops in a normal launch.
__device__ __forceinline__ void st_pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

typedef __nv_bfloat16 bf16;

__device__ __forceinline__ uint32_t lowmask(int t1) { return (1u << t1) - 1u; }

// row index of (pixel bp, diff frame t1+1) in a diff tensor; 0 = zero row
__device__ __forceinline__ int row_of(const DView &v, int64_t bp, int t1) {
    const uint32_t a = __ldg(v.act + bp);
    if (!((a >> t1) & 1u)) return 0;
    return 1 + __ldg(v.pbase + bp) + __popc(__ldg(v.slot + bp) & lowmask(t1));
}

// ---- delta-row storage type T: float (FP32 mode) or bf16 (BF16 mode, R22-BF16)
template <class T> __device__ __forceinline__ float ldr(const T *p);
template <> __device__ __forceinline__ float ldr<float>(const float *p) { return *p; }
template <> __device__ __forceinline__ float ldr<bf16>(const bf16 *p) { return __bfloat162float(*p); }
template <class T> __device__ __forceinline__ void str(T *p, float v);
template <> __device__ __forceinline__ void str<float>(float *p, float v) { *p = v; }
template <> __device__ __forceinline__ void str<bf16>(bf16 *p, float v) { *p = __float2bfloat16_rn(v); }
// the value as it will be stored (the emitted delta)
template <class T> __device__ __forceinline__ float rnd(float v);
template <> __device__ __forceinline__ float rnd<float>(float v) { return v; }
template <> __device__ __forceinline__ float rnd<bf16>(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
// a pair rounded to the stored type (bf16: one cvt.rn.bf16x2 -- RNE per lane)
template <class T> __device__ __forceinline__ float2 rnd2(float2 v);
template <> __device__ __forceinline__ float2 rnd2<float>(float2 v) { return v; }
template <> __device__ __forceinline__ float2 rnd2<bf16>(float2 v) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v.y), "f"(v.x));
    return make_float2(__uint_as_float(r << 16), __uint_as_float(r & 0xFFFF0000u));
}
// RNE bf16 rounding of an fp32 value, kept as fp32 (BF16-mode conv operands)
__device__ __forceinline__ float bf16_round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
// 4 consecutive elements -> float4 (p 4-element aligned)
template <class T> __device__ __forceinline__ float4 ld4(const T *p);
template <> __device__ __forceinline__ float4 ld4<float>(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
template <> __device__ __forceinline__ float4 ld4<bf16>(const bf16 *p) {
    const uint2 u = __ldg(reinterpret_cast<const uint2 *>(p));
    float4 f;
    f.x = __uint_as_float(u.x << 16);
    f.y = __uint_as_float(u.x & 0xFFFF0000u);
    f.z = __uint_as_float(u.y << 16);
    f.w = __uint_as_float(u.y & 0xFFFF0000u);
    return f;
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
// BF16 mode (tolerance parity, R22-BF16): single-precision MUFU exp and
// approximate division -- within a few fp32 ulp of the exact form, far below
// the bf16 rounding of every emitted delta.
// x * 1 / (1 + 2^(-x log2 e)) with the flush-to-zero MUFU forms (ex2.approx.ftz,
// rcp.approx.ftz): five instructions, no denormal range fix-ups (ncu: the
// __fdividef(x, 1 + __expf(-x)) form cost ~12 per channel in the site kernels,
// whose per-row instruction count bounds them)
__device__ __forceinline__ float silu_fast(float x) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return x * r;
}

// ---- packed fp32x2 (FADD2 / FMUL2 / FFMA2, sm_100): each lane of a pair is
// rounded exactly as the scalar operation, so results are bit-identical
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// a - b as fma(b, -1, a): one rounding of the exact difference, the same bits
// as __fsub_rn(a, b) including the signs of zeros
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a); }
__device__ __forceinline__ float2 silu2_fast(float2 x) {
    const float2 t = mul2(x, make_float2(-1.4426950408889634f, -1.4426950408889634f));
    float e0, e1, r0, r1;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(t.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(t.y));
    const float2 d = add2(make_float2(e0, e1), make_float2(1.0f, 1.0f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
    return mul2(x, make_float2(r0, r1));
}

// pointwise non-linearity f of a site (kind fixed at compile time / at run time)
template <int ACT>
__device__ __forceinline__ float actf(float x) {
    return ACT == ACT_RELU ? relu_f(x) : ACT == ACT_SILU ? silu_f(x) : silu_fast(x);
}
// the same on a pair (silu2_fast is silu_fast lane by lane: x * -log2e, 1 + e
// and x * r round like their scalar forms)
template <int ACT>
__device__ __forceinline__ float2 actf2(float2 x) {
    if constexpr (ACT == ACT_SILU_FAST) return silu2_fast(x);
    else return make_float2(actf<ACT>(x.x), actf<ACT>(x.y));
}
__device__ __forceinline__ float act_rt(int kind, float x) {
    return kind == ACT_RELU ? relu_f(x) : kind == ACT_SILU ? silu_f(x) : silu_fast(x);
}

// lanes of this thread's pixel group (G lanes, G a power of two <= 32)
template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        const int lane = threadIdx.x & 31;
        return ((1u << G) - 1u) << (lane & ~(G - 1));
    }
}

template <int G>
__device__ __forceinline__ float gmax(float v, unsigned mask) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(mask, v, o, G));
    return v;
}

inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// grid of a grid-stride kernel: at most one wave of resident CTAs (the
// occupancy calculator's count x SMs), so no partial last wave idles SMs;
// ST_SITE_GRID=old keeps the caller's cap instead
// (the occupancy query runs once per kernel, on the eager first step: no CUDA
// calls of that kind inside a graph capture)
template <class K>
inline int resident_grid(K kernel, int threads, size_t smem, int64_t want, int old_cap) {
    const char *v = getenv("ST_SITE_GRID");
    if (v && v[0] == 'o') return (int)std::max<int64_t>(1, std::min<int64_t>(want, old_cap));
    static int sms = 0;
    static std::unordered_map<const void *, int> per_sm;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    auto it = per_sm.find(reinterpret_cast<const void *>(kernel));
    int per = 0;
    if (it == per_sm.end()) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess) per = 0;
        per_sm[reinterpret_cast<const void *>(kernel)] = per;
    } else {
        per = it->second;
    }
    if (per <= 0) return (int)std::max<int64_t>(1, std::min<int64_t>(want, old_cap));
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per * sms));
}

// host-side dispatch on the row type
#define ST_ROW_DISPATCH(bf, ...)            \
    do {                                    \
        if (bf) {                           \
            typedef ::st::bf16 T;           \
            __VA_ARGS__;                    \
        } else {                            \
            typedef float T;                \
            __VA_ARGS__;                    \
        }                                   \
    } while (0)

}  // namespace st
