// rowio.cuh -- vectorized per-lane access to a pixel's channel row (internal).
//
// Site kernels own one pixel per group of G lanes; lane l holds the CPL
// consecutive channels [l*CPL, (l+1)*CPL) ("blocked" mapping), so a row is
// moved with the widest aligned vector per lane (16 B for 8 bf16 / 4 fp32).
// When C != G*CPL the tail lanes fall back to guarded scalar access.
#pragma once
#include "common.cuh"

namespace st {

template <class T, int CPL>
struct RowIO {
    // full row chunk of this lane: p points at channel l*CPL
    static __device__ __forceinline__ void load(const T *p, float (&v)[CPL]) {
        if constexpr (sizeof(T) == 2 && CPL % 8 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 8) {
                const uint4 u = *reinterpret_cast<const uint4 *>(p + i);
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    v[i + 2 * k] = __uint_as_float(w[k] << 16);
                    v[i + 2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
                }
            }
        } else if constexpr (sizeof(T) == 2 && CPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 4) {
                const uint2 u = *reinterpret_cast<const uint2 *>(p + i);
                v[i] = __uint_as_float(u.x << 16);
                v[i + 1] = __uint_as_float(u.x & 0xFFFF0000u);
                v[i + 2] = __uint_as_float(u.y << 16);
                v[i + 3] = __uint_as_float(u.y & 0xFFFF0000u);
            }
        } else if constexpr (sizeof(T) == 2 && CPL % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 2) {
                const uint32_t u = *reinterpret_cast<const uint32_t *>(p + i);
                v[i] = __uint_as_float(u << 16);
                v[i + 1] = __uint_as_float(u & 0xFFFF0000u);
            }
        } else if constexpr (sizeof(T) == 4 && CPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 4) {
                const float4 f = *reinterpret_cast<const float4 *>(p + i);
                v[i] = f.x; v[i + 1] = f.y; v[i + 2] = f.z; v[i + 3] = f.w;
            }
        } else if constexpr (sizeof(T) == 4 && CPL % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 2) {
                const float2 f = *reinterpret_cast<const float2 *>(p + i);
                v[i] = f.x; v[i + 1] = f.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < CPL; i++) v[i] = ldr<T>(p + i);
        }
    }
    static __device__ __forceinline__ void store(T *p, const float (&v)[CPL]) {
        if constexpr (sizeof(T) == 2 && CPL % 8 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 8) {
                uint4 u;
                u.x = pack(v[i], v[i + 1]);
                u.y = pack(v[i + 2], v[i + 3]);
                u.z = pack(v[i + 4], v[i + 5]);
                u.w = pack(v[i + 6], v[i + 7]);
                *reinterpret_cast<uint4 *>(p + i) = u;
            }
        } else if constexpr (sizeof(T) == 2 && CPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 4) {
                uint2 u;
                u.x = pack(v[i], v[i + 1]);
                u.y = pack(v[i + 2], v[i + 3]);
                *reinterpret_cast<uint2 *>(p + i) = u;
            }
        } else if constexpr (sizeof(T) == 2 && CPL % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 2) *reinterpret_cast<uint32_t *>(p + i) = pack(v[i], v[i + 1]);
        } else if constexpr (sizeof(T) == 4 && CPL % 4 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 4)
                *reinterpret_cast<float4 *>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else if constexpr (sizeof(T) == 4 && CPL % 2 == 0) {
#pragma unroll
            for (int i = 0; i < CPL; i += 2) *reinterpret_cast<float2 *>(p + i) = make_float2(v[i], v[i + 1]);
        } else {
#pragma unroll
            for (int i = 0; i < CPL; i++) str<T>(p + i, v[i]);
        }
    }
    // guarded variants (tail lanes when C != G*CPL); c0 = l*CPL
    static __device__ __forceinline__ void load_g(const T *row, int c0, int C, float (&v)[CPL]) {
#pragma unroll
        for (int i = 0; i < CPL; i++) v[i] = c0 + i < C ? ldr<T>(row + c0 + i) : 0.0f;
    }
    static __device__ __forceinline__ void store_g(T *row, int c0, int C, const float (&v)[CPL]) {
#pragma unroll
        for (int i = 0; i < CPL; i++)
            if (c0 + i < C) str<T>(row + c0 + i, v[i]);
    }
    static __device__ __forceinline__ uint32_t pack(float lo, float hi) {
        uint32_t r;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
        return r;
    }
};

// row chunk of this lane, vectorized when the lane's chunk lies fully inside C
template <class T, int CPL>
__device__ __forceinline__ void row_load(const T *row, int c0, int C, bool full, float (&v)[CPL]) {
    if (full) RowIO<T, CPL>::load(row + c0, v);
    else RowIO<T, CPL>::load_g(row, c0, C, v);
}
template <class T, int CPL>
__device__ __forceinline__ void row_store(T *row, int c0, int C, bool full, const float (&v)[CPL]) {
    if (full) RowIO<T, CPL>::store(row + c0, v);
    else RowIO<T, CPL>::store_g(row, c0, C, v);
}

}  // namespace st
