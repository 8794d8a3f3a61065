// kernels_site.cu -- non-linear correction + truncation sites, residual joins
// and Accumulation on sm_100a.
//
// Non-linear correction (Eq.(3), reading R7): per
// touched pixel, sequentially over diff frames with x_acc / y_acc held in
// registers (the SparseBatch "N" order: the state is born from the
// reference frame's x0 and dies with the kernel -- no per-layer cache is
// kept in HBM):
//     x_acc += Delta_t;  c = f(x_acc) - y_acc;
//     emit iff max_c |c| > theta (pixel granularity, R1/R2);
//     e = c as stored (fp32, or bf16-rounded in BF16 mode); y_acc += e.
// A pixel is owned by a group of G lanes (G = 32 for C >= 32, else the next
// power of two >= C); lane l holds channels [l*CPL, (l+1)*CPL) and moves
// them with 16-byte vectors (rowio.cuh); the channel max is a group shuffle
// reduction.  The frame loop is serial in its arithmetic but not in its
// loads: rows of the next P active frames are fetched together (P = frames
// prefetched per batch, sized so ~16 values per lane are in flight), which
// turns a chain of dependent DRAM round trips into batches.  Emitted rows
// are written in the input's slot layout (in place), so no compaction pass
// follows a site.  Delta rows are of type T (fp32 / bf16).
#include <math_constants.h>

#include "rowio.cuh"

namespace st {

// frames whose rows are fetched per batch (~16 prefetched values per lane:
// deeper batches cost more registers than they save in latency -- measured)
constexpr int prefetch_depth(int cpl) { return cpl <= 2 ? 8 : cpl <= 4 ? 4 : cpl <= 8 ? 2 : 1; }

// ---------------------------------------------------------------- dense ops
__device__ __forceinline__ void put_bf(void *ybf, int64_t i, float v) {
    if (ybf) static_cast<bf16 *>(ybf)[i] = __float2bfloat16_rn(v);
}

template <int ACT>
__global__ void k_dense_act(const float *__restrict__ x, float *__restrict__ y, int64_t n, void *ybf) {
    st_pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = actf<ACT>(x[i]);
        y[i] = v;
        put_bf(ybf, i, v);
    }
}

void launch_dense_act(const float *x, float *y, int64_t n, int act, void *ybf, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(cdiv(n, 256), 148 * 16);
    if (grid <= 0) return;
    if (act == ACT_RELU) k_dense_act<ACT_RELU><<<grid, 256, 0, s>>>(x, y, n, ybf);
    else if (act == ACT_SILU) k_dense_act<ACT_SILU><<<grid, 256, 0, s>>>(x, y, n, ybf);
    else k_dense_act<ACT_SILU_FAST><<<grid, 256, 0, s>>>(x, y, n, ybf);
}

// relu_in: x is the pre-activation of a ReLU whose only consumer is this pool
// (fused pair): y = relu(window max) == window max of relu(x) exactly (ReLU is
// monotone, max is exact), so the ReLU's dense output is never materialised
__global__ void k_dense_maxpool(const float *__restrict__ x, float *__restrict__ y, int B, Geo g, void *ybf,
                                bool relu_in) {
    st_pdl_enter();
    const int No = g.Hout * g.Wout;
    const int64_t n = (int64_t)B * No * g.Cin;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.Cin);
        const int64_t bq = i / g.Cin;
        const int b = (int)(bq / No), q = (int)(bq % No);
        const int oy = q / g.Wout, ox = q % g.Wout;
        float m = -CUDART_INF_F;
        for (int dy = 0; dy < g.kh; dy++) {
            const int iy = oy * g.sh - g.ph + dy;
            if (iy < 0 || iy >= g.Hin) continue;
            for (int dx = 0; dx < g.kw; dx++) {
                const int ix = ox * g.sw - g.pw + dx;
                if (ix < 0 || ix >= g.Win) continue;
                const float v = __ldg(x + (((int64_t)b * g.Hin + iy) * g.Win + ix) * g.Cin + c);
                m = v > m ? v : m;
            }
        }
        if (relu_in) m = relu_f(m);
        y[i] = m;
        put_bf(ybf, i, m);
    }
}

// C % 4 == 0: one thread per (output pixel, 4 channels), float4 window loads,
// 32-bit index math (the scalar kernel above spends most of its time in 64-bit
// divisions); the same max / relu per element
__global__ void k_dense_maxpool4(const float *__restrict__ x, float *__restrict__ y, int B, Geo g, void *ybf,
                                 bool relu_in) {
    st_pdl_enter();
    const int No = g.Hout * g.Wout, C4 = g.Cin >> 2;
    const int n = B * No * C4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int c4 = i % C4, bq = i / C4;
        const int b = bq / No, q = bq - b * No;
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        float4 m = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
        for (int dy = 0; dy < g.kh; dy++) {
            const int iy = oy * g.sh - g.ph + dy;
            if (iy < 0 || iy >= g.Hin) continue;
            for (int dx = 0; dx < g.kw; dx++) {
                const int ix = ox * g.sw - g.pw + dx;
                if (ix < 0 || ix >= g.Win) continue;
                const float4 v =
                    __ldg(reinterpret_cast<const float4 *>(x + ((int64_t)(b * g.Hin + iy) * g.Win + ix) * g.Cin) + c4);
                m.x = v.x > m.x ? v.x : m.x;
                m.y = v.y > m.y ? v.y : m.y;
                m.z = v.z > m.z ? v.z : m.z;
                m.w = v.w > m.w ? v.w : m.w;
            }
        }
        if (relu_in) {
            m.x = relu_f(m.x);
            m.y = relu_f(m.y);
            m.z = relu_f(m.z);
            m.w = relu_f(m.w);
        }
        reinterpret_cast<float4 *>(y)[i] = m;
        if (ybf) {
            uint2 u;
            u.x = RowIO<bf16, 2>::pack(m.x, m.y);
            u.y = RowIO<bf16, 2>::pack(m.z, m.w);
            reinterpret_cast<uint2 *>(ybf)[i] = u;
        }
    }
}

void launch_dense_maxpool(const float *x, float *y, int B, const Geo &g, void *ybf, cudaStream_t s, bool relu_in) {
    const int64_t n = (int64_t)B * g.Hout * g.Wout * g.Cin;
    if (g.Cin % 4 == 0 && n < (int64_t)1 << 31) {
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n / 4, 256), 148 * 16));
        k_dense_maxpool4<<<grid, 256, 0, s>>>(x, y, B, g, ybf, relu_in);
        return;
    }
    const int grid = (int)std::min<int64_t>(cdiv(n, 256), 148 * 16);
    if (grid > 0) k_dense_maxpool<<<grid, 256, 0, s>>>(x, y, B, g, ybf, relu_in);
}

__global__ void k_dense_add(const float *__restrict__ a, const float *__restrict__ b, float *__restrict__ y, int64_t n,
                            void *ybf) {
    st_pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float v = __fadd_rn(a[i], b[i]);
        y[i] = v;
        put_bf(ybf, i, v);
    }
}

void launch_dense_add(const float *a, const float *b, float *y, int64_t n, void *ybf, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(cdiv(n, 256), 148 * 16);
    if (grid > 0) k_dense_add<<<grid, 256, 0, s>>>(a, b, y, n, ybf);
}

// bf16 shadow of a dense activation produced by another kernel (4 per thread)
__global__ void k_to_bf16(const float *__restrict__ x, bf16 *__restrict__ y, int64_t n) {
    st_pdl_enter();
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < n;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
        if (i + 4 <= n) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(x + i));
            uint2 u;
            u.x = RowIO<bf16, 2>::pack(v.x, v.y);
            u.y = RowIO<bf16, 2>::pack(v.z, v.w);
            *reinterpret_cast<uint2 *>(y + i) = u;
        } else {
            for (int64_t j = i; j < n; j++) y[j] = __float2bfloat16_rn(x[j]);
        }
    }
}

void launch_to_bf16(const float *x, void *ybf, int64_t n, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(cdiv(n, 1024), 148 * 16);
    if (grid > 0) k_to_bf16<<<grid, 256, 0, s>>>(x, static_cast<bf16 *>(ybf), n);
}

// ------------------------------------------------------- pointwise site
template <int G, int CPL, int ACT, class T>
__global__ void __launch_bounds__(256) k_site_pw(DView in, const float *__restrict__ x0, int64_t BN, int C,
                                                 const float *__restrict__ theta_p, uint32_t *__restrict__ out_act,
                                                 T *out_rows, SiteState sst, bool zero_gaps) {
    st_pdl_enter();
    const float theta = __ldg(theta_p);
    constexpr int P = prefetch_depth(CPL);
    const int lane = threadIdx.x & (G - 1);
    const int c0 = lane * CPL;
    const bool full = (C % 8 == 0) && (c0 + CPL <= C);
    const unsigned mask = group_mask<G>();
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const T *rows = static_cast<const T *>(in.rows);
    // software pipeline over this group's pixels: while pixel k runs, the
    // frame word of pixel k+2 and the metadata + x0 of pixel k+1 are in flight
    int64_t bp = grp;
    uint32_t a_nx = bp < BN ? __ldg(in.act + bp) : 0u;                      // pixel k
    int base_nx = 0;
    uint32_t sl_nx = 0;
    float x_nx[CPL];
    if (a_nx) {
        base_nx = 1 + __ldg(in.pbase + bp);
        sl_nx = __ldg(in.slot + bp);
        row_load<float, CPL>(x0 + bp * C, c0, C, full, x_nx);
    }
    uint32_t a_nn = bp + ngrp < BN ? __ldg(in.act + bp + ngrp) : 0u;         // pixel k+1
    for (; bp < BN; bp += ngrp) {
        uint32_t a = a_nx;
        const int base = base_nx;
        const uint32_t sl = sl_nx;
        float xa[CPL], ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) xa[i] = x_nx[i];
        // prefetch: metadata + x0 of pixel k+1, frame word of pixel k+2
        const int64_t b1 = bp + ngrp;
        a_nx = a_nn;
        if (a_nx) {
            base_nx = 1 + __ldg(in.pbase + b1);
            sl_nx = __ldg(in.slot + b1);
            row_load<float, CPL>(x0 + b1 * C, c0, C, full, x_nx);
        }
        a_nn = b1 + ngrp < BN ? __ldg(in.act + b1 + ngrp) : 0u;
        if (!a) {
            if (lane == 0) out_act[bp] = 0;
            continue;
        }
        if (sst.y_init)   // streaming continuation: the saved y_acc
            row_load<float, CPL>(sst.y_init + bp * C, c0, C, full, ya);
        else
#pragma unroll
            for (int i = 0; i < CPL; i++) ya[i] = actf<ACT>(xa[i]);
        uint32_t emit = 0;
        while (a) {
            int t1s[P];
            int64_t rws[P];
            float v[P][CPL];
#pragma unroll
            for (int j = 0; j < P; j++) {            // the next P frames (absent: row 0 = zeros)
                const int t1 = __ffs(a) - 1;         // -1 when a == 0
                t1s[j] = t1;
                rws[j] = t1 >= 0 ? base + __popc(sl & lowmask(t1)) : 0;
                a &= a - 1;
            }
#pragma unroll
            for (int j = 0; j < P; j++) {            // issue all P row loads before any use
                ST_CHECK(rws[j] >= 0 && rws[j] < in.nrows);
                row_load<T, CPL>(rows + rws[j] * C, c0, C, full, v[j]);
            }
#pragma unroll
            for (int j = 0; j < P; j++) {            // then step the frames in order
                if (t1s[j] < 0) continue;
                float cand[CPL];
                float mx = 0.0f;
                if constexpr (CPL % 2 == 0) {        // fp32x2 pairs: the same bits as the scalar form
#pragma unroll
                    for (int i = 0; i < CPL; i += 2) {
                        const float2 x = add2(f2(xa[i], xa[i + 1]), f2(v[j][i], v[j][i + 1]));   // Eq.3
                        const float2 cd = sub2(actf2<ACT>(x), f2(ya[i], ya[i + 1]));
                        xa[i] = x.x;
                        xa[i + 1] = x.y;
                        cand[i] = cd.x;
                        cand[i + 1] = cd.y;
                        mx = fmaxf(mx, fmaxf(fabsf(cd.x), fabsf(cd.y)));
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        xa[i] = __fadd_rn(xa[i], v[j][i]);                 // reconstruct x (Eq.3)
                        cand[i] = __fsub_rn(actf<ACT>(xa[i]), ya[i]);      // restore the delta
                        mx = fmaxf(mx, fabsf(cand[i]));
                    }
                }
                mx = gmax<G>(mx, mask);
                if (mx > theta) {                                      // truncation
                    if constexpr (CPL % 2 == 0) {
#pragma unroll
                        for (int i = 0; i < CPL; i += 2) {
                            const float2 r = rnd2<T>(f2(cand[i], cand[i + 1]));
                            const float2 y = add2(f2(ya[i], ya[i + 1]), r);
                            cand[i] = r.x;
                            cand[i + 1] = r.y;
                            ya[i] = y.x;
                            ya[i + 1] = y.y;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < CPL; i++) {
                            cand[i] = rnd<T>(cand[i]);
                            ya[i] = __fadd_rn(ya[i], cand[i]);
                        }
                    }
                    row_store<T, CPL>(out_rows + rws[j] * C, c0, C, full, cand);
                    emit |= 1u << t1s[j];
                } else if (zero_gaps) {   // a rowmap conv reads this slot as a row
                    float z[CPL];
#pragma unroll
                    for (int i = 0; i < CPL; i++) z[i] = 0.0f;
                    row_store<T, CPL>(out_rows + rws[j] * C, c0, C, full, z);
                }
            }
        }
        if (lane == 0) out_act[bp] = emit;
        if (sst.x_save) {   // streaming: state of a touched pixel (in place)
            row_store<float, CPL>(sst.x_save + bp * C, c0, C, full, xa);
            row_store<float, CPL>(sst.y_save + bp * C, c0, C, full, ya);
        }
    }
}

// Wide pointwise site (C > 1280, C % 8 == 0: the 2048-channel stages of
// ResNet-152).  One warp per pixel; the pixel's x_acc,
// y_acc and the frame's candidate live in shared memory (3 x C fp32 per
// warp) instead of registers, walked in 256-channel chunks (8 per lane).
// Per frame: x += Delta, c = f(x) - y over all chunks with the running
// max; warp max; if it exceeds theta, y += rnd(c) and the row is written.
// Same per-channel operations in the same order as k_site_pw (FP32 mode
// bit-exact).
constexpr int PW_WIDE_WARPS = 4;
template <int ACT, class T>
__global__ void __launch_bounds__(32 * PW_WIDE_WARPS) k_site_pw_wide(DView in, const float *__restrict__ x0, int64_t BN,
                                                                  int C, const float *__restrict__ theta_p,
                                                                  uint32_t *__restrict__ out_act, T *out_rows,
                                                                  SiteState sst, bool zero_gaps) {
    st_pdl_enter();
    extern __shared__ float pw_sm[];
    const float theta = __ldg(theta_p);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *xs = pw_sm + (size_t)wid * 3 * C, *ys = xs + C, *cs = ys + C;
    const T *rows = static_cast<const T *>(in.rows);
    for (int64_t bp = (int64_t)blockIdx.x * PW_WIDE_WARPS + wid; bp < BN; bp += (int64_t)gridDim.x * PW_WIDE_WARPS) {
        uint32_t a = __ldg(in.act + bp);
        if (!a) {
            if (lane == 0) out_act[bp] = 0;
            continue;
        }
        const int base = 1 + __ldg(in.pbase + bp);
        const uint32_t sl = __ldg(in.slot + bp);
        for (int c0 = lane * 8; c0 < C; c0 += 256) {
            float x[8], y[8];
            RowIO<float, 8>::load(x0 + bp * C + c0, x);
            if (sst.y_init) RowIO<float, 8>::load(sst.y_init + bp * C + c0, y);
            else
#pragma unroll
                for (int i = 0; i < 8; i++) y[i] = actf<ACT>(x[i]);
            RowIO<float, 8>::store(xs + c0, x);
            RowIO<float, 8>::store(ys + c0, y);
        }
        __syncwarp();
        uint32_t emit = 0;
        while (a) {
            const int t1 = __ffs(a) - 1;
            a &= a - 1;
            const int64_t row = base + __popc(sl & lowmask(t1));
            float mx = 0.0f;
            for (int c0 = lane * 8; c0 < C; c0 += 256) {
                float v[8], x[8], y[8], cand[8];
                RowIO<T, 8>::load(rows + row * C + c0, v);
                RowIO<float, 8>::load(xs + c0, x);
                RowIO<float, 8>::load(ys + c0, y);
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    x[i] = __fadd_rn(x[i], v[i]);                     // reconstruct x (Eq.3)
                    cand[i] = __fsub_rn(actf<ACT>(x[i]), y[i]);       // restore the delta
                    mx = fmaxf(mx, fabsf(cand[i]));
                }
                RowIO<float, 8>::store(xs + c0, x);
                RowIO<float, 8>::store(cs + c0, cand);
            }
            mx = gmax<32>(mx, 0xffffffffu);
            if (mx > theta) {                                          // truncation
                for (int c0 = lane * 8; c0 < C; c0 += 256) {
                    float y[8], cand[8];
                    RowIO<float, 8>::load(cs + c0, cand);
                    RowIO<float, 8>::load(ys + c0, y);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        cand[i] = rnd<T>(cand[i]);
                        y[i] = __fadd_rn(y[i], cand[i]);
                    }
                    RowIO<float, 8>::store(ys + c0, y);
                    RowIO<T, 8>::store(out_rows + row * C + c0, cand);
                }
                emit |= 1u << t1;
            } else if (zero_gaps) {   // a rowmap conv reads this slot as a row
                const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int c0 = lane * 8; c0 < C; c0 += 256) RowIO<T, 8>::store(out_rows + row * C + c0, z);
            }
        }
        if (lane == 0) out_act[bp] = emit;
        if (sst.x_save)
            for (int c0 = lane * 8; c0 < C; c0 += 256) {
                float x[8], y[8];
                RowIO<float, 8>::load(xs + c0, x);
                RowIO<float, 8>::load(ys + c0, y);
                RowIO<float, 8>::store(sst.x_save + bp * C + c0, x);
                RowIO<float, 8>::store(sst.y_save + bp * C + c0, y);
            }
        __syncwarp();   // state rows reused by the next pixel
    }
}

#define CH_DISPATCH(C_, LAUNCH)                                    \
    if ((C_) <= 1) { LAUNCH(1, 1); }                               \
    else if ((C_) <= 2) { LAUNCH(2, 1); }                          \
    else if ((C_) <= 4) { LAUNCH(4, 1); }                          \
    else if ((C_) <= 8) { LAUNCH(8, 1); }                          \
    else if ((C_) <= 16) { LAUNCH(16, 1); }                        \
    else if ((C_) <= 32) { LAUNCH(32, 1); }                        \
    else if ((C_) <= 64) { LAUNCH(32, 2); }                        \
    else if ((C_) <= 96) { LAUNCH(32, 3); }                        \
    else if ((C_) <= 128) { LAUNCH(32, 4); }                       \
    else if ((C_) <= 160) { LAUNCH(32, 5); }                       \
    else if ((C_) <= 256) { LAUNCH(32, 8); }                       \
    else if ((C_) <= 480) { LAUNCH(32, 15); }                      \
    else if ((C_) <= 512) { LAUNCH(32, 16); }                      \
    else if ((C_) <= 672) { LAUNCH(32, 21); }                      \
    else { LAUNCH(32, 36); }

// Pixel-group shape for the site / join / accumulate kernels: 8 channels
// (16 bytes of bf16) per lane when C % 8 == 0, so narrow layers put several
// pixels in one warp (C = 64 -> 8 lanes per pixel, 4 pixels per warp) and a
// lane always moves whole 16-byte vectors; wide layers use 32 lanes.
#define SITE_DISPATCH(C_, LAUNCH)                                  \
    if ((C_) % 8 != 0 || (C_) <= 8) {                              \
        if ((C_) <= 1) { LAUNCH(1, 1); }                           \
        else if ((C_) <= 2) { LAUNCH(2, 1); }                      \
        else if ((C_) <= 4) { LAUNCH(4, 1); }                      \
        else if ((C_) <= 8) { LAUNCH(8, 1); }                      \
        else if ((C_) <= 16) { LAUNCH(16, 1); }                    \
        else if ((C_) <= 32) { LAUNCH(32, 1); }                    \
        else if ((C_) <= 64) { LAUNCH(32, 2); }                    \
        else if ((C_) <= 128) { LAUNCH(32, 4); }                   \
        else if ((C_) <= 256) { LAUNCH(32, 8); }                   \
        else if ((C_) <= 512) { LAUNCH(32, 16); }                  \
        else if ((C_) <= 768) { LAUNCH(32, 24); }                  \
        else { LAUNCH(32, 40); }                                   \
    } else if ((C_) <= 16) { LAUNCH(2, 8); }                       \
    else if ((C_) <= 32) { LAUNCH(4, 8); }                         \
    else if ((C_) <= 64) { LAUNCH(8, 8); }                         \
    else if ((C_) <= 128) { LAUNCH(16, 8); }                       \
    else if ((C_) <= 256) { LAUNCH(32, 8); }                       \
    else if ((C_) <= 512) { LAUNCH(32, 16); }                      \
    else if ((C_) <= 768) { LAUNCH(32, 24); }                      \
    else if ((C_) <= 1280) { LAUNCH(32, 40); }                     \
    else { LAUNCH(32, 64); }

static int groups_grid(int64_t n_groups, int G) {
    const int64_t threads = n_groups * G;
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(threads, 256), 148 * 8));
}

void launch_site_pointwise(DView in, const float *x0, int B, int N, int C, int act, const float *theta, bool bf,
                           uint32_t *out_act, void *out_rows, const SiteState &st, cudaStream_t s, bool zero_gaps) {
    const int64_t BN = (int64_t)B * N;
    if (C > 1280 && C % 8 == 0) {
        const size_t sm = (size_t)PW_WIDE_WARPS * 3 * C * sizeof(float);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(BN, PW_WIDE_WARPS), 148 * 8));
#define L_PWW(ACT_)                                                                                    \
    {                                                                                                  \
        auto kf = k_site_pw_wide<ACT_, T>;                                                             \
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                \
        kf<<<grid, 32 * PW_WIDE_WARPS, sm, s>>>(in, x0, BN, C, theta, out_act, static_cast<T *>(out_rows), st,   \
                                                zero_gaps);                                                    \
    }
        ST_ROW_DISPATCH(bf, if (act == ACT_RELU) L_PWW(ACT_RELU) else if (sizeof(T) == 4) L_PWW(ACT_SILU) else L_PWW(ACT_SILU_FAST));
#undef L_PWW
        return;
    }

#define L_PW(G_, CPL_)                                                                                 \
    {                                                                                                  \
        const int64_t want = cdiv(BN * G_, 256);                                                       \
        if (act == ACT_RELU) {                                                                         \
            auto kf = k_site_pw<G_, CPL_, ACT_RELU, T>;                                                \
            kf<<<resident_grid(kf, 256, 0, want, 148 * 8), 256, 0, s>>>(in, x0, BN, C, theta, out_act,  \
                                                                  static_cast<T *>(out_rows), st,      \
                                                                  zero_gaps);                          \
        } else { /* SiLU: exact (double exp) in FP32 mode, fast in BF16 mode */                        \
            auto kf = k_site_pw<G_, CPL_, (sizeof(T) == 4 ? ACT_SILU : ACT_SILU_FAST), T>;             \
            kf<<<resident_grid(kf, 256, 0, want, 148 * 8), 256, 0, s>>>(                               \
                in, x0, BN, C, theta, out_act, static_cast<T *>(out_rows), st, zero_gaps);             \
        }                                                                                              \
    }
    ST_ROW_DISPATCH(bf, SITE_DISPATCH(C, L_PW));
#undef L_PW
}

// --------------------------------------------------------- maxpool site
// Touched set T = footprint dilation of the input mask (R7);
// each touched window is re-evaluated from x_acc of its input pixels.  The
// window pixels' frame words are read once per output pixel; the rows of
// the next P touched frames are fetched together.
template <int G, int CPL, int KMAX, class T>
__global__ void __launch_bounds__(256) k_site_maxpool(DView in, const float *__restrict__ x0, int B, Geo g,
                                                      const float *__restrict__ theta_p,
                                                      const uint32_t *__restrict__ t_slot,
                                                      const int32_t *__restrict__ t_pbase,
                                                      uint32_t *__restrict__ out_act, T *__restrict__ out_rows,
                                                      SiteState sst) {
    st_pdl_enter();
    const float theta = __ldg(theta_p);
    constexpr int P = CPL <= 2 ? 4 : CPL <= 4 ? 2 : 1;
    const int lane = threadIdx.x & (G - 1);
    const int C = g.Cin;
    const int c0 = lane * CPL;
    const bool full = (C % 8 == 0) && (c0 + CPL <= C);
    const unsigned mask = group_mask<G>();
    const int Nin = g.Hin * g.Win, No = g.Hout * g.Wout;
    const int64_t BN = (int64_t)B * No;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const T *rows = static_cast<const T *>(in.rows);
    for (int64_t bq = grp; bq < BN; bq += ngrp) {
        const uint32_t Tw = __ldg(t_slot + bq);
        if (!Tw) {
            if (lane == 0) out_act[bq] = 0;
            continue;
        }
        const int b = (int)(bq / No), q = (int)(bq % No);
        const int oy = q / g.Wout, ox = q % g.Wout;
        uint32_t wa[KMAX], wsl[KMAX];
        int wbase[KMAX];
        uint32_t valid = 0;
        float xa[KMAX][CPL];
#pragma unroll
        for (int w = 0; w < KMAX; w++) {
            const int dy = w / g.kw, dx = w % g.kw;
            const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
            wa[w] = 0;
            wsl[w] = 0;
            wbase[w] = 0;
            if (w < g.kh * g.kw && iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                const int64_t p = (int64_t)b * Nin + iy * g.Win + ix;
                valid |= 1u << w;
                wa[w] = __ldg(in.act + p);
                if (wa[w]) {
                    wsl[w] = __ldg(in.slot + p);
                    wbase[w] = 1 + __ldg(in.pbase + p);
                }
                row_load<float, CPL>(x0 + p * C, c0, C, full, xa[w]);
            } else {
#pragma unroll
                for (int i = 0; i < CPL; i++) xa[w][i] = -CUDART_INF_F;
            }
        }
        float ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            float m = -CUDART_INF_F;
#pragma unroll
            for (int w = 0; w < KMAX; w++)
                if ((valid >> w) & 1u) m = xa[w][i] > m ? xa[w][i] : m;
            ya[i] = m;
        }
        if (sst.y_init) row_load<float, CPL>(sst.y_init + bq * C, c0, C, full, ya);   // streaming continuation
        const int base = 1 + __ldg(t_pbase + bq);
        uint32_t bits = Tw, emit = 0;
        while (bits) {
            int t1s[P];
            uint32_t has[P];
            float v[P][KMAX][CPL];
            int64_t wrow[P][KMAX];
#pragma unroll
            for (int j = 0; j < P; j++) {            // the next P touched frames
                const int t1 = __ffs(bits) - 1;      // -1 when bits == 0
                bits &= bits - 1;
                t1s[j] = t1;
                has[j] = 0;
#pragma unroll
                for (int w = 0; w < KMAX; w++) {
                    const bool on = t1 >= 0 && ((wa[w] >> t1) & 1u);
                    has[j] |= (uint32_t)on << w;
                    wrow[j][w] = on ? wbase[w] + __popc(wsl[w] & lowmask(t1)) : 0;   // row 0 = zeros
                }
            }
#pragma unroll
            for (int j = 0; j < P; j++)              // issue every window row load before any use
#pragma unroll
                for (int w = 0; w < KMAX; w++) row_load<T, CPL>(rows + wrow[j][w] * C, c0, C, full, v[j][w]);
#pragma unroll
            for (int j = 0; j < P; j++) {
                if (t1s[j] < 0) continue;
#pragma unroll
                for (int w = 0; w < KMAX; w++)
                    if ((has[j] >> w) & 1u)
#pragma unroll
                        for (int i = 0; i < CPL; i++) xa[w][i] = __fadd_rn(xa[w][i], v[j][w][i]);
                float cand[CPL];
                float mx = 0.0f;
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    float m = -CUDART_INF_F;
#pragma unroll
                    for (int w = 0; w < KMAX; w++)
                        if ((valid >> w) & 1u) m = xa[w][i] > m ? xa[w][i] : m;
                    cand[i] = c0 + i < C ? __fsub_rn(m, ya[i]) : 0.0f;
                    mx = fmaxf(mx, fabsf(cand[i]));
                }
                mx = gmax<G>(mx, mask);
                if (mx > theta) {
                    const int64_t orow = base + __popc(Tw & lowmask(t1s[j]));
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        cand[i] = rnd<T>(cand[i]);
                        ya[i] = __fadd_rn(ya[i], cand[i]);
                    }
                    row_store<T, CPL>(out_rows + orow * C, c0, C, full, cand);
                    emit |= 1u << t1s[j];
                }
            }
        }
        if (lane == 0) out_act[bq] = emit;
        if (sst.x_save) {   // streaming: x_acc of the window pixels that changed (overlapping
                            // windows write identical values), y_acc of this output
#pragma unroll
            for (int w = 0; w < KMAX; w++)
                if (wa[w]) {
                    const int dy = w / g.kw, dx = w % g.kw;
                    const int64_t p = (int64_t)b * Nin + (oy * g.sh - g.ph + dy) * g.Win + ox * g.sw - g.pw + dx;
                    row_store<float, CPL>(sst.x_save + p * C, c0, C, full, xa[w]);
                }
            row_store<float, CPL>(sst.y_save + bq * C, c0, C, full, ya);
        }
    }
}

// Tile-resident variant (C = G*CPL, G a power of two <= 32).  A CTA owns
// a TOH x TOW tile of output pixels of one chunk; the x_acc state of the
// tile's input footprint lives in shared memory (one fp32 row per input
// pixel, shared by the overlapping windows instead of one register copy per
// window), the y_acc of each output in the registers of its lane group.
// Frames of the tile's union word run in order.  Each thread owns fixed
// (footprint pixel, lane chunk) units; the delta pieces of its units for the
// frame MP_NS-1 ahead are staged with cp.async into a ring of MP_NS frame
// stages (thread-private slots, so a per-thread cp.async.wait_group is the
// only completion needed), so DRAM latency overlaps the frames in between.
// Per frame: x_acc += Delta_t at the active footprint pixels, then every
// touched output re-evaluates its window max (R7).  Per-pixel
// arithmetic is identical to k_site_maxpool (x_acc += Delta in frame order,
// max over the valid window, c = max - y_acc), so FP32 mode stays bit-exact.
//
// FUSE: the ReLU site that feeds the pool runs in the same pass (ReLU ->
// maxpool with the ReLU output consumed only by the pool).  `in` is then the
// CONV delta tensor and x0 the conv's dense pre-activation; each unit keeps
// the ReLU x_acc in registers and the ReLU y_acc -- which is, bit for bit,
// the pool's x_acc (both start from relu(x0) and advance by the same emitted
// values) -- in shared memory.  Per frame a unit runs the pointwise site
// step of k_site_pw (x += Delta; c = relu(x) - y; emit iff max_c |c| > theta_r;
// y += rnd(c)), records the emission in a per-pixel word, and the pool's
// touched set is the window-OR of those words (the footprint dilation of the
// ReLU's emitted mask, R7).  The pool's row layout (t_slot, t_pbase) is the
// dilation of the CONV mask, a superset of the touched frames (rows of
// untouched frames stay unused).  The ReLU delta rows never go to HBM
// (written only when r_rows != nullptr, debug); its mask words are written
// for the statistics.  Requires every ReLU pixel to lie in some window.
constexpr int MP_NS = 4;    // frame stages in flight
constexpr int MP_KU = 4;    // units per thread (footprint pixels x G <= 1024)

template <int G, int CPL, int OPT, class T, bool FUSE>
__global__ void __launch_bounds__(256) k_site_maxpool_t(DView in, const float *__restrict__ x0, int B, Geo g,
                                                        int TOH, int TOW, const float *__restrict__ theta_p,
                                                        const uint32_t *__restrict__ t_slot,
                                                        const int32_t *__restrict__ t_pbase,
                                                        uint32_t *__restrict__ out_act, T *__restrict__ out_rows,
                                                        const float *__restrict__ theta_rp, uint32_t *__restrict__ r_act,
                                                        T *__restrict__ r_rows, SiteState sst) {
    st_pdl_enter();
    constexpr int NGR = 256 / G;                          // output groups per CTA
    constexpr int PIECES = CPL * (int)sizeof(T) / 16;     // 16-byte pieces per unit
    constexpr int XR = FUSE ? MP_KU : 1;                  // ReLU x_acc register rows
    extern __shared__ __align__(16) unsigned char smem_mp[];
    const int C = G * CPL;
    const float theta = __ldg(theta_p);
    const float theta_r = FUSE ? __ldg(theta_rp) : 0.0f;
    const int tid = threadIdx.x, lane = tid & (G - 1), gr = tid / G;
    const unsigned gmask = group_mask<G>();
    const int Nin = g.Hin * g.Win, No = g.Hout * g.Wout;
    const int ntx = (g.Wout + TOW - 1) / TOW, nty = (g.Hout + TOH - 1) / TOH;
    const int b = blockIdx.x / (ntx * nty);
    const int tr = blockIdx.x - b * ntx * nty;
    const int ty = tr / ntx, tx = tr - ty * ntx;
    const int FH = (TOH - 1) * g.sh + g.kh, FW = (TOW - 1) * g.sw + g.kw, FP = FH * FW;
    const int fy0 = ty * TOH * g.sh - g.ph, fx0 = tx * TOW * g.sw - g.pw;
    float *xs = reinterpret_cast<float *>(smem_mp);
    T *stg = reinterpret_cast<T *>(xs + (size_t)FP * C);                // [MP_NS][ku][256][CPL]
    uint32_t *u_word = reinterpret_cast<uint32_t *>(stg + (size_t)MP_NS * ((FP * G + 255) / 256) * 256 * CPL);
    uint32_t *r_em = u_word + 4;                                         // FUSE: [FP] ReLU emitted words
    const T *rows = static_cast<const T *>(in.rows);
    if (tid == 0) *u_word = 0u;
    if (FUSE)
        for (int p = tid; p < FP; p += 256) r_em[p] = 0u;
    // ---- this thread's units: metadata in registers, x0 into x_acc (-inf outside the map, R11)
    uint32_t u_act[MP_KU], u_sl[MP_KU], r_emit[MP_KU];
    int u_r1[MP_KU], u_off[MP_KU];
    float xr[XR][CPL];
    uint32_t uw = 0;
#pragma unroll
    for (int k = 0; k < MP_KU; k++) {
        const int u = tid + k * 256;
        const int p = u / G, l = u - (u / G) * G;
        u_act[k] = 0;
        u_sl[k] = 0;
        u_r1[k] = 0;
        r_emit[k] = 0;
        u_off[k] = p * C + l * CPL;
        if (p < FP) {
            const int iy = fy0 + p / FW, ix = fx0 + p % FW;
            float v[CPL];
            if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                const int64_t gp = (int64_t)b * Nin + iy * g.Win + ix;
                u_act[k] = __ldg(in.act + gp);
                if (u_act[k]) {
                    u_sl[k] = __ldg(in.slot + gp);
                    u_r1[k] = 1 + __ldg(in.pbase + gp);
                }
                RowIO<float, CPL>::load(x0 + gp * C + l * CPL, v);
                if constexpr (FUSE) {
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        xr[k][i] = v[i];
                        v[i] = relu_f(v[i]);   // y0 of the ReLU = x0 of the pool
                    }
                    if (sst.ry_init) RowIO<float, CPL>::load(sst.ry_init + gp * C + l * CPL, v);   // continuation
                }
            } else {
#pragma unroll
                for (int i = 0; i < CPL; i++) v[i] = -CUDART_INF_F;
            }
            RowIO<float, CPL>::store(xs + u_off[k], v);
            uw |= u_act[k];
        }
    }
    uw = __reduce_or_sync(0xffffffffu, uw);
    __syncthreads();
    if ((tid & 31) == 0 && uw) atomicOr(u_word, uw);
    __syncthreads();
    // ---- outputs of this group: y_acc = window max of x0 (= y0)
    int64_t ob[OPT];
    uint32_t Tw[OPT], emit[OPT];
    int obase[OPT], wo[OPT];   // wo: footprint index of the window's top-left pixel
    float ya[OPT][CPL];
#pragma unroll
    for (int j = 0; j < OPT; j++) {
        const int o = gr + j * NGR;
        const int loy = o / TOW, lox = o - (o / TOW) * TOW;
        const int oy = ty * TOH + loy, ox = tx * TOW + lox;
        ob[j] = -1;
        Tw[j] = 0;
        emit[j] = 0;
        obase[j] = 0;
        wo[j] = loy * g.sh * FW + lox * g.sw;
        if (o < TOH * TOW && oy < g.Hout && ox < g.Wout) {
            ob[j] = (int64_t)b * No + oy * g.Wout + ox;
            Tw[j] = __ldg(t_slot + ob[j]);
            obase[j] = 1 + __ldg(t_pbase + ob[j]);
        }
#pragma unroll
        for (int i = 0; i < CPL; i++) ya[j][i] = -CUDART_INF_F;
        if (ob[j] >= 0)
            for (int dy = 0; dy < g.kh; dy++)
                for (int dx = 0; dx < g.kw; dx++) {
                    float w[CPL];
                    RowIO<float, CPL>::load(xs + (size_t)(wo[j] + dy * FW + dx) * C + lane * CPL, w);
#pragma unroll
                    for (int i = 0; i < CPL; i++) ya[j][i] = w[i] > ya[j][i] ? w[i] : ya[j][i];
                }
        if (sst.y_init && ob[j] >= 0) RowIO<float, CPL>::load(sst.y_init + ob[j] * C + lane * CPL, ya[j]);
    }
    __syncthreads();   // every window's y_acc taken from x0 before frame 1 updates x_acc
    const uint32_t U = *u_word;
    const int ku = (FP * G + 255) / 256;   // units per thread in use (<= MP_KU): stage stride
    // stage the active units of frame bit t1 (t1 < 0: nothing) into ring slot st
    auto issue = [&](int t1, int st) {
        if (t1 < 0) return;
#pragma unroll
        for (int k = 0; k < MP_KU; k++)
            if ((u_act[k] >> t1) & 1u) {
                const int row = u_r1[k] + __popc(u_sl[k] & lowmask(t1));
                const unsigned char *src =
                    reinterpret_cast<const unsigned char *>(rows + (int64_t)row * C + (u_off[k] % C));
                unsigned char *dst =
                    reinterpret_cast<unsigned char *>(stg + ((size_t)(st * ku + k) * 256 + tid) * CPL);
#pragma unroll
                for (int q = 0; q < PIECES; q++)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(dst + 16 * q)),
                                 "l"(src + 16 * q)
                                 : "memory");
            }
    };
    // prologue: frames 0 .. MP_NS-2 of U in flight
    uint32_t Ui = U;   // frames not yet issued
    for (int s = 0; s < MP_NS - 1; s++) {
        const int t1 = Ui ? __ffs(Ui) - 1 : -1;
        if (Ui) Ui &= Ui - 1;
        issue(t1, s);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    uint32_t Uc = U;   // frames not yet consumed
    int it = 0;
    while (Uc) {
        const int t1 = __ffs(Uc) - 1;
        Uc &= Uc - 1;
        {   // frame MP_NS-1 ahead into the slot consumed MP_NS-1 frames from now
            const int tn = Ui ? __ffs(Ui) - 1 : -1;
            if (Ui) Ui &= Ui - 1;
            issue(tn, (it + MP_NS - 1) % MP_NS);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.wait_group %0;" ::"n"(MP_NS - 1) : "memory");
        const int st = it % MP_NS;
        if constexpr (FUSE) {
            // (a') ReLU site step at this thread's active units (pixel-uniform branch)
#pragma unroll
            for (int k = 0; k < MP_KU; k++)
                if ((u_act[k] >> t1) & 1u) {
                    float v[CPL], y[CPL], cand[CPL];
                    RowIO<T, CPL>::load(stg + ((size_t)(st * ku + k) * 256 + tid) * CPL, v);
                    RowIO<float, CPL>::load(xs + u_off[k], y);
                    float mx = 0.0f;
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        xr[k][i] = __fadd_rn(xr[k][i], v[i]);
                        cand[i] = __fsub_rn(relu_f(xr[k][i]), y[i]);
                        mx = fmaxf(mx, fabsf(cand[i]));
                    }
                    mx = gmax<G>(mx, gmask);
                    if (mx > theta_r) {
#pragma unroll
                        for (int i = 0; i < CPL; i++) {
                            cand[i] = rnd<T>(cand[i]);
                            y[i] = __fadd_rn(y[i], cand[i]);
                        }
                        RowIO<float, CPL>::store(xs + u_off[k], y);
                        r_emit[k] |= 1u << t1;
                        if ((tid & (G - 1)) == 0) r_em[(tid + k * 256) / G] |= 1u << t1;
                        if (r_rows) {
                            const int row = u_r1[k] + __popc(u_sl[k] & lowmask(t1));
                            RowIO<T, CPL>::store(r_rows + (int64_t)row * C + (u_off[k] % C), cand);
                        }
                    }
                }
        } else {
            // (a) x_acc += Delta_t at this thread's active units (own staged pieces)
#pragma unroll
            for (int k = 0; k < MP_KU; k++)
                if ((u_act[k] >> t1) & 1u) {
                    float v[CPL], w[CPL];
                    RowIO<T, CPL>::load(stg + ((size_t)(st * ku + k) * 256 + tid) * CPL, v);
                    RowIO<float, CPL>::load(xs + u_off[k], w);
#pragma unroll
                    for (int i = 0; i < CPL; i++) w[i] = __fadd_rn(w[i], v[i]);
                    RowIO<float, CPL>::store(xs + u_off[k], w);
                }
        }
        __syncthreads();
        // (b) touched outputs: candidate = window max - y_acc, truncation
#pragma unroll
        for (int j = 0; j < OPT; j++) {
            if (!((Tw[j] >> t1) & 1u)) continue;   // group-uniform
            if constexpr (FUSE) {   // touched iff some window pixel's ReLU emitted at t1
                uint32_t tch = 0;
                for (int dy = 0; dy < g.kh; dy++)
                    for (int dx = 0; dx < g.kw; dx++) tch |= r_em[wo[j] + dy * FW + dx];
                if (!((tch >> t1) & 1u)) continue;
            }
            float m[CPL];
#pragma unroll
            for (int i = 0; i < CPL; i++) m[i] = -CUDART_INF_F;
            for (int dy = 0; dy < g.kh; dy++)
                for (int dx = 0; dx < g.kw; dx++) {
                    float w[CPL];
                    RowIO<float, CPL>::load(xs + (size_t)(wo[j] + dy * FW + dx) * C + lane * CPL, w);
#pragma unroll
                    for (int i = 0; i < CPL; i++) m[i] = w[i] > m[i] ? w[i] : m[i];
                }
            float cand[CPL];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                cand[i] = __fsub_rn(m[i], ya[j][i]);
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            mx = gmax<G>(mx, gmask);
            if (mx > theta) {
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    cand[i] = rnd<T>(cand[i]);
                    ya[j][i] = __fadd_rn(ya[j][i], cand[i]);
                }
                RowIO<T, CPL>::store(out_rows + (int64_t)(obase[j] + __popc(Tw[j] & lowmask(t1))) * C + lane * CPL,
                                     cand);
                emit[j] |= 1u << t1;
            }
        }
        __syncthreads();
        it++;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
    for (int j = 0; j < OPT; j++)
        if (ob[j] >= 0 && lane == 0) out_act[ob[j]] = emit[j];
    if (sst.y_save) {   // streaming: pool y_acc of the outputs (in place), x_acc of the footprint
#pragma unroll
        for (int j = 0; j < OPT; j++)
            if (ob[j] >= 0) RowIO<float, CPL>::store(sst.y_save + ob[j] * C + lane * CPL, ya[j]);
#pragma unroll
        for (int k = 0; k < MP_KU; k++) {
            const int u = tid + k * 256;
            const int p = u / G;
            if (p >= FP) continue;
            const int iy = fy0 + p / FW, ix = fx0 + p % FW;
            if (iy < 0 || iy >= g.Hin || ix < 0 || ix >= g.Win) continue;
            const int64_t o = ((int64_t)b * Nin + iy * g.Win + ix) * C + (u_off[k] % C);
            if constexpr (FUSE) {   // every footprint pixel (ping-pong buffers, halo: identical writes)
                float w[CPL];
                RowIO<float, CPL>::load(xs + u_off[k], w);
                RowIO<float, CPL>::store(sst.ry_save + o, w);
                RowIO<float, CPL>::store(sst.rx_save + o, xr[k]);
            } else if (u_act[k]) {  // pixels that changed (the rest was pre-copied)
                float w[CPL];
                RowIO<float, CPL>::load(xs + u_off[k], w);
                RowIO<float, CPL>::store(sst.x_save + o, w);
            }
        }
    }
    if constexpr (FUSE) {   // ReLU mask words of the footprint (halo pixels: identical duplicate writes)
#pragma unroll
        for (int k = 0; k < MP_KU; k++) {
            const int u = tid + k * 256;
            const int p = u / G;
            if (p >= FP || (u & (G - 1))) continue;
            const int iy = fy0 + p / FW, ix = fx0 + p % FW;
            if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) r_act[(int64_t)b * Nin + iy * g.Win + ix] = r_emit[k];
        }
    }
}

// output tile for the tile-resident maxpool: the most outputs per CTA whose
// input footprint's fp32 x_acc fits in 64 KiB
static size_t mp_smem(int FP, int C, int G, int esz) {
    // x_acc rows | cp.async frame ring | u_word (+pad) | FUSE: per-pixel ReLU emitted words
    return (size_t)FP * C * 4 + (size_t)MP_NS * ((FP * G + 255) / 256) * 256 * (C / G) * esz + 16 + (size_t)FP * 4;
}
static bool mp_tile(const Geo &g, int C, int G, int esz, int max_out, int &TOH, int &TOW) {
    int fp_max = std::min(16384 / C, 256 * MP_KU / G);
    while (fp_max > 1 && mp_smem(fp_max, C, G, esz) > 200 * 1024) fp_max--;
    int best = 0;
    TOH = TOW = 0;
    for (int h = 1; h <= std::min(g.Hout, 32); h++)
        for (int w = 1; w <= std::min(g.Wout, 64); w++) {
            const int fp = ((h - 1) * g.sh + g.kh) * ((w - 1) * g.sw + g.kw);
            if (h * w > max_out || fp > fp_max) continue;
            // most outputs; ties: fewest footprint pixels
            if (h * w > best || (h * w == best && fp < ((TOH - 1) * g.sh + g.kh) * ((TOW - 1) * g.sw + g.kw))) {
                best = h * w;
                TOH = h;
                TOW = w;
            }
        }
    return best > 0;
}

constexpr int MP_OPT = 2;   // outputs per lane group
struct MpPlan {
    int TG = 0, TCPL = 0, TOH = 0, TOW = 0;
};
// tile-resident kernel when C = G * CPL (G a power of two <= 32, CPL 8 or 16)
static bool mp_plan(const Geo &g, bool bf, MpPlan &pl) {
    const int C = g.Cin;
    if (C % 8 != 0 || C < 16) return false;
    const int cpl = std::max(8, C / 32), gg = C / cpl;
    if (gg * cpl != C || (gg & (gg - 1)) != 0 || (cpl != 8 && cpl != 16)) return false;
    pl.TG = gg;
    pl.TCPL = cpl;
    return mp_tile(g, C, gg, bf ? 2 : 4, MP_OPT * (256 / gg), pl.TOH, pl.TOW);
}

bool site_relu_maxpool_fusable(const Geo &g, bool bf) {
    MpPlan pl;
    if (!mp_plan(g, bf, pl)) return false;
    // every input pixel inside some window (the fused pass runs the ReLU site
    // only on window footprints): no gaps between windows, last window reaches the edge
    auto covers = [](int in, int out, int k, int st, int pd) { return st <= k && (out - 1) * st - pd + k >= in; };
    return covers(g.Hin, g.Hout, g.kh, g.sh, g.ph) && covers(g.Win, g.Wout, g.kw, g.sw, g.pw);
}

template <bool FUSE>
static bool launch_mp_tile(const MpPlan &pl, DView in, const float *x0, int B, const Geo &g, const float *theta,
                           bool bf, const uint32_t *t_slot, const int32_t *t_pbase, uint32_t *out_act, void *out_rows,
                           const float *theta_r, uint32_t *r_act, void *r_rows, const SiteState &st,
                           cudaStream_t s) {
    const int C = g.Cin, TG = pl.TG, TCPL = pl.TCPL, TOH = pl.TOH, TOW = pl.TOW;
    const int FP = ((TOH - 1) * g.sh + g.kh) * ((TOW - 1) * g.sw + g.kw);
    const size_t sm = mp_smem(FP, C, TG, bf ? 2 : 4);
    const int64_t tiles = (int64_t)B * ((g.Hout + TOH - 1) / TOH) * ((g.Wout + TOW - 1) / TOW);
#define L_MPT(G_, CPL_)                                                                                      \
    {                                                                                                        \
        auto kf = k_site_maxpool_t<G_, CPL_, MP_OPT, T, FUSE>;                                               \
        cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                      \
        kf<<<(unsigned)tiles, 256, sm, s>>>(in, x0, B, g, TOH, TOW, theta, t_slot, t_pbase, out_act,         \
                                            static_cast<T *>(out_rows), theta_r, r_act,                      \
                                            static_cast<T *>(r_rows), st);                                   \
    }
#define L_MPT_C(...)                                                                                         \
    if (TG == 2) L_MPT(2, 8) else if (TG == 4) L_MPT(4, 8) else if (TG == 8) L_MPT(8, 8)                     \
    else if (TG == 16) L_MPT(16, 8) else if (TCPL == 8) L_MPT(32, 8) else L_MPT(32, 16)
    ST_ROW_DISPATCH(bf, L_MPT_C());
#undef L_MPT_C
#undef L_MPT
    return true;
}

void launch_site_relu_maxpool(DView conv, const float *x0_conv, int B, const Geo &g, const float *theta_r,
                              const float *theta, bool bf, const uint32_t *t_slot, const int32_t *t_pbase,
                              uint32_t *r_act, void *r_rows, uint32_t *out_act, void *out_rows, const SiteState &st,
                              cudaStream_t s) {
    MpPlan pl;
    if (!mp_plan(g, bf, pl)) return;   // callers check site_relu_maxpool_fusable first
    launch_mp_tile<true>(pl, conv, x0_conv, B, g, theta, bf, t_slot, t_pbase, out_act, out_rows, theta_r, r_act,
                         r_rows, st, s);
}

void launch_site_maxpool(DView in, const float *x0, int B, const Geo &g, const float *theta, bool bf,
                         const uint32_t *t_slot, const int32_t *t_pbase, uint32_t *out_act, void *out_rows,
                         const SiteState &st, cudaStream_t s) {
    const int64_t BN = (int64_t)B * g.Hout * g.Wout;
    const int kk = g.kh * g.kw;
    MpPlan pl;
    if (mp_plan(g, bf, pl)) {
        launch_mp_tile<false>(pl, in, x0, B, g, theta, bf, t_slot, t_pbase, out_act, out_rows, nullptr, nullptr,
                              nullptr, st, s);
        return;
    }
#define L_MP(G_, CPL_)                                                                                       \
    {                                                                                                        \
        const int grid = groups_grid(BN, G_);                                                                \
        if (kk <= 4)                                                                                         \
            k_site_maxpool<G_, CPL_, 4, T><<<grid, 256, 0, s>>>(in, x0, B, g, theta, t_slot, t_pbase,        \
                                                                out_act, static_cast<T *>(out_rows), st);    \
        else                                                                                                 \
            k_site_maxpool<G_, CPL_, 9, T><<<grid, 256, 0, s>>>(in, x0, B, g, theta, t_slot, t_pbase,        \
                                                                out_act, static_cast<T *>(out_rows), st);    \
    }
    ST_ROW_DISPATCH(bf, SITE_DISPATCH(g.Cin, L_MP));
#undef L_MP
}

// ---------------------------------------------------------- residual add
template <int G, int CPL, class T>
__global__ void __launch_bounds__(256) k_add_rows(DView a, DView b, const uint32_t *__restrict__ slot,
                                                  const int32_t *__restrict__ pbase, int64_t BN, int C,
                                                  T *__restrict__ out) {
    st_pdl_enter();
    const int lane = threadIdx.x & (G - 1);
    const int c0 = lane * CPL;
    const bool full = (C % 8 == 0) && (c0 + CPL <= C);
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const T *ra_rows = static_cast<const T *>(a.rows);
    const T *rb_rows = static_cast<const T *>(b.rows);
    for (int64_t bp = grp; bp < BN; bp += ngrp) {
        uint32_t w = __ldg(slot + bp);
        if (!w) continue;
        int64_t row = 1 + __ldg(pbase + bp);
        while (w) {
            const int t1 = __ffs(w) - 1;
            w &= w - 1;
            const int ra = row_of(a, bp, t1), rb = row_of(b, bp, t1);
            float va[CPL], vb[CPL];
            if (ra) row_load<T, CPL>(ra_rows + (int64_t)ra * C, c0, C, full, va);
            else
#pragma unroll
                for (int i = 0; i < CPL; i++) va[i] = 0.0f;
            if (rb) row_load<T, CPL>(rb_rows + (int64_t)rb * C, c0, C, full, vb);
            else
#pragma unroll
                for (int i = 0; i < CPL; i++) vb[i] = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) va[i] = __fadd_rn(va[i], vb[i]);
            row_store<T, CPL>(out + row * C, c0, C, full, va);
            row++;
        }
    }
}

void launch_add_rows(DView a, DView b, const uint32_t *slot, const int32_t *pbase, int B, int N, int C, bool bf,
                     void *out_rows, cudaStream_t s) {
    const int64_t BN = (int64_t)B * N;
#define L_ADD(G_, CPL_) \
    k_add_rows<G_, CPL_, T><<<groups_grid(BN, G_), 256, 0, s>>>(a, b, slot, pbase, BN, C, static_cast<T *>(out_rows));
    ST_ROW_DISPATCH(bf, SITE_DISPATCH(C, L_ADD));
#undef L_ADD
}

// ---------------------------------------------------------- accumulation
// O_t = O_{t-1} + Delta_t, dense per-frame outputs [B][L][N][C].
template <int G, int CPL, class T>
__global__ void __launch_bounds__(256) k_accumulate(DView in, const float *y0, int B, int N, int C,
                                                    int n_diff, float *__restrict__ out, float *o_save) {
    st_pdl_enter();
    const int lane = threadIdx.x & (G - 1);
    const int c0 = lane * CPL;
    const bool full = (C % 8 == 0) && (c0 + CPL <= C);
    const int64_t BN = (int64_t)B * N;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const int64_t fstride = (int64_t)N * C;
    const T *rows = static_cast<const T *>(in.rows);
    for (int64_t bq = grp; bq < BN; bq += ngrp) {
        const int b = (int)(bq / N), q = (int)(bq % N);
        const uint32_t a = n_diff ? __ldg(in.act + bq) : 0u;
        const int base = a ? 1 + __ldg(in.pbase + bq) : 0;
        const uint32_t sl = a ? __ldg(in.slot + bq) : 0u;
        float O[CPL];
        float *o = out + (int64_t)b * (n_diff + 1) * fstride + (int64_t)q * C;
        row_load<float, CPL>(y0 + bq * C, c0, C, full, O);
        row_store<float, CPL>(o, c0, C, full, O);
        for (int t1 = 0; t1 < n_diff; t1++) {
            o += fstride;
            if ((a >> t1) & 1u) {
                const int64_t row = base + __popc(sl & lowmask(t1));
                float v[CPL];
                row_load<T, CPL>(rows + row * C, c0, C, full, v);
#pragma unroll
                for (int i = 0; i < CPL; i++) O[i] = __fadd_rn(O[i], v[i]);
            }
            row_store<float, CPL>(o, c0, C, full, O);
        }
        if (o_save) row_store<float, CPL>(o_save + bq * C, c0, C, full, O);   // streaming: next call's start
    }
}

void launch_accumulate(DView in, const float *y0, int B, int N, int C, int n_diff, bool bf, float *out,
                       float *o_save, cudaStream_t s) {
    const int64_t BN = (int64_t)B * N;
#define L_ACC(G_, CPL_) \
    k_accumulate<G_, CPL_, T><<<groups_grid(BN, G_), 256, 0, s>>>(in, y0, B, N, C, n_diff, out, o_save);
    ST_ROW_DISPATCH(bf, SITE_DISPATCH(C, L_ACC));
#undef L_ACC
}

}  // namespace st
