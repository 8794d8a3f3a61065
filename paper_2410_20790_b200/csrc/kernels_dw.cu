// kernels_dw.cu -- depthwise convolution (groups == C_in == C_out, reading R9)
// on compacted deltas and on the dense reference frame, sm_100a.
//
// Eq.(2) per channel: Delta_out[c] = sum over the
// kxk taps (dy, dx ascending) of W[c][dy][dx] * Delta_in[c], bias absent;
// dense mode adds the bias last.  Depthwise work is HBM-bound (1.8-12.5
// flop/B), so the kernel is organised around memory
// parallelism: one output row per group of G lanes; the tap row indices of
// the row are resolved once (32-bit, into registers), then the channels are
// walked in chunks of G*8 -- lane l owns 8 channels of a chunk, moved as one
// 16-byte bf16 vector (two float4 in FP32 mode) -- and a batch of tap loads
// is issued before its FMAs.  FP32-mode results are bit-identical to the
// oracle (fmaf chain in tap order from +0).
#include "rowio.cuh"

namespace st {

template <int G, int CPL, int KMAX, class T>
__global__ void __launch_bounds__(256, 2) k_dwconv(ConvCall c) {
    constexpr int TB = KMAX > 9 ? 5 : 3;      // taps per load batch
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int M = c.dense ? c.B * Nout : *c.m_dev;
    const int C = g.Cin;
    const int lane = threadIdx.x & (G - 1);
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const int ntaps = g.kh * g.kw;
    const T *A = c.dense ? reinterpret_cast<const T *>(c.a_dense) : static_cast<const T *>(c.a.rows);
    for (int64_t r = grp; r < M; r += ngrp) {
        int b, q, t1 = 0;
        if (c.dense) {
            b = (int)(r / Nout);
            q = (int)(r - (int64_t)b * Nout);
        } else {
            const int code = __ldg(c.ridx + r);
            const int gq = code >> 5;
            t1 = code & 31;
            b = gq / Nout;
            q = gq - b * Nout;
        }
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        int idx[KMAX];                         // input row per tap, -1 = zero
#pragma unroll
        for (int tap = 0; tap < KMAX; tap++) {
            idx[tap] = -1;
            if (tap < ntaps) {
                const int dy = tap / g.kw, dx = tap - dy * g.kw;
                const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                    const int64_t bp = (int64_t)b * Nin + iy * g.Win + ix;
                    if (c.dense) {
                        idx[tap] = (int)bp;
                    } else {
                        const int row = row_of(c.a, bp, t1);
                        if (row) idx[tap] = row;
                    }
                }
            }
        }
        for (int cb = 0; cb < C; cb += G * CPL) {
            const int c0 = cb + lane * CPL;
            const bool full = (C % 8 == 0) && (c0 + CPL <= C);
            float acc[CPL];
#pragma unroll
            for (int i = 0; i < CPL; i++) acc[i] = 0.0f;
#pragma unroll
            for (int t0 = 0; t0 < KMAX; t0 += TB) {
                float v[TB][CPL];
#pragma unroll
                for (int j = 0; j < TB; j++)
                    if (t0 + j < KMAX && idx[t0 + j] >= 0)
                        row_load<T, CPL>(A + (int64_t)idx[t0 + j] * C, c0, C, full, v[j]);
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    if (t0 + j >= KMAX || idx[t0 + j] < 0) continue;
                    float w[CPL];
                    row_load<float, CPL>(c.wk + (int64_t)(t0 + j) * C, c0, C, full, w);
#pragma unroll
                    for (int i = 0; i < CPL; i++) acc[i] = fmaf(w[i], v[j][i], acc[i]);
                }
            }
            if (c0 >= C) continue;
            if (c.dense) {
                float bb[CPL];
                row_load<float, CPL>(c.bias, c0, C, full, bb);
#pragma unroll
                for (int i = 0; i < CPL; i++) acc[i] = __fadd_rn(acc[i], bb[i]);
                row_store<float, CPL>(static_cast<float *>(c.out) + r * C, c0, C, full, acc);
            } else {
                row_store<T, CPL>(static_cast<T *>(c.out) + (r + 1) * C, c0, C, full, acc);
            }
        }
    }
}

// Sparse mode, pixel-major: one group per OUTPUT PIXEL.  Its output rows are
// its active frames, consecutive in the (b, p, t) row order (base = 1 +
// out_pbase, j-th set bit -> row base + j), and every tap's frame word,
// slot word and row base are read once per pixel instead of once per
// (output row, tap); per frame the active taps' rows are loaded in a batch.
// The tap metadata (frame word, slot word, row base) is gathered by the
// group's lanes in parallel (lane j: taps j, j+G, ...) into shared memory,
// then read back as one 16-byte broadcast per tap, so 5x5 kernels keep the
// register budget of two CTAs per SM.
template <int G, int CPL, int KMAX, class T>
__global__ void __launch_bounds__(256, 2) k_dwconv_pm(ConvCall c, const uint32_t *__restrict__ out_act,
                                                      const int32_t *__restrict__ out_pbase) {
    constexpr int TB = KMAX > 9 ? 5 : 3;
    extern __shared__ int4 dw_meta[];   // [256/G groups][KMAX] {act, slot, 1 + pbase, 0}
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int C = g.Cin;
    const int lane = threadIdx.x & (G - 1);
    const uint32_t gmask = G == 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    int4 *meta = dw_meta + (threadIdx.x / G) * KMAX;
    const int64_t BNo = (int64_t)c.B * Nout;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const int ntaps = g.kh * g.kw;
    const T *A = static_cast<const T *>(c.a.rows);
    T *O = static_cast<T *>(c.out);
    for (int64_t bq = grp; bq < BNo; bq += ngrp) {
        uint32_t w = __ldg(out_act + bq);
        if (!w) continue;
        const int b = (int)(bq / Nout), q = (int)(bq - (int64_t)b * Nout);
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        __syncwarp(gmask);   // previous pixel's metadata fully consumed
        for (int tap = lane; tap < KMAX; tap += G) {
            int4 m = make_int4(0, 0, 0, 0);
            if (tap < ntaps) {
                const int dy = tap / g.kw, dx = tap - dy * g.kw;
                const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                    const int64_t bp = (int64_t)b * Nin + iy * g.Win + ix;
                    m.x = (int)__ldg(c.a.act + bp);
                    m.y = (int)__ldg(c.a.slot + bp);
                    m.z = 1 + __ldg(c.a.pbase + bp);
                }
            }
            meta[tap] = m;
        }
        __syncwarp(gmask);
        int64_t orow = 1 + __ldg(out_pbase + bq);
        while (w) {
            const int t1 = __ffs(w) - 1;
            w &= w - 1;
            const uint32_t lm = lowmask(t1);
            for (int cb = 0; cb < C; cb += G * CPL) {
                const int c0 = cb + lane * CPL;
                const bool full = (C % 8 == 0) && (c0 + CPL <= C);
                float acc[CPL];
#pragma unroll
                for (int i = 0; i < CPL; i++) acc[i] = 0.0f;
#pragma unroll
                for (int t0 = 0; t0 < KMAX; t0 += TB) {
                    float v[TB][CPL];
                    bool on[TB];
#pragma unroll
                    for (int j = 0; j < TB; j++) {
                        const int tap = t0 + j;
                        on[j] = false;
                        if (tap < KMAX) {
                            const int4 m = meta[tap];
                            on[j] = ((uint32_t)m.x >> t1) & 1u;
                            if (on[j]) {
                                const int64_t row = m.z + __popc((uint32_t)m.y & lm);
                                row_load<T, CPL>(A + row * C, c0, C, full, v[j]);
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < TB; j++) {
                        if (!on[j]) continue;
                        float wv[CPL];
                        row_load<float, CPL>(c.wk + (int64_t)(t0 + j) * C, c0, C, full, wv);
#pragma unroll
                        for (int i = 0; i < CPL; i++) acc[i] = fmaf(wv[i], v[j][i], acc[i]);
                    }
                }
                if (c0 < C) row_store<T, CPL>(O + orow * C, c0, C, full, acc);
            }
            orow++;
        }
    }
}

// lanes per row: 8 channels per lane when C % 8 == 0 (G*8 channels per chunk)
#define DW_SHAPE(C_, L)                                            \
    if ((C_) % 8 != 0) {                                           \
        if ((C_) <= 1) { L(1, 1); }                                \
        else if ((C_) <= 2) { L(2, 1); }                           \
        else if ((C_) <= 4) { L(4, 1); }                           \
        else if ((C_) <= 8) { L(8, 1); }                           \
        else if ((C_) <= 16) { L(16, 1); }                         \
        else { L(32, 1); }                                         \
    } else if ((C_) <= 8) { L(1, 8); }                             \
    else if ((C_) <= 16) { L(2, 8); }                              \
    else if ((C_) <= 32) { L(4, 8); }                              \
    else if ((C_) <= 64) { L(8, 8); }                              \
    else if ((C_) <= 128) { L(16, 8); }                            \
    else { L(32, 8); }

template <class T>
static void launch_dw_t(const ConvCall &c, cudaStream_t s) {
    const int64_t m_up = c.dense ? (int64_t)c.B * c.g.Hout * c.g.Wout : c.m_cap;
    const int kk = c.g.kh * c.g.kw;
    auto grid_for = [&](int G) {
        return (int)std::max<int64_t>(1, std::min<int64_t>((m_up * G + 255) / 256, 148 * 16));
    };
#define L_DW(G_, CPL_)                                                                   \
    {                                                                                    \
        if (kk <= 9) k_dwconv<G_, CPL_, 9, T><<<grid_for(G_), 256, 0, s>>>(c);           \
        else k_dwconv<G_, CPL_, 25, T><<<grid_for(G_), 256, 0, s>>>(c);                  \
    }
    DW_SHAPE(c.g.Cin, L_DW);
#undef L_DW
}

void launch_dwconv_f32(const ConvCall &c, cudaStream_t s) {
    if (c.dense || !c.bf) launch_dw_t<float>(c, s);
    else launch_dw_t<bf16>(c, s);
}

template <int G, int CPL, int KMAX, class T>
static void launch_dw_pm_k(const ConvCall &c, const uint32_t *out_act, const int32_t *out_pbase, int64_t BNo,
                           cudaStream_t s) {
    constexpr int smem = (256 / G) * KMAX * 16;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dwconv_pm<G, CPL, KMAX, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((BNo * G + 255) / 256, 148 * 16));
    k_dwconv_pm<G, CPL, KMAX, T><<<grid, 256, smem, s>>>(c, out_act, out_pbase);
}

template <class T>
static void launch_dw_pm_t(const ConvCall &c, const uint32_t *out_act, const int32_t *out_pbase, cudaStream_t s) {
    const int64_t BNo = (int64_t)c.B * c.g.Hout * c.g.Wout;
    const int kk = c.g.kh * c.g.kw;
#define L_DWPM(G_, CPL_)                                                                 \
    {                                                                                    \
        if (kk <= 9) launch_dw_pm_k<G_, CPL_, 9, T>(c, out_act, out_pbase, BNo, s);      \
        else launch_dw_pm_k<G_, CPL_, 25, T>(c, out_act, out_pbase, BNo, s);             \
    }
    DW_SHAPE(c.g.Cin, L_DWPM);
#undef L_DWPM
}

void launch_dwconv_pm(const ConvCall &c, const uint32_t *out_act, const int32_t *out_pbase, cudaStream_t s) {
    if (!c.bf) launch_dw_pm_t<float>(c, out_act, out_pbase, s);
    else launch_dw_pm_t<bf16>(c, out_act, out_pbase, s);
}

}  // namespace st
