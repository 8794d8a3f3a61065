// kernels_se.cu -- squeeze-excitation site (EfficientNet blocks), sm_100a.
//
// The paper is silent on SE (SPEC excludes it); reading R8
// (DESIGN.md): the gate s = sigmoid(W2 silu(W1 mean(x) + b1) + b2) depends
// on the mean over ALL pixels, so per diff frame t
//   mean_t = (sum over pixels of x0 + sum_{t' <= t} sum over rows of Delta_t') / N
//   s_t    = gate(mean_t)
//   refresh iff max_c |s_t - s_emit| > theta_site  (then s_emit = s_t and every
//          pixel is touched at t), else the touched set is the input mask;
//   on touched pixels: c = x_acc * s_emit - y_acc, truncate, y_acc += c.
// Kernels: (i) fp64 channel sums of the reference activations and of every
// frame's delta rows; (ii) one CTA per chunk runs the sequential gate
// schedule (frames are sequential, channels parallel); (iii) the pixel loop
// with x_acc / y_acc in registers, like the pointwise site.
#include <math_constants.h>

#include "common.cuh"

namespace st {

// ---- (i-a) dense channel sums: sums[b][c] += sum_p x[b][p][c]  (fp64)
__global__ void __launch_bounds__(256) k_se_colsum(const float *__restrict__ x, int N, int C, int ppb,
                                                   double *__restrict__ sums) {
    const int b = blockIdx.z, c = blockIdx.y * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
    const int p0 = blockIdx.x * ppb;
    const int p1 = min(N, p0 + ppb);
    double acc = 0.0;
    if (c < C)
        for (int p = p0 + w; p < p1; p += 8) acc += (double)__ldg(x + ((int64_t)b * N + p) * C + c);
    __shared__ double red[8][32];
    red[w][threadIdx.x & 31] = acc;
    __syncthreads();
    if (w == 0 && c < C) {
        double s = 0.0;
        for (int i = 0; i < 8; i++) s += red[i][threadIdx.x];
        atomicAdd(sums + (int64_t)b * C + c, s);
    }
}

// ---- (i-b) per-frame channel sums of the delta rows: dsum[b][t][c] (fp64)
template <class T>
__global__ void __launch_bounds__(256) k_se_delta_sums(DView in, int N, int C, int F, int ppb,
                                                       double *__restrict__ dsum) {
    extern __shared__ double sacc[];   // [8 warps][32 frames][32 lanes]
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.y * 32 + lane;
    double *my = sacc + w * 32 * 32;
    for (int t = 0; t < 32; t++) my[t * 32 + lane] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    for (int p = p0 + w; p < p1; p += 8) {
        const int64_t bp = (int64_t)b * N + p;
        uint32_t a = __ldg(in.act + bp);
        if (!a) continue;
        const int base = 1 + __ldg(in.pbase + bp);
        const uint32_t sl = __ldg(in.slot + bp);
        while (a) {
            const int t1 = __ffs(a) - 1;
            a &= a - 1;
            const int64_t row = base + __popc(sl & lowmask(t1));
            if (c < C) my[t1 * 32 + lane] += (double)ldr<T>(rows + row * C + c);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
        const int t1 = i >> 5, l = i & 31, cc = blockIdx.y * 32 + l;
        if (t1 >= F || cc >= C) continue;
        double s = 0.0;
        for (int ww = 0; ww < 8; ww++) s += sacc[ww * 1024 + i];
        if (s != 0.0) atomicAdd(dsum + ((int64_t)b * F + t1) * C + cc, s);
    }
}

// gate of one chunk from fp32 means m[C] (block-wide; hid/gate in smem)
__device__ void se_gate_block(const float *m, int C, int H, const float *w1, const float *b1, const float *w2,
                              const float *b2, float *hid, float *gate) {
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        float acc = 0.0f;
        for (int c = 0; c < C; c++) acc = fmaf(__ldg(w1 + (int64_t)j * C + c), m[c], acc);
        hid[j] = silu_f(__fadd_rn(acc, __ldg(b1 + j)));
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float acc = 0.0f;
        for (int j = 0; j < H; j++) acc = fmaf(__ldg(w2 + (int64_t)c * H + j), hid[j], acc);
        gate[c] = sigm_f(__fadd_rn(acc, __ldg(b2 + c)));
    }
    __syncthreads();
}

// ---- (ii) gate schedule, one CTA per chunk.  s_tab[b][t][c] = s_emit in
// force at frame t (t = 0: reference gate); refresh[b] bit t-1 = refresh at t.
__global__ void __launch_bounds__(256) k_se_schedule(const double *__restrict__ sum0, const double *__restrict__ dsum,
                                                     int N, int C, int H, int F, const float *w1, const float *b1,
                                                     const float *w2, const float *b2,
                                                     const float *__restrict__ theta_p,
                                                     float *__restrict__ s_tab, uint32_t *__restrict__ refresh) {
    const float theta = __ldg(theta_p);
    extern __shared__ float sm[];
    float *mean = sm;            // [C]
    float *gate = mean + C;      // [C]
    float *semit = gate + C;     // [C]
    float *hid = semit + C;      // [H]
    double *run = reinterpret_cast<double *>(
        (reinterpret_cast<uintptr_t>(hid + H) + 7) & ~uintptr_t(7));   // [C], 8-byte aligned
    __shared__ float red[8];
    __shared__ int do_refresh;
    const int b = blockIdx.x;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        run[c] = sum0[(int64_t)b * C + c];
        mean[c] = (float)(run[c] / (double)N);
    }
    __syncthreads();
    se_gate_block(mean, C, H, w1, b1, w2, b2, hid, gate);
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        semit[c] = gate[c];
        s_tab[(int64_t)b * (F + 1) * C + c] = gate[c];
    }
    uint32_t bits = 0;
    for (int t1 = 0; t1 < F; t1++) {
        __syncthreads();
        for (int c = threadIdx.x; c < C; c += blockDim.x) {
            run[c] += dsum[((int64_t)b * F + t1) * C + c];
            mean[c] = (float)(run[c] / (double)N);
        }
        __syncthreads();
        se_gate_block(mean, C, H, w1, b1, w2, b2, hid, gate);
        float mx = 0.0f;
        for (int c = threadIdx.x; c < C; c += blockDim.x) mx = fmaxf(mx, fabsf(__fsub_rn(gate[c], semit[c])));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            float m = 0.0f;
            for (int i = 0; i < (int)(blockDim.x >> 5); i++) m = fmaxf(m, red[i]);
            do_refresh = m > theta;
        }
        __syncthreads();
        if (do_refresh) {
            bits |= 1u << t1;
            for (int c = threadIdx.x; c < C; c += blockDim.x) semit[c] = gate[c];
        }
        __syncthreads();
        for (int c = threadIdx.x; c < C; c += blockDim.x) s_tab[((int64_t)b * (F + 1) + t1 + 1) * C + c] = semit[c];
    }
    if (threadIdx.x == 0) refresh[b] = bits;
}

// dense reference SE: y0 = x0 * s_tab[b][0]
__global__ void k_se_dense_apply(const float *__restrict__ x, const float *__restrict__ s_tab, int N, int C, int F,
                                 int64_t n, float *__restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        const int b = (int)(i / ((int64_t)N * C));
        y[i] = __fmul_rn(x[i], s_tab[(int64_t)b * (F + 1) * C + c]);
    }
}

// slot[b][p] = act[b][p] | refresh[b]
__global__ void k_se_slots(const uint32_t *__restrict__ act, const uint32_t *__restrict__ refresh, int N, int64_t n,
                           uint32_t *__restrict__ slot) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) slot[i] = act[i] | refresh[i / N];
}

// ---- (iii) SE site pixel loop
template <int G, int CPL, class T>
__global__ void __launch_bounds__(256) k_se_site(DView in, const float *__restrict__ x0, const float *__restrict__ s_tab,
                                                 int N, int C, int F, int64_t BN, const float *__restrict__ theta_p,
                                                 const uint32_t *__restrict__ slot, const int32_t *__restrict__ pbase,
                                                 uint32_t *__restrict__ out_act, T *__restrict__ out_rows) {
    const float theta = __ldg(theta_p);
    const T *rows = static_cast<const T *>(in.rows);
    const int lane = threadIdx.x & (G - 1);
    unsigned mask = 0xffffffffu;
    if constexpr (G < 32) mask = ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t bp = grp; bp < BN; bp += ngrp) {
        const uint32_t Tw = __ldg(slot + bp);
        if (!Tw) {
            if (lane == 0) out_act[bp] = 0;
            continue;
        }
        const int b = (int)(bp / N);
        const float *st = s_tab + (int64_t)b * (F + 1) * C;
        const uint32_t a = __ldg(in.act + bp);
        float xa[CPL], ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            const int ch = lane + G * i;
            xa[i] = ch < C ? __ldg(x0 + bp * C + ch) : 0.0f;
            ya[i] = ch < C ? __fmul_rn(xa[i], __ldg(st + ch)) : 0.0f;   // y0 = x0 * s_emit(0)
        }
        const int ibase = a ? 1 + __ldg(in.pbase + bp) : 0;
        const uint32_t isl = a ? __ldg(in.slot + bp) : 0u;
        const int obase = 1 + __ldg(pbase + bp);
        uint32_t bits = Tw, emit = 0;
        while (bits) {
            const int t1 = __ffs(bits) - 1;
            bits &= bits - 1;
            const bool act = (a >> t1) & 1u;
            const int64_t irow = act ? ibase + __popc(isl & lowmask(t1)) : 0;
            const float *s_now = st + (int64_t)(t1 + 1) * C;
            float cand[CPL];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                const int ch = lane + G * i;
                cand[i] = 0.0f;
                if (ch < C) {
                    if (act) xa[i] = __fadd_rn(xa[i], ldr<T>(rows + irow * C + ch));
                    cand[i] = __fsub_rn(__fmul_rn(xa[i], __ldg(s_now + ch)), ya[i]);
                    mx = fmaxf(mx, fabsf(cand[i]));
                }
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(mask, mx, o, G));
            if (mx > theta) {
                const int64_t orow = obase + __popc(Tw & lowmask(t1));
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    const int ch = lane + G * i;
                    if (ch < C) {
                        const float e = rnd<T>(cand[i]);
                        ya[i] = __fadd_rn(ya[i], e);
                        str<T>(out_rows + orow * C + ch, e);
                    }
                }
                emit |= 1u << t1;
            }
        }
        if (lane == 0) out_act[bp] = emit;
    }
}

void launch_se_colsum(const float *x, int B, int N, int C, double *sum0, cudaStream_t s) {
    cudaMemsetAsync(sum0, 0, (size_t)B * C * 8, s);
    const int ppb = 2048;
    dim3 grid(cdiv(N, ppb), cdiv(C, 32), B);
    k_se_colsum<<<grid, 256, 0, s>>>(x, N, C, ppb, sum0);
}

void launch_se_schedule(const double *sum0, const double *dsum, int B, int N, int C, int H, int F, const float *w1,
                        const float *b1, const float *w2, const float *b2, const float *theta, float *s_tab,
                        uint32_t *refresh, cudaStream_t s) {
    const size_t smem = (size_t)(3 * C + ((H + 1) & ~1)) * 4 + (size_t)C * 8 + 64;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_se_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_se_schedule<<<B, 256, smem, s>>>(sum0, dsum, N, C, H, F, w1, b1, w2, b2, theta, s_tab, refresh);
}

void launch_se_dense_apply(const float *x, const float *s_tab, int B, int N, int C, int F, float *y, cudaStream_t s) {
    const int64_t n = (int64_t)B * N * C;
    const int grid = (int)std::min<int64_t>(cdiv(n, 256), 148 * 16);
    if (grid > 0) k_se_dense_apply<<<grid, 256, 0, s>>>(x, s_tab, N, C, F, n, y);
}

template <class T>
static void se_delta_sums_t(DView in, int B, int N, int C, int F, double *dsum, cudaStream_t s) {
    const int ppb = 1024;
    dim3 grid(cdiv(N, ppb), cdiv(C, 32), B);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_se_delta_sums<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 32 * 8);
        attr = true;
    }
    k_se_delta_sums<T><<<grid, 256, 8 * 32 * 32 * 8, s>>>(in, N, C, F, ppb, dsum);
}

void launch_se_delta_sums(DView in, int B, int N, int C, int F, bool bf, double *dsum, cudaStream_t s) {
    cudaMemsetAsync(dsum, 0, (size_t)B * F * C * 8, s);
    if (bf) se_delta_sums_t<bf16>(in, B, N, C, F, dsum, s);
    else se_delta_sums_t<float>(in, B, N, C, F, dsum, s);
}

void launch_se_slots(const uint32_t *act, const uint32_t *refresh, int B, int N, uint32_t *slot, cudaStream_t s) {
    const int64_t n = (int64_t)B * N;
    k_se_slots<<<cdiv(n, 256), 256, 0, s>>>(act, refresh, N, n, slot);
}

void launch_se_site(DView in, const float *x0, const float *s_tab, int B, int N, int C, int F, const float *theta, bool bf,
                    const uint32_t *slot, const int32_t *pbase, uint32_t *out_act, void *out_rows, cudaStream_t s) {
    const int64_t BN = (int64_t)B * N;
    auto grid_for = [&](int G) {
        return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(BN * G, 256), 148 * 8));
    };
#define L_SE(G_, CPL_)                                                                                      \
    k_se_site<G_, CPL_, T><<<grid_for(G_), 256, 0, s>>>(in, x0, s_tab, N, C, F, BN, theta, slot, pbase, out_act, \
                                                        static_cast<T *>(out_rows))
#define SE_CH                          \
    if (C <= 8) L_SE(8, 1);            \
    else if (C <= 16) L_SE(16, 1);     \
    else if (C <= 32) L_SE(32, 1);     \
    else if (C <= 64) L_SE(32, 2);     \
    else if (C <= 96) L_SE(32, 3);     \
    else if (C <= 160) L_SE(32, 5);    \
    else if (C <= 256) L_SE(32, 8);    \
    else if (C <= 480) L_SE(32, 15);   \
    else if (C <= 672) L_SE(32, 21);   \
    else L_SE(32, 36);
    ST_ROW_DISPATCH(bf, SE_CH);
#undef SE_CH
#undef L_SE
}

}  // namespace st
