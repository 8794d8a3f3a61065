// kernels_conv.cu -- convolution on compacted deltas and the
// dense reference-frame convolution (a1) on CUDA cores.
//
// Eq.(2): Delta_out = W x Delta_in, bias absent (R5).
// As an implicit GEMM: M = output rows (sparse: the dilated output mask's
// (b, q, t) rows from `ridx`; dense: every reference pixel), N = c_out,
// K = k_h*k_w*c_in in the fixed order (dy, dx, ci) (reading R18).  Each
// output is one thread's sequential fmaf chain over K starting from +0.0f,
// so FP32-mode results are bit-identical to the oracle; inactive taps read
// nothing (fma(w, 0, acc) == acc, so skipping them is exact).  Used for every
// conv in FP32 mode and, in BF16 mode, for convs the tensor-core kernel does
// not take (small c_in such as the stems); delta rows are of type T (fp32 or
// bf16; bf16 rows are exact fp32 values, outputs are rounded on store).
//
// Tile: 128 rows x BN cols x 8 k, 256 threads, 8 x (BN/16) outputs per
// thread, register-prefetched double-buffered shared memory; per M tile a
// shared-memory table holds the gathered input row of every (row, tap).
// Persistent grid: each CTA strides over tiles, the sparse M is read from
// device memory (no host sync inside a step).
#include "common.cuh"

namespace st {

constexpr int CBM = 128, CBK = 8, CNT = 256, CAPAD = 4;

template <int BN, bool CINV, class T>
__global__ void __launch_bounds__(CNT, 2) k_conv_f32(ConvCall c) {
    st_pdl_enter();
    constexpr int TN = BN / 16;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float *As = reinterpret_cast<float *>(smem_raw);                 // [2][CBK][CBM+CAPAD]
    float *Bs = As + 2 * CBK * (CBM + CAPAD);                         // [2][CBK][BN]
    int *tab = reinterpret_cast<int *>(Bs + 2 * CBK * BN);             // [CBM][ntaps]

    const Geo g = c.g;
    const int ntaps = g.kh * g.kw;
    const int K = ntaps * g.Cin;
    const int Nin = g.Hin * g.Win, Nout = g.Hout * g.Wout;
    const int M = c.dense ? c.B * Nout : *c.m_dev;
    const int ntn = (g.Cout + BN - 1) / BN;
    const int ntiles = ((M + CBM - 1) / CBM) * ntn;
    // dense launches are instantiated with T = float
    // sparse mode reads either the compacted rows (via the frame-word lookup)
    // or, for convs on the network input, the dense per-frame delta
    const bool dd = !c.dense && c.ddelta != nullptr;
    const T *A = c.dense ? reinterpret_cast<const T *>(c.a_dense)
                         : dd ? static_cast<const T *>(c.ddelta) : static_cast<const T *>(c.a.rows);
    const int astride = dd ? 4 : g.Cin;   // ddelta pixels are padded to 4 channels
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const bool bvec = (g.Cout & 3) == 0;
    const int nk = (K + CBK - 1) / CBK;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int mt = tile / ntn, nt = tile % ntn;
        const int m0 = mt * CBM, n0 = nt * BN;
        __syncthreads();   // previous tile done with tab / smem
        // ---- gather table: input row of every (output row, tap), -1 = zero
        for (int i = tid; i < CBM * ntaps; i += CNT) {
            const int m = i / ntaps, tap = i - m * ntaps;
            const int r = m0 + m;
            int idx = -1;
            if (r < M && c.rowmap) {   // 1x1/s1 in the input's row layout
                idx = r + 1;
            } else if (r < M) {
                int b, q, t1 = 0;
                if (c.dense) {
                    b = r / Nout;
                    q = r - b * Nout;
                } else {
                    const int code = __ldg(c.ridx + r);
                    const int gq = code >> 5;
                    t1 = code & 31;
                    b = gq / Nout;
                    q = gq - b * Nout;
                }
                const int oy = q / g.Wout, ox = q - oy * g.Wout;
                const int dy = tap / g.kw, dx = tap - dy * g.kw;
                const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                    const int64_t bp = (int64_t)b * Nin + iy * g.Win + ix;
                    if (c.dense) {
                        idx = (int)bp;
                    } else if (dd) {   // zeros where the input was truncated: no lookup
                        // (4-channel-padded pixel pieces: element offset = idx * 4)
                        idx = (int)(((int64_t)b * c.F + t1) * Nin + iy * g.Win + ix);
                    } else {
                        const int row = row_of(c.a, bp, t1);
                        idx = row ? row : -1;
                    }
                }
            }
            tab[i] = idx;
        }
        __syncthreads();

        float acc[8][TN];
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
            for (int j = 0; j < TN; j++) acc[i][j] = 0.0f;

        float ra[4];     // A prefetch registers
        float4 rb;       // B prefetch
        auto load_tile = [&](int k0) {
            if (CINV) {
                // whole k-tile inside one tap: 8 contiguous channels per row
                const int tap = k0 / g.Cin, ci0 = k0 - tap * g.Cin;
                const int m = tid >> 1, half = tid & 1;
                const int idx = tab[m * ntaps + tap];
                if (idx >= 0) {
                    const float4 v = ld4<T>(A + (int64_t)idx * astride + ci0 + half * 4);
                    ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
                } else {
                    ra[0] = ra[1] = ra[2] = ra[3] = 0.0f;
                }
                if (c.rnd_a)
#pragma unroll
                    for (int j = 0; j < 4; j++) ra[j] = bf16_round(ra[j]);
            } else {
                const int kk = tid & 7;
                const int k = k0 + kk;
                const int tap = k / g.Cin, ci = k - tap * g.Cin;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int m = (tid >> 3) + 32 * j;
                    float v = 0.0f;
                    if (k < K) {
                        const int idx = tab[m * ntaps + tap];
                        if (idx >= 0) v = ldr<T>(A + (int64_t)idx * astride + ci);
                    }
                    ra[j] = c.rnd_a ? bf16_round(v) : v;
                }
            }
            // B: [K][Cout]
            constexpr int NV = CBK * BN / 4;   // float4 per tile
            rb = make_float4(0.f, 0.f, 0.f, 0.f);
            if (tid < NV) {
                const int kk = tid / (BN / 4), n4 = tid - kk * (BN / 4);
                const int k = k0 + kk, n = n0 + n4 * 4;
                if (k < K) {
                    const float *wp = c.wk + (int64_t)k * g.Cout + n;
                    if (bvec && n + 3 < g.Cout) {
                        rb = __ldg(reinterpret_cast<const float4 *>(wp));
                    } else {
                        if (n < g.Cout) rb.x = __ldg(wp);
                        if (n + 1 < g.Cout) rb.y = __ldg(wp + 1);
                        if (n + 2 < g.Cout) rb.z = __ldg(wp + 2);
                        if (n + 3 < g.Cout) rb.w = __ldg(wp + 3);
                    }
                }
            }
        };
        auto store_tile = [&](int buf) {
            float *as = As + buf * CBK * (CBM + CAPAD);
            if (CINV) {
                const int m = tid >> 1, half = tid & 1;
#pragma unroll
                for (int j = 0; j < 4; j++) as[(half * 4 + j) * (CBM + CAPAD) + m] = ra[j];
            } else {
                const int kk = tid & 7;
#pragma unroll
                for (int j = 0; j < 4; j++) as[kk * (CBM + CAPAD) + (tid >> 3) + 32 * j] = ra[j];
            }
            constexpr int NV = CBK * BN / 4;
            if (tid < NV) {
                const int kk = tid / (BN / 4), n4 = tid - kk * (BN / 4);
                *reinterpret_cast<float4 *>(Bs + buf * CBK * BN + kk * BN + n4 * 4) = rb;
            }
        };

        load_tile(0);
        store_tile(0);
        __syncthreads();
        for (int kt = 0; kt < nk; kt++) {
            const int cur = kt & 1;
            if (kt + 1 < nk) load_tile((kt + 1) * CBK);
            const float *as = As + cur * CBK * (CBM + CAPAD);
            const float *bs = Bs + cur * CBK * BN;
#pragma unroll
            for (int kk = 0; kk < CBK; kk++) {
                float a[8], b[TN];
                const float4 a0 = *reinterpret_cast<const float4 *>(as + kk * (CBM + CAPAD) + ty * 8);
                const float4 a1 = *reinterpret_cast<const float4 *>(as + kk * (CBM + CAPAD) + ty * 8 + 4);
                a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
                a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
#pragma unroll
                for (int j = 0; j < TN; j += 2) {
                    const float2 bv = *reinterpret_cast<const float2 *>(bs + kk * BN + tx * TN + j);
                    b[j] = bv.x;
                    b[j + 1] = bv.y;
                }
#pragma unroll
                for (int i = 0; i < 8; i++)
#pragma unroll
                    for (int j = 0; j < TN; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
            }
            if (kt + 1 < nk) store_tile(cur ^ 1);
            __syncthreads();
        }

        // ---- epilogue
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int r = m0 + ty * 8 + i;
            if (r >= M) continue;
            if (c.dense) {
                float *o = static_cast<float *>(c.out) + (int64_t)r * g.Cout;
#pragma unroll
                for (int j = 0; j < TN; j++) {
                    const int n = n0 + tx * TN + j;
                    if (n < g.Cout) {
                        const float x = __fadd_rn(acc[i][j], __ldg(c.bias + n));
                        o[n] = x;
                        if (c.act_out) {   // the consuming site's dense output f(x0)
                            const float y = act_rt(c.act_kind, x);
                            c.act_out[(int64_t)r * g.Cout + n] = y;
                            if (c.act_bf) static_cast<bf16 *>(c.act_bf)[(int64_t)r * g.Cout + n] = __float2bfloat16_rn(y);
                        }
                    }
                }
            } else {
                T *o = static_cast<T *>(c.out) + (int64_t)(r + 1) * g.Cout;
#pragma unroll
                for (int j = 0; j < TN; j++) {
                    const int n = n0 + tx * TN + j;
                    if (n < g.Cout) str<T>(o + n, acc[i][j]);
                }
            }
        }
    }
}

template <int BN, bool CINV, class T>
static void launch_one(const ConvCall &c, cudaStream_t s) {
    const int ntaps = c.g.kh * c.g.kw;
    const size_t smem = (2 * CBK * (CBM + CAPAD) + 2 * CBK * BN) * sizeof(float) + CBM * ntaps * sizeof(int);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_conv_f32<BN, CINV, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr_set = true;
    }
    const int ntn = (c.g.Cout + BN - 1) / BN;
    const int64_t m_up = c.dense ? (int64_t)c.B * c.g.Hout * c.g.Wout : c.m_cap;
    int64_t tiles = ((m_up + CBM - 1) / CBM) * ntn;
    int grid = (int)(tiles < 148 * 2 ? tiles : 148 * 2);
    if (grid < 1) grid = 1;
    k_conv_f32<BN, CINV, T><<<grid, CNT, smem, s>>>(c);
}

template <class T>
static void launch_conv_t(const ConvCall &c, cudaStream_t s) {
    const bool cinv = (c.g.Cin % CBK) == 0;
    if (c.g.Cout > 64) {
        cinv ? launch_one<128, true, T>(c, s) : launch_one<128, false, T>(c, s);
    } else if (c.g.Cout > 32) {
        cinv ? launch_one<64, true, T>(c, s) : launch_one<64, false, T>(c, s);
    } else {
        cinv ? launch_one<32, true, T>(c, s) : launch_one<32, false, T>(c, s);
    }
}

void launch_conv_f32(const ConvCall &c, cudaStream_t s) {
    if (c.dense || !c.bf) launch_conv_t<float>(c, s);
    else launch_conv_t<bf16>(c, s);
}

}  // namespace st
