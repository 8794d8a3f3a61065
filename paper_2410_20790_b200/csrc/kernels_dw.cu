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
#include <cstdlib>
#include <type_traits>

#include "rowio.cuh"

namespace st {

template <int G, int CPL, int KMAX, class T>
__global__ void __launch_bounds__(256, 2) k_dwconv(ConvCall c) {
    st_pdl_enter();
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
                    if (t0 + j < KMAX && idx[t0 + j] >= 0) {
                        row_load<T, CPL>(A + (int64_t)idx[t0 + j] * C, c0, C, full, v[j]);
                        if (c.rnd_a)
#pragma unroll
                            for (int i = 0; i < CPL; i++) v[j][i] = bf16_round(v[j][i]);
                    }
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
                if (c.act_out) {   // the consuming site's dense output f(x0)
#pragma unroll
                    for (int i = 0; i < CPL; i++) acc[i] = act_rt(c.act_kind, acc[i]);
                    row_store<float, CPL>(c.act_out + r * C, c0, C, full, acc);
                    if (c.act_bf) row_store<bf16, CPL>(static_cast<bf16 *>(c.act_bf) + r * C, c0, C, full, acc);
                }
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

// tap metadata of output pixel (b, oy, ox) into meta[tap] = {act, slot, 1 +
// pbase, -}, then the live taps (active in some frame of the step) in
// ascending order into meta[k].w; returns their number
template <int G, int KMAX>
__device__ __forceinline__ int dw_gather_meta(const ConvCall &c, int b, int oy, int ox, int lane, uint32_t gmask,
                                              int4 *meta) {
    const Geo &g = c.g;
    const int Nin = g.Hin * g.Win, ntaps = g.kh * g.kw;
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
    int nlive = 0;
    for (int r = 0; r < KMAX; r += G) {
        const int tap = r + lane;
        const bool live = tap < KMAX && meta[tap].x != 0;
        const uint32_t bal = __ballot_sync(gmask, live) >> ((threadIdx.x & 31) & ~(G - 1));
        if (live) meta[nlive + __popc(bal & ((1u << lane) - 1u))].w = tap;
        nlive += __popc(bal);
    }
    __syncwarp(gmask);
    return nlive;
}

// 8 bf16 channels [c0, c0+8) of a row as one raw 16-byte vector (zeros past C)
__device__ __forceinline__ uint4 dw_load_raw(const bf16 *A, int64_t row, int C, int c0, bool full) {
    if (full) return *reinterpret_cast<const uint4 *>(A + row * C + c0);
    const uint16_t *r16 = reinterpret_cast<const uint16_t *>(A + row * C);
    uint32_t h[8];
#pragma unroll
    for (int i = 0; i < 8; i++) h[i] = c0 + i < C ? r16[c0 + i] : 0u;
    return make_uint4(h[0] | h[1] << 16, h[2] | h[3] << 16, h[4] | h[5] << 16, h[6] | h[7] << 16);
}

// bf16 rows, 8 channels at c0: the depthwise deltas of frames tA and tB (tB <
// 0: none) in one pass over the live taps -- each batch loads the rows of TB
// taps for both frames, kept as raw 16-byte vectors until their FMA (the
// register cost of one frame's float rows), so one round trip serves up to
// 2*TB rows; every frame's chain stays in ascending tap order
template <int TB>
__device__ __forceinline__ void dw_acc_pair(const bf16 *A, const float *wk, int C, int c0, bool full,
                                            const int4 *meta, int nlive, int tA, int tB, float (&accA)[8],
                                            float (&accB)[8]) {
    const uint32_t lmA = lowmask(tA), lmB = tB >= 0 ? lowmask(tB) : 0u;
    const uint32_t fm = (1u << tA) | (tB >= 0 ? 1u << tB : 0u);
#pragma unroll
    for (int i = 0; i < 8; i++) accA[i] = accB[i] = 0.0f;
    int k = 0;
    while (k < nlive) {
        int tp[TB];
        uint4 vA[TB], vB[TB];
        uint32_t on = 0;   // bit 2j: tap j active in frame A, bit 2j+1: in frame B
#pragma unroll
        for (int j = 0; j < TB; j++) {
            tp[j] = -1;
            while (k < nlive) {
                const int tap = meta[k].w;
                k++;
                const int4 m = meta[tap];
                const uint32_t hit = (uint32_t)m.x & fm;
                if (hit) {
                    tp[j] = tap;
                    if ((hit >> tA) & 1u) {
                        vA[j] = dw_load_raw(A, m.z + __popc((uint32_t)m.y & lmA), C, c0, full);
                        on |= 1u << (2 * j);
                    }
                    if (tB >= 0 && ((hit >> tB) & 1u)) {
                        vB[j] = dw_load_raw(A, m.z + __popc((uint32_t)m.y & lmB), C, c0, full);
                        on |= 2u << (2 * j);
                    }
                    break;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < TB; j++) {
            if (tp[j] < 0) continue;
            float wv[8];
            row_load<float, 8>(wk + (int64_t)tp[j] * C, c0, C, full, wv);
            if ((on >> (2 * j)) & 1u) {
                const uint32_t u[4] = {vA[j].x, vA[j].y, vA[j].z, vA[j].w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    accA[2 * q] = fmaf(wv[2 * q], __uint_as_float(u[q] << 16), accA[2 * q]);
                    accA[2 * q + 1] = fmaf(wv[2 * q + 1], __uint_as_float(u[q] & 0xFFFF0000u), accA[2 * q + 1]);
                }
            }
            if ((on >> (2 * j + 1)) & 1u) {
                const uint32_t u[4] = {vB[j].x, vB[j].y, vB[j].z, vB[j].w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    accB[2 * q] = fmaf(wv[2 * q], __uint_as_float(u[q] << 16), accB[2 * q]);
                    accB[2 * q + 1] = fmaf(wv[2 * q + 1], __uint_as_float(u[q] & 0xFFFF0000u), accB[2 * q + 1]);
                }
            }
        }
    }
}

// one frame t1, CPL channels at c0: batches of TB taps ACTIVE in t1 (found by
// walking the live list), loaded together; fmaf chain in ascending tap order
template <int TB, int CPL, class T>
__device__ __forceinline__ void dw_acc_one(const T *A, const float *wk, int C, int c0, bool full, const int4 *meta,
                                           int nlive, int t1, float (&acc)[CPL]) {
    const uint32_t lm = lowmask(t1);
#pragma unroll
    for (int i = 0; i < CPL; i++) acc[i] = 0.0f;
    int k = 0;
    while (k < nlive) {
        int tp[TB];
        float v[TB][CPL];
#pragma unroll
        for (int j = 0; j < TB; j++) {
            tp[j] = -1;
            while (k < nlive) {
                const int tap = meta[k].w;
                k++;
                const int4 m = meta[tap];
                if (((uint32_t)m.x >> t1) & 1u) {
                    tp[j] = tap;
                    const int64_t row = m.z + __popc((uint32_t)m.y & lm);
                    row_load<T, CPL>(A + row * C, c0, C, full, v[j]);
                    break;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < TB; j++) {
            if (tp[j] < 0) continue;
            float wv[CPL];
            row_load<float, CPL>(wk + (int64_t)tp[j] * C, c0, C, full, wv);
#pragma unroll
            for (int i = 0; i < CPL; i++) acc[i] = fmaf(wv[i], v[j][i], acc[i]);
        }
    }
}

template <int G, int CPL, int KMAX, class T>
__global__ void __launch_bounds__(256, 3) k_dwconv_pm(ConvCall c, const uint32_t *__restrict__ out_act,
                                                      const int32_t *__restrict__ out_pbase) {
    st_pdl_enter();
    constexpr int TB = KMAX > 9 ? 4 : 3;   // active taps loaded per batch
    constexpr bool PAIR = sizeof(T) == 2 && CPL == 8;   // two frames per pass (dw_acc_pair)
    extern __shared__ int4 dw_meta[];   // [256/G groups][KMAX] {act, slot, 1 + pbase, live tap}
    const Geo g = c.g;
    const int Nout = g.Wout * g.Hout;
    const int C = g.Cin;
    const int lane = threadIdx.x & (G - 1);
    const uint32_t gmask = group_mask<G>();
    int4 *meta = dw_meta + (threadIdx.x / G) * KMAX;
    const int64_t BNo = (int64_t)c.B * Nout;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const T *A = static_cast<const T *>(c.a.rows);
    T *O = static_cast<T *>(c.out);
    for (int64_t bq = grp; bq < BNo; bq += ngrp) {
        uint32_t w = __ldg(out_act + bq);
        if (!w) continue;
        const int b = (int)(bq / Nout), q = (int)(bq - (int64_t)b * Nout);
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        const int nlive = dw_gather_meta<G, KMAX>(c, b, oy, ox, lane, gmask, meta);
        int64_t orow = 1 + __ldg(out_pbase + bq);
        if constexpr (PAIR) {
            while (w) {
                const int tA = __ffs(w) - 1;
                w &= w - 1;
                const int tB = w ? __ffs(w) - 1 : -1;
                if (w) w &= w - 1;
                for (int cb = 0; cb < C; cb += G * CPL) {
                    const int c0 = cb + lane * CPL;
                    const bool full = c0 + CPL <= C;
                    float accA[8], accB[8];
                    dw_acc_pair<TB>(A, c.wk, C, c0, full, meta, nlive, tA, tB, accA, accB);
                    if (c0 < C) {
                        row_store<T, 8>(O + orow * C, c0, C, full, accA);
                        if (tB >= 0) row_store<T, 8>(O + (orow + 1) * C, c0, C, full, accB);
                    }
                }
                orow += tB >= 0 ? 2 : 1;
            }
        } else {
            while (w) {
                const int t1 = __ffs(w) - 1;
                w &= w - 1;
                for (int cb = 0; cb < C; cb += G * CPL) {
                    const int c0 = cb + lane * CPL;
                    const bool full = (C % 8 == 0) && (c0 + CPL <= C);
                    float acc[CPL];
                    dw_acc_one<TB, CPL, T>(A, c.wk, C, c0, full, meta, nlive, t1, acc);
                    if (c0 < C) row_store<T, CPL>(O + orow * C, c0, C, full, acc);
                }
                orow++;
            }
        }
    }
}

// ---- sparse depthwise + pointwise site in one pass (SURVEY §8(f) N2 for
// depthwise convs; Eq.2 then Eq.3).  The group that owns an
// output pixel computes its delta rows frame by frame in ascending order (as
// k_dwconv_pm), rounds each to the stored row type (the value the separate
// conv kernel would write, R22-BF16) and steps the site right away:
//     x_acc += Delta; c = f(x_acc) - y_acc; emit iff max_c |c| > theta;
//     y_acc += rnd(c)   (the operations of k_site_pw, in its order)
// x_acc starts from the conv's dense reference output x0, y_acc = f(x0).
// The site's emitted rows go to the conv's row layout (the in-place layout of
// the separate site kernel), so the conv's delta rows never reach HBM
// (written only when d.conv_rows is set: debug_retain).  Narrow form: C <=
// G*8, one 8-channel chunk per lane, state in registers.
template <int G, int KMAX, class T, int ACT, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_dwconv_site(ConvCall c, DwSite d) {
    st_pdl_enter();
    constexpr int TB = KMAX > 9 ? 4 : 3;
    constexpr bool PAIR = sizeof(T) == 2;
    extern __shared__ int4 dw_meta[];
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nout = g.Wout * g.Hout;
    const int C = g.Cin;
    const int lane = threadIdx.x & (G - 1);
    const uint32_t gmask = group_mask<G>();
    int4 *meta = dw_meta + (threadIdx.x / G) * KMAX;
    const int64_t BNo = (int64_t)c.B * Nout;
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    const T *A = static_cast<const T *>(c.a.rows);
    T *SR = static_cast<T *>(d.site_rows);
    T *CR = static_cast<T *>(d.conv_rows);
    const int c0 = lane * 8;
    const bool full = c0 + 8 <= C;   // C % 8 == 0: a lane's chunk is whole or past C
    for (int64_t bq = grp; bq < BNo; bq += ngrp) {
        uint32_t w = __ldg(d.out_act + bq);
        if (!w) {
            if (lane == 0) d.site_act[bq] = 0u;
            continue;
        }
        const int b = (int)(bq / Nout), q = (int)(bq - (int64_t)b * Nout);
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        const int nlive = dw_gather_meta<G, KMAX>(c, b, oy, ox, lane, gmask, meta);
        float xa[8], ya[8];
        row_load<float, 8>(d.x0 + bq * C, c0, C, full, xa);
#pragma unroll
        for (int i = 0; i < 8; i++) ya[i] = actf<ACT>(xa[i]);
        uint32_t emit = 0;
        int64_t orow = 1 + __ldg(d.out_pbase + bq);
        auto step = [&](const float (&acc)[8], int64_t row, int t1) {
            float cand[8];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const float v = rnd<T>(acc[i]);                        // the conv's stored delta
                xa[i] = __fadd_rn(xa[i], v);                           // reconstruct x (Eq.3)
                cand[i] = __fsub_rn(actf<ACT>(xa[i]), ya[i]);          // restore the delta
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            if (CR && c0 < C) row_store<T, 8>(CR + row * C, c0, C, full, acc);
            mx = gmax<G>(mx, gmask);
            if (mx > theta) {                                          // truncation
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    cand[i] = rnd<T>(cand[i]);
                    ya[i] = __fadd_rn(ya[i], cand[i]);
                }
                if (c0 < C) row_store<T, 8>(SR + row * C, c0, C, full, cand);
                emit |= 1u << t1;
            } else if (d.zero_gaps && c0 < C) {   // a rowmap conv reads this slot as a row
                const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                row_store<T, 8>(SR + row * C, c0, C, full, z);
            }
        };
        if constexpr (PAIR) {
            while (w) {
                const int tA = __ffs(w) - 1;
                w &= w - 1;
                const int tB = w ? __ffs(w) - 1 : -1;
                if (w) w &= w - 1;
                float accA[8], accB[8];
                dw_acc_pair<TB>(reinterpret_cast<const bf16 *>(A), c.wk, C, c0, full, meta, nlive, tA, tB, accA, accB);
                step(accA, orow, tA);
                if (tB >= 0) step(accB, orow + 1, tB);
                orow += tB >= 0 ? 2 : 1;
            }
        } else {
            while (w) {
                const int t1 = __ffs(w) - 1;
                w &= w - 1;
                float acc[8];
                dw_acc_one<TB, 8, T>(A, c.wk, C, c0, full, meta, nlive, t1, acc);
                step(acc, orow, t1);
                orow++;
            }
        }
        if (lane == 0) d.site_act[bq] = emit;
    }
}

// Warp form (C <= 256; ST_DW_TEAM=0 -- the team form in kernels_dw_team.cu is the
// default): ONE WARP PER OUTPUT PIXEL, lane l owns
// channels l, l+32, ... (CPL = ceil(C/32)), so every warp's control flow --
// the frame loop, the live-tap walk, the emit decision -- is uniform (ncu on
// the 8-pixels-per-warp form: 2.3 G instructions for one 540x960x32 layer,
// issue-bound with 15 % branch-resolving stalls from the divergent per-pixel
// loops).  Lane t < k*k holds tap t's metadata {frame word, slot word, row
// base} in registers; the row indices of a frame pair are computed by their
// owner lanes and broadcast by shuffles, and the rows of up to TB active taps
// x 2 frames are loaded (coalesced: the warp reads 64 contiguous bytes per
// load instruction) before their FMAs.  Depthwise weights are staged in
// shared memory once per CTA.  Per channel the fmaf chain runs over the taps
// in ascending order from +0 (FP32 bit-exact), then the site step of
// k_site_pw (x_acc += rnd(Delta); c = f(x_acc) - y_acc; warp max; emit).
constexpr int DWW_WARPS = 8;
template <int CPL, int KMAX, class T, int ACT>
__global__ void __launch_bounds__(32 * DWW_WARPS) k_dwconv_site_w(ConvCall c, DwSite d) {
    st_pdl_enter();
    constexpr int TB = CPL == 1 ? 9 : CPL <= 2 ? 6 : CPL <= 4 ? 4 : 2;   // active taps per load batch
    extern __shared__ float dww_w[];   // [KMAX][C] depthwise weights
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int C = g.Cin, ntaps = g.kh * g.kw;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < ntaps * C; i += blockDim.x) dww_w[i] = __ldg(c.wk + i);
    __syncthreads();
    const int64_t BNo = (int64_t)c.B * Nout;
    const T *A = static_cast<const T *>(c.a.rows);
    T *SR = static_cast<T *>(d.site_rows);
    T *CR = static_cast<T *>(d.conv_rows);
    // this lane's tap geometry (fixed)
    const int tdy = lane < ntaps ? lane / g.kw : 0, tdx = lane < ntaps ? lane - tdy * g.kw : 0;
    // strided pixels per warp (active pixels cluster in space: contiguous
    // chunks per warp were measured 2-3x slower from load imbalance); the tap
    // metadata and x0 of the warp's next pixel are loaded while the current
    // one is computed
    uint32_t ma = 0, ms = 0, n_ma = 0, n_ms = 0, n_w = 0;
    int mz = 0, n_mz = 0;
    float xa[CPL], ya[CPL], n_x[CPL];
    auto fetch = [&](int64_t bq) {   // frame word; tap lanes: {act, slot, 1 + pbase}; x0 row
        n_w = 0;
        n_ma = n_ms = 0;
        n_mz = 0;
        if (bq >= BNo) return;
        n_w = __ldg(d.out_act + bq);
        if (!n_w) return;
        const int b = (int)(bq / Nout), q = (int)(bq - (int64_t)b * Nout);
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        if (lane < ntaps) {
            const int iy = oy * g.sh - g.ph + tdy, ix = ox * g.sw - g.pw + tdx;
            if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                const int64_t bp = (int64_t)b * Nin + iy * g.Win + ix;
                n_ma = __ldg(c.a.act + bp);
                n_ms = __ldg(c.a.slot + bp);
                n_mz = 1 + __ldg(c.a.pbase + bp);
            }
        }
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            const int ch = lane + 32 * i;
            n_x[i] = ch < C ? __ldg(d.x0 + bq * C + ch) : 0.0f;
        }
    };
    const int64_t stride = (int64_t)gridDim.x * DWW_WARPS;
    int64_t bq = (int64_t)blockIdx.x * DWW_WARPS + wid;
    fetch(bq);
    for (; bq < BNo; bq += stride) {
        uint32_t w = n_w;
        ma = n_ma;
        ms = n_ms;
        mz = n_mz;
#pragma unroll
        for (int i = 0; i < CPL; i++) xa[i] = n_x[i];
        fetch(bq + stride);   // the next pixel's loads in flight
        if (!w) {
            if (lane == 0) d.site_act[bq] = 0u;
            continue;
        }
#pragma unroll
        for (int i = 0; i < CPL; i++) ya[i] = actf<ACT>(xa[i]);
        uint32_t emit = 0;
        int64_t orow = 1 + __ldg(d.out_pbase + bq);
        auto step = [&](const float (&acc)[CPL], int64_t row, int t1) {
            float cand[CPL];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                const float v = rnd<T>(acc[i]);                    // the conv's stored delta
                xa[i] = __fadd_rn(xa[i], v);                       // reconstruct x (Eq.3)
                cand[i] = __fsub_rn(actf<ACT>(xa[i]), ya[i]);      // restore the delta
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            if (CR)
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) str<T>(CR + row * C + lane + 32 * i, acc[i]);
            mx = gmax<32>(mx, 0xffffffffu);
            if (mx > theta) {                                      // truncation
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    cand[i] = rnd<T>(cand[i]);
                    ya[i] = __fadd_rn(ya[i], cand[i]);
                    if (lane + 32 * i < C) str<T>(SR + row * C + lane + 32 * i, cand[i]);
                }
                emit |= 1u << t1;
            } else if (d.zero_gaps) {                              // a rowmap conv reads this slot as a row
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) str<T>(SR + row * C + lane + 32 * i, 0.0f);
            }
        };
        while (w) {
            const int tA = __ffs(w) - 1;
            w &= w - 1;
            const int tB = w ? __ffs(w) - 1 : -1;
            if (w) w &= w - 1;
            // tap lanes: hit bits and row indices of both frames
            const bool hA = (ma >> tA) & 1u, hB = tB >= 0 && ((ma >> tB) & 1u);
            const int rA = mz + __popc(ms & lowmask(tA)), rB = tB >= 0 ? mz + __popc(ms & lowmask(tB)) : 0;
            uint32_t todo = __ballot_sync(0xffffffffu, hA || hB);   // taps active in A or B, ascending
            const uint32_t bA = __ballot_sync(0xffffffffu, hA), bB = __ballot_sync(0xffffffffu, hB);
            float accA[CPL], accB[CPL];
#pragma unroll
            for (int i = 0; i < CPL; i++) accA[i] = accB[i] = 0.0f;
            while (todo) {
                int tp[TB];
                float vA[TB][CPL], vB[TB][CPL];
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    tp[j] = todo ? __ffs(todo) - 1 : -1;
                    if (todo) todo &= todo - 1;
                    const int t = tp[j] < 0 ? 0 : tp[j];
                    const int64_t ra = __shfl_sync(0xffffffffu, rA, t), rb = __shfl_sync(0xffffffffu, rB, t);
                    const bool ia = tp[j] >= 0 && ((bA >> t) & 1u), ib = tp[j] >= 0 && ((bB >> t) & 1u);
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        const int ch = lane + 32 * i;
                        vA[j][i] = (ia && ch < C) ? ldr<T>(A + ra * C + ch) : 0.0f;
                        vB[j][i] = (ib && ch < C) ? ldr<T>(A + rb * C + ch) : 0.0f;
                    }
                }
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    if (tp[j] < 0) continue;
                    const bool ia = (bA >> tp[j]) & 1u, ib = (bB >> tp[j]) & 1u;
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        const int ch = lane + 32 * i;
                        const float wv = ch < C ? dww_w[tp[j] * C + ch] : 0.0f;
                        if (ia) accA[i] = fmaf(wv, vA[j][i], accA[i]);
                        if (ib) accB[i] = fmaf(wv, vB[j][i], accB[i]);
                    }
                }
            }
            step(accA, orow, tA);
            if (tB >= 0) step(accB, orow + 1, tB);
            orow += tB >= 0 ? 2 : 1;
        }
        if (lane == 0) d.site_act[bq] = emit;
    }
}

// Wide form (C > 256): one warp per output pixel, the pixel's x_acc / y_acc
// (and, for the second frame of a bf16 pair, its stored delta) in shared
// memory, walked in 256-channel chunks.  Per frame: pass 1 adds the delta to
// x_acc and takes the running max of |f(x_acc) - y_acc|; on emission pass 2
// recomputes the candidate from the stored state (the same operations, so
// the same bits), rounds it, advances y_acc and writes the row.
constexpr int DWS_WARPS = 8;
template <int KMAX, class T, int ACT>
__global__ void __launch_bounds__(32 * DWS_WARPS, 2) k_dwconv_site_wide(ConvCall c, DwSite d) {
    st_pdl_enter();
    constexpr int TB = KMAX > 9 ? 4 : 3;
    constexpr bool PAIR = sizeof(T) == 2;
    extern __shared__ int4 dw_meta[];   // [warps][KMAX] metadata, then [warps][3][C] fp32 state
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nout = g.Wout * g.Hout;
    const int C = g.Cin;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int4 *meta = dw_meta + wid * KMAX;
    float *xs = reinterpret_cast<float *>(dw_meta + DWS_WARPS * KMAX) + (size_t)wid * 3 * C;
    float *ys = xs + C, *bs = ys + C;
    const int64_t BNo = (int64_t)c.B * Nout;
    const T *A = static_cast<const T *>(c.a.rows);
    T *SR = static_cast<T *>(d.site_rows);
    T *CR = static_cast<T *>(d.conv_rows);
    // pass 2 of one frame: the emitted row from the stored state
    auto emit_row = [&](int64_t row) {
        for (int c0 = lane * 8; c0 < C; c0 += 256) {
            float x[8], y[8], cand[8];
            RowIO<float, 8>::load(xs + c0, x);
            RowIO<float, 8>::load(ys + c0, y);
#pragma unroll
            for (int i = 0; i < 8; i++) {
                cand[i] = rnd<T>(__fsub_rn(actf<ACT>(x[i]), y[i]));
                y[i] = __fadd_rn(y[i], cand[i]);
            }
            RowIO<float, 8>::store(ys + c0, y);
            RowIO<T, 8>::store(SR + row * C + c0, cand);
        }
    };
    auto zero_row = [&](int64_t row) {   // a rowmap conv reads non-emitted slots as rows
        const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int c0 = lane * 8; c0 < C; c0 += 256) RowIO<T, 8>::store(SR + row * C + c0, z);
    };
    for (int64_t bq = (int64_t)blockIdx.x * DWS_WARPS + wid; bq < BNo; bq += (int64_t)gridDim.x * DWS_WARPS) {
        uint32_t w = __ldg(d.out_act + bq);
        if (!w) {
            if (lane == 0) d.site_act[bq] = 0u;
            continue;
        }
        const int b = (int)(bq / Nout), q = (int)(bq - (int64_t)b * Nout);
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        const int nlive = dw_gather_meta<32, KMAX>(c, b, oy, ox, lane, 0xffffffffu, meta);
        for (int c0 = lane * 8; c0 < C; c0 += 256) {
            float x[8], y[8];
            RowIO<float, 8>::load(d.x0 + bq * C + c0, x);
#pragma unroll
            for (int i = 0; i < 8; i++) y[i] = actf<ACT>(x[i]);
            RowIO<float, 8>::store(xs + c0, x);
            RowIO<float, 8>::store(ys + c0, y);
        }
        uint32_t emit = 0;
        int64_t orow = 1 + __ldg(d.out_pbase + bq);
        while (w) {
            const int tA = __ffs(w) - 1;
            w &= w - 1;
            int tB = -1;
            if (PAIR && w) {
                tB = __ffs(w) - 1;
                w &= w - 1;
            }
            // pass 1 of frame A (+ the delta of frame B into bs)
            float mx = 0.0f;
            for (int c0 = lane * 8; c0 < C; c0 += 256) {
                float accA[8], accB[8], x[8], y[8];
                if constexpr (PAIR)
                    dw_acc_pair<TB>(reinterpret_cast<const bf16 *>(A), c.wk, C, c0, true, meta, nlive, tA, tB, accA,
                                    accB);
                else
                    dw_acc_one<TB, 8, T>(A, c.wk, C, c0, true, meta, nlive, tA, accA);
                RowIO<float, 8>::load(xs + c0, x);
                RowIO<float, 8>::load(ys + c0, y);
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    x[i] = __fadd_rn(x[i], rnd<T>(accA[i]));
                    mx = fmaxf(mx, fabsf(__fsub_rn(actf<ACT>(x[i]), y[i])));
                }
                RowIO<float, 8>::store(xs + c0, x);
                if (CR) RowIO<T, 8>::store(CR + orow * C + c0, accA);
                if (PAIR && tB >= 0) {
#pragma unroll
                    for (int i = 0; i < 8; i++) accB[i] = rnd<T>(accB[i]);
                    RowIO<float, 8>::store(bs + c0, accB);
                    if (CR) RowIO<T, 8>::store(CR + (orow + 1) * C + c0, accB);
                }
            }
            if (gmax<32>(mx, 0xffffffffu) > theta) {   // truncation
                emit_row(orow);
                emit |= 1u << tA;
            } else if (d.zero_gaps) {
                zero_row(orow);
            }
            orow++;
            if (tB < 0) continue;
            mx = 0.0f;
            for (int c0 = lane * 8; c0 < C; c0 += 256) {
                float x[8], y[8], v[8];
                RowIO<float, 8>::load(xs + c0, x);
                RowIO<float, 8>::load(ys + c0, y);
                RowIO<float, 8>::load(bs + c0, v);
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    x[i] = __fadd_rn(x[i], v[i]);
                    mx = fmaxf(mx, fabsf(__fsub_rn(actf<ACT>(x[i]), y[i])));
                }
                RowIO<float, 8>::store(xs + c0, x);
            }
            if (gmax<32>(mx, 0xffffffffu) > theta) {
                emit_row(orow);
                emit |= 1u << tB;
            } else if (d.zero_gaps) {
                zero_row(orow);
            }
            orow++;
        }
        if (lane == 0) d.site_act[bq] = emit;
    }
}

// Tile-resident depthwise (C % 8 == 0).  A CTA owns an output tile of one
// chunk and one channel slice (<= 64 channels).  Depthwise deltas are linear
// per frame (Eq.2, no state across frames), so the CTA stages the footprint's
// delta rows of a GROUP of frames at once -- [pixel][frame in group][slice]
// in shared memory, only the rows that exist (active) are copied, with
// cp.async 16-byte pieces -- then every active output of every frame of the
// group reads its k x k taps from shared memory (absent taps = 0).  Each input
// row is fetched once per (tile, slice) instead of once per tap of every
// output that touches it, and one round trip serves a whole frame group.
// DENSE (reference frame): fp32 activations in, fp32 + bias out, one frame.
// FP32 mode keeps the oracle's fmaf chain over taps in (dy, dx) order from +0.
constexpr int DWT_CS = 64;                 // max channels per slice
constexpr int DWT_STG = 96 * 1024;         // staging bytes per CTA (two CTAs per SM)

template <class TI>
struct DwTile {
    static constexpr int EPL = 16 / (int)sizeof(TI);   // elements per 16-byte piece
    static size_t smem(int FP, int TO, int kk, size_t stg) {
        return (size_t)kk * DWT_CS * 4 + (size_t)FP * 12 + (size_t)TO * 8 + stg + 64;
    }
};

template <class T, bool DENSE>
__global__ void __launch_bounds__(256) k_dw_tile(ConvCall c, const uint32_t *__restrict__ out_act,
                                                 const int32_t *__restrict__ out_pbase, int TOH, int TOW) {
    st_pdl_enter();
    using TI = typename std::conditional<DENSE, float, T>::type;   // staged input element
    using TO = typename std::conditional<DENSE, float, T>::type;   // output element
    constexpr int EPL = DwTile<TI>::EPL;
    extern __shared__ __align__(16) unsigned char dwt_smem[];
    const Geo g = c.g;
    const int C = g.Cin, kk = g.kh * g.kw;
    const int Nin = g.Hin * g.Win, Nout = g.Hout * g.Wout;
    const int nsl = (C + DWT_CS - 1) / DWT_CS;
    const int ntx = (g.Wout + TOW - 1) / TOW, nty = (g.Hout + TOH - 1) / TOH;
    int bid = blockIdx.x;
    const int sl = bid % nsl;
    bid /= nsl;
    const int tile = bid % (ntx * nty), b = bid / (ntx * nty);
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int cs0 = sl * DWT_CS, csw = min(DWT_CS, C - cs0);   // slice channels (multiple of 8)
    const int FH = (TOH - 1) * g.sh + g.kh, FW = (TOW - 1) * g.sw + g.kw, FP = FH * FW, TOc = TOH * TOW;
    const int fy0 = ty * TOH * g.sh - g.ph, fx0 = tx * TOW * g.sw - g.pw;
    // frames per staged group: the whole [FP][FG][csw] block fits the staging area
    const int FG = DENSE ? 1 : min(32, (int)(DWT_STG / ((size_t)FP * csw * sizeof(TI))));
    float *w_s = reinterpret_cast<float *>(dwt_smem);                 // [kk][csw]
    uint32_t *f_act = reinterpret_cast<uint32_t *>(w_s + kk * DWT_CS); // [FP]
    uint32_t *f_sl = f_act + FP;
    int32_t *f_row = reinterpret_cast<int32_t *>(f_sl + FP);          // sparse: 1 + pbase; dense: pixel; -1 outside
    uint32_t *o_act = reinterpret_cast<uint32_t *>(f_row + FP);       // [TO]
    int32_t *o_row = reinterpret_cast<int32_t *>(o_act + TOc);        // sparse: 1 + out pbase; dense: out pixel; -1
    uintptr_t sp = reinterpret_cast<uintptr_t>(o_row + TOc);
    TI *stg = reinterpret_cast<TI *>((sp + 15) & ~uintptr_t(15));     // [FP][FG][csw]
    __shared__ uint32_t u_word;
    const int tid = threadIdx.x;
    if (tid == 0) u_word = 0u;
    for (int i = tid; i < kk * csw; i += 256) {
        const int tap = i / csw, j = i - tap * csw;
        w_s[i] = __ldg(c.wk + (int64_t)tap * C + cs0 + j);
    }
    for (int p = tid; p < FP; p += 256) {
        const int iy = fy0 + p / FW, ix = fx0 + p % FW;
        uint32_t a = 0, sl2 = 0;
        int row = -1;
        if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
            const int64_t gp = (int64_t)b * Nin + iy * g.Win + ix;
            if (DENSE) {
                a = 1u;
                row = (int)gp;
            } else {
                a = __ldg(c.a.act + gp);
                if (a) {
                    sl2 = __ldg(c.a.slot + gp);
                    row = 1 + __ldg(c.a.pbase + gp);
                }
            }
        }
        f_act[p] = a;
        f_sl[p] = sl2;
        f_row[p] = row;
    }
    __syncthreads();
    uint32_t uw = 0;
    for (int o = tid; o < TOc; o += 256) {
        const int oy = ty * TOH + o / TOW, ox = tx * TOW + o % TOW;
        uint32_t a = 0;
        int row = -1;
        if (oy < g.Hout && ox < g.Wout) {
            const int64_t bo = (int64_t)b * Nout + oy * g.Wout + ox;
            if (DENSE) {
                a = 1u;
                row = (int)bo;
            } else {
                a = __ldg(out_act + bo);
                row = 1 + __ldg(out_pbase + bo);
            }
        }
        o_act[o] = a;
        o_row[o] = row;
        uw |= a;
    }
    uw = __reduce_or_sync(0xffffffffu, uw);
    if ((tid & 31) == 0 && uw) atomicOr(&u_word, uw);
    __syncthreads();
    const uint32_t U = u_word;
    const TI *src_base = DENSE ? reinterpret_cast<const TI *>(c.a_dense) : static_cast<const TI *>(c.a.rows);
    const int ppp = csw / EPL;   // 16-byte pieces per staged row
    const int ncg = csw / 8;     // 8-channel groups per output
    uint32_t Ur = U;
    while (Ur) {
        const int ta = __ffs(Ur) - 1;                                   // group = frames [ta, ta + FG)
        const uint32_t gmask = (ta + FG >= 32) ? ~lowmask(ta) : (lowmask(ta + FG) & ~lowmask(ta));
        // ---- stage every existing row of the group (absent rows are never read)
        for (int u = tid; u < FP * FG * ppp; u += 256) {
            const int k = u % ppp, pj = u / ppp;
            const int j = pj % FG, p = pj / FG;
            const int t1 = ta + j;
            if (t1 < 32 && f_row[p] >= 0 && ((f_act[p] >> t1) & 1u)) {
                const int64_t row = DENSE ? (int64_t)f_row[p] : (int64_t)f_row[p] + __popc(f_sl[p] & lowmask(t1));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(
                                 stg + ((size_t)p * FG + j) * csw + k * EPL)),
                             "l"(src_base + row * C + cs0 + k * EPL)
                             : "memory");
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // ---- every active output of every frame of the group
        uint32_t Ug = U & gmask;
        while (Ug) {
            const int t1 = __ffs(Ug) - 1;
            Ug &= Ug - 1;
            const int j = t1 - ta;
            for (int u = tid; u < TOc * ncg; u += 256) {
                const int o = u / ncg, cg = u - (u / ncg) * ncg;
                const uint32_t oa = o_act[o];
                if (!((oa >> t1) & 1u)) continue;
                const int loy = o / TOW, lox = o - (o / TOW) * TOW;
                float acc[8];
#pragma unroll
                for (int i = 0; i < 8; i++) acc[i] = 0.0f;
                for (int dy = 0; dy < g.kh; dy++)
                    for (int dx = 0; dx < g.kw; dx++) {
                        const int p = (loy * g.sh + dy) * FW + lox * g.sw + dx;
                        float v[8], w[8];
                        if (f_row[p] >= 0 && ((f_act[p] >> t1) & 1u)) {
                            RowIO<TI, 8>::load(stg + ((size_t)p * FG + j) * csw + cg * 8, v);
                            if (DENSE && c.rnd_a)
#pragma unroll
                                for (int i = 0; i < 8; i++) v[i] = bf16_round(v[i]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 8; i++) v[i] = 0.0f;
                        }
                        RowIO<float, 8>::load(w_s + (dy * g.kw + dx) * csw + cg * 8, w);
#pragma unroll
                        for (int i = 0; i < 8; i++) acc[i] = fmaf(w[i], v[i], acc[i]);
                    }
                if (DENSE) {
                    float bb[8];
                    RowIO<float, 8>::load(c.bias + cs0 + cg * 8, bb);
#pragma unroll
                    for (int i = 0; i < 8; i++) acc[i] = __fadd_rn(acc[i], bb[i]);
                    RowIO<float, 8>::store(static_cast<float *>(c.out) + (int64_t)o_row[o] * C + cs0 + cg * 8, acc);
                    if (c.act_out) {   // the consuming site's dense output f(x0)
#pragma unroll
                        for (int i = 0; i < 8; i++) acc[i] = act_rt(c.act_kind, acc[i]);
                        RowIO<float, 8>::store(c.act_out + (int64_t)o_row[o] * C + cs0 + cg * 8, acc);
                        if (c.act_bf)
                            RowIO<bf16, 8>::store(static_cast<bf16 *>(c.act_bf) + (int64_t)o_row[o] * C + cs0 + cg * 8,
                                                  acc);
                    }
                } else {
                    const int64_t orow = (int64_t)o_row[o] + __popc(oa & lowmask(t1));
                    RowIO<TO, 8>::store(static_cast<TO *>(c.out) + orow * C + cs0 + cg * 8, acc);
                }
            }
        }
        __syncthreads();   // staging area reused by the next group
        Ur &= ~gmask;
    }
}

// output tile of the tile-resident depthwise: most outputs whose footprint fits
static bool dw_tile_dims(const Geo &g, int fp_max, int &TOH, int &TOW) {
    int best = 0;
    TOH = TOW = 0;
    for (int h = 1; h <= std::min(g.Hout, 32); h++)
        for (int w = 1; w <= std::min(g.Wout, 64); w++) {
            const int fp = ((h - 1) * g.sh + g.kh) * ((w - 1) * g.sw + g.kw);
            if (fp > fp_max || h * w > 256) continue;
            if (h * w > best) { best = h * w; TOH = h; TOW = w; }
        }
    return best > 0;
}

template <class T, bool DENSE>
static bool launch_dw_tile_t(const ConvCall &c, const uint32_t *out_act, const int32_t *out_pbase, cudaStream_t s) {
    using TI = typename std::conditional<DENSE, float, T>::type;
    const Geo &g = c.g;
    if (g.Cin % 8 != 0) return false;
    // footprint small enough that a group holds >= 4 frames (sparse) / 1 frame (dense)
    const int csw = std::min(DWT_CS, g.Cin);
    // dense: a smaller staging budget -> more resident CTAs overlap their
    // staging round trips (the sparse frame-group path keeps DWT_STG)
    static const int dense_stg = [] {
        const char *v = getenv("ST_DW_DENSE_STG_KB");
        return (v ? atoi(v) : 48) * 1024;   // measured: 48 KB best of 96 / 48 / 32 on cfg5
    }();
    const int stg_budget = DENSE ? std::min(dense_stg, DWT_STG) : DWT_STG;
    const int fp_max = std::min<int>(512, (int)(stg_budget / ((DENSE ? 1 : 4) * csw * sizeof(TI))));
    int TOH, TOW;
    if (!dw_tile_dims(g, fp_max, TOH, TOW)) return false;
    const int FP = ((TOH - 1) * g.sh + g.kh) * ((TOW - 1) * g.sw + g.kw);
    const size_t sm = DwTile<TI>::smem(FP, TOH * TOW, g.kh * g.kw,
                                       DENSE ? (size_t)FP * csw * sizeof(TI) + 16 : (size_t)DWT_STG);
    const int64_t grid = (int64_t)c.B * ((g.Hout + TOH - 1) / TOH) * ((g.Wout + TOW - 1) / TOW) *
                         ((g.Cin + DWT_CS - 1) / DWT_CS);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dw_tile<T, DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
        attr = true;
    }
    k_dw_tile<T, DENSE><<<(unsigned)grid, 256, sm, s>>>(c, out_act, out_pbase, TOH, TOW);
    return true;
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

// Dense (reference-frame) depthwise, register form.  A CTA owns an output
// tile of one chunk and a channel slice of <= 64 channels (8-channel groups;
// every thread keeps ONE group for the whole tile, the threads past the last
// whole pixel group idle when the group count does not divide 256).  The tile's
// input footprint is staged once into shared memory, zero-padded, already in
// the contract's operand precision (BF16 mode: bf16-rounded values stored as
// bf16, R22-BF16; FP32 mode: fp32), so the inner loop is per tap one
// shared-memory vector load and 8 FMAs with the group's weights and bias in
// registers (k x k <= 9; 5x5 reads them from shared memory).  Per channel
// the fmaf chain runs over the taps in (dy, dx) order from +0, bias last
// (R18; FP32 mode bit-identical to k_dw_tile and the oracle).  Epilogue: the
// fp32 output, and for a fused site its dense output f(x0) (+ bf16 shadow).
template <class TS, int KK, int MINB>
__global__ void __launch_bounds__(256, MINB) k_dw_dense(ConvCall c, int TOH, int TOW) {
    constexpr bool WREG = KK == 9 && MINB < 3;   // 3x3 weights in registers (72 floats) unless occupancy is asked for
    st_pdl_enter();
    extern __shared__ __align__(16) unsigned char dwd_smem[];
    const Geo g = c.g;
    const int C = g.Cin, kk = g.kh * g.kw;
    const int Nin = g.Hin * g.Win, Nout = g.Hout * g.Wout;
    const int nsl = (C + 63) / 64;
    const int ntx = (g.Wout + TOW - 1) / TOW, nty = (g.Hout + TOH - 1) / TOH;
    int bid = blockIdx.x;
    const int sl = bid % nsl;
    bid /= nsl;
    const int tile = bid % (ntx * nty), b = bid / (ntx * nty);
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int cs0 = sl * 64, csw = min(64, C - cs0), ncg = csw / 8;
    const int FH = (TOH - 1) * g.sh + g.kh, FW = (TOW - 1) * g.sw + g.kw, FP = FH * FW;
    const int fy0 = ty * TOH * g.sh - g.ph, fx0 = tx * TOW * g.sw - g.pw;
    float *w_s = reinterpret_cast<float *>(dwd_smem);           // [kk][csw]
    TS *stg = reinterpret_cast<TS *>(w_s + kk * 64);              // [FP][csw]
    const int tid = threadIdx.x;
    for (int i = tid; i < kk * csw; i += 256) {
        const int tap = i / csw, j = i - tap * csw;
        float wv = __ldg(c.wk + (int64_t)tap * C + cs0 + j);
        if (c.rnd_a) wv = bf16_round(wv);   // weights are bf16 values already in BF16 mode (idempotent)
        w_s[i] = wv;
    }
    // stage the footprint: 8-channel pieces, zeros outside the map
    const float *X = c.a_dense;
    for (int u = tid; u < FP * ncg; u += 256) {
        const int p = u / ncg, cg = u - p * ncg;
        const int iy = fy0 + p / FW, ix = fx0 + p % FW;
        float v[8];
        if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
            RowIO<float, 8>::load(X + ((int64_t)b * Nin + iy * g.Win + ix) * C + cs0 + cg * 8, v);
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] = 0.0f;
        }
        RowIO<TS, 8>::store(stg + (size_t)p * csw + cg * 8, v);   // bf16 staging rounds (RNE)
    }
    __syncthreads();
    const int cg = tid % ncg;               // fixed per thread
    const int c0 = cs0 + cg * 8;
    float bb[8];
    RowIO<float, 8>::load(c.bias + c0, bb);
    float wr[WREG ? KK * 8 : 1];
    if constexpr (WREG) {
#pragma unroll
        for (int t = 0; t < KK; t++) RowIO<float, 8>::load(w_s + t * csw + cg * 8, *reinterpret_cast<float(*)[8]>(wr + 8 * t));
    }
    const int TOc = TOH * TOW;
    // ncg need not divide 256: the threads past the last whole pixel group idle
    const int o0 = tid < (256 / ncg) * ncg ? tid / ncg : TOc;
    for (int o = o0; o < TOc; o += 256 / ncg) {
        const int loy = o / TOW, lox = o - loy * TOW;
        const int oy = ty * TOH + loy, ox = tx * TOW + lox;
        if (oy >= g.Hout || ox >= g.Wout) continue;
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; i++) acc[i] = 0.0f;
        const TS *base = stg + (size_t)(loy * g.sh * FW + lox * g.sw) * csw + cg * 8;
        if constexpr (WREG) {
#pragma unroll
            for (int t = 0; t < KK; t++) {
                const int dy = t / (KK == 25 ? 5 : 3), dx = t - dy * (KK == 25 ? 5 : 3);
                float v[8];
                RowIO<TS, 8>::load(base + (size_t)(dy * FW + dx) * csw, v);
#pragma unroll
                for (int i = 0; i < 8; i++) acc[i] = fmaf(wr[8 * t + i], v[i], acc[i]);
            }
        } else if constexpr (KK > 0) {
#pragma unroll
            for (int t = 0; t < KK; t++) {
                const int dy = t / (KK == 25 ? 5 : 3), dx = t - dy * (KK == 25 ? 5 : 3);
                float v[8], wv[8];
                RowIO<TS, 8>::load(base + (size_t)(dy * FW + dx) * csw, v);
                RowIO<float, 8>::load(w_s + t * csw + cg * 8, wv);
#pragma unroll
                for (int i = 0; i < 8; i += 2) {   // FFMA2: per lane the scalar fmaf
                    const float2 r = fma2(f2(wv[i], wv[i + 1]), f2(v[i], v[i + 1]), f2(acc[i], acc[i + 1]));
                    acc[i] = r.x;
                    acc[i + 1] = r.y;
                }
            }
        } else {
            for (int dy = 0; dy < g.kh; dy++)
                for (int dx = 0; dx < g.kw; dx++) {
                    float v[8], wv[8];
                    RowIO<TS, 8>::load(base + (size_t)(dy * FW + dx) * csw, v);
                    RowIO<float, 8>::load(w_s + (dy * g.kw + dx) * csw + cg * 8, wv);
#pragma unroll
                    for (int i = 0; i < 8; i++) acc[i] = fmaf(wv[i], v[i], acc[i]);
                }
        }
#pragma unroll
        for (int i = 0; i < 8; i++) acc[i] = __fadd_rn(acc[i], bb[i]);
        const int64_t oi = ((int64_t)b * Nout + oy * g.Wout + ox) * C + c0;
        RowIO<float, 8>::store(static_cast<float *>(c.out) + oi, acc);
        if (c.act_out) {
#pragma unroll
            for (int i = 0; i < 8; i++) acc[i] = act_rt(c.act_kind, acc[i]);
            RowIO<float, 8>::store(c.act_out + oi, acc);
            if (c.act_bf) RowIO<bf16, 8>::store(static_cast<bf16 *>(c.act_bf) + oi, acc);
        }
    }
}

template <class TS>
static bool launch_dw_dense_t(const ConvCall &c, cudaStream_t s) {
    const Geo &g = c.g;
    if (g.Cin % 8 != 0) return false;
    const int csw = std::min(64, g.Cin);
    const int stg_budget = 64 * 1024;
    const int fp_max = std::min<int>(1024, stg_budget / (csw * (int)sizeof(TS)));
    int TOH, TOW;
    if (!dw_tile_dims(g, fp_max, TOH, TOW)) return false;
    const int FP = ((TOH - 1) * g.sh + g.kh) * ((TOW - 1) * g.sw + g.kw);
    const size_t sm = (size_t)g.kh * g.kw * 64 * 4 + (size_t)FP * csw * sizeof(TS) + 64;
    const int64_t grid = (int64_t)c.B * ((g.Hout + TOH - 1) / TOH) * ((g.Wout + TOW - 1) / TOW) * ((g.Cin + 63) / 64);
    const bool k3 = g.kh == 3 && g.kw == 3, k5 = g.kh == 5 && g.kw == 5;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dw_dense<TS, 9, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        cudaFuncSetAttribute(k_dw_dense<TS, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        cudaFuncSetAttribute(k_dw_dense<TS, 9, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        cudaFuncSetAttribute(k_dw_dense<TS, 25, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        cudaFuncSetAttribute(k_dw_dense<TS, 0, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        attr = true;
    }
    // default: weights from shared memory, <= 80 registers (3 CTAs / SM)
    const char *mb = getenv("ST_DW_DENSE_MINB");   // 2: weights in registers (measured 6 % slower on cfg5)
    const bool occ = !mb || atoi(mb) >= 3;
    if (occ) {   // 3x3 / 5x5 unrolled (weights from shared memory), other shapes looped
        if (k3) k_dw_dense<TS, 9, 3><<<(unsigned)grid, 256, sm, s>>>(c, TOH, TOW);
        else if (k5) k_dw_dense<TS, 25, 3><<<(unsigned)grid, 256, sm, s>>>(c, TOH, TOW);
        else k_dw_dense<TS, 0, 3><<<(unsigned)grid, 256, sm, s>>>(c, TOH, TOW);
    } else {
        if (k3) k_dw_dense<TS, 9, 2><<<(unsigned)grid, 256, sm, s>>>(c, TOH, TOW);
        else k_dw_dense<TS, 0, 2><<<(unsigned)grid, 256, sm, s>>>(c, TOH, TOW);
    }
    return true;
}

void launch_dwconv_f32(const ConvCall &c, cudaStream_t s) {
    static const bool old_dense = [] { const char *v = getenv("ST_DW_DENSE_TILE"); return v && v[0] == '1'; }();
    if (c.dense && !old_dense &&
        (c.rnd_a ? launch_dw_dense_t<bf16>(c, s) : launch_dw_dense_t<float>(c, s)))
        return;
    if (c.dense && launch_dw_tile_t<float, true>(c, nullptr, nullptr, s)) return;
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
    static const int tile_mode = [] { const char *v = getenv("ST_DW_SPARSE_TILE"); return v ? atoi(v) : 0; }();
    if (tile_mode == 1 || (tile_mode == 2 && c.g.kh * c.g.kw <= 9)) {
        if (c.bf ? launch_dw_tile_t<bf16, false>(c, out_act, out_pbase, s)
                 : launch_dw_tile_t<float, false>(c, out_act, out_pbase, s))
            return;
    }
    if (!c.bf) launch_dw_pm_t<float>(c, out_act, out_pbase, s);
    else launch_dw_pm_t<bf16>(c, out_act, out_pbase, s);
}

bool dwconv_site_fusable(const Geo &g) {
    return g.Cin % 8 == 0 && g.kh * g.kw <= 25 &&
           (g.Cin <= DWT_MAXC || DWS_WARPS * (25 * 16 + 3 * g.Cin * 4) <= 200 * 1024);
}

template <int G, int KMAX, class T, int ACT>
static void launch_dws_k(const ConvCall &c, const DwSite &d, int64_t BNo, cudaStream_t s) {
    constexpr int smem = (256 / G) * KMAX * 16;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((BNo * G + 255) / 256, 148 * 16));
    // ST_DWN_MINB: resident CTAs per SM the narrow form is compiled for (2: <= 128
    // registers; 3: <= 80; 4: <= 64)
    const char *mb = getenv("ST_DWN_MINB");
    const int minb = mb ? atoi(mb) : 2;
    static bool attr = false;
    if (!attr && smem > 48 * 1024) {
        cudaFuncSetAttribute(k_dwconv_site<G, KMAX, T, ACT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_dwconv_site<G, KMAX, T, ACT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_dwconv_site<G, KMAX, T, ACT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    }
    attr = true;
    if (minb == 3) k_dwconv_site<G, KMAX, T, ACT, 3><<<grid, 256, smem, s>>>(c, d);
    else if (minb == 4) k_dwconv_site<G, KMAX, T, ACT, 4><<<grid, 256, smem, s>>>(c, d);
    else k_dwconv_site<G, KMAX, T, ACT, 2><<<grid, 256, smem, s>>>(c, d);
}

template <int KMAX, class T, int ACT>
static void launch_dws_wide_k(const ConvCall &c, const DwSite &d, int64_t BNo, cudaStream_t s) {
    const int smem = DWS_WARPS * KMAX * 16 + DWS_WARPS * 3 * c.g.Cin * 4;   // <= 200 KB (dwconv_site_fusable)
    static int attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_dwconv_site_wide<KMAX, T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = smem;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((BNo + DWS_WARPS - 1) / DWS_WARPS, 148 * 8));
    k_dwconv_site_wide<KMAX, T, ACT><<<grid, 32 * DWS_WARPS, smem, s>>>(c, d);
}

template <int CPL, int KMAX, class T, int ACT>
static void launch_dww_k(const ConvCall &c, const DwSite &d, int64_t BNo, cudaStream_t s) {
    const int smem = KMAX * c.g.Cin * 4;
    static int attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_dwconv_site_w<CPL, KMAX, T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = smem;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((BNo + DWW_WARPS - 1) / DWW_WARPS, 148 * 8));
    k_dwconv_site_w<CPL, KMAX, T, ACT><<<grid, 32 * DWW_WARPS, smem, s>>>(c, d);
}

template <class T, int ACT>
static void launch_dws_t(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int64_t BNo = (int64_t)c.B * c.g.Hout * c.g.Wout;
    const int C = c.g.Cin;
    const bool k9 = c.g.kh * c.g.kw <= 9;
    static const bool grouped = [] { const char *v = getenv("ST_DW_GROUPED"); return v && v[0] == '1'; }();
    // ST_DW_TEAM: 0 = never the team form, 1 (default) = C > 32, 2 = every C
    // (cfg5: 17.9 -> 12.3 ms of depthwise sites per step with the default;
    // at C <= 32 the team form idles 28 of 32 lanes: 4.0 -> 10.0 ms)
    const char *tv = getenv("ST_DW_TEAM");   // read per launch (graph capture): tests switch it
    const int team = tv ? atoi(tv) : 1;
    // ST_DW_TILE (default 1): the tile form for C <= 32, k x k <= 9 (shared-memory
    // staged footprint rows; cfg5 540x960x32: 4.05 -> 3.47 ms, cfg3 0.70 -> 0.49)
    const char *tl = getenv("ST_DW_TILE");
    if (!(tl && tl[0] == '0') && team != 0 && dwconv_site_tile_ok(c.g)) {
        launch_dwconv_site_tile(c, d, s);
        return;
    }
    if (team != 0 && C <= DWT_MAXC && ((team >= 1 && C > 32) || team == 2)) {
        launch_dwconv_site_team(c, d, s);
        return;
    }
    if (!grouped && C > 32 && C <= 256) {   // warp per pixel (uniform control flow); C <= 32: 8+ pixels per warp
#define L_DWW(CPL_)                                                             \
    {                                                                           \
        if (k9) launch_dww_k<CPL_, 9, T, ACT>(c, d, BNo, s);                    \
        else launch_dww_k<CPL_, 25, T, ACT>(c, d, BNo, s);                      \
        return;                                                                 \
    }
        if (C <= 32) L_DWW(1)
        if (C <= 64) L_DWW(2)
        if (C <= 96) L_DWW(3)
        if (C <= 128) L_DWW(4)
        if (C <= 160) L_DWW(5)
        if (C <= 192) L_DWW(6)
        L_DWW(8)
#undef L_DWW
    }
#define L_DWS(G_)                                                               \
    {                                                                           \
        if (k9) launch_dws_k<G_, 9, T, ACT>(c, d, BNo, s);                      \
        else launch_dws_k<G_, 25, T, ACT>(c, d, BNo, s);                        \
    }
    if (C <= 8) L_DWS(1)
    else if (C <= 16) L_DWS(2)
    else if (C <= 32) L_DWS(4)
    else if (C <= 64) L_DWS(8)
    else if (C <= 128) L_DWS(16)
    else if (C <= 256) L_DWS(32)
    else if (k9) launch_dws_wide_k<9, T, ACT>(c, d, BNo, s);
    else launch_dws_wide_k<25, T, ACT>(c, d, BNo, s);
#undef L_DWS
}

void launch_dwconv_site(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    if (c.bf) {
        if (d.act == ACT_RELU) launch_dws_t<bf16, ACT_RELU>(c, d, s);
        else launch_dws_t<bf16, ACT_SILU_FAST>(c, d, s);   // BF16 mode: the fast SiLU of the site kernels
    } else {
        if (d.act == ACT_RELU) launch_dws_t<float, ACT_RELU>(c, d, s);
        else launch_dws_t<float, ACT_SILU>(c, d, s);
    }
}

}  // namespace st
