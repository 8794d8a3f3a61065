// kernels_dw_team.cu -- sparse depthwise conv + its pointwise site in one
// pass, team form (SURVEY §8(f) N2 for depthwise convs; Eq.2 then Eq.3,
// PAPER.md P:124-139; truncation P:143), sm_100a.  The other forms
// (narrow, warp, wide) and the dispatch are in kernels_dw.cu.
#include <cstdlib>

#include "rowio.cuh"

namespace st {

// Team form (the default for C > 256, and for 32 < C <= 256 when 8-channel
// lanes beat channel-strided ones): ONE CTA = a team of NW warps per output
// pixel; warp v owns channels [256v, 256v + 256), lane l the 8 channels at
// 256v + 8l, so a tap row moves as one 16-byte vector per lane (bf16) and the
// site state x_acc / y_acc stays in registers -- no shared-memory state and
// no serial walk over channel chunks.  Every warp holds the tap metadata in
// its tap lanes (as k_dwconv_site_w); per frame pair the rows of a batch of
// TB active taps x 2 frames are loaded before their FMAs.  The truncation
// decision needs max_c |c| over the whole pixel: each warp reduces by
// shuffles, then the team through a double-buffered shared slot and one
// barrier per frame (a warp reads frame k's slot before it arrives at frame
// k+1's barrier, so frame k+2 may reuse it).  Per channel the operations are
// those of k_dwconv_site_w (fmaf chain over taps in ascending order from +0,
// x += rnd(Delta), c = f(x) - y, emit iff max > theta, y += rnd(c)), so the
// results are bit-identical to the other forms and to the separate kernels.
template <class T>
struct DwVec {   // one lane's 8 channels of a row, raw
    static constexpr int NV = sizeof(T) == 2 ? 1 : 2;
    uint4 u[NV];
    __device__ __forceinline__ void load(const T *p) {
#pragma unroll
        for (int i = 0; i < NV; i++) u[i] = __ldg(reinterpret_cast<const uint4 *>(p) + i);
    }
    __device__ __forceinline__ void fma_into(const float (&w)[8], float (&acc)[8]) const {
        if constexpr (sizeof(T) == 2) {   // FFMA2: per lane the fmaf of the scalar chain
            const uint32_t v[4] = {u[0].x, u[0].y, u[0].z, u[0].w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const float2 r = fma2(f2(w[2 * q], w[2 * q + 1]),
                                      f2(__uint_as_float(v[q] << 16), __uint_as_float(v[q] & 0xFFFF0000u)),
                                      f2(acc[2 * q], acc[2 * q + 1]));
                acc[2 * q] = r.x;
                acc[2 * q + 1] = r.y;
            }
        } else {
            const uint32_t v[8] = {u[0].x, u[0].y, u[0].z, u[0].w, u[1].x, u[1].y, u[1].z, u[1].w};
#pragma unroll
            for (int q = 0; q < 8; q++) acc[q] = fmaf(w[q], __uint_as_float(v[q]), acc[q]);
        }
    }
};

constexpr int DWT_MAXNW = 16;   // team form: C <= 16 * 256
#ifndef DWT_MAXREG
#define DWT_MAXREG __launch_bounds__(32 * DWT_MAXNW)
#endif
template <int KMAX, int TB, class T, int ACT>
__global__ void DWT_MAXREG k_dwconv_site_team(ConvCall c, DwSite d) {
    st_pdl_enter();
    __shared__ float red[2][DWT_MAXNW];
    const int NW = blockDim.x >> 5;
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int C = g.Cin, ntaps = g.kh * g.kw;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c0 = wid * 256 + lane * 8;
    const bool on = c0 < C;   // C % 8 == 0: a lane's 8 channels are whole or past C
    const int64_t BNo = (int64_t)c.B * Nout;
    const T *A = static_cast<const T *>(c.a.rows);
    T *SR = static_cast<T *>(d.site_rows);
    T *CR = static_cast<T *>(d.conv_rows);
    const int tdy = lane < ntaps ? lane / g.kw : 0, tdx = lane < ntaps ? lane - tdy * g.kw : 0;
    int par = 0;
    uint32_t n_w = 0, n_ma = 0, n_ms = 0;
    int n_mz = 0;
    float n_x[8];
    auto fetch = [&](int64_t bq) {   // frame word; tap lanes: {act, slot, 1 + pbase}; x0 chunk
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
        if (on) RowIO<float, 8>::load(d.x0 + bq * C + c0, n_x);
    };
    auto team_max = [&](float mx) {
        mx = gmax<32>(mx, 0xffffffffu);
        if (NW > 1) {
            if (lane == 0) red[par][wid] = mx;
            __syncthreads();
            for (int v = 0; v < NW; v++) mx = fmaxf(mx, red[par][v]);
            par ^= 1;
        }
        return mx;
    };
    fetch(blockIdx.x);
    for (int64_t bq = blockIdx.x; bq < BNo; bq += gridDim.x) {
        uint32_t w = n_w;
        const uint32_t ma = n_ma, ms = n_ms;
        const int mz = n_mz;
        float xa[8], ya[8];
#pragma unroll
        for (int i = 0; i < 8; i++) xa[i] = n_x[i];
        fetch(bq + gridDim.x);   // the next pixel's loads in flight
        if (!w) {
            if (threadIdx.x == 0) d.site_act[bq] = 0u;
            continue;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) ya[i] = actf<ACT>(xa[i]);
        uint32_t emit = 0;
        int64_t orow = 1 + __ldg(d.out_pbase + bq);
        auto step = [&](const float (&acc)[8], int64_t row, int t1) {
            float cand[8];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const float v = rnd<T>(acc[i]);                    // the conv's stored delta
                xa[i] = __fadd_rn(xa[i], v);                       // reconstruct x (Eq.3)
                cand[i] = __fsub_rn(actf<ACT>(xa[i]), ya[i]);      // restore the delta
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            if (CR && on) RowIO<T, 8>::store(CR + row * C + c0, acc);
            if (team_max(mx) > theta) {                            // truncation
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    cand[i] = rnd<T>(cand[i]);
                    ya[i] = __fadd_rn(ya[i], cand[i]);
                }
                if (on) RowIO<T, 8>::store(SR + row * C + c0, cand);
                emit |= 1u << t1;
            } else if (d.zero_gaps && on) {                        // a rowmap conv reads this slot as a row
                const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                RowIO<T, 8>::store(SR + row * C + c0, z);
            }
        };
        while (w) {
            const int tA = __ffs(w) - 1;
            w &= w - 1;
            const int tB = w ? __ffs(w) - 1 : -1;
            if (w) w &= w - 1;
            const bool hA = (ma >> tA) & 1u, hB = tB >= 0 && ((ma >> tB) & 1u);
            const int rA = mz + __popc(ms & lowmask(tA)), rB = tB >= 0 ? mz + __popc(ms & lowmask(tB)) : 0;
            uint32_t todo = __ballot_sync(0xffffffffu, hA || hB);   // taps active in A or B, ascending
            const uint32_t bA = __ballot_sync(0xffffffffu, hA), bB = __ballot_sync(0xffffffffu, hB);
            float accA[8], accB[8];
#pragma unroll
            for (int i = 0; i < 8; i++) accA[i] = accB[i] = 0.0f;
            while (todo) {
                int tp[TB];
                DwVec<T> vA[TB], vB[TB];
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    tp[j] = todo ? __ffs(todo) - 1 : -1;
                    if (todo) todo &= todo - 1;
                    const int t = tp[j] < 0 ? 0 : tp[j];
                    const int64_t ra = __shfl_sync(0xffffffffu, rA, t), rb = __shfl_sync(0xffffffffu, rB, t);
                    if (on && tp[j] >= 0 && ((bA >> t) & 1u)) vA[j].load(A + ra * C + c0);
                    if (on && tp[j] >= 0 && ((bB >> t) & 1u)) vB[j].load(A + rb * C + c0);
                }
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    if (tp[j] < 0 || !on) continue;
                    float wv[8];
                    RowIO<float, 8>::load(c.wk + (int64_t)tp[j] * C + c0, wv);
                    if ((bA >> tp[j]) & 1u) vA[j].fma_into(wv, accA);
                    if ((bB >> tp[j]) & 1u) vB[j].fma_into(wv, accB);
                }
            }
            step(accA, orow, tA);
            if (tB >= 0) step(accB, orow + 1, tB);
            orow += tB >= 0 ? 2 : 1;
        }
        if (threadIdx.x == 0) d.site_act[bq] = emit;
    }
}

// Sequential-pipeline team form (the default team kernel): one frame per
// step, with the rows of the NEXT touched frame's first TB active taps
// loaded while the current frame's site step (and its team barrier) runs --
// the memory parallelism of a frame pair at the register cost of one frame,
// and half the code (one site step per iteration).  32-bit pixel and row
// indices (the launcher checks B*N and the row count fit).
#ifndef DWS_SEQ_BOUNDS
#define DWS_SEQ_BOUNDS __launch_bounds__(32 * DWT_MAXNW)
#endif
template <int KMAX, int TB, class T, int ACT>
__global__ void DWS_SEQ_BOUNDS k_dwconv_site_seq(ConvCall c, DwSite d) {
    st_pdl_enter();
    __shared__ float red[2][DWT_MAXNW];
    const int NW = blockDim.x >> 5;
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int C = g.Cin, ntaps = g.kh * g.kw;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c0 = wid * 256 + lane * 8;
    const bool on = c0 < C;   // C % 8 == 0: a lane's 8 channels are whole or past C
    const int BNo = c.B * Nout;
    const T *A = static_cast<const T *>(c.a.rows) + (on ? c0 : 0);
    T *SR = static_cast<T *>(d.site_rows) + c0;
    T *CR = d.conv_rows ? static_cast<T *>(d.conv_rows) + c0 : nullptr;
    const float *W = c.wk + (on ? c0 : 0);
    const int tdy = lane < ntaps ? lane / g.kw : 0, tdx = lane < ntaps ? lane - tdy * g.kw : 0;
    int par = 0;
    for (int bq = blockIdx.x; bq < BNo; bq += gridDim.x) {
        uint32_t w = __ldg(d.out_act + bq);
        if (!w) {
            if (threadIdx.x == 0) d.site_act[bq] = 0u;
            continue;
        }
        const int b = bq / Nout, q = bq - b * Nout;
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        uint32_t ma = 0, ms = 0;
        int mz = 0;
        if (lane < ntaps) {   // tap lanes: {act, slot, 1 + pbase} of the tap's input pixel
            const int iy = oy * g.sh - g.ph + tdy, ix = ox * g.sw - g.pw + tdx;
            if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                const int bp = b * Nin + iy * g.Win + ix;
                ma = __ldg(c.a.act + bp);
                ms = __ldg(c.a.slot + bp);
                mz = 1 + __ldg(c.a.pbase + bp);
            }
        }
        float xa[8], ya[8];
        if (on) {
            RowIO<float, 8>::load(d.x0 + (int64_t)bq * C + c0, xa);
        } else {
#pragma unroll
            for (int i = 0; i < 8; i++) xa[i] = 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) ya[i] = actf<ACT>(xa[i]);
        int orow = 1 + __ldg(d.out_pbase + bq);
        uint32_t emit = 0;
        // the first TB taps active at frame tt: rows in flight; the rest stay in todo
        uint32_t todo = 0;
        int rcur = 0, tp[TB];
        DwVec<T> v[TB];
        auto issue = [&](int tt) {
            rcur = mz + __popc(ms & lowmask(tt));
            todo = __ballot_sync(0xffffffffu, (ma >> tt) & 1u);
#pragma unroll
            for (int j = 0; j < TB; j++) {
                tp[j] = todo ? __ffs(todo) - 1 : -1;
                if (todo) todo &= todo - 1;
                const int r = __shfl_sync(0xffffffffu, rcur, tp[j] < 0 ? 0 : tp[j]);
                if (on && tp[j] >= 0) {
                    ST_CHECK(r > 0 && r < c.a.nrows);
                    v[j].load(A + (int64_t)r * C);
                }
            }
        };
        auto consume = [&](float (&acc)[8]) {
#pragma unroll
            for (int j = 0; j < TB; j++) {
                if (tp[j] < 0 || !on) continue;
                float wv[8];
                RowIO<float, 8>::load(W + tp[j] * C, wv);
                v[j].fma_into(wv, acc);
            }
        };
        int t = __ffs(w) - 1;
        w &= w - 1;
        issue(t);
        while (true) {
            float acc[8];
#pragma unroll
            for (int i = 0; i < 8; i++) acc[i] = 0.0f;
            consume(acc);
            while (todo) {   // more than TB active taps (ascending order kept)
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    tp[j] = todo ? __ffs(todo) - 1 : -1;
                    if (todo) todo &= todo - 1;
                    const int r = __shfl_sync(0xffffffffu, rcur, tp[j] < 0 ? 0 : tp[j]);
                    if (on && tp[j] >= 0) v[j].load(A + (int64_t)r * C);
                }
                consume(acc);
            }
            const int tn = w ? __ffs(w) - 1 : -1;
            if (w) w &= w - 1;
            if (tn >= 0) issue(tn);   // next frame's rows in flight during the site step
            // site step (k_site_pw's operations, in its order; fp32x2 pairs)
            float cand[8];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                const float2 dv = rnd2<T>(f2(acc[i], acc[i + 1]));               // the conv's stored delta
                const float2 x = add2(f2(xa[i], xa[i + 1]), dv);                 // reconstruct x (Eq.3)
                const float2 cd = sub2(actf2<ACT>(x), f2(ya[i], ya[i + 1]));     // restore the delta
                xa[i] = x.x;
                xa[i + 1] = x.y;
                cand[i] = cd.x;
                cand[i + 1] = cd.y;
                mx = fmaxf(mx, fmaxf(fabsf(cd.x), fabsf(cd.y)));
            }
            ST_CHECK(orow > 0 && orow < d.site_nrows);
            if (CR && on) RowIO<T, 8>::store(CR + (int64_t)orow * C, acc);
            mx = gmax<32>(mx, 0xffffffffu);
            if (NW > 1) {
                if (lane == 0) red[par][wid] = mx;
                __syncthreads();
                for (int u = 0; u < NW; u++) mx = fmaxf(mx, red[par][u]);
                par ^= 1;
            }
            if (mx > theta) {                                      // truncation
#pragma unroll
                for (int i = 0; i < 8; i += 2) {
                    const float2 r = rnd2<T>(f2(cand[i], cand[i + 1]));
                    const float2 y = add2(f2(ya[i], ya[i + 1]), r);
                    cand[i] = r.x;
                    cand[i + 1] = r.y;
                    ya[i] = y.x;
                    ya[i + 1] = y.y;
                }
                if (on) RowIO<T, 8>::store(SR + (int64_t)orow * C, cand);
                emit |= 1u << t;
            } else if (d.zero_gaps && on) {                        // a rowmap conv reads this slot as a row
                const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                RowIO<T, 8>::store(SR + (int64_t)orow * C, z);
            }
            orow++;
            if (tn < 0) break;
            t = tn;
        }
        if (threadIdx.x == 0) d.site_act[bq] = emit;
    }
}

// Channel-strided sequential form (C <= 64): ONE WARP per output pixel, lane
// l owns channels l, l + 32 (CPL = ceil(C/32)), so a narrow row is one
// coalesced 2-byte access per lane and every lane works -- the 8-channel
// team form idles 28 of 32 lanes at C = 32.  Same pipeline (the next
// frame's tap rows in flight during the site step) and the same per-channel
// operations in the same order.
constexpr int DWS_SEQS_WARPS = 8;
template <int KMAX, int TB, int CPL, class T, int ACT>
__global__ void __launch_bounds__(32 * DWS_SEQS_WARPS) k_dwconv_site_seqs(ConvCall c, DwSite d) {
    st_pdl_enter();
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int Nin = g.Hin * g.Win, Nout = g.Wout * g.Hout;
    const int C = g.Cin, ntaps = g.kh * g.kw;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int BNo = c.B * Nout;
    const T *A = static_cast<const T *>(c.a.rows) + lane;
    T *SR = static_cast<T *>(d.site_rows) + lane;
    T *CR = d.conv_rows ? static_cast<T *>(d.conv_rows) + lane : nullptr;
    const float *W = c.wk + lane;
    const int tdy = lane < ntaps ? lane / g.kw : 0, tdx = lane < ntaps ? lane - tdy * g.kw : 0;
    const int nwarps = gridDim.x * DWS_SEQS_WARPS;
    for (int bq = blockIdx.x * DWS_SEQS_WARPS + wid; bq < BNo; bq += nwarps) {
        uint32_t w = __ldg(d.out_act + bq);
        if (!w) {
            if (lane == 0) d.site_act[bq] = 0u;
            continue;
        }
        const int b = bq / Nout, q = bq - b * Nout;
        const int oy = q / g.Wout, ox = q - oy * g.Wout;
        uint32_t ma = 0, ms = 0;
        int mz = 0;
        if (lane < ntaps) {   // tap lanes: {act, slot, 1 + pbase} of the tap's input pixel
            const int iy = oy * g.sh - g.ph + tdy, ix = ox * g.sw - g.pw + tdx;
            if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                const int bp = b * Nin + iy * g.Win + ix;
                ma = __ldg(c.a.act + bp);
                ms = __ldg(c.a.slot + bp);
                mz = 1 + __ldg(c.a.pbase + bp);
            }
        }
        float xa[CPL], ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            xa[i] = lane + 32 * i < C ? __ldg(d.x0 + (int64_t)bq * C + lane + 32 * i) : 0.0f;
            ya[i] = actf<ACT>(xa[i]);
        }
        int orow = 1 + __ldg(d.out_pbase + bq);
        uint32_t emit = 0;
        // the first TB taps active at frame tt: rows in flight; the rest stay in todo
        uint32_t todo = 0;
        int rcur = 0, tp[TB];
        float v[TB][CPL];
        auto issue = [&](int tt) {
            rcur = mz + __popc(ms & lowmask(tt));
            todo = __ballot_sync(0xffffffffu, (ma >> tt) & 1u);
#pragma unroll
            for (int j = 0; j < TB; j++) {
                tp[j] = todo ? __ffs(todo) - 1 : -1;
                if (todo) todo &= todo - 1;
                const int r = __shfl_sync(0xffffffffu, rcur, tp[j] < 0 ? 0 : tp[j]);
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    v[j][i] = (tp[j] >= 0 && lane + 32 * i < C) ? ldr<T>(A + (int64_t)r * C + 32 * i) : 0.0f;
            }
        };
        auto consume = [&](float (&acc)[CPL]) {
#pragma unroll
            for (int j = 0; j < TB; j++) {
                if (tp[j] < 0) continue;
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) acc[i] = fmaf(__ldg(W + tp[j] * C + 32 * i), v[j][i], acc[i]);
            }
        };
        int t = __ffs(w) - 1;
        w &= w - 1;
        issue(t);
        while (true) {
            float acc[CPL];
#pragma unroll
            for (int i = 0; i < CPL; i++) acc[i] = 0.0f;
            consume(acc);
            while (todo) {   // more than TB active taps (ascending order kept)
#pragma unroll
                for (int j = 0; j < TB; j++) {
                    tp[j] = todo ? __ffs(todo) - 1 : -1;
                    if (todo) todo &= todo - 1;
                    const int r = __shfl_sync(0xffffffffu, rcur, tp[j] < 0 ? 0 : tp[j]);
#pragma unroll
                    for (int i = 0; i < CPL; i++)
                        v[j][i] = (tp[j] >= 0 && lane + 32 * i < C) ? ldr<T>(A + (int64_t)r * C + 32 * i) : 0.0f;
                }
                consume(acc);
            }
            const int tn = w ? __ffs(w) - 1 : -1;
            if (w) w &= w - 1;
            if (tn >= 0) issue(tn);   // next frame's rows in flight during the site step
            // site step (k_site_pw's operations, in its order)
            float cand[CPL];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                const float dv = rnd<T>(acc[i]);                   // the conv's stored delta
                xa[i] = __fadd_rn(xa[i], dv);                      // reconstruct x (Eq.3)
                cand[i] = __fsub_rn(actf<ACT>(xa[i]), ya[i]);      // restore the delta
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            if (CR)
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) str<T>(CR + (int64_t)orow * C + 32 * i, acc[i]);
            mx = gmax<32>(mx, 0xffffffffu);
            if (mx > theta) {                                      // truncation
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    cand[i] = rnd<T>(cand[i]);
                    ya[i] = __fadd_rn(ya[i], cand[i]);
                    if (lane + 32 * i < C) str<T>(SR + (int64_t)orow * C + 32 * i, cand[i]);
                }
                emit |= 1u << t;
            } else if (d.zero_gaps) {                              // a rowmap conv reads this slot as a row
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) str<T>(SR + (int64_t)orow * C + 32 * i, 0.0f);
            }
            orow++;
            if (tn < 0) break;
            t = tn;
        }
        if (lane == 0) d.site_act[bq] = emit;
    }
}

// Tile form for narrow layers (C <= 32, k x k <= 9; the default there): a CTA
// owns an output tile of one chunk -- 256 / G pixels, G = ceil(C/8) lanes per
// pixel, 8 channels per lane.  Rows are ordered (chunk, pixel, frame), so the
// delta rows of one image row of the tile's input footprint are ONE contiguous
// range: the CTA copies those ranges (every frame's rows, cp.async 16-byte
// pieces) into shared memory once, then each pixel group walks its touched
// frames with the tap rows read from shared memory -- no per-frame global
// round trips, no per-group metadata walk (the 9 taps' frame / slot words and
// staged row bases are registers).  A tile whose rows exceed the staging
// capacity reads its taps from global memory instead (same operations).  Per
// channel: the fmaf chain over active taps in ascending order from +0, then
// the site step of k_site_pw -- bit-identical to the other forms.
constexpr int DWT_TILE_STG = 32 * 1024;   // staged row bytes per CTA
template <int G, class T, int ACT>
__global__ void __launch_bounds__(256) k_dwconv_site_tile(ConvCall c, DwSite d, int TH, int TW) {
    st_pdl_enter();
    __shared__ float w_s[9 * 32];
    __shared__ uint32_t f_act[17 * 33], f_sl[17 * 33];
    __shared__ int32_t f_off[17 * 33];            // staged row of the pixel's first row (-1: outside)
    __shared__ int32_t r_lo[17], r_len[17], r_so[18];
    __shared__ int ovf;
    extern __shared__ __align__(16) unsigned char dwt_stage[];
    const T *stg = reinterpret_cast<const T *>(dwt_stage);
    const float theta = __ldg(d.theta);
    const Geo g = c.g;
    const int C = g.Cin, kk = g.kh * g.kw;
    const int Nin = g.Hin * g.Win, Nout = g.Hout * g.Wout;
    const int ntx = (g.Wout + TW - 1) / TW, nty = (g.Hout + TH - 1) / TH;
    const int tile = blockIdx.x % (ntx * nty), b = blockIdx.x / (ntx * nty);
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int FH = (TH - 1) * g.sh + g.kh, FW = (TW - 1) * g.sw + g.kw, FP = FH * FW;
    const int fy0 = ty * TH * g.sh - g.ph, fx0 = tx * TW * g.sw - g.pw;
    const int tid = threadIdx.x;
    const T *A = static_cast<const T *>(c.a.rows);
    for (int i = tid; i < kk * C; i += 256) w_s[(i / C) * 32 + i % C] = __ldg(c.wk + i);
    // footprint metadata; per footprint image row the contiguous range of rows
    for (int p = tid; p < FP; p += 256) {
        const int iy = fy0 + p / FW, ix = fx0 + p % FW;
        uint32_t a = 0, sl = 0;
        int off = -1;
        if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
            const int gp = b * Nin + iy * g.Win + ix;
            a = __ldg(c.a.act + gp);
            sl = __ldg(c.a.slot + gp);
            off = 1 + __ldg(c.a.pbase + gp);   // global row for now
        }
        f_act[p] = a;
        f_sl[p] = sl;
        f_off[p] = off;
    }
    __syncthreads();
    if (tid < FH) {   // row range of footprint row tid (pixels inside the map)
        int lo = -1, hi = -1;
        for (int x = 0; x < FW; x++) {
            const int p = tid * FW + x;
            if (f_off[p] < 0) continue;
            if (lo < 0) lo = f_off[p];
            hi = f_off[p] + __popc(f_sl[p]);
        }
        r_lo[tid] = lo;
        r_len[tid] = lo < 0 ? 0 : hi - lo;
    }
    __syncthreads();
    if (tid == 0) {
        int so = 0;
        for (int y = 0; y < FH; y++) {
            r_so[y] = so;
            so += r_len[y];
        }
        r_so[FH] = so;
        ovf = so * C * (int)sizeof(T) > DWT_TILE_STG;
    }
    __syncthreads();
    const bool use_smem = !ovf;
    if (use_smem) {
        // copy the ranges: 16-byte pieces (C % 8 == 0 -> a row is whole pieces)
        const int ppr = C * (int)sizeof(T) / 16;   // pieces per row
        const int total = r_so[FH] * ppr;
        for (int k = tid; k < total; k += 256) {
            const int srow = k / ppr, pc = k - srow * ppr;
            int y = 0;
            while (r_so[y + 1] <= srow) y++;
            const int64_t grow = r_lo[y] + (srow - r_so[y]);
            ST_CHECK(grow > 0 && grow < c.a.nrows);
            const unsigned char *src = reinterpret_cast<const unsigned char *>(A + grow * C) + pc * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(
                             dwt_stage + (size_t)srow * C * sizeof(T) + pc * 16)),
                         "l"(src));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // staged row of each footprint pixel's first row
        for (int p = tid; p < FP; p += 256)
            if (f_off[p] >= 0) {
                const int y = p / FW;
                f_off[p] = r_so[y] + (f_off[p] - r_lo[y]);
            }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    // ---- the pixel groups
    const int pix = tid / G, lane = tid % G;
    const int ly = pix / TW, lx = pix - ly * TW;
    const int oy = ty * TH + ly, ox = tx * TW + lx;
    const unsigned gmask = group_mask<G == 3 ? 4 : G>();
    if (oy >= g.Hout || ox >= g.Wout) return;   // whole groups (G | 32)
    const int bq = b * Nout + oy * g.Wout + ox;
    uint32_t w = __ldg(d.out_act + bq);
    const int c0 = lane * 8;
    const bool on = c0 < C;
    if (!w) {
        if (lane == 0) d.site_act[bq] = 0u;
        return;
    }
    // the 9 taps: frame word, slot word, first row (staged or global)
    uint32_t ta[9], ts[9];
    int tr[9];
#pragma unroll
    for (int k = 0; k < 9; k++) {
        ta[k] = 0u;
        ts[k] = 0u;
        tr[k] = 0;
        if (k < kk) {
            const int dy = k / g.kw, dx = k - dy * g.kw;
            const int p = (ly * g.sh + dy) * FW + lx * g.sw + dx;
            ta[k] = f_act[p];
            ts[k] = f_sl[p];
            tr[k] = f_off[p];
        }
    }
    if (!use_smem)   // global rows: recompute the first rows from the map
#pragma unroll
        for (int k = 0; k < 9; k++)
            if (k < kk && ta[k]) {
                const int dy = k / g.kw, dx = k - dy * g.kw;
                const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                tr[k] = 1 + __ldg(c.a.pbase + b * Nin + iy * g.Win + ix);
            }
    float xa[8], ya[8];
    if (on) {
        RowIO<float, 8>::load(d.x0 + (int64_t)bq * C + c0, xa);
    } else {
#pragma unroll
        for (int i = 0; i < 8; i++) xa[i] = 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) ya[i] = actf<ACT>(xa[i]);
    T *SR = static_cast<T *>(d.site_rows);
    T *CR = static_cast<T *>(d.conv_rows);
    int orow = 1 + __ldg(d.out_pbase + bq);
    uint32_t emit = 0;
    while (w) {
        const int t = __ffs(w) - 1;
        w &= w - 1;
        const uint32_t lm = lowmask(t);
        float acc[8];
#pragma unroll
        for (int i = 0; i < 8; i++) acc[i] = 0.0f;
#pragma unroll
        for (int k = 0; k < 9; k++) {
            if (k >= kk || !((ta[k] >> t) & 1u) || !on) continue;
            const int r = tr[k] + __popc(ts[k] & lm);
            ST_CHECK(use_smem ? (r >= 0 && r < r_so[FH]) : (r > 0 && r < c.a.nrows));
            float v[8], wv[8];
            if (use_smem) RowIO<T, 8>::load(stg + (size_t)r * C + c0, v);
            else RowIO<T, 8>::load(A + (int64_t)r * C + c0, v);
            RowIO<float, 8>::load(w_s + k * 32 + c0, wv);
#pragma unroll
            for (int i = 0; i < 8; i += 2) {   // FFMA2: per lane the fmaf of the scalar chain
                const float2 r = fma2(f2(wv[i], wv[i + 1]), f2(v[i], v[i + 1]), f2(acc[i], acc[i + 1]));
                acc[i] = r.x;
                acc[i + 1] = r.y;
            }
        }
        float cand[8];
        float mx = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const float2 dv = rnd2<T>(f2(acc[i], acc[i + 1]));               // the conv's stored delta
            const float2 x = add2(f2(xa[i], xa[i + 1]), dv);                 // reconstruct x (Eq.3)
            const float2 cd = sub2(actf2<ACT>(x), f2(ya[i], ya[i + 1]));     // restore the delta
            xa[i] = x.x;
            xa[i + 1] = x.y;
            cand[i] = cd.x;
            cand[i + 1] = cd.y;
            mx = fmaxf(mx, fmaxf(fabsf(cd.x), fabsf(cd.y)));
        }
        ST_CHECK(orow > 0 && orow < d.site_nrows);
        if (CR && on) RowIO<T, 8>::store(CR + (int64_t)orow * C + c0, acc);
        mx = gmax<G == 3 ? 4 : G>(mx, gmask);
        if (mx > theta) {                                      // truncation
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                const float2 r = rnd2<T>(f2(cand[i], cand[i + 1]));
                const float2 y = add2(f2(ya[i], ya[i + 1]), r);
                cand[i] = r.x;
                cand[i + 1] = r.y;
                ya[i] = y.x;
                ya[i + 1] = y.y;
            }
            if (on) RowIO<T, 8>::store(SR + (int64_t)orow * C + c0, cand);
            emit |= 1u << t;
        } else if (d.zero_gaps && on) {                        // a rowmap conv reads this slot as a row
            const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            RowIO<T, 8>::store(SR + (int64_t)orow * C + c0, z);
        }
        orow++;
    }
    if (lane == 0) d.site_act[bq] = emit;
}

static int dw_sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// team form: one CTA of ceil(C/256) warps per pixel; one wave of resident CTAs
// walks the pixels interleaved (active pixels cluster in space)
template <int KMAX, int TB, class T, int ACT>
static void launch_team_k(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int64_t BNo = (int64_t)c.B * c.g.Hout * c.g.Wout;
    const int NW = (c.g.Cin + 255) / 256;
    static int per_sm[DWT_MAXNW + 1] = {};
    if (!per_sm[NW]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[NW], k_dwconv_site_team<KMAX, TB, T, ACT>, 32 * NW, 0);
        if (per_sm[NW] <= 0) per_sm[NW] = 1;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(BNo, (int64_t)dw_sm_count() * per_sm[NW]));
    k_dwconv_site_team<KMAX, TB, T, ACT><<<grid, 32 * NW, 0, s>>>(c, d);
}

template <int KMAX, int CPL, class T, int ACT>
static void launch_seqs_k(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int64_t BNo = (int64_t)c.B * c.g.Hout * c.g.Wout;
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dwconv_site_seqs<KMAX, 4, CPL, T, ACT>,
                                                      32 * DWS_SEQS_WARPS, 0);
        if (per_sm <= 0) per_sm = 1;
    }
    const int64_t want = (BNo + DWS_SEQS_WARPS - 1) / DWS_SEQS_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)dw_sm_count() * per_sm));
    k_dwconv_site_seqs<KMAX, 4, CPL, T, ACT><<<grid, 32 * DWS_SEQS_WARPS, 0, s>>>(c, d);
}

template <int KMAX, class T, int ACT>
static void launch_seq_k(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int64_t BNo = (int64_t)c.B * c.g.Hout * c.g.Wout;
    const int NW = (c.g.Cin + 255) / 256;
    static int per_sm[DWT_MAXNW + 1] = {};
    if (!per_sm[NW]) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[NW], k_dwconv_site_seq<KMAX, 4, T, ACT>, 32 * NW, 0);
        if (per_sm[NW] <= 0) per_sm[NW] = 1;
    }
    // ST_DWT_OCC: fraction of the resident capacity the persistent grid takes
    // (below 1 leaves room for the overlapped dense pass)
    const char *oc = getenv("ST_DWT_OCC");
    const double occ = oc ? atof(oc) : 1.0;
    const int64_t cap = std::max<int64_t>(1, (int64_t)(dw_sm_count() * per_sm[NW] * occ));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(BNo, cap));
    k_dwconv_site_seq<KMAX, 4, T, ACT><<<grid, 32 * NW, 0, s>>>(c, d);
}

template <class T, int ACT>
static void launch_team_t(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    // ST_DWT_TB: 0 (default) = the sequential-pipeline kernel; 2 / 4 = the
    // frame-pair kernel with that many active taps per load batch (x 2 frames)
    const char *tb = getenv("ST_DWT_TB");
    const int tbv = tb ? atoi(tb) : 0;
    const bool tb4 = tbv == 4;
    if (tbv != 2 && tbv != 4 && (int64_t)c.B * c.g.Hout * c.g.Wout < (1ll << 31)) {   // row indices are int32 (pbase)
        // ST_DW_STRIDED=1: the channel-strided warp form for C <= 64 (opt-in: cfg5's
        // 540x960x32 layer 4.0 -> 6.3 ms against the narrow form, cfg3's 0.70 -> 0.95)
        const char *sv = getenv("ST_DW_STRIDED");
        if (c.g.Cin <= 64 && sv && sv[0] == '1') {
            const bool k9 = c.g.kh * c.g.kw <= 9;
            if (c.g.Cin <= 32) {
                if (k9) launch_seqs_k<9, 1, T, ACT>(c, d, s);
                else launch_seqs_k<25, 1, T, ACT>(c, d, s);
            } else {
                if (k9) launch_seqs_k<9, 2, T, ACT>(c, d, s);
                else launch_seqs_k<25, 2, T, ACT>(c, d, s);
            }
            return;
        }
        if (c.g.kh * c.g.kw <= 9) launch_seq_k<9, T, ACT>(c, d, s);
        else launch_seq_k<25, T, ACT>(c, d, s);
        return;
    }
    if (c.g.kh * c.g.kw <= 9) {
        if (tb4) launch_team_k<9, 4, T, ACT>(c, d, s);
        else launch_team_k<9, 2, T, ACT>(c, d, s);
    } else {
        if (tb4) launch_team_k<25, 4, T, ACT>(c, d, s);
        else launch_team_k<25, 2, T, ACT>(c, d, s);
    }
}

void launch_dwconv_site_team(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    if (c.bf) {
        if (d.act == ACT_RELU) launch_team_t<bf16, ACT_RELU>(c, d, s);
        else launch_team_t<bf16, ACT_SILU_FAST>(c, d, s);   // BF16 mode: the fast SiLU of the site kernels
    } else {
        if (d.act == ACT_RELU) launch_team_t<float, ACT_RELU>(c, d, s);
        else launch_team_t<float, ACT_SILU>(c, d, s);
    }
}


// tile form: C <= 32 (C % 8 == 0), k x k <= 9, stride <= 2 (footprint <= 17 x 33)
template <int G, class T, int ACT>
static void launch_tile_k(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int TW = G >= 4 ? 8 : 16, TH = (256 / G) / TW;
    const int ntx = (c.g.Wout + TW - 1) / TW, nty = (c.g.Hout + TH - 1) / TH;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_dwconv_site_tile<G, T, ACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, DWT_TILE_STG);
        attr = true;
    }
    k_dwconv_site_tile<G, T, ACT><<<c.B * ntx * nty, 256, DWT_TILE_STG, s>>>(c, d, TH, TW);
}

template <class T, int ACT>
static void launch_tile_t(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    const int C = c.g.Cin;
    if (C <= 8) launch_tile_k<1, T, ACT>(c, d, s);
    else if (C <= 16) launch_tile_k<2, T, ACT>(c, d, s);
    else launch_tile_k<4, T, ACT>(c, d, s);
}

bool dwconv_site_tile_ok(const Geo &g) {
    if (g.Cin > 32 || g.Cin % 8 != 0 || g.kh * g.kw > 9 || g.sh > 2 || g.sw > 2) return false;
    const int G = g.Cin <= 8 ? 1 : g.Cin <= 16 ? 2 : 4;
    const int TW = G >= 4 ? 8 : 16, TH = (256 / G) / TW;
    return (TH - 1) * g.sh + g.kh <= 17 && (TW - 1) * g.sw + g.kw <= 33;
}

void launch_dwconv_site_tile(const ConvCall &c, const DwSite &d, cudaStream_t s) {
    if (c.bf) {
        if (d.act == ACT_RELU) launch_tile_t<bf16, ACT_RELU>(c, d, s);
        else launch_tile_t<bf16, ACT_SILU_FAST>(c, d, s);
    } else {
        if (d.act == ACT_RELU) launch_tile_t<float, ACT_RELU>(c, d, s);
        else launch_tile_t<float, ACT_SILU>(c, d, s);
    }
}

}  // namespace st
