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
#include <cstdlib>

#include <math_constants.h>

#include "rowio.cuh"

namespace st {

// ---- (i-a) dense channel sums: sums[b][c] += sum_p x[b][p][c]  (fp64;
// four independent partial sums per lane keep four loads in flight)
__global__ void __launch_bounds__(256) k_se_colsum(const float *__restrict__ x, int N, int C, int ppb,
                                                   double *__restrict__ sums) {
    st_pdl_enter();
    const int b = blockIdx.z, c = blockIdx.y * 32 + (threadIdx.x & 31), w = threadIdx.x >> 5;
    const int p0 = blockIdx.x * ppb;
    const int p1 = min(N, p0 + ppb);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (c < C) {
        const float *xb = x + (int64_t)b * N * C + c;
        int p = p0 + w;
        for (; p + 24 < p1; p += 32) {
            const float v0 = __ldg(xb + (int64_t)p * C), v1 = __ldg(xb + (int64_t)(p + 8) * C);
            const float v2 = __ldg(xb + (int64_t)(p + 16) * C), v3 = __ldg(xb + (int64_t)(p + 24) * C);
            a0 += (double)v0;
            a1 += (double)v1;
            a2 += (double)v2;
            a3 += (double)v3;
        }
        for (; p < p1; p += 8) a0 += (double)__ldg(xb + (int64_t)p * C);
    }
    __shared__ double red[8][32];
    red[w][threadIdx.x & 31] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (w == 0 && c < C) {
        double s = 0.0;
        for (int i = 0; i < 8; i++) s += red[i][threadIdx.x];
        atomicAdd(sums + (int64_t)b * C + c, s);
    }
}

// ---- (i-b) per-frame channel sums of the delta rows: dsum[b][t][c] (fp64).
// Each warp reads 32 frame words at once and walks the active pixels of the
// ballot (lanes = 32 channels of the block's channel slice).
template <class T>
__global__ void __launch_bounds__(256) k_se_delta_sums(DView in, int N, int C, int F, int ppb,
                                                       double *__restrict__ dsum) {
    st_pdl_enter();
    extern __shared__ double sacc[];   // [8 warps][32 frames][32 lanes]
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.y * 32 + lane;
    double *my = sacc + w * 32 * 32;
    for (int t = 0; t < 32; t++) my[t * 32 + lane] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    for (int pw = p0 + w * 32; pw < p1; pw += 8 * 32) {
        const int p = pw + lane;
        const int64_t bp = (int64_t)b * N + p;
        const uint32_t a_l = p < p1 ? __ldg(in.act + bp) : 0u;
        uint32_t bal = __ballot_sync(0xffffffffu, a_l != 0);
        const int base_l = a_l ? 1 + __ldg(in.pbase + bp) : 0;
        const uint32_t sl_l = a_l ? __ldg(in.slot + bp) : 0u;
        while (bal) {
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            uint32_t a = __shfl_sync(0xffffffffu, a_l, src);
            const int base = __shfl_sync(0xffffffffu, base_l, src);
            const uint32_t sl = __shfl_sync(0xffffffffu, sl_l, src);
            while (a) {
                const int t1 = __ffs(a) - 1;
                a &= a - 1;
                const int64_t row = base + __popc(sl & lowmask(t1));
                if (c < C) my[t1 * 32 + lane] += (double)ldr<T>(rows + row * C + c);
            }
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

// ---- (i-b') the same sums, thread-per-(frame, 8-channel group): thread
// (t, cg) accumulates frame t's rows of its 8 channels in fp64 registers
// while the CTA sweeps its pixel range; the frame words / slots / row bases
// of 256 pixels are staged in shared memory and every active (pixel, t) row
// slice is one 16-byte vector load, consecutive threads reading consecutive
// pieces of a row (rows of a pixel are contiguous), several pixels in flight.
// Exact fp64 sums of bf16 / fp32 values do not depend on the order (R8).
template <class T>
__global__ void __launch_bounds__(256) k_se_delta_sums_v(DView in, int N, int C, int F, int ppb, int CS,
                                                         double *__restrict__ dsum) {
    st_pdl_enter();
    __shared__ uint32_t m_act[256], m_sl[256];
    __shared__ int32_t m_row[256];
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, ncg = CS / 8;
    const int t = threadIdx.x / ncg, cg = threadIdx.x - (threadIdx.x / ncg) * ncg;
    const int c0 = blockIdx.y * CS + cg * 8;
    const bool mine = t < F && c0 < C;   // C % 8 == 0
    const uint32_t tbit = mine ? 1u << t : 0u;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    for (int pb = p0; pb < p1; pb += 256) {
        const int p = pb + threadIdx.x;
        uint32_t a = 0, sl = 0;
        int r1 = 0;
        if (p < p1) {
            const int64_t bp = (int64_t)b * N + p;
            a = __ldg(in.act + bp);
            if (a) {
                sl = __ldg(in.slot + bp);
                r1 = 1 + __ldg(in.pbase + bp);
            }
        }
        m_act[threadIdx.x] = a;
        m_sl[threadIdx.x] = sl;
        m_row[threadIdx.x] = r1;
        __syncthreads();
        const int np = mine ? min(256, p1 - pb) : 0;   // threads without a (frame, channel group) only stage
        for (int k0 = 0; k0 < np; k0 += 8) {
            float v[8][8];
            uint32_t on = 0;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int k = k0 + u;
                const bool o = k < np && (m_act[k] & tbit);
                on |= (uint32_t)o << u;
                const int64_t row = o ? m_row[k] + __popc(m_sl[k] & lowmask(t)) : 0;   // row 0 = zeros
                RowIO<T, 8>::load(rows + row * C + (mine ? c0 : 0), v[u]);
            }
            if (on) {
#pragma unroll
                for (int u = 0; u < 8; u++)
#pragma unroll
                    for (int i = 0; i < 8; i++) acc[i] += (double)v[u][i];   // zeros where off
            }
        }
        __syncthreads();
    }
    if (mine)
#pragma unroll
        for (int i = 0; i < 8; i++)
            if (acc[i] != 0.0) atomicAdd(dsum + ((int64_t)b * F + t) * C + c0 + i, acc[i]);
}

// ---- (i-b'') the same sums over ACTIVE pixels only: the CTA compacts the
// active pixels of each 256-pixel batch of its range (frame word, slot, row
// base) into shared memory; thread (replica, t, cg) walks every R-th entry
// of the list and adds frame t's row (8 channels, one 16-byte load) of the
// entries active at t into fp64 registers, several entries per batch in
// flight; the R replica partials meet in shared memory at the end.  Threads
// = R x F x (CS / 8) <= 256, so short chunks do not idle most of the CTA.
template <class T>
__global__ void __launch_bounds__(256) k_se_delta_sums_c(DView in, int N, int C, int F, int ppb, int CS, int R,
                                                         double *__restrict__ dsum) {
    st_pdl_enter();
    __shared__ uint32_t m_act[256], m_sl[256];
    __shared__ int32_t m_row[256];
    __shared__ int n_list;
    extern __shared__ double part[];   // [R][F][CS]
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, ncg = CS / 8;
    const int per = F * ncg;
    const int rep = threadIdx.x / per, rem = threadIdx.x - rep * per;
    const int t = rem / ncg, cg = rem - t * ncg;
    const int c0 = blockIdx.y * CS + cg * 8;
    const bool mine = rep < R && c0 < C;   // C % 8 == 0
    const uint32_t tbit = 1u << t;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int wcount[8];
    for (int pb = p0; pb < p1; pb += 256) {
        const int p = pb + threadIdx.x;
        uint32_t a = 0;
        const int64_t bp = (int64_t)b * N + p;
        if (p < p1) a = __ldg(in.act + bp);
        // ordered compaction of the batch's active pixels
        const uint32_t bal = __ballot_sync(0xffffffffu, a != 0);
        if (lane == 0) wcount[wid] = __popc(bal);
        __syncthreads();
        int off = 0;
        for (int w = 0; w < wid; w++) off += wcount[w];
        if (a) {
            const int k = off + __popc(bal & ((1u << lane) - 1u));
            m_act[k] = a;
            m_sl[k] = __ldg(in.slot + bp);
            m_row[k] = 1 + __ldg(in.pbase + bp);
        }
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < 8; w++) tot += wcount[w];
            n_list = tot;
        }
        __syncthreads();
        const int nl = n_list;
        if (mine) {
            for (int k0 = rep; k0 < nl; k0 += 4 * R) {
                float v[4][8];
                bool on[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int k = k0 + u * R;
                    on[u] = k < nl && (m_act[k] & tbit);
                    if (on[u]) RowIO<T, 8>::load(rows + (int64_t)(m_row[k] + __popc(m_sl[k] & lowmask(t))) * C + c0, v[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (on[u])
#pragma unroll
                        for (int i = 0; i < 8; i++) acc[i] += (double)v[u][i];
            }
        }
        __syncthreads();   // list reused by the next batch
    }
    if (mine)
#pragma unroll
        for (int i = 0; i < 8; i++) part[((size_t)rep * F + t) * CS + cg * 8 + i] = acc[i];
    __syncthreads();
    for (int j = threadIdx.x; j < F * CS; j += blockDim.x) {
        const int tt = j / CS, cc = blockIdx.y * CS + (j - tt * CS);
        if (cc >= C) continue;
        double sum = 0.0;
        for (int r = 0; r < R; r++) sum += part[((size_t)r * F) * CS + j];
        if (sum != 0.0) atomicAdd(dsum + ((int64_t)b * F + tt) * C + cc, sum);
    }
}

// ---- (i-b4) the same sums from per-frame row lists: the CTA bins the
// active (pixel, frame) rows of each 256-pixel batch by frame in shared
// memory (ordered: per frame a ballot rank inside the warp plus the earlier
// warps' counts, so a list is in pixel order and the sums are reproducible),
// then thread (replica, t, 8-channel group) adds every R-th row of frame t's
// list -- only rows that exist are loaded (the sweep forms above test every
// pixel of the batch for every frame), four in flight per thread.
template <class T>
__global__ void __launch_bounds__(256) k_se_delta_sums_f(DView in, int N, int C, int F, int ppb, int CS, int R,
                                                         double *__restrict__ dsum) {
    st_pdl_enter();
    extern __shared__ double part[];                    // [R][F][CS], then the lists [F][256] int32
    int *lst = reinterpret_cast<int *>(part + (size_t)R * F * CS);
    __shared__ int wcnt[8][32], foff[8][32], fcnt[32];
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, ncg = CS / 8;
    const int per = F * ncg;
    const int rep = threadIdx.x / per, rem = threadIdx.x - rep * per;
    const int t = rem / ncg, cg = rem - t * ncg;
    const int c0 = blockIdx.y * CS + cg * 8;
    const bool mine = rep < R && c0 < C;   // C % 8 == 0
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int pb = p0; pb < p1; pb += 256) {
        const int p = pb + threadIdx.x;
        uint32_t a = 0, sl = 0;
        int r1 = 0;
        if (p < p1) {
            const int64_t bp = (int64_t)b * N + p;
            a = __ldg(in.act + bp);
            if (a) {
                sl = __ldg(in.slot + bp);
                r1 = 1 + __ldg(in.pbase + bp);
            }
        }
        for (int f = 0; f < F; f++) {
            const uint32_t bal = __ballot_sync(0xffffffffu, (a >> f) & 1u);
            if (lane == 0) wcnt[wid][f] = __popc(bal);
        }
        __syncthreads();
        if (threadIdx.x < F) {
            int o = 0;
            for (int w = 0; w < 8; w++) {
                foff[w][threadIdx.x] = o;
                o += wcnt[w][threadIdx.x];
            }
            fcnt[threadIdx.x] = o;
        }
        __syncthreads();
        for (int f = 0; f < F; f++) {   // uniform loop: the ballot again gives this lane's rank at f
            const uint32_t bal = __ballot_sync(0xffffffffu, (a >> f) & 1u);
            if ((a >> f) & 1u)
                lst[f * 256 + foff[wid][f] + __popc(bal & lowmask(lane))] = r1 + __popc(sl & lowmask(f));
        }
        __syncthreads();
        if (mine) {
            const int n = fcnt[t];
            const int *L = lst + t * 256;
            for (int k0 = rep; k0 < n; k0 += 4 * R) {
                float v[4][8];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int k = k0 + u * R;
                    const int row = k < n ? L[k] : 0;   // row 0 = zeros
                    ST_CHECK(row >= 0 && row < in.nrows);
                    RowIO<T, 8>::load(rows + (int64_t)row * C + c0, v[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int i = 0; i < 8; i++) acc[i] += (double)v[u][i];
            }
        }
        __syncthreads();   // lists reused by the next batch
    }
    if (mine)
#pragma unroll
        for (int i = 0; i < 8; i++) part[((size_t)rep * F + t) * CS + cg * 8 + i] = acc[i];
    __syncthreads();
    for (int j = threadIdx.x; j < F * CS; j += blockDim.x) {
        const int tt = j / CS, cc = blockIdx.y * CS + (j - tt * CS);
        if (cc >= C) continue;
        double sum = 0.0;
        for (int r = 0; r < R; r++) sum += part[((size_t)r * F) * CS + j];
        if (sum != 0.0) atomicAdd(dsum + ((int64_t)b * F + tt) * C + cc, sum);
    }
}

// ---- (i-b3) the same sums with uniform control flow: the CTA compacts the
// active pixels of each 256-pixel batch (frame word, slot, row base) into
// shared memory; warp w owns frames t = w, w + 8, ... and walks the list --
// for an entry active at t every lane adds its channels of the row (lane l:
// channels c0 + l + 32 i, one coalesced 64-byte load per i) into fp64
// registers.  Channel chunks of 256 (CPL <= 8) for wide layers.
template <int CPL, class T>
__global__ void __launch_bounds__(256) k_se_delta_sums_w(DView in, int N, int C, int F, int ppb,
                                                         double *__restrict__ dsum) {
    st_pdl_enter();
    __shared__ uint32_t m_act[256], m_sl[256];
    __shared__ int32_t m_row[256];
    __shared__ int wcount[8];
    const T *rows = static_cast<const T *>(in.rows);
    const int b = blockIdx.z, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c0 = blockIdx.y * 32 * CPL;
    constexpr int FW = 4;   // frames per warp (F <= 32)
    double acc[FW][CPL];
#pragma unroll
    for (int f = 0; f < FW; f++)
#pragma unroll
        for (int i = 0; i < CPL; i++) acc[f][i] = 0.0;
    const int p0 = blockIdx.x * ppb, p1 = min(N, p0 + ppb);
    for (int pb = p0; pb < p1; pb += 256) {
        const int p = pb + threadIdx.x;
        const int64_t bp = (int64_t)b * N + p;
        const uint32_t a = p < p1 ? __ldg(in.act + bp) : 0u;
        const uint32_t bal = __ballot_sync(0xffffffffu, a != 0);
        if (lane == 0) wcount[wid] = __popc(bal);
        __syncthreads();
        int off = 0, nl = 0;
        for (int w = 0; w < 8; w++) {
            off += w < wid ? wcount[w] : 0;
            nl += wcount[w];
        }
        if (a) {
            const int k = off + __popc(bal & ((1u << lane) - 1u));
            m_act[k] = a;
            m_sl[k] = __ldg(in.slot + bp);
            m_row[k] = 1 + __ldg(in.pbase + bp);
        }
        __syncthreads();
#pragma unroll
        for (int f = 0; f < FW; f++) {
            const int t = wid + 8 * f;
            if (t >= F) break;
            for (int k = 0; k < nl; k++) {
                const uint32_t ak = m_act[k];
                if (!((ak >> t) & 1u)) continue;
                const int64_t row = m_row[k] + __popc(m_sl[k] & lowmask(t));
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    const int ch = c0 + lane + 32 * i;
                    if (ch < C) acc[f][i] += (double)ldr<T>(rows + row * C + ch);
                }
            }
        }
        __syncthreads();   // list reused by the next batch
    }
#pragma unroll
    for (int f = 0; f < FW; f++) {
        const int t = wid + 8 * f;
        if (t >= F) break;
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            const int ch = c0 + lane + 32 * i;
            if (ch < C && acc[f][i] != 0.0) atomicAdd(dsum + ((int64_t)b * F + t) * C + ch, acc[f][i]);
        }
    }
}

// gate of one chunk from fp32 means m[C] (block-wide; hid/gate in smem)
// SE_WCH: channels of W1 staged per round (row stride SE_WCH + 1: conflict-free)
constexpr int SE_WCH = 128;
__device__ void se_gate_block(const float *m, int C, int H, const float *w1, const float *b1, const float *w2,
                              const float *b2, float *hid, float *gate, float *wbuf) {
    if (H <= (int)blockDim.x) {
        // W1 staged through shared memory in SE_WCH-channel rounds (coalesced,
        // all threads loading): the per-output fmaf chain over c ascending is
        // unchanged, but its operands no longer wait on one global load each
        const int j = threadIdx.x;
        float acc = 0.0f;
        for (int c0 = 0; c0 < C; c0 += SE_WCH) {
            const int cw = min(SE_WCH, C - c0);
            for (int i = threadIdx.x; i < H * cw; i += blockDim.x) {
                const int jj = i / cw, k = i - jj * cw;
                wbuf[jj * (SE_WCH + 1) + k] = __ldg(w1 + (int64_t)jj * C + c0 + k);
            }
            __syncthreads();
            if (j < H)
                for (int k = 0; k < cw; k++) acc = fmaf(wbuf[j * (SE_WCH + 1) + k], m[c0 + k], acc);
            __syncthreads();
        }
        if (j < H) hid[j] = silu_f(__fadd_rn(acc, __ldg(b1 + j)));
    } else {
        for (int j = threadIdx.x; j < H; j += blockDim.x) {
            float acc = 0.0f;
            for (int c = 0; c < C; c++) acc = fmaf(__ldg(w1 + (int64_t)j * C + c), m[c], acc);
            hid[j] = silu_f(__fadd_rn(acc, __ldg(b1 + j)));
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float acc = 0.0f;
        for (int j = 0; j < H; j++) acc = fmaf(__ldg(w2 + (int64_t)c * H + j), hid[j], acc);
        gate[c] = sigm_f(__fadd_rn(acc, __ldg(b2 + c)));
    }
    __syncthreads();
}

// ---- (ii-a) gates of every frame, one CTA per (frame t, chunk b): the means
// mean_t = (sum0 + dsum_1 + ... + dsum_t) / N do not depend on the refresh
// decisions, so the F+1 gate evaluations run in parallel.  The running sum
// is accumulated in frame order (as the sequential schedule would).
__global__ void __launch_bounds__(1024) k_se_gates(const double *__restrict__ sum0, const double *__restrict__ dsum,
                                                  int N, int C, int H, int F, const float *w1, const float *b1,
                                                  const float *w2, const float *b2, int t0, float *__restrict__ gate_tab) {
    st_pdl_enter();
    extern __shared__ float sm[];
    float *mean = sm;          // [C]
    float *hid = mean + C;     // [H]
    float *wbuf = hid + H;     // [H][SE_WCH + 1] (H <= blockDim.x)
    const int t = t0 + blockIdx.x, b = blockIdx.y;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        double run = sum0[(int64_t)b * C + c];
        for (int t1 = 0; t1 < t; t1++) run += dsum[((int64_t)b * F + t1) * C + c];
        mean[c] = (float)(run / (double)N);
    }
    __syncthreads();
    se_gate_block(mean, C, H, w1, b1, w2, b2, hid, gate_tab + ((int64_t)b * (F + 1) + t) * C, wbuf);
}

// ---- (ii-b) refresh schedule, one CTA per chunk (frames sequential):
// s_tab[b][t][c] = s_emit in force at frame t (t = 0: reference gate);
// refresh[b] bit t-1 = refresh at t.
__global__ void __launch_bounds__(1024) k_se_schedule(const float *__restrict__ gate_tab, int C, int F,
                                                     const float *__restrict__ theta_p, float *__restrict__ s_tab,
                                                     uint32_t *__restrict__ refresh) {
    st_pdl_enter();
    const float theta = __ldg(theta_p);
    extern __shared__ float semit[];   // [C]
    __shared__ float red[32];
    __shared__ int do_refresh;
    const int b = blockIdx.x;
    const float *gt = gate_tab + (int64_t)b * (F + 1) * C;
    float *st = s_tab + (int64_t)b * (F + 1) * C;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        semit[c] = gt[c];
        st[c] = gt[c];
    }
    uint32_t bits = 0;
    for (int t1 = 0; t1 < F; t1++) {
        __syncthreads();
        const float *g = gt + (int64_t)(t1 + 1) * C;
        float mx = 0.0f;
        for (int c = threadIdx.x; c < C; c += blockDim.x) mx = fmaxf(mx, fabsf(__fsub_rn(g[c], semit[c])));
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
            for (int c = threadIdx.x; c < C; c += blockDim.x) semit[c] = g[c];
        }
        __syncthreads();
        for (int c = threadIdx.x; c < C; c += blockDim.x) st[(int64_t)(t1 + 1) * C + c] = semit[c];
    }
    if (threadIdx.x == 0) refresh[b] = bits;
}

// dense reference SE: y0 = x0 * s_tab[b][0]; grid (pixel blocks, chunk),
// float4 over channels when C % 4 == 0.  y (fp32) and ybf (its bf16 shadow,
// read by a tensor-core conv in dense mode) are each optional: an SE whose
// consumers are all tensor-core convs gets only the shadow (BF16 mode)
__global__ void k_se_dense_apply(const float *__restrict__ x, const float *__restrict__ s_tab, int N, int C, int F,
                                 float *__restrict__ y, bf16 *__restrict__ ybf) {
    st_pdl_enter();
    const int b = blockIdx.y;
    const float *sb = s_tab + (int64_t)b * (F + 1) * C;
    const int64_t n = (int64_t)N * C;
    const float *xb = x + (int64_t)b * n;
    float *yb = y ? y + (int64_t)b * n : nullptr;
    bf16 *hb = ybf ? ybf + (int64_t)b * n : nullptr;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if ((C & 3) == 0) {
        const int64_t n4 = n >> 2;
        const int C4 = C >> 2;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
            const int c = (int)(i % C4) * 4;
            const float4 v = __ldg(reinterpret_cast<const float4 *>(xb) + i);
            const float4 sc = __ldg(reinterpret_cast<const float4 *>(sb + c));
            float4 o;
            o.x = __fmul_rn(v.x, sc.x);
            o.y = __fmul_rn(v.y, sc.y);
            o.z = __fmul_rn(v.z, sc.z);
            o.w = __fmul_rn(v.w, sc.w);
            if (yb) reinterpret_cast<float4 *>(yb)[i] = o;
            if (hb) {
                uint2 u;
                u.x = RowIO<bf16, 2>::pack(o.x, o.y);
                u.y = RowIO<bf16, 2>::pack(o.z, o.w);
                reinterpret_cast<uint2 *>(hb)[i] = u;
            }
        }
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            const float o = __fmul_rn(xb[i], __ldg(sb + (int)(i % C)));
            if (yb) yb[i] = o;
            if (hb) hb[i] = __float2bfloat16_rn(o);
        }
    }
}

// slot[b][p] = act[b][p] | refresh[b]
__global__ void k_se_slots(const uint32_t *__restrict__ act, const uint32_t *__restrict__ refresh, int N, int64_t n,
                           uint32_t *__restrict__ slot) {
    st_pdl_enter();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) slot[i] = act[i] | refresh[i / N];
}

// ---- (iii) SE site pixel loop
template <int G, int CPL, class T>
__global__ void __launch_bounds__(256) k_se_site(DView in, const float *__restrict__ x0, const float *__restrict__ s_tab,
                                                 int N, int C, int F, int64_t BN, const float *__restrict__ theta_p,
                                                 const uint32_t *__restrict__ slot, const int32_t *__restrict__ pbase,
                                                 uint32_t *__restrict__ out_act, T *__restrict__ out_rows,
                                                 bool zero_gaps) {
    st_pdl_enter();
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
        const int b = BN < (1ll << 31) ? (int)bp / N : (int)(bp / N);   // 32-bit division when it fits
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
            } else if (zero_gaps) {   // a rowmap conv reads this slot as a row
                const int64_t orow = obase + __popc(Tw & lowmask(t1));
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + G * i < C) str<T>(out_rows + orow * C + lane + G * i, 0.0f);
            }
        }
        if (lane == 0) out_act[bp] = emit;
    }
}

// ---- (iii') SE site pixel loop, C % 8 == 0: lane l of a pixel's group owns
// the CPL consecutive channels [l*CPL, (l+1)*CPL) and moves x0, the delta
// rows and the frame's gate as 16-byte vectors (rowio.cuh); the rows of the
// next P touched frames are fetched together; while pixel k runs, the touched
// word of pixel k+2 and the metadata + x0 of pixel k+1 are in flight.  Same
// per-channel operations in the same order as k_se_site (FP32 bit-exact).
template <int G, int CPL, class T>
__global__ void __launch_bounds__(256) k_se_site_v(DView in, const float *__restrict__ x0,
                                                   const float *__restrict__ s_tab, int N, int C, int F, int64_t BN,
                                                   const float *__restrict__ theta_p, const uint32_t *__restrict__ slot,
                                                   const int32_t *__restrict__ pbase, uint32_t *__restrict__ out_act,
                                                   T *__restrict__ out_rows, bool zero_gaps) {
    st_pdl_enter();
    constexpr int P = CPL <= 8 ? 2 : 1;   // frames prefetched per batch (~16 values per lane)
    const float theta = __ldg(theta_p);
    const T *rows = static_cast<const T *>(in.rows);
    const int lane = threadIdx.x & (G - 1);
    const int c0 = lane * CPL;
    const bool full = c0 + CPL <= C;   // C % 8 == 0: whole or past C
    const unsigned mask = group_mask<G>();
    const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / G;
    int64_t bp = grp;
    uint32_t T_nx = bp < BN ? __ldg(slot + bp) : 0u;
    uint32_t a_nx = 0, isl_nx = 0;
    int ib_nx = 0, ob_nx = 0;
    float x_nx[CPL];
    auto meta = [&](int64_t q, uint32_t Tw) {
        if (!Tw) return;
        a_nx = __ldg(in.act + q);
        ib_nx = a_nx ? 1 + __ldg(in.pbase + q) : 0;
        isl_nx = a_nx ? __ldg(in.slot + q) : 0u;
        ob_nx = 1 + __ldg(pbase + q);
        row_load<float, CPL>(x0 + q * C, c0, C, full, x_nx);
    };
    meta(bp, T_nx);
    uint32_t T_nn = bp + ngrp < BN ? __ldg(slot + bp + ngrp) : 0u;
    for (; bp < BN; bp += ngrp) {
        const uint32_t Tw = T_nx, a = a_nx, isl = isl_nx;
        const int ibase = ib_nx, obase = ob_nx;
        float xa[CPL], ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) xa[i] = x_nx[i];
        const int64_t b1 = bp + ngrp;
        T_nx = T_nn;
        meta(b1, T_nx);
        T_nn = b1 + ngrp < BN ? __ldg(slot + b1 + ngrp) : 0u;
        if (!Tw) {
            if (lane == 0) out_act[bp] = 0;
            continue;
        }
        const int b = BN < (1ll << 31) ? (int)bp / N : (int)(bp / N);   // 32-bit division when it fits
        const float *st = s_tab + (int64_t)b * (F + 1) * C;
        {
            float s0[CPL];
            row_load<float, CPL>(st, c0, C, full, s0);
#pragma unroll
            for (int i = 0; i < CPL; i++) ya[i] = __fmul_rn(xa[i], s0[i]);   // y0 = x0 * s_emit(0)
        }
        uint32_t bits = Tw, emit = 0;
        while (bits) {
            int t1s[P];
            float v[P][CPL], sn[P][CPL];
#pragma unroll
            for (int j = 0; j < P; j++) {   // the next P touched frames (absent: row 0 = zeros)
                const int t1 = __ffs(bits) - 1;
                t1s[j] = t1;
                bits &= bits - 1;
                const int64_t irow = (t1 >= 0 && ((a >> t1) & 1u)) ? ibase + __popc(isl & lowmask(t1)) : 0;
                row_load<T, CPL>(rows + irow * C, c0, C, full, v[j]);
                row_load<float, CPL>(st + (int64_t)(t1 >= 0 ? t1 + 1 : 0) * C, c0, C, full, sn[j]);
            }
#pragma unroll
            for (int j = 0; j < P; j++) {
                const int t1 = t1s[j];
                if (t1 < 0) continue;
                const bool act = (a >> t1) & 1u;
                float cand[CPL];
                float mx = 0.0f;
                if constexpr (CPL % 2 == 0) {   // fp32x2 pairs: the scalar form's bits per lane
#pragma unroll
                    for (int i = 0; i < CPL; i += 2) {
                        float2 x = f2(xa[i], xa[i + 1]);
                        if (act) x = add2(x, f2(v[j][i], v[j][i + 1]));
                        const float2 cd = sub2(mul2(x, f2(sn[j][i], sn[j][i + 1])), f2(ya[i], ya[i + 1]));
                        xa[i] = x.x;
                        xa[i + 1] = x.y;
                        cand[i] = cd.x;
                        cand[i + 1] = cd.y;
                        mx = fmaxf(mx, fmaxf(fabsf(cd.x), fabsf(cd.y)));
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < CPL; i++) {
                        if (act) xa[i] = __fadd_rn(xa[i], v[j][i]);
                        cand[i] = __fsub_rn(__fmul_rn(xa[i], sn[j][i]), ya[i]);
                        mx = fmaxf(mx, fabsf(cand[i]));
                    }
                }
                mx = gmax<G>(mx, mask);
                if (mx > theta) {
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
                    if (c0 < C) row_store<T, CPL>(out_rows + (obase + __popc(Tw & lowmask(t1))) * (int64_t)C, c0, C,
                                                  full, cand);
                    emit |= 1u << t1;
                } else if (zero_gaps && c0 < C) {   // a rowmap conv reads this slot as a row
                    float z[CPL];
#pragma unroll
                    for (int i = 0; i < CPL; i++) z[i] = 0.0f;
                    row_store<T, CPL>(out_rows + (obase + __popc(Tw & lowmask(t1))) * (int64_t)C, c0, C, full, z);
                }
            }
        }
        if (lane == 0) out_act[bp] = emit;
    }
}

// ---- (iii'') SE site for wide layers (C > 1280, C % 8 == 0: the expanded
// stages of EfficientNet-B4..B6): one warp per pixel, x_acc /
// y_acc in shared memory, 256-channel chunks (8 per lane).  Per touched frame
// pass 1 adds the delta and takes the running max of |x_acc * s - y_acc|; on
// emission pass 2 recomputes the candidate from the stored state (same
// operations, same bits), rounds it, advances y_acc and writes the row.
constexpr int SE_WIDE_WARPS = 4;
template <class T>
__global__ void __launch_bounds__(32 * SE_WIDE_WARPS) k_se_site_wide(DView in, const float *__restrict__ x0,
                                                                     const float *__restrict__ s_tab, int N, int C,
                                                                     int F, int64_t BN, const float *__restrict__ theta_p,
                                                                     const uint32_t *__restrict__ slot,
                                                                     const int32_t *__restrict__ pbase,
                                                                     uint32_t *__restrict__ out_act,
                                                                     T *__restrict__ out_rows, bool zero_gaps) {
    st_pdl_enter();
    extern __shared__ float sew_sm[];
    const float theta = __ldg(theta_p);
    const T *rows = static_cast<const T *>(in.rows);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *xs = sew_sm + (size_t)wid * 2 * C, *ys = xs + C;
    for (int64_t bp = (int64_t)blockIdx.x * SE_WIDE_WARPS + wid; bp < BN; bp += (int64_t)gridDim.x * SE_WIDE_WARPS) {
        const uint32_t Tw = __ldg(slot + bp);
        if (!Tw) {
            if (lane == 0) out_act[bp] = 0;
            continue;
        }
        const int b = BN < (1ll << 31) ? (int)bp / N : (int)(bp / N);   // 32-bit division when it fits
        const float *st = s_tab + (int64_t)b * (F + 1) * C;
        const uint32_t a = __ldg(in.act + bp);
        const int ibase = a ? 1 + __ldg(in.pbase + bp) : 0;
        const uint32_t isl = a ? __ldg(in.slot + bp) : 0u;
        const int obase = 1 + __ldg(pbase + bp);
        for (int c0 = lane * 8; c0 < C; c0 += 256) {
            float x[8], s0[8], y[8];
            RowIO<float, 8>::load(x0 + bp * C + c0, x);
            RowIO<float, 8>::load(st + c0, s0);
#pragma unroll
            for (int i = 0; i < 8; i++) y[i] = __fmul_rn(x[i], s0[i]);   // y0 = x0 * s_emit(0)
            RowIO<float, 8>::store(xs + c0, x);
            RowIO<float, 8>::store(ys + c0, y);
        }
        uint32_t bits = Tw, emit = 0;
        while (bits) {
            const int t1 = __ffs(bits) - 1;
            bits &= bits - 1;
            const bool act = (a >> t1) & 1u;
            const int64_t irow = act ? ibase + __popc(isl & lowmask(t1)) : 0;
            const float *s_now = st + (int64_t)(t1 + 1) * C;
            float mx = 0.0f;
            for (int c0 = lane * 8; c0 < C; c0 += 256) {
                float x[8], y[8], v[8], sn[8];
                RowIO<float, 8>::load(xs + c0, x);
                RowIO<float, 8>::load(ys + c0, y);
                RowIO<float, 8>::load(s_now + c0, sn);
                if (act) {
                    RowIO<T, 8>::load(rows + irow * C + c0, v);
#pragma unroll
                    for (int i = 0; i < 8; i++) x[i] = __fadd_rn(x[i], v[i]);
                    RowIO<float, 8>::store(xs + c0, x);
                }
#pragma unroll
                for (int i = 0; i < 8; i++) mx = fmaxf(mx, fabsf(__fsub_rn(__fmul_rn(x[i], sn[i]), y[i])));
            }
            mx = gmax<32>(mx, 0xffffffffu);
            if (mx > theta) {
                const int64_t orow = obase + __popc(Tw & lowmask(t1));
                for (int c0 = lane * 8; c0 < C; c0 += 256) {
                    float x[8], y[8], sn[8], e[8];
                    RowIO<float, 8>::load(xs + c0, x);
                    RowIO<float, 8>::load(ys + c0, y);
                    RowIO<float, 8>::load(s_now + c0, sn);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        e[i] = rnd<T>(__fsub_rn(__fmul_rn(x[i], sn[i]), y[i]));
                        y[i] = __fadd_rn(y[i], e[i]);
                    }
                    RowIO<float, 8>::store(ys + c0, y);
                    RowIO<T, 8>::store(out_rows + orow * C + c0, e);
                }
                emit |= 1u << t1;
            } else if (zero_gaps) {   // a rowmap conv reads this slot as a row
                const int64_t orow = obase + __popc(Tw & lowmask(t1));
                const float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int c0 = lane * 8; c0 < C; c0 += 256) RowIO<T, 8>::store(out_rows + orow * C + c0, z);
            }
        }
        if (lane == 0) out_act[bp] = emit;
    }
}

void launch_se_colsum(const float *x, int B, int N, int C, double *sum0, cudaStream_t s) {
    cudaMemsetAsync(sum0, 0, (size_t)B * C * 8, s);
    const int ppb = 1024;
    dim3 grid(cdiv(N, ppb), cdiv(C, 32), B);
    k_se_colsum<<<grid, 256, 0, s>>>(x, N, C, ppb, sum0);
}

// threads per block of the per-chunk gate kernels: one CTA per (frame, chunk)
// or per chunk, latency-bound chains -- wide layers spread over 1024 threads
static int se_threads(int C) { return C > 256 ? 1024 : 256; }

void launch_se_schedule(const double *sum0, const double *dsum, int B, int N, int C, int H, int F, const float *w1,
                        const float *b1, const float *w2, const float *b2, const float *theta, float *gate_tab,
                        float *s_tab, uint32_t *refresh, cudaStream_t s) {
    const int nth = se_threads(C);
    const size_t smem = (size_t)(C + H + (H <= nth ? H * (SE_WCH + 1) : 0)) * 4;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_se_gates, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_se_gates<<<dim3(F + 1, B), nth, smem, s>>>(sum0, dsum, N, C, H, F, w1, b1, w2, b2, 0, gate_tab);
    static size_t attr2 = 0;
    const size_t smem2 = (size_t)C * 4;
    if (smem2 > 48 * 1024 && smem2 > attr2) {
        cudaFuncSetAttribute(k_se_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        attr2 = smem2;
    }
    k_se_schedule<<<B, se_threads(C), smem2, s>>>(gate_tab, C, F, theta, s_tab, refresh);
}

void launch_se_gates(const double *sum0, const double *dsum, int B, int N, int C, int H, int F, const float *w1,
                     const float *b1, const float *w2, const float *b2, int t0, int nt, float *gate_tab, cudaStream_t s) {
    if (nt <= 0) return;
    const int nth = se_threads(C);
    const size_t smem = (size_t)(C + H + (H <= nth ? H * (SE_WCH + 1) : 0)) * 4;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaFuncSetAttribute(k_se_gates, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    k_se_gates<<<dim3(nt, B), nth, smem, s>>>(sum0, dsum, N, C, H, F, w1, b1, w2, b2, t0, gate_tab);
}

void launch_se_sched(const float *gate_tab, int B, int C, int F, const float *theta, float *s_tab, uint32_t *refresh,
                     cudaStream_t s) {
    static size_t attr2 = 0;
    const size_t smem2 = (size_t)C * 4;
    if (smem2 > 48 * 1024 && smem2 > attr2) {
        cudaFuncSetAttribute(k_se_schedule, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        attr2 = smem2;
    }
    k_se_schedule<<<B, se_threads(C), smem2, s>>>(gate_tab, C, F, theta, s_tab, refresh);
}

void launch_se_dense_apply(const float *x, const float *s_tab, int B, int N, int C, int F, float *y, void *ybf,
                           cudaStream_t s) {
    const int64_t n = (int64_t)N * C / ((C & 3) == 0 ? 4 : 1);
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16 / std::max(B, 1) + 1));
    if (n > 0 && B > 0) k_se_dense_apply<<<dim3(gx, B), 256, 0, s>>>(x, s_tab, N, C, F, y, static_cast<bf16 *>(ybf));
}

template <class T>
static void se_delta_sums_t(DView in, int B, int N, int C, int F, double *dsum, cudaStream_t s) {
    const int ppb = 2048;
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
    if (C % 8 == 0 && F >= 1 && F <= 32) {
        // channel slice: as many 8-channel groups as fit 256 threads at F frames
        const int CS = std::max(8, std::min((C + 7) / 8 * 8, (256 / F) * 8));
        // pixels per block: enough blocks for two waves of the 148 SMs (small
        // late-stage maps otherwise ran 32 blocks), 256-pixel granules, <= 2048
        const int nsl = cdiv(C, CS);
        const int want = std::max(1, 296 / std::max(1, nsl * B));
        const int ppb = std::min(2048, std::max(256, (cdiv(N, want) + 255) / 256 * 256));
        dim3 grid(cdiv(N, ppb), cdiv(C, CS), B);
        const int R = std::max(1, 256 / (F * (CS / 8)));   // replicas of the (t, cg) threads
        const size_t sm = (size_t)R * F * CS * sizeof(double);
        // 3 (default): per-frame row lists (cfg5 delta sums 4.2 -> 2.0 ms per step);
        // 0: the per-(frame, channel group) sweep; 1 / 2: compacted-pixel forms
        const char *mv = getenv("ST_SE_SUMS");   // read per launch (graph capture): tests switch it
        const int mode = mv ? atoi(mv) : 3;
        if (mode == 2) {   // warp per frame over the compacted active pixels
            const int cpl = std::min(8, (C + 31) / 32);
            dim3 gw(cdiv(N, ppb), cdiv(C, 32 * (cpl == 3 ? 4 : cpl > 4 ? 8 : cpl)), B);
            if (cpl == 1) {
                if (bf) k_se_delta_sums_w<1, bf16><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
                else k_se_delta_sums_w<1, float><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
            } else if (cpl == 2) {
                if (bf) k_se_delta_sums_w<2, bf16><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
                else k_se_delta_sums_w<2, float><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
            } else if (cpl <= 4) {
                if (bf) k_se_delta_sums_w<4, bf16><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
                else k_se_delta_sums_w<4, float><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
            } else {
                if (bf) k_se_delta_sums_w<8, bf16><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
                else k_se_delta_sums_w<8, float><<<gw, 256, 0, s>>>(in, N, C, F, ppb, dsum);
            }
            return;
        }
        const size_t smf = sm + (size_t)F * 256 * 4;
        if (mode == 3 && smf <= 200 * 1024) {
            static size_t attr = 0;
            if (smf > 48 * 1024 && smf > attr) {
                cudaFuncSetAttribute(k_se_delta_sums_f<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf);
                cudaFuncSetAttribute(k_se_delta_sums_f<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smf);
                attr = smf;
            }
            if (bf) k_se_delta_sums_f<bf16><<<grid, 256, smf, s>>>(in, N, C, F, ppb, CS, R, dsum);
            else k_se_delta_sums_f<float><<<grid, 256, smf, s>>>(in, N, C, F, ppb, CS, R, dsum);
            return;
        }
        if (mode == 1 && sm <= 48 * 1024) {
            if (bf) k_se_delta_sums_c<bf16><<<grid, 256, sm, s>>>(in, N, C, F, ppb, CS, R, dsum);
            else k_se_delta_sums_c<float><<<grid, 256, sm, s>>>(in, N, C, F, ppb, CS, R, dsum);
            return;
        }
        if (bf) k_se_delta_sums_v<bf16><<<grid, 256, 0, s>>>(in, N, C, F, ppb, CS, dsum);
        else k_se_delta_sums_v<float><<<grid, 256, 0, s>>>(in, N, C, F, ppb, CS, dsum);
        return;
    }
    if (bf) se_delta_sums_t<bf16>(in, B, N, C, F, dsum, s);
    else se_delta_sums_t<float>(in, B, N, C, F, dsum, s);
}

void launch_se_slots(const uint32_t *act, const uint32_t *refresh, int B, int N, uint32_t *slot, cudaStream_t s) {
    const int64_t n = (int64_t)B * N;
    k_se_slots<<<cdiv(n, 256), 256, 0, s>>>(act, refresh, N, n, slot);
}

void launch_se_site(DView in, const float *x0, const float *s_tab, int B, int N, int C, int F, const float *theta, bool bf,
                    const uint32_t *slot, const int32_t *pbase, uint32_t *out_act, void *out_rows, cudaStream_t s,
                    bool zero_gaps) {
    const int64_t BN = (int64_t)B * N;
    auto grid_for = [&](int G) {
        return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(BN * G, 256), 148 * 8));
    };
    if (C % 8 == 0 && C > 1280) {   // wide layers: state in shared memory
        const size_t sm = (size_t)SE_WIDE_WARPS * 2 * C * sizeof(float);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(BN, SE_WIDE_WARPS), 148 * 8));
#define L_SEW                                                                                               \
    {                                                                                                       \
        cudaFuncSetAttribute(k_se_site_wide<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);      \
        k_se_site_wide<T><<<grid, 32 * SE_WIDE_WARPS, sm, s>>>(in, x0, s_tab, N, C, F, BN, theta, slot, pbase, \
                                                              out_act, static_cast<T *>(out_rows), zero_gaps); \
    }
        ST_ROW_DISPATCH(bf, L_SEW);
#undef L_SEW
        return;
    }
    if (C % 8 == 0 && C <= 1280) {   // vectorised blocked form
#define L_SEV(G_, CPL_)                                                                                          \
    k_se_site_v<G_, CPL_, T><<<resident_grid(k_se_site_v<G_, CPL_, T>, 256, 0, cdiv(BN * G_, 256), 148 * 8), 256, 0, s>>>( \
        in, x0, s_tab, N, C, F, BN, theta, slot, pbase, out_act, static_cast<T *>(out_rows), zero_gaps)
#define SEV_CH                            \
    if (C <= 8) L_SEV(1, 8);              \
    else if (C <= 16) L_SEV(2, 8);        \
    else if (C <= 32) L_SEV(4, 8);        \
    else if (C <= 64) L_SEV(8, 8);        \
    else if (C <= 128) L_SEV(16, 8);      \
    else if (C <= 256) L_SEV(32, 8);      \
    else if (C <= 512) L_SEV(32, 16);     \
    else if (C <= 768) L_SEV(32, 24);     \
    else L_SEV(32, 40);
        ST_ROW_DISPATCH(bf, SEV_CH);
#undef SEV_CH
#undef L_SEV
        return;
    }
#define L_SE(G_, CPL_)                                                                                      \
    k_se_site<G_, CPL_, T><<<grid_for(G_), 256, 0, s>>>(in, x0, s_tab, N, C, F, BN, theta, slot, pbase, out_act, \
                                                        static_cast<T *>(out_rows), zero_gaps)
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
