// kernels_mask.cu -- Subtraction, truncation, mask dilation and ordered
// compaction on sm_100a.
//
// Subtraction + pixel-granular truncation
// (readings R1-R3): per pixel, sequential over diff frames with the
// Subtraction buffer S in registers, raw = X_t - S, active iff
// max_c |raw| > theta_0, S += raw when active.  Masks are pixel-major frame
// words (one uint32 per pixel, bit t-1 = frame t) so a warp reads 32
// consecutive pixels' words with one coalesced 128-byte load and a pixel's
// frames are one register.  Compaction is an ordered exclusive scan of
// popc(word) -- deterministic, no atomics on the data path.
#include "rowio.cuh"

namespace st {

// ------------------------------------------------------------ subtraction
// Frame element -> fp32: float frames as they are; uint8 frames v / 255.0f
// (reading R20; IEEE division, the same value the fp32 input path receives).
__device__ __forceinline__ float frame_val(const float *p, const float *) { return __ldg(p); }
// uint8: the value v / 255.0f (IEEE division) from a per-CTA table of the
// 256 quotients -- the same bits, without a division per element
__device__ __forceinline__ float frame_val(const uint8_t *p, const float *tab) { return tab[__ldg(p)]; }
__device__ __forceinline__ void fill_u8_table(float *tab) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tab[i] = __fdiv_rn((float)i, 255.0f);
    __syncthreads();
}

template <int C, class T, class FT>
__global__ void __launch_bounds__(256) k_subtract_mask(const float *__restrict__ ref, int64_t ref_stride,
                                                       const FT *__restrict__ fr, int64_t fr_stride, int B,
                                                       int N, int n_diff, const float *__restrict__ theta_p,
                                                       uint32_t *__restrict__ act, T *__restrict__ ddelta) {
    st_pdl_enter();
    __shared__ float u8tab[256];
    if (sizeof(FT) == 1) fill_u8_table(u8tab);
    const float theta = __ldg(theta_p);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * N) return;
    const int b = (int)(i / N), p = (int)(i % N);
    const float *r = ref + b * ref_stride + (int64_t)p * C;
    float S[C];
#pragma unroll
    for (int c = 0; c < C; c++) S[c] = __ldg(r + c);
    const FT *f = fr + b * fr_stride + (int64_t)p * C;
    const int64_t fs = (int64_t)N * C;
    // optional dense per-frame copy of the emitted delta [B][n_diff][N][C]
    // (zeros where truncated) for convs that read the input directly
    // channel-padded to 4 (one aligned 8-byte bf16 piece per pixel; zeros in
    // the pad channels) so tensor-core stems gather a tap with one copy
    T *dd = ddelta ? ddelta + ((int64_t)b * n_diff * N + p) * 4 : nullptr;
    const int64_t dfs = (int64_t)N * 4;
    uint32_t w = 0;
#pragma unroll 4
    for (int t1 = 0; t1 < n_diff; ++t1) {
        float raw[C];
        float mx = 0.0f;
#pragma unroll
        for (int c = 0; c < C; c++) {
            raw[c] = __fsub_rn(frame_val(f + t1 * fs + c, u8tab), S[c]);
            mx = fmaxf(mx, fabsf(raw[c]));
        }
        const bool on = mx > theta;             // R1: strict comparison
        float e4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c = 0; c < C; c++) {
            const float e = on ? rnd<T>(raw[c]) : 0.0f;
            if (on) S[c] = __fadd_rn(S[c], e);  // R3: S += emitted
            e4[c] = e;
        }
        if (dd) RowIO<T, 4>::store(dd + t1 * dfs, e4);   // one 8-byte (bf16) / 16-byte (fp32) store
        if (on) w |= 1u << t1;
    }
    act[i] = w;
}

template <int C, class T, class FT>
__global__ void __launch_bounds__(256) k_subtract_rows(const float *__restrict__ ref, int64_t ref_stride,
                                                       const FT *__restrict__ fr, int64_t fr_stride, int B,
                                                       int N, const uint32_t *__restrict__ act,
                                                       const int32_t *__restrict__ pbase, T *__restrict__ rows,
                                                       float *s_save) {
    st_pdl_enter();
    __shared__ float u8tab[256];
    if (sizeof(FT) == 1) fill_u8_table(u8tab);
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * N) return;
    uint32_t w = act[i];
    if (!w) return;
    const int b = (int)(i / N), p = (int)(i % N);
    const float *r = ref + b * ref_stride + (int64_t)p * C;
    float S[C];
#pragma unroll
    for (int c = 0; c < C; c++) S[c] = __ldg(r + c);
    const FT *f = fr + b * fr_stride + (int64_t)p * C;
    const int64_t fs = (int64_t)N * C;
    T *o = rows + (int64_t)(1 + pbase[i]) * C;
    while (w) {
        const int t1 = __ffs(w) - 1;
        w &= w - 1;
#pragma unroll
        for (int c = 0; c < C; c++) {
            const float e = rnd<T>(__fsub_rn(frame_val(f + t1 * fs + c, u8tab), S[c]));   // emitted delta
            S[c] = __fadd_rn(S[c], e);
            str<T>(o + c, e);
        }
        o += C;
    }
    if (s_save)
#pragma unroll
        for (int c = 0; c < C; c++) s_save[i * C + c] = S[c];
}

#define SUB_DISPATCH(C_, KERNEL, FT, FR, ...)                                                               \
    switch (C_) {                                                                                           \
    case 1: KERNEL<1, T, FT><<<grid, 256, 0, s>>>(ref, ref_stride, static_cast<const FT *>(FR), __VA_ARGS__); break; \
    case 2: KERNEL<2, T, FT><<<grid, 256, 0, s>>>(ref, ref_stride, static_cast<const FT *>(FR), __VA_ARGS__); break; \
    case 3: KERNEL<3, T, FT><<<grid, 256, 0, s>>>(ref, ref_stride, static_cast<const FT *>(FR), __VA_ARGS__); break; \
    case 4: KERNEL<4, T, FT><<<grid, 256, 0, s>>>(ref, ref_stride, static_cast<const FT *>(FR), __VA_ARGS__); break; \
    default: break;                                                                                         \
    }

void launch_subtract_mask(const float *ref, int64_t ref_stride, const void *frames, bool u8, int64_t fr_stride,
                          int B, int N, int C, int n_diff, const float *theta_p, bool bf, uint32_t *act, void *ddelta,
                          cudaStream_t s) {
    const int grid = cdiv((int64_t)B * N, 256);
    if (u8)
        ST_ROW_DISPATCH(bf, SUB_DISPATCH(C, k_subtract_mask, uint8_t, frames, fr_stride, B, N, n_diff, theta_p, act,
                                         static_cast<T *>(ddelta)));
    else
        ST_ROW_DISPATCH(bf, SUB_DISPATCH(C, k_subtract_mask, float, frames, fr_stride, B, N, n_diff, theta_p, act,
                                         static_cast<T *>(ddelta)));
}

void launch_subtract_rows(const float *ref, int64_t ref_stride, const void *frames, bool u8, int64_t fr_stride,
                          int B, int N, int C, const uint32_t *act, const int32_t *pbase, void *rows, bool bf,
                          float *s_save, cudaStream_t s) {
    const int grid = cdiv((int64_t)B * N, 256);
    if (u8)
        ST_ROW_DISPATCH(bf, SUB_DISPATCH(C, k_subtract_rows, uint8_t, frames, fr_stride, B, N, act, pbase,
                                         static_cast<T *>(rows), s_save));
    else
        ST_ROW_DISPATCH(bf, SUB_DISPATCH(C, k_subtract_rows, float, frames, fr_stride, B, N, act, pbase,
                                         static_cast<T *>(rows), s_save));
}

// uint8 frames -> fp32 v / 255.0f (reading R20): the staged reference frames
__global__ void __launch_bounds__(256) k_u8_to_f32(const uint8_t *__restrict__ src, int64_t src_stride,
                                                   int64_t per, int n, float *__restrict__ dst) {
    st_pdl_enter();
    const int64_t tot = per * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / per, k = i - c * per;
        dst[i] = __fdiv_rn((float)__ldg(src + c * src_stride + k), 255.0f);
    }
}

void launch_u8_to_f32(const uint8_t *src, int64_t src_stride, int64_t per, int n, float *dst, cudaStream_t s) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(per * n, 256), 148 * 16));
    k_u8_to_f32<<<grid, 256, 0, s>>>(src, src_stride, per, n, dst);
}

// --------------------------------------------------------------- dilation
__global__ void __launch_bounds__(256) k_dilate(const uint32_t *__restrict__ in, int B, Geo g,
                                                uint32_t *__restrict__ out) {
    st_pdl_enter();
    const int No = g.Hout * g.Wout;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)B * No) return;
    const int b = (int)(i / No), q = (int)(i % No);
    const int oy = q / g.Wout, ox = q % g.Wout;
    const uint32_t *src = in + (int64_t)b * g.Hin * g.Win;
    uint32_t w = 0;
    for (int dy = 0; dy < g.kh; dy++) {
        const int iy = oy * g.sh - g.ph + dy;
        if (iy < 0 || iy >= g.Hin) continue;
        for (int dx = 0; dx < g.kw; dx++) {
            const int ix = ox * g.sw - g.pw + dx;
            if (ix < 0 || ix >= g.Win) continue;
            w |= __ldg(src + iy * g.Win + ix);
        }
    }
    out[i] = w;
}

void launch_dilate(const uint32_t *in, int B, const Geo &g, uint32_t *out, cudaStream_t s) {
    const int64_t n = (int64_t)B * g.Hout * g.Wout;
    k_dilate<<<cdiv(n, 256), 256, 0, s>>>(in, B, g, out);
}

// ------------------------------------------------------------------- scan
constexpr int SCAN_T = 256, SCAN_E = 8, SCAN_TILE = SCAN_T * SCAN_E;

int64_t scan_tmp_ints(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE + 2; }

__device__ __forceinline__ int block_excl_scan(int v, int *warp_sums, int &block_total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int ws = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += y;
        }
        if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = ws;
    }
    __syncthreads();
    block_total = warp_sums[(blockDim.x >> 5) - 1];
    const int res = (wid ? warp_sums[wid - 1] : 0) + x - v;
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(SCAN_T) k_scan1(const uint32_t *__restrict__ w, int64_t n, int32_t *tmp) {
    st_pdl_enter();
    __shared__ int ws[32];
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * SCAN_E;
    int s = 0;
#pragma unroll
    for (int e = 0; e < SCAN_E; e++)
        if (base + e < n) s += __popc(__ldg(w + base + e));
    int tot;
    block_excl_scan(s, ws, tot);
    if (threadIdx.x == 0) tmp[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan2(int32_t *tmp, int nb, int32_t *total, long long *stat,
                                                long long *peak) {
    st_pdl_enter();
    __shared__ int ws[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? tmp[i] : 0;
        int tot;
        const int ex = block_excl_scan(v, ws, tot);
        if (i < nb) tmp[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *total = carry;
        if (stat) atomicAdd((unsigned long long *)stat, (unsigned long long)carry);
        if (peak) atomicMax(peak, (long long)carry);
    }
}

// Row capacity (reading of SURVEY §8(a) a9: buffers sized from measured
// occupancy): a word whose rows would end past `cap` is cleared -- with the
// ordered prefix, exactly the words from the first one that does not fit on
// -- so no kernel of the step writes past the buffer; the first cleared
// word's offset becomes the tensor's total and *ovf is raised (the step's
// results are invalid; the host re-plans and re-issues it).
__device__ __forceinline__ bool fits_cap(uint32_t *w, int64_t i, int off, int c, int64_t cap, int32_t *total,
                                         int32_t *ovf) {
    if ((int64_t)off + c <= cap) return true;
    if (c) {
        w[i] = 0u;
        if ((int64_t)off <= cap) {   // the first word that does not fit (unique)
            *total = off;
            *ovf = 1;
        }
    }
    return false;
}

// ridx (optional): the conv M-row list, ((b*N+q) << 5) | (t-1) for every set
// bit in (b, p, t) order -- enumerated here from the word's own offset
__device__ __forceinline__ void emit_codes(uint32_t w, int64_t i, int off, int32_t *ridx) {
    int32_t *o = ridx + off;
    const int32_t code = (int32_t)(i << 5);
    while (w) {
        const int t1 = __ffs(w) - 1;
        w &= w - 1;
        *o++ = code | t1;
    }
}

__global__ void __launch_bounds__(SCAN_T) k_scan3(uint32_t *w, int64_t n, const int32_t *__restrict__ tmp,
                                                  int32_t *__restrict__ pbase, int32_t *__restrict__ ridx,
                                                  int64_t cap, int32_t *total, int32_t *ovf) {
    st_pdl_enter();
    __shared__ int ws[32];
    const int64_t base = blockIdx.x * (int64_t)SCAN_TILE + threadIdx.x * SCAN_E;
    int c[SCAN_E];
    int s = 0;
#pragma unroll
    for (int e = 0; e < SCAN_E; e++) {
        c[e] = base + e < n ? __popc(w[base + e]) : 0;
        s += c[e];
    }
    int tot;
    int off = block_excl_scan(s, ws, tot) + tmp[blockIdx.x];
#pragma unroll
    for (int e = 0; e < SCAN_E; e++) {
        if (base + e < n) {
            pbase[base + e] = off;
            if (fits_cap(w, base + e, off, c[e], cap, total, ovf) && ridx && c[e])
                emit_codes(w[base + e], base + e, off, ridx);
        }
        off += c[e];
    }
}

// one CTA for small word arrays: the whole scan (+ optional enumeration) in
// one launch instead of scan1 / scan2 / scan3 / enumerate
constexpr int SCAN_SMALL_T = 1024, SCAN_SMALL_MAX = 2048;   // larger arrays: the enumeration parallelises better over 3 passes
__global__ void __launch_bounds__(SCAN_SMALL_T) k_scan_small(uint32_t *w, int64_t n, int32_t *__restrict__ pbase,
                                                             int32_t *total, long long *stat,
                                                             int32_t *__restrict__ ridx, int64_t cap, int32_t *ovf,
                                                             long long *peak) {
    st_pdl_enter();
    __shared__ int ws[32];
    int carry = 0;
    for (int64_t b0 = 0; b0 < n; b0 += (int64_t)SCAN_SMALL_T * 4) {
        const int64_t base = b0 + threadIdx.x * 4;
        uint32_t v[4];
        int c[4], sum = 0;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            v[e] = base + e < n ? w[base + e] : 0u;
            c[e] = __popc(v[e]);
            sum += c[e];
        }
        int tot;
        int off = carry + block_excl_scan(sum, ws, tot);
#pragma unroll
        for (int e = 0; e < 4; e++) {
            if (base + e < n) {
                pbase[base + e] = off;
                if (fits_cap(w, base + e, off, c[e], cap, total, ovf) && ridx && c[e]) emit_codes(v[e], base + e, off, ridx);
            }
            off += c[e];
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        if (stat) atomicAdd((unsigned long long *)stat, (unsigned long long)carry);
        if (peak) atomicMax(peak, (long long)carry);
        if ((int64_t)carry <= cap) *total = carry;   // else: set by the first word that did not fit
    }
}

void launch_scan_popc(uint32_t *words, int64_t n, int32_t *pbase, int32_t *total, int32_t *tmp, long long *stat,
                      cudaStream_t s, int32_t *ridx, const ScanCap &cap) {
    const int nb = cdiv(n, SCAN_TILE);
    if (nb == 0) {
        cudaMemsetAsync(total, 0, sizeof(int32_t), s);
        return;
    }
    const int64_t cp = cap.ovf ? cap.cap : INT64_MAX;
    if (n <= SCAN_SMALL_MAX) {
        k_scan_small<<<1, SCAN_SMALL_T, 0, s>>>(words, n, pbase, total, stat, ridx, cp, cap.ovf, cap.peak);
        return;
    }
    k_scan1<<<nb, SCAN_T, 0, s>>>(words, n, tmp);
    k_scan2<<<1, 1024, 0, s>>>(tmp, nb, total, stat, cap.peak);
    // enumeration in its own pass: one thread per word (up to 32 codes each)
    // parallelises 8x better than the scan's 8-words-per-thread layout
    k_scan3<<<nb, SCAN_T, 0, s>>>(words, n, tmp, pbase, nullptr, cp, total, cap.ovf);
    if (ridx) launch_enumerate(words, pbase, n, ridx, s);
}

// -------------------------------------------------------------- enumerate
__global__ void __launch_bounds__(256) k_enumerate(const uint32_t *__restrict__ slot, const int32_t *__restrict__ pbase,
                                                   int64_t n, int32_t *__restrict__ ridx) {
    st_pdl_enter();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t w = slot[i];
    if (!w) return;
    int32_t *o = ridx + pbase[i];
    const int32_t code = (int32_t)(i << 5);
    while (w) {
        const int t1 = __ffs(w) - 1;
        w &= w - 1;
        *o++ = code | t1;
    }
}

void launch_enumerate(const uint32_t *slot, const int32_t *pbase, int64_t n, int32_t *ridx, cudaStream_t s) {
    k_enumerate<<<cdiv(n, 256), 256, 0, s>>>(slot, pbase, n, ridx);
}

// ----------------------------------------------------------------- counts
constexpr int CNT_E = 8;
// Per-frame popcounts by bit transposition: for each frame bit t a warp
// ballots bit t of its 32 words, so lane t accumulates popc(ballot) -- one
// ballot per word and no per-bit atomics (dense words would otherwise
// serialise on 31 shared counters).
__global__ void __launch_bounds__(256) k_frame_counts(const uint32_t *__restrict__ act, int N, long long *counts,
                                                      int64_t cstride, long long *stat, long long *stat_nz) {
    st_pdl_enter();
    __shared__ int cnt[32];
    __shared__ int nz;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
    if (threadIdx.x == 0) nz = 0;
    __syncthreads();
    const int b = blockIdx.y;
    const uint32_t *a = act + (int64_t)b * N;
    // block covers 256 * CNT_E consecutive words; warp w takes CNT_E runs of 32
    const int64_t base = (int64_t)blockIdx.x * 256 * CNT_E + (int64_t)warp * 32 * CNT_E;
    uint32_t w[CNT_E];
#pragma unroll
    for (int e = 0; e < CNT_E; e++) {
        const int64_t p = base + e * 32 + lane;
        w[e] = p < N ? __ldg(a + p) : 0u;
    }
    int mine = 0, nzw = 0;
#pragma unroll
    for (int e = 0; e < CNT_E; e++) {
        nzw += __popc(__ballot_sync(0xffffffffu, w[e] != 0u));
        uint32_t any = __reduce_or_sync(0xffffffffu, w[e]);
        while (any) {   // only frames with at least one active pixel in these 32 words
            const int t = __ffs(any) - 1;
            any &= any - 1;
            const int cbit = __popc(__ballot_sync(0xffffffffu, (w[e] >> t) & 1u));
            if (lane == t) mine += cbit;
        }
    }
    if (mine) atomicAdd(&cnt[lane], mine);
    if (lane == 0 && nzw) atomicAdd(&nz, nzw);
    __syncthreads();
    if (threadIdx.x < 32) {
        const int v = cnt[threadIdx.x];
        if (v) {
            if (counts) atomicAdd((unsigned long long *)(counts + b * cstride + threadIdx.x), (unsigned long long)v);
            if (stat) atomicAdd((unsigned long long *)stat, (unsigned long long)v);
        }
        if (threadIdx.x == 0 && stat_nz && nz) atomicAdd((unsigned long long *)stat_nz, (unsigned long long)nz);
    }
}

void launch_frame_counts(const uint32_t *act, int B, int N, long long *counts, int64_t cstride, long long *stat,
                         long long *stat_nz, cudaStream_t s) {
    dim3 grid(cdiv(N, 256 * CNT_E), B);
    k_frame_counts<<<grid, 256, 0, s>>>(act, N, counts, cstride, stat, stat_nz);
}

__global__ void k_or_words(const uint32_t *a, const uint32_t *b, int64_t n, uint32_t *o) {
    st_pdl_enter();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) o[i] = a[i] | b[i];
}

void launch_or_words(const uint32_t *a, const uint32_t *b, int64_t n, uint32_t *out, cudaStream_t s) {
    k_or_words<<<cdiv(n, 256), 256, 0, s>>>(a, b, n, out);
}

}  // namespace st
