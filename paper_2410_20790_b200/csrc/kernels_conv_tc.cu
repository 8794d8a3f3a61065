// kernels_conv_tc.cu -- BF16 mode sparse / dense convolution on the 5th-gen
// tensor cores (tcgen05, TMEM accumulators), sm_100a.
//
// Eq.(2) as a gathered implicit GEMM:
//   D[M x Cout] = A[M x K] * B[K x Cout],  K = k_h*k_w*c_in in (dy, dx, ci) order,
// A rows gathered from the compacted bf16 delta rows (sparse) or the fp32
// dense reference activations (dense), B = bf16 weights.  Used where the
// active-row batch is a real dense contraction (3x3 convs of the CRNN and
// ResNet encoders, EfficientNet 1x1 expand/project convs; c_in % 8 == 0, each
// tap's channels zero-padded to a multiple of the 64-wide k-block).
//
// Precision contract of BF16 mode (R22-BF16): operands are bf16
// (delta rows are stored bf16; dense activations and weights are rounded
// RNE when staged), products are exact in fp32, accumulation is fp32 in TMEM;
// sparse outputs are stored as bf16 delta rows, dense outputs as fp32 + bias.
//
// CTA = 9 warps, persistent over (M tile, N tile):
//   warps 0-3  producers: thread m owns A row m of the tile.  Per k-block
//              (64 channels of one tap): sparse -> 8 x cp.async 16 B of the
//              bf16 row into the 128B-swizzled K-major layout (zero-fill for
//              an inactive tap), completion tracked by
//              cp.async.mbarrier.arrive.noinc; dense -> 16 x LDG.128 fp32 ->
//              cvt.bf16x2 -> 8 x STS.128 + fence.proxy.async + arrive.
//              Thread 0 also issues the B tile as one TMA 2D load
//              (box 64 x BN, 128B swizzle) with expect_tx.
//   warp 4     MMA issuer: one lane issues 4 x tcgen05.mma (M=128, N=BN,
//              K=16) per k-block, tcgen05.commit -> empty[s]; after the last
//              k-block commit -> tmem_full[acc].
//   warps 5-8  epilogue: tcgen05.ld 32x32b (TMEM lane = tile row) -> row
//              stores, arrive tmem_empty[acc].
// Stages: 4-deep smem ring; TMEM: 2 accumulators x BN columns.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace st {

namespace tc {

// warps 0-3 producers, 4 MMA issuer, 5 .. 5 + NEPI - 1 epilogue: two warps per
// TMEM lane quarter (each half of the accumulator's 32-column chunks), since
// the epilogue of one CTA per SM bounds the dense and 1x1 convs
constexpr int NEPI = 8;
constexpr int BM = 128, BK = 64, NPROD = 128, NTHREADS = 160 + 32 * NEPI;
constexpr int SMEM_MAX = 232448;   // 227 KB opt-in dynamic shared memory per CTA
constexpr int TAPS = 9;   // max k_h*k_w taken by the tensor-core path (1x1, 2x2, 3x3)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// TMA 2D load multicast to the CTAs of `mask` (same smem offsets in each;
// complete_tx lands on the barrier at the same offset in each destination)
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, int x, int y, uint64_t *bar,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 16-byte cp.async, zero-filled when src_bytes == 0
__device__ __forceinline__ void cp_async16(void *dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
// 8-byte cp.async (.ca), zero-filled when src_bytes == 0
__device__ __forceinline__ void cp_async8(void *dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// commit arriving on the barrier at the same offset in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// 2-SM MMA (issued by the leader CTA of the pair): A rows 0-127 from the
// leader's smem and 128-255 from the peer's, B rows (N) split likewise, D rows
// 0-127 in the leader's TMEM and 128-255 in the peer's (same addresses)
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// completion of the leader's prior 2-SM MMAs -> barrier at this offset in both CTAs
__device__ __forceinline__ void tc_commit2_mc(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}
// arrive (release, cluster scope) on the barrier at this offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// SWIZZLE_128B K-major smem descriptor (sm_100 version 1): start>>4 [0,14),
// LBO>>4 [16,30) (unused for swizzled K-major), SBO>>4 [32,46) = 1024 B
// between 8-row core-matrix groups, version bits [46,48) = 1, layout
// [61,64) = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(16 >> 4) << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, K-major both, N>>3, M>>4.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// 8 independent 16-byte read-only loads issued back to back in one asm
// block (ptxas otherwise chains them through one destination register)
__device__ __forceinline__ void ldg4x8(const float *const (&p)[8], float4 (&v)[8]) {
    asm volatile(
        "ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%32];\n\t"
        "ld.global.nc.v4.f32 {%4,%5,%6,%7}, [%33];\n\t"
        "ld.global.nc.v4.f32 {%8,%9,%10,%11}, [%34];\n\t"
        "ld.global.nc.v4.f32 {%12,%13,%14,%15}, [%35];\n\t"
        "ld.global.nc.v4.f32 {%16,%17,%18,%19}, [%36];\n\t"
        "ld.global.nc.v4.f32 {%20,%21,%22,%23}, [%37];\n\t"
        "ld.global.nc.v4.f32 {%24,%25,%26,%27}, [%38];\n\t"
        "ld.global.nc.v4.f32 {%28,%29,%30,%31}, [%39];"
        : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[0].z), "=f"(v[0].w), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[1].z),
          "=f"(v[1].w), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[2].z), "=f"(v[2].w), "=f"(v[3].x), "=f"(v[3].y),
          "=f"(v[3].z), "=f"(v[3].w), "=f"(v[4].x), "=f"(v[4].y), "=f"(v[4].z), "=f"(v[4].w), "=f"(v[5].x),
          "=f"(v[5].y), "=f"(v[5].z), "=f"(v[5].w), "=f"(v[6].x), "=f"(v[6].y), "=f"(v[6].z), "=f"(v[6].w),
          "=f"(v[7].x), "=f"(v[7].y), "=f"(v[7].z), "=f"(v[7].w)
        : "l"(p[0]), "l"(p[1]), "l"(p[2]), "l"(p[3]), "l"(p[4]), "l"(p[5]), "l"(p[6]), "l"(p[7]));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int BN, bool SITE = false, bool DSTG = false>
struct Smem {
    static constexpr int A_BYTES = BM * BK * 2;          // 16 KB: this CTA's 128 rows of the M=256 tile
    static constexpr int B_BYTES = (BN / 2) * BK * 2;    // this CTA's half of the BN weight rows
    static constexpr int STAGE = A_BYTES + B_BYTES;
    // SITE: the tile's 128 delta rows (bf16, row stride BN + 8 elements) and
    // their row codes, read back by the site step of the epilogue
    static constexpr int SROW = BN + 8;
    static constexpr int SITE_BYTES = SITE ? BM * SROW * 2 + BM * 4 + 64 : 0;
    // DSTG (dense mode): per epilogue warp a 32 x 32 fp32 transpose buffer (row
    // stride 33), so each store instruction writes whole 128-byte row pieces
    static constexpr int DSTG_BYTES = DSTG ? NEPI * 32 * 33 * 4 : 0;
    static constexpr int STAGES_FIT = (SMEM_MAX - 256 - 1024 - SITE_BYTES - DSTG_BYTES) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int SITE_OFF = STAGES * STAGE;
    static constexpr int DSTG_OFF = SITE_OFF + SITE_BYTES;
    static constexpr int BAR_OFF = DSTG_OFF + DSTG_BYTES;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024;   // + barriers, + alignment slack
};

}  // namespace tc

// ---- conv-epilogue non-linear correction (Eq.2 then Eq.3,
// PAPER.md P:124-139).  A sparse conv whose only consumer is a ReLU /
// SiLU site and whose c_out fits one N tile (BN >= c_out) runs the site in
// its epilogue: the tile's 128 delta rows (rounded to the stored bf16 value,
// R22-BF16) go from TMEM to shared memory, the accumulator is released, and
// each epilogue warp takes the pixels that START in its 32-row slice: the
// M rows are in (b, q, t) order, so a pixel's frames are consecutive rows.
// Per pixel (lanes own channels l + 32 i): x_acc from the conv's dense x0,
// y_acc = f(x0); per frame x_acc += Delta; c = f(x_acc) - y_acc; warp max;
// emit iff > theta; y_acc += rnd(c); the emitted row goes to the conv's row
// layout (in place, as the separate site kernel writes it).  The conv's own
// delta rows never reach HBM -- except those of the <= 2 pixels per tile that
// continue into a neighbouring tile, whose rows are written and finished by
// k_tc_site_fixup (one warp per tile boundary).
template <int BN>
__device__ __forceinline__ void site_epilogue(const ConvCall &c, uint32_t taddr, unsigned char *sbuf, int M, int mt,
                                              int quarter, int lane, bool releaser, uint64_t *tempty_bar) {
    using namespace tc;
    using S = Smem<BN, true>;
    constexpr int SR = S::SROW;
    constexpr int CPL = BN / 32;
    bf16 *stg = reinterpret_cast<bf16 *>(sbuf);
    int32_t *codes = reinterpret_cast<int32_t *>(sbuf + BM * SR * 2);
    const int C = c.g.Cout;
    const int rt = quarter * 32 + lane;
    const int r = mt * BM + rt;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint4 *dst = reinterpret_cast<uint4 *>(stg + rt * SR + c0);
#pragma unroll
        for (int j = 0; j < 32; j += 8)
            dst[j / 8] = make_uint4(pack_bf16x2(__uint_as_float(v[j]), __uint_as_float(v[j + 1])),
                                    pack_bf16x2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3])),
                                    pack_bf16x2(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5])),
                                    pack_bf16x2(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7])));
    }
    codes[rt] = r < M ? __ldg(c.ridx + r) : -1;
    tc_fence_before();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (releaser) mbar_arrive_remote(tempty_bar, 0);   // the accumulator is free for the next tile
    // pixels continuing into the previous / next tile (finished by the fix-up kernel)
    const int r0 = mt * BM;
    const int g_first = codes[0] >= 0 ? codes[0] >> 5 : -1;
    const int head = (r0 > 0 && g_first >= 0 && (__ldg(c.ridx + r0 - 1) >> 5) == g_first) ? g_first : -2;
    const int last = min(BM, M - r0) - 1;
    const int g_last = last >= 0 ? codes[last] >> 5 : -1;
    const int tail = (last == BM - 1 && r0 + BM < M && (__ldg(c.ridx + r0 + BM) >> 5) == g_last) ? g_last : -2;
    const int my = codes[rt];
    const int gq = my >= 0 ? my >> 5 : -1;
    bf16 *out = static_cast<bf16 *>(c.out);
    if (gq >= 0 && (gq == head || gq == tail)) {   // straddler: its delta row, as the conv kernel writes it
        const uint4 *src = reinterpret_cast<const uint4 *>(stg + rt * SR);
        for (int j = 0; j < C / 8; j++) reinterpret_cast<uint4 *>(out + (int64_t)(r + 1) * C)[j] = src[j];
    }
    const bool start = gq >= 0 && gq != head && gq != tail && (rt == 0 || (codes[rt - 1] >> 5) != gq);
    uint32_t starts = __ballot_sync(0xffffffffu, start);
    const float theta = __ldg(c.site.theta);
    const int kind = c.site.act;
    // x0 rows (and rowmap touched words) of the next two pixels in flight
    // while the current one is stepped: the dense x0 of scattered pixels is
    // an HBM round trip each
    float p0[CPL], p1[CPL];
    uint32_t tw0 = 0xFFFFFFFFu, tw1 = 0xFFFFFFFFu;
    auto fetch = [&](uint32_t st, float (&dst)[CPL], uint32_t &tw) {
        if (!st) return;
        const int g = codes[quarter * 32 + __ffs(st) - 1] >> 5;
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            const int ch = lane + 32 * i;
            dst[i] = ch < C ? __ldg(c.site.x0 + (int64_t)g * C + ch) : 0.0f;
        }
        tw = c.rowmap ? __ldg(c.a.act + g) : 0xFFFFFFFFu;   // rowmap: gap slots are not touched
    };
    fetch(starts, p0, tw0);
    fetch(starts & (starts - 1), p1, tw1);
    while (starts) {
        const int s = quarter * 32 + __ffs(starts) - 1;
        starts &= starts - 1;
        const int g = codes[s] >> 5;
        const uint32_t touched = tw0;
        float xa[CPL], ya[CPL];
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            xa[i] = p0[i];
            ya[i] = act_rt(kind, xa[i]);
            p0[i] = p1[i];
        }
        tw0 = tw1;
        fetch(starts & (starts - 1), p1, tw1);   // the pixel after the next
        uint32_t emit = 0;
        for (int j = s; j < BM; j++) {
            const int cj = codes[j];
            if (cj < 0 || (cj >> 5) != g) break;
            if (!((touched >> (cj & 31)) & 1u)) {   // gap slot: zero Delta, no site step
                if (c.site.zero_gaps) {
                    bf16 *o = out + (int64_t)(r0 + j + 1) * C;
#pragma unroll
                    for (int i = 0; i < CPL; i++)
                        if (lane + 32 * i < C) o[lane + 32 * i] = __float2bfloat16_rn(0.0f);
                }
                continue;
            }
            float cand[CPL];
            float mx = 0.0f;
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                const int ch = lane + 32 * i;
                const float v = ch < C ? __bfloat162float(stg[j * SR + ch]) : 0.0f;
                xa[i] = __fadd_rn(xa[i], v);                            // reconstruct x (Eq.3)
                cand[i] = __fsub_rn(act_rt(kind, xa[i]), ya[i]);        // restore the delta
                mx = fmaxf(mx, fabsf(cand[i]));
            }
            mx = gmax<32>(mx, 0xffffffffu);
            if (mx > theta) {                                           // truncation
                bf16 *o = out + (int64_t)(r0 + j + 1) * C;
#pragma unroll
                for (int i = 0; i < CPL; i++) {
                    const int ch = lane + 32 * i;
                    cand[i] = bf16_round(cand[i]);
                    ya[i] = __fadd_rn(ya[i], cand[i]);
                    if (ch < C) o[ch] = __float2bfloat16_rn(cand[i]);
                }
                emit |= 1u << (cj & 31);
            } else if (c.site.zero_gaps) {
                bf16 *o = out + (int64_t)(r0 + j + 1) * C;
#pragma unroll
                for (int i = 0; i < CPL; i++)
                    if (lane + 32 * i < C) o[lane + 32 * i] = __float2bfloat16_rn(0.0f);
            }
        }
        if (lane == 0) c.site.words[g] = emit;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");   // shared rows read before the next tile overwrites them
}

// SMALL: convs on the network input with c_in <= 4 (stems).  The input delta
// is the dense per-frame array padded to 4 channels (one aligned 8-byte bf16
// piece per pixel), so a 64-wide k-block holds 16 taps x 4 channels and is
// gathered with 16 x 8-byte cp.async per row -- no frame-word lookups (the
// dense array holds zeros where the Subtraction truncated).  Dense mode
// packs the fp32 reference frame's <= 4 channels into the same layout.
// Weights are [Cout][ceil(taps/16)*64] with tap-major 4-channel pieces.
template <int BN, bool DENSE, bool SMALL = false, bool SITE = false>
__global__ void __launch_bounds__(tc::NTHREADS, 1) k_conv_tc(ConvCall c, const __grid_constant__ CUtensorMap tmap_b,
                                                             const __grid_constant__ CUtensorMap tmap_a) {
    st_pdl_enter();
    using namespace tc;
    using S = Smem<BN, SITE, DENSE>;
    constexpr int STAGES = S::STAGES;
    constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + S::BAR_OFF);   // this CTA's stage landed
    uint64_t *pfull = full + STAGES;     // leader only: the peer's stage landed (relayed)
    uint64_t *empty = pfull + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const Geo g = c.g;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Nin = g.Hin * g.Win, Nout = g.Hout * g.Wout;
    const int M = DENSE ? c.B * Nout : *c.m_dev;
    // K layout (dy, dx, ci) with each tap's channels zero-padded to Cpad, a
    // multiple of the 64-wide k-block (Cpad == c_in when c_in % 64 == 0)
    const int Cpad = (g.Cin + BK - 1) / BK * BK;
    const int nkb = SMALL ? ((c.sr > 0 ? g.kh * c.sr : g.kh * g.kw) + 15) / 16 : g.kh * g.kw * Cpad / BK;
    const int ntn = (g.Cout + BN - 1) / BN;
    // CTA pair (cta_group::2): work item w = (M-tile pair, N tile) is one
    // M=256 x N=BN MMA tile; this CTA stages A rows of M tile 2*pair + rank and
    // weight rows [rank*BN/2, (rank+1)*BN/2) of the N tile, the leader (rank 0)
    // issues the MMAs over both CTAs' shared memory, each CTA's TMEM receives
    // its own 128 rows.
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int mtiles = (M + BM - 1) / BM;
    const int nwork = ((mtiles + 1) >> 1) * ntn;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(full + s, NPROD + 1);   // 128 producer arrivals + the TMA expect_tx arrival
            mbar_init(pfull + s, 1);          // the peer's relay
            mbar_init(empty + s, 1);          // the leader's multicast MMA commit
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(tfull + a, 1);          // the leader's multicast MMA commit
            mbar_init(tempty + a, 2);         // both CTAs' epilogues drained the accumulator
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();   // peer barriers initialised before any multicast targets them
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (SMALL && warp < 4) {
        // ===================== producers (stem, c_in <= 4) =====================
        // A source: the 4-channel-padded bf16 input delta per frame (sparse)
        // or the padded bf16 reference frames (dense); 8 bytes per pixel
        const int m = threadIdx.x;
        int stage = 0;
        uint32_t phase = 0;
        const int ntaps = g.kh * g.kw;
        const bf16 *dd = static_cast<const bf16 *>(DENSE ? c.a_dense_bf : c.ddelta);
        const int wrow0 = warp * 32;
        // sparse: the row code of the next work item is loaded one item ahead,
        // so a tile boundary costs no dependent DRAM round trip (a stem tile
        // is one or a few k-blocks)
        auto row_code = [&](int w) -> int {
            const int r = (2 * (w / ntn) + (int)rank) * BM + m;
            return (!DENSE && w < nwork && r < M) ? __ldg(c.ridx + r) : 0;
        };
        int code_cur = row_code(cid);
        for (int w = cid; w < nwork; w += ncl) {
            const int mt = 2 * (w / ntn) + (int)rank, nt = w % ntn;
            const int r = mt * BM + m;
            const int code_nxt = row_code(w + ncl);
            // this thread's row: input plane (chunk, or chunk x frame) and the
            // receptive-field origin; invalid rows get an origin no tap reaches
            int plane = 0, iy0 = -(1 << 20), ix0 = -(1 << 20);
            if (r < M) {
                int b, q;
                if (DENSE) {
                    b = r / Nout;
                    q = r - b * Nout;
                    plane = b;
                } else {
                    const int code = code_cur;
                    b = (code >> 5) / Nout;
                    q = (code >> 5) - b * Nout;
                    plane = b * c.F + (code & 31);
                }
                const int oy = q / g.Wout, ox = q - oy * g.Wout;
                iy0 = oy * g.sh - g.ph;
                ix0 = ox * g.sw - g.pw;
            }
            // the rows this lane stages are fixed for the whole tile: fetch their
            // plane / origin from the owning lanes once, not once per k-block
            int pl_r[16], iy_r[16], ix_r[16];
#pragma unroll
            for (int i = 0; i < 16; i++) {
                const int rl = c.sr > 0 ? (4 * (i & 7) + (lane >> 3)) : (2 * i + (lane >> 4));
                pl_r[i] = __shfl_sync(0xffffffffu, plane, rl);
                iy_r[i] = __shfl_sync(0xffffffffu, iy0, rl);
                ix_r[i] = __shfl_sync(0xffffffffu, ix0, rl);
            }
            for (int kb = 0; kb < nkb; kb++) {
                mbar_wait(empty + stage, phase ^ 1);
                unsigned char *sa = smem + stage * S::STAGE;
                unsigned char *sb = sa + S::A_BYTES;
                if (c.sr > 0) {
                    // paired layout: lane (l & 7) stages the 16-byte slot pair
                    // p of rows 4i + (l >> 3): pixels (ix, ix+1) of kernel row dy
                    const int p = lane & 7;
                    const int s0 = kb * 16 + 2 * p;
                    const int dy = s0 / c.sr, dxp = s0 - dy * c.sr - c.shift;   // dx of the pair's first pixel
                    const bool sv = dy < g.kh;
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int rl = 4 * i + (lane >> 3), row = wrow0 + rl;
                        const int pl = pl_r[i];
                        const int iy = iy_r[i] + dy;
                        const int ix = ix_r[i] + dxp;   // even
                        const bool valid = sv && iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win;
                        const bf16 *src = dd + (valid ? ((int64_t)pl * Nin + iy * g.Win + ix) * 4 : 0);
                        cp_async16(sa + row * 128 + ((p ^ (row & 7)) << 4), src, valid ? 16u : 0u);
                    }
                } else {
                    // 16 taps per k-block: lane l stages tap (l & 15) of rows 2i + (l >> 4)
                    const int j = lane & 15;
                    const int tap = kb * 16 + j;
                    const bool tv = tap < ntaps;
                    const int dy = tv ? tap / g.kw : 0, dx = tv ? tap - (tap / g.kw) * g.kw : 0;
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int rl = 2 * i + (lane >> 4), row = wrow0 + rl;
                        const int pl = pl_r[i];
                        const int iy = iy_r[i] + dy;
                        const int ix = ix_r[i] + dx;
                        const bool valid = tv && iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win;
                        const int64_t pix = (int64_t)pl * Nin + iy * g.Win + ix;
                        cp_async8(sa + row * 128 + ((((j >> 1) ^ (row & 7)) << 4) | ((j & 1) << 3)),
                                  dd + (valid ? pix * 4 : 0), valid ? 8u : 0u);
                    }
                }
                cp_async_arrive_noinc(full + stage);
                if (m == 0) {   // this CTA's half of the weight tile
                    mbar_arrive_tx(full + stage, S::B_BYTES);
                    tma_load_2d(sb, &tmap_b, kb * BK, nt * BN + (int)rank * (BN / 2), full + stage);
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            code_cur = code_nxt;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp < 4) {
        // ===================== producers =====================
        const int m = threadIdx.x;   // tile row owned by this thread
        int stage = 0;
        uint32_t phase = 0;
        const float *Ad = c.a_dense;
        // bf16 rows gathered with cp.async: the delta rows (sparse), or the bf16
        // shadow of the dense activation when the producer wrote one (dense)
        const bool async_a = !DENSE || c.a_dense_bf != nullptr;
        const bf16 *As = static_cast<const bf16 *>(DENSE ? c.a_dense_bf : c.a.rows);
        const int ntaps = g.kh * g.kw;   // <= TAPS (conv_tc_eligible)
        // Sparse: a tile's tap lookups (frame word, base, slot of each of the
        // <= 9 input pixels) are issued one tile ahead -- while the current
        // tile streams -- and the row code two tiles ahead, so a tile boundary
        // costs no dependent memory round trip (short-K layers have only a
        // few k-blocks per tile).
        uint32_t n_a[TAPS], n_sl[TAPS];
        int n_pb[TAPS], n_t1 = 0;
        auto fetch_taps = [&](int w, int code) {
            const int r = (2 * (w / ntn) + (int)rank) * BM + m;
            const bool ok = w < nwork && r < M;
            const int gq = code >> 5;
            const int b = gq / Nout, q = gq - (gq / Nout) * Nout;
            const int oy = q / g.Wout, ox = q - oy * g.Wout;
            n_t1 = code & 31;
#pragma unroll
            for (int t = 0; t < TAPS; t++) {
                n_a[t] = 0;
                n_sl[t] = 0;
                n_pb[t] = 0;
                if (ok && t < ntaps) {
                    const int dy = t / g.kw, dx = t - dy * g.kw;
                    const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                    if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) {
                        const int64_t bp = (int64_t)b * Nin + iy * g.Win + ix;
                        n_a[t] = __ldg(c.a.act + bp);
                        n_pb[t] = __ldg(c.a.pbase + bp);
                        n_sl[t] = __ldg(c.a.slot + bp);
                    }
                }
            }
        };
        auto code_of = [&](int w) {
            const int r = (2 * (w / ntn) + (int)rank) * BM + m;
            return (w < nwork && r < M) ? __ldg(c.ridx + r) : 0;
        };
        int code_nx = 0;
        const bool rowmap = !DENSE && c.rowmap;   // 1x1/s1: tile row r reads input row r + 1
        if (!DENSE && !rowmap) {
            fetch_taps(cid, code_of(cid));
            code_nx = code_of(cid + ncl);
        }
        for (int w = cid; w < nwork; w += ncl) {
            const int mt = 2 * (w / ntn) + (int)rank, nt = w % ntn;
            const int r = mt * BM + m;
            const bool rv = r < M;
            int tapidx[TAPS];
            if (DENSE) {
                // dense rows are (chunk, pixel): taps are pixel indices
                const int b = rv ? r / Nout : 0, q = rv ? r - b * Nout : 0;
                const int oy = q / g.Wout, ox = q - oy * g.Wout;
#pragma unroll
                for (int t = 0; t < TAPS; t++) {
                    tapidx[t] = -1;
                    if (rv && t < ntaps) {
                        const int dy = t / g.kw, dx = t - dy * g.kw;
                        const int iy = oy * g.sh - g.ph + dy, ix = ox * g.sw - g.pw + dx;
                        if (iy >= 0 && iy < g.Hin && ix >= 0 && ix < g.Win) tapidx[t] = b * Nin + iy * g.Win + ix;
                    }
                }
            } else if (rowmap) {
#pragma unroll
                for (int t = 0; t < TAPS; t++) tapidx[t] = (t == 0 && rv) ? r + 1 : -1;
            } else {
                // this tile's lookups (issued a tile ago) -> delta-row index per tap (-1 = zero)
#pragma unroll
                for (int t = 0; t < TAPS; t++) {
                    tapidx[t] = ((n_a[t] >> n_t1) & 1u) ? 1 + n_pb[t] + __popc(n_sl[t] & lowmask(n_t1)) : -1;
                    ST_CHECK(tapidx[t] < 0 || tapidx[t] < c.a.nrows);
                }
                fetch_taps(w + ncl, code_nx);    // next tile's lookups in flight
                code_nx = code_of(w + 2 * ncl);  // and the row code after that
            }
            // the K loop walks (tap, 64-channel block) without divisions
            int tap = 0, ci0 = 0;
            for (int kb = 0; kb < nkb; kb++) {
                const int nval = min(8, (g.Cin - ci0) >> 3);   // real 8-channel chunks (c_in % 8 == 0)
                int idx = -1;
#pragma unroll
                for (int t = 0; t < TAPS; t++)
                    if (t == tap) idx = tapidx[t];
                const int64_t src = idx >= 0 ? (int64_t)idx * g.Cin : -1;   // element offset, -1 = zero
                const int k0 = kb * BK;
                mbar_wait(empty + stage, phase ^ 1);
                unsigned char *sa = smem + stage * S::STAGE;
                unsigned char *sb = sa + S::A_BYTES;
                // Warp-cooperative, coalesced staging: the warp's 32 rows are
                // moved a few rows per instruction (lanes split a row's
                // 128-byte k-block slice), each row's source index taken from
                // its owner lane by shuffle.  One row per thread would touch
                // 32 lines per instruction (8x the L1tex wavefronts).
                const int wrow0 = warp * 32;
                if (c.tma_a) {
                    // 1x1/s1 with contiguous A rows (dense bf16 shadow, or the
                    // rowmap layout): the tile's 128 rows x 64 channels arrive as
                    // one TMA 2D load into the same 128B-swizzled layout (rows /
                    // channels past the tensor zero-filled); thread 0 issues it
                    // with the weight tile below, the others only arrive
                    if (m == 0) {   // thread 0's producer arrival carries the A bytes
                        mbar_arrive_tx(full + stage, S::A_BYTES);
                        tma_load_2d(sa, &tmap_a, ci0, mt * BM, full + stage);
                    } else {
                        mbar_arrive(full + stage);
                    }
                } else if (!async_a) {
                    // ---- fp32 activations -> bf16 (RNE): 2 rows x 16 float4 per instruction,
                    // two batches of 8 unconditional loads (an invalid source reads a safe
                    // address and is zeroed after), so the loads issue back to back
                    // an absent tap / padding chunk reads the zero block, so no
                    // per-load validity has to stay live (8+ live predicates make
                    // ptxas serialise the loads)
                    float4 v[16];
                    const float *pp[16];
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int rl = 2 * i + (lane >> 4), j4 = lane & 15;
                        const int64_t si = __shfl_sync(0xffffffffu, src, rl);
                        pp[i] = (si >= 0 && (j4 >> 1) < nval) ? Ad + si + ci0 + 4 * j4 : c.zeros + 4 * j4;
                    }
                    ldg4x8(*reinterpret_cast<const float *const(*)[8]>(pp), *reinterpret_cast<float4(*)[8]>(v));
                    ldg4x8(*reinterpret_cast<const float *const(*)[8]>(pp + 8), *reinterpret_cast<float4(*)[8]>(v + 8));
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const int row = wrow0 + 2 * i + (lane >> 4), j4 = lane & 15;
                        *reinterpret_cast<uint2 *>(sa + row * 128 + ((((j4 >> 1) ^ (row & 7)) << 4) | ((j4 & 1) << 3))) =
                            make_uint2(pack_bf16x2(v[i].x, v[i].y), pack_bf16x2(v[i].z, v[i].w));
                    }
                    fence_proxy_async();
                    mbar_arrive(full + stage);
                } else {
                    // ---- bf16 delta rows: 4 rows x 8 x 16 B cp.async per instruction, zero-fill if inactive
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        const int rl = 4 * i + (lane >> 3), j = lane & 7;
                        const int64_t si = __shfl_sync(0xffffffffu, src, rl);
                        const int row = wrow0 + rl;
                        const bool ok = si >= 0 && j < nval;
                        cp_async16(sa + row * 128 + ((j ^ (row & 7)) << 4), ok ? As + si + ci0 + j * 8 : As,
                                   ok ? 16u : 0u);
                    }
                    cp_async_arrive_noinc(full + stage);
                }
                // ---- B tile: one TMA 2D load by thread 0 (rows past Cout zero-filled)
                if (m == 0) {   // this CTA's half of the weight tile
                    mbar_arrive_tx(full + stage, S::B_BYTES);
                    tma_load_2d(sb, &tmap_b, k0, nt * BN + (int)rank * (BN / 2), full + stage);
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
                ci0 += BK;
                if (ci0 == Cpad) { ci0 = 0; tap++; }
            }
        }
        if (async_a && !c.tma_a) asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (warp == 4) {
        if (rank == 0) {
            // ===================== MMA issuer (leader) =====================
            constexpr uint32_t IDESC = idesc_bf16(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int w = cid; w < nwork; w += ncl, it++) {
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                mbar_wait(tempty + acc, acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; kb++) {
                    mbar_wait(full + stage, phase);
                    mbar_wait(pfull + stage, phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = smem_u32(smem + stage * S::STAGE);
                        const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
                        for (int k = 0; k < BK / 16; k++)
                            tc_mma2(tmem_d, sdesc(sa + k * 32), sdesc(sb + k * 32), IDESC, (kb | k) != 0);
                        tc_commit2_mc(empty + stage);                 // both CTAs' stage reusable
                        if (kb == nkb - 1) tc_commit2_mc(tfull + acc);  // both CTAs' epilogues
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        } else if (lane == 0) {
            // ===================== relay (peer) =====================
            // forwards "this CTA's stage landed" to the leader's pfull barrier
            int stage = 0;
            uint32_t phase = 0;
            for (int w = cid; w < nwork; w += ncl)
                for (int kb = 0; kb < nkb; kb++) {
                    mbar_wait(full + stage, phase);
                    mbar_arrive_remote(pfull + stage, 0);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
        }
    } else {
        // ===================== epilogue =====================
        const int quarter = warp & 3;            // TMEM lane quarter accessible by this warp
        const int half = (warp - 5) >> 2;        // which 32-column chunks of the accumulator
        const int row_in_tile = quarter * 32 + lane;
        int it = 0;
        // the site epilogue (SITE) runs in warps 5-8 only (its barriers count 128 threads)
        for (int w = cid; w < nwork && !(SITE && !DENSE && half > 0); w += ncl, it++) {
            const int mt = 2 * (w / ntn) + (int)rank, nt = w % ntn;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(tfull + acc, acc_phase);
            tc_fence_after();
            const int r = mt * BM + row_in_tile;
            if constexpr (SITE && !DENSE) {
                site_epilogue<BN>(c, tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN,
                                  smem + S::SITE_OFF, M, mt, quarter, lane, warp == 5 && lane == 0, tempty + acc);
            } else {
#pragma unroll 1
                for (int c0 = 32 * half; c0 < BN; c0 += 32 * (NEPI / 4)) {
                    uint32_t v[32];
                    const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0;
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
                          "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
                          "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                        : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    const int n0 = nt * BN + c0;
                    if (DENSE) {
                        // bias, then a transpose through shared memory: lane l of the
                        // copy-out covers row 4k + l/8, columns 4(l%8)..+3 -- four whole
                        // 128-byte row pieces per store instruction (a row per thread
                        // wrote 32 row pieces of 16 bytes per instruction); the
                        // consuming site's dense output f(x0) (+ bf16 shadow) from the
                        // same registers
                        if (n0 >= g.Cout) continue;   // warp-uniform
                        float *stg = reinterpret_cast<float *>(smem + S::DSTG_OFF) + (warp - 5) * (32 * 33);
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            stg[lane * 33 + j] =
                                __fadd_rn(__uint_as_float(v[j]), n0 + j < g.Cout ? __ldg(c.bias + n0 + j) : 0.0f);
                        __syncwarp();
                        const int cc = (lane & 7) * 4;
#pragma unroll
                        for (int k = 0; k < 8; k++) {
                            const int rl = 4 * k + (lane >> 3);
                            const int rr = mt * BM + quarter * 32 + rl;
                            if (rr < M && n0 + cc < g.Cout) {
                                float4 f;
                                f.x = stg[rl * 33 + cc];
                                f.y = stg[rl * 33 + cc + 1];
                                f.z = stg[rl * 33 + cc + 2];
                                f.w = stg[rl * 33 + cc + 3];
                                const int64_t oi = (int64_t)rr * g.Cout + n0 + cc;
                                *reinterpret_cast<float4 *>(static_cast<float *>(c.out) + oi) = f;
                                if (c.act_out) {
                                    f.x = act_rt(c.act_kind, f.x);
                                    f.y = act_rt(c.act_kind, f.y);
                                    f.z = act_rt(c.act_kind, f.z);
                                    f.w = act_rt(c.act_kind, f.w);
                                    *reinterpret_cast<float4 *>(c.act_out + oi) = f;
                                    if (c.act_bf) {
                                        uint2 u;
                                        u.x = pack_bf16x2(f.x, f.y);
                                        u.y = pack_bf16x2(f.z, f.w);
                                        *reinterpret_cast<uint2 *>(static_cast<bf16 *>(c.act_bf) + oi) = u;
                                    }
                                }
                            }
                        }
                        __syncwarp();   // buffer reused by the next chunk
                        continue;
                    }
                    if (r >= M || n0 >= g.Cout) continue;
                    const bool full_chunk = n0 + 32 <= g.Cout;
                    if (DENSE) {
                        float *o = static_cast<float *>(c.out) + (int64_t)r * g.Cout + n0;
                        if (full_chunk) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                float4 f;
                                f.x = __fadd_rn(__uint_as_float(v[j]), __ldg(c.bias + n0 + j));
                                f.y = __fadd_rn(__uint_as_float(v[j + 1]), __ldg(c.bias + n0 + j + 1));
                                f.z = __fadd_rn(__uint_as_float(v[j + 2]), __ldg(c.bias + n0 + j + 2));
                                f.w = __fadd_rn(__uint_as_float(v[j + 3]), __ldg(c.bias + n0 + j + 3));
                                *reinterpret_cast<float4 *>(o + j) = f;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; j++)   // unrolled: v[] stays in registers
                                if (n0 + j < g.Cout) o[j] = __fadd_rn(__uint_as_float(v[j]), __ldg(c.bias + n0 + j));
                        }
                    } else {
                        bf16 *o = static_cast<bf16 *>(c.out) + (int64_t)(r + 1) * g.Cout + n0;
                        if (full_chunk) {
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                uint4 u;
                                u.x = pack_bf16x2(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                                u.y = pack_bf16x2(__uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
                                u.z = pack_bf16x2(__uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
                                u.w = pack_bf16x2(__uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
                                *reinterpret_cast<uint4 *>(o + j) = u;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; j++)
                                if (n0 + j < g.Cout) o[j] = __float2bfloat16_rn(__uint_as_float(v[j]));
                        }
                    }
                }
                tc_fence_before();
                asm volatile("bar.sync 1, %0;" ::"n"(32 * NEPI) : "memory");   // all epilogue warps done with acc
                if (warp == 5 && lane == 0) mbar_arrive_remote(tempty + acc, 0);
            }
        }
    }
    __syncwarp();     // reconverge role-divergent warps before the .aligned cluster barrier
    tc_fence_before();
    cluster_sync();   // no CTA leaves while its peer may still signal it / its MMAs target it
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

template <int BN, bool DENSE, bool SMALL = false, bool SITE = false>
static void launch_tc(const ConvCall &c, const CUtensorMap *tmap, cudaStream_t s, int num_sms,
                      const CUtensorMap *tmap_a = nullptr) {
    using S = tc::Smem<BN, SITE, DENSE>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_conv_tc<BN, DENSE, SMALL, SITE>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL);
        attr = true;
    }
    const int ntn = (c.g.Cout + BN - 1) / BN;
    const int64_t m_up = DENSE ? (int64_t)c.B * c.g.Hout * c.g.Wout : c.m_cap;
    const int64_t work = ((m_up + 2 * tc::BM - 1) / (2 * tc::BM)) * ntn;   // (M-tile pair, N tile)
    int grid = 2 * (int)std::min<int64_t>(work, num_sms / 2);              // whole 2-CTA clusters
    if (grid < 2) grid = 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NTHREADS);
    cfg.dynamicSmemBytes = S::TOTAL;
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = 2;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_conv_tc<BN, DENSE, SMALL, SITE>, c, *tmap, tmap_a ? *tmap_a : *tmap);
}

// c_in % 8 == 0 (16-byte bf16 row pieces; each tap zero-padded to a multiple
// of 64 channels), c_out % 8 == 0 (the TMA zero-fills weight rows past c_out)
bool conv_tc_eligible(const Geo &g) {
    return g.groups == 1 && g.Cin % 8 == 0 && g.Cout % 8 == 0 && g.kh * g.kw <= tc::TAPS;
}
int conv_tc_cpad(int cin) { return (cin + tc::BK - 1) / tc::BK * tc::BK; }

// stems: the network input (c_in <= 4) on tensor cores, taps packed 16 per
// 64-wide k-block (kernel SMALL variant); weights K = ceil(taps/16)*64
bool conv_tc_small_eligible(const Geo &g) {
    return g.groups == 1 && g.Cin <= 4 && g.Cout % 16 == 0 && g.kh * g.kw <= 64;
}
void conv_tc_small_layout(const Geo &g, int &sr, int &shift) {
    // stride 2 -> ix0 = 2*ox - pw has the parity of pw for every output
    // pixel; even map width keeps pixel pairs 16-byte aligned in memory
    sr = shift = 0;
    if (g.sw == 2 && g.Win % 2 == 0 && g.kw + (g.pw & 1) <= 16) {
        shift = g.pw & 1;
        sr = (g.kw + shift + 1) / 2 * 2;
    }
}
int conv_tc_small_k(const Geo &g) {
    int sr, shift;
    conv_tc_small_layout(g, sr, shift);
    const int slots = sr ? g.kh * sr : g.kh * g.kw;
    return (slots + 15) / 16 * tc::BK;
}

__global__ void k_pad4_bf16(const float *__restrict__ x, int64_t n, int C, uint2 *__restrict__ out) {
    st_pdl_enter();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int c = 0; c < C && c < 4; c++) v[c] = __ldg(x + i * C + c);
        out[i] = make_uint2(tc::pack_bf16x2(v[0], v[1]), tc::pack_bf16x2(v[2], v[3]));
    }
}
void launch_pad4_bf16(const float *x, int64_t n, int C, void *out, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    if (grid > 0) k_pad4_bf16<<<grid, 256, 0, s>>>(x, n, C, static_cast<uint2 *>(out));
}

int conv_tc_bn(int cout) { return cout >= 256 ? 256 : cout >= 128 ? 128 : cout >= 64 ? 64 : 32; }

// TMA descriptor of the bf16 weights [Cout][K] (K contiguous): box 64 x BN,
// 128-byte swizzle matching the UMMA SWIZZLE_128B K-major smem layout,
// out-of-bounds rows (Cout not a multiple of BN) zero-filled.
static bool make_weight_tmap_bn(void *tmap_out, const void *wbf, int K, int Cout, int BN);
bool make_weight_tmap(void *tmap_out, const void *wbf, int K, int Cout) {
    return make_weight_tmap_bn(tmap_out, wbf, K, Cout, conv_tc_bn(Cout));
}
static int conv_tc_site_bn(int cout);
bool make_weight_tmap_site(void *tmap_out, const void *wbf, int K, int Cout) {
    return make_weight_tmap_bn(tmap_out, wbf, K, Cout, conv_tc_site_bn(Cout));
}
static bool make_weight_tmap_bn(void *tmap_out, const void *wbf, int K, int Cout, int BN) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)Cout};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)(BN / 2)};   // half tile per CTA of a pair
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap *>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void *>(wbf), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// A-operand map of a 1x1/s1 conv: [rows][C] bf16, box 64 channels x 128 rows,
// 128B swizzle (the MMA's K-major A layout), out-of-range rows / channels read 0
bool make_act_tmap(void *tmap_out, const void *base, int64_t rows, int C) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (C % 8 != 0 || rows < 1 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {(cuuint32_t)tc::BK, (cuuint32_t)tc::BM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(reinterpret_cast<CUtensorMap *>(tmap_out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                        const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

void launch_conv_tc(const ConvCall &c, const void *tmap_v, cudaStream_t s, const void *tmap_a_v) {
    const CUtensorMap *tmap = static_cast<const CUtensorMap *>(tmap_v);
    const CUtensorMap *tmap_a = static_cast<const CUtensorMap *>(tmap_a_v);
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (!c.dense && c.site.on) {   // one N tile covering c_out, the site in the epilogue
        switch (conv_tc_site_bn(c.g.Cout)) {
        case 32: launch_tc<32, false, false, true>(c, tmap, s, num_sms, tmap_a); break;
        case 64: launch_tc<64, false, false, true>(c, tmap, s, num_sms, tmap_a); break;
        case 128: launch_tc<128, false, false, true>(c, tmap, s, num_sms, tmap_a); break;
        default: launch_tc<256, false, false, true>(c, tmap, s, num_sms, tmap_a); break;
        }
        return;
    }
#define TC_BN(BN_) \
    (c.dense ? launch_tc<BN_, true>(c, tmap, s, num_sms, tmap_a) : launch_tc<BN_, false>(c, tmap, s, num_sms, tmap_a))
    switch (conv_tc_bn(c.g.Cout)) {
    case 256: TC_BN(256); break;
    case 128: TC_BN(128); break;
    case 64: TC_BN(64); break;
    default: TC_BN(32); break;
    }
#undef TC_BN
}


// ---- conv + site: pixels whose M rows continue across a 128-row tile
// boundary (their delta rows were written by both tiles' epilogues): one warp
// per boundary runs the site step of k_site_pw over the pixel's rows (the
// conv's row layout: rows 1 + pbase .. + popc(act)), in place.
template <int CPL>
__global__ void __launch_bounds__(256) k_tc_site_fixup(ConvCall c, DView conv) {
    st_pdl_enter();
    const int M = *c.m_dev;
    const int C = c.g.Cout;
    const int lane = threadIdx.x & 31;
    const int nb = (M + tc::BM - 1) / tc::BM;   // boundaries 1 .. nb-1
    const int k = 1 + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    if (k >= nb) return;
    const int rb = k * tc::BM;
    const int ga = __ldg(c.ridx + rb - 1) >> 5, gb = __ldg(c.ridx + rb) >> 5;
    if (ga != gb) return;
    const int g = ga;
    uint32_t a = __ldg(conv.act + g);
    const uint32_t sl = __ldg(conv.slot + g);
    const int64_t base = 1 + __ldg(conv.pbase + g);
    const float theta = __ldg(c.site.theta);
    const int kind = c.site.act;
    bf16 *out = static_cast<bf16 *>(c.out);
    float xa[CPL], ya[CPL];
#pragma unroll
    for (int i = 0; i < CPL; i++) {
        const int ch = lane + 32 * i;
        xa[i] = ch < C ? __ldg(c.site.x0 + (int64_t)g * C + ch) : 0.0f;
        ya[i] = act_rt(kind, xa[i]);
    }
    uint32_t emit = 0;
    while (a) {
        const int t1 = __ffs(a) - 1;
        a &= a - 1;
        const int64_t row = base + __popc(sl & lowmask(t1));
        float cand[CPL];
        float mx = 0.0f;
#pragma unroll
        for (int i = 0; i < CPL; i++) {
            const int ch = lane + 32 * i;
            const float v = ch < C ? __bfloat162float(out[row * C + ch]) : 0.0f;
            xa[i] = __fadd_rn(xa[i], v);
            cand[i] = __fsub_rn(act_rt(kind, xa[i]), ya[i]);
            mx = fmaxf(mx, fabsf(cand[i]));
        }
        mx = gmax<32>(mx, 0xffffffffu);
        if (mx > theta) {
#pragma unroll
            for (int i = 0; i < CPL; i++) {
                const int ch = lane + 32 * i;
                cand[i] = bf16_round(cand[i]);
                ya[i] = __fadd_rn(ya[i], cand[i]);
                if (ch < C) out[row * C + ch] = __float2bfloat16_rn(cand[i]);
            }
            emit |= 1u << t1;
        } else if (c.site.zero_gaps) {
#pragma unroll
            for (int i = 0; i < CPL; i++)
                if (lane + 32 * i < C) out[row * C + lane + 32 * i] = __float2bfloat16_rn(0.0f);
        }
    }
    if (lane == 0) c.site.words[g] = emit;
}

bool conv_tc_site_eligible(const Geo &g) { return conv_tc_eligible(g) && g.Cout <= 256; }
static int conv_tc_site_bn(int cout) { return cout <= 32 ? 32 : cout <= 64 ? 64 : cout <= 128 ? 128 : 256; }

void launch_tc_site_fixup(const ConvCall &c, DView conv, cudaStream_t s) {
    const int64_t nb = (c.m_cap + tc::BM - 1) / tc::BM;   // upper bound of the boundaries
    const int grid = (int)std::max<int64_t>(1, (nb + 7) / 8);
    switch (conv_tc_site_bn(c.g.Cout)) {
    case 32: k_tc_site_fixup<1><<<grid, 256, 0, s>>>(c, conv); break;
    case 64: k_tc_site_fixup<2><<<grid, 256, 0, s>>>(c, conv); break;
    case 128: k_tc_site_fixup<4><<<grid, 256, 0, s>>>(c, conv); break;
    default: k_tc_site_fixup<8><<<grid, 256, 0, s>>>(c, conv); break;
    }
}

}  // namespace st

namespace st {
void launch_conv_tc_small(const ConvCall &c, const void *tmap_v, cudaStream_t s) {
    const CUtensorMap *tmap = static_cast<const CUtensorMap *>(tmap_v);
    static int num_sms = 0;
    if (!num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
#define TC_BN(BN_) \
    (c.dense ? launch_tc<BN_, true, true>(c, tmap, s, num_sms) : launch_tc<BN_, false, true>(c, tmap, s, num_sms))
    switch (conv_tc_bn(c.g.Cout)) {
    case 256: TC_BN(256); break;
    case 128: TC_BN(128); break;
    case 64: TC_BN(64); break;
    default: TC_BN(32); break;
    }
#undef TC_BN
}
}  // namespace st
