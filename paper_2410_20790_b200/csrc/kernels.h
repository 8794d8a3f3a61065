// kernels.h -- host-side launchers of the sm_100a kernels (internal, not ABI).
//
// Data layout of a diff tensor (one layer boundary, all chunks of a step;
// DESIGN.md "Data layout in HBM"):
//   act  [B][N] uint32   bit (t-1) set <=> pixel active in diff frame t
//                        (pixel-major "frame words", so L-1 <= 32, R25)
//   slot [B][N] uint32   frame bits that own a row (superset of act)
//   pbase[B][N] int32    exclusive prefix over (b,p) of popc(slot)
//   rows [1+cap][C]      packed delta rows in (b, p, t) order; row 0 = zeros;
//                        fp32 in FP32 mode, bf16 in BF16 mode (`bf` flags)
// Row of (b,p,t) = 1 + pbase[b,p] + popc(slot[b,p] & ((1<<(t-1))-1)) when the
// act bit is set, else row 0.  Consumers never read rows of inactive bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace st {

struct DView {
    const uint32_t *act = nullptr;
    const uint32_t *slot = nullptr;
    const int32_t *pbase = nullptr;
    const void *rows = nullptr;   // float or bf16 [1+cap][C]
    int64_t nrows = INT64_MAX;    // 1 + cap (ST_CHECK bounds in the checked build)
};

struct Geo {   // conv / pool geometry
    int Hin, Win, Cin, Hout, Wout, Cout, kh, kw, sh, sw, ph, pw, groups;
};

// Thresholds are read by the kernels from device memory (theta points at one
// fp32 site threshold), so a captured CUDA graph serves every step.
// ---- masks, compaction (kernels_mask.cu) ----
// Subtraction pass 1 (site 0): act bits per pixel, sequential over frames;
// optionally also the dense per-frame emitted delta ddelta [B][n_diff][N][C]
// (zeros where truncated; row type) for convs reading the input directly.
// frames: fp32, or uint8 (u8: value v / 255.0f, reading R20); fr_stride in elements
void launch_subtract_mask(const float *ref, int64_t ref_stride, const void *frames, bool u8, int64_t fr_stride,
                          int B, int N, int C, int n_diff, const float *theta, bool bf, uint32_t *act, void *ddelta,
                          cudaStream_t s);
// Subtraction pass 2: write emitted rows at the slots of `act`; s_save
// (streaming, nullable): final S of every pixel with an emission, [B][N][C]
// (may alias ref when ref_stride == N*C: each pixel is read, then written, by
// its own thread).
void launch_subtract_rows(const float *ref, int64_t ref_stride, const void *frames, bool u8, int64_t fr_stride,
                          int B, int N, int C, const uint32_t *act, const int32_t *pbase, void *rows, bool bf,
                          float *s_save, cudaStream_t s);
// n uint8 frames of `per` elements (frame c at src + c*src_stride) -> fp32 v / 255.0f, packed
void launch_u8_to_f32(const uint8_t *src, int64_t src_stride, int64_t per, int n, float *dst, cudaStream_t s);
// out[b][q] = OR of in[b][p] over the receptive field (dense amplification)
void launch_dilate(const uint32_t *in, int B, const Geo &g, uint32_t *out, cudaStream_t s);
// pbase = exclusive prefix of popc(words) over n words; *total = sum; also
// adds the total into *stat (int64) if stat != nullptr.  tmp: scan scratch
// (scan_tmp_ints(n) int32).
int64_t scan_tmp_ints(int64_t n);
// ridx (optional): also enumerate the conv M-row list (replaces launch_enumerate)
// cap (optional): row capacity of the tensor -- words whose rows would end
// past cap are cleared, *total becomes the rows that fit and *ovf is set;
// peak (optional): running max of the unclamped totals (int64 atomicMax)
struct ScanCap {
    int64_t cap = 0;
    int32_t *ovf = nullptr;   // null: no capacity check
    long long *peak = nullptr;
};
void launch_scan_popc(uint32_t *words, int64_t n, int32_t *pbase, int32_t *total, int32_t *tmp, long long *stat,
                      cudaStream_t s, int32_t *ridx = nullptr, const ScanCap &cap = ScanCap());
// ridx[pbase+j] = ((b*N+q) << 5) | t1 for every set bit of slot (conv M rows)
void launch_enumerate(const uint32_t *slot, const int32_t *pbase, int64_t n, int32_t *ridx, cudaStream_t s);
// per (b, t1) popcounts of act into counts[b*cstride + t1] (int64 atomics,
// counts may be null); sum of popc into *stat, number of non-zero words into
// *stat_nz (either may be null).
void launch_frame_counts(const uint32_t *act, int B, int N, long long *counts, int64_t cstride,
                         long long *stat, long long *stat_nz, cudaStream_t s);
void launch_or_words(const uint32_t *a, const uint32_t *b, int64_t n, uint32_t *out, cudaStream_t s);

// ---- convolution (kernels_conv.cu) ----
struct ConvCall {
    Geo g;
    int B;
    bool dense;             // reference-frame mode (fp32 activations in and out)
    bool bf;                // sparse mode: rows are bf16 (BF16 mode)
    bool rnd_a;             // dense mode, BF16 mode: round the fp32 A operand to bf16 (RNE, R22-BF16)
    // A operand
    const float *a_dense;   // dense: [B][Nin][Cin]
    const float *zeros;     // >= 1 KiB of device zeros (source of absent taps / padding)
    const void *a_dense_bf; // dense, optional: bf16 shadow of a_dense (tcgen05 path gathers it with cp.async)
    DView a;                // sparse
    const int32_t *ridx;    // sparse: M-row list
    const int32_t *m_dev;   // sparse: device M
    int64_t m_cap;          // sparse: upper bound of M (grid sizing)
    const void *ddelta;     // sparse, optional: dense per-frame input delta [B][F][Nin][Cin]
    int F;                  // diff frames (ddelta indexing)
    int sr, shift;          // stems: paired K layout (sr > 0), see conv_tc_small_layout
    bool rowmap = false;    // sparse 1x1/s1: M row r = input row r + 1 -> output row r + 1 (no ridx)
    bool tma_a = false;     // tcgen05, 1x1/s1 with contiguous A rows: A tiles by TMA (launch_conv_tc tmap_a)
    // tcgen05 sparse conv + its ReLU / SiLU site in the epilogue (N2; BF16 mode, c_out <= 256):
    // the emitted rows go to `out` (the conv's row layout), the site's frame words to `words`
    struct {
        bool on = false;
        const float *x0 = nullptr;     // conv dense output of the reference frame (the site's x_acc start)
        const float *theta = nullptr;
        int act = 0;                   // Act
        uint32_t *words = nullptr;     // site emitted frame words [B][N] (zeroed before the launch)
        bool zero_gaps = false;
    } site;
    // B operand / output
    const float *wk;        // [K][Cout] (K order dy,dx,ci; R18)
    const float *bias;      // dense only
    void *out;              // dense: float [B*Nout][Cout]; sparse: rows_out (row 1+r)
    // dense depthwise only, optional: the consuming pointwise site's dense
    // output f(out) (act_kind: Act) written by the same epilogue
    float *act_out = nullptr;
    void *act_bf = nullptr;   // optional bf16 (RNE) shadow of act_out (a tensor-core conv reads it densely)
    int act_kind = 0;
};
void launch_conv_f32(const ConvCall &c, cudaStream_t s);
void launch_dwconv_f32(const ConvCall &c, cudaStream_t s);
// sparse depthwise, pixel-major over the output frame words (no M-row list)
void launch_dwconv_pm(const ConvCall &c, const uint32_t *out_act, const int32_t *out_pbase, cudaStream_t s);
// Sparse depthwise conv + the pointwise site (ReLU / SiLU) that is its only
// consumer, in one pass (conv-epilogue non-linear correction, SURVEY §8(f)
// N2): the group that computes an output pixel's delta rows (frames in
// order) steps the site's x_acc / y_acc on them at once, so the conv's delta
// rows never reach HBM.  Requires C % 8 == 0.
struct DwSite {
    const uint32_t *out_act = nullptr;   // conv output frame words (the site's touched set and row layout)
    const int32_t *out_pbase = nullptr;  // their row bases
    const float *x0 = nullptr;           // conv dense output of the reference frame = the site's x_acc start
    const float *theta = nullptr;        // the site's threshold (device)
    int act = 0;                         // Act
    uint32_t *site_act = nullptr;        // site emitted frame words [B][N]
    void *site_rows = nullptr;           // site emitted rows, in the conv's row layout
    void *conv_rows = nullptr;           // optional (debug_retain): the conv's own delta rows
    bool zero_gaps = false;              // zero rows at touched, not emitted slots (rowmap consumer)
    int64_t site_nrows = INT64_MAX;      // rows of site_rows / conv_rows (ST_CHECK)
};
bool dwconv_site_fusable(const Geo &g);
void launch_dwconv_site(const ConvCall &c, const DwSite &d, cudaStream_t s);
// team form (kernels_dw_team.cu): one CTA of ceil(C/256) warps per output pixel, C <= DWT_MAXC
constexpr int DWT_MAXC = 16 * 256;
void launch_dwconv_site_team(const ConvCall &c, const DwSite &d, cudaStream_t s);
// tile form (kernels_dw_team.cu): C <= 32, k x k <= 9, stride <= 2
bool dwconv_site_tile_ok(const Geo &g);
void launch_dwconv_site_tile(const ConvCall &c, const DwSite &d, cudaStream_t s);
// BF16 mode, tcgen05 tensor cores (kernels_conv_tc.cu).  Weights bf16
// [Cout][K] are read through a TMA descriptor (CUtensorMap, 128 bytes)
// built once at create by make_weight_tmap.
bool conv_tc_eligible(const Geo &g);
int conv_tc_cpad(int cin);   // per-tap channel stride of the bf16 weight K layout (zero padded)
bool make_weight_tmap(void *tmap_out, const void *wbf, int K, int Cout);
void launch_conv_tc(const ConvCall &c, const void *tmap, cudaStream_t s, const void *tmap_a = nullptr);
// A-operand TMA map of a 1x1/s1 conv over a [rows][C] bf16 matrix (c.tma_a)
bool make_act_tmap(void *tmap_out, const void *base, int64_t rows, int C);
// conv + site in the epilogue: eligibility, the weight map with the one-tile
// N width it needs, and the fix-up of pixels continuing across tile
// boundaries (conv = the conv's delta tensor view: act / pbase)
bool conv_tc_site_eligible(const Geo &g);
bool make_weight_tmap_site(void *tmap_out, const void *wbf, int K, int Cout);
void launch_tc_site_fixup(const ConvCall &c, DView conv, cudaStream_t s);
// stems on tensor cores: the network input (c_in <= 4); sparse mode reads the
// 4-channel-padded dense input delta (c.ddelta), dense mode the fp32 frames
bool conv_tc_small_eligible(const Geo &g);
// stem K layout: "paired" for stride-2 stems on even-width maps (each kernel row
// padded to sr tap slots, slot = dy*sr + dx + shift, so 16-byte pieces of two
// 4-channel pixels land on 16-byte slot pairs); else 16 taps per 64-wide k-block.
// slot_of gives the 4-channel slot of tap (dy, dx); K = conv_tc_small_k
void conv_tc_small_layout(const Geo &g, int &sr, int &shift);
int conv_tc_small_k(const Geo &g);
// bf16 copy of the fp32 reference frames [n][C] padded to 4 channels [n][4]
void launch_pad4_bf16(const float *x, int64_t n, int C, void *out, cudaStream_t s);
void launch_conv_tc_small(const ConvCall &c, const void *tmap, cudaStream_t s);

// ---- sites, joins, accumulation (kernels_site.cu) ----
enum Act { ACT_RELU = 0, ACT_SILU = 1, ACT_SILU_FAST = 2 };   // FAST: BF16 mode only
// dense reference-frame ops; ybf (optional, may be null): bf16 (RNE) shadow
// of y for a tensor-core conv that consumes y in dense mode
void launch_dense_act(const float *x, float *y, int64_t n, int act, void *ybf, cudaStream_t s);
void launch_dense_maxpool(const float *x, float *y, int B, const Geo &g, void *ybf, cudaStream_t s,
                          bool relu_in = false);   // relu_in: x = pre-activation of a fused ReLU
void launch_dense_add(const float *a, const float *b, float *y, int64_t n, void *ybf, cudaStream_t s);
void launch_to_bf16(const float *x, void *ybf, int64_t n, cudaStream_t s);
// Streaming state of a site (the per-site caches of the
// vanilla DeltaCNN schedule, kept so st_encode_diff can continue a
// chunk).  All pointers nullable (SparseBatch: none).  x0 passed to a site
// launch is the x_acc at call start (dense reference activation on the
// first call, the saved state on a continuation); y_init the y_acc at call
// start (null: derived from x0).  Saves cover every pixel the call changed;
// the encoder pre-fills save buffers that are not updated in place.
struct SiteState {
    const float *y_init = nullptr;   // y_acc at start [B][N_out][C]
    float *x_save = nullptr;         // x_acc at end [B][N_in][C]
    float *y_save = nullptr;         // y_acc at end [B][N_out][C]
    const float *ry_init = nullptr;  // fused ReLU -> pool: ReLU y_acc at start [B][N_in][C]
    float *rx_save = nullptr;        //                     ReLU x_acc at end
    float *ry_save = nullptr;        //                     ReLU y_acc at end
};
// pointwise site: emitted rows written into out_rows at the input slots
// zero_gaps: also write zero rows at touched frames that were not emitted
// (the layout is read as a plain matrix by a rowmap 1x1 conv)
void launch_site_pointwise(DView in, const float *x0, int B, int N, int C, int act, const float *theta, bool bf,
                           uint32_t *out_act, void *out_rows, const SiteState &st, cudaStream_t s,
                           bool zero_gaps = false);
// maxpool site: touched layout (t_slot, t_pbase) = dilation of in.act
void launch_site_maxpool(DView in, const float *x0, int B, const Geo &g, const float *theta, bool bf,
                         const uint32_t *t_slot, const int32_t *t_pbase, uint32_t *out_act, void *out_rows,
                         const SiteState &st, cudaStream_t s);
// ReLU site + maxpool site in one tile-resident pass (ReLU output consumed
// only by the pool): conv = the conv's delta tensor, x0_conv its dense
// pre-activation; (t_slot, t_pbase) = dilation of conv.act (row capacity of
// the pool); writes the ReLU mask words r_act (+ its rows into r_rows at the
// conv slots when r_rows != nullptr) and the pool's act / rows.
bool site_relu_maxpool_fusable(const Geo &g, bool bf);
void launch_site_relu_maxpool(DView conv, const float *x0_conv, int B, const Geo &g, const float *theta_r,
                              const float *theta, bool bf, const uint32_t *t_slot, const int32_t *t_pbase,
                              uint32_t *r_act, void *r_rows, uint32_t *out_act, void *out_rows, const SiteState &st,
                              cudaStream_t s);
// residual add: out slot layout = act_a | act_b (already scanned into pbase)
void launch_add_rows(DView a, DView b, const uint32_t *slot, const int32_t *pbase, int B, int N, int C, bool bf,
                     void *out_rows, cudaStream_t s);
// ---- squeeze-excitation site (kernels_se.cu, reading R8) ----
void launch_se_colsum(const float *x, int B, int N, int C, double *sum0, cudaStream_t s);
void launch_se_delta_sums(DView in, int B, int N, int C, int F, bool bf, double *dsum, cudaStream_t s);
void launch_se_schedule(const double *sum0, const double *dsum, int B, int N, int C, int H, int F, const float *w1,
                        const float *b1, const float *w2, const float *b2, const float *theta, float *gate_tab,
                        float *s_tab, uint32_t *refresh, cudaStream_t s);
// split form of launch_se_schedule: gates of frames t0 .. t0 + nt - 1 (frame 0 =
// the reference, from sum0 alone: the dense pass computes it, the diff pass
// frames 1 .. F), then the sequential refresh schedule over frames 1 .. F
void launch_se_gates(const double *sum0, const double *dsum, int B, int N, int C, int H, int F, const float *w1,
                     const float *b1, const float *w2, const float *b2, int t0, int nt, float *gate_tab, cudaStream_t s);
void launch_se_sched(const float *gate_tab, int B, int C, int F, const float *theta, float *s_tab, uint32_t *refresh,
                     cudaStream_t s);
// y (fp32) and ybf (bf16 shadow) each nullable
void launch_se_dense_apply(const float *x, const float *s_tab, int B, int N, int C, int F, float *y, void *ybf,
                           cudaStream_t s);
void launch_se_slots(const uint32_t *act, const uint32_t *refresh, int B, int N, uint32_t *slot, cudaStream_t s);
void launch_se_site(DView in, const float *x0, const float *s_tab, int B, int N, int C, int F, const float *theta, bool bf,
                    const uint32_t *slot, const int32_t *pbase, uint32_t *out_act, void *out_rows, cudaStream_t s,
                    bool zero_gaps = false);
// Accumulation at a tap: out[b][t][N][C], t = 0..n_diff (frame 0 = y0, the
// start state [B][N][C]); o_save (streaming, nullable, may alias y0): the
// last frame's output, the start of the next call
void launch_accumulate(DView in, const float *y0, int B, int N, int C, int n_diff, bool bf, float *out,
                       float *o_save, cudaStream_t s);

}  // namespace st
