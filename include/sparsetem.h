/*
 * sparsetem.h -- C ABI of libsparsetem.so, the B200 (sm_100a) Diff Computation
 * hot path of SparseTem (arXiv 2410.20790).  Citations "P:n" are lines of the
 * paper text; "Rn" are the readings listed in DESIGN.md.
 *
 * The calls follow the paper's problem statement:
 *   st_encoder_create      -- network from layer specs + weights (Eq.1)
 *   st_encode_reference    -- stage the reference frame of each chunk
 *   st_encode_diff         -- one SparseBatch pass over all diff frames of all
 *                             chunks: dense on the reference frame,
 *                             Subtraction -> mask -> compaction -> sparse conv
 *                             (Eq.2) -> non-linear correction (Eq.3) ->
 *                             truncation -> Accumulation
 *   st_get_sparsity        -- measured per-site sparsity (input of P:171-181)
 *   st_get_output          -- dense per-frame outputs at the taps
 *   st_controller_*        -- BST/IBST online threshold adjustment
 *
 * Conventions (apply to every call):
 *   - Every call returns st_status; no C++ exception crosses the ABI.  On
 *     error, st_last_error(enc) holds a one-line message.
 *   - Pointers named *_dev are CUDA device pointers on the encoder's device;
 *     *_host / plain pointers are host memory.  The caller owns every buffer
 *     it passes; the encoder owns all device memory it allocates (one arena,
 *     allocated at create; the encode calls never allocate).
 *   - Tensors are NHWC fp32: pixel p = y*W + x, element [p*C + c].  Input
 *     frames are in [0,1] (R20).
 *   - Stream-ordered: calls taking `stream` (a cudaStream_t; NULL = legacy
 *     default stream) only enqueue work.  st_get_sparsity, st_get_layer_counts
 *     and the debug getters synchronize the stream of the last encode call.
 *   - One encoder per device per host thread; encoders are not thread-safe.
 *   - There is no CPU fallback: without a usable sm_100 device, create fails
 *     with ST_ERR_CUDA.
 */
#ifndef SPARSETEM_H_
#define SPARSETEM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct st_encoder st_encoder;   /* opaque */

typedef enum {
    ST_OK = 0,
    ST_ERR_ARG = 1,          /* null pointer, out-of-range value              */
    ST_ERR_SHAPE = 2,        /* inconsistent geometry or chunk/frame counts   */
    ST_ERR_STATE = 3,        /* call out of order (diff without reference)    */
    ST_ERR_UNSUPPORTED = 4,  /* valid but not implemented (e.g. L-1 > 32)     */
    ST_ERR_OOM = 5,          /* arena allocation failed                       */
    ST_ERR_CUDA = 6,         /* CUDA runtime error (message has the detail)   */
    ST_ERR_INTERNAL = 7,     /* invariant violated                                  */
    ST_ERR_CAPACITY = 8,     /* a delta tensor of the last step needed more rows than
                                its capacity (row_frac / st_encoder_fit_capacity): the
                                step's outputs and statistics are invalid; re-plan
                                with st_encoder_fit_capacity and re-issue the step */
} st_status;

/* Layer kinds.  CONV is Eq.(1) (zero padding, groups; groups == c_in is
 * depthwise, R9).  RELU/SILU/MAXPOOL/SE are non-linear and are
 * truncation sites (R6).  ADD is a residual join (linear).  OUTPUT
 * marks an output tap where Accumulation happens. */
typedef enum { ST_CONV = 0, ST_RELU = 1, ST_SILU = 2, ST_MAXPOOL = 3, ST_ADD = 4,
               ST_SE = 5, ST_OUTPUT = 6 } st_kind;

typedef enum { ST_FP32 = 0, ST_BF16 = 1 } st_precision;

typedef struct {
    int32_t kind;          /* st_kind                                              */
    int32_t src;           /* producer layer index, -1 = network input; < own index */
    int32_t src2;          /* ADD only: second producer                            */
    int32_t c_out;         /* CONV output channels                                 */
    int32_t groups;        /* CONV groups (1 = dense, c_in = depthwise)            */
    int32_t k_h, k_w;      /* CONV / MAXPOOL window                                */
    int32_t s_h, s_w;      /* stride                                               */
    int32_t p_h, p_w;      /* padding (CONV zeros, MAXPOOL -inf; R11)              */
    int32_t se_hidden;     /* SE reduced width                                     */
    const float *w, *b;    /* host fp32. CONV: w OIHW [c_out][c_in/groups][k_h][k_w],
                              b [c_out] (BatchNorm folded).  SE: w [hidden][C],
                              b [hidden].  Copied at create.                       */
    const float *w2, *b2;  /* SE only: w2 [C][hidden], b2 [C]                      */
} st_layer_spec;

typedef struct {
    int32_t in_c, in_h, in_w;    /* network input geometry                       */
    int32_t max_chunks;          /* B: chunks per encode call (upper bound)       */
    int32_t max_frames;          /* L: frames per chunk incl. reference, 2..33    */
    int32_t precision;           /* st_precision                                  */
    int32_t device;              /* CUDA device ordinal                           */
    int32_t debug_retain;        /* 1: keep every layer's buffers for st_debug_*  */
    int32_t streaming;           /* 1: streaming continuation:  *
                                  * the per-site caches of the vanilla DeltaCNN   *
                                  * schedule -- S, each site's x_acc /    *
                                  * y_acc, each tap's last output -- are kept in  *
                                  * persistent device buffers, so st_encode_diff  *
                                  * called again without st_encode_reference      *
                                  * continues every chunk from its last frame     *
                                  * (chunks longer than max_frames, live video).  *
                                  * Memory: those caches (st_memory_report).      *
                                  * ST_ERR_UNSUPPORTED with SE layers.            */
    float row_frac;              /* row capacity of every delta tensor (SURVEY    *
                                  * §8(a) a9; P:139, P:152 -- memory, not time,   *
                                  * is the claim): 0 or >= 1 = the all-active     *
                                  * bound B*(L-1)*N rows; in (0,1) = that         *
                                  * fraction of it (>= 4096 rows).  A step that   *
                                  * needs more rows is clamped on the device and  *
                                  * reported as ST_ERR_CAPACITY; see              *
                                  * st_encoder_fit_capacity.                      */
} st_encoder_config;

/* Validate specs, infer shapes, number the sites, repack weights, plan the
 * SparseBatch buffer lifetimes and allocate one device arena.
 * Sites: 0 = network input, then every non-linear layer in spec order. */
st_status st_encoder_create(const st_encoder_config *cfg, const st_layer_spec *layers,
                            int32_t n_layers, st_encoder **out);
void st_encoder_destroy(st_encoder *enc);
int32_t st_encoder_num_sites(const st_encoder *enc);
/* shape of layer `layer`'s output (-1 = network input) */
st_status st_layer_shape(const st_encoder *enc, int32_t layer, int32_t hwc[3]);

/* Stage the reference frame (frame 0) of n_chunks chunks as slot 0.
 * ref_dev: [n_chunks] frames of [H][W][C] fp32, chunk c at ref_dev +
 * c*chunk_stride elements (chunk_stride 0 = packed H*W*C).  Copied
 * (stream-ordered); the dense reference pass itself runs inside
 * st_encode_diff, layer-interleaved (reading R-B1). */
st_status st_encode_reference(st_encoder *enc, const float *ref_dev, int32_t n_chunks,
                              int64_t chunk_stride, void *stream);

/* One SparseBatch pass over n_diff diff frames of every staged
 * chunk.  With cfg.streaming, a call after a previous st_encode_diff (no
 * st_encode_reference in between) continues each chunk: its frame 0 is the
 * previous call's last frame (state and outputs), the dense reference pass
 * is skipped, and the results equal one call over all frames of the chunk.
 * frames_dev: chunk c, diff frame t (1..n_diff) at frames_dev +
 * c*chunk_stride + (t-1)*H*W*C (chunk_stride 0 = packed n_diff*H*W*C).
 * thresholds: host [n_sites] fp32 truncation thresholds, constant for the
 * call (R15).  n_diff = 0 runs the dense pass only.  Without streaming, a
 * repeated call (no new st_encode_reference) recomputes the chunks from the
 * staged reference frames.  Errors: ST_ERR_STATE
 * without a staged reference; ST_ERR_SHAPE if n_diff+1 > max_frames. */
st_status st_encode_diff(st_encoder *enc, const float *frames_dev, int32_t n_diff,
                         int64_t chunk_stride, const float *thresholds, void *stream);

/* uint8 video frames (the camera / decoder format; 4x fewer bytes over PCIe
 * and out of HBM).  Identical to the fp32 calls on frames v / 255.0f
 * (reading R20; the conversion happens in the Subtraction kernels and, for
 * the reference, in a staging kernel), so results are bit-identical to
 * st_encode_reference / st_encode_diff on the converted frames.  Layout,
 * strides (in elements), state rules and errors as the fp32 calls. */
st_status st_encode_reference_u8(st_encoder *enc, const uint8_t *ref_dev, int32_t n_chunks,
                                 int64_t chunk_stride, void *stream);
st_status st_encode_diff_u8(st_encoder *enc, const uint8_t *frames_dev, int32_t n_diff,
                            int64_t chunk_stride, const float *thresholds, void *stream);

/* Per-site sparsity statistics of the last encode (synchronizes).
 * active: host [n_chunks][n_sites][n_diff] emitted-pixel counts (or NULL);
 * site_active / site_pixels: host [n_sites] step sums (or NULL).
 * Sparsity of site s = 1 - site_active[s]/site_pixels[s] (R14). */
st_status st_get_sparsity(st_encoder *enc, int64_t *active, int64_t *site_active,
                          int64_t *site_pixels);
/* Async copy of int64 [2*n_sites] = {site_active..., site_pixels...} into a
 * device buffer (for the NCCL all-gather of the statistics). */
st_status st_copy_site_counts(st_encoder *enc, int64_t *dst_dev, void *stream);
/* Step totals per layer (synchronizes): rows_in = active input rows read,
 * rows_out = output rows produced (conv: dilated mask; site: emitted),
 * touched = pixels with any active input frame.  host [n_layers] each (any
 * may be NULL).  rows_in / touched are collected only while profiling is on
 * (st_set_profiling; 0 otherwise), rows_out always.  Used for the
 * algorithmic bytes/flops of the roofline. */
st_status st_get_layer_counts(st_encoder *enc, int64_t *rows_in, int64_t *rows_out,
                              int64_t *touched);

/* Dense fp32 output of OUTPUT layer `tap` for (chunk, frame), frame 0 = the
 * reference frame, 1..n_diff the accumulated diff frames.  Borrowed device
 * pointer, valid until the next encode call or destroy. */
st_status st_get_output(st_encoder *enc, int32_t tap, int32_t chunk, int32_t frame,
                        const float **dev_ptr, int32_t hwc[3]);

/* Debug (requires debug_retain; synchronizes).  Mask of layer `layer`'s
 * output delta (-1 = network input site) for (chunk, diff frame 1..n_diff)
 * as bitmask words (bit i of word j = pixel 32j+i), host [ceil(H*W/32)].
 * st_debug_get_rows: ascending active pixel list idx_host [n] and their
 * delta rows rows_host [n][C]; returns n in *n_out (buffers may be NULL to
 * query n).  Mask of a conv layer is its structural (dilated) output mask. */
st_status st_debug_get_mask(st_encoder *enc, int32_t layer, int32_t chunk, int32_t frame,
                            uint32_t *words_host);
st_status st_debug_get_rows(st_encoder *enc, int32_t layer, int32_t chunk, int32_t frame,
                            int32_t *idx_host, float *rows_host, int64_t *n_out);
/* Debug: dense reference-frame output of layer `layer` for `chunk`
 * (requires debug_retain), host [H*W*C]. */
st_status st_debug_get_dense0(st_encoder *enc, int32_t layer, int32_t chunk, float *host);

/* Debug: mask export for parity checks in the production launch
 * configuration (no debug_retain, arena reuse, CUDA-graph replay).  After
 * st_debug_export_chunk(enc, chunk), every following st_encode_diff also
 * copies, for that chunk only, the frame words of every layer boundary --
 * uint32 per pixel, bit t-1 set <=> pixel active in diff frame t (the
 * emitted mask at a site, the dilated structural mask at a conv) -- into a
 * buffer the encoder owns (sum over layers of H*W words); chunk = -1 turns it
 * off.  The copies are stream-ordered nodes of the step.  ST_ERR_ARG for a
 * chunk >= max_chunks, ST_ERR_OOM if the buffer cannot be allocated.
 * st_debug_get_words: host copy of layer `layer`'s words (-1 = input site)
 * [H_l*W_l]; syncs the stream; ST_ERR_STATE before an exporting diff call. */
st_status st_debug_export_chunk(st_encoder *enc, int32_t chunk);
st_status st_debug_get_words(st_encoder *enc, int32_t layer, uint32_t *words_host);

/* Memory report of the SparseBatch plan (bytes): persistent (staged
 * reference + outputs), peak transient (max live set), arena total. */
st_status st_memory_report(const st_encoder *enc, int64_t *persistent, int64_t *peak_transient,
                           int64_t *arena_total);
/* Total device bytes the encoder holds: the arena plus the fixed areas
 * (staged reference, counts, scan scratch) and the device weights. */
st_status st_device_bytes(const st_encoder *enc, int64_t *total);

/* Row capacity.  Every scan of a delta tensor checks its
 * row capacity on the device; words whose rows would not fit are cleared
 * (nothing is written past a buffer) and the step is flagged.
 * st_step_status: synchronizes the last encode's stream; ST_ERR_CAPACITY if
 *   that step was clamped, else ST_OK.
 * st_get_capacity: per delta tensor (layer i at [i], the input site at
 *   [n_layers]; -1 for layers without their own rows) the current capacity
 *   and the largest row count any step needed since create (host arrays of
 *   n_layers + 1, either may be NULL; synchronizes).
 * st_encoder_fit_capacity: re-plan the arena with every capacity = ceil(
 *   headroom * largest row count seen) (>= 4096, <= the all-active bound;
 *   headroom >= 1), i.e. from measured occupancy instead of the all-active
 *   bound.  Frees and reallocates the arena: borrowed output pointers and
 *   the last step's results become invalid, captured graphs are dropped.
 *   The staged reference frames survive, so the same step can be re-issued
 *   with st_encode_diff.  ST_ERR_UNSUPPORTED for streaming encoders (their
 *   caches live in the arena), ST_ERR_ARG for headroom < 1, ST_ERR_OOM if
 *   the new arena cannot be allocated (the encoder then has none: destroy
 *   it). */
st_status st_step_status(st_encoder *enc);
st_status st_get_capacity(st_encoder *enc, int64_t *rows_cap, int64_t *rows_peak);
st_status st_encoder_fit_capacity(st_encoder *enc, double headroom);

/* Optional per-kernel timing with CUDA events on the launch stream (adds an
 * event pair per launch; off by default).  Kernel classes are named by
 * st_kernel_class_name(i) for i < st_num_kernel_classes(). */
st_status st_set_profiling(st_encoder *enc, int32_t on);
int32_t st_num_kernel_classes(void);
const char *st_kernel_class_name(int32_t i);
/* per class: accumulated ms, launches, algorithmic bytes, algorithmic flops
 * since the last reset (synchronizes). */
st_status st_get_kernel_times(st_encoder *enc, double *ms, int64_t *launches, double *bytes,
                              double *flops, int32_t reset);
int32_t st_last_launch_count(const st_encoder *enc);   /* kernels launched by the last encode */

const char *st_status_string(st_status s);
const char *st_last_error(const st_encoder *enc);

/* ---- online threshold controller (host, readings R15/R16) ----
 * policy 0 fixed, 1 BST, 2 IBST.  One observation per site per step. */
typedef struct st_controller st_controller;
typedef struct {
    int32_t policy;
    float T, eps, theta_max, theta_res, theta_fixed;
    int32_t cycle;           /* IBST restart period in observations */
} st_ctl_config;
st_status st_controller_create(const st_ctl_config *cfg, int32_t n_sites, st_controller **out);
st_status st_controller_observe(st_controller *c, const int64_t *site_active,
                                const int64_t *site_pixels);
st_status st_controller_thresholds(const st_controller *c, float *out);
st_status st_controller_state(const st_controller *c, double *theta, double *lo, double *hi,
                              int32_t *frozen);
void st_controller_destroy(st_controller *c);

#ifdef __cplusplus
}
#endif
#endif /* SPARSETEM_H_ */
