// encoder.cu -- host runtime of libsparsetem.so: validation, shape inference,
// the SparseBatch cache-lifetime planner and arena, the
// per-step executor (a1-a8) and the C ABI of include/sparsetem.h.
//
// SparseBatch: one pass per step.  Layers run in
// topological order; for each layer the reference-frame dense op runs first,
// then the layer's diff op over ALL diff frames of ALL chunks ("N" order).
// A layer's dense reference output (x0 / y0) and its diff tensor live only
// until their last consumer has run; the planner turns those lifetimes into
// arena offsets (greedy first-fit by size over overlapping intervals), so
// the per-layer caches of DeltaCNN never exist.  Only the staged
// reference frames ("one buffer for Subtraction") and the output taps ("one
// for Accumulation") persist across the step.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "sparsetem.h"

using namespace st;

namespace {

constexpr int KC_SUBTRACT = 0, KC_DILATE = 1, KC_SCAN = 2, KC_ENUM = 3, KC_CONV_SPARSE = 4, KC_CONV_DENSE = 5,
              KC_SITE_PW = 6, KC_SITE_MP = 7, KC_ADD = 8, KC_ACCUM = 9, KC_DENSE_MISC = 10, KC_COUNTS = 11,
              KC_DW_SPARSE = 12, KC_DW_DENSE = 13, KC_TC_SPARSE = 14, KC_TC_DENSE = 15, KC_SE = 16,
              KC_STEM_SPARSE = 17, KC_STEM_DENSE = 18, KC_PROF_STATS = 19, KC_SE_SUMS = 20, KC_DW_SITE = 21,
              KC_TC_SITE_FIX = 22, KC_N = 23;
const char *KC_NAMES[KC_N] = {"subtract",   "dilate",       "scan",      "enumerate", "conv_sparse",
                              "conv_dense", "site_pointwise", "site_maxpool", "add",     "accumulate",
                              "dense_misc", "counts",       "dwconv_sparse", "dwconv_dense",
                              "conv_tc_sparse", "conv_tc_dense", "se", "conv_tc_stem_sparse",
                              "conv_tc_stem_dense", "prof_stats", "se_sums", "dwconv_site", "tc_site_fixup"};

struct Buf {
    int64_t bytes = 0;
    int first = 0, last = 0;   // live interval in step time (0 = input site, l+1 = layer l)
    int64_t off = -1;
};

struct LayerRT {
    st_layer_spec spec{};
    int kind = 0, src = -1, src2 = -1;
    int H = 0, W = 0, C = 0;   // output shape
    int site = 0;
    Geo geo{};
    bool depthwise = false;
    bool tc = false;          // BF16 mode: tcgen05 tensor-core conv
    bool tc_small = false;    // BF16 mode: tcgen05 stem on the network input (c_in <= 4)
    int n_consumers = 0, last_consumer = 0;
    int fused_pool = -1;      // ReLU: the maxpool that runs this site in its own pass
    int fused_relu = -1;      // MAXPOOL: the ReLU site folded into this layer's pass
    int fused_dw = -1;        // ReLU/SiLU: the depthwise conv whose pass runs this site (N2)
    int dw_site = -1;         // depthwise CONV: the pointwise site its sparse pass runs
    int act_site = -1;        // non-depthwise CONV: the ReLU/SiLU whose dense output its epilogue writes
    int act_of = -1;          // ReLU/SiLU: the conv that writes its dense output
    int tc_site = -1;         // tcgen05 CONV: the ReLU/SiLU site its sparse epilogue runs (N2)
    int fused_tc = -1;        // ReLU/SiLU: the tcgen05 conv whose epilogue runs this site
    // streaming state (N1, persistent): pointwise site sx[0]/sy[0] in place;
    // maxpool sx[0..1] ping-pong x_acc + spy y_acc; fused pool (on the pool
    // layer) sx[0..1] ReLU x_acc, sy[0..1] ReLU y_acc, spy pool y_acc; OUTPUT sx[0]
    int sx[2] = {-1, -1}, sy[2] = {-1, -1}, spy = -1;
    // device weights (separate allocation)
    float *wk = nullptr, *bias = nullptr;
    uint16_t *wbf = nullptr;  // bf16 [Cout][K] (tc layers)
    alignas(64) unsigned char tmap[128] = {};   // CUtensorMap of wbf (tc layers)
    alignas(64) unsigned char tmap_site[128] = {};   // the same weights with the one-tile N box (tc_site)
    // 1x1/s1 tc convs: A-operand TMA maps over contiguous rows (dense: the
    // input's bf16 shadow; sparse: the rowmap layout's rows), re-encoded per plan
    alignas(64) unsigned char tmap_ad[128] = {};
    alignas(64) unsigned char tmap_as[128] = {};
    bool tma_ad = false, tma_as = false;
    float *se_w1 = nullptr, *se_b1 = nullptr, *se_w2 = nullptr, *se_b2 = nullptr;   // SE MLP
    int b_se = -1;            // SE scratch: sum0 [B][C] f64 | dsum [B][F][C] f64 | s_tab [B][F+1][C] | refresh [B]
    // buffer ids (-1 = none / alias)
    int b_y0 = -1, b_act = -1, b_slot = -1, b_pbase = -1, b_rows = -1, b_ridx = -1, b_out = -1;
    int b_ybf = -1;           // bf16 shadow of y0 (BF16 mode: feeds a tcgen05 conv in dense mode)
    int alias_rows_of = -1;   // rows / slot / pbase borrowed from another tensor
    int64_t rows_cap = 0;     // rows excluding the zero row
    bool rowmap = false;      // CONV 1x1/s1/p0: output rows in the input's row layout, A row r = input row r
                              // (no dilation / scan / gather; reading R26 tiles of the input layout)
    bool zero_gaps = false;   // site: also writes zero rows at touched-but-not-emitted slots (a rowmap
                              // conv reads its layout's rows as a plain matrix)
    bool bf_only = false;     // BF16 mode: the dense output is kept only as its bf16 shadow (every
                              // consumer is a tensor-core conv reading the shadow; SE layers)
};

struct LaunchRec {
    int cls, layer;
    cudaEvent_t e0, e1;
};

struct GraphKey {
    const void *frames;
    int64_t stride;
    int n_diff, chunks;
    int smode;   // streaming: 0 off / first call after a reference, 1 + ping-pong parity on continuations
    bool u8;     // uint8 frames
    bool operator==(const GraphKey &o) const {
        return frames == o.frames && stride == o.stride && n_diff == o.n_diff && chunks == o.chunks &&
               smode == o.smode && u8 == o.u8;
    }
};
struct GraphEnt {
    GraphKey key;
    cudaGraphExec_t exec;
    int launches;
};

}  // namespace

struct st_encoder {
    st_encoder_config cfg{};
    std::vector<LayerRT> L;
    int n_sites = 1;
    int in_H = 0, in_W = 0, in_C = 0;
    int B = 0, F = 0;   // max chunks, max diff frames
    // input site tensor buffers
    int in_act = -1, in_pbase = -1, in_rows = -1;
    int in_dd = -1;              // dense per-frame input delta for CUDA-core convs on the input
    int in_refbf = -1;           // reference frames as 4-channel-padded bf16 (tensor-core stems)
    int64_t in_rows_cap = 0;
    // row capacity (a9): per delta tensor (layer i at i, the input at n) the
    // fitted capacity (-1: none; then cfg.row_frac of the all-active bound)
    std::vector<int64_t> cap_fit;
    int32_t *ovf = nullptr;      // device: a scan clamped a tensor this step
    long long *rows_peak = nullptr;   // device [n + 1]: max unclamped rows per tensor since create
    int64_t fixed_bytes = 0;     // device bytes outside the arena (fixed areas, staged reference, weights)
    bool bf = false;             // BF16 mode: delta rows stored as bf16 (R22-BF16)
    int esz = 4;                 // delta-row element size in bytes
    std::vector<Buf> bufs;
    char *arena = nullptr;
    int64_t arena_bytes = 0, persistent_bytes = 0, peak_transient = 0;
    // small fixed device areas
    char *smallmem = nullptr;
    int32_t *totals = nullptr;   // [n_layers + 1] device row counts
    long long *counts = nullptr; // [B][n_sites][32]
    long long *stats = nullptr;  // [n_layers + 1][3] rows_in, rows_out, touched
    long long *site_sum = nullptr; // [n_sites]
    int32_t *scan_tmp = nullptr;
    float *ref = nullptr;        // staged reference frames [B][N][C]
    float *weights_mem = nullptr;
    uint16_t *wbf_mem = nullptr;
    // thresholds: pinned host staging -> device (a graph node), one fp32 per site
    float *thr_dev = nullptr, *thr_host = nullptr;
    float *zeros = nullptr;   // 1 KiB of device zeros (gather source of absent taps)
    cudaEvent_t thr_ev = nullptr;
    bool thr_pending = false;
    // CUDA graphs of whole steps, keyed by (frames, stride, n_diff, chunks)
    bool use_graphs = true;
    bool use_pdl = false;        // programmatic kernel->kernel edges in captured steps (ST_PDL=1)
    bool dw_rowmajor = false;
    bool prof_trace = false;
    std::vector<GraphEnt> graphs;
    cudaStream_t gstream = nullptr;            // capture / replay stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // dense / diff overlap: the reference (dense) pass of every layer runs on
    // dstream up to ov_k layers ahead of the diff pass (0 = one stream)
    int ov_k = 0;
    cudaStream_t dstream = nullptr;
    std::vector<cudaEvent_t> ev_d, ev_s;
    cudaEvent_t ev_dfork = nullptr, ev_djoin = nullptr;
    // state
    int staged_chunks = 0;       // >0 after encode_reference
    // streaming continuation (N1): cont = the chunks already ran a diff call
    // since their reference; par = ping-pong parity of the shared-halo states
    bool cont = false;
    int par = 0;
    int in_S = -1;               // Subtraction buffer S [B][N][C] (streaming)
    int last_chunks = 0, last_ndiff = -1;
    cudaStream_t last_stream = nullptr;
    std::string err;
    // mask export of one chunk (st_debug_export_chunk): words per layer boundary
    int exp_chunk = -1;
    uint32_t *exp_words = nullptr;
    std::vector<int64_t> exp_off;   // [n_layers + 1]: input site, then layer l at l + 1 (-1 = none)
    bool exp_valid = false;
    // profiling
    bool prof = false;
    std::vector<LaunchRec> recs;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int launches = 0;
    double prof_ms[KC_N] = {0};
    int64_t prof_n[KC_N] = {0};
    double prof_bytes[KC_N] = {0}, prof_flops[KC_N] = {0};

    char *ptr(int id) const { return id < 0 ? nullptr : arena + bufs[id].off; }
    template <class T> T *p(int id) const { return reinterpret_cast<T *>(ptr(id)); }
};

static st_status fail(st_encoder *e, st_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (e) e->err = buf;
    return s;
}

#define CUDA_OK(e, call)                                                                          \
    do {                                                                                          \
        cudaError_t _r = (call);                                                                  \
        if (_r != cudaSuccess) return fail(e, ST_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(_r)); \
    } while (0)

static bool is_site(int k) { return k == ST_RELU || k == ST_SILU || k == ST_MAXPOOL || k == ST_SE; }
static int out_dim(int n, int k, int s, int p) { return (n + 2 * p - k) / s + 1; }

// ----------------------------------------------------------------- profiling
static void prof_begin(st_encoder *e, int cls, int layer, cudaStream_t s) {
    e->launches++;
    if (!e->prof) return;
    while (e->ev_used + 2 > e->ev_pool.size()) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        e->ev_pool.push_back(ev);
    }
    LaunchRec r{cls, layer, e->ev_pool[e->ev_used], e->ev_pool[e->ev_used + 1]};
    e->ev_used += 2;
    cudaEventRecord(r.e0, s);
    e->recs.push_back(r);
}
static void prof_end(st_encoder *e, cudaStream_t s) {
    if (!e->prof) return;
    cudaEventRecord(e->recs.back().e1, s);
}
#define LAUNCH(e, cls, layer, s, stmt) \
    do {                               \
        prof_begin(e, cls, layer, s);  \
        stmt;                          \
        prof_end(e, s);                \
    } while (0)

// ------------------------------------------------------------------- create
static st_status plan(st_encoder *e);
static st_status alloc_fixed(st_encoder *e);
static void encode_act_maps(st_encoder *e);

extern "C" st_status st_encoder_create(const st_encoder_config *cfg, const st_layer_spec *layers, int32_t n,
                                       st_encoder **out) {
    if (!cfg || !out || (n > 0 && !layers) || n < 1) return ST_ERR_ARG;
    *out = nullptr;
    std::unique_ptr<st_encoder> e(new st_encoder());
    e->cfg = *cfg;
    if (cfg->in_c < 1 || cfg->in_c > 4 || cfg->in_h < 1 || cfg->in_w < 1)
        return ST_ERR_SHAPE;
    if (cfg->max_chunks < 1 || cfg->max_frames < 1) return ST_ERR_SHAPE;
    if (cfg->max_frames > 33) return ST_ERR_UNSUPPORTED;   // frame words hold L-1 <= 32 (R25)
    if (cfg->precision != ST_FP32 && cfg->precision != ST_BF16) return ST_ERR_UNSUPPORTED;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return ST_ERR_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10) return ST_ERR_CUDA;
    if (cudaSetDevice(cfg->device) != cudaSuccess) return ST_ERR_CUDA;
    e->in_H = cfg->in_h;
    e->in_W = cfg->in_w;
    e->in_C = cfg->in_c;
    e->B = cfg->max_chunks;
    e->F = cfg->max_frames - 1;
    e->bf = cfg->precision == ST_BF16;
    e->esz = e->bf ? 2 : 4;
    e->L.resize(n);
    // ---- validate + shapes
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        l.spec = layers[i];
        l.kind = layers[i].kind;
        l.src = layers[i].src;
        l.src2 = layers[i].src2;
        if (l.src < -1 || l.src >= i) return ST_ERR_ARG;
        const int sh = l.src < 0 ? e->in_H : e->L[l.src].H, sw = l.src < 0 ? e->in_W : e->L[l.src].W,
                  sc = l.src < 0 ? e->in_C : e->L[l.src].C;
        switch (l.kind) {
        case ST_CONV: {
            const st_layer_spec &s = layers[i];
            if (!s.w || !s.b || s.c_out < 1 || s.groups < 1 || s.k_h < 1 || s.k_w < 1 || s.s_h < 1 || s.s_w < 1 ||
                s.p_h < 0 || s.p_w < 0)
                return ST_ERR_ARG;
            if (s.groups != 1 && !(s.groups == sc && s.c_out == sc)) return ST_ERR_UNSUPPORTED;
            l.depthwise = s.groups != 1;
            l.H = out_dim(sh, s.k_h, s.s_h, s.p_h);
            l.W = out_dim(sw, s.k_w, s.s_w, s.p_w);
            l.C = s.c_out;
            if (s.k_h * s.k_w > 49) return ST_ERR_UNSUPPORTED;
            if (l.depthwise && s.k_h * s.k_w > 25) return ST_ERR_UNSUPPORTED;   // depthwise kernels: <= 5x5 taps
            break;
        }
        case ST_MAXPOOL: {
            const st_layer_spec &s = layers[i];
            if (s.k_h < 1 || s.k_w < 1 || s.s_h < 1 || s.s_w < 1 || s.p_h < 0 || s.p_w < 0) return ST_ERR_ARG;
            if (s.k_h * s.k_w > 9) return ST_ERR_UNSUPPORTED;
            l.H = out_dim(sh, s.k_h, s.s_h, s.p_h);
            l.W = out_dim(sw, s.k_w, s.s_w, s.p_w);
            l.C = sc;
            break;
        }
        case ST_ADD: {
            if (l.src2 < -1 || l.src2 >= i) return ST_ERR_ARG;
            const int h2 = l.src2 < 0 ? e->in_H : e->L[l.src2].H, w2 = l.src2 < 0 ? e->in_W : e->L[l.src2].W,
                      c2 = l.src2 < 0 ? e->in_C : e->L[l.src2].C;
            if (h2 != sh || w2 != sw || c2 != sc) return ST_ERR_SHAPE;
            l.H = sh; l.W = sw; l.C = sc;
            break;
        }
        case ST_RELU: case ST_SILU: case ST_OUTPUT:
            l.H = sh; l.W = sw; l.C = sc;
            break;
        case ST_SE:
            if (!layers[i].w || !layers[i].b || !layers[i].w2 || !layers[i].b2 || layers[i].se_hidden < 1)
                return ST_ERR_ARG;
            l.H = sh; l.W = sw; l.C = sc;
            break;
        default:
            return ST_ERR_ARG;
        }
        if (l.H < 1 || l.W < 1) return ST_ERR_SHAPE;
        if (l.kind == ST_CONV || l.kind == ST_MAXPOOL) {
            const st_layer_spec &s = layers[i];
            l.geo = Geo{sh, sw, sc, l.H, l.W, l.C, s.k_h, s.k_w, s.s_h, s.s_w, s.p_h, s.p_w, s.groups};
        }
        if (is_site(l.kind)) l.site = e->n_sites++;
        // register-resident site kernels: <= 1152 channels at maxpool / SE
        // sites; pointwise sites, joins and taps up to 2048 (wide kernels)
        if (l.C > 4096 || (l.kind == ST_MAXPOOL && l.C > 1152) || (l.kind == ST_SE && l.C > 1152 && l.C % 8 != 0))
            return ST_ERR_UNSUPPORTED;
        if ((l.kind == ST_ADD || l.kind == ST_OUTPUT) && l.C > 2048) return ST_ERR_UNSUPPORTED;
        if ((l.kind == ST_RELU || l.kind == ST_SILU) && l.C > 1280 && l.C % 8 != 0) return ST_ERR_UNSUPPORTED;
    }
    // consumers
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        for (int s : {l.src, l.kind == ST_ADD ? l.src2 : -2}) {
            if (s >= 0) {
                e->L[s].n_consumers++;
                e->L[s].last_consumer = std::max(e->L[s].last_consumer, i);
            }
        }
    }
    if (cfg->streaming)
        for (auto &l : e->L)
            if (l.kind == ST_SE) return ST_ERR_UNSUPPORTED;   // SE gate schedule spans the call (R8)
    // ReLU -> maxpool pairs run as one tile-resident pass (the ReLU output is
    // read only by the pool, its input is a conv tensor, windows cover the map)
    {
        const char *nf = getenv("ST_NO_FUSE");   // A/B switch
        if (!(nf && nf[0] == '1'))
            for (int i = 0; i < n; i++) {
                LayerRT &p = e->L[i];
                if (p.kind != ST_MAXPOOL || p.src < 0) continue;
                LayerRT &r = e->L[p.src];
                if (r.kind != ST_RELU || r.n_consumers != 1 || r.src < 0 || e->L[r.src].kind != ST_CONV) continue;
                if (!site_relu_maxpool_fusable(p.geo, e->bf)) continue;
                p.fused_relu = p.src;
                r.fused_pool = i;
            }
    }
    // depthwise conv -> pointwise site (ReLU / SiLU, the conv's only consumer):
    // the site's state machine runs in the conv's pixel loop
    {
        const char *nf = getenv("ST_NO_FUSE_DW");   // A/B switch
        const char *dr = getenv("ST_DW_ROWMAJOR");
        if (!(nf && nf[0] == '1') && !(dr && dr[0] == '1') && !cfg->streaming)
            for (int i = 0; i < n; i++) {
                LayerRT &r = e->L[i];
                if ((r.kind != ST_RELU && r.kind != ST_SILU) || r.src < 0) continue;
                LayerRT &cv = e->L[r.src];
                if (cv.kind != ST_CONV || !cv.depthwise || cv.n_consumers != 1 || !dwconv_site_fusable(cv.geo)) continue;
                r.fused_dw = r.src;
                cv.dw_site = i;
            }
    }
    // 1x1/s1 convs in the input's row layout (rowmap): the layout must have no
    // stale rows at touched-but-not-emitted slots -- input site, convs, adds
    // have none; ReLU / SiLU / SE sites are asked to zero theirs (zero_gaps);
    // maxpool layouts are not used
    {
        const char *nr = getenv("ST_NO_ROWMAP");   // A/B switch
        if (!(nr && nr[0] == '1'))
            for (int i = 0; i < n; i++) {
                LayerRT &l = e->L[i];
                if (l.kind != ST_CONV || l.depthwise || l.spec.groups != 1 || l.spec.k_h != 1 || l.spec.k_w != 1 ||
                    l.spec.s_h != 1 || l.spec.s_w != 1 || l.spec.p_h != 0 || l.spec.p_w != 0 || l.src < 0)
                    continue;
                int o = l.src;
                while (o >= 0 && e->L[o].kind == ST_OUTPUT) o = e->L[o].src;
                if (o < 0) continue;
                // the layout's owner chain: sites / rowmap convs borrow their source's layout
                bool ok = true;
                for (int t = o; t >= 0;) {
                    const LayerRT &q = e->L[t];
                    // maxpool layouts hold the footprint dilation; an SE layout holds
                    // every pixel of a gate-refresh frame (R8): both can be far denser
                    // than the emitted rows, so those convs keep the gathered M list
                    if (q.kind == ST_MAXPOOL || q.kind == ST_SE || q.fused_pool >= 0) { ok = false; break; }
                    if (q.kind == ST_RELU || q.kind == ST_SILU || (q.kind == ST_CONV && q.rowmap)) {
                        t = q.src;
                        while (t >= 0 && e->L[t].kind == ST_OUTPUT) t = e->L[t].src;
                        continue;
                    }
                    break;
                }
                if (!ok) continue;
                l.rowmap = true;
                for (int t = o; t >= 0;) {   // every site on the chain zero-fills its gaps
                    LayerRT &q = e->L[t];
                    if (q.kind == ST_RELU || q.kind == ST_SILU || q.kind == ST_SE) q.zero_gaps = true;
                    if (q.kind == ST_RELU || q.kind == ST_SILU || (q.kind == ST_CONV && q.rowmap)) {
                        t = q.src;
                        while (t >= 0 && e->L[t].kind == ST_OUTPUT) t = e->L[t].src;
                        continue;
                    }
                    break;
                }
            }
    }
    // ---- weights (K-major repack: wk[(dy*kw+dx)*cin_g + ci][co], reading R18)
    int64_t wfloats = 0;
    for (auto &l : e->L)
        if (l.kind == ST_CONV) {
            const int cin_g = l.geo.Cin / l.spec.groups;
            wfloats += ((int64_t)l.spec.k_h * l.spec.k_w * cin_g * l.C + 63) / 64 * 64 + (l.C + 63) / 64 * 64;
        } else if (l.kind == ST_SE) {
            const int64_t hc = (int64_t)l.spec.se_hidden * l.C;
            wfloats += 2 * ((hc + 63) / 64 * 64) + (l.spec.se_hidden + 63) / 64 * 64 + (l.C + 63) / 64 * 64;
        }
    CUDA_OK(e.get(), cudaMalloc(&e->weights_mem, std::max<int64_t>(wfloats, 1) * sizeof(float)));
    e->fixed_bytes += std::max<int64_t>(wfloats, 1) * (int64_t)sizeof(float);
    {
        std::vector<float> host(std::max<int64_t>(wfloats, 1));
        int64_t o = 0;
        auto put = [&](const float *src, int64_t n) {
            float *dst = e->weights_mem + o;
            for (int64_t k = 0; k < n; k++) host[o + k] = src[k];
            o += (n + 63) / 64 * 64;
            return dst;
        };
        for (auto &l : e->L) {
            if (l.kind == ST_SE) {
                const int64_t hc = (int64_t)l.spec.se_hidden * l.C;
                l.se_w1 = put(l.spec.w, hc);
                l.se_b1 = put(l.spec.b, l.spec.se_hidden);
                l.se_w2 = put(l.spec.w2, hc);
                l.se_b2 = put(l.spec.b2, l.C);
                continue;
            }
            if (l.kind != ST_CONV) continue;
            const int kh = l.spec.k_h, kw = l.spec.k_w, cin_g = l.geo.Cin / l.spec.groups, co = l.C;
            l.wk = e->weights_mem + o;
            // BF16 mode (R22-BF16): every conv multiplies bf16-rounded weights,
            // so the CUDA-core convs (depthwise, small c_in) get RNE-rounded values too
            const bool rw = cfg->precision == ST_BF16;
            for (int dy = 0; dy < kh; dy++)
                for (int dx = 0; dx < kw; dx++)
                    for (int ci = 0; ci < cin_g; ci++)
                        for (int c = 0; c < co; c++) {
                            float v = l.spec.w[(((int64_t)c * cin_g + ci) * kh + dy) * kw + dx];
                            if (rw) {
                                uint32_t u;
                                std::memcpy(&u, &v, 4);
                                u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
                                std::memcpy(&v, &u, 4);
                            }
                            host[o + ((int64_t)(dy * kw + dx) * cin_g + ci) * co + c] = v;
                        }
            o += ((int64_t)kh * kw * cin_g * co + 63) / 64 * 64;   // 256-byte aligned (float4 loads)
            l.bias = e->weights_mem + o;
            for (int c = 0; c < co; c++) host[o + c] = l.spec.b[c];
            o += (co + 63) / 64 * 64;
        }
        CUDA_OK(e.get(), cudaMemcpy(e->weights_mem, host.data(), host.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    // ---- BF16 mode: tensor-core layers get bf16 [Cout][K] weights (RNE)
    if (cfg->precision == ST_BF16) {
        // weight K per tc layer: kh*kw*Cpad in (dy, dx, ci) order, each tap's
        // channels zero-padded to a multiple of 64; stems pack each tap as a
        // 4-channel piece (zero pad) and round K up to 64
        auto tc_k = [](const LayerRT &l) -> int64_t {
            return l.tc_small ? conv_tc_small_k(l.geo) : (int64_t)l.spec.k_h * l.spec.k_w * conv_tc_cpad(l.geo.Cin);
        };
        int64_t nbf = 0;
        for (auto &l : e->L) {
            if (l.kind != ST_CONV) continue;
            if (conv_tc_eligible(l.geo)) l.tc = true;
            else if (l.src == -1 && conv_tc_small_eligible(l.geo)) l.tc_small = true;
            if (l.tc || l.tc_small) nbf += (tc_k(l) * l.C + 127) / 128 * 128;
        }
        if (nbf) {
            CUDA_OK(e.get(), cudaMalloc(&e->wbf_mem, nbf * 2));
            e->fixed_bytes += nbf * 2;
            std::vector<uint16_t> hb(nbf, 0);
            int64_t o = 0;
            for (auto &l : e->L) {
                if (!l.tc && !l.tc_small) continue;
                const int kh = l.spec.k_h, kw = l.spec.k_w, ci_n = l.geo.Cin, co = l.C;
                const int64_t K = tc_k(l);
                const int cstep = l.tc_small ? 4 : conv_tc_cpad(ci_n);   // elements per tap in the K layout
                int sr = 0, shift = 0;
                if (l.tc_small) conv_tc_small_layout(l.geo, sr, shift);
                l.wbf = e->wbf_mem + o;
                for (int c = 0; c < co; c++)
                    for (int dy = 0; dy < kh; dy++)
                        for (int dx = 0; dx < kw; dx++)
                            for (int ci = 0; ci < ci_n; ci++) {
                                float v = l.spec.w[(((int64_t)c * ci_n + ci) * kh + dy) * kw + dx];
                                uint32_t u;
                                std::memcpy(&u, &v, 4);
                                u += 0x7FFFu + ((u >> 16) & 1u);   // round to nearest even
                                const int slot = sr ? dy * sr + dx + shift : dy * kw + dx;
                                hb[o + (int64_t)c * K + slot * cstep + ci] = (uint16_t)(u >> 16);
                            }
                o += (K * co + 127) / 128 * 128;
            }
            CUDA_OK(e.get(), cudaMemcpy(e->wbf_mem, hb.data(), nbf * 2, cudaMemcpyHostToDevice));
            for (auto &l : e->L)
                if ((l.tc || l.tc_small) && !make_weight_tmap(l.tmap, l.wbf, (int)tc_k(l), l.C))
                    return fail(e.get(), ST_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        }
    }
    // conv -> ReLU / SiLU (its only consumer): the conv's dense epilogue also
    // writes the site's dense output (no separate activation pass); not for a
    // ReLU fused into a maxpool (the pool's dense pass applies it) or streaming
    if (!cfg->streaming)
        for (int i = 0; i < n; i++) {
            LayerRT &r = e->L[i];
            if ((r.kind != ST_RELU && r.kind != ST_SILU) || r.src < 0 || r.fused_dw >= 0 || r.fused_pool >= 0) continue;
            LayerRT &cv = e->L[r.src];
            // tensor-core convs: the dense epilogue stages 32 x 32 blocks through
            // shared memory and writes f(x0) (+ bf16 shadow) with the same coalesced
            // stores (ST_TC_ACT=0: the separate activation pass, as when the
            // epilogue wrote a row per thread and measured slower)
            const char *tca = getenv("ST_TC_ACT");   // read per create (tests switch it)
            const bool tc_act = tca && tca[0] == '1';
            if (cv.kind != ST_CONV || cv.depthwise || cv.n_consumers != 1) continue;
            if ((cv.tc || cv.tc_small) && !tc_act) continue;
            cv.act_site = i;
            r.act_of = r.src;
        }
    // tcgen05 conv -> ReLU / SiLU (its only consumer, c_out <= 256): the site
    // runs in the conv's epilogue, with a weight map for the
    // one-tile N width.  Opt-in (ST_FUSE_TC=1): measured slower on every
    // workload -- the per-pixel site chain in the 4 epilogue warps of one CTA
    // per SM cannot keep up with the MMA pipeline (cfg5 sparse convs 3.1 ->
    // 19.7 ms for 3.2 ms of site kernels saved; cfg4 +3 ms; cfg2 +0.1 ms)
    {
        const char *ff = getenv("ST_FUSE_TC");
        if (e->bf && (ff && ff[0] == '1') && !cfg->streaming && !cfg->debug_retain)
            for (int i = 0; i < n; i++) {
                LayerRT &r = e->L[i];
                if ((r.kind != ST_RELU && r.kind != ST_SILU) || r.src < 0 || r.fused_dw >= 0 || r.fused_pool >= 0 ||
                    r.act_of >= 0)
                    continue;
                LayerRT &cv = e->L[r.src];
                if (cv.kind != ST_CONV || !cv.tc || cv.n_consumers != 1 || !conv_tc_site_eligible(cv.geo)) continue;
                const int64_t K = (int64_t)cv.spec.k_h * cv.spec.k_w * conv_tc_cpad(cv.geo.Cin);
                if (!make_weight_tmap_site(cv.tmap_site, cv.wbf, (int)K, cv.C))
                    return fail(e.get(), ST_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                cv.tc_site = i;
                r.fused_tc = r.src;
            }
    }
    for (auto &l : e->L) { l.spec.w = l.spec.b = l.spec.w2 = l.spec.b2 = nullptr; }
    e->cap_fit.assign(n + 1, -1);
    {   // ST_OVERLAP=0: one stream; ST_OVERLAP_K: lookahead in layers (default 6)
        const char *ov = getenv("ST_OVERLAP"), *ok = getenv("ST_OVERLAP_K"), *np = getenv("ST_PDL");
        const bool off = (ov && ov[0] == '0') || cfg->streaming || cfg->debug_retain || (np && np[0] == '1');
        e->ov_k = off ? 0 : std::max(1, ok ? atoi(ok) : 6);
    }
    st_status r = plan(e.get());
    if (r == ST_OK) r = alloc_fixed(e.get());
    if (r == ST_OK) encode_act_maps(e.get());
    if (r != ST_OK) {
        cudaFree(e->weights_mem);
        return r;
    }
    *out = e.release();
    return ST_OK;
}

// ------------------------------------------------------------------- planner
// row capacity of delta tensor `idx` (layer i, or n = the input site) whose
// all-active bound is `full` rows (B * (L-1) * N): the fitted capacity, else
// cfg.row_frac of the bound (at least 4096 rows), else the bound
static int64_t cap_for(const st_encoder *e, int idx, int64_t full) {
    if (e->cap_fit[idx] >= 0) return std::min(full, e->cap_fit[idx]);
    const double f = e->cfg.row_frac;
    if (f > 0.0 && f < 1.0) return std::min(full, std::max<int64_t>((int64_t)std::ceil(f * (double)full), 4096));
    return full;
}

// the tensor whose slot / pbase (row layout) a layer's delta tensor uses:
// sites and rowmap convs borrow their source's layout; n = the input site
static int layout_owner(const st_encoder *e, int t) {
    while (t >= 0) {
        const LayerRT &l = e->L[t];
        if (l.kind == ST_OUTPUT || l.kind == ST_RELU || l.kind == ST_SILU || (l.kind == ST_CONV && l.rowmap)) t = l.src;
        else return t;
    }
    return (int)e->L.size();
}

static st_status plan(st_encoder *e) {
    const int n = (int)e->L.size();
    const int64_t B = e->B, F = e->F;
    const int END = n + 1;   // step end
    e->bufs.clear();
    e->in_act = e->in_pbase = e->in_rows = e->in_dd = e->in_refbf = e->in_S = -1;
    for (auto &l : e->L) {
        l.b_y0 = l.b_act = l.b_slot = l.b_pbase = l.b_rows = l.b_ridx = l.b_out = l.b_ybf = l.b_se = -1;
        l.alias_rows_of = -1;
        l.sx[0] = l.sx[1] = l.sy[0] = l.sy[1] = l.spy = -1;
    }
    // SE outputs whose every consumer is a tensor-core conv (the 1x1 project
    // conv of an MBConv block) keep only the bf16 shadow of their dense output
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        l.bf_only = false;
        if (l.kind != ST_SE || !e->bf || e->cfg.debug_retain || e->cfg.streaming || l.n_consumers == 0) continue;
        bool ok = true;
        for (int j = i + 1; j < n; j++) {
            const LayerRT &c = e->L[j];
            if (c.src == i || (c.kind == ST_ADD && c.src2 == i)) ok = ok && c.kind == ST_CONV && c.tc;
        }
        l.bf_only = ok;
    }
    auto add = [&](int64_t bytes, int first, int last) {
        Buf b;
        b.bytes = (bytes + 255) / 256 * 256;
        if (e->cfg.debug_retain) { first = 0; last = END; }
        b.first = first;
        b.last = last;
        e->bufs.push_back(b);
        return (int)e->bufs.size() - 1;
    };
    auto t_of = [](int layer) { return layer + 1; };   // step time of a layer
    // input site: consumers of -1
    int in_last = 0;
    for (int i = 0; i < n; i++)
        if (e->L[i].src == -1 || (e->L[i].kind == ST_ADD && e->L[i].src2 == -1)) in_last = std::max(in_last, t_of(i));
    const int64_t Nin = (int64_t)e->in_H * e->in_W;
    e->in_rows_cap = cap_for(e, n, B * F * Nin);
    e->in_act = add(B * Nin * 4, 0, in_last);
    e->in_pbase = add(B * Nin * 4, 0, in_last);
    const int64_t ES = e->esz;   // delta-row element size: 4 (FP32 mode) or 2 (BF16 mode)
    e->in_rows = add((e->in_rows_cap + 1) * e->in_C * ES, 0, in_last);
    // convs reading the network input on CUDA cores (c_in <= 4 stems) gather
    // from a dense per-frame delta written by the Subtraction pass instead of
    // resolving every tap through the frame words
    bool want_dd = false;
    for (auto &l : e->L)
        if (l.kind == ST_CONV && l.src == -1 && !l.depthwise && !l.tc) want_dd = true;   // incl. tc_small
    if (want_dd) e->in_dd = add(B * F * Nin * 4 * ES, 0, in_last);   // pixels padded to 4 channels
    bool want_refbf = false;   // stems on tensor cores read the reference frames as padded bf16
    for (auto &l : e->L)
        if (l.kind == ST_CONV && l.tc_small) want_refbf = true;
    if (want_refbf) e->in_refbf = add(B * Nin * 4 * 2, 0, in_last);
    // per-layer tensors
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        const int64_t N = (int64_t)l.H * l.W;
        const int tdef = t_of(i);
        const int tlast = std::max(tdef, l.n_consumers ? t_of(l.last_consumer) : tdef);
        if (l.kind == ST_OUTPUT) {
            // Accumulation buffer: persistent [B][L][N][C]
            l.b_out = add(B * (F + 1) * N * l.C * 4, 0, END);
            continue;
        }
        l.b_y0 = l.bf_only ? -1 : add(B * N * l.C * 4, tdef, tlast);
        if (l.bf_only) l.b_ybf = add(B * N * l.C * 2, tdef, tlast);
        if (l.kind == ST_CONV && l.rowmap) {
            // rows in the input's layout (same capacity); frame words borrowed
            const int o = layout_owner(e, l.src);
            l.rows_cap = o == n ? e->in_rows_cap : e->L[o].rows_cap;
            l.b_rows = add((l.rows_cap + 1) * l.C * ES, tdef, tlast);
            if (l.tc_site >= 0) l.b_ridx = add(std::max<int64_t>(l.rows_cap, 1) * 4, tdef, tdef);   // row codes
            continue;
        }
        l.b_act = add(B * N * 4, tdef, tlast);
        l.rows_cap = cap_for(e, i, B * F * N);
        switch (l.kind) {
        case ST_CONV:
            l.b_pbase = add(B * N * 4, tdef, tlast);
            l.b_rows = add((l.rows_cap + 1) * l.C * ES, tdef, tlast);
            l.b_ridx = add(std::max<int64_t>(l.rows_cap, 1) * 4, tdef, tdef);
            break;
        case ST_MAXPOOL: case ST_ADD: case ST_SE:
            l.b_slot = add(B * N * 4, tdef, tlast);
            l.b_pbase = add(B * N * 4, tdef, tlast);
            l.b_rows = add((l.rows_cap + 1) * l.C * ES, tdef, tlast);
            if (l.kind == ST_SE)   // sum0 | dsum | s_tab | refresh, used only while the layer runs
                l.b_se = add(B * l.C * 8 + B * F * l.C * 8 + 2 * B * (F + 1) * l.C * 4 + B * 4 + 128, tdef, tdef);
            break;
        case ST_RELU: case ST_SILU: {
            // emitted rows go into the input's slot layout; in place when
            // this site is the input's only consumer (and not debugging)
            const LayerRT *sl = l.src >= 0 ? &e->L[l.src] : nullptr;
            const bool sole = sl ? sl->n_consumers == 1 : false;
            if (sole && !e->cfg.debug_retain) {
                l.alias_rows_of = l.src;
            } else {
                l.alias_rows_of = l.src;   // slot/pbase still borrowed
                const int64_t cap = sl ? sl->rows_cap : e->in_rows_cap;
                l.b_rows = add((cap + 1) * l.C * ES, tdef, tlast);
            }
            break;
        }
        default:
            break;
        }
    }
    // bf16 shadows of dense activations read by tcgen05 convs in dense mode
    // (same live interval as the fp32 y0 they shadow)
    for (int i = 0; i < n; i++) {
        const LayerRT &c = e->L[i];
        if (c.kind != ST_CONV || !c.tc || c.src < 0) continue;
        int o = c.src;
        while (o >= 0 && e->L[o].kind == ST_OUTPUT) o = e->L[o].src;
        if (o < 0 || e->L[o].b_y0 < 0 || e->L[o].b_ybf >= 0) continue;   // (bf_only: shadow already planned)
        const LayerRT &ol = e->L[o];
        const Buf &yb = e->bufs[ol.b_y0];
        e->L[o].b_ybf = add(B * (int64_t)ol.H * ol.W * ol.C * 2, yb.first, yb.last);
    }
    // aliases extend the lifetime of the borrowed buffers
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        const bool rm = l.kind == ST_CONV && l.rowmap;
        if (l.alias_rows_of < 0 && !(l.kind == ST_RELU || l.kind == ST_SILU) && !rm) continue;
        const int tlast = std::max(t_of(i), l.n_consumers ? t_of(l.last_consumer) : t_of(i));
        int s = l.src;
        bool rows_too = !rm;   // a rowmap conv borrows frame words only
        while (true) {   // walk to the tensor that owns slot/pbase (and maybe rows)
            while (s >= 0 && e->L[s].kind == ST_OUTPUT) s = e->L[s].src;
            if (s < 0) {
                for (int id : {e->in_act, e->in_pbase}) e->bufs[id].last = std::max(e->bufs[id].last, tlast);
                if (rows_too) e->bufs[e->in_rows].last = std::max(e->bufs[e->in_rows].last, tlast);
                break;
            }
            LayerRT &o = e->L[s];
            for (int id : {o.b_act, o.b_slot, o.b_pbase})
                if (id >= 0) e->bufs[id].last = std::max(e->bufs[id].last, tlast);
            if (rows_too && o.b_rows >= 0) e->bufs[o.b_rows].last = std::max(e->bufs[o.b_rows].last, tlast);
            if (o.kind == ST_RELU || o.kind == ST_SILU) { s = o.src; continue; }
            if (o.kind == ST_CONV && o.rowmap) { s = o.src; rows_too = false; continue; }
            break;
        }
    }
    // streaming state (N1): the vanilla schedule's persistent caches
    if (e->cfg.streaming) {
        e->in_S = add(B * Nin * e->in_C * 4, 0, END);
        for (int i = 0; i < n; i++) {
            LayerRT &l = e->L[i];
            const int64_t No = (int64_t)l.H * l.W * l.C;
            const int64_t Ni = l.src < 0 ? Nin * e->in_C : (int64_t)e->L[l.src].H * e->L[l.src].W * e->L[l.src].C;
            if (l.kind == ST_OUTPUT) {
                l.sx[0] = add(B * No * 4, 0, END);
            } else if ((l.kind == ST_RELU || l.kind == ST_SILU) && l.fused_pool < 0) {
                l.sx[0] = add(B * No * 4, 0, END);
                l.sy[0] = add(B * No * 4, 0, END);
            } else if (l.kind == ST_MAXPOOL) {
                for (int k = 0; k < 2; k++) l.sx[k] = add(B * Ni * 4, 0, END);
                if (l.fused_relu >= 0)
                    for (int k = 0; k < 2; k++) l.sy[k] = add(B * Ni * 4, 0, END);
                l.spy = add(B * No * 4, 0, END);
            }
        }
    }
    // a depthwise conv's pass writes its fused site's dense output (dense
    // epilogue) and frame words (sparse pass) at the conv's step time
    for (int i = 0; i < n; i++)
        if (e->L[i].fused_tc >= 0) {
            const int tc = t_of(e->L[i].fused_tc);
            for (int id : {e->L[i].b_act, e->L[i].b_rows})
                if (id >= 0) e->bufs[id].first = std::min(e->bufs[id].first, tc);
        }
    for (int i = 0; i < n; i++)
        if (e->L[i].act_of >= 0) {
            const int tc = t_of(e->L[i].act_of);
            for (int id : {e->L[i].b_y0, e->L[i].b_ybf})
                if (id >= 0) e->bufs[id].first = std::min(e->bufs[id].first, tc);
        }
    for (int i = 0; i < n; i++)
        if (e->L[i].fused_dw >= 0) {
            const int tc = t_of(e->L[i].fused_dw);
            for (int id : {e->L[i].b_y0, e->L[i].b_ybf, e->L[i].b_act, e->L[i].b_rows})
                if (id >= 0) e->bufs[id].first = std::min(e->bufs[id].first, tc);
        }
    // a fused ReLU -> maxpool pass reads the conv's dense pre-activation (the
    // ReLU's x0) at the pool's step time
    for (int i = 0; i < n; i++)
        if (e->L[i].fused_relu >= 0) {
            const LayerRT &cv = e->L[e->L[e->L[i].fused_relu].src];
            if (cv.b_y0 >= 0) e->bufs[cv.b_y0].last = std::max(e->bufs[cv.b_y0].last, t_of(i));
        }
    // dense / diff overlap: a layer's dense op may run up to ov_k layers ahead of
    // its step (it waits for the diff pass of layer i - ov_k), so every buffer a
    // dense op writes -- y0, its bf16 shadow, the SE's sums / gate table -- is
    // live from ov_k steps earlier; consumers still finish by their own step
    // (a diff op waits for the dense op of its layer)
    if (e->ov_k > 0)
        for (auto &l : e->L)
            for (int id : {l.b_y0, l.b_ybf, l.b_se})
                if (id >= 0) e->bufs[id].first = std::max(0, e->bufs[id].first - e->ov_k);
    // ---- first-fit arena assignment, largest first
    std::vector<int> order(e->bufs.size());
    for (size_t i = 0; i < order.size(); i++) order[i] = (int)i;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return e->bufs[a].bytes > e->bufs[b].bytes; });
    std::vector<int> placed;
    int64_t total = 0;
    for (int id : order) {
        Buf &b = e->bufs[id];
        std::vector<std::pair<int64_t, int64_t>> busy;
        for (int pid : placed) {
            const Buf &o = e->bufs[pid];
            if (o.first <= b.last && b.first <= o.last) busy.push_back({o.off, o.off + o.bytes});
        }
        std::sort(busy.begin(), busy.end());
        int64_t off = 0;
        for (auto &iv : busy) {
            if (off + b.bytes <= iv.first) break;
            off = std::max(off, iv.second);
        }
        b.off = off;
        total = std::max(total, off + b.bytes);
        placed.push_back(id);
    }
    e->arena_bytes = total;
    // memory report
    int64_t persistent = 0;
    for (auto &l : e->L)
        if (l.b_out >= 0) persistent += e->bufs[l.b_out].bytes;
    persistent += B * Nin * e->in_C * 4;   // staged reference (Subtraction buffer)
    if (e->in_S >= 0) persistent += e->bufs[e->in_S].bytes;   // streaming caches (N1)
    for (auto &l : e->L)
        for (int id : {l.sx[0], l.sx[1], l.sy[0], l.sy[1], l.spy})
            if (id >= 0) persistent += e->bufs[id].bytes;
    e->persistent_bytes = persistent;
    int64_t peak = 0;
    for (int t = 0; t <= END; t++) {
        int64_t live = 0;
        for (auto &b : e->bufs)
            if (b.first <= t && t <= b.last && b.first != 0) live += b.bytes;
        for (auto &b : e->bufs)
            if (b.first == 0 && b.last != END && t <= b.last) live += b.bytes;
        peak = std::max(peak, live);
    }
    e->peak_transient = peak;
    if (cudaMalloc(&e->arena, std::max<int64_t>(total, 256)) != cudaSuccess) {
        cudaGetLastError();
        e->arena = nullptr;
        return fail(e, ST_ERR_OOM, "arena of %lld bytes failed", (long long)total);
    }
    return ST_OK;
}

// fixed device areas (counts, scan scratch, thresholds, staged reference ...),
// streams and events: allocated once at create
static st_status alloc_fixed(st_encoder *e) {
    const int n = (int)e->L.size();
    const int64_t B = e->B;
    const int64_t Nin = (int64_t)e->in_H * e->in_W;
    int64_t max_words = B * Nin;
    for (auto &l : e->L) max_words = std::max<int64_t>(max_words, B * l.H * l.W);
    const int64_t small = (n + 1) * 4 + B * e->n_sites * 32 * 8 + (n + 1) * 3 * 8 + e->n_sites * 8 +
                          scan_tmp_ints(max_words) * 4 + e->n_sites * 4 + 1024 + (n + 1) * 8 + 256 + 10 * 256;
    CUDA_OK(e, cudaMalloc(&e->smallmem, small));
    char *p = e->smallmem;
    auto take = [&](int64_t bytes) { char *r = p; p += (bytes + 255) / 256 * 256; return r; };
    e->totals = (int32_t *)take((n + 1) * 4);
    e->counts = (long long *)take(B * e->n_sites * 32 * 8);
    e->stats = (long long *)take((n + 1) * 3 * 8);
    e->site_sum = (long long *)take(e->n_sites * 8);
    e->scan_tmp = (int32_t *)take(scan_tmp_ints(max_words) * 4);
    e->thr_dev = (float *)take(e->n_sites * 4);
    e->zeros = (float *)take(1024);
    CUDA_OK(e, cudaMemset(e->zeros, 0, 1024));
    e->rows_peak = (long long *)take((n + 1) * 8);
    e->ovf = (int32_t *)take(256);
    CUDA_OK(e, cudaMemset(e->rows_peak, 0, (n + 1) * 8));
    CUDA_OK(e, cudaMemset(e->ovf, 0, 4));
    CUDA_OK(e, cudaMallocHost(&e->thr_host, e->n_sites * 4));
    CUDA_OK(e, cudaEventCreateWithFlags(&e->thr_ev, cudaEventDisableTiming));
    const char *ng = getenv("ST_NO_GRAPHS");
    e->use_graphs = !(ng && ng[0] == '1');
    // programmatic edges measured neutral-to-slower on cfg2/cfg4 (592.9K vs
    // 582.6K diff-frames/s, profiles/r01i_bench_cfg2_pdl.json): opt-in
    const char *np = getenv("ST_PDL");
    e->use_pdl = np && np[0] == '1';
    const char *dr = getenv("ST_DW_ROWMAJOR");   // A/B switch: the M-row depthwise kernel
    e->dw_rowmajor = dr && dr[0] == '1';
    const char *pt = getenv("ST_PROF_TRACE");    // per-launch profile lines on stderr
    e->prof_trace = pt && pt[0] == '1';
    CUDA_OK(e, cudaStreamCreateWithFlags(&e->gstream, cudaStreamNonBlocking));
    CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
    CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    if (e->ov_k > 0) {
        // ST_OVERLAP_PRIO: the dense stream's priority relative to the diff pass
        // (-1 lower -- the default: the diff pass is the critical path --, 0 equal,
        // 1 higher); the capture / replay stream carries the diff pass
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        const char *pp = getenv("ST_OVERLAP_PRIO");
        const int pr = pp ? atoi(pp) : -1;
        if (pr != 0) {
            cudaStreamDestroy(e->gstream);
            CUDA_OK(e, cudaStreamCreateWithPriority(&e->gstream, cudaStreamNonBlocking, pr < 0 ? greatest : least));
        }
        CUDA_OK(e, cudaStreamCreateWithPriority(&e->dstream, cudaStreamNonBlocking,
                                                pr < 0 ? least : pr > 0 ? greatest : least));
        CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_dfork, cudaEventDisableTiming));
        CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_djoin, cudaEventDisableTiming));
        e->ev_d.resize(e->L.size());
        e->ev_s.resize(e->L.size());
        for (size_t i = 0; i < e->L.size(); i++) {
            CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_d[i], cudaEventDisableTiming));
            CUDA_OK(e, cudaEventCreateWithFlags(&e->ev_s[i], cudaEventDisableTiming));
        }
    }
    (void)take(0);
    CUDA_OK(e, cudaMalloc(&e->ref, B * Nin * e->in_C * 4));
    // zero rows (row 0 of every rows buffer) are written per step (arena reuse)
    e->fixed_bytes += small + B * Nin * e->in_C * 4;
    return ST_OK;
}

extern "C" void st_encoder_destroy(st_encoder *e) {
    if (!e) return;
    cudaFree(e->exp_words);
    cudaFree(e->arena);
    cudaFree(e->smallmem);
    cudaFree(e->ref);
    cudaFree(e->weights_mem);
    cudaFree(e->wbf_mem);
    for (auto &g : e->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (e->thr_host) cudaFreeHost(e->thr_host);
    if (e->thr_ev) cudaEventDestroy(e->thr_ev);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    if (e->gstream) cudaStreamDestroy(e->gstream);
    if (e->dstream) cudaStreamDestroy(e->dstream);
    if (e->ev_dfork) cudaEventDestroy(e->ev_dfork);
    if (e->ev_djoin) cudaEventDestroy(e->ev_djoin);
    for (auto ev : e->ev_d) cudaEventDestroy(ev);
    for (auto ev : e->ev_s) cudaEventDestroy(ev);
    for (auto ev : e->ev_pool) cudaEventDestroy(ev);
    delete e;
}

extern "C" int32_t st_encoder_num_sites(const st_encoder *e) { return e ? e->n_sites : 0; }

extern "C" st_status st_layer_shape(const st_encoder *e, int32_t layer, int32_t hwc[3]) {
    if (!e || !hwc || layer < -1 || layer >= (int)e->L.size()) return ST_ERR_ARG;
    if (layer < 0) { hwc[0] = e->in_H; hwc[1] = e->in_W; hwc[2] = e->in_C; }
    else { hwc[0] = e->L[layer].H; hwc[1] = e->L[layer].W; hwc[2] = e->L[layer].C; }
    return ST_OK;
}

// ------------------------------------------------------------ encode calls
extern "C" st_status st_encode_reference(st_encoder *e, const float *ref_dev, int32_t n_chunks, int64_t chunk_stride,
                                         void *stream) {
    if (!e) return ST_ERR_ARG;
    if (!ref_dev) return fail(e, ST_ERR_ARG, "ref_dev is null");
    if (n_chunks < 1 || n_chunks > e->B) return fail(e, ST_ERR_SHAPE, "n_chunks %d outside [1, %d]", n_chunks, e->B);
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t per = (int64_t)e->in_H * e->in_W * e->in_C;
    const int64_t stride = chunk_stride ? chunk_stride : per;
    if (stride < per) return fail(e, ST_ERR_ARG, "chunk_stride smaller than a frame");
    CUDA_OK(e, cudaSetDevice(e->cfg.device));
    CUDA_OK(e, cudaMemcpy2DAsync(e->ref, per * 4, ref_dev, stride * 4, per * 4, n_chunks, cudaMemcpyDeviceToDevice, s));
    e->staged_chunks = n_chunks;
    e->cont = false;
    e->par = 0;
    return ST_OK;
}

extern "C" st_status st_encode_reference_u8(st_encoder *e, const uint8_t *ref_dev, int32_t n_chunks,
                                            int64_t chunk_stride, void *stream) {
    if (!e) return ST_ERR_ARG;
    if (!ref_dev) return fail(e, ST_ERR_ARG, "ref_dev is null");
    if (n_chunks < 1 || n_chunks > e->B) return fail(e, ST_ERR_SHAPE, "n_chunks %d outside [1, %d]", n_chunks, e->B);
    const int64_t per = (int64_t)e->in_H * e->in_W * e->in_C;
    const int64_t stride = chunk_stride ? chunk_stride : per;
    if (stride < per) return fail(e, ST_ERR_ARG, "chunk_stride smaller than a frame");
    CUDA_OK(e, cudaSetDevice(e->cfg.device));
    launch_u8_to_f32(ref_dev, stride, per, n_chunks, e->ref, (cudaStream_t)stream);
    CUDA_OK(e, cudaGetLastError());
    e->staged_chunks = n_chunks;
    e->cont = false;
    e->par = 0;
    return ST_OK;
}

static int64_t rows_cap_of(const st_encoder *e, int t);
static DView view_of_(const st_encoder *e, int t);
static DView view_of(const st_encoder *e, int t) {
    DView v = view_of_(e, t);
    v.nrows = rows_cap_of(e, t) + 1;
    return v;
}
static DView view_of_(const st_encoder *e, int t) {
    DView v;
    if (t < 0) {
        v.act = e->p<uint32_t>(e->in_act);
        v.slot = v.act;
        v.pbase = e->p<int32_t>(e->in_pbase);
        v.rows = e->ptr(e->in_rows);
        return v;
    }
    const LayerRT &l = e->L[t];
    if (l.kind == ST_OUTPUT) return view_of(e, l.src);
    if (l.kind == ST_CONV && l.rowmap) {   // the input's frame words and row layout, own rows
        DView s = view_of(e, l.src);
        s.rows = e->ptr(l.b_rows);
        return s;
    }
    v.act = e->p<uint32_t>(l.b_act);
    if (l.kind == ST_RELU || l.kind == ST_SILU) {
        DView s = view_of(e, l.src);
        v.slot = s.slot;
        v.pbase = s.pbase;
        v.rows = l.b_rows >= 0 ? static_cast<const void *>(e->ptr(l.b_rows)) : s.rows;
        return v;
    }
    v.slot = l.b_slot >= 0 ? e->p<uint32_t>(l.b_slot) : v.act;
    v.pbase = e->p<int32_t>(l.b_pbase);
    v.rows = e->ptr(l.b_rows);
    return v;
}

static void *ybf_of(st_encoder *e, int t) { return e->L[t].b_ybf >= 0 ? e->ptr(e->L[t].b_ybf) : nullptr; }
// bf16 shadow of the dense tensor a layer reads (through OUTPUT taps), or null
static const void *dense_bf_of(st_encoder *e, int t) {
    while (t >= 0 && e->L[t].kind == ST_OUTPUT) t = e->L[t].src;
    return t >= 0 ? ybf_of(e, t) : nullptr;
}
static const float *dense_of(const st_encoder *e, int t) {
    if (t < 0) return e->ref;
    const LayerRT &l = e->L[t];
    if (l.kind == ST_OUTPUT) return dense_of(e, l.src);
    return e->p<float>(l.b_y0);
}

// A-operand TMA maps of the 1x1/s1 tensor-core convs for the current arena
static void encode_act_maps(st_encoder *e) {
    const char *nt = getenv("ST_NO_TMA_A");   // A/B switch
    const bool off = nt && nt[0] == '1';
    for (int i = 0; i < (int)e->L.size(); i++) {
        LayerRT &l = e->L[i];
        l.tma_ad = l.tma_as = false;
        if (off || l.kind != ST_CONV || !l.tc || l.src < 0 || l.spec.k_h != 1 || l.spec.k_w != 1 || l.spec.s_h != 1 ||
            l.spec.s_w != 1 || l.spec.p_h != 0 || l.spec.p_w != 0)
            continue;
        const int Cin = l.geo.Cin;
        const void *bfsrc = dense_bf_of(e, l.src);
        if (bfsrc) l.tma_ad = make_act_tmap(l.tmap_ad, bfsrc, (int64_t)e->B * l.geo.Hin * l.geo.Win, Cin);
        if (l.rowmap) {
            const char *rows = static_cast<const char *>(view_of(e, l.src).rows);
            if (rows) l.tma_as = make_act_tmap(l.tmap_as, rows + (size_t)Cin * e->esz, l.rows_cap, Cin);
        }
    }
}

static int64_t rows_cap_of(const st_encoder *e, int t) {
    if (t < 0) return e->in_rows_cap;
    const LayerRT &l = e->L[t];
    if (l.kind == ST_RELU || l.kind == ST_SILU || l.kind == ST_OUTPUT) return rows_cap_of(e, l.src);
    return l.rows_cap;
}

// Turn every kernel -> kernel edge of a captured step into a programmatic
// dependency (PDL): the dependent kernel is scheduled while its predecessor
// drains and blocks in griddepcontrol.wait (st_pdl_enter, the first statement
// of every kernel) until the predecessor completed and its writes are
// visible.  Edges touching memset / memcpy nodes stay full dependencies.  On
// any API failure the graph keeps its plain edges.
static void make_edges_programmatic(cudaGraph_t g) {
    size_t ne = 0;
    if (cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne) != cudaSuccess || ne == 0) {
        cudaGetLastError();
        return;
    }
    std::vector<cudaGraphNode_t> from(ne), to(ne);
    std::vector<cudaGraphEdgeData> ed(ne);
    if (cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    for (size_t i = 0; i < ne; i++) {
        cudaGraphNodeType tf, tt;
        if (cudaGraphNodeGetType(from[i], &tf) != cudaSuccess || cudaGraphNodeGetType(to[i], &tt) != cudaSuccess) break;
        if (tf != cudaGraphNodeTypeKernel || tt != cudaGraphNodeTypeKernel) continue;
        if (ed[i].type != cudaGraphDependencyTypeDefault) continue;
        cudaGraphEdgeData pe{};
        pe.from_port = cudaGraphKernelNodePortProgrammatic;
        pe.type = cudaGraphDependencyTypeProgrammatic;
        if (cudaGraphRemoveDependencies_v2(g, &from[i], &to[i], &ed[i], 1) != cudaSuccess) break;
        if (cudaGraphAddDependencies_v2(g, &from[i], &to[i], &pe, 1) != cudaSuccess) {
            cudaGraphAddDependencies_v2(g, &from[i], &to[i], &ed[i], 1);   // restore the plain edge
            break;
        }
    }
    cudaGetLastError();
}

// Enqueue one SparseBatch step on stream s (everything st_encode_diff does on
// the device).  Thresholds are read by the kernels from e->thr_dev, which the
// first node refreshes from the pinned host staging buffer, so the same
// captured graph serves every step.
static st_status issue_step(st_encoder *e, const void *frames_dev, bool u8, int F, int64_t fstride, cudaStream_t s);

static st_status encode_diff(st_encoder *e, const void *frames_dev, bool u8, int32_t n_diff, int64_t chunk_stride,
                             const float *thresholds, void *stream) {
    if (!e) return ST_ERR_ARG;
    if (!thresholds) return fail(e, ST_ERR_ARG, "thresholds is null");
    if (n_diff < 0 || n_diff > e->F) return fail(e, ST_ERR_SHAPE, "n_diff %d outside [0, %d]", n_diff, e->F);
    if (n_diff > 0 && !frames_dev) return fail(e, ST_ERR_ARG, "frames_dev is null");
    if (e->staged_chunks <= 0) return fail(e, ST_ERR_STATE, "st_encode_diff without st_encode_reference");
    for (int i = 0; i < e->n_sites; i++)
        if (!(thresholds[i] >= 0.0f)) return fail(e, ST_ERR_ARG, "threshold %d is negative or NaN", i);
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_OK(e, cudaSetDevice(e->cfg.device));
    const int64_t per = (int64_t)e->in_H * e->in_W * e->in_C;
    const int64_t fstride = chunk_stride ? chunk_stride : (int64_t)n_diff * per;
    // the previous step's threshold copy must have consumed the staging buffer
    if (e->thr_pending) CUDA_OK(e, cudaEventSynchronize(e->thr_ev));
    std::memcpy(e->thr_host, thresholds, sizeof(float) * e->n_sites);
    e->last_chunks = e->staged_chunks;
    e->last_ndiff = n_diff;
    e->last_stream = s;
    const bool graphs = e->use_graphs && !e->prof && !e->cfg.debug_retain;
    if (!graphs) {
        st_status r = issue_step(e, frames_dev, u8, n_diff, fstride, s);
        if (r) return r;
    } else {
        GraphKey key{frames_dev, fstride, n_diff, e->staged_chunks, e->cont ? 1 + e->par : 0, u8};
        GraphEnt *ent = nullptr;
        for (auto &g : e->graphs)
            if (g.key == key) ent = &g;
        if (!ent) {   // first sight: run eagerly (lazy kernel attributes get set), capture next time
            e->graphs.push_back(GraphEnt{key, nullptr, 0});
            st_status r = issue_step(e, frames_dev, u8, n_diff, fstride, s);
            if (r) return r;
        } else {
            // capture and replay on the encoder's own stream, forked from / joined
            // back to the caller's stream (the legacy default stream cannot be captured)
            cudaStream_t g_s = e->gstream;
            if (!ent->exec) {
                cudaGraph_t g = nullptr;
                CUDA_OK(e, cudaStreamBeginCapture(g_s, cudaStreamCaptureModeThreadLocal));
                st_status r = issue_step(e, frames_dev, u8, n_diff, fstride, g_s);
                cudaError_t ce = cudaStreamEndCapture(g_s, &g);
                if (r) return r;
                if (ce != cudaSuccess) return fail(e, ST_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ce));
                if (e->use_pdl) make_edges_programmatic(g);
                // node priorities from the capturing streams (dense / diff overlap)
                CUDA_OK(e, cudaGraphInstantiate(&ent->exec, g, e->ov_k > 0 ? cudaGraphInstantiateFlagUseNodePriority : 0));
                cudaGraphDestroy(g);
                ent->launches = e->launches;
            }
            CUDA_OK(e, cudaEventRecord(e->ev_fork, s));
            CUDA_OK(e, cudaStreamWaitEvent(g_s, e->ev_fork, 0));
            CUDA_OK(e, cudaGraphLaunch(ent->exec, g_s));
            CUDA_OK(e, cudaEventRecord(e->ev_join, g_s));
            CUDA_OK(e, cudaStreamWaitEvent(s, e->ev_join, 0));
            e->launches = ent->launches;
        }
    }
    CUDA_OK(e, cudaEventRecord(e->thr_ev, s));
    e->thr_pending = true;
    e->exp_valid = e->exp_chunk >= 0 && e->exp_chunk < e->staged_chunks && n_diff > 0;
    if (e->cfg.streaming) {   // the chunks continue from the saved state next call
        e->cont = true;
        e->par ^= 1;
    }
    CUDA_OK(e, cudaGetLastError());
    return ST_OK;
}

extern "C" st_status st_encode_diff(st_encoder *e, const float *frames_dev, int32_t n_diff, int64_t chunk_stride,
                                    const float *thresholds, void *stream) {
    return encode_diff(e, frames_dev, false, n_diff, chunk_stride, thresholds, stream);
}

extern "C" st_status st_encode_diff_u8(st_encoder *e, const uint8_t *frames_dev, int32_t n_diff, int64_t chunk_stride,
                                       const float *thresholds, void *stream) {
    return encode_diff(e, frames_dev, true, n_diff, chunk_stride, thresholds, stream);
}

// conv + site in the tcgen05 epilogue: the site's frame words start at zero
// (pixels without rows are never visited), emitted rows in place
static void tc_site_setup(st_encoder *e, const LayerRT &l, ConvCall &c, cudaStream_t s) {
    const LayerRT &r = e->L[l.tc_site];
    cudaMemsetAsync(e->ptr(r.b_act), 0, (size_t)e->staged_chunks * r.H * r.W * 4, s);
    c.site.on = true;
    c.site.x0 = e->p<float>(l.b_y0);
    c.site.theta = e->thr_dev + r.site;
    c.site.act = r.kind == ST_RELU ? ACT_RELU : ACT_SILU_FAST;
    c.site.words = e->p<uint32_t>(r.b_act);
    c.site.zero_gaps = r.zero_gaps;
}

static st_status issue_step(st_encoder *e, const void *frames_dev, bool u8, int F, int64_t fstride, cudaStream_t s) {
    const int B = e->staged_chunks, n = (int)e->L.size();
    const int64_t Nin = (int64_t)e->in_H * e->in_W;
    const int64_t per = Nin * e->in_C;
    e->launches = 0;
    if (e->prof) { e->recs.clear(); e->ev_used = 0; }
    CUDA_OK(e, cudaMemcpyAsync(e->thr_dev, e->thr_host, sizeof(float) * e->n_sites, cudaMemcpyHostToDevice, s));
    const float *thresholds = e->thr_dev;   // device copy, one fp32 per site
    CUDA_OK(e, cudaMemsetAsync(e->counts, 0, (size_t)e->B * e->n_sites * 32 * 8, s));
    CUDA_OK(e, cudaMemsetAsync(e->stats, 0, (size_t)(n + 1) * 3 * 8, s));
    CUDA_OK(e, cudaMemsetAsync(e->site_sum, 0, (size_t)e->n_sites * 8, s));
    CUDA_OK(e, cudaMemsetAsync(e->ovf, 0, 4, s));
    auto capv = [&](int idx, int64_t cap) {   // row capacity check of one scanned tensor (a9)
        ScanCap c;
        c.cap = cap;
        c.ovf = e->ovf;
        c.peak = e->rows_peak + idx;
        return c;
    };
    const int64_t cstride = (int64_t)e->n_sites * 32;
    auto zero_row = [&](int buf, int C) {
        if (buf >= 0) cudaMemsetAsync(e->ptr(buf), 0, (size_t)C * e->esz, s);
    };
    const bool bf = e->bf;
    // streaming (N1): on a continuation the dense reference pass is skipped and
    // every site starts from its saved state; par selects the ping-pong halves
    const bool strm = e->cfg.streaming != 0, cont = strm && e->cont;
    const int par = e->par;
    auto fcopy = [&](int dst_buf, const float *src, int64_t n_floats) {
        cudaMemcpyAsync(e->ptr(dst_buf), src, (size_t)n_floats * 4, cudaMemcpyDeviceToDevice, s);
    };
    const float *S0 = cont ? e->p<float>(e->in_S) : e->ref;   // Subtraction buffer at call start
    if (strm && !cont) fcopy(e->in_S, e->ref, B * per);
    // dense / diff overlap: dense ops on sD, diff ops on s; the diff
    // ops of layer i wait for its dense op, the dense op of layer i for the
    // diff ops of layer i - ov_k (the arena's lifetimes assume that bound)
    // (profiled passes run on one stream: their per-launch event times are the
    // kernels' own, not the overlap's; the arena's lifetimes hold either way)
    const bool ov = e->ov_k > 0 && !strm && F > 0 && !e->prof;
    cudaStream_t sD = ov ? e->dstream : s;
    if (ov) {
        CUDA_OK(e, cudaEventRecord(e->ev_dfork, s));
        CUDA_OK(e, cudaStreamWaitEvent(sD, e->ev_dfork, 0));
    }
    auto dense_done = [&](int i) {
        if (!ov) return;
        cudaEventRecord(e->ev_d[i], sD);
        cudaStreamWaitEvent(s, e->ev_d[i], 0);
    };

    // ---------------- input site: Subtraction + truncation + compaction (a2)
    if (F > 0) {
        uint32_t *act = e->p<uint32_t>(e->in_act);
        int32_t *pb = e->p<int32_t>(e->in_pbase);
        void *rows = e->ptr(e->in_rows);
        const void *fr = frames_dev;
        LAUNCH(e, KC_SUBTRACT, -1, s,
               launch_subtract_mask(S0, per, fr, u8, fstride, B, (int)Nin, e->in_C, F, thresholds, bf, act,
                                    e->in_dd >= 0 ? e->ptr(e->in_dd) : nullptr, s));
        LAUNCH(e, KC_SCAN, -1, s,
               launch_scan_popc(act, B * Nin, pb, e->totals + n, e->scan_tmp, e->stats + 3 * n + 1, s, nullptr,
                                capv(n, e->in_rows_cap)));
        zero_row(e->in_rows, e->in_C);
        LAUNCH(e, KC_SUBTRACT, -1, s,
               launch_subtract_rows(S0, per, fr, u8, fstride, B, (int)Nin, e->in_C, act, pb, rows, bf,
                                    strm ? e->p<float>(e->in_S) : nullptr, s));
        LAUNCH(e, KC_COUNTS, -1, s,
               launch_frame_counts(act, B, (int)Nin, e->counts, cstride, e->site_sum, nullptr, s));
    }
    // mask export (st_debug_export_chunk): the chunk's words of a layer boundary
    const bool exporting = e->exp_chunk >= 0 && e->exp_chunk < B && F > 0;
    auto export_words = [&](int layer) {
        if (!exporting) return;
        const int64_t Nl = layer < 0 ? Nin : (int64_t)e->L[layer].H * e->L[layer].W;
        const uint32_t *src = view_of(e, layer).act;
        cudaMemcpyAsync(e->exp_words + e->exp_off[layer + 1], src + (int64_t)e->exp_chunk * Nl, Nl * 4,
                        cudaMemcpyDeviceToDevice, s);
    };
    export_words(-1);

    if (e->in_refbf >= 0 && !cont)
        LAUNCH(e, KC_DENSE_MISC, -1, sD, launch_pad4_bf16(e->ref, (int64_t)B * Nin, e->in_C, e->ptr(e->in_refbf), sD));
    // ---------------- layers in topological order, dense then diff ("N")
    for (int i = 0; i < n; i++) {
        LayerRT &l = e->L[i];
        const int64_t N = (int64_t)l.H * l.W;
        const int64_t Ns = l.src < 0 ? Nin : (int64_t)e->L[l.src].H * e->L[l.src].W;
        const int Cs = l.src < 0 ? e->in_C : e->L[l.src].C;
        const float *x_src = dense_of(e, l.src);
        long long *st = e->stats + 3 * i;
        DView in = F > 0 ? view_of(e, l.src) : DView{};
        if (ov && i >= e->ov_k) cudaStreamWaitEvent(sD, e->ev_s[i - e->ov_k], 0);
        // rows_in / touched of this layer: roofline accounting only, collected
        // when profiling is on (st_set_profiling) so the timed step skips them
        if (F > 0 && l.kind != ST_OUTPUT && e->prof && l.fused_relu < 0)
            LAUNCH(e, KC_PROF_STATS, i, s, launch_frame_counts(in.act, B, (int)Ns, nullptr, 0, st, st + 2, s));
        switch (l.kind) {
        case ST_CONV: {
            ConvCall c{};
            c.g = l.geo;
            c.B = B;
            c.dense = true;
            c.a_dense = x_src;
            c.zeros = e->zeros;
            c.a_dense_bf = l.tc ? dense_bf_of(e, l.src) : l.tc_small ? e->ptr(e->in_refbf) : nullptr;
            if (l.tc_small) conv_tc_small_layout(l.geo, c.sr, c.shift);
            c.wk = l.wk;
            c.bias = l.bias;
            c.rnd_a = bf;   // BF16 mode: the dense A operand is bf16-rounded (R22-BF16)
            c.out = e->p<float>(l.b_y0);
            if (l.dw_site >= 0 || l.act_site >= 0) {   // the site's dense output from the same epilogue
                const int si = l.dw_site >= 0 ? l.dw_site : l.act_site;
                const LayerRT &r = e->L[si];
                c.act_out = e->p<float>(r.b_y0);
                c.act_bf = ybf_of(e, si);
                c.act_kind = r.kind == ST_RELU ? ACT_RELU : bf ? ACT_SILU_FAST : ACT_SILU;
            }
            if (!cont)
                LAUNCH(e, l.depthwise ? KC_DW_DENSE : l.tc ? KC_TC_DENSE : l.tc_small ? KC_STEM_DENSE : KC_CONV_DENSE, i, sD,
                       l.depthwise  ? launch_dwconv_f32(c, sD)
                       : l.tc       ? (c.tma_a = l.tma_ad, launch_conv_tc(c, l.tmap, sD, l.tma_ad ? l.tmap_ad : nullptr))
                       : l.tc_small ? launch_conv_tc_small(c, l.tmap, sD)
                                    : launch_conv_f32(c, sD));
            c.tma_a = false;
            if (l.b_ybf >= 0 && !cont)
                LAUNCH(e, KC_DENSE_MISC, i, sD, launch_to_bf16(e->p<float>(l.b_y0), ybf_of(e, i), (int64_t)B * N * l.C, sD));
            dense_done(i);
            if (F == 0) break;
            if (l.rowmap) {   // 1x1/s1: a plain GEMM over the rows of the input's layout
                zero_row(l.b_rows, l.C);
                c.dense = false;
                c.rnd_a = false;
                c.bf = bf;
                c.a = in;
                c.rowmap = true;
                c.ridx = nullptr;
                c.F = F;
                c.ddelta = nullptr;
                c.m_dev = e->totals + layout_owner(e, l.src);
                c.m_cap = l.rows_cap;
                c.out = e->ptr(l.b_rows);
                c.act_out = nullptr;
                c.act_bf = nullptr;
                c.tma_a = l.tma_as;
                if (l.tc_site >= 0) {   // the site in the epilogue: row codes of the layout's slots
                    const int o = layout_owner(e, l.src);
                    const uint32_t *sw = o == n ? e->p<uint32_t>(e->in_act) : e->p<uint32_t>(e->L[o].b_slot >= 0 ? e->L[o].b_slot : e->L[o].b_act);
                    const int32_t *pw = o == n ? e->p<int32_t>(e->in_pbase) : e->p<int32_t>(e->L[o].b_pbase);
                    const int64_t Nn = o == n ? Nin : (int64_t)e->L[o].H * e->L[o].W;
                    LAUNCH(e, KC_ENUM, i, s, launch_enumerate(sw, pw, B * Nn, e->p<int32_t>(l.b_ridx), s));
                    c.ridx = e->p<int32_t>(l.b_ridx);
                    tc_site_setup(e, l, c, s);
                }
                LAUNCH(e, l.tc ? KC_TC_SPARSE : KC_CONV_SPARSE, i, s,
                       l.tc ? launch_conv_tc(c, l.tc_site >= 0 ? l.tmap_site : l.tmap, s, l.tma_as ? l.tmap_as : nullptr)
                            : launch_conv_f32(c, s));
                if (l.tc_site >= 0) LAUNCH(e, KC_TC_SITE_FIX, l.tc_site, s, launch_tc_site_fixup(c, in, s));
                c.tma_a = false;
                c.site.on = false;
                break;
            }
            uint32_t *act = e->p<uint32_t>(l.b_act);
            int32_t *pb = e->p<int32_t>(l.b_pbase);
            LAUNCH(e, KC_DILATE, i, s, launch_dilate(in.act, B, l.geo, act, s));
            const bool dw_pm = l.depthwise && !e->dw_rowmajor;   // pixel-major depthwise needs no M-row list
            // scan of the output frame words; the M-row list is enumerated in the same pass
            LAUNCH(e, KC_SCAN, i, s,
                   launch_scan_popc(act, B * N, pb, e->totals + i, e->scan_tmp, st + 1, s,
                                    dw_pm ? nullptr : e->p<int32_t>(l.b_ridx), capv(i, l.rows_cap)));
            zero_row(l.b_rows, l.C);
            c.dense = false;
            c.rnd_a = false;   // delta rows are already bf16 values in BF16 mode
            c.bf = bf;
            c.a = in;
            c.ridx = e->p<int32_t>(l.b_ridx);
            c.F = F;
            c.ddelta = (l.src == -1 && !l.depthwise && !l.tc && e->in_dd >= 0) ? e->ptr(e->in_dd) : nullptr;
            c.m_dev = e->totals + i;
            c.m_cap = l.rows_cap;
            c.out = e->ptr(l.b_rows);
            c.act_out = nullptr;
            c.act_bf = nullptr;
            if (l.dw_site >= 0) {   // depthwise conv + its site in one pass (N2)
                const LayerRT &r = e->L[l.dw_site];
                DwSite d;
                d.out_act = act;
                d.out_pbase = pb;
                d.x0 = e->p<float>(l.b_y0);
                d.theta = thresholds + r.site;
                d.act = r.kind == ST_RELU ? ACT_RELU : ACT_SILU;
                d.site_act = e->p<uint32_t>(r.b_act);
                d.site_rows = const_cast<void *>(view_of(e, l.dw_site).rows);
                d.conv_rows = r.b_rows >= 0 ? e->ptr(l.b_rows) : nullptr;   // own site rows: keep the conv's too
                d.zero_gaps = r.zero_gaps;
                d.site_nrows = std::min(view_of(e, l.dw_site).nrows, l.rows_cap + 1);
                LAUNCH(e, KC_DW_SITE, i, s, launch_dwconv_site(c, d, s));
                break;
            }
            if (l.tc_site >= 0) tc_site_setup(e, l, c, s);
            LAUNCH(e, l.depthwise ? KC_DW_SPARSE : l.tc ? KC_TC_SPARSE : l.tc_small ? KC_STEM_SPARSE : KC_CONV_SPARSE, i, s,
                   dw_pm        ? launch_dwconv_pm(c, act, pb, s)
                   : l.depthwise ? launch_dwconv_f32(c, s)
                   : l.tc       ? launch_conv_tc(c, l.tc_site >= 0 ? l.tmap_site : l.tmap, s)
                   : l.tc_small ? launch_conv_tc_small(c, l.tmap, s)
                                : launch_conv_f32(c, s));
            if (l.tc_site >= 0) {
                DView cv;
                cv.act = act;
                cv.slot = act;
                cv.pbase = pb;
                LAUNCH(e, KC_TC_SITE_FIX, l.tc_site, s, launch_tc_site_fixup(c, cv, s));
            }
            c.site.on = false;
            break;
        }
        case ST_RELU: case ST_SILU: {
            const int act_kind = l.kind == ST_RELU ? ACT_RELU : ACT_SILU;
            // the dense reference activation uses the same SiLU form as the site (fast in BF16 mode)
            const int dense_kind = (act_kind == ACT_SILU && bf) ? ACT_SILU_FAST : act_kind;
            // a fused ReLU's dense output is read only by the pool's dense pass,
            // which applies the ReLU itself (kept when streaming or debugging)
            const bool skip_dense = (l.fused_pool >= 0 && !strm && !e->cfg.debug_retain) || l.fused_dw >= 0 ||
                                    l.act_of >= 0;
            if (!cont && !skip_dense)
                LAUNCH(e, KC_DENSE_MISC, i, sD,
                       launch_dense_act(x_src, e->p<float>(l.b_y0), (int64_t)B * N * l.C, dense_kind, ybf_of(e, i), sD));
            dense_done(i);
            SiteState sst;
            const float *x_init = x_src;
            if (strm && l.sx[0] >= 0) {   // in-place state; first call: from the dense reference pass
                if (!cont) {
                    fcopy(l.sx[0], x_src, B * N * l.C);
                    fcopy(l.sy[0], e->p<float>(l.b_y0), B * N * l.C);
                }
                x_init = e->p<float>(l.sx[0]);
                sst.y_init = e->p<float>(l.sy[0]);
                sst.x_save = e->p<float>(l.sx[0]);
                sst.y_save = e->p<float>(l.sy[0]);
            }
            if (F == 0) break;
            DView me = view_of(e, i);
            if (l.b_rows >= 0) zero_row(l.b_rows, l.C);   // own buffer (not in place)
            if (l.fused_pool >= 0) break;                 // runs inside the pool's pass
            if (l.fused_dw < 0 && l.fused_tc < 0)         // else: ran inside the conv's pass
                LAUNCH(e, KC_SITE_PW, i, s,
                   launch_site_pointwise(in, x_init, B, (int)N, l.C, act_kind, thresholds + l.site, bf,
                                         e->p<uint32_t>(l.b_act), const_cast<void *>(me.rows), sst, s, l.zero_gaps));
            LAUNCH(e, KC_COUNTS, i, s,
                   launch_frame_counts(e->p<uint32_t>(l.b_act), B, (int)N, e->counts + l.site * 32, cstride,
                                       e->site_sum + l.site, nullptr, s));
            break;
        }
        case ST_MAXPOOL: {
            if (!cont) {
                const bool relu_in = l.fused_relu >= 0 && !strm && !e->cfg.debug_retain;
                LAUNCH(e, KC_DENSE_MISC, i, sD,
                       launch_dense_maxpool(relu_in ? dense_of(e, e->L[l.fused_relu].src) : x_src,
                                            e->p<float>(l.b_y0), B, l.geo, ybf_of(e, i), sD, relu_in));
            }
            dense_done(i);
            // streaming state: x_acc of the input pixels ping-pongs (windows of
            // neighbouring tiles share pixels), y_acc of the outputs in place
            SiteState sst;
            const float *x_init = x_src;
            const int64_t NiC = Ns * Cs;
            if (strm) {
                if (!cont) fcopy(l.spy, e->p<float>(l.b_y0), B * N * l.C);
                sst.y_init = e->p<float>(l.spy);
                sst.y_save = e->p<float>(l.spy);
                if (l.fused_relu >= 0) {
                    const LayerRT &r = e->L[l.fused_relu];
                    x_init = cont ? e->p<float>(l.sx[par]) : dense_of(e, r.src);
                    sst.ry_init = cont ? e->p<float>(l.sy[par]) : e->p<float>(r.b_y0);
                    sst.rx_save = e->p<float>(l.sx[par ^ 1]);
                    sst.ry_save = e->p<float>(l.sy[par ^ 1]);
                    if (F == 0) {   // the pass writes every footprint pixel; without it, carry over
                        fcopy(l.sx[par ^ 1], x_init, B * NiC);
                        fcopy(l.sy[par ^ 1], sst.ry_init, B * NiC);
                    }
                } else {
                    x_init = cont ? e->p<float>(l.sx[par]) : x_src;
                    fcopy(l.sx[par ^ 1], x_init, B * NiC);   // the kernels save changed pixels only
                    sst.x_save = e->p<float>(l.sx[par ^ 1]);
                }
            }
            if (F == 0) break;
            uint32_t *slot = e->p<uint32_t>(l.b_slot);
            int32_t *pb = e->p<int32_t>(l.b_pbase);
            if (l.fused_relu >= 0) {
                // ReLU site + pool in one pass; the pool's row capacity is the
                // dilation of the conv mask (superset of the ReLU's emitted mask)
                const LayerRT &r = e->L[l.fused_relu];
                const DView cv = view_of(e, r.src);
                LAUNCH(e, KC_DILATE, i, s, launch_dilate(cv.act, B, l.geo, slot, s));
                LAUNCH(e, KC_SCAN, i, s, launch_scan_popc(slot, B * N, pb, e->totals + i, e->scan_tmp, nullptr, s, nullptr, capv(i, l.rows_cap)));
                zero_row(l.b_rows, l.C);
                LAUNCH(e, KC_SITE_MP, i, s,
                       launch_site_relu_maxpool(cv, strm ? x_init : dense_of(e, r.src), B, l.geo, thresholds + r.site,
                                                thresholds + l.site, bf, slot, pb, e->p<uint32_t>(r.b_act),
                                                r.b_rows >= 0 ? e->ptr(r.b_rows) : nullptr,
                                                e->p<uint32_t>(l.b_act), e->ptr(l.b_rows), sst, s));
                LAUNCH(e, KC_COUNTS, l.fused_relu, s,
                       launch_frame_counts(e->p<uint32_t>(r.b_act), B, (int)Ns, e->counts + r.site * 32, cstride,
                                           e->site_sum + r.site, nullptr, s));
                LAUNCH(e, KC_COUNTS, i, s,
                       launch_frame_counts(e->p<uint32_t>(l.b_act), B, (int)N, e->counts + l.site * 32, cstride,
                                           e->site_sum + l.site, nullptr, s));
                if (e->prof)
                    LAUNCH(e, KC_PROF_STATS, i, s, launch_frame_counts(in.act, B, (int)Ns, nullptr, 0, st, st + 2, s));
                break;
            }
            LAUNCH(e, KC_DILATE, i, s, launch_dilate(in.act, B, l.geo, slot, s));
            LAUNCH(e, KC_SCAN, i, s, launch_scan_popc(slot, B * N, pb, e->totals + i, e->scan_tmp, nullptr, s, nullptr, capv(i, l.rows_cap)));
            zero_row(l.b_rows, l.C);
            LAUNCH(e, KC_SITE_MP, i, s,
                   launch_site_maxpool(in, x_init, B, l.geo, thresholds + l.site, bf, slot, pb,
                                       e->p<uint32_t>(l.b_act), e->ptr(l.b_rows), sst, s));
            LAUNCH(e, KC_COUNTS, i, s,
                   launch_frame_counts(e->p<uint32_t>(l.b_act), B, (int)N, e->counts + l.site * 32, cstride,
                                       e->site_sum + l.site, nullptr, s));
            break;
        }
        case ST_ADD: {
            const float *x2 = dense_of(e, l.src2);
            if (!cont)
                LAUNCH(e, KC_DENSE_MISC, i, sD,
                       launch_dense_add(x_src, x2, e->p<float>(l.b_y0), (int64_t)B * N * l.C, ybf_of(e, i), sD));
            dense_done(i);
            if (F == 0) break;
            DView in2 = view_of(e, l.src2);
            uint32_t *slot = e->p<uint32_t>(l.b_slot);
            int32_t *pb = e->p<int32_t>(l.b_pbase);
            LAUNCH(e, KC_ADD, i, s, launch_or_words(in.act, in2.act, B * N, slot, s));
            LAUNCH(e, KC_SCAN, i, s, launch_scan_popc(slot, B * N, pb, e->totals + i, e->scan_tmp, nullptr, s, nullptr, capv(i, l.rows_cap)));
            zero_row(l.b_rows, l.C);
            LAUNCH(e, KC_ADD, i, s, launch_add_rows(in, in2, slot, pb, B, (int)N, l.C, bf, e->ptr(l.b_rows), s));
            CUDA_OK(e, cudaMemcpyAsync(e->p<uint32_t>(l.b_act), slot, (size_t)B * N * 4, cudaMemcpyDeviceToDevice, s));
            break;
        }
        case ST_SE: {
            // reading R8: sums of x0 and of every frame's delta rows -> sequential
            // gate schedule per chunk -> dense apply + pixel loop
            char *sb = e->ptr(l.b_se);
            double *sum0 = reinterpret_cast<double *>(sb);
            double *dsum = sum0 + (int64_t)B * l.C;
            float *s_tab = reinterpret_cast<float *>(dsum + (int64_t)B * F * l.C);
            uint32_t *refresh = reinterpret_cast<uint32_t *>(s_tab + (int64_t)B * (F + 1) * l.C);
            float *gate_tab = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(refresh + B) + 63) & ~uintptr_t(63));
            const int H = l.spec.se_hidden;
            // dense part: the reference gates (frame 0) depend on sum0 alone; the
            // dense apply reads gate_tab row 0 (= s_tab row 0, same layout)
            LAUNCH(e, KC_SE_SUMS, i, sD, launch_se_colsum(x_src, B, (int)N, l.C, sum0, sD));
            LAUNCH(e, KC_SE_SUMS, i, sD,
                   launch_se_gates(sum0, dsum, B, (int)N, l.C, H, F, l.se_w1, l.se_b1, l.se_w2, l.se_b2, 0, 1,
                                   gate_tab, sD));
            LAUNCH(e, KC_SE_SUMS, i, sD,
                   launch_se_dense_apply(x_src, gate_tab, B, (int)N, l.C, F, e->p<float>(l.b_y0), ybf_of(e, i), sD));
            dense_done(i);
            if (F == 0) break;
            LAUNCH(e, KC_SE_SUMS, i, s, launch_se_delta_sums(in, B, (int)N, l.C, F, bf, dsum, s));
            LAUNCH(e, KC_SE_SUMS, i, s,
                   launch_se_gates(sum0, dsum, B, (int)N, l.C, H, F, l.se_w1, l.se_b1, l.se_w2, l.se_b2, 1, F,
                                   gate_tab, s));
            LAUNCH(e, KC_SE_SUMS, i, s, launch_se_sched(gate_tab, B, l.C, F, thresholds + l.site, s_tab, refresh, s));
            uint32_t *slot = e->p<uint32_t>(l.b_slot);
            int32_t *pb = e->p<int32_t>(l.b_pbase);
            LAUNCH(e, KC_SE_SUMS, i, s, launch_se_slots(in.act, refresh, B, (int)N, slot, s));
            LAUNCH(e, KC_SCAN, i, s, launch_scan_popc(slot, B * N, pb, e->totals + i, e->scan_tmp, nullptr, s, nullptr, capv(i, l.rows_cap)));
            zero_row(l.b_rows, l.C);
            LAUNCH(e, KC_SE, i, s,
                   launch_se_site(in, x_src, s_tab, B, (int)N, l.C, F, thresholds + l.site, bf, slot, pb,
                                  e->p<uint32_t>(l.b_act), e->ptr(l.b_rows), s, l.zero_gaps));
            LAUNCH(e, KC_COUNTS, i, s,
                   launch_frame_counts(e->p<uint32_t>(l.b_act), B, (int)N, e->counts + l.site * 32, cstride,
                                       e->site_sum + l.site, nullptr, s));
            break;
        }
        case ST_OUTPUT: {
            dense_done(i);
            DView v = F > 0 ? in : DView{};
            float *o_state = strm ? e->p<float>(l.sx[0]) : nullptr;   // last output = next call's frame 0
            LAUNCH(e, KC_ACCUM, i, s,
                   launch_accumulate(v, cont ? o_state : x_src, B, (int)N, l.C, F, bf, e->p<float>(l.b_out), o_state,
                                     s));
            break;
        }
        default:
            return fail(e, ST_ERR_INTERNAL, "layer kind %d not executable", l.kind);
        }
        // a fused ReLU's words are written by its pool's pass
        if (l.kind != ST_OUTPUT && l.fused_pool < 0) export_words(i);
        if (l.fused_relu >= 0) export_words(l.fused_relu);
        if (ov) cudaEventRecord(e->ev_s[i], s);
        (void)Cs;
    }
    if (ov) {   // join the dense stream back
        CUDA_OK(e, cudaEventRecord(e->ev_djoin, sD));
        CUDA_OK(e, cudaStreamWaitEvent(s, e->ev_djoin, 0));
    }
    CUDA_OK(e, cudaGetLastError());
    return ST_OK;
}

// ------------------------------------------------------------- statistics
extern "C" st_status st_get_sparsity(st_encoder *e, int64_t *active, int64_t *site_active, int64_t *site_pixels) {
    if (!e) return ST_ERR_ARG;
    if (e->last_ndiff < 0) return fail(e, ST_ERR_STATE, "no encode_diff yet");
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    const int B = e->last_chunks, F = e->last_ndiff, S = e->n_sites;
    int32_t ov = 0;
    CUDA_OK(e, cudaMemcpy(&ov, e->ovf, 4, cudaMemcpyDeviceToHost));
    if (ov) return fail(e, ST_ERR_CAPACITY, "the last step exceeded a row capacity; its statistics are invalid");
    if (active) {
        std::vector<long long> h((size_t)e->B * S * 32);
        CUDA_OK(e, cudaMemcpy(h.data(), e->counts, h.size() * 8, cudaMemcpyDeviceToHost));
        for (int b = 0; b < B; b++)
            for (int si = 0; si < S; si++)
                for (int t = 0; t < F; t++) active[((int64_t)b * S + si) * F + t] = h[((size_t)b * S + si) * 32 + t];
    }
    if (site_active) {
        std::vector<long long> h(S);
        CUDA_OK(e, cudaMemcpy(h.data(), e->site_sum, S * 8, cudaMemcpyDeviceToHost));
        for (int si = 0; si < S; si++) site_active[si] = h[si];
    }
    if (site_pixels) {
        site_pixels[0] = (int64_t)B * F * e->in_H * e->in_W;
        for (auto &l : e->L)
            if (l.site) site_pixels[l.site] = (int64_t)B * F * l.H * l.W;
    }
    return ST_OK;
}

extern "C" st_status st_copy_site_counts(st_encoder *e, int64_t *dst_dev, void *stream) {
    if (!e || !dst_dev) return ST_ERR_ARG;
    if (e->last_ndiff < 0) return fail(e, ST_ERR_STATE, "no encode_diff yet");
    cudaStream_t s = (cudaStream_t)stream;
    const int S = e->n_sites;
    CUDA_OK(e, cudaMemcpyAsync(dst_dev, e->site_sum, S * 8, cudaMemcpyDeviceToDevice, s));
    std::vector<long long> pix(S);
    pix[0] = (long long)e->last_chunks * e->last_ndiff * e->in_H * e->in_W;
    for (auto &l : e->L)
        if (l.site) pix[l.site] = (long long)e->last_chunks * e->last_ndiff * l.H * l.W;
    // pixel counts are host-known constants: small H2D copy (pageable -> staged by the driver)
    CUDA_OK(e, cudaMemcpyAsync(dst_dev + S, pix.data(), S * 8, cudaMemcpyHostToDevice, s));
    CUDA_OK(e, cudaStreamSynchronize(s));
    return ST_OK;
}

extern "C" st_status st_get_layer_counts(st_encoder *e, int64_t *rows_in, int64_t *rows_out, int64_t *touched) {
    if (!e) return ST_ERR_ARG;
    if (e->last_ndiff < 0) return fail(e, ST_ERR_STATE, "no encode_diff yet");
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    const int n = (int)e->L.size();
    std::vector<long long> h((size_t)(n + 1) * 3);
    CUDA_OK(e, cudaMemcpy(h.data(), e->stats, h.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<int32_t> tot(n + 1);
    CUDA_OK(e, cudaMemcpy(tot.data(), e->totals, tot.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<long long> ss(e->n_sites);
    CUDA_OK(e, cudaMemcpy(ss.data(), e->site_sum, ss.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; i++) {
        const LayerRT &l = e->L[i];
        int64_t out = 0;
        if (l.kind == ST_CONV) out = l.rowmap ? (int64_t)h[3 * i] : (int64_t)tot[i];   // rowmap: the input's rows
        else if (is_site(l.kind)) out = ss[l.site];
        else if (l.kind == ST_ADD) out = tot[i];
        if (rows_in) rows_in[i] = h[3 * i];
        if (rows_out) rows_out[i] = out;
        if (touched) touched[i] = h[3 * i + 2];
    }
    return ST_OK;
}

extern "C" st_status st_get_output(st_encoder *e, int32_t tap, int32_t chunk, int32_t frame, const float **dev_ptr,
                                   int32_t hwc[3]) {
    if (!e || !dev_ptr) return ST_ERR_ARG;
    if (tap < 0 || tap >= (int)e->L.size() || e->L[tap].kind != ST_OUTPUT)
        return fail(e, ST_ERR_ARG, "layer %d is not an OUTPUT tap", tap);
    if (e->last_ndiff < 0) return fail(e, ST_ERR_STATE, "no encode yet");
    if (chunk < 0 || chunk >= e->last_chunks || frame < 0 || frame > e->last_ndiff)
        return fail(e, ST_ERR_ARG, "chunk/frame out of range");
    const LayerRT &l = e->L[tap];
    const int64_t fs = (int64_t)l.H * l.W * l.C;
    *dev_ptr = e->p<float>(l.b_out) + ((int64_t)chunk * (e->last_ndiff + 1) + frame) * fs;
    if (hwc) { hwc[0] = l.H; hwc[1] = l.W; hwc[2] = l.C; }
    return ST_OK;
}

// ------------------------------------------------------------------ debug
static st_status debug_words(st_encoder *e, int layer, int chunk, int frame, std::vector<uint32_t> &act,
                             std::vector<uint32_t> &slot, std::vector<int32_t> &pbase, int &H, int &W, int &C,
                             DView &v) {
    if (!e->cfg.debug_retain) return fail(e, ST_ERR_STATE, "debug getters need debug_retain");
    if (e->last_ndiff < 1) return fail(e, ST_ERR_STATE, "no diff frames encoded");
    if (layer < -1 || layer >= (int)e->L.size()) return fail(e, ST_ERR_ARG, "bad layer");
    if (chunk < 0 || chunk >= e->last_chunks || frame < 1 || frame > e->last_ndiff)
        return fail(e, ST_ERR_ARG, "chunk/frame out of range");
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    if (layer < 0) { H = e->in_H; W = e->in_W; C = e->in_C; }
    else { H = e->L[layer].H; W = e->L[layer].W; C = e->L[layer].C; }
    v = view_of(e, layer);
    const int64_t N = (int64_t)H * W;
    act.resize(N); slot.resize(N); pbase.resize(N);
    CUDA_OK(e, cudaMemcpy(act.data(), v.act + chunk * N, N * 4, cudaMemcpyDeviceToHost));
    CUDA_OK(e, cudaMemcpy(slot.data(), v.slot + chunk * N, N * 4, cudaMemcpyDeviceToHost));
    CUDA_OK(e, cudaMemcpy(pbase.data(), v.pbase + chunk * N, N * 4, cudaMemcpyDeviceToHost));
    return ST_OK;
}

extern "C" st_status st_debug_get_mask(st_encoder *e, int32_t layer, int32_t chunk, int32_t frame, uint32_t *words) {
    if (!e || !words) return ST_ERR_ARG;
    std::vector<uint32_t> act, slot;
    std::vector<int32_t> pb;
    int H, W, C;
    DView v;
    st_status r = debug_words(e, layer, chunk, frame, act, slot, pb, H, W, C, v);
    if (r) return r;
    const int64_t N = (int64_t)H * W;
    for (int64_t j = 0; j < (N + 31) / 32; j++) words[j] = 0;
    for (int64_t p = 0; p < N; p++)
        if ((act[p] >> (frame - 1)) & 1u) words[p / 32] |= 1u << (p % 32);
    return ST_OK;
}

extern "C" st_status st_debug_get_rows(st_encoder *e, int32_t layer, int32_t chunk, int32_t frame, int32_t *idx,
                                       float *rows, int64_t *n_out) {
    if (!e) return ST_ERR_ARG;
    std::vector<uint32_t> act, slot;
    std::vector<int32_t> pb;
    int H, W, C;
    DView v;
    st_status r = debug_words(e, layer, chunk, frame, act, slot, pb, H, W, C, v);
    if (r) return r;
    const int64_t N = (int64_t)H * W;
    const int t1 = frame - 1;
    int64_t k = 0;
    for (int64_t p = 0; p < N; p++) {
        if (!((act[p] >> t1) & 1u)) continue;
        if (idx) idx[k] = (int32_t)p;
        if (rows) {
            const int64_t row = 1 + pb[p] + __builtin_popcount(slot[p] & ((1u << t1) - 1u));
            const char *src = static_cast<const char *>(v.rows) + row * C * e->esz;
            if (e->esz == 4) {
                CUDA_OK(e, cudaMemcpy(rows + k * C, src, C * 4, cudaMemcpyDeviceToHost));
            } else {   // bf16 -> fp32 (exact)
                std::vector<uint16_t> hb(C);
                CUDA_OK(e, cudaMemcpy(hb.data(), src, C * 2, cudaMemcpyDeviceToHost));
                for (int ch = 0; ch < C; ch++) {
                    const uint32_t u = (uint32_t)hb[ch] << 16;
                    std::memcpy(rows + k * C + ch, &u, 4);
                }
            }
        }
        k++;
    }
    if (n_out) *n_out = k;
    return ST_OK;
}

extern "C" st_status st_debug_get_dense0(st_encoder *e, int32_t layer, int32_t chunk, float *host) {
    if (!e || !host) return ST_ERR_ARG;
    if (!e->cfg.debug_retain) return fail(e, ST_ERR_STATE, "debug getters need debug_retain");
    if (layer < 0 || layer >= (int)e->L.size() || chunk < 0 || chunk >= e->last_chunks)
        return fail(e, ST_ERR_ARG, "bad layer/chunk");
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    const LayerRT &l = e->L[layer];
    const int64_t ne = (int64_t)l.H * l.W * l.C;
    CUDA_OK(e, cudaMemcpy(host, dense_of(e, layer) + chunk * ne, ne * 4, cudaMemcpyDeviceToHost));
    return ST_OK;
}

extern "C" st_status st_debug_export_chunk(st_encoder *e, int32_t chunk) {
    if (!e) return ST_ERR_ARG;
    if (chunk < -1 || chunk >= e->B) return fail(e, ST_ERR_ARG, "export chunk %d outside [-1, %d)", chunk, e->B);
    CUDA_OK(e, cudaSetDevice(e->cfg.device));
    if (chunk >= 0 && !e->exp_words) {
        const int n = (int)e->L.size();
        e->exp_off.assign(n + 1, -1);
        int64_t o = 0;
        e->exp_off[0] = o;
        o += (int64_t)e->in_H * e->in_W;
        for (int i = 0; i < n; i++)
            if (e->L[i].kind != ST_OUTPUT) {
                e->exp_off[i + 1] = o;
                o += (int64_t)e->L[i].H * e->L[i].W;
            }
        if (cudaMalloc(&e->exp_words, o * 4) != cudaSuccess) {
            cudaGetLastError();
            e->exp_words = nullptr;
            return fail(e, ST_ERR_OOM, "mask export buffer of %lld bytes", (long long)o * 4);
        }
    }
    if (chunk != e->exp_chunk) {   // the issued step changes: drop captured graphs
        CUDA_OK(e, cudaDeviceSynchronize());
        for (auto &g : e->graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        e->graphs.clear();
    }
    e->exp_chunk = chunk;
    e->exp_valid = false;
    return ST_OK;
}

extern "C" st_status st_debug_get_words(st_encoder *e, int32_t layer, uint32_t *words) {
    if (!e || !words) return ST_ERR_ARG;
    if (layer < -1 || layer >= (int)e->L.size()) return fail(e, ST_ERR_ARG, "bad layer %d", layer);
    if (!e->exp_valid || e->exp_chunk < 0) return fail(e, ST_ERR_STATE, "no exporting st_encode_diff yet");
    int t = layer;
    while (t >= 0 && e->L[t].kind == ST_OUTPUT) t = e->L[t].src;
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    const int64_t N = t < 0 ? (int64_t)e->in_H * e->in_W : (int64_t)e->L[t].H * e->L[t].W;
    CUDA_OK(e, cudaMemcpy(words, e->exp_words + e->exp_off[t + 1], N * 4, cudaMemcpyDeviceToHost));
    return ST_OK;
}

extern "C" st_status st_device_bytes(const st_encoder *e, int64_t *total) {
    if (!e || !total) return ST_ERR_ARG;
    *total = e->arena_bytes + e->fixed_bytes;
    return ST_OK;
}

extern "C" st_status st_step_status(st_encoder *e) {
    if (!e) return ST_ERR_ARG;
    if (e->last_ndiff < 0) return ST_OK;
    CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    int32_t ov = 0;
    CUDA_OK(e, cudaMemcpy(&ov, e->ovf, 4, cudaMemcpyDeviceToHost));
    return ov ? fail(e, ST_ERR_CAPACITY, "the last step exceeded a row capacity") : ST_OK;
}

extern "C" st_status st_get_capacity(st_encoder *e, int64_t *rows_cap, int64_t *rows_peak) {
    if (!e) return ST_ERR_ARG;
    const int n = (int)e->L.size();
    if (e->last_stream) CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    std::vector<long long> pk(n + 1);
    CUDA_OK(e, cudaMemcpy(pk.data(), e->rows_peak, (n + 1) * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i <= n; i++) {
        const bool own = i == n || e->L[i].b_rows >= 0 || e->L[i].kind == ST_CONV || e->L[i].kind == ST_MAXPOOL ||
                         e->L[i].kind == ST_ADD || e->L[i].kind == ST_SE;
        if (rows_cap) rows_cap[i] = !own ? -1 : i == n ? e->in_rows_cap : e->L[i].rows_cap;
        if (rows_peak) rows_peak[i] = own ? pk[i] : -1;
    }
    return ST_OK;
}

extern "C" st_status st_encoder_fit_capacity(st_encoder *e, double headroom) {
    if (!e) return ST_ERR_ARG;
    if (!(headroom >= 1.0)) return fail(e, ST_ERR_ARG, "headroom %g < 1", headroom);
    if (e->cfg.streaming) return fail(e, ST_ERR_UNSUPPORTED, "streaming caches live in the arena");
    CUDA_OK(e, cudaSetDevice(e->cfg.device));
    CUDA_OK(e, cudaDeviceSynchronize());
    const int n = (int)e->L.size();
    std::vector<long long> pk(n + 1);
    CUDA_OK(e, cudaMemcpy(pk.data(), e->rows_peak, (n + 1) * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i <= n; i++) e->cap_fit[i] = std::max<int64_t>((int64_t)std::ceil(headroom * (double)pk[i]), 4096);
    for (auto &g : e->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    e->graphs.clear();
    cudaFree(e->arena);
    e->arena = nullptr;
    e->arena_bytes = 0;
    e->last_ndiff = -1;   // the last step's results are gone
    st_status r = plan(e);
    if (r == ST_OK) encode_act_maps(e);
    return r;
}

extern "C" st_status st_memory_report(const st_encoder *e, int64_t *persistent, int64_t *peak, int64_t *arena) {
    if (!e) return ST_ERR_ARG;
    if (persistent) *persistent = e->persistent_bytes;
    if (peak) *peak = e->peak_transient;
    if (arena) *arena = e->arena_bytes;
    return ST_OK;
}

// ---------------------------------------------------------------- profiling
extern "C" st_status st_set_profiling(st_encoder *e, int32_t on) {
    if (!e) return ST_ERR_ARG;
    e->prof = on != 0;
    e->recs.clear();
    e->ev_used = 0;
    return ST_OK;
}
extern "C" int32_t st_num_kernel_classes(void) { return KC_N; }
extern "C" const char *st_kernel_class_name(int32_t i) { return i >= 0 && i < KC_N ? KC_NAMES[i] : ""; }

extern "C" st_status st_get_kernel_times(st_encoder *e, double *ms, int64_t *launches, double *bytes, double *flops,
                                         int32_t reset) {
    if (!e) return ST_ERR_ARG;
    if (e->last_stream || e->last_ndiff >= 0) CUDA_OK(e, cudaStreamSynchronize(e->last_stream));
    // fold pending records of the last encode call
    if (!e->recs.empty()) {
        std::vector<int64_t> rin(e->L.size()), rout(e->L.size()), tch(e->L.size());
        if (e->last_ndiff > 0) st_get_layer_counts(e, rin.data(), rout.data(), tch.data());
        for (auto &r : e->recs) {
            float t = 0;
            cudaEventElapsedTime(&t, r.e0, r.e1);
            e->prof_ms[r.cls] += t;
            e->prof_n[r.cls] += 1;
            const bool sparse = r.cls == KC_CONV_SPARSE || r.cls == KC_DW_SPARSE || r.cls == KC_TC_SPARSE ||
                                r.cls == KC_STEM_SPARSE;
            const bool dense = r.cls == KC_CONV_DENSE || r.cls == KC_DW_DENSE || r.cls == KC_TC_DENSE ||
                               r.cls == KC_STEM_DENSE;
            if (r.layer >= 0 && (sparse || dense)) {
                const LayerRT &l = e->L[r.layer];
                const int64_t K = (int64_t)l.geo.kh * l.geo.kw * (l.geo.Cin / l.geo.groups);
                const int64_t M = sparse ? rout[r.layer] : (int64_t)e->last_chunks * l.H * l.W;
                const int64_t Min = sparse ? rin[r.layer] : (int64_t)e->last_chunks * l.geo.Hin * l.geo.Win;
                e->prof_flops[r.cls] += 2.0 * K * l.C * M;
                // algorithmic bytes: each active input row once, each output row once (+ its
                // 4-byte row index when sparse), weights once (bf16 on the tensor-core path)
                const double wbytes = (r.cls == KC_TC_SPARSE || r.cls == KC_TC_DENSE || r.cls == KC_STEM_SPARSE ||
                                       r.cls == KC_STEM_DENSE) ? 2.0 : 4.0;
                const double ebytes = sparse && e->cfg.precision == ST_BF16 ? 2.0 : 4.0;   // row element size
                const double b = ebytes * ((double)Min * l.geo.Cin + (double)M * l.C) + wbytes * K * l.C +
                                 (sparse && r.cls != KC_DW_SPARSE ? 4.0 * M : 0.0);
                e->prof_bytes[r.cls] += b;
                if (e->prof_trace)
                    fprintf(stderr, "[st-prof] bf=%d cls=%d layer=%d ms=%.4f M=%lld Min=%lld K=%lld C=%d GBps=%.1f\n",
                            (int)(e->cfg.precision == ST_BF16), r.cls, r.layer, t, (long long)M, (long long)Min, (long long)K, l.C, t > 0 ? b / t * 1e-6 : 0.0);
            } else if (r.layer >= 0 && r.cls == KC_DW_SITE && e->last_ndiff > 0) {
                // depthwise conv + its site: active input rows once, x0 of the touched
                // output pixels once, the site's emitted rows once, frame words; the
                // conv's own delta rows never leave the chip
                const LayerRT &l = e->L[r.layer];
                const int si = l.dw_site;
                const double eb = e->cfg.precision == ST_BF16 ? 2.0 : 4.0;
                const double C = l.C, Bc = e->last_chunks;
                const int64_t K = (int64_t)l.geo.kh * l.geo.kw;
                e->prof_flops[r.cls] += 2.0 * K * l.C * (double)rout[r.layer];
                const double b = eb * ((double)rin[r.layer] + (double)rout[si]) * C + 4.0 * tch[si] * C +
                                 12.0 * tch[si] + 4.0 * Bc * ((double)l.geo.Hin * l.geo.Win + 2.0 * l.H * l.W) +
                                 4.0 * K * C;
                e->prof_bytes[r.cls] += b;
                if (e->prof_trace)
                    fprintf(stderr, "[st-prof] bf=%d cls=%d layer=%d ms=%.4f M=%lld Min=%lld GBps=%.1f\n",
                            (int)(e->cfg.precision == ST_BF16), r.cls, r.layer, t, (long long)rout[r.layer],
                            (long long)rin[r.layer], t > 0 ? b / t * 1e-6 : 0.0);
            } else if (r.layer >= 0 && e->last_ndiff > 0 &&
                       (r.cls == KC_SITE_PW || r.cls == KC_SITE_MP || r.cls == KC_ACCUM || r.cls == KC_SE)) {
                // algorithmic bytes of the HBM-bound per-pixel kernels:
                // input delta rows once, x0 of the touched input pixels once, emitted
                // rows once, frame words in/out; Accumulation writes the dense outputs
                const LayerRT &l = e->L[r.layer];
                const double eb = e->cfg.precision == ST_BF16 ? 2.0 : 4.0;
                const double C = l.C, Bc = e->last_chunks, F = e->last_ndiff;
                const double Nout = (double)l.H * l.W;
                const double Nin = l.src < 0 ? (double)e->in_H * e->in_W : (double)e->L[l.src].H * e->L[l.src].W;
                double b = 0;
                if (r.cls == KC_ACCUM)
                    b = 4.0 * Bc * (F + 1) * Nout * C + 4.0 * Bc * Nout * C + eb * rin[r.layer] * C + 4.0 * Bc * Nin;
                else if (l.fused_relu >= 0)   // ReLU + pool pass: conv rows in, x0 of the touched conv
                    // pixels, pool rows out; the ReLU rows never leave the chip
                    b = eb * ((double)rin[l.fused_relu] + (double)rout[r.layer]) * C + 4.0 * tch[l.fused_relu] * C +
                        12.0 * tch[l.fused_relu] + 4.0 * Bc * (2 * Nin + Nout);
                else
                    b = eb * ((double)rin[r.layer] + (double)rout[r.layer]) * C + 4.0 * tch[r.layer] * C +
                        12.0 * tch[r.layer] + 4.0 * Bc * (Nin + Nout);
                e->prof_bytes[r.cls] += b;
                if (e->prof_trace)
                    fprintf(stderr, "[st-prof] bf=%d cls=%d layer=%d ms=%.4f GBps=%.1f\n",
                            (int)(e->cfg.precision == ST_BF16), r.cls, r.layer, t, t > 0 ? b / t * 1e-6 : 0.0);
            } else if (r.layer >= 0 && r.cls == KC_SE_SUMS) {
                // SE sums / schedule / dense apply of one layer (5 launches with diff
                // frames, 4 without): x0 column sums, delta-row sums, dense x -> y;
                // the layer total is spread evenly over its launches
                const LayerRT &l = e->L[r.layer];
                const double eb = e->cfg.precision == ST_BF16 ? 2.0 : 4.0;
                const double BNC = (double)e->last_chunks * l.H * l.W * l.C;
                const double tot = 3.0 * 4.0 * BNC + (e->last_ndiff > 0 ? eb * (double)rin[r.layer] * l.C : 0.0);
                e->prof_bytes[r.cls] += tot / (e->last_ndiff > 0 ? 5.0 : 4.0);
                if (e->prof_trace)
                    fprintf(stderr, "[st-prof] bf=%d cls=%d layer=%d ms=%.4f\n", (int)(e->cfg.precision == ST_BF16),
                            r.cls, r.layer, t);
            } else if (e->prof_trace) {
                fprintf(stderr, "[st-prof] bf=%d cls=%d layer=%d ms=%.4f\n", (int)(e->cfg.precision == ST_BF16), r.cls, r.layer, t);
            }
        }
        e->recs.clear();
        e->ev_used = 0;
    }
    for (int i = 0; i < KC_N; i++) {
        if (ms) ms[i] = e->prof_ms[i];
        if (launches) launches[i] = e->prof_n[i];
        if (bytes) bytes[i] = e->prof_bytes[i];
        if (flops) flops[i] = e->prof_flops[i];
    }
    if (reset)
        for (int i = 0; i < KC_N; i++) { e->prof_ms[i] = 0; e->prof_n[i] = 0; e->prof_bytes[i] = 0; e->prof_flops[i] = 0; }
    return ST_OK;
}

extern "C" int32_t st_last_launch_count(const st_encoder *e) { return e ? e->launches : 0; }

extern "C" const char *st_status_string(st_status s) {
    switch (s) {
    case ST_OK: return "ok";
    case ST_ERR_ARG: return "invalid argument";
    case ST_ERR_SHAPE: return "shape mismatch";
    case ST_ERR_STATE: return "call out of order";
    case ST_ERR_UNSUPPORTED: return "unsupported";
    case ST_ERR_OOM: return "out of device memory";
    case ST_ERR_CUDA: return "CUDA error";
    case ST_ERR_INTERNAL: return "internal error";
    case ST_ERR_CAPACITY: return "row capacity exceeded (re-plan with st_encoder_fit_capacity and re-issue)";
    }
    return "unknown status";
}

extern "C" const char *st_last_error(const st_encoder *e) { return e ? e->err.c_str() : ""; }
