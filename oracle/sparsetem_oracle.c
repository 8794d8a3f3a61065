/*
 * sparsetem_oracle.c -- CPU oracle of SparseTem's Diff Computation
 * (arXiv 2410.20790, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` legs may load this file.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2410_20790_b200/csrc); neither includes the other.
 *
 * What it computes, step by step in the paper's order (citations are
 * PAPER.md line numbers "P:n"; SURVEY readings "Rn" are listed in DESIGN.md):
 *
 *   dense_layer   Eq.(1) P:119-122 convolution (+bias), ReLU, SiLU, maxpool,
 *                 add, squeeze-excitation -- the dense forward used on the
 *                 reference frame and as the "original model".
 *   subtraction   P:115-116 + truncation P:143: raw = X_t - S,
 *                 active iff max_c |raw| > theta_0 (R1/R2), S += emitted (R3).
 *   conv delta    Eq.(2): output mask = dilation of the input mask
 *                 (dense amplification), values = full receptive-field
 *                 dot product of the delta, NO bias (R5).
 *   nonlinear     Eq.(3): x_acc += delta; c = f(x_acc) - y_acc;
 *                 emit iff max_c |c| > theta_site; y_acc += emitted (R7).
 *   SE site       reading R8 (gate refresh when max_c |s_t - s_emit| > theta).
 *   accumulation  P:116: O_t = O_{t-1} + delta at the taps.
 *   order         frame-outer (DeltaCNN / vanilla) or layer-outer
 *                 (SparseBatch "N" order); values are identical.
 *
 * Arithmetic: IEEE fp32, round-to-nearest; every multiply-add is an explicit
 * fmaf() in the fixed K order (dy, dx, ci) starting from +0.0f, bias added
 * last (reading R18); compiled with -ffp-contract=off so no other fusion
 * happens.  exp() is evaluated in double and rounded to float (reading R10).
 * The SE mean is summed in double in raster order (reading R8).
 * Storage is NHWC: pixel p = y*W + x, value [p*C + c].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_CONV = 0, ORC_RELU = 1, ORC_SILU = 2, ORC_MAXPOOL = 3, ORC_ADD = 4,
       ORC_SE = 5, ORC_OUTPUT = 6 };

typedef struct {
    int32_t kind, src, src2, c_out, groups, k_h, k_w, s_h, s_w, p_h, p_w, se_hidden;
    const float *w, *b, *w2, *b2;
} orc_layer;

typedef struct { int h, w, c; } shp;

static int is_nonlinear(int k) {
    return k == ORC_RELU || k == ORC_SILU || k == ORC_MAXPOOL || k == ORC_SE;
}

/* geometry */
static int out_dim(int n, int k, int s, int p) { return (n + 2 * p - k) / s + 1; }

/* ---------------------------------------------------------------- shapes */
static int infer(const orc_layer *L, int n, shp in, shp *out) {
    for (int i = 0; i < n; i++) {
        const orc_layer *l = &L[i];
        if (l->src >= i || l->src < -1) return -1;
        shp s = l->src < 0 ? in : out[l->src];
        switch (l->kind) {
        case ORC_CONV:
            if (l->groups < 1 || s.c % l->groups || l->c_out % l->groups) return -2;
            out[i].h = out_dim(s.h, l->k_h, l->s_h, l->p_h);
            out[i].w = out_dim(s.w, l->k_w, l->s_w, l->p_w);
            out[i].c = l->c_out;
            break;
        case ORC_MAXPOOL:
            out[i].h = out_dim(s.h, l->k_h, l->s_h, l->p_h);
            out[i].w = out_dim(s.w, l->k_w, l->s_w, l->p_w);
            out[i].c = s.c;
            break;
        case ORC_ADD: {
            if (l->src2 >= i || l->src2 < -1) return -1;
            shp s2 = l->src2 < 0 ? in : out[l->src2];
            if (s2.h != s.h || s2.w != s.w || s2.c != s.c) return -3;
            out[i] = s;
            break;
        }
        case ORC_RELU: case ORC_SILU: case ORC_SE: case ORC_OUTPUT:
            out[i] = s;
            break;
        default:
            return -4;
        }
        if (out[i].h < 1 || out[i].w < 1) return -5;
    }
    return 0;
}

int orc_shapes(const orc_layer *L, int n, int in_h, int in_w, int in_c, int32_t *hwc) {
    shp in = {in_h, in_w, in_c};
    shp *o = (shp *)malloc(sizeof(shp) * (n > 0 ? n : 1));
    int r = infer(L, n, in, o);
    if (r == 0)
        for (int i = 0; i < n; i++) { hwc[3 * i] = o[i].h; hwc[3 * i + 1] = o[i].w; hwc[3 * i + 2] = o[i].c; }
    free(o);
    return r;
}

int orc_num_sites(const orc_layer *L, int n) {
    int s = 1;
    for (int i = 0; i < n; i++) s += is_nonlinear(L[i].kind);
    return s;
}

/* ------------------------------------------------------- scalar functions */
static float exp_r(float v) { return (float)exp((double)v); }           /* R10 */
static float relu_f(float x) { return x > 0.0f ? x : 0.0f; }
static float silu_f(float x) { return x / (1.0f + exp_r(-x)); }          /* R10 */
static float sigm_f(float x) { return 1.0f / (1.0f + exp_r(-x)); }       /* R10 */

/* Precision mode (R22-BF16).  0 = FP32 mode.  1 = BF16 mode, a
 * contract stated without reference to how the GPU dispatches its kernels:
 *  - every emitted delta (input Subtraction, conv output, residual add, every
 *    non-linear site) is stored rounded to bf16 (round-to-nearest-even); the
 *    truncation decision is taken on the fp32 value, and the Subtraction
 *    buffer S and each site's y_acc advance by the rounded (emitted) value;
 *  - EVERY convolution (dense or delta, any groups / kernel size) multiplies
 *    bf16-rounded operands (weight and input value) and accumulates in fp32;
 *  - dense reference activations, site states, SE gates and outputs stay fp32. */
static int g_bf16 = 0;
void orc_set_precision(int bf16) { g_bf16 = bf16 ? 1 : 0; }

static float bf16r(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    memcpy(&v, &u, 4);
    return v;
}
static float emit_r(float v) { return g_bf16 ? bf16r(v) : v; }

/* ------------------------------------------------------------ dense ops */

/* Eq.(1): O[q][co] = sum_{dy,dx,ci} W[co][ci][dy][dx] * X[p(q,dy,dx)][g*cin_g+ci]
 * (+ b[co] when with_bias).  If mask_in != NULL, input pixels outside the mask
 * are treated as exact zeros; if mask_out != NULL only masked outputs are
 * computed (others set to 0). */
static void conv_apply(const orc_layer *l, shp si, shp so, const float *x, const uint8_t *mask_out,
                       int with_bias, float *out) {
    const int cin_g = si.c / l->groups, cout_g = l->c_out / l->groups;
    const int No = so.h * so.w;
    const int rb = g_bf16;   /* R22-BF16: every conv multiplies bf16-rounded operands */
#pragma omp parallel for schedule(static)
    for (int q = 0; q < No; q++) {
        float *o = out + (size_t)q * so.c;
        if (mask_out && !mask_out[q]) {
            for (int co = 0; co < so.c; co++) o[co] = 0.0f;
            continue;
        }
        const int oy = q / so.w, ox = q % so.w;
        for (int co = 0; co < so.c; co++) {
            const int g = co / cout_g;
            float acc = 0.0f;
            for (int dy = 0; dy < l->k_h; dy++) {
                const int iy = oy * l->s_h - l->p_h + dy;
                if (iy < 0 || iy >= si.h) continue;            /* zero padding */
                for (int dx = 0; dx < l->k_w; dx++) {
                    const int ix = ox * l->s_w - l->p_w + dx;
                    if (ix < 0 || ix >= si.w) continue;
                    const float *xp = x + ((size_t)iy * si.w + ix) * si.c + (size_t)g * cin_g;
                    for (int ci = 0; ci < cin_g; ci++) {
                        const float wv = l->w[(((size_t)co * cin_g + ci) * l->k_h + dy) * l->k_w + dx];
                        acc = rb ? fmaf(bf16r(wv), bf16r(xp[ci]), acc) : fmaf(wv, xp[ci], acc);
                    }
                }
            }
            o[co] = with_bias ? acc + l->b[co] : acc;
        }
    }
}

/* window max with -inf padding (R11) at output pixel q */
static void maxwin(const orc_layer *l, shp si, shp so, const float *x, int q, float *o) {
    const int oy = q / so.w, ox = q % so.w;
    for (int c = 0; c < si.c; c++) {
        float m = -INFINITY;
        for (int dy = 0; dy < l->k_h; dy++) {
            const int iy = oy * l->s_h - l->p_h + dy;
            if (iy < 0 || iy >= si.h) continue;
            for (int dx = 0; dx < l->k_w; dx++) {
                const int ix = ox * l->s_w - l->p_w + dx;
                if (ix < 0 || ix >= si.w) continue;
                const float v = x[((size_t)iy * si.w + ix) * si.c + c];
                m = v > m ? v : m;
            }
        }
        o[c] = m;
    }
}

/* SE gate s = sigmoid(W2 silu(W1 mean(x) + b1) + b2)  (reading R8) */
static void se_gate(const orc_layer *l, shp s, const float *x, float *gate) {
    const int C = s.c, N = s.h * s.w, H = l->se_hidden;
    float *mean = (float *)malloc(sizeof(float) * C);
    float *hid = (float *)malloc(sizeof(float) * (H > 0 ? H : 1));
    for (int c = 0; c < C; c++) {
        double acc = 0.0;
        for (int p = 0; p < N; p++) acc += (double)x[(size_t)p * C + c];
        mean[c] = (float)(acc / (double)N);
    }
    for (int j = 0; j < H; j++) {
        float acc = 0.0f;
        for (int c = 0; c < C; c++) acc = fmaf(l->w[(size_t)j * C + c], mean[c], acc);
        hid[j] = silu_f(acc + l->b[j]);
    }
    for (int c = 0; c < C; c++) {
        float acc = 0.0f;
        for (int j = 0; j < H; j++) acc = fmaf(l->w2[(size_t)c * H + j], hid[j], acc);
        gate[c] = sigm_f(acc + l->b2[c]);
    }
    free(mean);
    free(hid);
}

/* one dense layer on one frame */
static void dense_layer(const orc_layer *l, shp si, shp so, const float *x, const float *x2, float *y) {
    const size_t ni = (size_t)si.h * si.w * si.c;
    switch (l->kind) {
    case ORC_CONV: conv_apply(l, si, so, x, NULL, 1, y); break;
    case ORC_RELU: for (size_t i = 0; i < ni; i++) y[i] = relu_f(x[i]); break;
    case ORC_SILU: for (size_t i = 0; i < ni; i++) y[i] = silu_f(x[i]); break;
    case ORC_MAXPOOL:
        for (int q = 0; q < so.h * so.w; q++) maxwin(l, si, so, x, q, y + (size_t)q * so.c);
        break;
    case ORC_ADD: for (size_t i = 0; i < ni; i++) y[i] = x[i] + x2[i]; break;
    case ORC_SE: {
        float *g = (float *)malloc(sizeof(float) * si.c);
        se_gate(l, si, x, g);
        for (size_t i = 0; i < ni; i++) y[i] = x[i] * g[i % si.c];
        free(g);
        break;
    }
    case ORC_OUTPUT: memcpy(y, x, ni * sizeof(float)); break;
    }
}

static size_t numel(shp s) { return (size_t)s.h * s.w * s.c; }

/* Dense forward of one frame.  outs[l] (caller buffers, may be NULL)
 * receive every layer's output. */
int orc_dense_forward(const orc_layer *L, int n, int in_h, int in_w, int in_c,
                      const float *x, float **outs) {
    shp in = {in_h, in_w, in_c};
    shp *s = (shp *)malloc(sizeof(shp) * n);
    int r = infer(L, n, in, s);
    if (r) { free(s); return r; }
    float **y = (float **)calloc(n, sizeof(float *));
    for (int i = 0; i < n; i++) {
        y[i] = (float *)malloc(numel(s[i]) * sizeof(float));
        const orc_layer *l = &L[i];
        const float *a = l->src < 0 ? x : y[l->src];
        shp sa = l->src < 0 ? in : s[l->src];
        const float *b = l->kind == ORC_ADD ? (l->src2 < 0 ? x : y[l->src2]) : NULL;
        dense_layer(l, sa, s[i], a, b, y[i]);
        if (outs && outs[i]) memcpy(outs[i], y[i], numel(s[i]) * sizeof(float));
    }
    for (int i = 0; i < n; i++) free(y[i]);
    free(y);
    free(s);
    return 0;
}

/* Mask dilation (dense amplification): output pixel is
 * active iff its receptive field (stride/pad aware) holds an active input. */
static void dilate(const uint8_t *m, int H, int W, int kh, int kw, int sh, int sw, int ph, int pw,
                   int Ho, int Wo, uint8_t *mo) {
    for (int oy = 0; oy < Ho; oy++)
        for (int ox = 0; ox < Wo; ox++) {
            uint8_t a = 0;
            for (int dy = 0; dy < kh && !a; dy++) {
                const int iy = oy * sh - ph + dy;
                if (iy < 0 || iy >= H) continue;
                for (int dx = 0; dx < kw; dx++) {
                    const int ix = ox * sw - pw + dx;
                    if (ix < 0 || ix >= W) continue;
                    if (m[iy * W + ix]) { a = 1; break; }
                }
            }
            mo[oy * Wo + ox] = a;
        }
}

void orc_dilate(const uint8_t *m, int H, int W, int kh, int kw, int sh, int sw, int ph, int pw,
                int Ho, int Wo, uint8_t *mo) {
    dilate(m, H, W, kh, kw, sh, sw, ph, pw, Ho, Wo, mo);
}

/* ------------------------------------------------------ diff computation */

/* O12 band-follow (reading R23).  A truncation decision
 * compares max_c |c| with theta; where the two sides' values of c are not
 * bit-matched (BF16 mode, SiLU / SE), every decision whose value lies inside
 * the ambiguity band |max_c|c| - theta| <= tau is a correct one.  With follow
 * masks given (the GPU's emitted masks of one chunk, per site layer [F][N_l]),
 * the oracle adopts the GPU's decision ONLY inside the band; every other
 * decision stays its own, and a disagreement there is counted as a violation.
 * tau = a_theta * theta + a_rms * rms + a_abs, rms = root mean square of the
 * site's current output f(x_acc) (= candidate + y_acc) over the touched pixels
 * of that site and frame: the candidate is a difference of two activation-
 * sized values, so the two sides' candidates differ by amounts relative to
 * the activations (bf16 roundings of x_acc / y_acc), not to the candidate.
 * stats per layer: [0] decisions, [1] inside the band, [2] adopted (the GPU's
 * decision differed from the oracle's own), [3] violations. */
typedef struct {
    const uint8_t *const *masks;   /* [n] per layer ([F][N_l]) or NULL entries */
    float a_theta, a_rms, a_abs;
    int64_t *stats;                /* [n][4] */
} follow_t;

typedef struct {
    const orc_layer *L;
    int n, L_frames;
    shp in;
    shp *s;
    int *site;             /* site index of layer l (0 if linear) */
    const float *theta;    /* [n_sites] */
    /* per-layer transient state (nonlinear layers only) */
    float **xacc, **yacc, **semit;
    float **otap;          /* running output at OUTPUT layers */
    float *S;              /* Subtraction buffer */
    int64_t *counts;       /* [n_sites][L-1] */
    const follow_t *fl;    /* band-follow (NULL = off) */
    /* scratch of one site step: candidate rows [N][C], max_c |cand| [N], touched [N] */
    float *cand, *mx;
    uint8_t *T;
} ctx_t;

static shp src_shape(const ctx_t *c, int i) { return i < 0 ? c->in : c->s[i]; }

/* Subtraction + input truncation for diff frame t (site 0). */
static void step_input(ctx_t *c, int t, const float *X, float *d, uint8_t *m) {
    const int N = c->in.h * c->in.w, C = c->in.c;
    const float th = c->theta[0];
    int64_t cnt = 0;
    for (int p = 0; p < N; p++) {
        float raw[64];
        float mx = 0.0f;
        for (int ch = 0; ch < C; ch++) {
            raw[ch] = X[(size_t)p * C + ch] - c->S[(size_t)p * C + ch];
            const float a = fabsf(raw[ch]);
            mx = a > mx ? a : mx;
        }
        if (mx > th) {                                      /* R1: strict */
            m[p] = 1;
            cnt++;
            for (int ch = 0; ch < C; ch++) {
                const float e = emit_r(raw[ch]);                   /* stored delta */
                d[(size_t)p * C + ch] = e;
                c->S[(size_t)p * C + ch] = c->S[(size_t)p * C + ch] + e;   /* R3 */
            }
        } else {
            m[p] = 0;
            for (int ch = 0; ch < C; ch++) d[(size_t)p * C + ch] = 0.0f;
        }
    }
    if (c->counts) c->counts[(size_t)0 * (c->L_frames - 1) + (t - 1)] = cnt;
}

static float row_absmax(const float *v, int C) {
    float mx = 0.0f;
    for (int ch = 0; ch < C; ch++) {
        const float a = fabsf(v[ch]);
        mx = a > mx ? a : mx;
    }
    return mx;
}

/* Truncation of one non-linear site for one frame (R1/R2/R7): the
 * candidate rows c->cand of the touched pixels c->T are already computed,
 * c->mx[p] = max_c |cand|.  Keep iff max_c |cand| > theta (strict); a kept
 * row is emitted (stored rounded in BF16 mode) and y_acc advances by the
 * emitted value; everything else is exactly 0.  Returns the emitted count. */
static int64_t truncate_site(ctx_t *c, int i, int t, int No, int C, float *ya, float *d, uint8_t *m) {
    const float th = c->theta[c->site[i]];
    const uint8_t *fm = (c->fl && c->fl->masks && c->fl->masks[i]) ? c->fl->masks[i] + (size_t)(t - 1) * No : NULL;
    double tau = 0.0;
    int64_t *fs = fm ? c->fl->stats + (size_t)4 * i : NULL;
    if (fm) {
        double ss = 0.0;
        int64_t n = 0;
        for (int p = 0; p < No; p++)
            if (c->T[p]) {
                for (int ch = 0; ch < C; ch++) {   /* the site's current output f(x_acc) = cand + y_acc */
                    const double v = (double)c->cand[(size_t)p * C + ch] + (double)ya[(size_t)p * C + ch];
                    ss += v * v;
                }
                n += C;
            }
        const double rms = n ? sqrt(ss / (double)n) : 0.0;
        tau = (double)c->fl->a_theta * th + (double)c->fl->a_rms * rms + (double)c->fl->a_abs;
    }
    int64_t cnt = 0;
    for (int p = 0; p < No; p++) {
        float *dp = d + (size_t)p * C;
        int keep = 0;
        if (c->T[p]) {
            keep = c->mx[p] > th;                                   /* R1: strict */
            if (fm) {
                fs[0]++;
                if (fabs((double)c->mx[p] - (double)th) <= tau) {
                    fs[1]++;
                    if ((int)fm[p] != keep) { fs[2]++; keep = fm[p]; }
                } else if ((int)fm[p] != keep) {
                    fs[3]++;
                }
            }
        } else if (fm && fm[p]) {
            fs[3]++;                                                /* GPU emitted an untouched pixel */
        }
        m[p] = (uint8_t)keep;
        if (keep) {
            const float *cp = c->cand + (size_t)p * C;
            float *yp = ya + (size_t)p * C;
            for (int ch = 0; ch < C; ch++) {
                const float e = emit_r(cp[ch]);    /* stored delta; y_acc advances by it */
                yp[ch] = yp[ch] + e;
                dp[ch] = e;
            }
            cnt++;
        } else {
            for (int ch = 0; ch < C; ch++) dp[ch] = 0.0f;
        }
    }
    return cnt;
}

/* one layer, one diff frame t.  d_a/m_a: src delta; d_b/m_b: src2 delta (ADD). */
static void step_layer(ctx_t *c, int i, int t, const float *d_a, const uint8_t *m_a,
                       const float *d_b, const uint8_t *m_b, float *d, uint8_t *m) {
    const orc_layer *l = &c->L[i];
    const shp si = src_shape(c, l->src), so = c->s[i];
    const int Ni = si.h * si.w, No = so.h * so.w, C = so.c;
    int64_t cnt = 0;
    switch (l->kind) {
    case ORC_CONV:
        dilate(m_a, si.h, si.w, l->k_h, l->k_w, l->s_h, l->s_w, l->p_h, l->p_w, so.h, so.w, m);
        conv_apply(l, si, so, d_a, m, 0, d);                        /* Eq.(2): no bias */
        if (g_bf16)
            for (size_t k = 0; k < (size_t)No * C; k++) d[k] = emit_r(d[k]);
        break;
    case ORC_ADD:
        for (int p = 0; p < No; p++) {
            m[p] = (uint8_t)(m_a[p] | m_b[p]);
            for (int ch = 0; ch < C; ch++)
                d[(size_t)p * C + ch] = emit_r(d_a[(size_t)p * C + ch] + d_b[(size_t)p * C + ch]);
        }
        break;
    case ORC_OUTPUT: {
        float *O = c->otap[i];
        for (int p = 0; p < No; p++) {
            m[p] = m_a[p];
            for (int ch = 0; ch < C; ch++) {
                const float v = d_a[(size_t)p * C + ch];
                d[(size_t)p * C + ch] = v;
                if (m_a[p]) O[(size_t)p * C + ch] = O[(size_t)p * C + ch] + v;   /* Accumulation */
            }
        }
        break;
    }
    case ORC_RELU: case ORC_SILU: {
        float *xa = c->xacc[i], *ya = c->yacc[i];
        const int relu = l->kind == ORC_RELU;
#pragma omp parallel for schedule(static)
        for (int p = 0; p < No; p++) {
            c->T[p] = m_a[p];                                       /* touched = input mask (R7) */
            if (!m_a[p]) continue;
            float *cp = c->cand + (size_t)p * C;
            for (int ch = 0; ch < C; ch++) {
                const size_t k = (size_t)p * C + ch;
                xa[k] = xa[k] + d_a[k];                             /* reconstruct input */
                const float f = relu ? relu_f(xa[k]) : silu_f(xa[k]);
                cp[ch] = f - ya[k];                                 /* restore delta (Eq.3) */
            }
            c->mx[p] = row_absmax(cp, C);
        }
        cnt = truncate_site(c, i, t, No, C, ya, d, m);
        break;
    }
    case ORC_MAXPOOL: {
        float *xa = c->xacc[i], *ya = c->yacc[i];
        for (int p = 0; p < Ni; p++)
            if (m_a[p])
                for (int ch = 0; ch < C; ch++) xa[(size_t)p * C + ch] = xa[(size_t)p * C + ch] + d_a[(size_t)p * C + ch];
        /* touched = pool-footprint dilation of the input mask (R7) */
        dilate(m_a, si.h, si.w, l->k_h, l->k_w, l->s_h, l->s_w, l->p_h, l->p_w, so.h, so.w, c->T);
#pragma omp parallel for schedule(static)
        for (int q = 0; q < No; q++) {
            if (!c->T[q]) continue;
            float *cp = c->cand + (size_t)q * C;
            maxwin(l, si, so, xa, q, cp);
            for (int ch = 0; ch < C; ch++) cp[ch] = cp[ch] - ya[(size_t)q * C + ch];
            c->mx[q] = row_absmax(cp, C);
        }
        cnt = truncate_site(c, i, t, No, C, ya, d, m);
        break;
    }
    case ORC_SE: {
        float *xa = c->xacc[i], *ya = c->yacc[i], *se = c->semit[i];
        for (int p = 0; p < Ni; p++)
            if (m_a[p])
                for (int ch = 0; ch < C; ch++) xa[(size_t)p * C + ch] = xa[(size_t)p * C + ch] + d_a[(size_t)p * C + ch];
        float *st = (float *)malloc(sizeof(float) * C);
        se_gate(l, si, xa, st);                                     /* s_t = gate(x_acc) */
        float ds = 0.0f;
        for (int ch = 0; ch < C; ch++) {
            const float a = fabsf(st[ch] - se[ch]);
            ds = a > ds ? a : ds;
        }
        const int refresh = ds > c->theta[c->site[i]];              /* R8, theta_gate = theta_site */
        if (refresh) memcpy(se, st, sizeof(float) * C);
#pragma omp parallel for schedule(static)
        for (int p = 0; p < No; p++) {
            c->T[p] = (uint8_t)(refresh || m_a[p]);                  /* refresh touches every pixel */
            if (!c->T[p]) continue;
            float *cp = c->cand + (size_t)p * C;
            for (int ch = 0; ch < C; ch++) cp[ch] = xa[(size_t)p * C + ch] * se[ch] - ya[(size_t)p * C + ch];
            c->mx[p] = row_absmax(cp, C);
        }
        cnt = truncate_site(c, i, t, No, C, ya, d, m);
        free(st);
        break;
    }
    }
    if (is_nonlinear(l->kind) && c->counts)
        c->counts[(size_t)c->site[i] * (c->L_frames - 1) + (t - 1)] = cnt;
}

/*
 * Run one chunk: frame 0 dense (reference frame), frames 1..L-1 as
 * diff frames.  layer_outer = 0: frame-outer order; 1: layer-outer SparseBatch
 * order.  Outputs (caller-allocated; any pointer or entry may be NULL):
 *   masks[l]   uint8 [(L-1)][N_l]        output mask of layer l per diff frame
 *   deltas[l]  float [(L-1)][N_l][C_l]   output delta of layer l (0 off-mask)
 *   dense0[l]  float [N_l][C_l]          frame-0 dense output of layer l
 *   taps[l]    float [L][N_l][C_l]       accumulated outputs of OUTPUT layers
 *   counts     int64 [n_sites][L-1]      emitted-pixel counts per site/frame
 *   in_mask    uint8 [(L-1)][N_in]       input-site (Subtraction) mask
 *   in_delta   float [(L-1)][N_in][C]    input-site emitted delta
 * thresholds: float [n_sites]; site 0 = input, then nonlinear layers in order.
 */
/* follow (nullable): band-follow mode, see follow_t above */
int orc_run_chunk_follow(const orc_layer *L, int n, int in_h, int in_w, int in_c, int Lf,
                         const float *frames, const float *thresholds, int layer_outer,
                         uint8_t **masks, float **deltas, float **dense0, float **taps, int64_t *counts,
                         uint8_t *in_mask, float *in_delta, const follow_t *follow) {
    if (Lf < 1 || in_c > 64) return -10;
    ctx_t c;
    memset(&c, 0, sizeof c);
    c.L = L; c.n = n; c.L_frames = Lf; c.theta = thresholds; c.counts = counts;
    c.in.h = in_h; c.in.w = in_w; c.in.c = in_c;
    c.fl = follow;
    c.s = (shp *)malloc(sizeof(shp) * n);
    int r = infer(L, n, c.in, c.s);
    if (r) { free(c.s); return r; }
    size_t max_nc = 1, max_n = 1;
    for (int i = 0; i < n; i++)
        if (is_nonlinear(L[i].kind)) {
            const size_t No = (size_t)c.s[i].h * c.s[i].w;
            if (No * c.s[i].c > max_nc) max_nc = No * c.s[i].c;
            if (No > max_n) max_n = No;
        }
    c.cand = (float *)malloc(max_nc * sizeof(float));
    c.mx = (float *)malloc(max_n * sizeof(float));
    c.T = (uint8_t *)malloc(max_n);
    c.site = (int *)calloc(n, sizeof(int));
    for (int i = 0, s = 1; i < n; i++) if (is_nonlinear(L[i].kind)) c.site[i] = s++;
    c.xacc = (float **)calloc(n, sizeof(float *));
    c.yacc = (float **)calloc(n, sizeof(float *));
    c.semit = (float **)calloc(n, sizeof(float *));
    c.otap = (float **)calloc(n, sizeof(float *));
    const size_t nin = numel(c.in);

    /* ---- reference frame: dense forward; seed buffers and states ---- */
    float **y0 = (float **)calloc(n, sizeof(float *));
    for (int i = 0; i < n; i++) y0[i] = (float *)malloc(numel(c.s[i]) * sizeof(float));
    orc_dense_forward(L, n, in_h, in_w, in_c, frames, y0);
    c.S = (float *)malloc(nin * sizeof(float));
    memcpy(c.S, frames, nin * sizeof(float));
    for (int i = 0; i < n; i++) {
        const orc_layer *l = &L[i];
        if (dense0 && dense0[i]) memcpy(dense0[i], y0[i], numel(c.s[i]) * sizeof(float));
        if (is_nonlinear(l->kind)) {
            const shp si = src_shape(&c, l->src);
            const float *x0 = l->src < 0 ? frames : y0[l->src];
            c.xacc[i] = (float *)malloc(numel(si) * sizeof(float));
            memcpy(c.xacc[i], x0, numel(si) * sizeof(float));
            c.yacc[i] = (float *)malloc(numel(c.s[i]) * sizeof(float));
            memcpy(c.yacc[i], y0[i], numel(c.s[i]) * sizeof(float));
            if (l->kind == ORC_SE) {
                c.semit[i] = (float *)malloc(sizeof(float) * si.c);
                se_gate(l, si, x0, c.semit[i]);
            }
        }
        if (l->kind == ORC_OUTPUT) {
            c.otap[i] = (float *)malloc(numel(c.s[i]) * sizeof(float));
            memcpy(c.otap[i], y0[i], numel(c.s[i]) * sizeof(float));
            if (taps && taps[i]) memcpy(taps[i], y0[i], numel(c.s[i]) * sizeof(float));
        }
    }

    if (Lf > 1) {
        const int F = Lf - 1;
        if (!layer_outer) {
            /* frame-outer: per-frame buffers for every layer */
            float **d = (float **)calloc(n, sizeof(float *));
            uint8_t **m = (uint8_t **)calloc(n, sizeof(uint8_t *));
            for (int i = 0; i < n; i++) {
                d[i] = (float *)malloc(numel(c.s[i]) * sizeof(float));
                m[i] = (uint8_t *)malloc((size_t)c.s[i].h * c.s[i].w);
            }
            float *din = (float *)malloc(nin * sizeof(float));
            uint8_t *min = (uint8_t *)malloc((size_t)in_h * in_w);
            for (int t = 1; t < Lf; t++) {
                step_input(&c, t, frames + (size_t)t * nin, din, min);
                if (in_mask) memcpy(in_mask + (size_t)(t - 1) * in_h * in_w, min, (size_t)in_h * in_w);
                if (in_delta) memcpy(in_delta + (size_t)(t - 1) * nin, din, nin * sizeof(float));
                for (int i = 0; i < n; i++) {
                    const orc_layer *l = &L[i];
                    const float *da = l->src < 0 ? din : d[l->src];
                    const uint8_t *ma = l->src < 0 ? min : m[l->src];
                    const float *db = NULL;
                    const uint8_t *mb = NULL;
                    if (l->kind == ORC_ADD) { db = l->src2 < 0 ? din : d[l->src2]; mb = l->src2 < 0 ? min : m[l->src2]; }
                    step_layer(&c, i, t, da, ma, db, mb, d[i], m[i]);
                    const size_t No = (size_t)c.s[i].h * c.s[i].w;
                    if (masks && masks[i]) memcpy(masks[i] + (size_t)(t - 1) * No, m[i], No);
                    if (deltas && deltas[i]) memcpy(deltas[i] + (size_t)(t - 1) * numel(c.s[i]), d[i], numel(c.s[i]) * sizeof(float));
                    if (l->kind == ORC_OUTPUT && taps && taps[i])
                        memcpy(taps[i] + (size_t)t * numel(c.s[i]), c.otap[i], numel(c.s[i]) * sizeof(float));
                }
            }
            for (int i = 0; i < n; i++) { free(d[i]); free(m[i]); }
            free(d); free(m); free(din); free(min);
        } else {
            /* layer-outer (SparseBatch "N" order): every layer sees all F frames
             * before the next layer runs; per-layer state could be dropped after. */
            float **D = (float **)calloc(n, sizeof(float *));
            uint8_t **M = (uint8_t **)calloc(n, sizeof(uint8_t *));
            float *Din = (float *)malloc((size_t)F * nin * sizeof(float));
            uint8_t *Min = (uint8_t *)malloc((size_t)F * in_h * in_w);
            const size_t Nin = (size_t)in_h * in_w;
            for (int t = 1; t < Lf; t++)
                step_input(&c, t, frames + (size_t)t * nin, Din + (size_t)(t - 1) * nin, Min + (size_t)(t - 1) * Nin);
            if (in_mask) memcpy(in_mask, Min, (size_t)F * Nin);
            if (in_delta) memcpy(in_delta, Din, (size_t)F * nin * sizeof(float));
            for (int i = 0; i < n; i++) {
                const orc_layer *l = &L[i];
                const size_t ne = numel(c.s[i]), No = (size_t)c.s[i].h * c.s[i].w;
                D[i] = (float *)malloc((size_t)F * ne * sizeof(float));
                M[i] = (uint8_t *)malloc((size_t)F * No);
                const shp sa = src_shape(&c, l->src);
                const size_t nea = numel(sa), Na = (size_t)sa.h * sa.w;
                for (int t = 1; t < Lf; t++) {
                    const float *da = (l->src < 0 ? Din : D[l->src]) + (size_t)(t - 1) * nea;
                    const uint8_t *ma = (l->src < 0 ? Min : M[l->src]) + (size_t)(t - 1) * Na;
                    const float *db = NULL;
                    const uint8_t *mb = NULL;
                    if (l->kind == ORC_ADD) {
                        db = (l->src2 < 0 ? Din : D[l->src2]) + (size_t)(t - 1) * nea;
                        mb = (l->src2 < 0 ? Min : M[l->src2]) + (size_t)(t - 1) * Na;
                    }
                    step_layer(&c, i, t, da, ma, db, mb, D[i] + (size_t)(t - 1) * ne, M[i] + (size_t)(t - 1) * No);
                    if (l->kind == ORC_OUTPUT && taps && taps[i])
                        memcpy(taps[i] + (size_t)t * ne, c.otap[i], ne * sizeof(float));
                }
                /* SparseBatch: the layer's transient state dies here */
                free(c.xacc[i]); c.xacc[i] = NULL;
                free(c.yacc[i]); c.yacc[i] = NULL;
                free(c.semit[i]); c.semit[i] = NULL;
                if (masks && masks[i]) memcpy(masks[i], M[i], (size_t)F * No);
                if (deltas && deltas[i]) memcpy(deltas[i], D[i], (size_t)F * ne * sizeof(float));
            }
            for (int i = 0; i < n; i++) { free(D[i]); free(M[i]); }
            free(D); free(M); free(Din); free(Min);
        }
    }

    for (int i = 0; i < n; i++) {
        free(y0[i]); free(c.xacc[i]); free(c.yacc[i]); free(c.semit[i]); free(c.otap[i]);
    }
    free(y0); free(c.xacc); free(c.yacc); free(c.semit); free(c.otap);
    free(c.S); free(c.site); free(c.s);
    free(c.cand); free(c.mx); free(c.T);
    return 0;
}

int orc_run_chunk(const orc_layer *L, int n, int in_h, int in_w, int in_c, int Lf,
                  const float *frames, const float *thresholds, int layer_outer,
                  uint8_t **masks, float **deltas, float **dense0, float **taps, int64_t *counts,
                  uint8_t *in_mask, float *in_delta) {
    return orc_run_chunk_follow(L, n, in_h, in_w, in_c, Lf, frames, thresholds, layer_outer, masks, deltas,
                                dense0, taps, counts, in_mask, in_delta, NULL);
}
