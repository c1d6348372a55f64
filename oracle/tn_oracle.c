/*
 * tn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU statement of what the TernaryNet
 * inference hot path computes (Heinrich, Blendowski, Oktay, arXiv 1801.09449;
 * cited as PAPER.md:<line> with the section / equation it falls in).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library.  It shares no code, header, table or constant
 * generator with the CUDA path (paper_1801_09449_b200/) and neither side
 * imports the other.  Inputs come from synth/ (random numbers only).
 *
 * Representation: ternary tensors are int8 codes in {-1,0,+1} in PyTorch's
 * NCDHW order (deliberately NOT the GPU's channel-last bit-packed layout).
 * The convolution is the plain definition of a cross-correlation with zero
 * padding, summed as acc += w*a in int32.  Eq. 9's popcount identity is NOT
 * used here: the method reaches exactly (no rounding) the integer dot product
 * of the codes, so the oracle is that dot product written out.  The one
 * bit-level function is oracle_pack, written independently so that packed
 * bytes can be compared byte for byte.
 *
 * Every function pinned by tests/test_oracle_*.py (brute force against
 * torch float64, closed forms, worked examples, exhaustive tables).  See
 * DESIGN.md "Oracle pins".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX5(a, b, c, d, e, B, C, D, E) \
    (((((int64_t)(a) * (B) + (b)) * (C) + (c)) * (D) + (d)) * (E) + (e))

/* ------------------------------------------------------------------------- */
/* Eq. 6 hard ternarisation of the float input (Eq. 6) with  */
/* the zero-mean/unit-variance normalisation of PAPER.md:180 folded into the */
/* float thresholds t_lo = mu - 0.5 sigma, t_hi = mu + 0.5 sigma (DESIGN.md  */
/* reading R7).  +1 if x > t_hi; -1 if x < t_lo; 0 otherwise (closed band,   */
/* |x| <= 0.5 -> 0).  Returns the first flat index holding NaN/Inf, else -1. */
/* ------------------------------------------------------------------------- */
int64_t oracle_tern_f32(const float* x, int64_t count, float t_lo, float t_hi, int8_t* t)
{
    int64_t bad = -1;
    for (int64_t i = 0; i < count; ++i) {
        float v = x[i];
        if (!isfinite(v)) {
            if (bad < 0) bad = i;
            t[i] = 0;
            continue;
        }
        if (v > t_hi)      t[i] = 1;
        else if (v < t_lo) t[i] = -1;
        else               t[i] = 0;
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* 2-bit encoding ("2 bits per entry that encode the sign and   */
/* value"; Fig. 3 caption PAPER.md:130).  Reading R2: mask bit = 1 <=> the   */
/* entry is nonzero, sign bit = 1 <=> the entry is +1, zero = (0,0).         */
/* Reading R3: 32-bit little-endian words, channel c -> bit (c % 32) of word */
/* (c / 32); per voxel the CW sign words come first, then the CW mask words; */
/* voxels in N,D,H,W order (channel-last).  Padding lanes are zero.          */
/* x is int8 NCDHW; xp is uint32 [n][d][h][w][2][cw].  Returns the first     */
/* flat NCDHW index whose code is outside {-1,0,+1}, else -1.                */
/* ------------------------------------------------------------------------- */
int64_t oracle_pack(const int8_t* x, int n, int c, int d, int h, int w, uint32_t* xp)
{
    int cw = (c + 31) / 32;
    int64_t bad = -1;
    for (int in = 0; in < n; ++in)
    for (int z = 0; z < d; ++z)
    for (int y = 0; y < h; ++y)
    for (int xx = 0; xx < w; ++xx) {
        int64_t vox = (((int64_t)in * d + z) * h + y) * w + xx;
        uint32_t* sign = xp + vox * 2 * cw;
        uint32_t* mask = sign + cw;
        for (int j = 0; j < cw; ++j) { sign[j] = 0; mask[j] = 0; }
        for (int ch = 0; ch < c; ++ch) {
            int64_t src = IDX5(in, ch, z, y, xx, c, d, h, w);
            int8_t v = x[src];
            if (v != -1 && v != 0 && v != 1) {
                if (bad < 0 || src < bad) bad = src;
                continue;
            }
            uint32_t bit = 1u << (ch % 32);
            if (v != 0) mask[ch / 32] |= bit;
            if (v == 1) sign[ch / 32] |= bit;
        }
    }
    return bad;
}

/* Inverse of oracle_pack.  Returns the first flat NCDHW index whose bits are */
/* not canonical (sign set on a zero), or the first padding lane  */
/* that is set (reported as the voxel's flat index of channel c), else -1.    */
int64_t oracle_unpack(const uint32_t* xp, int n, int c, int d, int h, int w, int8_t* x)
{
    int cw = (c + 31) / 32;
    int64_t bad = -1;
    for (int in = 0; in < n; ++in)
    for (int z = 0; z < d; ++z)
    for (int y = 0; y < h; ++y)
    for (int xx = 0; xx < w; ++xx) {
        int64_t vox = (((int64_t)in * d + z) * h + y) * w + xx;
        const uint32_t* sign = xp + vox * 2 * cw;
        const uint32_t* mask = sign + cw;
        for (int lane = 0; lane < cw * 32; ++lane) {
            int s = (sign[lane / 32] >> (lane % 32)) & 1;
            int m = (mask[lane / 32] >> (lane % 32)) & 1;
            if (lane >= c) {
                if (s || m) {
                    int64_t at = IDX5(in, c - 1, z, y, xx, c, d, h, w);
                    if (bad < 0 || at < bad) bad = at;
                }
                continue;
            }
            int64_t dst = IDX5(in, lane, z, y, xx, c, d, h, w);
            if (s && !m) {
                if (bad < 0 || dst < bad) bad = dst;
                x[dst] = 0;
                continue;
            }
            x[dst] = (int8_t)(m ? (s ? 1 : -1) : 0);
        }
    }
    return bad;
}

/* Weights: int8 [k][c][3][3][3] -> packed [k][27][2][cw], tap t = (dz*3+dy)*3+dx. */
int64_t oracle_pack_weights(const int8_t* wt, int k, int c, uint32_t* wp)
{
    int cw = (c + 31) / 32;
    int64_t bad = -1;
    for (int ko = 0; ko < k; ++ko)
    for (int t = 0; t < 27; ++t) {
        uint32_t* sign = wp + ((int64_t)ko * 27 + t) * 2 * cw;
        uint32_t* mask = sign + cw;
        for (int j = 0; j < cw; ++j) { sign[j] = 0; mask[j] = 0; }
        for (int ch = 0; ch < c; ++ch) {
            int64_t src = ((int64_t)ko * c + ch) * 27 + t;
            int8_t v = wt[src];
            if (v != -1 && v != 0 && v != 1) {
                if (bad < 0 || src < bad) bad = src;
                continue;
            }
            uint32_t bit = 1u << (ch % 32);
            if (v != 0) mask[ch / 32] |= bit;
            if (v == 1) sign[ch / 32] |= bit;
        }
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Ternary 3x3x3 convolution ("inner products of an input       */
/* tensor I and a filter bank W"; Eq. 9 PAPER.md:118-123 computes exactly    */
/* this integer sum; dilation PAPER.md:135).  PyTorch cross-correlation      */
/* semantics with zero padding:                                              */
/*   y[n][k][zo][yo][xo] = sum_c sum_{a,b,e in 0..2} w[k][c][a][b][e] *      */
/*        x[n][c][zo*s - p + a*dil][yo*s - p + b*dil][xo*s - p + e*dil]      */
/* Output extent per axis: (D + 2p - 2*dil - 1) / s + 1.                     */
/* g = {sz, sy, sx, pz, py, px, dilz, dily, dilx}.  y is int32 NCDHW.        */
/* ------------------------------------------------------------------------- */
static int out_extent(int len, int s, int p, int dil)
{
    int span = len + 2 * p - 2 * dil - 1;   /* last valid window start */
    if (span < 0) return 0;
    return span / s + 1;
}

static int32_t conv_one(const int8_t* x, int c, int d, int h, int w,
                        const int8_t* wt, const int* g, int in, int ko, int zo, int yo, int xo)
{
    int32_t acc = 0;
    for (int ch = 0; ch < c; ++ch)
    for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
    for (int e = 0; e < 3; ++e) {
        int zi = zo * g[0] - g[3] + a * g[6];
        int yi = yo * g[1] - g[4] + b * g[7];
        int xi = xo * g[2] - g[5] + e * g[8];
        if (zi < 0 || zi >= d || yi < 0 || yi >= h || xi < 0 || xi >= w) continue; /* zero padding */
        int32_t wv = wt[(((int64_t)ko * c + ch) * 3 + a) * 9 + b * 3 + e];
        int32_t av = x[IDX5(in, ch, zi, yi, xi, c, d, h, w)];
        acc += wv * av;
    }
    return acc;
}

void oracle_conv3d(const int8_t* x, int n, int c, int d, int h, int w,
                   const int8_t* wt, int k, const int* g, int32_t* y)
{
    int dout = out_extent(d, g[0], g[3], g[6]);
    int hout = out_extent(h, g[1], g[4], g[7]);
    int wout = out_extent(w, g[2], g[5], g[8]);
    if (dout <= 0 || hout <= 0 || wout <= 0) return;
    int64_t jobs = (int64_t)n * k * dout;
    #pragma omp parallel for schedule(dynamic)
    for (int64_t job = 0; job < jobs; ++job) {
        int in = (int)(job / ((int64_t)k * dout));
        int ko = (int)((job / dout) % k);
        int zo = (int)(job % dout);
        for (int yo = 0; yo < hout; ++yo)
        for (int xo = 0; xo < wout; ++xo)
            y[IDX5(in, ko, zo, yo, xo, k, dout, hout, wout)] =
                conv_one(x, c, d, h, w, wt, g, in, ko, zo, yo, xo);
    }
}

/* Same sum at sampled output coordinates: at[i] = {n, k, zo, yo, xo}. */
void oracle_conv3d_at(const int8_t* x, int n, int c, int d, int h, int w,
                      const int8_t* wt, int k, const int* g,
                      const int32_t* at, int64_t count, int32_t* out)
{
    (void)n; (void)k;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const int32_t* q = at + 5 * i;
        out[i] = conv_one(x, c, d, h, w, wt, g, q[0], q[1], q[2], q[3], q[4]);
    }
}

/* ------------------------------------------------------------------------- */
/* Requantisation between layers ("The output is batch          */
/* normalised and passed on to the nonlinearity"; PAPER.md:135 hard          */
/* quantisation at inference; Eq. 6).  The per-channel scale  */
/* alpha, batch norm and Eq. 6's +-0.5 band fold into integer  */
/* thresholds (reading R5/R6):                                               */
/*   t = +1 if acc >= hi[k]; else -1 if acc <= lo[k]; else 0                 */
/* evaluated in that order.  acc is int32 [n][k][dhw], t int8 same shape.    */
/* ------------------------------------------------------------------------- */
void oracle_requant(const int32_t* acc, int n, int k, int64_t dhw,
                    const int32_t* lo, const int32_t* hi, int8_t* t)
{
    for (int in = 0; in < n; ++in)
    for (int ko = 0; ko < k; ++ko)
    for (int64_t v = 0; v < dhw; ++v) {
        int64_t i = ((int64_t)in * k + ko) * dhw + v;
        int32_t a = acc[i];
        if (a >= hi[ko])      t[i] = 1;
        else if (a <= lo[ko]) t[i] = -1;
        else                  t[i] = 0;
    }
}

/* Nearest-neighbour x2 upsampling ("Upsample2D 2x2";  */
/* reading R10): y[n][c][z][yy][x] = x[n][c][z/2][yy/2][x/2].               */
void oracle_upsample2(const int8_t* x, int n, int c, int d, int h, int w, int8_t* y)
{
    int d2 = 2 * d, h2 = 2 * h, w2 = 2 * w;
    for (int in = 0; in < n; ++in)
    for (int ch = 0; ch < c; ++ch)
    for (int z = 0; z < d2; ++z)
    for (int yy = 0; yy < h2; ++yy)
    for (int xx = 0; xx < w2; ++xx)
        y[IDX5(in, ch, z, yy, xx, c, d2, h2, w2)] = x[IDX5(in, ch, z / 2, yy / 2, xx / 2, c, d, h, w)];
}

/* Upsample2D of Table 1 (the 2D decoder's 2x2     */
/* upsampling; reading R18): nearest x2 in y and x only, planes unchanged.    */
void oracle_upsample2_yx(const int8_t* x, int n, int c, int d, int h, int w, int8_t* y)
{
    int h2 = 2 * h, w2 = 2 * w;
    for (int in = 0; in < n; ++in)
    for (int ch = 0; ch < c; ++ch)
    for (int z = 0; z < d; ++z)
    for (int yy = 0; yy < h2; ++yy)
    for (int xx = 0; xx < w2; ++xx)
        y[IDX5(in, ch, z, yy, xx, c, d, h2, w2)] = x[IDX5(in, ch, z, yy / 2, xx / 2, c, d, h, w)];
}

/* Channel concatenation [a, b] ("skip connections ... dense   */
/* feature concatenation"; Table 1 skip column PAPER.md:154-171).           */
void oracle_concat(const int8_t* a, int ca, const int8_t* b, int cb, int n, int64_t dhw, int8_t* y)
{
    for (int in = 0; in < n; ++in) {
        memcpy(y + (int64_t)in * (ca + cb) * dhw, a + (int64_t)in * ca * dhw, (size_t)(ca * dhw));
        memcpy(y + ((int64_t)in * (ca + cb) + ca) * dhw, b + (int64_t)in * cb * dhw, (size_t)(cb * dhw));
    }
}

/* Prediction layer ("hyperbolic tangents (except for the final */
/* prediction layer)"; Table 1 "Prediction ... 2" PAPER.md:173; reading R12: */
/* 1x1x1, float weights/bias).  logits[n][j][v] = b[j] + sum_c w[j][c]*t,    */
/* summed in double and rounded once to float.                               */
void oracle_predict(const int8_t* t, int n, int c, int64_t dhw, int nclass,
                    const float* w, const float* b, float* logits)
{
    for (int in = 0; in < n; ++in)
    for (int j = 0; j < nclass; ++j)
    for (int64_t v = 0; v < dhw; ++v) {
        double s = (double)b[j];
        for (int ch = 0; ch < c; ++ch)
            s += (double)w[j * c + ch] * (double)t[((int64_t)in * c + ch) * dhw + v];
        logits[((int64_t)in * nclass + j) * dhw + v] = (float)s;
    }
}

/* ------------------------------------------------------------------------- */
/* The ternary FCN (reading R9: the Table-1 analogue of PAPER.md:143-176 in  */
/* 3D with channels 16-32-64-64, stride-2 convolutions in place of AvgPool   */
/* (reading R8), nearest x2 upsampling (R10), concat order [upsampled, skip],*/
/* 1x1x1 float prediction (R12)).  This is the oracle's own statement of the */
/* table; it is not shared with the GPU path.                                */
/*   #1  1->16  R0            #8  64->64 R3                                  */
/*   #2 16->16  R0 [skip #13] #9  [up(#8) 64 | #6 64] -> 64 R2               */
/*   #3 16->16  s2 -> R1      #10 64->32 R2                                  */
/*   #4 16->32  R1 [skip #11] #11 [up(#10) 32 | #4 32] -> 32 R1              */
/*   #5 32->32  s2 -> R2      #12 32->16 R1                                  */
/*   #6 32->64  R2 [skip #9]  #13 [up(#12) 16 | #2 16] -> 16 R0              */
/*   #7 64->64  s2 -> R3      #14 16->16 R0     pred 16 -> 2                 */
/* All convs 3x3x3, pad 1, dilation 1.  W[i] is int8 [cout][cin][3][3][3],   */
/* lo[i]/hi[i] int32 [cout].  x is float [n][1][d][h][w]; d,h,w divisible by */
/* 8.  logits float [n][2][d][h][w].  acts (optional, may be NULL): 14       */
/* caller buffers receiving each layer's int8 NCDHW codes.  Returns the      */
/* first non-finite input index, else -1.                                    */
/* ------------------------------------------------------------------------- */
typedef struct { int cin, cout, stride; } ofcn_layer;

static const ofcn_layer OFCN[14] = {
    {1, 16, 1}, {16, 16, 1}, {16, 16, 2}, {16, 32, 1}, {32, 32, 2}, {32, 64, 1}, {64, 64, 2},
    {64, 64, 1}, {128, 64, 1}, {64, 32, 1}, {64, 32, 1}, {32, 16, 1}, {32, 16, 1}, {16, 16, 1},
};

static int8_t* conv_block(const int8_t* in, int n, int c, int d, int h, int w,
                          const int8_t* wt, int k, int s, const int32_t* lo, const int32_t* hi,
                          int* od, int* oh, int* ow)
{
    int g[9] = {s, s, s, 1, 1, 1, 1, 1, 1};
    *od = out_extent(d, s, 1, 1);
    *oh = out_extent(h, s, 1, 1);
    *ow = out_extent(w, s, 1, 1);
    int64_t dhw = (int64_t)(*od) * (*oh) * (*ow);
    int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * k * dhw));
    int8_t* out = (int8_t*)malloc((size_t)(n * k * dhw));
    oracle_conv3d(in, n, c, d, h, w, wt, k, g, acc);
    oracle_requant(acc, n, k, dhw, lo, hi, out);
    free(acc);
    return out;
}

static int8_t* up_cat(const int8_t* low, int cl, const int8_t* skip, int cs, int n, int d, int h, int w)
{
    /* d,h,w: the low-resolution extents */
    int64_t dhw2 = (int64_t)8 * d * h * w;
    int8_t* up = (int8_t*)malloc((size_t)(n * cl * dhw2));
    int8_t* cat = (int8_t*)malloc((size_t)(n * (cl + cs) * dhw2));
    oracle_upsample2(low, n, cl, d, h, w, up);
    oracle_concat(up, cl, skip, cs, n, dhw2, cat);
    free(up);
    return cat;
}

int64_t oracle_fcn_forward(const float* x, int n, int d, int h, int w, float t_lo, float t_hi,
                           const int8_t* const* W, const int32_t* const* lo, const int32_t* const* hi,
                           const float* pred_w, const float* pred_b, float* logits, int8_t* const* acts)
{
    int64_t v0 = (int64_t)n * d * h * w;
    int8_t* t0 = (int8_t*)malloc((size_t)v0);
    int64_t bad = oracle_tern_f32(x, v0, t_lo, t_hi, t0);

    int8_t* a[15] = {0};
    int dd[15], hh[15], ww[15];
    int od, oh, ow;
    /* encoder */
    a[1] = conv_block(t0, n, 1, d, h, w, W[0], 16, 1, lo[0], hi[0], &od, &oh, &ow);
    dd[1] = od; hh[1] = oh; ww[1] = ow;
    for (int i = 2; i <= 8; ++i) {
        const ofcn_layer* L = &OFCN[i - 1];
        a[i] = conv_block(a[i - 1], n, L->cin, dd[i - 1], hh[i - 1], ww[i - 1], W[i - 1], L->cout,
                          L->stride, lo[i - 1], hi[i - 1], &od, &oh, &ow);
        dd[i] = od; hh[i] = oh; ww[i] = ow;
    }
    /* decoder: (layer, low-res source, skip source) */
    const int dec[3][2] = {{8, 6}, {10, 4}, {12, 2}};
    for (int j = 0; j < 3; ++j) {
        int i = 9 + 2 * j;
        int low = dec[j][0], skip = dec[j][1];
        const ofcn_layer* L = &OFCN[i - 1];
        int cl = OFCN[low - 1].cout, cs = OFCN[skip - 1].cout;
        int8_t* cat = up_cat(a[low], cl, a[skip], cs, n, dd[low], hh[low], ww[low]);
        a[i] = conv_block(cat, n, cl + cs, dd[skip], hh[skip], ww[skip], W[i - 1], L->cout, 1,
                          lo[i - 1], hi[i - 1], &od, &oh, &ow);
        dd[i] = od; hh[i] = oh; ww[i] = ow;
        free(cat);
        const ofcn_layer* L2 = &OFCN[i];
        a[i + 1] = conv_block(a[i], n, L2->cin, dd[i], hh[i], ww[i], W[i], L2->cout, 1,
                              lo[i], hi[i], &od, &oh, &ow);
        dd[i + 1] = od; hh[i + 1] = oh; ww[i + 1] = ow;
    }
    oracle_predict(a[14], n, 16, (int64_t)dd[14] * hh[14] * ww[14], 2, pred_w, pred_b, logits);

    for (int i = 1; i <= 14; ++i) {
        if (acts && acts[i - 1]) {
            int64_t bytes = (int64_t)n * OFCN[i - 1].cout * dd[i] * hh[i] * ww[i];
            memcpy(acts[i - 1], a[i], (size_t)bytes);
        }
        free(a[i]);
    }
    free(t0);
    return bad;
}

/* Number of threads the OpenMP runtime will use (reported by bench.py). */
int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
