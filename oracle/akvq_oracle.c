/*
 * akvq_oracle.c -- plain, slow, obviously-correct CPU oracle of the AKVQ-VL
 * hot path (arXiv 2501.15021).  TEST INFRASTRUCTURE: see akvq_oracle.h for
 * who may use it.  Shares nothing with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fPIC -shared
 *        (no -ffast-math: the fp32 decisions must be plain IEEE single ops;
 *         -ffp-contract=off forbids fusing a*b+c into an FMA).
 *
 * The method, in the paper's order:
 *  1. Walsh-Hadamard matrix (Eq. 7) and the equivalent
 *     transformation of Q/K after RoPE (Fig. 6) and of V/O
 *     (Fig. 7; applied online here, R4).
 *  2. Salient tokens: text tokens in TSA layers, pivot tokens in
 *     PSA layers (top-k over accumulated attention column sums per
 *     north_star BJ:5, R2), recent tokens always.
 *  3. Pivot + recent tokens at the original 16-bit precision, text tokens at
 *     4 bits, the rest at 2 bits, with Eqs. 3-6 and
 *     clip ratios 0.8 / 1.0, group size G.  K per channel
 *     over G-token blocks, V per token over G-channel groups (BJ:5, R1).
 *  4. Decode attention over the cache (Eq. 2 "update the KV cache", P:112-119;
 *     softmax(q K^T / sqrt d) V), computed as the plain definition on
 *     the dequantized view.
 */
#include "akvq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

struct orc_cache {
  orc_config cfg;
  int cap;        /* capacity rounded up to a multiple of G              */
  int side_cap;   /* PSA: top_k; TSA: cap                                 */
  int L, nq;      /* tokens stored; tokens in the quantized region        */
  double *H;      /* normalized Walsh-Hadamard matrix, d x d (Eq. 7)      */
  double *Hs;     /* +-1 Walsh-Hadamard matrix H_s = sqrt(d) H            */
  uint16_t *K, *V;      /* [U][cap][d] original 16-bit rows, every token  */
  uint8_t *sal;         /* [U][cap] salient flag                           */
  double *xk, *xv;      /* [U][cap][d] K.H_s, V.H_s decision inputs: fp64, or
                           rounded once to fp32 in the fp32-decision mode  */
  uint8_t *kc, *vc;     /* [U][cap][d] unpacked 2-bit codes                */
  double *ks;           /* [U][cap/G][d] K scale (unnormalized units)      */
  int32_t *kz;          /* [U][cap/G][d] K zero point                      */
  double *kzp;          /* [U][cap/G][d] clipped_min / scale before rounding */
  double *vs;           /* [U][cap][d/G] V scale (unnormalized units)      */
  int32_t *vz;          /* [U][cap][d/G] V zero point                      */
  double *vzp;          /* [U][cap][d/G] clipped_min / scale before rounding */
  int32_t *side_idx;    /* [U][side_cap] token index of each side entry    */
  int32_t *side_cnt;    /* [U]                                             */
  int32_t *side_pos;    /* [U][cap] side entry of token t (or -1)          */
  uint8_t *s4c;         /* [U][side_cap][2][d] unpacked 4-bit codes (TSA)  */
  double *s4s;          /* [U][side_cap][2][d/G]                           */
  int32_t *s4z;         /* [U][side_cap][2][d/G]                           */
  double *s4zp;         /* [U][side_cap][2][d/G]                           */
};

static int is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

/* ------------------------------------------------------------------ */
/* Eq. 7: H_1 = [1];                                        */
/*   H_{2^k} = (1/sqrt 2) [[H_{2^(k-1)},  H_{2^(k-1)}],                 */
/*                         [H_{2^(k-1)}, -H_{2^(k-1)}]].                */
/* Built literally by the recursion, one doubling at a time.            */
int orc_hadamard(int d, int normalized, double *H) {
  if (!is_pow2(d)) return ORC_EINVAL;
  const double f = normalized ? 1.0 / sqrt(2.0) : 1.0;
  H[0] = 1.0;                                   /* H_1 = [1] */
  for (int n = 1; n < d; n *= 2) {              /* H_n -> H_2n, in place */
    /* copy H_n (stored with row stride d) into the four quadrants,
     * bottom-right negated; go from the last row up so the top-left
     * quadrant is read before it is overwritten. */
    for (int i = n - 1; i >= 0; --i) {
      for (int j = n - 1; j >= 0; --j) {
        const double h = H[i * d + j];
        H[i * d + j] = f * h;
        H[i * d + j + n] = f * h;
        H[(i + n) * d + j] = f * h;
        H[(i + n) * d + j + n] = -f * h;
      }
    }
  }
  return ORC_OK;
}

/* y = x . H  (explicit vector-matrix product in fp64). */
int orc_rotate(int d, int normalized, const double *x, double *y) {
  if (!is_pow2(d)) return ORC_EINVAL;
  double *H = (double *)malloc(sizeof(double) * d * d);
  orc_hadamard(d, normalized, H);
  for (int j = 0; j < d; ++j) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += x[i] * H[i * d + j];
    y[j] = s;
  }
  free(H);
  return ORC_OK;
}

static void matvec(int d, const double *H, const double *x, double *y) {
  for (int j = 0; j < d; ++j) {
    double s = 0.0;
    for (int i = 0; i < d; ++i) s += x[i] * H[i * d + j];
    y[j] = s;
  }
}

/* ------------------------------------------------------------------ */
/* 16-bit inputs are widened exactly.                                   */
double orc_half_to_double(uint16_t h, int dtype16) {
  if (dtype16 == ORC_BF16) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
  }
  /* IEEE binary16: 1 sign, 5 exponent (bias 15), 10 mantissa bits. */
  const int s = (h >> 15) & 1, e = (h >> 10) & 0x1f, m = h & 0x3ff;
  double v;
  if (e == 0) v = ldexp((double)m, -24);                 /* subnormal */
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = ldexp((double)(m | 0x400), e - 25);           /* 1.m * 2^(e-15) */
  return s ? -v : v;
}

/* ------------------------------------------------------------------ */
/* Eqs. 3, 5, 6 on one group of n elements (stride apart).  */
/*   clipped_max = clip * max, clipped_min = clip * min   (R3)   */
/*   scale = (clipped_max - clipped_min) / (2^n - 1)           Eq. 5    */
/*   zero  = -round(clipped_min / scale)                       Eq. 6    */
/*   Q(X)  = clamp(round(X / scale) + zero, 0, 2^n - 1)        Eq. 3    */
/* round = round-half-to-even (R7).  Degenerate group (clipped range <  */
/* 1e-12): scale = the constant, zero 0, codes 1 (R8).  Empty    */
/* group (all elements skipped): scale 0, zero 0, codes 0 (R8).         */
/* Skipped (salient) elements get code 0.                                */
/* Two decision precisions (R6): fp64 (the default of the cache, SURVEY  */
/* 8(c)) and IEEE fp32 (the kernel's precision, used as a second,        */
/* bit-exact cross-check).  The clip ratio is the fp32 constant widened  */
/* exactly in both.  zpre receives clipped_min / scale before rounding   */
/* (the zero-point tie test of the parity checker).                      */
static int32_t zero_to_i32(double zf) {
  if (zf > 2147483647.0) return 2147483647;
  if (zf < -2147483648.0) return (int32_t)0x80000000u;
  return (int32_t)zf;
}

static void qgroup64(const double *x, const uint8_t *skip, int n, int stride, int bits,
                     double clip, double *scale, int32_t *zero, double *zpre,
                     uint8_t *codes, int code_stride) {
  const int levels = (1 << bits) - 1;
  int any = 0;
  double mx = 0.0, mn = 0.0;
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) continue;
    const double v = x[(long)i * stride];
    if (!any) { mx = v; mn = v; any = 1; }
    else { if (v > mx) mx = v; if (v < mn) mn = v; }
  }
  *zpre = NAN;                               /* no rounding decision      */
  if (!any) {
    *scale = 0.0; *zero = 0;
    for (int i = 0; i < n; ++i) codes[(long)i * code_stride] = 0;
    return;
  }
  const double cmx = clip * mx;              /* clipped_max(X) */
  const double cmn = clip * mn;              /* clipped_min(X) */
  const double range = cmx - cmn;
  if (range < 1e-12) {                       /* degenerate constant group */
    *scale = mx; *zero = 0;
    for (int i = 0; i < n; ++i)
      codes[(long)i * code_stride] = (skip && skip[i]) ? 0 : 1;
    return;
  }
  const double s = range / (double)levels;   /* Eq. 5 */
  *zpre = cmn / s;
  const double zf = -rint(cmn / s);          /* Eq. 6 */
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) { codes[(long)i * code_stride] = 0; continue; }
    double q = rint(x[(long)i * stride] / s) + zf;               /* Eq. 3 */
    if (q < 0.0) q = 0.0;
    if (q > (double)levels) q = (double)levels;
    codes[(long)i * code_stride] = (uint8_t)q;
  }
  *scale = s;
  *zero = zero_to_i32(zf);
}

/* The same steps with every operation an IEEE fp32 operation (R6). */
static void qgroup32(const double *x, const uint8_t *skip, int n, int stride, int bits,
                     float clip, double *scale, int32_t *zero, double *zpre,
                     uint8_t *codes, int code_stride) {
  const int levels = (1 << bits) - 1;
  int any = 0;
  float mx = 0.0f, mn = 0.0f;
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) continue;
    const float v = (float)x[(long)i * stride];
    if (!any) { mx = v; mn = v; any = 1; }
    else { if (v > mx) mx = v; if (v < mn) mn = v; }
  }
  *zpre = NAN;                               /* no rounding decision      */
  if (!any) {
    *scale = 0.0; *zero = 0;
    for (int i = 0; i < n; ++i) codes[(long)i * code_stride] = 0;
    return;
  }
  const float cmx = clip * mx;               /* clipped_max(X) */
  const float cmn = clip * mn;               /* clipped_min(X) */
  const float range = cmx - cmn;
  if (range < 1e-12f) {                      /* degenerate constant group */
    *scale = mx; *zero = 0;
    for (int i = 0; i < n; ++i)
      codes[(long)i * code_stride] = (skip && skip[i]) ? 0 : 1;
    return;
  }
  const float s = range / (float)levels;     /* Eq. 5 */
  const float zq = cmn / s;
  *zpre = zq;
  const float zf = -rintf(zq);               /* Eq. 6 */
  for (int i = 0; i < n; ++i) {
    if (skip && skip[i]) { codes[(long)i * code_stride] = 0; continue; }
    const float r = rintf((float)x[(long)i * stride] / s);      /* Eq. 3 */
    double q = (double)r + (double)zf;
    if (q < 0.0) q = 0.0;
    if (q > (double)levels) q = (double)levels;
    codes[(long)i * code_stride] = (uint8_t)q;
  }
  *scale = s;
  *zero = zero_to_i32(zf);
}

static void qgroup(int decide64, const double *x, const uint8_t *skip, int n, int stride,
                   int bits, float clip, double *scale, int32_t *zero, double *zpre,
                   uint8_t *codes, int code_stride) {
  if (decide64)
    qgroup64(x, skip, n, stride, bits, (double)clip, scale, zero, zpre, codes, code_stride);
  else
    qgroup32(x, skip, n, stride, bits, clip, scale, zero, zpre, codes, code_stride);
}

void orc_quantize_group(const float *x, const uint8_t *skip, int n, int stride,
                        int bits, float clip, float *scale, int32_t *zero,
                        uint8_t *codes, int code_stride) {
  double *xd = (double *)malloc(sizeof(double) * (n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) xd[i] = (double)x[(long)i * stride];
  double s, zp;
  qgroup32(xd, skip, n, 1, bits, clip, &s, zero, &zp, codes, code_stride);
  *scale = (float)s;
  free(xd);
}

void orc_quantize_group64(const double *x, const uint8_t *skip, int n, int bits, float clip,
                          double *scale, int32_t *zero, double *zpre, uint8_t *codes) {
  qgroup64(x, skip, n, 1, bits, (double)clip, scale, zero, zpre, codes, 1);
}

/* 2-bit code i -> bits [2(i mod 4), 2(i mod 4)+1] of byte i/4;
 *        4-bit code i -> low nibble of byte i/2 if i even, else high.   */
void orc_pack(const uint8_t *codes, int n, int bits, uint8_t *out) {
  const int per = 8 / bits;
  memset(out, 0, (size_t)((n + per - 1) / per));
  for (int i = 0; i < n; ++i)
    out[i / per] |= (uint8_t)((codes[i] & ((1 << bits) - 1)) << (bits * (i % per)));
}
void orc_unpack(const uint8_t *in, int n, int bits, uint8_t *codes) {
  const int per = 8 / bits;
  for (int i = 0; i < n; ++i)
    codes[i] = (in[i / per] >> (bits * (i % per))) & ((1 << bits) - 1);
}

/* ------------------------------------------------------------------ */
/* Salient-token selection for one unit (BJ:5, R2).          */
/*  TSA: salient = text tokens (type 1).                                */
/*  PSA: score_t = sum_{j<g} colsum[j][t] (fp32, j ascending: R6), the   */
/*       min(top_k, L0) tokens first in the order (score desc, t asc).   */
static const float *g_sort_scores;
static int cmp_desc_score_asc_idx(const void *a, const void *b) {
  const int i = *(const int *)a, j = *(const int *)b;
  const float si = g_sort_scores[i], sj = g_sort_scores[j];
  if (si > sj) return -1;
  if (si < sj) return 1;
  return (i > j) - (i < j);
}
void orc_select_salient(int kind, int g, int L0, int top_k,
                        const uint8_t *types, const float *colsum,
                        uint8_t *salient) {
  memset(salient, 0, (size_t)L0);
  if (kind == ORC_TSA) {
    for (int t = 0; t < L0; ++t) salient[t] = types[t] == 1;
    return;
  }
  if (L0 <= 0) return;
  float *score = (float *)malloc(sizeof(float) * L0);
  int *order = (int *)malloc(sizeof(int) * L0);
  for (int t = 0; t < L0; ++t) {
    float s = 0.0f;
    for (int j = 0; j < g; ++j) s += colsum[(long)j * L0 + t];
    score[t] = s;
    order[t] = t;
  }
  /* a library sort is a permitted step; qsort is not reentrant-safe with
   * the global, so this runs under a critical section when threaded. */
#ifdef _OPENMP
#pragma omp critical(orc_sort)
#endif
  {
    g_sort_scores = score;
    qsort(order, (size_t)L0, sizeof(int), cmp_desc_score_asc_idx);
  }
  const int k = top_k < L0 ? top_k : L0;
  for (int r = 0; r < k; ++r) salient[order[r]] = 1;
  free(score);
  free(order);
}

/* ------------------------------------------------------------------ */
/* Massive-activation pivot detection (SPEC S:317-321,        */
/* SURVEY NEXT-2) for one residual stream [L0][hidden] (16-bit):         */
/*   score(t) = max_c |residual[t][c]|            (exact, stored fp32)   */
/*   m = median over tokens of score: the middle value for odd L0, the   */
/*       fp32 mean (a + b) * 0.5 of the two middle values for even L0    */
/*       (R22)                                                 */
/*   pivots = tokens with score > tau * m (fp32 product, R6), ordered by */
/*       (score desc, index asc), truncated to n_max; none -> [0].       */
static int cmp_float_asc(const void *a, const void *b) {
  const float x = *(const float *)a, y = *(const float *)b;
  return (x > y) - (x < y);
}
int orc_detect_pivots(int L0, int hidden, const uint16_t *residual, int dtype16, float tau,
                      int n_max, int32_t *out) {
  if (L0 <= 0 || hidden <= 0 || n_max <= 0) return 0;
  float *score = (float *)malloc(sizeof(float) * L0);
  float *sorted = (float *)malloc(sizeof(float) * L0);
  int *order = (int *)malloc(sizeof(int) * L0);
  for (int t = 0; t < L0; ++t) {
    double mx = 0.0;
    for (int c = 0; c < hidden; ++c) {
      const double a = fabs(orc_half_to_double(residual[(long)t * hidden + c], dtype16));
      if (a > mx) mx = a;
    }
    score[t] = (float)mx;                 /* exact: |16-bit| fits fp32 */
    sorted[t] = score[t];
  }
  qsort(sorted, (size_t)L0, sizeof(float), cmp_float_asc);
  const float m = (L0 & 1) ? sorted[L0 / 2] : (sorted[L0 / 2 - 1] + sorted[L0 / 2]) * 0.5f;
  const float thr = tau * m;
  int n = 0;
  for (int t = 0; t < L0; ++t)
    if (score[t] > thr) order[n++] = t;
#ifdef _OPENMP
#pragma omp critical(orc_sort)
#endif
  {
    g_sort_scores = score;
    qsort(order, (size_t)n, sizeof(int), cmp_desc_score_asc_idx);
  }
  if (n > n_max) n = n_max;
  for (int i = 0; i < n; ++i) out[i] = order[i];
  if (n == 0) { out[0] = 0; n = 1; }      /* attention-sink fallback */
  free(score); free(sorted); free(order);
  return n;
}

/* ------------------------------------------------------------------ */
static long ROW(const orc_cache *c, int u, int t) {
  return ((long)u * c->cap + t) * c->cfg.d;
}

orc_cache *orc_new(const orc_config *cfg, int *status) {
  const int d = cfg->d, G = cfg->G;
  if (!is_pow2(d) || d > 512 || !is_pow2(G) || G > d || cfg->U < 1 || cfg->g < 1 ||
      cfg->R < 0 || cfg->capacity < 1 || cfg->top_k < 0 ||
      !(cfg->clip2 > 0.0f && cfg->clip2 <= 1.0f) ||
      !(cfg->clip4 > 0.0f && cfg->clip4 <= 1.0f) ||
      (cfg->kind != ORC_TSA && cfg->kind != ORC_PSA) ||
      (cfg->k_axis != 0 && cfg->k_axis != 1) ||
      (cfg->decide64 != 0 && cfg->decide64 != 1) ||
      (cfg->exact_r != 0 && cfg->exact_r != 1) || (cfg->exact_r && cfg->k_axis != 1)) {
    if (status) *status = ORC_EINVAL;
    return NULL;
  }
  orc_cache *c = (orc_cache *)calloc(1, sizeof(orc_cache));
  c->cfg = *cfg;
  c->cap = (cfg->capacity + G - 1) / G * G;
  c->side_cap = cfg->kind == ORC_PSA ? cfg->top_k : c->cap;
  const long U = cfg->U, cap = c->cap, sc = c->side_cap > 0 ? c->side_cap : 1;
  c->H = (double *)malloc(sizeof(double) * d * d);
  c->Hs = (double *)malloc(sizeof(double) * d * d);
  orc_hadamard(d, 1, c->H);
  orc_hadamard(d, 0, c->Hs);
  c->K = (uint16_t *)calloc((size_t)(U * cap * d), 2);
  c->V = (uint16_t *)calloc((size_t)(U * cap * d), 2);
  c->sal = (uint8_t *)calloc((size_t)(U * cap), 1);
  c->xk = (double *)calloc((size_t)(U * cap * d), 8);
  c->xv = (double *)calloc((size_t)(U * cap * d), 8);
  c->kc = (uint8_t *)calloc((size_t)(U * cap * d), 1);
  c->vc = (uint8_t *)calloc((size_t)(U * cap * d), 1);
  c->ks = (double *)calloc((size_t)(U * (cap / G) * d), 8);
  c->kz = (int32_t *)calloc((size_t)(U * (cap / G) * d), 4);
  c->kzp = (double *)calloc((size_t)(U * (cap / G) * d), 8);
  c->vs = (double *)calloc((size_t)(U * cap * (d / G)), 8);
  c->vz = (int32_t *)calloc((size_t)(U * cap * (d / G)), 4);
  c->vzp = (double *)calloc((size_t)(U * cap * (d / G)), 8);
  c->side_idx = (int32_t *)calloc((size_t)(U * sc), 4);
  c->side_cnt = (int32_t *)calloc((size_t)U, 4);
  c->side_pos = (int32_t *)malloc(sizeof(int32_t) * U * cap);
  for (long i = 0; i < U * cap; ++i) c->side_pos[i] = -1;
  c->s4c = (uint8_t *)calloc((size_t)(U * sc * 2 * d), 1);
  c->s4s = (double *)calloc((size_t)(U * sc * 2 * (d / G)), 8);
  c->s4z = (int32_t *)calloc((size_t)(U * sc * 2 * (d / G)), 4);
  c->s4zp = (double *)calloc((size_t)(U * sc * 2 * (d / G)), 8);
  if (status) *status = ORC_OK;
  return c;
}

void orc_free(orc_cache *c) {
  if (!c) return;
  free(c->H); free(c->Hs); free(c->K); free(c->V); free(c->sal);
  free(c->xk); free(c->xv); free(c->kc); free(c->vc);
  free(c->ks); free(c->kz); free(c->kzp); free(c->vs); free(c->vz); free(c->vzp);
  free(c->side_idx); free(c->side_cnt); free(c->side_pos);
  free(c->s4c); free(c->s4s); free(c->s4z); free(c->s4zp);
  free(c);
}

int orc_L(const orc_cache *c) { return c->L; }
int orc_nq(const orc_cache *c) { return c->nq; }
int orc_cap_rounded(const orc_cache *c) { return c->cap; }
int orc_side_cap(const orc_cache *c) { return c->side_cap; }
int orc_nthreads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* x.H_s of a stored 16-bit row by the explicit fp64 product (R5); in the
 * fp32-decision mode rounded once to fp32 (R6). */
static void rotate_row(const orc_cache *c, const uint16_t *row, double *out) {
  const int d = c->cfg.d;
  double x[512], y[512];
  for (int i = 0; i < d; ++i) x[i] = orc_half_to_double(row[i], c->cfg.dtype16);
  matvec(d, c->Hs, x, y);
  for (int i = 0; i < d; ++i) out[i] = c->cfg.decide64 ? y[i] : (double)(float)y[i];
}

/* Quantize block j = tokens [jG, (j+1)G) of unit u (R1):     */
/*  K: per channel c over the block's non-salient tokens (2-bit, clip2), */
/*     or (k_axis 1, P:246 literally) per token over G-channel groups    */
/*     exactly like V, meta at [token][group] in the same arrays.        */
/*  V: per token over G-channel groups (2-bit, clip2); salient tokens    */
/*     get codes 0 and meta (0, 0).                                      */
/*  Salient tokens enter the side table in ascending token order:        */
/*   PSA -> original 16-bit rows;                            */
/*   TSA -> 4-bit per-token groups of K.H_s and V.H_s, clip4.    */
static void quantize_block(orc_cache *c, int u, int j) {
  const int d = c->cfg.d, G = c->cfg.G, t0 = j * G;
  for (int t = t0; t < t0 + G; ++t) {
    rotate_row(c, c->K + ROW(c, u, t), c->xk + ROW(c, u, t));
    rotate_row(c, c->V + ROW(c, u, t), c->xv + ROW(c, u, t));
  }
  const uint8_t *skip = c->sal + (long)u * c->cap + t0;
  const long mb = ((long)u * (c->cap / G) + j) * d;
  const int ng = d / G, D64 = c->cfg.decide64;
  if (c->cfg.k_axis == 0) {
    for (int ch = 0; ch < d; ++ch)         /* K per channel over G tokens */
      qgroup(D64, c->xk + ROW(c, u, t0) + ch, skip, G, d, 2, c->cfg.clip2,
             &c->ks[mb + ch], &c->kz[mb + ch], &c->kzp[mb + ch],
             c->kc + ROW(c, u, t0) + ch, d);
  } else {
    for (int t = t0; t < t0 + G; ++t) {    /* K per token over G channels */
      const long km = ((long)u * c->cap + t) * ng;
      for (int gi = 0; gi < ng; ++gi) {
        if (c->sal[(long)u * c->cap + t]) {
          c->ks[km + gi] = 0.0; c->kz[km + gi] = 0; c->kzp[km + gi] = NAN;
          memset(c->kc + ROW(c, u, t) + gi * G, 0, (size_t)G);
        } else {
          qgroup(D64, c->xk + ROW(c, u, t) + gi * G, NULL, G, 1, 2, c->cfg.clip2,
                 &c->ks[km + gi], &c->kz[km + gi], &c->kzp[km + gi],
                 c->kc + ROW(c, u, t) + gi * G, 1);
        }
      }
    }
  }
  for (int t = t0; t < t0 + G; ++t) {      /* V per token over G channels */
    const long vm = ((long)u * c->cap + t) * ng;
    for (int gi = 0; gi < ng; ++gi) {
      if (c->sal[(long)u * c->cap + t]) {
        c->vs[vm + gi] = 0.0; c->vz[vm + gi] = 0; c->vzp[vm + gi] = NAN;
        memset(c->vc + ROW(c, u, t) + gi * G, 0, (size_t)G);
      } else {
        qgroup(D64, c->xv + ROW(c, u, t) + gi * G, NULL, G, 1, 2, c->cfg.clip2,
               &c->vs[vm + gi], &c->vz[vm + gi], &c->vzp[vm + gi],
               c->vc + ROW(c, u, t) + gi * G, 1);
      }
    }
  }
  for (int t = t0; t < t0 + G; ++t) {      /* side table, ascending t */
    if (!c->sal[(long)u * c->cap + t]) continue;
    const int e = c->side_cnt[u]++;
    c->side_idx[(long)u * c->side_cap + e] = t;
    c->side_pos[(long)u * c->cap + t] = e;
    if (c->cfg.kind == ORC_TSA) {
      for (int kv = 0; kv < 2; ++kv) {
        const double *x = (kv == 0 ? c->xk : c->xv) + ROW(c, u, t);
        const long base = (((long)u * c->side_cap + e) * 2 + kv);
        for (int gi = 0; gi < ng; ++gi)
          qgroup(D64, x + gi * G, NULL, G, 1, 4, c->cfg.clip4,
                 &c->s4s[base * ng + gi], &c->s4z[base * ng + gi], &c->s4zp[base * ng + gi],
                 c->s4c + base * d + gi * G, 1);
      }
    }
  }
}

/* One token leaving the window under the exact-R schedule (R26; per-token */
/* K only): the per-token steps of quantize_block for token t alone --     */
/* K and V per token over G-channel groups (Eqs. 3-6, clip2), salient ->   */
/* codes 0 and meta (0, 0) plus the side entry (TSA: 4-bit rows, clip4).    */
static void quantize_token(orc_cache *c, int u, int t) {
  const int d = c->cfg.d, G = c->cfg.G, ng = d / G, D64 = c->cfg.decide64;
  const int sal = c->sal[(long)u * c->cap + t];
  rotate_row(c, c->K + ROW(c, u, t), c->xk + ROW(c, u, t));
  rotate_row(c, c->V + ROW(c, u, t), c->xv + ROW(c, u, t));
  const long m = ((long)u * c->cap + t) * ng;
  for (int kv = 0; kv < 2; ++kv) {
    double *sc = kv ? c->vs : c->ks, *zp = kv ? c->vzp : c->kzp;
    int32_t *z = kv ? c->vz : c->kz;
    uint8_t *codes = (kv ? c->vc : c->kc) + ROW(c, u, t);
    const double *x = (kv ? c->xv : c->xk) + ROW(c, u, t);
    for (int gi = 0; gi < ng; ++gi) {
      if (sal) {
        sc[m + gi] = 0.0; z[m + gi] = 0; zp[m + gi] = NAN;
        memset(codes + gi * G, 0, (size_t)G);
      } else {
        qgroup(D64, x + gi * G, NULL, G, 1, 2, c->cfg.clip2, &sc[m + gi], &z[m + gi],
               &zp[m + gi], codes + gi * G, 1);
      }
    }
  }
  if (!sal) return;
  const int e = c->side_cnt[u]++;
  c->side_idx[(long)u * c->side_cap + e] = t;
  c->side_pos[(long)u * c->cap + t] = e;
  if (c->cfg.kind == ORC_TSA) {
    for (int kv = 0; kv < 2; ++kv) {
      const double *x = (kv == 0 ? c->xk : c->xv) + ROW(c, u, t);
      const long base = (((long)u * c->side_cap + e) * 2 + kv);
      for (int gi = 0; gi < ng; ++gi)
        qgroup(D64, x + gi * G, NULL, G, 1, 4, c->cfg.clip4,
               &c->s4s[base * ng + gi], &c->s4z[base * ng + gi], &c->s4zp[base * ng + gi],
               c->s4c + base * d + gi * G, 1);
    }
  }
}

/* Prefill: store rows, select salient tokens,     */
/* quantize blocks [0, n_q) with n_q = G floor(max(0, L0 - R)/G) (R9).    */
/* mask != NULL (PSA with explicit pivots, NEXT-2): salient = mask[u][t]. */
static int prefill_impl(orc_cache *c, const uint16_t *K, const uint16_t *V, int L0,
                        const uint8_t *types, const float *colsum, const uint8_t *mask) {
  const orc_config *f = &c->cfg;
  if (c->L != 0) return ORC_ESTATE;
  if (L0 < 0) return ORC_EINVAL;
  if (L0 > f->capacity) return ORC_ECAPACITY;
  if (f->kind == ORC_PSA && L0 > 0 && !colsum && !mask) return ORC_EINVAL;
  if (f->kind == ORC_TSA && L0 > 0 && !types) return ORC_EINVAL;
  if (mask) {                                /* at most top_k pivots per unit */
    if (f->kind != ORC_PSA) return ORC_EINVAL;
    for (int u = 0; u < f->U; ++u) {
      int n = 0;
      for (int t = 0; t < L0; ++t) n += mask[(long)u * L0 + t] != 0;
      if (n > f->top_k) return ORC_EINVAL;
    }
  }
  const int d = f->d;
  const int nq = L0 > f->R ? (f->exact_r ? L0 - f->R : (L0 - f->R) / f->G * f->G) : 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
  for (int u = 0; u < f->U; ++u) {
    for (int t = 0; t < L0; ++t) {
      memcpy(c->K + ROW(c, u, t), K + ((long)u * L0 + t) * d, (size_t)d * 2);
      memcpy(c->V + ROW(c, u, t), V + ((long)u * L0 + t) * d, (size_t)d * 2);
    }
    if (mask) {
      for (int t = 0; t < L0; ++t) c->sal[(long)u * c->cap + t] = mask[(long)u * L0 + t] != 0;
    } else {
      orc_select_salient(f->kind, f->g, L0, f->top_k,
                         types ? types + (long)u * L0 : NULL,
                         colsum ? colsum + (long)u * f->g * L0 : NULL,
                         c->sal + (long)u * c->cap);
    }
    if (f->exact_r)
      for (int t = 0; t < nq; ++t) quantize_token(c, u, t);
    else
      for (int j = 0; j < nq / f->G; ++j) quantize_block(c, u, j);
  }
  c->L = L0;
  c->nq = nq;
  return ORC_OK;
}

int orc_prefill(orc_cache *c, const uint16_t *K, const uint16_t *V, int L0,
                const uint8_t *types, const float *colsum) {
  return prefill_impl(c, K, V, L0, types, colsum, NULL);
}
int orc_prefill_pivots(orc_cache *c, const uint16_t *K, const uint16_t *V, int L0,
                       const uint8_t *pivot_mask) {
  return prefill_impl(c, K, V, L0, NULL, NULL, pivot_mask);
}

/* Append one decode token per unit (Eq. 2).        */
/* The new token enters the 16-bit recent window; in TSA layers a text    */
/* token is salient.  When L - R - n_q >= G the oldest block      */
/* leaves the window and is quantized exactly as prefill would.   */
int orc_append(orc_cache *c, const uint16_t *k, const uint16_t *v,
               const uint8_t *types) {
  const orc_config *f = &c->cfg;
  if (c->L >= f->capacity) return ORC_ECAPACITY;
  const int d = f->d, t = c->L;
  for (int u = 0; u < f->U; ++u) {
    memcpy(c->K + ROW(c, u, t), k + (long)u * d, (size_t)d * 2);
    memcpy(c->V + ROW(c, u, t), v + (long)u * d, (size_t)d * 2);
    c->sal[(long)u * c->cap + t] =
        (f->kind == ORC_TSA && types && types[u] == 1) ? 1 : 0;
  }
  c->L = t + 1;
  if (f->exact_r && c->L - f->R > c->nq) {   /* token n_q leaves the window (R26) */
    for (int u = 0; u < f->U; ++u) quantize_token(c, u, c->nq);
    c->nq += 1;
  } else if (!f->exact_r && c->L - f->R - c->nq >= f->G) {
    const int j = c->nq / f->G;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
    for (int u = 0; u < f->U; ++u) quantize_block(c, u, j);
    c->nq += f->G;
  }
  return ORC_OK;
}

/* Dequantized row of token t in the rotated normalized basis (Eq. 4).   */
static void view_row(const orc_cache *c, int u, int t, double *Kh, double *Vh) {
  const int d = c->cfg.d, G = c->cfg.G, ng = d / G;
  const double rs = 1.0 / sqrt((double)d);   /* stored scale = scale/sqrt d */
  const int sal = c->sal[(long)u * c->cap + t];
  if (t >= c->nq || (sal && c->cfg.kind == ORC_PSA)) {
    /* 16-bit tier (recent window / PSA pivots): original row . H */
    double x[512];
    for (int i = 0; i < d; ++i)
      x[i] = orc_half_to_double(c->K[ROW(c, u, t) + i], c->cfg.dtype16);
    matvec(d, c->H, x, Kh);
    for (int i = 0; i < d; ++i)
      x[i] = orc_half_to_double(c->V[ROW(c, u, t) + i], c->cfg.dtype16);
    matvec(d, c->H, x, Vh);
    return;
  }
  if (sal) {                                 /* TSA text token, 4-bit */
    const int e = c->side_pos[(long)u * c->cap + t];
    for (int kv = 0; kv < 2; ++kv) {
      const long base = ((long)u * c->side_cap + e) * 2 + kv;
      double *out = kv == 0 ? Kh : Vh;
      for (int i = 0; i < d; ++i) {
        const double s = c->s4s[base * ng + i / G] * rs;
        out[i] = s * ((double)c->s4c[base * d + i] - (double)c->s4z[base * ng + i / G]);
      }
    }
    return;
  }
  const int j = t / G;                       /* 2-bit tier */
  const long mb = ((long)u * (c->cap / G) + j) * d;
  const long vm = ((long)u * c->cap + t) * ng;
  for (int i = 0; i < d; ++i) {
    const long ki = c->cfg.k_axis == 0 ? mb + i : vm + i / G;   /* per channel | per token */
    Kh[i] = c->ks[ki] * rs *
            ((double)c->kc[ROW(c, u, t) + i] - (double)c->kz[ki]);
    Vh[i] = c->vs[vm + i / G] * rs *
            ((double)c->vc[ROW(c, u, t) + i] - (double)c->vz[vm + i / G]);
  }
}

int orc_view(const orc_cache *c, double *K, double *V) {
  const int d = c->cfg.d, L = c->L;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
  for (int u = 0; u < c->cfg.U; ++u)
    for (int t = 0; t < L; ++t)
      view_row(c, u, t, K + ((long)u * L + t) * d, V + ((long)u * L + t) * d);
  return ORC_OK;
}

/* Decode attention for one query per head: with q~ = q.H,     */
/*   s_t = q~ . K^_t / sqrt(d),  p = softmax(s),  o' = sum_t p_t V^_t,      */
/*   o = o' . H   (H symmetric orthonormal, so H^-1 = H; Fig. 7).    */
/* GQA: the g query heads of unit u all read unit u's cache.        */
int orc_decode(const orc_cache *c, const uint16_t *q, double *out,
               int out_rotated, int unit_lo, int unit_hi) {
  const orc_config *f = &c->cfg;
  const int d = f->d, g = f->g, L = c->L;
  if (L == 0) return ORC_ESTATE;
  if (unit_lo < 0) unit_lo = 0;
  if (unit_hi > f->U || unit_hi < 0) unit_hi = f->U;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic)
#endif
  for (int u = unit_lo; u < unit_hi; ++u) {
    double *Kh = (double *)malloc(sizeof(double) * L * d);
    double *Vh = (double *)malloc(sizeof(double) * L * d);
    double *s = (double *)malloc(sizeof(double) * L);
    double qx[512], qt[512], o[512];
    for (int t = 0; t < L; ++t) view_row(c, u, t, Kh + (long)t * d, Vh + (long)t * d);
    for (int h = 0; h < g; ++h) {
      const uint16_t *qr = q + ((long)u * g + h) * d;
      for (int i = 0; i < d; ++i) qx[i] = orc_half_to_double(qr[i], f->dtype16);
      matvec(d, c->H, qx, qt);                              /* q~ = q.H */
      double m = -INFINITY;
      for (int t = 0; t < L; ++t) {
        double a = 0.0;
        for (int i = 0; i < d; ++i) a += qt[i] * Kh[(long)t * d + i];
        s[t] = a / sqrt((double)d);
        if (s[t] > m) m = s[t];
      }
      double Z = 0.0;
      for (int t = 0; t < L; ++t) { s[t] = exp(s[t] - m); Z += s[t]; }
      for (int i = 0; i < d; ++i) o[i] = 0.0;
      for (int t = 0; t < L; ++t) {
        const double p = s[t] / Z;
        for (int i = 0; i < d; ++i) o[i] += p * Vh[(long)t * d + i];
      }
      double *dst = out + ((long)u * g + h) * d;
      if (out_rotated) memcpy(dst, o, sizeof(double) * d);
      else matvec(d, c->H, o, dst);                          /* o = o'.H */
    }
    free(Kh); free(Vh); free(s);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* x / scale before rounding, in the decision precision (NaN where no code
 * was decided: salient slot, empty or degenerate group). */
static double pre_round(const orc_cache *c, double x, double s, double zpre, int skip) {
  if (skip || isnan(zpre)) return NAN;
  return c->cfg.decide64 ? x / s : (double)((float)x / (float)s);
}

int orc_export(const orc_cache *c, const orc_export_t *ex) {
  const orc_config *f = &c->cfg;
  const long U = f->U, cap = c->cap, d = f->d, G = f->G, ng = d / G;
  const long sc = c->side_cap;
  const double rs = 1.0 / sqrt((double)d);
  for (long u = 0; u < U; ++u) {
    for (long t = 0; t < cap; ++t) {
      if (ex->kcodes) orc_pack(c->kc + ROW(c, (int)u, (int)t), (int)d, 2, ex->kcodes + (u * cap + t) * (d / 4));
      if (ex->vcodes) orc_pack(c->vc + ROW(c, (int)u, (int)t), (int)d, 2, ex->vcodes + (u * cap + t) * (d / 4));
      if (ex->salient) ex->salient[u * cap + t] = c->sal[u * cap + t];
      const int sal = c->sal[u * cap + t];
      for (long i = 0; i < d; ++i) {
        const long e = ROW(c, (int)u, (int)t) + i;
        const long km = f->k_axis == 0 ? (u * (cap / G) + t / G) * d + i : (u * cap + t) * ng + i / G;
        const long vm = (u * cap + t) * ng + i / G;
        if (ex->kpre) ex->kpre[e] = pre_round(c, c->xk[e], c->ks[km], c->kzp[km], sal);
        if (ex->vpre) ex->vpre[e] = pre_round(c, c->xv[e], c->vs[vm], c->vzp[vm], sal);
      }
    }
    if (ex->side_count) ex->side_count[u] = c->side_cnt[u];
    for (long e = 0; e < sc; ++e) {
      const int have = e < c->side_cnt[u];
      const int t = have ? c->side_idx[u * sc + e] : -1;
      if (ex->side_index) ex->side_index[u * sc + e] = t;
      if (ex->side16) {
        uint16_t *dst = ex->side16 + (u * sc + e) * 2 * d;
        if (have) {
          memcpy(dst, c->K + ROW(c, (int)u, t), (size_t)d * 2);
          memcpy(dst + d, c->V + ROW(c, (int)u, t), (size_t)d * 2);
        } else {
          memset(dst, 0, (size_t)d * 4);
        }
      }
      for (int kv = 0; kv < 2; ++kv) {
        const long base = (u * sc + e) * 2 + kv;
        if (ex->side4) orc_pack(c->s4c + base * d, (int)d, 4, ex->side4 + base * (d / 2));
        for (long gi = 0; gi < ng; ++gi) {
          if (ex->side4_scale) ex->side4_scale[base * ng + gi] = c->s4s[base * ng + gi] * rs;
          if (ex->side4_zero) ex->side4_zero[base * ng + gi] = c->s4z[base * ng + gi];
          if (ex->side4_zpre) ex->side4_zpre[base * ng + gi] = have ? c->s4zp[base * ng + gi] : NAN;
        }
        if (ex->side4_pre)
          for (long i = 0; i < d; ++i) {
            const double x = have ? (kv == 0 ? c->xk : c->xv)[ROW(c, (int)u, t) + i] : 0.0;
            ex->side4_pre[base * d + i] =
                have && f->kind == ORC_TSA
                    ? pre_round(c, x, c->s4s[base * ng + i / G], c->s4zp[base * ng + i / G], 0)
                    : NAN;
          }
      }
    }
  }
  const long nk = U * (cap / G) * d, nv = U * cap * ng;
  for (long i = 0; i < nk; ++i) {
    if (ex->kscale) ex->kscale[i] = c->ks[i] * rs;
    if (ex->kscale_raw) ex->kscale_raw[i] = c->ks[i];
    if (ex->kzero) ex->kzero[i] = c->kz[i];
    if (ex->kzpre) ex->kzpre[i] = c->kzp[i];
  }
  for (long i = 0; i < nv; ++i) {
    if (ex->vscale) ex->vscale[i] = c->vs[i] * rs;
    if (ex->vscale_raw) ex->vscale_raw[i] = c->vs[i];
    if (ex->vzero) ex->vzero[i] = c->vz[i];
    if (ex->vzpre) ex->vzpre[i] = c->vzp[i];
  }
  if (ex->xs_k) memcpy(ex->xs_k, c->xk, sizeof(double) * U * cap * d);
  if (ex->xs_v) memcpy(ex->xs_v, c->xv, sizeof(double) * U * cap * d);
  return ORC_OK;
}
