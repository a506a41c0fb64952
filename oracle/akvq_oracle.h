/*
 * akvq_oracle.h -- plain, slow CPU ORACLE for the AKVQ-VL hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2501_15021_b200/csrc, include/akvq.h) and neither side includes the
 * other.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (arXiv 2501.15021),
 * S:n = SPEC.md line n, BJ:n = BASELINE.json line n.  Readings where the
 * paper is silent are the DESIGN.md "Readings" list (R1..Rn).
 *
 * Arithmetic: fp64 everywhere, with an explicit d x d Walsh-Hadamard matrix
 * built by the recursion of Eq. 7.  The integer decisions of
 * Eqs. 3, 5, 6 -- min/max, clipping, scale, zero point and code --
 * are taken in fp64 by default; orc_config.decide64 = 0 takes
 * them in IEEE fp32 instead, the kernel's precision (R6), as a second
 * cross-check in which codes agree bit for bit.
 */
#ifndef AKVQ_ORACLE_H
#define AKVQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_TSA = 0, ORC_PSA = 1 };          /* Table I layer kinds */
enum { ORC_BF16 = 0, ORC_FP16 = 1 };        /* "original 16-bit" type  */

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ECAPACITY = 3, ORC_ESTATE = 4 };

typedef struct {
  int U;          /* units = batch x kv-heads                              */
  int g;          /* query heads per kv head (GQA)                   */
  int d;          /* head_dim, power of two (Eq. 7 domain)                  */
  int G;          /* quantization group size                        */
  int R;          /* recent / residual window                */
  int capacity;   /* max tokens per unit                                    */
  int top_k;      /* PSA pivot count                                */
  int kind;       /* ORC_TSA / ORC_PSA                                      */
  int dtype16;    /* ORC_BF16 / ORC_FP16                                    */
  float clip2;    /* clip ratio for 2-bit (0.8)                      */
  float clip4;    /* clip ratio for 4-bit (1.0)                      */
  int k_axis;     /* 0: K per channel over G-token blocks (R1, graded);
                     1: K per token over G-channel groups, the paper-literal
                     "per-token dynamic" rule of P:246       */
  int decide64;   /* 1: quantizer decisions in fp64 (default); 0: in IEEE
                     fp32 on the fp32-rounded x.H_s (R6)                     */
  int exact_r;    /* per-token K only (k_axis 1): 1 = exactly the last R
                     tokens stay 16-bit, n_q = max(0, L - R), every token
                     quantized on its own when it leaves the window (P:246,
                     "residual" R, DESIGN R26); 0 = the block schedule R9    */
} orc_config;

typedef struct orc_cache orc_cache;

/* ---- primitives (each pinned by tests/test_oracle_pins.py) ---------- */
/* Eq. 7: H_1 = [1], H_{2^k} = 1/sqrt2 [[H, H], [H, -H]].  normalized=0
 * builds the same recursion without the 1/sqrt2 factor (the +-1 matrix H_s). */
int  orc_hadamard(int d, int normalized, double *H);
/* y = x . H (normalized=1) or x . H_s (normalized=0); explicit mat-vec.   */
int  orc_rotate(int d, int normalized, const double *x, double *y);
/* Eqs. 3,5,6 on one group, decisions in fp32 (R6).  skip[i]!=0 excludes
 * element i (salient token) from the statistics and gives it code 0.
 * Returns the (unnormalized-unit) scale, the zero point and the codes.   */
void orc_quantize_group(const float *x, const uint8_t *skip, int n, int stride,
                        int bits, float clip, float *scale, int32_t *zero,
                        uint8_t *codes, int code_stride);
/* The same in fp64 (clip is the fp32 constant widened exactly); zpre =
 * clipped_min / scale before rounding (NaN for empty / degenerate groups). */
void orc_quantize_group64(const double *x, const uint8_t *skip, int n, int bits, float clip,
                          double *scale, int32_t *zero, double *zpre, uint8_t *codes);
/* S:146 bit layout. */
void orc_pack(const uint8_t *codes, int n, int bits, uint8_t *out);
void orc_unpack(const uint8_t *in, int n, int bits, uint8_t *codes);
/* 16-bit decode (exact widening). */
double orc_half_to_double(uint16_t h, int dtype16);
/* PSA top-k over summed column scores / TSA text mask -> salient[0..L0). */
void orc_select_salient(int kind, int g, int L0, int top_k,
                        const uint8_t *types, const float *colsum,
                        uint8_t *salient);

/* ---- one layer's mixed-precision cache ------------------------------ */
orc_cache *orc_new(const orc_config *cfg, int *status);
void orc_free(orc_cache *c);
int  orc_L(const orc_cache *c);
int  orc_nq(const orc_cache *c);
int  orc_nthreads(void);
/* K, V [U][L0][d] 16-bit bit patterns; types [U][L0]; colsum [U][g][L0]. */
int  orc_prefill(orc_cache *c, const uint16_t *K, const uint16_t *V, int L0,
                 const uint8_t *types, const float *colsum);
/* Massive-activation pivots of one residual stream [L0][hidden] 16-bit
 * (NEXT-2); writes <= n_max token indices (>= 1), returns
 * the count. */
int  orc_detect_pivots(int L0, int hidden, const uint16_t *residual, int dtype16, float tau,
                       int n_max, int32_t *out);
/* PSA prefill with an explicit pivot mask [U][L0] (<= top_k per unit). */
int  orc_prefill_pivots(orc_cache *c, const uint16_t *K, const uint16_t *V, int L0,
                        const uint8_t *pivot_mask);
/* k, v [U][d]; types [U] */
int  orc_append(orc_cache *c, const uint16_t *k, const uint16_t *v,
                const uint8_t *types);
/* q [U][g][d] 16-bit; out [U][g][d] fp64.  out_rotated: return o' = sum p V^
 * in the rotated basis instead of o = o'.H.  unit_lo..unit_hi restricts the
 * work to a unit range (bench sampling); other rows are untouched.        */
int  orc_decode(const orc_cache *c, const uint16_t *q, double *out,
                int out_rotated, int unit_lo, int unit_hi);
/* Dequantized view in the rotated (normalized) basis: K^, V^ [U][L][d].  */
int  orc_view(const orc_cache *c, double *K, double *V);

/* Export of the packed representation in the oracle's own natural layout:
 *  kcodes, vcodes [U][cap][d/4] (S:146 packing along channels)
 *  kscale [U][cap/G][d] (normalized, fp64), kzero [U][cap/G][d]
 *  vscale [U][cap][d/G], vzero [U][cap][d/G]
 *  kscale_raw / vscale_raw: the unnormalized decision scales
 *  kzpre / vzpre: clipped_min / scale before rounding (zero-point tie test;
 *      NaN where no zero point was decided)
 *  kpre, vpre [U][cap][d]: x / scale before rounding (code tie test; NaN for
 *      salient slots, empty and degenerate groups), in decision precision
 *  salient [U][cap] (0/1)
 *  side_index [U][side_cap], side_count [U]
 *  side16 [U][side_cap][2][d]   (PSA: original 16-bit K row then V row)
 *  side4 [U][side_cap][2][d/2], side4_scale/zero/zpre [U][side_cap][2][d/G],
 *  side4_pre [U][side_cap][2][d] (TSA)
 *  xs_k, xs_v [U][cap][d]: the K.H_s / V.H_s values the decisions used.
 * Any pointer may be NULL.  cap is rounded up to a multiple of G.          */
typedef struct {
  uint8_t *kcodes, *vcodes;
  double *kscale; int32_t *kzero;
  double *vscale; int32_t *vzero;
  double *kscale_raw, *vscale_raw;
  double *kzpre, *vzpre;
  double *kpre, *vpre;
  uint8_t *salient;
  int32_t *side_index, *side_count;
  uint16_t *side16;
  uint8_t *side4; double *side4_scale; int32_t *side4_zero;
  double *side4_zpre, *side4_pre;
  double *xs_k, *xs_v;
} orc_export_t;
int orc_export(const orc_cache *c, const orc_export_t *ex);
int orc_cap_rounded(const orc_cache *c);
int orc_side_cap(const orc_cache *c);

#ifdef __cplusplus
}
#endif
#endif
