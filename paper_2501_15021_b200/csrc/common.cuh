// common.cuh -- device-side helpers shared by the libakvq.so kernels (sm_100a).
// AKVQ-VL (arXiv 2501.15021).  Nothing here is shared with oracle/.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "akvq.h"

namespace akvq {

constexpr float kLog2e = 1.4426950408889634f;

// Device view of one layer's cache (pointers resolved on the host from
// akvq_layout; see include/akvq.h for the byte layout).
struct DevCache {
  uint8_t *pages;          // [U][n_pages][page_bytes], or the page pool (paged)
  const int32_t *btab;     // paged: [U][n_pages] pool page of (unit, page); else null
  uint16_t *ring;          // [U][slots][2][d]
  uint32_t *bitmask;       // [U][bm_words]
  int32_t *side_idx;       // [U][side_cap]
  int32_t *side_cnt;       // [U]
  uint8_t *side;           // [U][side_cap][side_entry]
  uint32_t *ticket;        // [U * hg] decode-merge tickets (zero between launches)
  float2 *umax;            // [U] (max |K scale|, max |V scale|) of the unit's pages
  struct State { int32_t L; uint32_t done; int32_t pad[2]; };
  State *dstate;           // device copy of the token count L (+ launch exit counter)
  uint32_t page_bytes, pg_kscale, pg_kzero, pg_kcodes, pg_vscale, pg_vzero, pg_vcodes;
  uint32_t side_entry;
  int32_t n_pages, slots, bm_words, side_cap;
  int32_t U, g, d, G, R, ng, kind, k_axis;
  float clip2, clip4, inv_sqrt_d;
};

__device__ __forceinline__ uint8_t *page_ptr(const DevCache &c, int u, int p) {
  if (c.btab) return c.pages + (size_t)__ldg(c.btab + (size_t)u * c.n_pages + p) * c.page_bytes;
  return c.pages + ((size_t)u * c.n_pages + p) * c.page_bytes;
}
__device__ __forceinline__ uint16_t *ring_row(const DevCache &c, int u, int slot) {
  return c.ring + ((size_t)u * c.slots + slot) * 2 * c.d;   // K row; V row at +d
}
__device__ __forceinline__ uint8_t *side_ptr(const DevCache &c, int u, int e) {
  return c.side + ((size_t)u * c.side_cap + e) * c.side_entry;
}

// ---- 2-bit code layout inside a page (include/akvq.h) ----
// Both code regions are arrays of 32-bit words, each a 4 x 4 tile of (token,
// channel) codes; TQ = G/4 token quads, CQ = d/4 channel quads.
//  K word ((cq>>2)*TQ + tq)*4 + (cq&3): byte b = channel 4cq+b, bits 2s..2s+1 of
//    that byte = token 4tq+s.  A mask w & (3<<2s per byte) yields the 4 channels'
//    codes (x4^s) of ONE token: one A-fragment register of the page MMA (rows =
//    tokens, K = channels).
//  V word ((tq>>2)*CQ + cq)*4 + (tq&3): byte b = token 4tq+b (that byte is the
//    token's S:146 byte for channels 4cq..4cq+3), bits 2s = channel 4cq+s.  A
//    mask yields 4 tokens' codes (x4^s) of ONE channel: one A-fragment register
//    of the value MMA (rows = channels, K = tokens).
// Codes themselves are exactly the paper's (Eqs. 3-6); only their byte order is
// chosen for the decode kernel.
__host__ __device__ __forceinline__ int kword_idx(int cq, int tq, int TQ) {
  return ((cq >> 2) * TQ + tq) * 4 + (cq & 3);
}
__host__ __device__ __forceinline__ int vword_idx(int cq, int tq, int CQ) {
  return ((tq >> 2) * CQ + cq) * 4 + (tq & 3);
}
// code of token t (in page), channel ch
__device__ __forceinline__ uint32_t kcode_at(const uint8_t *kc, int t, int ch, int G) {
  return (kc[4 * kword_idx(ch >> 2, t >> 2, G >> 2) + (ch & 3)] >> (2 * (t & 3))) & 3u;
}
__device__ __forceinline__ uint32_t vcode_at(const uint8_t *vc, int t, int ch, int D) {
  return (vc[4 * vword_idx(ch >> 2, t >> 2, D >> 2) + (t & 3)] >> (2 * (ch & 3))) & 3u;
}
// S:146 byte of token t for channels 4cq..4cq+3 (V region)
__device__ __forceinline__ uint32_t vbyte_at(const uint8_t *vc, int t, int cq, int D) {
  return vc[4 * vword_idx(cq, t >> 2, D >> 2) + (t & 3)];
}

// ---- 16-bit element types --------------------------------------------------
template <int DT> struct H16;
template <> struct H16<AKVQ_BF16> {
  static __device__ __forceinline__ float to_f(uint16_t h) {
    return __uint_as_float((uint32_t)h << 16);
  }
};
template <> struct H16<AKVQ_FP16> {
  static __device__ __forceinline__ float to_f(uint16_t h) {
    return __half2float(__ushort_as_half(h));
  }
};

// Unpack 8 16-bit values held in a uint4.
template <int DT>
__device__ __forceinline__ void cvt8(const uint4 v, float *o) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = H16<DT>::to_f((uint16_t)(w[i] & 0xffff));
    o[2 * i + 1] = H16<DT>::to_f((uint16_t)(w[i] >> 16));
  }
}

// Load a row of D 16-bit values into fp32 registers.
template <int D, int DT>
__device__ __forceinline__ void load_row(const uint16_t *__restrict__ src, float (&x)[D]) {
  const uint4 *s = reinterpret_cast<const uint4 *>(src);
#pragma unroll
  for (int i = 0; i < D / 8; ++i) cvt8<DT>(__ldg(s + i), x + 8 * i);
}

// In-register fast Walsh-Hadamard transform: x <- x . H_s, the +-1
// Sylvester matrix in natural order (Eq. 7 without the 1/sqrt2 factors, R5).
template <int D>
__device__ __forceinline__ void fwht_reg(float (&x)[D]) {
#pragma unroll
  for (int h = 1; h < D; h <<= 1) {
#pragma unroll
    for (int i = 0; i < D; i += 2 * h) {
#pragma unroll
      for (int j = i; j < i + h; ++j) {
        const float a = x[j], b = x[j + h];
        x[j] = __fadd_rn(a, b);
        x[j + h] = __fsub_rn(a, b);
      }
    }
  }
}

// ---- Eqs. 3, 5, 6 with fp32 decisions (R3, R6, R7, R8) ------
struct QMeta {
  float s;    // scale in x.H_s units (normal), constant (degenerate), 0 (empty)
  float zf;   // zero point as an integer-valued float
  int mode;   // 0 normal, 1 degenerate (codes 1), 2 empty (codes 0)
};

// IEEE single operations only (explicit _rn intrinsics: no FMA contraction).
__device__ __forceinline__ QMeta q_meta(float mn, float mx, bool any, float clip,
                                        float levels) {
  QMeta m;
  if (!any) { m.s = 0.f; m.zf = 0.f; m.mode = 2; return m; }
  const float cmx = __fmul_rn(clip, mx);            // clipped_max(X)
  const float cmn = __fmul_rn(clip, mn);            // clipped_min(X)
  const float range = __fsub_rn(cmx, cmn);
  if (range < 1e-12f) { m.s = mx; m.zf = 0.f; m.mode = 1; return m; }
  m.s = __fdiv_rn(range, levels);                   // Eq. 5
  m.zf = -rintf(__fdiv_rn(cmn, m.s));               // Eq. 6
  m.mode = 0;
  return m;
}

__device__ __forceinline__ uint32_t q_code(float x, const QMeta &m, float levels) {
  if (m.mode == 2) return 0u;
  if (m.mode == 1) return 1u;
  const float r = rintf(__fdiv_rn(x, m.s));         // Eq. 3
  float q = __fadd_rn(r, m.zf);
  q = fminf(fmaxf(q, 0.f), levels);
  return (uint32_t)q;
}

// Same result as q_code (bit for bit), cheaper: with rs = 1/s rounded, x * rs is
// within 2 ulp of the IEEE quotient RN(x / s), so their round-half-to-even agree
// unless the product lies within a few ulp of a half-integer; only then is the
// IEEE division evaluated.
__device__ __forceinline__ uint32_t q_code_fast(float x, const QMeta &m, float rs, float levels) {
  if (m.mode == 2) return 0u;
  if (m.mode == 1) return 1u;
  float y = __fmul_rn(x, rs);
  const float f = __fsub_rn(y, floorf(y));          // fractional part, exact
  if (fabsf(__fsub_rn(f, 0.5f)) <= 8.f * 1.1920929e-07f * fmaxf(fabsf(y), 1.f))
    y = __fdiv_rn(x, m.s);                          // near a tie: exact quotient
  float q = __fadd_rn(rintf(y), m.zf);
  q = fminf(fmaxf(q, 0.f), levels);
  return (uint32_t)q;
}

__device__ __forceinline__ int32_t zero_i32(float zf) { return __float2int_rz(zf); }


// N codes of one group (same meta) packed at 2 * i bits, i < N: branch-free
// except once per group.  Equal, bit for bit, to q_code on each element: the
// product x * rs lies within 2 ulp of the IEEE quotient x / s, so both round to
// the same integer unless the product is within 1e-6 (|y| + 1) of a half-integer;
// if any element of the group is that close, the group is redone with IEEE
// division (rare).  mode 1 / 2 groups (degenerate / empty) are uniform.
template <int N>
__device__ __forceinline__ uint32_t q_codes2(const float (&x)[N], const QMeta &m, float rs) {
  if (m.mode == 2) return 0u;
  if (m.mode == 1) return 0x55555555u & ((N >= 16) ? 0xffffffffu : ((1u << (2 * N)) - 1u));
  uint32_t w = 0;
  bool near = false;
#ifndef AKVQ_QCODES_V1
  // |x rs - x / s| <= 2 ulp(|y|) < 2.4e-7 |y|: for |y| <= 99 the two round alike
  // unless y is within 2.4e-5 of a half-integer, which |y - rint(y)| > 0.4999
  // flags; |y| > 99 (a large zero point) always takes the IEEE path.  Codes are
  // packed exactly in fp32 (8 per float, values < 2^16) instead of per-code
  // conversions and shifts.
  float acc[(N + 7) / 8];
#pragma unroll
  for (int i = 0; i < (N + 7) / 8; ++i) acc[i] = 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float y = __fmul_rn(x[i], rs);
    const float r = rintf(y);
    near |= fabsf(__fsub_rn(y, r)) > 0.4999f;
    near |= fabsf(y) > 99.f;
    const float q = fminf(fmaxf(__fadd_rn(r, m.zf), 0.f), 3.f);
    acc[i / 8] = __fmaf_rn(q, (float)(1u << (2 * (i % 8))), acc[i / 8]);
  }
#pragma unroll
  for (int i = 0; i < (N + 7) / 8; ++i) w |= (uint32_t)acc[i] << (16 * i);
#else
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float y = __fmul_rn(x[i], rs);
    const float r = rintf(y);
    near |= fabsf(__fsub_rn(y, r)) > __fsub_rn(0.5f, __fmul_rn(1e-6f, __fadd_rn(fabsf(y), 1.f)));
    const float q = fminf(fmaxf(__fadd_rn(r, m.zf), 0.f), 3.f);
    w |= (uint32_t)q << (2 * i);
  }
#endif
  if (near) {
    w = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) w |= q_code(x[i], m, 3.f) << (2 * i);
  }
  return w;
}

// ---- warp helpers --------------------------------------------------------
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace akvq
