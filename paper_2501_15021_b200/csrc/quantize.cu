// quantize.cu -- prefill / flush side of the AKVQ-VL hot path on sm_100a:
//   K2  select_salient   (TSA text mask, PSA block top-k)       P:199-213, BJ:5
//   K1  quantize_blocks  (FWHT -> per-channel K / per-token V 2-bit, side table)
//                                                                 Eqs. 3-7
//   K1t ring_fill / K3 append (16-bit recent window, Eq. 2)
#include "common.cuh"
#include "kernels.h"

namespace akvq {

// ============================================================ K2: saliency
// TSA: salient = text tokens.  One warp per 32 tokens, ballot.
__global__ void k_salient_tsa(DevCache c, const uint8_t *__restrict__ types, int L0) {
  const int u = blockIdx.y;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool text = t < L0 && types[(size_t)u * L0 + t] == 1;
  const uint32_t b = __ballot_sync(0xffffffffu, text);
  if ((threadIdx.x & 31) == 0 && t < L0) c.bitmask[(size_t)u * c.bm_words + t / 32] = b;
}

// Orderable 64-bit key: larger = earlier in (score desc, index asc) (R2).
__device__ __forceinline__ uint64_t sal_key(float s, int t) {
  uint32_t b = __float_as_uint(s);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((uint64_t)b << 32) | (uint32_t)(0xffffffffu - (uint32_t)t);
}

// PSA (P:205-213 in BJ:5's form): score_t = sum_j colsum[u][j][t] (fp32, j
// ascending, R6); select the top_k keys by k rounds of a block-wide max over
// keys strictly below the previous winner.  One CTA per unit; scores live in
// dynamic shared memory.
__global__ void __launch_bounds__(1024) k_salient_psa(DevCache c, const float *__restrict__ colsum,
                                                      int L0, int top_k) {
  extern __shared__ float sc[];
  __shared__ uint64_t red[32];
  const int u = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const float *cs = colsum + (size_t)u * c.g * L0;
  for (int t = tid; t < L0; t += nt) {
    float s = 0.f;
    for (int j = 0; j < c.g; ++j) s = __fadd_rn(s, cs[(size_t)j * L0 + t]);
    sc[t] = s;
  }
  __syncthreads();
  const int k = top_k < L0 ? top_k : L0;
  uint64_t prev = ~0ull;
  for (int r = 0; r < k; ++r) {
    uint64_t best = 0;
    for (int t = tid; t < L0; t += nt) {
      const uint64_t key = sal_key(sc[t], t);
      if (key < prev && key > best) best = key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t x = __shfl_xor_sync(0xffffffffu, best, o);
      best = x > best ? x : best;
    }
    if ((tid & 31) == 0) red[tid >> 5] = best;
    __syncthreads();
    if (tid < 32) {
      uint64_t v = tid < (nt >> 5) ? red[tid] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x > v ? x : v;
      }
      if (tid == 0) {
        red[0] = v;
        const int t = (int)(0xffffffffu - (uint32_t)(v & 0xffffffffu));
        c.bitmask[(size_t)u * c.bm_words + t / 32] |= 1u << (t % 32);
      }
    }
    __syncthreads();
    prev = red[0];
    __syncthreads();
  }
}

// ============================================================ K1: quantize
// One CTA (8 warps) per (G-token block j, unit u).  Rows are processed by
// 8-lane groups, CPL = d/8 channels per lane, 4 rows per warp at a time:
//   1. row -> fp32 -> FWHT x.H_s (R5): log2(CPL) in-lane butterfly stages, then
//      3 shuffle stages across the 8 lanes (the same addition sequence as a
//      sequential in-register FWHT, so results are bit-identical to it)
//   2. K row -> smem (fp32) for the per-channel block stats (R1)
//   3. V row: per-token stats over each G-channel group (lane reductions),
//      Eqs. 5-6 -> V meta, codes -> S:146 bytes in smem
//   4. salient rows -> side table (PSA: original 16-bit rows; TSA: 4-bit per
//      token over G-channel groups with clip4, R11)
//   5. thread ch: min/max of K channel ch over the block's non-salient tokens,
//      Eqs. 5-6 -> K meta; then all threads build the 4x4-tile code words of K
//      and V (common.cuh kword_idx / vword_idx) with coalesced stores.
// Source rows come from the prefill inputs or, for a flush, from the ring.
constexpr int kQThreads = 256;
// packed fp32x2 FWHT and cheaper code rounding (A/B knob; results are identical)
#ifndef AKVQ_QPACKED
#define AKVQ_QPACKED 1
#endif
#ifndef AKVQ_QPREFETCH
#define AKVQ_QPREFETCH 1
#endif

// Staged K rows xs[t][P]: 16-byte chunk c of a row is stored at chunk
// c ^ ((c >> 2) & 7), so the 8 lanes of a row (16 consecutive channels each)
// store to distinct banks and a warp reading 32 consecutive chunks stays
// conflict-free.
__device__ __forceinline__ int xs_col(int ch) { return ((((ch >> 2) ^ (ch >> 4)) & 7) | ((ch >> 2) & ~7)) * 4 + (ch & 3); }

template <int CPL>
__device__ __forceinline__ void fwht_lanes8(float (&x)[CPL], int cl) {
#if AKVQ_QPACKED
  // stage h = 1 scalar; stages h >= 2 pair the adjacent lower elements (j, j+1)
  // with (j+h, j+h+1) as packed fp32x2 (FADD2 / FFMA2); a - b is fma(b, -1, a),
  // one rounding like the scalar subtraction: bit-identical results
#pragma unroll
  for (int i = 0; i < CPL; i += 2) {
    const float a = x[i], b = x[i + 1];
    x[i] = __fadd_rn(a, b);
    x[i + 1] = __fsub_rn(a, b);
  }
#pragma unroll
  for (int h = 2; h < CPL; h <<= 1)
#pragma unroll
    for (int i = 0; i < CPL; i += 2 * h)
#pragma unroll
      for (int j = i; j < i + h; j += 2) {
        const float2 a = make_float2(x[j], x[j + 1]), b = make_float2(x[j + h], x[j + h + 1]);
        const float2 sm = __fadd2_rn(a, b), df = __ffma2_rn(b, make_float2(-1.f, -1.f), a);
        x[j] = sm.x; x[j + 1] = sm.y; x[j + h] = df.x; x[j + h + 1] = df.y;
      }
#pragma unroll
  for (int lm = 1; lm < 8; lm <<= 1) {
    const float sg = (cl & lm) ? -1.f : 1.f;     // upper: partner - own; lower: own + partner
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      const float2 pr = make_float2(__shfl_xor_sync(0xffffffffu, x[k], lm), __shfl_xor_sync(0xffffffffu, x[k + 1], lm));
      const float2 r = __ffma2_rn(make_float2(sg, sg), make_float2(x[k], x[k + 1]), pr);
      x[k] = r.x; x[k + 1] = r.y;
    }
  }
#else
#pragma unroll
  for (int h = 1; h < CPL; h <<= 1)
#pragma unroll
    for (int i = 0; i < CPL; i += 2 * h)
#pragma unroll
      for (int j = i; j < i + h; ++j) {
        const float a = x[j], b = x[j + h];
        x[j] = __fadd_rn(a, b);
        x[j + h] = __fsub_rn(a, b);
      }
#pragma unroll
  for (int lm = 1; lm < 8; lm <<= 1) {
    const float sg = (cl & lm) ? -1.f : 1.f;     // upper: partner - own; lower: own + partner
#pragma unroll
    for (int k = 0; k < CPL; ++k) x[k] = __fmaf_rn(sg, x[k], __shfl_xor_sync(0xffffffffu, x[k], lm));
  }
#endif
}

// min / max over the lanes of a channel group of GL lanes (within the 8-lane row group)
template <int GL>
__device__ __forceinline__ void group_minmax(float &mn, float &mx) {
#pragma unroll
  for (int o = 1; o < GL; o <<= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
}

template <int D, int G, int DT, bool KT>
__global__ void __launch_bounds__(kQThreads, 2) k_quantize_blocks(DevCache c, QuantSrc src, int block0,
                                                               int last_block) {
  constexpr int CPL = D / 8;                 // channels per lane
  constexpr int GL = G / CPL;                // lanes per V channel group
  constexpr int P = D + 4;                   // smem pitch (floats), 16-byte rows
  constexpr int NG = D / G;
  constexpr int NW = kQThreads / 32;
  extern __shared__ __align__(16) float xs[];     // [G][P] rotated K rows
  __shared__ float s_s[D], s_z[D], s_rs[D];
  __shared__ int s_mode[D];
  __shared__ uint32_t s_bits[G / 32];
  __shared__ __align__(16) uint8_t vb8[G * D / 4];   // V S:146 bytes per token
  __shared__ int s_base;
  __shared__ unsigned s_kmax, s_vmax;     // block max of |stored K / V scale| (float bits)

  const int u = blockIdx.y, j = block0 + blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, rg = lane >> 3, cl = lane & 7;
  const uint32_t *bm = c.bitmask + (size_t)u * c.bm_words;
  if (tid < G / 32) s_bits[tid] = bm[j * (G / 32) + tid];
  if (tid == 0) { s_base = 0; s_kmax = 0u; s_vmax = 0u; }
  __syncthreads();
  {  // salient entries before this block -> first side slot of the block
    int cnt = 0;
    for (int w = tid; w < j * (G / 32); w += kQThreads) cnt += __popc(bm[w]);
    if (cnt) atomicAdd(&s_base, cnt);
  }
  __syncthreads();
  uint8_t *pg = page_ptr(c, u, j);
  const bool tsa = c.kind == AKVQ_TSA;
  float *vs_g = reinterpret_cast<float *>(pg + c.pg_vscale);
  int32_t *vz_g = reinterpret_cast<int32_t *>(pg + c.pg_vzero);

  // ---------------- rows: FWHT of K and V, V quantization, side entries
  unsigned kmax_l = 0u, vmax_l = 0u;          // this lane's largest |stored scale| (bits)
  auto row_off = [&](int t) -> size_t {     // element offset of token t's row
    const int tok = j * G + t;
    return (size_t)u * src.unit_stride +
           (size_t)(src.ring_slots ? tok % src.ring_slots : tok) * src.tok_stride + cl * CPL;
  };
#if AKVQ_QPREFETCH
  // the next row group's loads are issued before this one is processed
  uint4 knx[CPL / 8], vnx[CPL / 8];
  {
    const size_t o = row_off(warp * 4 + rg);
#pragma unroll
    for (int i = 0; i < CPL / 8; ++i) {
      knx[i] = reinterpret_cast<const uint4 *>(src.K + o)[i];
      vnx[i] = reinterpret_cast<const uint4 *>(src.V + o)[i];
    }
  }
#endif
  for (int r0 = warp * 4; r0 < G; r0 += NW * 4) {
    const int t = r0 + rg;                   // token within the block
    const int tok = j * G + t;
    const bool sal = (s_bits[t >> 5] >> (t & 31)) & 1u;
    uint4 kraw[CPL / 8], vraw[CPL / 8];
#if AKVQ_QPREFETCH
#pragma unroll
    for (int i = 0; i < CPL / 8; ++i) { kraw[i] = knx[i]; vraw[i] = vnx[i]; }
    if (r0 + NW * 4 < G) {
      const size_t o = row_off(t + NW * 4);
#pragma unroll
      for (int i = 0; i < CPL / 8; ++i) {
        knx[i] = reinterpret_cast<const uint4 *>(src.K + o)[i];
        vnx[i] = reinterpret_cast<const uint4 *>(src.V + o)[i];
      }
    }
#else
    {
      const size_t o = row_off(t);
#pragma unroll
      for (int i = 0; i < CPL / 8; ++i) {
        kraw[i] = reinterpret_cast<const uint4 *>(src.K + o)[i];
        vraw[i] = reinterpret_cast<const uint4 *>(src.V + o)[i];
      }
    }
#endif
    float k[CPL], v[CPL];
#pragma unroll
    for (int i = 0; i < CPL / 8; ++i) { cvt8<DT>(kraw[i], k + 8 * i); cvt8<DT>(vraw[i], v + 8 * i); }
    fwht_lanes8<CPL>(k, cl);
    fwht_lanes8<CPL>(v, cl);
    // staged K rows; a salient row is staged as NaN, which fminf / fmaxf skip in
    // the per-channel statistics (its codes are masked to 0 when packed)
    const float kst = sal && !KT ? __int_as_float(0x7fc00000) : 0.f;
#pragma unroll
    for (int i = 0; i < CPL / 4; ++i)
      *reinterpret_cast<float4 *>(xs + t * P + xs_col(cl * CPL + 4 * i)) =
          sal && !KT ? make_float4(kst, kst, kst, kst)
                     : make_float4(k[4 * i], k[4 * i + 1], k[4 * i + 2], k[4 * i + 3]);
    if constexpr (KT) {                   // K per token over G-channel groups (NEXT-1)
      const int gi = (cl * CPL) / G;
      float mn = k[0], mx = k[0];
#pragma unroll
      for (int i = 1; i < CPL; ++i) { mn = fminf(mn, k[i]); mx = fmaxf(mx, k[i]); }
      group_minmax<GL>(mn, mx);
      const QMeta m = q_meta(mn, mx, !sal, c.clip2, 3.f);
      if ((cl % GL) == 0) {
        const int mi = t * NG + gi;                  // meta [G][NG], same bytes as [D]
        s_s[mi] = m.s; s_z[mi] = m.zf; s_mode[mi] = m.mode;
        s_rs[mi] = m.mode == 0 ? __frcp_rn(m.s) : 0.f;
        const float ks = sal ? 0.f : __fmul_rn(m.s, c.inv_sqrt_d);
        reinterpret_cast<float *>(pg + c.pg_kscale)[mi] = ks;
        reinterpret_cast<int32_t *>(pg + c.pg_kzero)[mi] = sal ? 0 : zero_i32(m.zf);
        kmax_l = max(kmax_l, __float_as_uint(fabsf(ks)));
      }
    }

    // V: per token over the lane's channel group (Eqs. 3-6, clip2), salient -> 0
    {
      const int gi = (cl * CPL) / G;
      float mn = v[0], mx = v[0];
#pragma unroll
      for (int i = 1; i < CPL; ++i) { mn = fminf(mn, v[i]); mx = fmaxf(mx, v[i]); }
      group_minmax<GL>(mn, mx);
      const QMeta m = q_meta(mn, mx, !sal, c.clip2, 3.f);
      if ((cl % GL) == 0) {
        const float vsn = sal ? 0.f : __fmul_rn(m.s, c.inv_sqrt_d);
        vs_g[t * NG + gi] = vsn;
        vz_g[t * NG + gi] = sal ? 0 : zero_i32(m.zf);
        vmax_l = max(vmax_l, __float_as_uint(fabsf(vsn)));
      }
      static_assert(CPL == 8 || CPL == 16, "channels per lane");
      uint32_t w = 0;                         // the lane's CPL/4 S:146 bytes
      const float rs = m.mode == 0 ? __frcp_rn(m.s) : 0.f;
      w = q_codes2<CPL>(v, m, rs);            // salient row: m.mode == 2 -> codes 0
      if constexpr (CPL == 16) *reinterpret_cast<uint32_t *>(vb8 + t * (D / 4) + cl * 4) = w;
      else *reinterpret_cast<uint16_t *>(vb8 + t * (D / 4) + cl * 2) = (uint16_t)w;
    }
    // TSA 4-bit side stats (group reductions need every lane: computed for all rows)
    QMeta mk4, mv4;
    if (tsa && __any_sync(0xffffffffu, sal)) {
      float mnk = k[0], mxk = k[0], mnv = v[0], mxv = v[0];
#pragma unroll
      for (int i = 1; i < CPL; ++i) {
        mnk = fminf(mnk, k[i]); mxk = fmaxf(mxk, k[i]);
        mnv = fminf(mnv, v[i]); mxv = fmaxf(mxv, v[i]);
      }
      group_minmax<GL>(mnk, mxk);
      group_minmax<GL>(mnv, mxv);
      mk4 = q_meta(mnk, mxk, true, c.clip4, 15.f);
      mv4 = q_meta(mnv, mxv, true, c.clip4, 15.f);
    }
    // salient token -> side table (ascending token order); no shuffles below
    if (sal) {
      const uint32_t below = (t & 31) ? (s_bits[t >> 5] & ((1u << (t & 31)) - 1u)) : 0u;
      int pos = s_base + __popc(below);
      for (int w = 0; w < (t >> 5); ++w) pos += __popc(s_bits[w]);
      uint8_t *se = side_ptr(c, u, pos);
      if (cl == 0) c.side_idx[(size_t)u * c.side_cap + pos] = tok;
      if (tsa) {   // 4-bit per token over G-channel groups, clip4 (R11)
        const int gi = (cl * CPL) / G;
        const QMeta mk = mk4, mv = mv4;
        if ((cl % GL) == 0) {
          reinterpret_cast<float *>(se)[gi] = __fmul_rn(mk.s, c.inv_sqrt_d);
          reinterpret_cast<int32_t *>(se + 4 * NG)[gi] = zero_i32(mk.zf);
          reinterpret_cast<float *>(se + 8 * NG)[gi] = __fmul_rn(mv.s, c.inv_sqrt_d);
          reinterpret_cast<int32_t *>(se + 12 * NG)[gi] = zero_i32(mv.zf);
        }
        uint32_t ck[CPL / 8], cv[CPL / 8];
#pragma unroll
        for (int i = 0; i < CPL / 8; ++i) { ck[i] = 0; cv[i] = 0; }
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
          ck[i / 8] |= q_code(k[i], mk, 15.f) << (4 * (i % 8));
          cv[i / 8] |= q_code(v[i], mv, 15.f) << (4 * (i % 8));
        }
        uint32_t *dk = reinterpret_cast<uint32_t *>(se + 16 * NG + cl * (CPL / 2));
        uint32_t *dv = reinterpret_cast<uint32_t *>(se + 16 * NG + D / 2 + cl * (CPL / 2));
#pragma unroll
        for (int i = 0; i < CPL / 8; ++i) { dk[i] = ck[i]; dv[i] = cv[i]; }
      } else {     // PSA pivot: original 16-bit K and V rows (R10)
        uint4 *dk = reinterpret_cast<uint4 *>(se) + cl * (CPL / 8);
        uint4 *dv = reinterpret_cast<uint4 *>(se + 2 * D) + cl * (CPL / 8);
#pragma unroll
        for (int i = 0; i < CPL / 8; ++i) { dk[i] = kraw[i]; dv[i] = vraw[i]; }
      }
    }
  }
  {
    const unsigned kw = __reduce_max_sync(0xffffffffu, kmax_l), vw = __reduce_max_sync(0xffffffffu, vmax_l);
    if (lane == 0) { atomicMax(&s_kmax, kw); atomicMax(&s_vmax, vw); }
  }
  __syncthreads();

  // ---------------- K: per-channel block stats over non-salient tokens (R1);
  // NS threads per channel each scan G/NS rows, then one combines (min / max
  // are order-independent, so the result is exact)
  if constexpr (!KT) {
    constexpr int NS = kQThreads / D;
    float *red_mn = xs + G * P;                      // [NS][D] after the K rows
    float *red_mx = red_mn + NS * D;
    const int ch = tid % D, part = tid / D;
    float mn = INFINITY, mx = -INFINITY;
    for (int i = part * (G / NS); i < (part + 1) * (G / NS); ++i) {
      const float x = xs[i * P + xs_col(ch)];     // NaN for salient rows: skipped
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    red_mn[part * D + ch] = mn;
    red_mx[part * D + ch] = mx;
    __syncthreads();
    if (tid < D) {
      for (int p2 = 1; p2 < NS; ++p2) {
        mn = fminf(mn, red_mn[p2 * D + ch]);
        mx = fmaxf(mx, red_mx[p2 * D + ch]);
      }
      const bool any = mn <= mx;                     // some non-salient token seen
      const QMeta m = q_meta(any ? mn : 0.f, any ? mx : 0.f, any, c.clip2, 3.f);
      s_s[ch] = m.s; s_z[ch] = m.zf; s_mode[ch] = m.mode;
      s_rs[ch] = m.mode == 0 ? __frcp_rn(m.s) : 0.f;
      const float ks = __fmul_rn(m.s, c.inv_sqrt_d);
      reinterpret_cast<float *>(pg + c.pg_kscale)[ch] = ks;
      reinterpret_cast<int32_t *>(pg + c.pg_kzero)[ch] = zero_i32(m.zf);
      atomicMax(&s_kmax, __float_as_uint(fabsf(ks)));
    }
  }
  __syncthreads();
  if (tid == 0) {   // the unit's fixed-point ranges for the decode kernel (umax)
    atomicMax(reinterpret_cast<unsigned *>(&c.umax[u].x), s_kmax);
    atomicMax(reinterpret_cast<unsigned *>(&c.umax[u].y), s_vmax);
  }
  // ---------------- code words in the page's 4x4 tile layout
  {
    constexpr int TQ = G / 4, CQ = D / 4;
    uint32_t *dk = reinterpret_cast<uint32_t *>(pg + c.pg_kcodes);
    for (int wi = tid; wi < CQ * TQ; wi += kQThreads) {   // K word (cq, tq), cq fastest
      const int cq = wi % CQ, tq = wi / CQ;
      uint32_t word = 0;
      // salient tokens of this token quad: their codes are 0 (mask per byte)
      const uint32_t sb4 = (s_bits[(4 * tq) >> 5] >> ((4 * tq) & 31)) & 15u;
      uint32_t keep = 0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) keep |= ((sb4 >> s2) & 1u) ? 0u : (3u << (2 * s2));
      float xq[4][4];                                // [token s2][channel b]
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        const float4 x4 = *reinterpret_cast<const float4 *>(xs + (4 * tq + s2) * P + xs_col(4 * cq));
        xq[s2][0] = x4.x; xq[s2][1] = x4.y; xq[s2][2] = x4.z; xq[s2][3] = x4.w;
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int ch = 4 * cq + b;
        const float xv[4] = {xq[0][b], xq[1][b], xq[2][b], xq[3][b]};
        uint32_t c4;
        if constexpr (!KT) {                         // one channel's thresholds for the 4 tokens
          QMeta m; m.s = s_s[ch]; m.zf = s_z[ch]; m.mode = s_mode[ch];
          c4 = q_codes2<4>(xv, m, s_rs[ch]);
        } else {                                     // per-token meta
          c4 = 0;
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) {
            const int mi = (4 * tq + s2) * NG + ch / G;
            QMeta m; m.s = s_s[mi]; m.zf = s_z[mi]; m.mode = s_mode[mi];
            const float x1[1] = {xv[s2]};
            c4 |= q_codes2<1>(x1, m, s_rs[mi]) << (2 * s2);
          }
        }
        word |= (c4 & keep) << (8 * b);
      }
      dk[kword_idx(cq, tq, TQ)] = word;
    }
    uint32_t *dv = reinterpret_cast<uint32_t *>(pg + c.pg_vcodes);
    for (int wi = tid; wi < CQ * TQ; wi += kQThreads) {   // V word wi -> (cq, tq)
      const int tq = (wi & 3) + 4 * (wi / (4 * CQ)), cq = (wi / 4) % CQ;
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) word |= (uint32_t)vb8[(4 * tq + b) * (D / 4) + cq] << (8 * b);
      dv[wi] = word;
    }
  }
  if (j == last_block && tid == 0) {  // number of side entries after this block
    int n = s_base;
    for (int w = 0; w < G / 32; ++w) n += __popc(s_bits[w]);
    c.side_cnt[u] = n;
  }
}

// ============================================================ K1e: exact R
// Tokens [t0, t1) quantized one at a time (per-token K only; exact residual
// window, DESIGN R26): the per-token steps of k_quantize_blocks<KT> for
// each token alone -- FWHT, K and V meta per G-channel group (Eqs. 3-6, clip2),
// 2-bit codes written into the token's bits of the page's tile words (K words
// hold 4 tokens per byte: read-modify-write of the token's 2 bits), salient ->
// codes 0, meta (0, 0) and the next side entry (TSA 4-bit, clip4; PSA the
// 16-bit rows).  One warp per unit; the 4 row groups of 8 lanes all transform
// the same row (the shuffle FWHT needs every lane), row group 0 writes.  A
// token that opens a page first zeroes the page, so the decode kernels read
// scale 0 / codes 0 for the tokens not yet quantized (masked like salient).
template <int D, int G, int DT>
__global__ void __launch_bounds__(32) k_quantize_tokens(DevCache c, QuantSrc src, int t0, int t1) {
  constexpr int CPL = D / 8, GL = G / CPL, NG = D / G, TQ = G / 4, CQ = D / 4;
  const int u = blockIdx.x, lane = threadIdx.x, cl = lane & 7;
  const bool w0 = lane < 8;                  // row group 0 writes
  const uint32_t *bm = c.bitmask + (size_t)u * c.bm_words;
  const bool tsa = c.kind == AKVQ_TSA;
  int cnt = c.side_cnt[u];
  unsigned kmax_l = 0u, vmax_l = 0u;
  for (int tok = t0; tok < t1; ++tok) {
    const int j = tok / G, t = tok % G;
    uint8_t *pg = page_ptr(c, u, j);
    if (t == 0) {                            // a fresh page: zero it
      uint4 *z = reinterpret_cast<uint4 *>(pg);
      for (int i = lane; i < (int)(c.page_bytes / 16); i += 32) z[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
    }
    const bool sal = (bm[tok >> 5] >> (tok & 31)) & 1u;
    const size_t roff = (size_t)u * src.unit_stride +
                        (size_t)(src.ring_slots ? tok % src.ring_slots : tok) * src.tok_stride;
    const uint4 *kr = reinterpret_cast<const uint4 *>(src.K + roff + cl * CPL);
    const uint4 *vr = reinterpret_cast<const uint4 *>(src.V + roff + cl * CPL);
    uint4 kraw[CPL / 8], vraw[CPL / 8];
#pragma unroll
    for (int i = 0; i < CPL / 8; ++i) { kraw[i] = kr[i]; vraw[i] = vr[i]; }
    float k[CPL], v[CPL];
#pragma unroll
    for (int i = 0; i < CPL / 8; ++i) { cvt8<DT>(kraw[i], k + 8 * i); cvt8<DT>(vraw[i], v + 8 * i); }
    fwht_lanes8<CPL>(k, cl);
    fwht_lanes8<CPL>(v, cl);
    const int gi = (cl * CPL) / G, mi = t * NG + gi;
    float mnk = k[0], mxk = k[0], mnv = v[0], mxv = v[0];
#pragma unroll
    for (int i = 1; i < CPL; ++i) {
      mnk = fminf(mnk, k[i]); mxk = fmaxf(mxk, k[i]);
      mnv = fminf(mnv, v[i]); mxv = fmaxf(mxv, v[i]);
    }
    group_minmax<GL>(mnk, mxk);
    group_minmax<GL>(mnv, mxv);
    const QMeta mk = q_meta(mnk, mxk, !sal, c.clip2, 3.f);
    const QMeta mv = q_meta(mnv, mxv, !sal, c.clip2, 3.f);
    const uint32_t ck = q_codes2<CPL>(k, mk, mk.mode == 0 ? __frcp_rn(mk.s) : 0.f);
    const uint32_t cv = q_codes2<CPL>(v, mv, mv.mode == 0 ? __frcp_rn(mv.s) : 0.f);
    if (w0) {
      if ((cl % GL) == 0) {
        const float ks = sal ? 0.f : __fmul_rn(mk.s, c.inv_sqrt_d);
        const float vs = sal ? 0.f : __fmul_rn(mv.s, c.inv_sqrt_d);
        reinterpret_cast<float *>(pg + c.pg_kscale)[mi] = ks;
        reinterpret_cast<int32_t *>(pg + c.pg_kzero)[mi] = sal ? 0 : zero_i32(mk.zf);
        reinterpret_cast<float *>(pg + c.pg_vscale)[mi] = vs;
        reinterpret_cast<int32_t *>(pg + c.pg_vzero)[mi] = sal ? 0 : zero_i32(mv.zf);
        kmax_l = max(kmax_l, __float_as_uint(fabsf(ks)));
        vmax_l = max(vmax_l, __float_as_uint(fabsf(vs)));
      }
      uint8_t *kc = pg + c.pg_kcodes, *vc = pg + c.pg_vcodes;
      const int sh = 2 * (t & 3);
#pragma unroll
      for (int i = 0; i < CPL; ++i) {        // K: the token's 2 bits of channel ch's byte
        const int ch = cl * CPL + i;
        uint8_t *b = kc + 4 * kword_idx(ch >> 2, t >> 2, TQ) + (ch & 3);
        *b = (uint8_t)((*b & ~(3u << sh)) | (((ck >> (2 * i)) & 3u) << sh));
      }
#pragma unroll
      for (int i = 0; i < CPL / 4; ++i)      // V: the token's S:146 byte per channel quad
        vc[4 * vword_idx(cl * (CPL / 4) + i, t >> 2, CQ) + (t & 3)] = (uint8_t)(cv >> (8 * i));
    }
    if (sal) {                               // next side entry (ascending token order)
      uint8_t *se = side_ptr(c, u, cnt);
      if (lane == 0) c.side_idx[(size_t)u * c.side_cap + cnt] = tok;
      if (tsa) {   // 4-bit per token over G-channel groups, clip4 (R11)
        const QMeta mk4 = q_meta(mnk, mxk, true, c.clip4, 15.f);
        const QMeta mv4 = q_meta(mnv, mxv, true, c.clip4, 15.f);
        if (w0) {
          if ((cl % GL) == 0) {
            reinterpret_cast<float *>(se)[gi] = __fmul_rn(mk4.s, c.inv_sqrt_d);
            reinterpret_cast<int32_t *>(se + 4 * NG)[gi] = zero_i32(mk4.zf);
            reinterpret_cast<float *>(se + 8 * NG)[gi] = __fmul_rn(mv4.s, c.inv_sqrt_d);
            reinterpret_cast<int32_t *>(se + 12 * NG)[gi] = zero_i32(mv4.zf);
          }
          uint32_t c4k[CPL / 8], c4v[CPL / 8];
#pragma unroll
          for (int i = 0; i < CPL / 8; ++i) { c4k[i] = 0; c4v[i] = 0; }
#pragma unroll
          for (int i = 0; i < CPL; ++i) {
            c4k[i / 8] |= q_code(k[i], mk4, 15.f) << (4 * (i % 8));
            c4v[i / 8] |= q_code(v[i], mv4, 15.f) << (4 * (i % 8));
          }
          uint32_t *dk = reinterpret_cast<uint32_t *>(se + 16 * NG + cl * (CPL / 2));
          uint32_t *dv = reinterpret_cast<uint32_t *>(se + 16 * NG + D / 2 + cl * (CPL / 2));
#pragma unroll
          for (int i = 0; i < CPL / 8; ++i) { dk[i] = c4k[i]; dv[i] = c4v[i]; }
        }
      } else if (w0) {   // PSA pivot: original 16-bit K and V rows (R10)
        uint4 *dk = reinterpret_cast<uint4 *>(se) + cl * (CPL / 8);
        uint4 *dv = reinterpret_cast<uint4 *>(se + 2 * D) + cl * (CPL / 8);
#pragma unroll
        for (int i = 0; i < CPL / 8; ++i) { dk[i] = kraw[i]; dv[i] = vraw[i]; }
      }
      ++cnt;
    }
    __syncwarp();
  }
  const unsigned kw = __reduce_max_sync(0xffffffffu, kmax_l), vw = __reduce_max_sync(0xffffffffu, vmax_l);
  if (lane == 0) {
    c.side_cnt[u] = cnt;
    atomicMax(reinterpret_cast<unsigned *>(&c.umax[u].x), kw);
    atomicMax(reinterpret_cast<unsigned *>(&c.umax[u].y), vw);
  }
}

// ============================================================ K1t / K3
// Copy rows [t0, t1) of K and V (16-bit originals) into the ring (R10).
__global__ void k_ring_fill(DevCache c, const uint16_t *__restrict__ K,
                            const uint16_t *__restrict__ V, int L0, int t0, int t1) {
  const int u = blockIdx.y;
  const int chunks = c.d / 8;                         // uint4 per row
  const int n = (t1 - t0) * 2 * chunks;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int tok = t0 + i / (2 * chunks);
    const int kv = (i / chunks) & 1;
    const int ch = i % chunks;
    const uint16_t *s = (kv ? V : K) + ((size_t)u * L0 + tok) * c.d;
    uint16_t *d = ring_row(c, u, tok % c.slots) + kv * c.d;
    reinterpret_cast<uint4 *>(d)[ch] = reinterpret_cast<const uint4 *>(s)[ch];
  }
}

// Append one token per unit (Eq. 2): ring slot L % slots, salient bit for a
// TSA text token (R12).
__global__ void k_append(DevCache c, const uint16_t *__restrict__ k,
                         const uint16_t *__restrict__ v, const uint8_t *__restrict__ types,
                         int L) {
  const int u = blockIdx.x;
  const int chunks = c.d / 8;
  uint16_t *dst = ring_row(c, u, L % c.slots);
  for (int i = threadIdx.x; i < 2 * chunks; i += blockDim.x) {
    const uint16_t *s = (i < chunks ? k : v) + (size_t)u * c.d;
    reinterpret_cast<uint4 *>(dst + (i < chunks ? 0 : c.d))[i % chunks] =
        reinterpret_cast<const uint4 *>(s)[i % chunks];
  }
  if (threadIdx.x == 0 && c.kind == AKVQ_TSA && types && types[u] == 1)
    c.bitmask[(size_t)u * c.bm_words + L / 32] |= 1u << (L % 32);
  if (u == 0 && threadIdx.x == 0) c.dstate->L = L + 1;   // device copy of L
}

__global__ void k_state_set(DevCache c, int L) {
  c.dstate->L = L;
  c.dstate->done = 0u;
}

// ============================================================ launchers
cudaError_t launch_salient(const DevCache &c, const uint8_t *types, const float *colsum,
                           int L0, int top_k, cudaStream_t st) {
  if (L0 <= 0) return cudaSuccess;
  if (c.kind == AKVQ_TSA) {
    dim3 grid((L0 + 255) / 256, c.U);
    k_salient_tsa<<<grid, 256, 0, st>>>(c, types, L0);
  } else {
    if (top_k <= 0) return cudaSuccess;
    const size_t smem = (size_t)L0 * sizeof(float);
    {
      const cudaError_t ea = cudaFuncSetAttribute(k_salient_psa, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (ea != cudaSuccess) return ea;
    }
    const int nt = L0 >= 8192 ? 1024 : (L0 >= 1024 ? 512 : 128);
    k_salient_psa<<<c.U, nt, smem, st>>>(c, colsum, L0, top_k);
  }
  return cudaGetLastError();
}

template <int D, int G, int DT>
static cudaError_t launch_q(const DevCache &c, const QuantSrc &src, int block0, int nblocks,
                            int last_block, cudaStream_t st) {
  const size_t smem = ((size_t)G * (D + 4) + 2 * (size_t)kQThreads) * sizeof(float);
  auto kern = c.k_axis == AKVQ_K_PER_TOKEN ? k_quantize_blocks<D, G, DT, true>
                                           : k_quantize_blocks<D, G, DT, false>;
  {
    const cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
  }
  dim3 grid(nblocks, c.U);
  kern<<<grid, kQThreads, smem, st>>>(c, src, block0, last_block);
  return cudaGetLastError();
}

cudaError_t launch_quantize_blocks(const DevCache &c, int dtype16, const QuantSrc &src,
                                   int block0, int nblocks, int last_block, cudaStream_t st) {
  if (nblocks <= 0) return cudaSuccess;
#define AKVQ_QCASE(D_, G_)                                                              \
  if (c.d == D_ && c.G == G_)                                                           \
    return dtype16 == AKVQ_BF16 ? launch_q<D_, G_, AKVQ_BF16>(c, src, block0, nblocks, last_block, st) \
                                : launch_q<D_, G_, AKVQ_FP16>(c, src, block0, nblocks, last_block, st);
  AKVQ_QCASE(64, 32)
  AKVQ_QCASE(64, 64)
  AKVQ_QCASE(128, 32)
  AKVQ_QCASE(128, 64)
  AKVQ_QCASE(128, 128)
#undef AKVQ_QCASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_quantize_tokens(const DevCache &c, int dtype16, const QuantSrc &src, int t0,
                                   int t1, cudaStream_t st) {
  if (t1 <= t0) return cudaSuccess;
#define AKVQ_TCASE(D_, G_)                                                              \
  if (c.d == D_ && c.G == G_) {                                                         \
    if (dtype16 == AKVQ_BF16) k_quantize_tokens<D_, G_, AKVQ_BF16><<<c.U, 32, 0, st>>>(c, src, t0, t1); \
    else k_quantize_tokens<D_, G_, AKVQ_FP16><<<c.U, 32, 0, st>>>(c, src, t0, t1);       \
    return cudaGetLastError();                                                          \
  }
  AKVQ_TCASE(64, 32)
  AKVQ_TCASE(64, 64)
  AKVQ_TCASE(128, 32)
  AKVQ_TCASE(128, 64)
  AKVQ_TCASE(128, 128)
#undef AKVQ_TCASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_ring_fill(const DevCache &c, const void *K, const void *V, int L0, int t0,
                             int t1, cudaStream_t st) {
  if (t1 <= t0) return cudaSuccess;
  const int n = (t1 - t0) * 2 * (c.d / 8);
  dim3 grid((n + 255) / 256, c.U);
  k_ring_fill<<<grid, 256, 0, st>>>(c, (const uint16_t *)K, (const uint16_t *)V, L0, t0, t1);
  return cudaGetLastError();
}

cudaError_t launch_state_set(const DevCache &c, int L, cudaStream_t st) {
  k_state_set<<<1, 1, 0, st>>>(c, L);
  return cudaGetLastError();
}

cudaError_t launch_append(const DevCache &c, const void *k, const void *v, const uint8_t *types,
                          int L, cudaStream_t st) {
  k_append<<<c.U, 2 * (c.d / 8), 0, st>>>(c, (const uint16_t *)k, (const uint16_t *)v, types, L);
  return cudaGetLastError();
}

}  // namespace akvq
