// decode_pages.cu -- the hot loop of AKVQ-VL decode on sm_100a: single-query
// attention over the 2-bit pages (P:246-262 quantization, S:486-494 attention).
//
// Persistent warps stream the flattened (unit, page) list; each warp owns a
// contiguous range and double-buffers whole pages (one G-token block: K meta,
// K codes, V meta, V codes, contiguous in HBM) into shared memory with 1-D TMA
// bulk copies (cp.async.bulk + mbarrier).  Dequantize-and-dot runs on the
// integer dp4a path (profiles/r01_microbench_pipes.md):
//   logits:  q~ prescaled by the page's per-channel K scale, rounded to a 16-bit
//            fixed-point integer per page (2 int8 limbs), dotted with the codes
//            as bytes: sum_c Qq_c * (code_tc - z_c) exactly in int32, then
//            logit = alpha * delta * sum                           (Eqs. 3-4)
//   values:  softmax weights w_t = p_t * s^V_t rounded to 24-bit fixed point of
//            the page's largest weight (3 uint8 limbs); codes of 4 tokens are
//            transposed into bytes with PRMT and accumulated with dp4a:
//            o'_c += delta_w * sum_t W_t code_tc - sum_t w_t z_t
// Online softmax (base 2) per warp; each (warp, unit) segment writes a partial
// (m, l, o') that k_combine merges with the ring / side partials.
#include <math.h>

#include "decode_common.cuh"

namespace akvq {

constexpr int kPgWarps = 4;
constexpr int kStages = 3;
constexpr int kQMax = 32767;       // K-side fixed point: |Q| <= 2^15 - 1 (2 limbs)
constexpr int kWMax = 65535;       // V-side fixed point: W <= 2^16 - 1 (2 limbs)

// Per-warp shared-memory block (bytes): kStages half-page stages, q~, limbs,
// transposed value weights, barriers.  sb = stage bytes (>= either page half).
template <int D, int G, int NH>
struct PgSmem {
  static constexpr int NG = D / G;
  static __host__ __device__ size_t qh_off(size_t sb) { return kStages * sb; }
  static __host__ __device__ size_t limb_off(size_t sb) { return qh_off(sb) + NH * D * 4; }
  static __host__ __device__ size_t wt_off(size_t sb) { return limb_off(sb) + NH * 32 * 16; }
  static __host__ __device__ size_t bar_off(size_t sb) {
    return (wt_off(sb) + NH * NG * 2 * G + 15) / 16 * 16;
  }
  static __host__ __device__ size_t warp_bytes(size_t sb) {
    return (bar_off(sb) + kStages * 8 + 127) / 128 * 128;
  }
};

__host__ __device__ inline size_t pg_stage_bytes(size_t page_bytes, size_t pg_vscale) {
  const size_t a = pg_vscale, b = page_bytes - pg_vscale;
  return ((a > b ? a : b) + 127) / 128 * 128;
}

template <int D, int G, int DT, int NH>
__global__ void __launch_bounds__(kPgWarps * 32, 3)
    k_decode_pages(DevCache c, PagePlan pp, RowPlan rp, const uint16_t *__restrict__ q,
                   float *__restrict__ pg_part, const float *__restrict__ rw_part,
                   float *__restrict__ out, uint32_t flags) {
  using S = PgSmem<D, G, NH>;
  constexpr int NG = D / G;
  constexpr int KWL = D / 32;       // code words per lane in the K phase (2 lanes / token)
  constexpr int KPR = D / 16;       // code words per row = lanes per row in the V phase
  constexpr int NTG = 32 / KPR;     // token sub-groups in the V phase
  constexpr int PASSES = G / 16;    // K-phase passes of 16 tokens
  constexpr int GQ = G / 4;         // dp4a token groups of 4 (tokens gi + GQ*i)
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t SB = pg_stage_bytes(c.page_bytes, c.pg_vscale);
  uint8_t *wsm = smem + (size_t)warp * S::warp_bytes(SB);
  float *qh = reinterpret_cast<float *>(wsm + S::qh_off(SB));
  uint4 *limbs = reinterpret_cast<uint4 *>(wsm + S::limb_off(SB));
  uint8_t *wt = wsm + S::wt_off(SB);                    // [NH][NG][3 limbs][G] bytes
  uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + S::bar_off(SB));

  pdl_launch_dependents();                      // let the next layer's kernels queue up
  const int gw = blockIdx.x * kPgWarps + warp;
  if (gw >= (int)pp.W) return;
  const int ib = seg_begin((int)pp.T, (int)pp.W, gw), ie = seg_begin((int)pp.T, (int)pp.W, gw + 1);
  if (ib >= ie) return;
  const int npg = pp.n_pages;
  const int nsub = 2 * (ie - ib);               // two half-page loads per page
  const float alpha = kLog2e / (float)D;       // (q.H_s) . K^ / d in log2 units
  const uint32_t kbytes = c.pg_vscale, vbytes = c.page_bytes - c.pg_vscale;

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bar[s]);
    mbar_fence_init();
  }
  __syncwarp();
  // producer cursor (lane 0): sub-load pi is page (pu, pp_) K half (even) or V half (odd)
  int pi = 0, pu = ib / npg, ppg = ib - (ib / npg) * npg, pst = 0;
  auto issue_next = [&]() {
    const uint8_t *src = page_ptr(c, pu, ppg) + ((pi & 1) ? kbytes : 0u);
    const uint32_t nb = (pi & 1) ? vbytes : kbytes;
    mbar_expect_tx(&bar[pst], nb);
    bulk_g2s(wsm + (size_t)pst * SB, src, nb, &bar[pst]);
    if (pi & 1) { if (++ppg == npg) { ppg = 0; ++pu; } }
    ++pi;
    if (++pst == kStages) pst = 0;
  };
  if (lane == 0)
    for (int s = 0; s < kStages && s < nsub; ++s) issue_next();

  // per-head running state (online softmax, base 2)
  float m_run[NH], l_run[NH], Z[NH][NG], o[NH][16];
  float lgp[NH][PASSES];                        // page logits between the two halves
  int cur_u = -1;
  const int u_first = ib / npg;

  const int tq = lane >> 1, half = lane & 1;                // K phase
  const int kw = lane % KPR, tg = lane / KPR;               // V phase
  const int gam = (16 * kw) / G;                            // V channel group of this lane

  auto flush = [&](int u) {
    const size_t slot = (size_t)gw * pp.maxseg + (u - u_first);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      float zg = Z[h][0];
#pragma unroll
      for (int gi = 1; gi < NG; ++gi) if (gi == gam) zg = Z[h][gi];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float v = o[h][k];
#pragma unroll
        for (int off = KPR; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        o[h][k] = v - zg;
      }
      float *rec = pg_part + (slot * NH + h) * Rec<D>::P;
      if (tg == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          reinterpret_cast<float4 *>(rec + 16 * kw)[k] =
              make_float4(o[h][4 * k], o[h][4 * k + 1], o[h][4 * k + 2], o[h][4 * k + 3]);
      }
      if (lane == 0) { rec[D] = m_run[h]; rec[D + 1] = l_run[h]; }
    }
    // the last page warp of unit u merges it with the row kernel's segments
    int w_lo, w_hi;
    seg_range((int)pp.T, (int)pp.W, pp.n_pages, u, w_lo, w_hi);
    if (take_ticket(c, u, (int)(w_hi - w_lo + 1), lane)) {
      pdl_wait();                                  // row partials of the preceding grid
      merge_unit<D, NH>(c, pp, rp, pg_part, rw_part, u, out, flags, lane);
      if (lane == 0) c.ticket[u] = 0u;
    }
  };

  int u = u_first, pg = ib - u_first * npg;       // (unit, page) of the current sub-load
  int st = 0;
  uint32_t par = 0;
  for (int si = 0; si < nsub; ++si) {
    const uint8_t *B = wsm + (size_t)st * SB;
    if (pp.stream_only) {                          // profiling: pipeline only
      mbar_wait(&bar[st], par);
      __syncwarp();
      if (lane == 0 && pi < nsub) issue_next();
      if (++st == kStages) { st = 0; par ^= 1u; }
      continue;
    }
    if ((si & 1) == 0) {
      if (si > 0 && ++pg == npg) { pg = 0; ++u; }
      if (u != cur_u) {
        if (cur_u >= 0) flush(cur_u);
        cur_u = u;
        // q~ = q . H_s for this unit: lane holds D/32 contiguous channels,
        // in-register butterflies then shuffle butterflies (unnormalized FWHT)
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          constexpr int CPL = D / 32;
          float x[CPL];
          const uint16_t *qs = q + ((size_t)u * c.g + h) * D + CPL * lane;
          if constexpr (CPL == 4) {
            const uint2 v = *reinterpret_cast<const uint2 *>(qs);
            x[0] = H16<DT>::to_f((uint16_t)(v.x & 0xffff)); x[1] = H16<DT>::to_f((uint16_t)(v.x >> 16));
            x[2] = H16<DT>::to_f((uint16_t)(v.y & 0xffff)); x[3] = H16<DT>::to_f((uint16_t)(v.y >> 16));
          } else {
            const uint32_t v = *reinterpret_cast<const uint32_t *>(qs);
            x[0] = H16<DT>::to_f((uint16_t)(v & 0xffff)); x[1] = H16<DT>::to_f((uint16_t)(v >> 16));
          }
#pragma unroll
          for (int hs = 1; hs < CPL; hs <<= 1)
#pragma unroll
            for (int k = 0; k < CPL; ++k)
              if (!(k & hs)) { const float a = x[k], b = x[k + hs]; x[k] = a + b; x[k + hs] = a - b; }
#pragma unroll
          for (int lm = 1; lm < 32; lm <<= 1) {
            const bool upper = lane & lm;
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              const float o2 = __shfl_xor_sync(0xffffffffu, x[k], lm);
              x[k] = upper ? o2 - x[k] : x[k] + o2;
            }
          }
#pragma unroll
          for (int k = 0; k < CPL; ++k) qh[h * D + CPL * lane + k] = x[k];
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          m_run[h] = -INFINITY; l_run[h] = 0.f;
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) Z[h][gi] = 0.f;
#pragma unroll
          for (int k = 0; k < 16; ++k) o[h][k] = 0.f;
        }
      }
      mbar_wait(&bar[st], par);
      // ============== K half: logits of the page's G tokens
      const float *ks = reinterpret_cast<const float *>(B + c.pg_kscale);
      const int32_t *kz = reinterpret_cast<const int32_t *>(B + c.pg_kzero);
      const uint8_t *kc = B + c.pg_kcodes;
      const uint32_t *bmw = c.bitmask + (size_t)u * c.bm_words + (size_t)pg * (G / 32);
      uint32_t bits[G / 32];
#pragma unroll
      for (int w = 0; w < G / 32; ++w) bits[w] = __ldg(bmw + w);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        // per-page fixed-point limbs of qs_c = q~_c * s^K_c (22 bits, 3 bytes)
        float bias, delta;
        {
          const int k = lane >> 2, s = lane & 3;
          int Qv[4] = {0, 0, 0, 0};
          float qsb[4] = {0.f, 0.f, 0.f, 0.f};
          float am = 0.f;
          if (k < D / 16) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int ch = 16 * k + 4 * b + s;
              qsb[b] = qh[h * D + ch] * ks[ch];
              am = fmaxf(am, fabsf(qsb[b]));
            }
          }
          const float M = warp_max(am);
          const float inv = M > 0.f ? (float)kQMax / M : 0.f;
          delta = M > 0.f ? M / (float)kQMax : 0.f;
          long long bq = 0;   // zero-point bias from the same fixed-point q (exact, 64-bit)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            Qv[b] = __float2int_rn(qsb[b] * inv);
            if (k < D / 16) bq += (long long)Qv[b] * kz[16 * k + 4 * b + s];
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) bq += __shfl_xor_sync(0xffffffffu, bq, o);
          bias = delta * (float)bq;
          const uint32_t lo = prmt(prmt(Qv[0], Qv[1], 0x0040), prmt(Qv[2], Qv[3], 0x0040), 0x5410);
          const uint32_t hi = prmt(prmt(Qv[0], Qv[1], 0x0051), prmt(Qv[2], Qv[3], 0x0051), 0x5410);
          limbs[h * 32 + lane] = make_uint4(lo, hi, 0u, 0u);
        }
        __syncwarp();
        uint32_t lim[KWL][4][2];
#pragma unroll
        for (int w = 0; w < KWL; ++w)
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint2 v = *reinterpret_cast<const uint2 *>(&limbs[h * 32 + 4 * (half * KWL + w) + s]);
            lim[w][s][0] = v.x; lim[w][s][1] = v.y;
          }
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
          const int t = ps * 16 + tq;
          uint32_t wd[KWL];
          if constexpr (KWL == 4) {
            const uint4 v = *reinterpret_cast<const uint4 *>(kc + (size_t)t * (D / 4) + half * 16);
            wd[0] = v.x; wd[1] = v.y; wd[2] = v.z; wd[3] = v.w;
          } else {
            const uint2 v = *reinterpret_cast<const uint2 *>(kc + (size_t)t * (D / 4) + half * 8);
            wd[0] = v.x; wd[1] = v.y;
          }
          // two independent accumulator sets (even / odd words) to halve the
          // dp4a dependency chains
          int a0[2] = {0, 0}, a1[2] = {0, 0};
#pragma unroll
          for (int w = 0; w < KWL; ++w)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t x = (wd[w] >> (2 * s)) & 0x03030303u;
              a0[w & 1] = dp4a_uu(x, lim[w][s][0], a0[w & 1]);
              a1[w & 1] = dp4a_us(x, lim[w][s][1], a1[w & 1]);
            }
          int tot = (a1[0] + a1[1]) * 256 + (a0[0] + a0[1]);
          tot += __shfl_xor_sync(0xffffffffu, tot, 1);
          const bool sal = (bits[t >> 5] >> (t & 31)) & 1u;
          lgp[h][ps] = sal ? -INFINITY : alpha * fmaf((float)tot, delta, -bias);
        }
        __syncwarp();
      }
    } else {
      mbar_wait(&bar[st], par);
      // ============== V half: online softmax update and value accumulation
      const float *vs = reinterpret_cast<const float *>(B);
      const int32_t *vz = reinterpret_cast<const int32_t *>(B + (c.pg_vzero - c.pg_vscale));
      const uint8_t *vc = B + (c.pg_vcodes - c.pg_vscale);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        float mloc = lgp[h][0];
#pragma unroll
        for (int ps = 1; ps < PASSES; ++ps) mloc = fmaxf(mloc, lgp[h][ps]);
#pragma unroll
        for (int off = 2; off < 32; off <<= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, off));
        const float m_new = fmaxf(m_run[h], mloc);
        if (m_new == -INFINITY) continue;                  // nothing unmasked yet (warp-uniform)
        const float sc = exp2f(m_run[h] - m_new);
        float pr[PASSES], psum = 0.f;
#pragma unroll
        for (int ps = 0; ps < PASSES; ++ps) {
          pr[ps] = exp2f(lgp[h][ps] - m_new);
          psum += pr[ps];
        }
#pragma unroll
        for (int off = 2; off < 32; off <<= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
        l_run[h] = l_run[h] * sc + psum;
        m_run[h] = m_new;
        float dwl = 0.f;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          float wv[PASSES], wmax = 0.f;
#pragma unroll
          for (int ps = 0; ps < PASSES; ++ps) {
            const int t = ps * 16 + tq;
            wv[ps] = pr[ps] * vs[t * NG + gi];
            wmax = fmaxf(wmax, wv[ps]);
          }
#pragma unroll
          for (int off = 2; off < 32; off <<= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
          // 16-bit fixed point of the page's largest weight (2 uint8 limbs).  The
          // zero-point term uses the same rounded weights, so the rounding error
          // multiplies (code - z) -- a dequantized row -- and stays incoherent
          // across channels (with the exact w it multiplied code >= 0 and piled
          // up in output channel 0 under H).
          const float invw = wmax > 0.f ? (float)kWMax / wmax : 0.f;
          const float dw = wmax / (float)kWMax;
          if (gi == gam) dwl = dw;
          long long zq = 0;                          // sum_t W_t z_t, exact
          uint8_t *wl = wt + (h * NG + gi) * 2 * G;
#pragma unroll
          for (int ps = 0; ps < PASSES; ++ps) {
            const int t = ps * 16 + tq;
            const uint32_t W = min(__float2uint_rn(wv[ps] * invw), (uint32_t)kWMax);  // may round up
            if (half == 0) {
              zq += (long long)W * vz[t * NG + gi];
              const int idx = (t % GQ) * 4 + t / GQ;
              wl[idx] = (uint8_t)W;
              wl[G + idx] = (uint8_t)(W >> 8);
            }
          }
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) zq += __shfl_xor_sync(0xffffffffu, zq, off);
          Z[h][gi] = Z[h][gi] * sc + dw * (float)zq;
        }
        __syncwarp();
        // o'_c += sum_t W_t code_tc  (dp4a over 4 tokens, codes transposed by PRMT)
        int a0[16], a1[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) { a0[k] = 0; a1[k] = 0; }
        const uint8_t *wl = wt + (h * NG + gam) * 2 * G;
#pragma unroll 2
        for (int gi = tg; gi < GQ; gi += NTG) {
          const uint32_t w0 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi) * (D / 4) + 4 * kw);
          const uint32_t w1 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + GQ) * (D / 4) + 4 * kw);
          const uint32_t w2 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + 2 * GQ) * (D / 4) + 4 * kw);
          const uint32_t w3 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + 3 * GQ) * (D / 4) + 4 * kw);
          const uint32_t l0 = *reinterpret_cast<const uint32_t *>(wl + 4 * gi);
          const uint32_t l1 = *reinterpret_cast<const uint32_t *>(wl + G + 4 * gi);
          const uint32_t ta = prmt(w0, w1, 0x5140), tb = prmt(w0, w1, 0x7362);
          const uint32_t tc = prmt(w2, w3, 0x5140), td = prmt(w2, w3, 0x7362);
          const uint32_t Gb[4] = {prmt(ta, tc, 0x5410), prmt(ta, tc, 0x7632), prmt(tb, td, 0x5410),
                                  prmt(tb, td, 0x7632)};
#pragma unroll
          for (int bb = 0; bb < 4; ++bb)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint32_t x = Gb[bb] & (0x03030303u << (2 * s));   // code * 4^s per byte
              a0[bb * 4 + s] = dp4a_uu(x, l0, a0[bb * 4 + s]);
              a1[bb * 4 + s] = dp4a_uu(x, l1, a1[bb * 4 + s]);
            }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float sck = dwl * (1.0f / (float)(1 << (2 * (k & 3))));
          const float val = (float)(a1[k] * 256 + a0[k]);          // < 2^31: 32 tokens x 192 x 65535
          o[h][k] = fmaf(val, sck, o[h][k] * sc);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && pi < nsub) issue_next();        // refills stage st
    if (++st == kStages) { st = 0; par ^= 1u; }
  }
  if (cur_u >= 0 && !pp.stream_only) flush(cur_u);
}

// Shared memory bytes of one CTA of the page kernel.
template <int D, int G, int NH>
static size_t pg_smem(size_t sb) {
  return (size_t)kPgWarps * PgSmem<D, G, NH>::warp_bytes(sb);
}

template <int D, int G, int DT, int NH>
static cudaError_t launch_pg(const DevCache &c, const PagePlan &pp, const RowPlan &rp, const void *q,
                             float *pg_part, const float *rw_part, float *out, uint32_t flags,
                             cudaStream_t st) {
  const size_t smem = pg_smem<D, G, NH>(pg_stage_bytes(c.page_bytes, c.pg_vscale));
  auto kern = k_decode_pages<D, G, DT, NH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((pp.W + kPgWarps - 1) / kPgWarps));
  cfg.blockDim = dim3(kPgWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap the row kernel's tail
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c, pp, rp, (const uint16_t *)q, pg_part, rw_part, out, flags);
}

int pages_fast_supported(int d, int G, int g) {
  return (d == 128 || d == 64) && G >= 32 && G <= d && (g == 1 || g == 2 || g == 4);
}

int pages_warps_per_cta() { return kPgWarps; }

size_t pages_smem_bytes(int d, int G, int g, size_t page_bytes) {
#define AKVQ_SM(D_, G_)                                                               \
  if (d == D_ && G == G_)                                                             \
    return g == 1 ? pg_smem<D_, G_, 1>(page_bytes)                                    \
                  : (g == 2 ? pg_smem<D_, G_, 2>(page_bytes) : pg_smem<D_, G_, 4>(page_bytes));
  AKVQ_SM(64, 32)
  AKVQ_SM(64, 64)
  AKVQ_SM(128, 32)
  AKVQ_SM(128, 64)
  AKVQ_SM(128, 128)
#undef AKVQ_SM
  return 0;
}

template <int D, int G, int DT>
static cudaError_t launch_pg_g(const DevCache &c, const PagePlan &pp, const RowPlan &rp,
                               const void *q, float *pg_part, const float *rw_part, float *out,
                               uint32_t flags, cudaStream_t st) {
  if (c.g == 1) return launch_pg<D, G, DT, 1>(c, pp, rp, q, pg_part, rw_part, out, flags, st);
  if (c.g == 2) return launch_pg<D, G, DT, 2>(c, pp, rp, q, pg_part, rw_part, out, flags, st);
  return launch_pg<D, G, DT, 4>(c, pp, rp, q, pg_part, rw_part, out, flags, st);
}

cudaError_t launch_decode_pages(const DevCache &c, int dtype16, const PagePlan &pp,
                                const RowPlan &rp, const void *q, float *pg_part,
                                const float *rw_part, float *out, uint32_t flags, cudaStream_t st) {
  if (pp.T <= 0) return cudaSuccess;
#define AKVQ_PCASE(D_, G_)                                                                         \
  if (c.d == D_ && c.G == G_)                                                                      \
    return dtype16 == AKVQ_BF16                                                                    \
               ? launch_pg_g<D_, G_, AKVQ_BF16>(c, pp, rp, q, pg_part, rw_part, out, flags, st)   \
               : launch_pg_g<D_, G_, AKVQ_FP16>(c, pp, rp, q, pg_part, rw_part, out, flags, st);
  AKVQ_PCASE(64, 32)
  AKVQ_PCASE(64, 64)
  AKVQ_PCASE(128, 32)
  AKVQ_PCASE(128, 64)
  AKVQ_PCASE(128, 128)
#undef AKVQ_PCASE
  return cudaErrorInvalidValue;
}

}  // namespace akvq
