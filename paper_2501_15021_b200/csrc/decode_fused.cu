// decode_fused.cu -- one-launch decode step of the AKVQ-VL cache on sm_100a:
// (optional) append of the new token + single-query attention over every
// tier of one layer's cache + split merge + output H.
//
//   logit_t = q~ . K^_t / sqrt d,  o = softmax(logit) . V^ . H      (Fig. 6-7)
//
// Work: per unit u a cost-weighted item list
//     [P 2-bit pages][ring chunks of RC tokens][side splits]
// flattened over units; warp w of the persistent grid owns the items whose
// start cost lies in [w*T/W, (w+1)*T/W).  Each warp streams its items through a
// 3-stage shared-memory ring filled by 1-D TMA bulk copies (cp.async.bulk +
// mbarrier): a page is two loads (K half: K meta + K codes; V half: V meta + V
// codes), a ring chunk one or two (wrap), a side split one per RC entries.
//
// 2-bit pages use the integer dp4a path (profiles/r01_microbench_pipes.md):
//   K: q~ * s^K per channel as 22-bit fixed point (3 int8 limbs) dotted with
//      codes as bytes; V: softmax weights * s^V as 24-bit fixed point of the
//      page's largest weight (3 uint8 limbs), codes of 4 tokens transposed with
//      PRMT, accumulated with dp4a.
// 16-bit rows (ring, PSA pivots; original basis, R10) and 4-bit TSA rows
// (rotated basis, R11) use fp32 FMAs.
//
// Each (warp, unit) segment runs one online softmax (base 2) with two
// accumulators (rotated / original basis) and writes a partial; the last warp
// to finish a unit (per-unit ticket) merges the partials, applies H and
// writes the output row, then resets the ticket.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace akvq {

constexpr int kFWarps = 4;
constexpr int kFStages = 3;

__device__ __forceinline__ uint32_t f_smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void f_mbar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(f_smem_u32(b)) : "memory");
}
__device__ __forceinline__ void f_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(f_smem_u32(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void f_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "FWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra FWAIT_%=;\n}\n" ::"r"(
          f_smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void f_bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          f_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(f_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t f_prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}
__device__ __forceinline__ int f_dp4a_uu(uint32_t a, uint32_t b, int c) {
  int r;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ int f_dp4a_us(uint32_t a, uint32_t b, int c) {
  int r;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
template <int DT>
__device__ __forceinline__ void f_cvt2(uint32_t w, float &a, float &b) {
  if constexpr (DT == AKVQ_BF16) {
    a = __uint_as_float(w << 16);
    b = __uint_as_float(w & 0xffff0000u);
  } else {
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
    a = f.x;
    b = f.y;
  }
}

// Per-warp shared memory: stages, q~ (rotated, unnormalized) and q (original)
// per head, K limbs, V weight limbs, 16-bit-row probabilities, barriers.
template <int D, int G, int NH>
struct FSmem {
  static constexpr int NG = D / G;
  static __host__ __device__ size_t qh_off(size_t sb) { return kFStages * sb; }
  static __host__ __device__ size_t qo_off(size_t sb) { return qh_off(sb) + (size_t)NH * D * 4; }
  static __host__ __device__ size_t limb_off(size_t sb) { return qo_off(sb) + (size_t)NH * D * 4; }
  static __host__ __device__ size_t wt_off(size_t sb) { return limb_off(sb) + (size_t)NH * 32 * 16; }
  static __host__ __device__ size_t bar_off(size_t sb) {
    return (wt_off(sb) + (size_t)NH * NG * 3 * G + 15) / 16 * 16;
  }
  static __host__ __device__ size_t warp_bytes(size_t sb) {
    return (bar_off(sb) + kFStages * 8 + 127) / 128 * 128;
  }
};

// Load schedule of one warp: the flattened (unit, item, sub-load) sequence.
struct FCursor {
  int u, u_hi;          // current unit, last unit of the warp
  int item, item_end;   // current item index within the unit, end (exclusive)
  int sub, n_sub;       // sub-load within the item
  int kind, idx;        // 0 page, 1 ring chunk, 2 side split; index within kind
  int r0, nrows;        // ring / side: first row and rows of the item
  bool done;
};

template <int D, int G, int DT, int NH>
__global__ void __launch_bounds__(kFWarps * 32, 3)
    k_decode_fused(DevCache c, FusedPlan fp, const uint16_t *__restrict__ q,
                   const uint16_t *__restrict__ app_k, const uint16_t *__restrict__ app_v,
                   const uint8_t *__restrict__ app_types, float *__restrict__ part,
                   float *__restrict__ out, uint32_t flags) {
  using S = FSmem<D, G, NH>;
  constexpr int NG = D / G;
  constexpr int KWL = D / 32;       // page K phase: code words per lane (2 lanes / token)
  constexpr int KPR = D / 16;       // V phase: lanes per row (16 channels each)
  constexpr int NTG = 32 / KPR;     // V phase: token sub-groups
  constexpr int PASSES = G / 16;    // page K phase: passes of 16 tokens
  constexpr int GQ = G / 4;         // page V phase: dp4a token groups (tokens gi + GQ*i)
  constexpr int RC = FusedPlan::kRowChunk;   // 16-bit / 4-bit rows per sub-load
  constexpr int RQ = D / 4;         // row K phase: channels per lane (4 lanes / row)
  constexpr int RECH = 2 * D + 4;             // per head: rot[D], org[D], m, l, pad
  constexpr int REC = NH * RECH;              // floats per (slot, all heads) partial
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t SB = fp.stage_bytes;
  uint8_t *wsm = smem + (size_t)warp * S::warp_bytes(SB);
  float *qh = reinterpret_cast<float *>(wsm + S::qh_off(SB));
  float *qo = reinterpret_cast<float *>(wsm + S::qo_off(SB));
  uint4 *limbs = reinterpret_cast<uint4 *>(wsm + S::limb_off(SB));
  uint8_t *wt = wsm + S::wt_off(SB);
  uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + S::bar_off(SB));

  const long long gw = (long long)blockIdx.x * kFWarps + warp;
  if (gw >= fp.W) return;
  const long long cb = gw * fp.T / fp.W, ce = (gw + 1) * fp.T / fp.W;   // cost range
  if (cb >= ce) return;
  const int Cu = fp.cost_unit;
  const int u_lo = (int)(cb / Cu), u_hi = (int)((ce - 1) / Cu);
  const bool tsa = c.kind == AKVQ_TSA;
  const int n_ring = fp.L - fp.n_q;
  const float alpha_q = kLog2e / (float)D;          // (q.H_s) . K^ / d
  const float alpha_o = kLog2e * c.inv_sqrt_d;      // q . k / sqrt d

  if (lane == 0) {
    for (int s = 0; s < kFStages; ++s) f_mbar_init(&bar[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // ---- item schedule ---------------------------------------------------
  // item start costs within a unit: page k -> k*cp; ring r -> P*cp + r*cr;
  // side s -> P*cp + NR*cr + s*cs.  The warp owns items whose start cost is in
  // [cb, ce) (unit-relative window below).
  auto item_start = [&](int it) -> int {
    if (it < fp.P) return it * fp.cp;
    if (it < fp.P + fp.NR) return fp.P * fp.cp + (it - fp.P) * fp.cr;
    return fp.P * fp.cp + fp.NR * fp.cr + (it - fp.P - fp.NR) * fp.cs;
  };
  const int n_items = fp.P + fp.NR + fp.NS;
  // first item with start >= x (x unit-relative)
  auto first_item_ge = [&](int x) -> int {
    int it = 0;
    // pages
    if (x <= 0) return 0;
    const int pc = fp.P * fp.cp;
    if (x <= pc) return (x + fp.cp - 1) / fp.cp;
    it = fp.P;
    const int rc = pc + fp.NR * fp.cr;
    if (x <= rc) return it + (x - pc + fp.cr - 1) / fp.cr;
    it = fp.P + fp.NR;
    const int sc = rc + fp.NS * fp.cs;
    if (x <= sc) return it + (x - rc + fp.cs - 1) / fp.cs;
    return n_items;
  };
  auto set_item = [&](FCursor &k) {
    if (k.item < fp.P) {
      k.kind = 0; k.idx = k.item; k.n_sub = 2; k.r0 = 0; k.nrows = 0;
    } else if (k.item < fp.P + fp.NR) {
      k.kind = 1; k.idx = k.item - fp.P;
      k.r0 = k.idx * RC;
      k.nrows = min(RC, n_ring - k.r0);
      k.n_sub = k.nrows > 0 ? 1 : 0;
    } else {
      k.kind = 2; k.idx = k.item - fp.P - fp.NR;
      const int cnt = c.side_cnt[k.u];
      const int a = (int)((long long)k.idx * cnt / fp.NS);
      const int b = (int)((long long)(k.idx + 1) * cnt / fp.NS);
      k.r0 = a; k.nrows = b - a;
      k.n_sub = (k.nrows + RC - 1) / RC;
    }
    k.sub = 0;
  };
  auto unit_window = [&](FCursor &k) {
    const long long base = (long long)k.u * Cu;
    const int lo = (int)max(0LL, cb - base), hi = (int)min((long long)Cu, ce - base);
    k.item = first_item_ge(lo);
    k.item_end = first_item_ge(hi);
  };
  // advance to the next sub-load (skipping empty items); returns false at unit end
  auto next_in_unit = [&](FCursor &k) -> bool {
    while (true) {
      if (k.item >= k.item_end) return false;
      if (k.sub < k.n_sub) return true;
      ++k.item;
      if (k.item < k.item_end) set_item(k);
    }
  };
  auto start_unit = [&](FCursor &k, int u) {
    k.u = u;
    unit_window(k);
    if (k.item < k.item_end) set_item(k);
  };
  // producer side: issue one sub-load into stage st
  auto issue = [&](const FCursor &k, int st) {
    uint8_t *dst = wsm + (size_t)st * SB;
    if (k.kind == 0) {
      const uint8_t *pg = page_ptr(c, k.u, k.idx);
      const uint32_t kb = c.pg_vscale, vb = c.page_bytes - c.pg_vscale;
      if (k.sub == 0) { f_expect_tx(&bar[st], kb); f_bulk(dst, pg, kb, &bar[st]); }
      else { f_expect_tx(&bar[st], vb); f_bulk(dst, pg + kb, vb, &bar[st]); }
    } else if (k.kind == 1) {
      const int t0 = fp.n_q + k.r0;
      const int s0 = t0 % c.slots;
      const int n = k.nrows;
      const int n1 = min(n, c.slots - s0);
      const uint32_t rb = 4 * D;
      f_expect_tx(&bar[st], (uint32_t)n * rb);
      f_bulk(dst, ring_row(c, k.u, s0), (uint32_t)n1 * rb, &bar[st]);
      if (n1 < n) f_bulk(dst + (size_t)n1 * rb, ring_row(c, k.u, 0), (uint32_t)(n - n1) * rb, &bar[st]);
    } else {
      const int e0 = k.r0 + k.sub * RC;
      const int n = min(RC, k.r0 + k.nrows - e0);
      f_expect_tx(&bar[st], (uint32_t)n * c.side_entry);
      f_bulk(dst, side_ptr(c, k.u, e0), (uint32_t)n * c.side_entry, &bar[st]);
    }
  };

  // producer cursor (lane 0 issues; every lane keeps it in step, it is cheap)
  FCursor pc;
  pc.u_hi = u_hi;
  start_unit(pc, u_lo);
  auto producer_next = [&]() -> bool {   // position pc on the next sub-load
    while (true) {
      if (next_in_unit(pc)) return true;
      if (pc.u >= pc.u_hi) return false;
      start_unit(pc, pc.u + 1);
    }
  };
  bool p_ok = producer_next();
  for (int s = 0; s < kFStages && p_ok; ++s) {
    if (lane == 0) issue(pc, s);
    ++pc.sub;
    p_ok = producer_next();
  }

  // ---- per-lane roles ---------------------------------------------------
  const int tq = lane >> 1, half = lane & 1;         // page K phase
  const int kw = lane % KPR, tg = lane / KPR;        // V phases
  const int gam = (16 * kw) / G;                     // V channel group of this lane
  const int rq = lane >> 2, rc4 = lane & 3;          // row K phase: row, channel quarter

  float m_run[NH], l_run[NH], o_rot[NH][16], o_org[NH][16], Zu[NH], Zl[NH];
  float lgp[NH][PASSES];                            // page logits between the two halves
  int ci = 0;                                        // consumed sub-loads (stage counter)

  for (int u = u_lo; u <= u_hi; ++u) {
    // ---- unit setup: q, q~ and fresh softmax state
    for (int i = lane; i < NH * D; i += 32) {
      const float v = H16<DT>::to_f(q[(size_t)u * c.g * D + i]);
      qh[i] = v;
      qo[i] = v;
    }
    __syncwarp();
#pragma unroll
    for (int hs = 1; hs < D; hs <<= 1) {
      for (int idx = lane; idx < NH * D / 2; idx += 32) {
        const int h = idx / (D / 2), k = idx % (D / 2);
        const int i = (k / hs) * 2 * hs + (k % hs);
        const float a = qh[h * D + i], b = qh[h * D + i + hs];
        qh[h * D + i] = a + b;
        qh[h * D + i + hs] = a - b;
      }
      __syncwarp();
    }
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      m_run[h] = -INFINITY; l_run[h] = 0.f; Zu[h] = 0.f; Zl[h] = 0.f;
#pragma unroll
      for (int k = 0; k < 16; ++k) { o_rot[h][k] = 0.f; o_org[h][k] = 0.f; }
    }
    FCursor cc;
    cc.u_hi = u_hi;
    start_unit(cc, u);
    while (next_in_unit(cc)) {
      const int st = ci % kFStages;
      const uint32_t par = (uint32_t)((ci / kFStages) & 1);
      f_wait(&bar[st], par);
      const uint8_t *B = wsm + (size_t)st * SB;

      if (cc.kind == 0 && cc.sub == 0) {
        // =================== page, K half: logits of the G tokens
        const float *ks = reinterpret_cast<const float *>(B + c.pg_kscale);
        const int32_t *kz = reinterpret_cast<const int32_t *>(B + c.pg_kzero);
        const uint8_t *kc = B + c.pg_kcodes;
        const uint32_t *bmw = c.bitmask + (size_t)u * c.bm_words + (size_t)cc.idx * (G / 32);
        uint32_t bits[G / 32];
#pragma unroll
        for (int w = 0; w < G / 32; ++w) bits[w] = __ldg(bmw + w);
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          float bias, delta;
          {
            const int k = lane >> 2, s = lane & 3;
            int Qv[4] = {0, 0, 0, 0};
            float qsb[4] = {0.f, 0.f, 0.f, 0.f};
            float bp = 0.f, am = 0.f;
            if (k < D / 16) {
#pragma unroll
              for (int b = 0; b < 4; ++b) {
                const int ch = 16 * k + 4 * b + s;
                qsb[b] = qh[h * D + ch] * ks[ch];
                bp = fmaf(qsb[b], (float)kz[ch], bp);
                am = fmaxf(am, fabsf(qsb[b]));
              }
            }
            bias = warp_sum(bp);
            const float M = warp_max(am);
            const float inv = M > 0.f ? 2097151.0f / M : 0.f;   // |Q| <= 2^21 - 1
            delta = M > 0.f ? M / 2097151.0f : 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b) Qv[b] = __float2int_rn(qsb[b] * inv);
            const uint32_t lo = f_prmt(f_prmt(Qv[0], Qv[1], 0x0040), f_prmt(Qv[2], Qv[3], 0x0040), 0x5410);
            const uint32_t mi = f_prmt(f_prmt(Qv[0], Qv[1], 0x0051), f_prmt(Qv[2], Qv[3], 0x0051), 0x5410);
            const uint32_t hi = f_prmt(f_prmt(Qv[0], Qv[1], 0x0062), f_prmt(Qv[2], Qv[3], 0x0062), 0x5410);
            limbs[h * 32 + lane] = make_uint4(lo, mi, hi, 0u);
          }
          __syncwarp();
          uint32_t lim[KWL][4][3];
#pragma unroll
          for (int w = 0; w < KWL; ++w)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              const uint4 v = limbs[h * 32 + 4 * (half * KWL + w) + s];
              lim[w][s][0] = v.x; lim[w][s][1] = v.y; lim[w][s][2] = v.z;
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
            int a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int w = 0; w < KWL; ++w)
#pragma unroll
              for (int s = 0; s < 4; ++s) {
                const uint32_t x = (wd[w] >> (2 * s)) & 0x03030303u;
                a0 = f_dp4a_uu(x, lim[w][s][0], a0);
                a1 = f_dp4a_uu(x, lim[w][s][1], a1);
                a2 = f_dp4a_us(x, lim[w][s][2], a2);
              }
            int tot = a2 * 65536 + a1 * 256 + a0;
            tot += __shfl_xor_sync(0xffffffffu, tot, 1);
            const bool sal = (bits[t >> 5] >> (t & 31)) & 1u;
            lgp[h][ps] = sal ? -INFINITY : alpha_q * fmaf((float)tot, delta, -bias);
          }
          __syncwarp();
        }
      } else if (cc.kind == 0) {
        // =================== page, V half: softmax update and V accumulation
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
          if (m_new == -INFINITY) continue;
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
          Zu[h] *= sc; Zl[h] *= sc;
#pragma unroll
          for (int k = 0; k < 16; ++k) o_org[h][k] *= sc;
          float dwl = 0.f, zsum = 0.f;
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) {
            float wv[PASSES], wmax = 0.f, zs = 0.f;
#pragma unroll
            for (int ps = 0; ps < PASSES; ++ps) {
              const int t = ps * 16 + tq;
              wv[ps] = pr[ps] * vs[t * NG + gi];
              wmax = fmaxf(wmax, wv[ps]);
              zs = fmaf(wv[ps], (float)vz[t * NG + gi], zs);
            }
#pragma unroll
            for (int off = 2; off < 32; off <<= 1) {
              wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
              zs += __shfl_xor_sync(0xffffffffu, zs, off);
            }
            // 24-bit fixed point of the page's largest weight: per-token rounding
            // errors are shared by the token's d channels and add coherently
            // under the output H, so 16 bits are not enough.
            const float invw = wmax > 0.f ? 16777215.0f / wmax : 0.f;
            if (gi == gam) { dwl = wmax / 16777215.0f; zsum = zs; }
            if (half == 0) {
              uint8_t *wl = wt + (h * NG + gi) * 3 * G;
#pragma unroll
              for (int ps = 0; ps < PASSES; ++ps) {
                const int t = ps * 16 + tq;
                const uint32_t W = min(__float2uint_rn(wv[ps] * invw), 16777215u);
                const int idx = (t % GQ) * 4 + t / GQ;
                wl[idx] = (uint8_t)W;
                wl[G + idx] = (uint8_t)(W >> 8);
                wl[2 * G + idx] = (uint8_t)(W >> 16);
              }
            }
          }
          // the page's zero-point sum of this lane's channel group is a full
          // (warp-reduced) sum, so it is subtracted once at the flush, after the
          // token-subgroup reduction of o_rot (unlike the 4-bit rows' Zl).
          Zu[h] += zsum;
          __syncwarp();
          int a0[16], a1[16], a2[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) { a0[k] = 0; a1[k] = 0; a2[k] = 0; }
          const uint8_t *wl = wt + (h * NG + gam) * 3 * G;
#pragma unroll 2
          for (int gi = tg; gi < GQ; gi += NTG) {
            const uint32_t w0 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi) * (D / 4) + 4 * kw);
            const uint32_t w1 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + GQ) * (D / 4) + 4 * kw);
            const uint32_t w2 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + 2 * GQ) * (D / 4) + 4 * kw);
            const uint32_t w3 = *reinterpret_cast<const uint32_t *>(vc + (size_t)(gi + 3 * GQ) * (D / 4) + 4 * kw);
            const uint32_t l0 = *reinterpret_cast<const uint32_t *>(wl + 4 * gi);
            const uint32_t l1 = *reinterpret_cast<const uint32_t *>(wl + G + 4 * gi);
            const uint32_t l2 = *reinterpret_cast<const uint32_t *>(wl + 2 * G + 4 * gi);
            const uint32_t ta = f_prmt(w0, w1, 0x5140), tb = f_prmt(w0, w1, 0x7362);
            const uint32_t tc = f_prmt(w2, w3, 0x5140), td = f_prmt(w2, w3, 0x7362);
            const uint32_t Gb[4] = {f_prmt(ta, tc, 0x5410), f_prmt(ta, tc, 0x7632),
                                    f_prmt(tb, td, 0x5410), f_prmt(tb, td, 0x7632)};
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
#pragma unroll
              for (int s = 0; s < 4; ++s) {
                const uint32_t x = Gb[bb] & (0x03030303u << (2 * s));   // code * 4^s per byte
                a0[bb * 4 + s] = f_dp4a_uu(x, l0, a0[bb * 4 + s]);
                a1[bb * 4 + s] = f_dp4a_uu(x, l1, a1[bb * 4 + s]);
                a2[bb * 4 + s] = f_dp4a_uu(x, l2, a2[bb * 4 + s]);
              }
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const float sck = dwl * (1.0f / (float)(1 << (2 * (k & 3))));
            const float val = fmaf((float)a2[k], 65536.f, fmaf((float)a1[k], 256.f, (float)a0[k]));
            o_rot[h][k] = fmaf(val, sck, o_rot[h][k] * sc);
          }
        }
      } else {
        // =================== 16-bit rows (ring / PSA side) or TSA 4-bit rows
        const bool rows16 = cc.kind == 1 || !tsa;
        const int e0 = cc.kind == 1 ? cc.r0 : cc.r0 + cc.sub * RC;
        const int n = cc.kind == 1 ? cc.nrows : min(RC, cc.r0 + cc.nrows - e0);
        uint8_t *Bw = wsm + (size_t)st * SB;
        // the newest token: attend to the caller's row (the ring slot is written
        // here, after the stale copy was loaded), append it to the ring (Eq. 2)
        if (app_k != nullptr && cc.kind == 1) {
          const int tl = fp.L - 1 - (fp.n_q + e0);
          if (tl >= 0 && tl < n) {
            const uint16_t *sk = app_k + (size_t)u * D, *sv = app_v + (size_t)u * D;
            uint16_t *rr = ring_row(c, u, (fp.L - 1) % c.slots);
            for (int i = lane; i < D / 8; i += 32) {
              const uint4 kv = reinterpret_cast<const uint4 *>(sk)[i];
              const uint4 vv = reinterpret_cast<const uint4 *>(sv)[i];
              reinterpret_cast<uint4 *>(Bw + (size_t)tl * 4 * D)[i] = kv;
              reinterpret_cast<uint4 *>(Bw + (size_t)tl * 4 * D + 2 * D)[i] = vv;
              reinterpret_cast<uint4 *>(rr)[i] = kv;
              reinterpret_cast<uint4 *>(rr + D)[i] = vv;
            }
            if (lane == 0 && tsa && app_types != nullptr && app_types[u] == 1)
              c.bitmask[(size_t)u * c.bm_words + (fp.L - 1) / 32] |= 1u << ((fp.L - 1) % 32);
            __syncwarp();
          }
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          // K: row rq (4 lanes per row, RQ channels each)
          float dot = 0.f;
          if (rq < n) {
            if (rows16) {
              const uint4 *kr = reinterpret_cast<const uint4 *>(B + (size_t)rq * 4 * D + rc4 * (RQ * 2));
              const float *qq = qo + h * D + rc4 * RQ;
#pragma unroll
              for (int i = 0; i < RQ / 8; ++i) {
                const uint4 v = kr[i];
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float a, b;
                  f_cvt2<DT>(wv[j], a, b);
                  dot = fmaf(qq[8 * i + 2 * j], a, dot);
                  dot = fmaf(qq[8 * i + 2 * j + 1], b, dot);
                }
              }
              dot *= alpha_o;
            } else {
              const uint8_t *se = B + (size_t)rq * c.side_entry;
              const int gq = (rc4 * RQ) / G;                 // RQ <= G: one group per lane
              const float sk = reinterpret_cast<const float *>(se)[gq];
              const float zk = (float)reinterpret_cast<const int32_t *>(se + 4 * NG)[gq];
              const uint32_t *cw = reinterpret_cast<const uint32_t *>(se + 16 * NG + rc4 * (RQ / 2));
              const float *qq = qh + h * D + rc4 * RQ;
              float A = 0.f, Bs = 0.f;
#pragma unroll
              for (int w = 0; w < RQ / 8; ++w) {
                const uint32_t word = cw[w];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  A = fmaf(qq[8 * w + i], (float)((word >> (4 * i)) & 15u), A);
                  Bs += qq[8 * w + i];
                }
              }
              dot = alpha_q * sk * (A - zk * Bs);
            }
          }
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          const float lg = rq < n ? dot : -INFINITY;
          float mx = lg;
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
          const float m_new = fmaxf(m_run[h], mx);
          if (m_new == -INFINITY) continue;
          const float sc = exp2f(m_run[h] - m_new);
          const float p = exp2f(lg - m_new);
          float ps = rc4 == 0 ? p : 0.f;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
          l_run[h] = l_run[h] * sc + ps;
          m_run[h] = m_new;
          Zu[h] *= sc; Zl[h] *= sc;
#pragma unroll
          for (int k = 0; k < 16; ++k) { o_rot[h][k] *= sc; o_org[h][k] *= sc; }
          // V: lane (kw, tg) accumulates its 16 channels over rows tg, tg+NTG, ...
#pragma unroll
          for (int r = 0; r < RC / NTG; ++r) {
            const int row = tg + NTG * r;
            const float pr = __shfl_sync(0xffffffffu, p, 4 * row);
            if (row >= n) continue;
            if (rows16) {
              const uint4 *vr = reinterpret_cast<const uint4 *>(B + (size_t)row * 4 * D + 2 * D + 32 * kw);
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const uint4 v = vr[i];
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  float a, b;
                  f_cvt2<DT>(wv[j], a, b);
                  o_org[h][8 * i + 2 * j] = fmaf(pr, a, o_org[h][8 * i + 2 * j]);
                  o_org[h][8 * i + 2 * j + 1] = fmaf(pr, b, o_org[h][8 * i + 2 * j + 1]);
                }
              }
            } else {
              const uint8_t *se = B + (size_t)row * c.side_entry;
              const float sv = reinterpret_cast<const float *>(se + 8 * NG)[gam];
              const float zv = (float)reinterpret_cast<const int32_t *>(se + 12 * NG)[gam];
              const float w = pr * sv;
              const uint2 cv = *reinterpret_cast<const uint2 *>(se + 16 * NG + D / 2 + 8 * kw);
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const uint32_t word = k < 8 ? cv.x : cv.y;
                o_rot[h][k] = fmaf(w, (float)((word >> (4 * (k & 7))) & 15u), o_rot[h][k]);
              }
              Zl[h] = fmaf(w, zv, Zl[h]);
            }
          }
        }
      }
      __syncwarp();
      // refill this stage with the producer's next sub-load
      if (p_ok) {
        if (lane == 0) issue(pc, st);
        ++pc.sub;
        p_ok = producer_next();
      }
      ++ci;
      ++cc.sub;
    }

    // ---- write this unit's partial (slot = warp's k-th unit)
    const size_t slot = (size_t)gw * fp.maxseg + (u - u_lo);
    float *rec = part + slot * REC;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      float zl = Zl[h];
#pragma unroll
      for (int off = KPR; off < 32; off <<= 1) zl += __shfl_xor_sync(0xffffffffu, zl, off);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a = o_org[h][k], b = o_rot[h][k];
#pragma unroll
        for (int off = KPR; off < 32; off <<= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, off);
          b += __shfl_xor_sync(0xffffffffu, b, off);
        }
        o_org[h][k] = a;
        o_rot[h][k] = b - Zu[h] - zl;
      }
      float *rh = rec + h * RECH;
      if (tg == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          reinterpret_cast<float4 *>(rh + 16 * kw)[k] =
              make_float4(o_rot[h][4 * k], o_rot[h][4 * k + 1], o_rot[h][4 * k + 2], o_rot[h][4 * k + 3]);
          reinterpret_cast<float4 *>(rh + D + 16 * kw)[k] =
              make_float4(o_org[h][4 * k], o_org[h][4 * k + 1], o_org[h][4 * k + 2], o_org[h][4 * k + 3]);
        }
      }
      if (lane == 0) { rh[2 * D] = m_run[h]; rh[2 * D + 1] = l_run[h]; }
    }
    // ---- ticket: the last warp of this unit merges the partials
    __threadfence();
    __syncwarp();
    long long w_lo, w_hi;
    {
      const long long i0 = (long long)u * Cu, i1 = i0 + Cu;
      w_lo = i0 * fp.W / fp.T;
      while (w_lo > 0 && w_lo * fp.T / fp.W > i0) --w_lo;
      while ((w_lo + 1) * fp.T / fp.W <= i0) ++w_lo;
      w_hi = w_lo;
      while (w_hi + 1 < fp.W && (w_hi + 1) * fp.T / fp.W < i1) ++w_hi;
    }
    const int expected = (int)(w_hi - w_lo + 1);
    int last = 0;
    if (lane == 0) last = atomicAdd(&c.ticket[u], 1u) == (unsigned)(expected - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence();
      constexpr int CPL = D / 32;
      const bool out_rot = flags & AKVQ_OUT_ROTATED;
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        float M = -INFINITY;
        for (long long w = w_lo; w <= w_hi; ++w) {
          const long long ul = (w * fp.T / fp.W) / Cu;
          const float *r = part + ((size_t)w * fp.maxseg + (u - ul)) * REC + h * RECH;
          M = fmaxf(M, __ldcg(r + 2 * D));
        }
        float rot[CPL], org[CPL], lsum = 0.f;
#pragma unroll
        for (int k = 0; k < CPL; ++k) { rot[k] = 0.f; org[k] = 0.f; }
        if (M != -INFINITY) {
          for (long long w = w_lo; w <= w_hi; ++w) {
            const long long ul = (w * fp.T / fp.W) / Cu;
            const float *r = part + ((size_t)w * fp.maxseg + (u - ul)) * REC + h * RECH;
            const float ms = __ldcg(r + 2 * D);
            if (ms == -INFINITY) continue;
            const float f = exp2f(ms - M);
            lsum += f * __ldcg(r + 2 * D + 1);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              rot[k] = fmaf(f, __ldcg(r + CPL * lane + k), rot[k]);
              org[k] = fmaf(f, __ldcg(r + D + CPL * lane + k), org[k]);
            }
          }
        }
        float x[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) x[k] = out_rot ? org[k] : rot[k];
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
            const float o = __shfl_xor_sync(0xffffffffu, x[k], lm);
            x[k] = upper ? o - x[k] : x[k] + o;
          }
        }
        const float inv = 1.f / lsum;
        float *dst = out + ((size_t)u * c.g + h) * D + CPL * lane;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const float tr = x[k] * c.inv_sqrt_d;
          dst[k] = (out_rot ? rot[k] + tr : tr + org[k]) * inv;
        }
      }
      if (lane == 0) c.ticket[u] = 0u;
    }
  }
}

template <int D, int G, int NH>
static size_t f_smem(size_t sb) { return (size_t)kFWarps * FSmem<D, G, NH>::warp_bytes(sb); }

size_t fused_stage_bytes(int d, int G, size_t page_bytes, size_t pg_vscale, size_t side_entry) {
  const size_t half_k = pg_vscale, half_v = page_bytes - pg_vscale;
  size_t sb = half_k > half_v ? half_k : half_v;
  const size_t rows = (size_t)FusedPlan::kRowChunk * 4 * d;
  if (rows > sb) sb = rows;
  const size_t side = (size_t)FusedPlan::kRowChunk * side_entry;
  if (side > sb) sb = side;
  return (sb + 127) / 128 * 128;
}

template <int D, int G, int DT, int NH>
static cudaError_t launch_f(const DevCache &c, const FusedPlan &fp, const void *q, const void *k,
                            const void *v, const uint8_t *types, float *part, float *out,
                            uint32_t flags, cudaStream_t st) {
  const size_t smem = f_smem<D, G, NH>(fp.stage_bytes);
  auto kern = k_decode_fused<D, G, DT, NH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int ctas = (int)((fp.W + kFWarps - 1) / kFWarps);
  kern<<<ctas, kFWarps * 32, smem, st>>>(c, fp, (const uint16_t *)q, (const uint16_t *)k,
                                          (const uint16_t *)v, types, part, out, flags);
  return cudaGetLastError();
}

template <int D, int G, int DT>
static cudaError_t launch_f_g(const DevCache &c, const FusedPlan &fp, const void *q, const void *k,
                              const void *v, const uint8_t *types, float *part, float *out,
                              uint32_t flags, cudaStream_t st) {
  if (c.g == 1) return launch_f<D, G, DT, 1>(c, fp, q, k, v, types, part, out, flags, st);
  if (c.g == 2) return launch_f<D, G, DT, 2>(c, fp, q, k, v, types, part, out, flags, st);
  return launch_f<D, G, DT, 4>(c, fp, q, k, v, types, part, out, flags, st);
}

int fused_supported(int d, int G, int g) {
  return (d == 128 || d == 64) && G >= 32 && G <= d && (g == 1 || g == 2 || g == 4);
}
int fused_warps_per_cta() { return kFWarps; }
size_t fused_smem_bytes(int d, int G, int g, size_t stage_bytes) {
#define AKVQ_FS(D_, G_)                                                            \
  if (d == D_ && G == G_)                                                          \
    return g == 1 ? f_smem<D_, G_, 1>(stage_bytes)                                 \
                  : (g == 2 ? f_smem<D_, G_, 2>(stage_bytes) : f_smem<D_, G_, 4>(stage_bytes));
  AKVQ_FS(64, 32)
  AKVQ_FS(64, 64)
  AKVQ_FS(128, 32)
  AKVQ_FS(128, 64)
  AKVQ_FS(128, 128)
#undef AKVQ_FS
  return 0;
}

cudaError_t launch_decode_fused(const DevCache &c, int dtype16, const FusedPlan &fp, const void *q,
                                const void *k, const void *v, const uint8_t *types, float *part,
                                float *out, uint32_t flags, cudaStream_t st) {
#define AKVQ_FCASE(D_, G_)                                                                          \
  if (c.d == D_ && c.G == G_)                                                                       \
    return dtype16 == AKVQ_BF16                                                                     \
               ? launch_f_g<D_, G_, AKVQ_BF16>(c, fp, q, k, v, types, part, out, flags, st)        \
               : launch_f_g<D_, G_, AKVQ_FP16>(c, fp, q, k, v, types, part, out, flags, st);
  AKVQ_FCASE(64, 32)
  AKVQ_FCASE(64, 64)
  AKVQ_FCASE(128, 32)
  AKVQ_FCASE(128, 64)
  AKVQ_FCASE(128, 128)
#undef AKVQ_FCASE
  return cudaErrorInvalidValue;
}

}  // namespace akvq
