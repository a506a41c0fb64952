// decode_gqa.cu -- single-pass grouped-query decode (GQA models
// of the paper's evaluation): one read of a kv head's packed cache
// serves all NH (4 or 8) query heads of the group.  Same tiers, arithmetic and
// work list as k_decode_layer (decode_layer.cu); what differs is the layout of
// the per-head work across the warp:
//
//  Page contractions.  The page's K codes (and V codes) are masked into A
//  fragments ONCE and multiplied against NT = NH/4 + 1 B tiles of the warp MMA
//  (m16n8k32, int8): tiles 0 .. NH/4-1 hold limbs 0 and 1 of four heads each
//  (column j: head 4t + j/2, limb j%2), the last tile holds limb 2 of all heads
//  (column j: head j/2 + 4 (j%2)).  MMA lane (grp, mt) thus owns heads 4t + mt:
//  limbs 0 + 256 x 1 in tile t, limb 2 in column 2 mt + t of the last tile --
//  all of a head's limbs land in the same lane.  Logits and value sums stay in this
//  "heads across lanes" layout: the softmax of head 4t + mt runs on the eight
//  lanes grp = 0..7 (16 tokens each), and o_rot accumulates in registers
//  (channels 4 (8 cb + grp) + k).  Page logits pass through shared memory once
//  (K half -> V half of the same page).
//  Rows (ring, PSA side rows, TSA 4-bit text rows) are rare in the long-context
//  GQA shapes; they are processed one row at a time in the ROTATED basis (16-bit
//  rows get an in-warp FWHT), with their own online-softmax state, and joined
//  with the page state when the segment is flushed.
// Partial records are [o' (rotated) D][m][l] per head; the merge applies H (Fig.
// 7, R4) and writes the output.  Fixed points: decode_common.cuh (24-bit, 3 int8
// limbs, per-unit ranges).
#include <math.h>

#include "decode_common.cuh"

namespace akvq {

#ifndef AKVQ_GQ_WARPS
#define AKVQ_GQ_WARPS 4
#endif
#ifndef AKVQ_GQ_REGS
#define AKVQ_GQ_REGS 255
#endif
#ifndef AKVQ_GQ_CTAS
#define AKVQ_GQ_CTAS 2
#endif
// warps per CTA and CTAs per SM: a sub-partition holds 16K registers, so 2 warps
// per sub-partition (8 per SM) at up to 255 registers each
constexpr int kGqWarps = AKVQ_GQ_WARPS;

template <int D> struct RecG {
  static constexpr int R = D + 4;    // [o D][m][l][pad 2]
};

// Per-warp shared memory: stages | orr [NH][32][4] f32 (row accumulators, one
// 16-byte slot per lane) | un: K limbs [NH][3][CQ] u32, then the page logits
// [NH][G + 8] f32, then the V limbs [NG][NH][3][TQ + 2] u32 | barriers.
template <int D, int G, int NH>
struct GqSmem {
  static constexpr int NG = D / G, CQ = D / 4, TQ = G / 4;
  static constexpr int LGP = G + 8;                // logit row pitch (bank spread)
  static constexpr int VLP = TQ + 2;               // V limb row pitch (bank spread, 8-byte rows)
  static constexpr size_t ORR = (size_t)NH * 32 * 16;
  static constexpr size_t UNK = (size_t)NH * 3 * CQ * 4, UNL = (size_t)NH * LGP * 4,
                          UNV = (size_t)NG * NH * 3 * VLP * 4;
  static constexpr size_t UN = UNK > UNL ? (UNK > UNV ? UNK : UNV) : (UNL > UNV ? UNL : UNV);
  static __host__ __device__ size_t orr_off(size_t sb) { return kLyStages * sb; }
  static __host__ __device__ size_t un_off(size_t sb) { return orr_off(sb) + ORR; }
  static __host__ __device__ size_t bar_off(size_t sb) { return un_off(sb) + (UN + 15) / 16 * 16; }
  static __host__ __device__ size_t warp_bytes(size_t sb) { return (bar_off(sb) + kLyStages * 8 + 127) / 128 * 128; }
};

// Per-unit merge of the GQA partials: out = (sum_seg f_seg o_seg) . H / l
// (rotated-basis records only).
template <int D, int NH>
__device__ __noinline__ void merge_gqa_unit(const DevCache &c, const LayerPlan &lp, const float *part, int u,
                                            float *out_u, int nh, uint32_t flags, int lane) {
  constexpr int CPL = D / 32;
  const int w0 = ly_warp_of(lp, u, 0), w1 = ly_warp_of(lp, u, lp.per_u - 1);
  const int nseg = w1 - w0 + 1;
  const bool out_rot = flags & AKVQ_OUT_ROTATED;
  auto seg_rec = [&](int j, int h) -> const float * {
    const int w = w0 + j;
    const int slot = w * lp.maxseg + (u - ly_first_unit(lp, w));
    return part + ((size_t)slot * NH + h) * RecG<D>::R;
  };
  for (int h = 0; h < nh; ++h) {
    float M = -INFINITY;
    for (int b0 = 0; b0 < nseg; b0 += 32) {
      const float ms = b0 + lane < nseg ? __ldcg(seg_rec(b0 + lane, h) + D) : -INFINITY;
      M = fmaxf(M, warp_max(ms));
    }
    float acc[CPL], lsum = 0.f;
#pragma unroll
    for (int k = 0; k < CPL; ++k) acc[k] = 0.f;
    if (M != -INFINITY) {
      for (int b0 = 0; b0 < nseg; b0 += 32) {
        float f = 0.f, ls = 0.f;
        const float *rh = nullptr;
        if (b0 + lane < nseg) {
          rh = seg_rec(b0 + lane, h);
          const float ms = __ldcg(rh + D);
          ls = __ldcg(rh + D + 1);
          f = ms == -INFINITY ? 0.f : exp2f(ms - M);
        }
        lsum += warp_sum(f * ls);
        const int nb = min(32, nseg - b0);
        for (int j = 0; j < nb; ++j) {
          const float fj = __shfl_sync(0xffffffffu, f, j);
          const unsigned long long pj = __shfl_sync(0xffffffffu, (unsigned long long)(uintptr_t)rh, j);
          if (fj == 0.f) continue;                   // warp-uniform
          const float *r = reinterpret_cast<const float *>((uintptr_t)pj);
#pragma unroll
          for (int k = 0; k < CPL; ++k) acc[k] = fmaf(fj, __ldcg(r + CPL * lane + k), acc[k]);
        }
      }
    }
    float x[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) x[k] = acc[k];
    if (!out_rot) {                                 // o = o' . H (FWHT x 1/sqrt d)
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
#pragma unroll
      for (int k = 0; k < CPL; ++k) x[k] *= c.inv_sqrt_d;
    }
    const float inv = 1.f / lsum;
    float *dst = out_u + (size_t)h * D + CPL * lane;
#pragma unroll
    for (int k = 0; k < CPL; ++k) dst[k] = x[k] * inv;
  }
}

// Sum of NH int64 values across the warp, reduce-scatter style: on return lane
// L holds the total of slot rs_enc^-1(lane bits 4..2), i.e. slot m is held by
// lane rs_enc<NH, 32>(m) (and its neighbours in bits 0, 1).
template <int NH>
__device__ __forceinline__ long long rs_reduce_i64(long long (&v)[NH], int lane) {
  constexpr int L2 = NH == 8 ? 3 : 2;
#pragma unroll
  for (int step = 0; step < L2; ++step) {
    const int n = NH >> step, off = 16 >> step;
    const bool up = lane & off;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const long long send = up ? v[i] : v[i + n / 2];
      const long long keep = up ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  long long t = v[0];
#pragma unroll
  for (int off = 16 >> L2; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  return t;
}

template <int D, int G, int DT, int NH, bool TSA>
__global__ void __maxnreg__(AKVQ_GQ_REGS)
    k_decode_gqa(const __grid_constant__ DevCache c, const __grid_constant__ LayerPlan lp,
                 const uint16_t *__restrict__ q, const uint16_t *__restrict__ app_k,
                 const uint16_t *__restrict__ app_v, const uint8_t *__restrict__ app_types,
                 float *__restrict__ part, float *__restrict__ out, uint32_t flags) {
  using S = GqSmem<D, G, NH>;
  constexpr int NG = D / G;
  constexpr int CQ = D / 4, TQ = G / 4;
  constexpr int NT01 = NH / 4;              // limb-0/1 tiles (4 heads each)
  constexpr int NT = NT01 + 1;              // + the limb-2 tile (8 heads)
  constexpr int KC = D / 32, TC = G / 32;   // K-phase channel chunks, V-phase token chunks
  constexpr int NB = TQ / 8;                // token blocks (16 tokens) of a page per lane group
  constexpr int NCB = D / 32;               // V-phase channel blocks
  constexpr int VTS = 32 / CQ;              // lanes per channel quad (rows)
  static_assert(NH == 4 || NH == 8, "head group of 4 or 8");
  static_assert(TQ <= 32 && CQ <= 32 && G >= 32, "page shape");
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ unsigned cta_done;                 // warps of this CTA done (ly_exit)
  if (lp.dev_L) {                               // (uniform: the barrier is legal)
    if (threadIdx.x == 0) cta_done = 0u;
    __syncthreads();
  }
  const size_t SB = ly_stage_bytes(c);
  uint8_t *wsm = smem + (size_t)warp * S::warp_bytes(SB);
  float *orr = reinterpret_cast<float *>(wsm + S::orr_off(SB));             // [NH][32][4]
  uint32_t *un_u = reinterpret_cast<uint32_t *>(wsm + S::un_off(SB));
  float *un_f = reinterpret_cast<float *>(wsm + S::un_off(SB));
  uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + S::bar_off(SB));

  if (!lp.prologue) {
    pdl_wait();
    pdl_launch_dependents();
  }
  const int gw = blockIdx.x * kGqWarps + warp;
  if (gw >= lp.W) { ly_exit(c, lp, lane, &cta_done); return; }
  const int ib = ly_first_item_p(&lp, gw);       // (out of line: code size)
  const int ie = gw + 1 < lp.W ? ly_first_item_p(&lp, gw + 1) : lp.T;
  if (ib >= ie) { ly_exit(c, lp, lane, &cta_done); return; }
  // this launch's token count, the new token included when it appends (DEVICE_L
  // launches have no prologue: the griddepcontrol.wait above has been passed)
  const int Lc = lp.dev_L ? c.dstate->L + (lp.appends ? 1 : 0) : lp.L;
  constexpr bool tsa = TSA;
  const int HG = lp.hg;
  const float alpha_k = kLog2e / (float)D;      // q~_u . K^_n / d in log2 units (pages, 4-bit rows)
  const float rsd = c.inv_sqrt_d;
  const uint32_t kbytes = c.pg_vscale, vbytes = c.page_bytes - c.pg_vscale;

  // ---- producer (as k_decode_layer): warp-uniform item walk, lane 0 issues TMA
  if (lane == 0) {
    for (int s = 0; s < kLyStages; ++s) mbar_init(&bar[s]);
    mbar_fence_init();
  }
  __syncwarp();
  int pu = ib / lp.per_u, pj = ib - (ib / lp.per_u) * lp.per_u, left = ie - ib, part_i = 0;
  int pphys = pu / HG, phg = pu - (pu / HG) * HG;
  const uint8_t *ubase = c.pages + (size_t)pphys * c.n_pages * c.page_bytes;
  int eu = -1;                                  // last (virtual) unit a sub-load was issued for
  const uint8_t *vsrc = nullptr;
  uint2 vdesc = make_uint2(0u, 0u);
  auto produce = [&](int st) -> uint2 {
    uint8_t *dst = wsm + (size_t)st * SB;
    if (vsrc != nullptr) {
      if (lane == 0) {
        mbar_expect_tx(&bar[st], vbytes);
        bulk_g2s(dst, vsrc, vbytes, &bar[st]);
      }
      vsrc = nullptr;
      return vdesc;
    }
    LySub sb;
    sb.kind = -1;
    while (left > 0) {
      const uint32_t e = lp.tab[pj];
      const int kind = (int)(e & 3u);
      const int a = (int)(e >> 8), n = (int)((e >> 2) & 63u);
      bool ok = true, next = true;
      sb.u = pu;
      sb.pu = pphys;
      sb.ring = 0;
      sb.a = a;
      if (kind == 0) {
        sb.kind = 0; sb.n = 0;
      } else if (kind == 2) {
        sb.kind = 2; sb.ring = 1; sb.n = n;
        if (lp.dev_L) {                           // chunks of the period past L: skip
          sb.n = min(n, Lc - lp.n_q - a);
          ok = sb.n > 0;
        }
      } else {
        const int cnt = __ldg(c.side_cnt + pphys);
        auto fdiv = [&](int x) {
          int qd = __float2int_rz((float)x * lp.sc_inv);
          qd += (qd + 1) * lp.Sc <= x;
          qd -= qd * lp.Sc > x;
          return qd;
        };
        const int lo = fdiv(a * cnt), hi = fdiv((a + 1) * cnt);
        const int per = tsa ? kRows4 : kRows;
        sb.kind = tsa ? 3 : 2;
        sb.a = lo + part_i * per;
        sb.n = min(per, hi - sb.a);
        ok = sb.n > 0;
        next = !ok;
        part_i = ok ? part_i + 1 : 0;
      }
      const uint8_t *ub = ubase;                  // (pages: the unit before advancing)
      if (next) {
        if (++pj == lp.per_u) {
          pj = 0;
          ++pu;
          if (++phg == HG) { phg = 0; ++pphys; ubase += (size_t)c.n_pages * c.page_bytes; }
        }
        --left;
      }
      const bool unit_done = next && (pj == 0 || left == 0);   // the item closed its unit's run
      if (ok) {
        eu = sb.u;
        if (sb.kind == 0) {
          const uint8_t *pg = c.btab ? c.pages + (size_t)__ldg(c.btab + (size_t)sb.pu * c.n_pages + sb.a) * c.page_bytes
                                     : ub + (size_t)sb.a * c.page_bytes;
          if (lane == 0) {
            mbar_expect_tx(&bar[st], kbytes);
            bulk_g2s(dst, pg, kbytes, &bar[st]);
          }
          vsrc = pg + kbytes;
          LySub vb = sb;
          vb.kind = 1;
          vdesc = pack_sub(vb);
        } else if (sb.ring) {
          int s0 = lp.nq_mod + sb.a;
          if (s0 >= c.slots) s0 -= c.slots;
          const int n1 = min(sb.n, c.slots - s0);
          const uint32_t rowb = 4 * D;
          if (lane == 0) {
            mbar_expect_tx(&bar[st], (uint32_t)sb.n * rowb);
            bulk_g2s(dst, ring_row(c, sb.pu, s0), (uint32_t)n1 * rowb, &bar[st]);
            if (n1 < sb.n)
              bulk_g2s(dst + (size_t)n1 * rowb, ring_row(c, sb.pu, 0), (uint32_t)(sb.n - n1) * rowb, &bar[st]);
          }
        } else {
          const uint32_t eb = c.side_entry;
          if (lane == 0) {
            mbar_expect_tx(&bar[st], (uint32_t)sb.n * eb);
            bulk_g2s(dst, side_ptr(c, sb.pu, sb.a), (uint32_t)sb.n * eb, &bar[st]);
          }
        }
        break;
      }
      if (unit_done && eu != sb.u) {
        // every item of this unit in the range was empty (empty side splits, ring
        // chunks past L): an empty sub-load still reaches the consumer, which then
        // writes the (empty) partial the unit's merge ticket counts on
        eu = sb.u;
        sb.kind = 4;
        if (lane == 0) mbar_expect_tx(&bar[st], 0u);
        break;
      }
      sb.kind = -1;
    }
    return pack_sub(sb);
  };
  // stage descriptors, primed by the loop's single producer call site (code size)
  uint2 dsc0 = make_uint2(0u, 0u), dsc1 = make_uint2(0u, 0u);

  // lane roles
  const int mg = lane >> 2, mt = lane & 3;            // MMA fragment group / thread in group
  const int vcq = lane % CQ, vts = lane / CQ;         // rows: channel quad
  // this lane's B column in tile t: head 4t + mg/2, limb mg%2 (t < NT01); head mg, limb 2

  // per-segment state
  // qi = q~ kQMax / max|q~| per head (channel quad vcq; |qi| <= kQMax); a page's
  // Q_hc = rn(qi_hc s^K_c / umax.K) (|Q| <= kQMax); logit_t = dAh sum_c Q_hc
  // (code_tc - z_c) with dAh = alpha_k max|q~_h| umax.K / kQMax = rq_h umax.K
  float qi[NH][4];
  float rq[NH];                                       // alpha_k max|q~_h| / kQMax (rows: q~ = qi rq / alpha_k)
  float dAh[NH];                                      // page logit scale per head
  float dl[NT01];                                     // dAh of the lane's heads 4t + mt
  float o_rot[NT01][NCB][4];                          // pages, heads 4t + mt, channels 4 (8 cb + mg) + k
  float m_p[NT01], l_p[NT01], zl[NT01][NG];           // pages softmax (l, zl: lane partials)
  float m_r[NH], l_r[NH];                             // rows softmax (warp-uniform)
  float winv = 0.f, dwu = 0.f, skinv = 0.f;
  int cur_u = -1, cur_pu = 0, cur_hg = 0;
  const int u_first = ib / lp.per_u;

  auto flush = [&](int u) {
    const size_t slot = (size_t)gw * lp.maxseg + (u - u_first);
    const int hg = u % HG, nh = min(NH, c.g - hg * NH);
    __syncwarp();
#pragma unroll
    for (int t = 0; t < NT01; ++t) {
      const int h = 4 * t + mt;
      float lp_t = l_p[t];
      float zg[NG];
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) zg[gi] = zl[t][gi];
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        lp_t += __shfl_xor_sync(0xffffffffu, lp_t, off);
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) zg[gi] += __shfl_xor_sync(0xffffffffu, zg[gi], off);
      }
      // rows state of head h (warp-uniform arrays, static index via select)
      float mr = m_r[0], lr = l_r[0];
#pragma unroll
      for (int hh = 1; hh < NH; ++hh)
        if (h == hh) { mr = m_r[hh]; lr = l_r[hh]; }
      const float m = fmaxf(m_p[t], mr);
      const float fp = m == -INFINITY ? 0.f : ex2(m_p[t] - m);
      const float fr = m == -INFINITY ? 0.f : ex2(mr - m);
      float *rec = part + (slot * NH + h) * RecG<D>::R;
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) {
        const int cq = 8 * cb + mg;
        const float zsub = zg[(4 * cq) / G];
        const float4 rr = reinterpret_cast<const float4 *>(orr)[h * 32 + cq];
        float4 o;
        o.x = fmaf(o_rot[t][cb][0] - zsub, fp, rr.x * fr);
        o.y = fmaf(o_rot[t][cb][1] - zsub, fp, rr.y * fr);
        o.z = fmaf(o_rot[t][cb][2] - zsub, fp, rr.z * fr);
        o.w = fmaf(o_rot[t][cb][3] - zsub, fp, rr.w * fr);
        if (h < nh) reinterpret_cast<float4 *>(rec)[cq] = o;
      }
      if (mg == 0 && h < nh) { rec[D] = m; rec[D + 1] = fmaf(lp_t, fp, lr * fr); }
    }
    const int2 wsp = ly_warp_span_p(&lp, u);      // (out of line: code size)
    const int w_lo = wsp.x, w_hi = wsp.y;
    if (take_ticket(c, u, w_hi - w_lo + 1, lane)) {
      merge_gqa_unit<D, NH>(c, lp, part, u, out + ((size_t)(u / HG) * c.g + hg * NH) * D, nh, flags, lane);
      if (lane == 0) c.ticket[u] = 0u;
    }
  };

  // one row (rotated basis, normalized: k4 / v4 are this lane's channel quad)
  // joins the rows softmax of every head; lanes >= CQ (d = 64) duplicate lanes
  // < CQ and keep their own (unused) accumulator slots
  auto row_update = [&](const float (&k4)[4], const float (&v4)[4], bool valid) {
    float dot[NH];
#pragma unroll
    for (int h = 0; h < NH; ++h)
      dot[h] = rq[h] * fmaf(qi[h][0], k4[0], fmaf(qi[h][1], k4[1], fmaf(qi[h][2], k4[2], qi[h][3] * k4[3])));
    int mine;
    float t = rs_reduce<NH, CQ>(dot, vcq, mine);
    t = valid ? t : -INFINITY;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const float lg = __shfl_sync(0xffffffffu, t, (vts * CQ) | rs_enc<NH, CQ>(h));
      const float m_new = fmaxf(m_r[h], lg);
      if (m_new == -INFINITY) continue;               // warp-uniform
      const float sc = ex2(m_r[h] - m_new), p = ex2(lg - m_new);
      m_r[h] = m_new;
      l_r[h] = fmaf(l_r[h], sc, p);
      float4 *a = reinterpret_cast<float4 *>(orr) + h * 32 + lane;
      float4 r = *a;
      r.x = fmaf(p, v4[0], r.x * sc); r.y = fmaf(p, v4[1], r.y * sc);
      r.z = fmaf(p, v4[2], r.z * sc); r.w = fmaf(p, v4[3], r.w * sc);
      *a = r;
    }
  };

  int st = 0;
  uint32_t par = 0;
  int rf = 0, nrf = kLyStages;                      // stages to (re)fill: both at first
  bool first = true;
  for (;;) {
#pragma unroll 1
    for (; nrf > 0; --nrf, rf ^= 1) {               // the only producer call site
      const uint2 d = produce(rf);
      if (rf) dsc1 = d; else dsc0 = d;
    }
    if (first) {
      first = false;
      if (lp.prologue) {
        pdl_wait();
        pdl_launch_dependents();
      }
      // host-L mode: keep the device copy current (a later DEVICE_L launch reads it)
      if (!lp.dev_L && lp.appends && blockIdx.x == 0 && threadIdx.x == 0) c.dstate->L = lp.L;
    }
    const LySub s = unpack_sub(st ? dsc1 : dsc0);
    uint8_t *B = wsm + (size_t)st * SB;
    if (s.kind < 0 || s.u != cur_u) {               // segment boundary (one flush site)
      if (cur_u >= 0) flush(cur_u);
      if (s.kind < 0) break;
      cur_u = s.u;
      cur_pu = s.u / HG;
      cur_hg = s.u - cur_pu * HG;
      const float2 um = c.umax[cur_pu];
      const float skmax = um.x;
      skinv = skmax > 0.f ? __fdividef(1.0f, skmax) : 0.f;
      winv = um.y > 0.f ? __fdividef((float)kQMax, um.y) : 0.f;
      dwu = um.y * (1.0f / (float)kQMax);
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        // q~ = q . H_s for this lane's channel quad: in-lane butterflies, then shuffles
        float x[4];
        const uint2 v = *reinterpret_cast<const uint2 *>(
            q + ((size_t)cur_pu * c.g + min(cur_hg * NH + h, c.g - 1)) * D + 4 * vcq);
        cvt2<DT>(v.x, x[0], x[1]);
        cvt2<DT>(v.y, x[2], x[3]);
        { const float a = x[0], b = x[1]; x[0] = a + b; x[1] = a - b; }
        { const float a = x[2], b = x[3]; x[2] = a + b; x[3] = a - b; }
        { const float a = x[0], b = x[2]; x[0] = a + b; x[2] = a - b; }
        { const float a = x[1], b = x[3]; x[1] = a + b; x[3] = a - b; }
#pragma unroll 1
        for (int lm = 1; lm < CQ; lm <<= 1) {     // (not unrolled: once per unit, code size)
          const bool upper = lane & lm;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float o2 = __shfl_xor_sync(0xffffffffu, x[k], lm);
            x[k] = upper ? o2 - x[k] : x[k] + o2;
          }
        }
        const float qmax = warp_max(fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fmaxf(fabsf(x[2]), fabsf(x[3]))));
        const float iq = qmax > 0.f ? __fdividef((float)kQMax, qmax) : 0.f;
        rq[h] = alpha_k * qmax * (1.0f / (float)kQMax);
        dAh[h] = rq[h] * skmax;
#pragma unroll
        for (int k = 0; k < 4; ++k) qi[h][k] = x[k] * iq;
        m_r[h] = -INFINITY;
        l_r[h] = 0.f;
        reinterpret_cast<float4 *>(orr)[h * 32 + lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int t = 0; t < NT01; ++t) {
        dl[t] = dAh[4 * t];
#pragma unroll
        for (int j = 1; j < 4; ++j) if (mt == j) dl[t] = dAh[4 * t + j];
        m_p[t] = -INFINITY;
        l_p[t] = 0.f;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) zl[t][gi] = 0.f;
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb)
#pragma unroll
          for (int k = 0; k < 4; ++k) o_rot[t][cb][k] = 0.f;
      }
      __syncwarp();
    }

    if (s.kind == 0) {
      // ================= page K half: logits of the page's G tokens, all heads
      uint32_t sw[NB];                                // salient bits of the lane's token quads
#pragma unroll
      for (int blk = 0; blk < NB; ++blk) {
        const int tq = 8 * blk + mg;
        sw[blk] = (__ldg(c.bitmask + (size_t)cur_pu * c.bm_words + (size_t)s.a * (G / 32) + (tq >> 3)) >>
                   (4 * (tq & 7))) & 15u;
      }
      mbar_wait(&bar[st], par);
      const float4 *ks4 = reinterpret_cast<const float4 *>(B + c.pg_kscale);
      const int4 *kz4 = reinterpret_cast<const int4 *>(B + c.pg_kzero);
      // Q_hc = rn(q~_hc s^K_c inv_h), inv_h = kQMax / (max|q~_h| umax.K); bias
      // B_h = sum_c Q_hc z_c (int64); limbs -> un [h][limb][cq]
      long long bz[NH];
      float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
      int4 zq = make_int4(0, 0, 0, 0);
      if (lane < CQ) { sv = ks4[lane]; zq = kz4[lane]; }
      sv.x *= skinv; sv.y *= skinv; sv.z *= skinv; sv.w *= skinv;    // |s / umax.K| <= 1
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        uint32_t x[4];
        x[0] = (uint32_t)__float2int_rn(qi[h][0] * sv.x) + kQOff;
        x[1] = (uint32_t)__float2int_rn(qi[h][1] * sv.y) + kQOff;
        x[2] = (uint32_t)__float2int_rn(qi[h][2] * sv.z) + kQOff;
        x[3] = (uint32_t)__float2int_rn(qi[h][3] * sv.w) + kQOff;
        bz[h] = (long long)(int)(x[0] - kQOff) * zq.x + (long long)(int)(x[1] - kQOff) * zq.y +
                (long long)(int)(x[2] - kQOff) * zq.z + (long long)(int)(x[3] - kQOff) * zq.w;
        if (lane < CQ) {
          un_u[(h * 3) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0040), prmt(x[2], x[3], 0x0040), 0x5410) ^ 0x80808080u;
          un_u[(h * 3 + 1) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0051), prmt(x[2], x[3], 0x0051), 0x5410) ^ 0x80808080u;
          un_u[(h * 3 + 2) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0062), prmt(x[2], x[3], 0x0062), 0x5410) ^ 0x80808080u;
        }
      }
      const long long bsum = rs_reduce_i64<NH>(bz, lane);
      // the bias limbs this lane's accumulators start from: heads 4t + mt (limbs 0,
      // 1) and 2 mt, 2 mt + 1 (limb 2)
      int b01[NT01][2], b2[2];
      bool slow = lp.exact_logits != 0;
#pragma unroll
      for (int t = 0; t < NT01; ++t) {
        const long long Bh = __shfl_sync(0xffffffffu, bsum, rs_enc<NH, 32>(4 * t + mt));
        b01[t][0] = (int)(Bh & 255);
        b01[t][1] = (int)((Bh >> 8) & 255);
        const long long hi = Bh >> 16;
        slow |= hi >= (1 << 24) || hi <= -(1 << 24);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {      // limb-2 tile columns 2 mt, 2 mt + 1: heads mt, mt + 4
        const long long Bh = __shfl_sync(0xffffffffu, bsum, rs_enc<NH, 32>(min(mt + 4 * j, NH - 1)));
        const long long hi = Bh >> 16;
        b2[j] = (int)hi;
        slow |= hi >= (1 << 24) || hi <= -(1 << 24);
      }
      slow = __any_sync(0xffffffffu, slow);
      __syncwarp();
      if (slow) {
        // plain fp32 logits: alpha_k sum_c q~_hc s_c (code_tc - z_c), lane = heads
        // 4t + mt, tokens of its quads (rare: huge zero-point offsets, test hook)
        const float *ksf = reinterpret_cast<const float *>(B + c.pg_kscale);
        const int32_t *kzf = reinterpret_cast<const int32_t *>(B + c.pg_kzero);
        const uint8_t *kcb = B + c.pg_kcodes;
        // q~ of all channels: gather through the orr-free un area (K limbs unused here)
        float *qf = un_f;                             // [NH][D]
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (lane < CQ)
            reinterpret_cast<float4 *>(qf + h * D)[lane] =
                make_float4(qi[h][0] * rq[h], qi[h][1] * rq[h], qi[h][2] * rq[h], qi[h][3] * rq[h]);
        __syncwarp();
        float lgv[NT01][NB][4];
#pragma unroll
        for (int t = 0; t < NT01; ++t)
#pragma unroll
          for (int blk = 0; blk < NB; ++blk) {
            const int h = 4 * t + mt, tq = 8 * blk + mg;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              float acc = 0.f;
#pragma unroll 1
              for (int ch = 0; ch < D; ++ch)              // (rare fp32 path: not unrolled)
                acc = fmaf(qf[h * D + ch] * ksf[ch], (float)kcode_at(kcb, 4 * tq + k, ch, G) - (float)kzf[ch], acc);
              lgv[t][blk][k] = ((sw[blk] >> k) & 1u) ? -INFINITY : acc;   // q~ alpha_k . K^
            }
          }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < NT01; ++t)
#pragma unroll
          for (int blk = 0; blk < NB; ++blk) {
            const float4 r = make_float4(lgv[t][blk][0], lgv[t][blk][1], lgv[t][blk][2], lgv[t][blk][3]);
            reinterpret_cast<float4 *>(un_f + (4 * t + mt) * S::LGP)[8 * blk + mg] = r;
          }
      } else {
        // B fragments: tile t < NT01 column mg -> head 4t + mg/2, limb mg%2;
        // limb-2 tile column mg -> head mg
        uint32_t bq[NT][KC][2];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int row = t < NT01 ? (4 * t + (mg >> 1)) * 3 + (mg & 1) : min((mg >> 1) + 4 * (mg & 1), NH - 1) * 3 + 2;
#pragma unroll
          for (int cc = 0; cc < KC; ++cc) {
            const uint2 b = *reinterpret_cast<const uint2 *>(un_u + row * CQ + 8 * cc + 2 * mt);
            bq[t][cc][0] = b.x;
            bq[t][cc][1] = b.y;
          }
        }
        __syncwarp();                                 // un now free for the logits
        const uint32_t *kcw = reinterpret_cast<const uint32_t *>(B + c.pg_kcodes);
        const float fk[4] = {1.f, 0.25f, 0.0625f, 0.015625f};
#pragma unroll
        for (int blk = 0; blk < NB; ++blk) {
          const int tq = 8 * blk + mg;
          int acc[NT][8];
#pragma unroll
          for (int t = 0; t < NT01; ++t) {
            const int ba = b01[t][0], bb = b01[t][1];
            acc[t][0] = -ba; acc[t][1] = -bb; acc[t][2] = -4 * ba; acc[t][3] = -4 * bb;
            acc[t][4] = -16 * ba; acc[t][5] = -16 * bb; acc[t][6] = -64 * ba; acc[t][7] = -64 * bb;
          }
          acc[NT01][0] = -b2[0]; acc[NT01][1] = -b2[1]; acc[NT01][2] = -4 * b2[0]; acc[NT01][3] = -4 * b2[1];
          acc[NT01][4] = -16 * b2[0]; acc[NT01][5] = -16 * b2[1]; acc[NT01][6] = -64 * b2[0]; acc[NT01][7] = -64 * b2[1];
#pragma unroll
          for (int cc = 0; cc < KC; ++cc) {
            const uint2 w = *reinterpret_cast<const uint2 *>(kcw + kword_idx(8 * cc + 2 * mt, tq, TQ));
            const uint32_t a0 = fmask(w.x, 0), a1 = fmask(w.x, 1), a2 = fmask(w.y, 0), a3 = fmask(w.y, 1);
            const uint32_t e0 = fmask(w.x, 2), e1 = fmask(w.x, 3), e2 = fmask(w.y, 2), e3 = fmask(w.y, 3);
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              int *c01 = acc[t], *c23 = acc[t] + 4;
              mma_u8s8(*reinterpret_cast<int(*)[4]>(c01), a0, a1, a2, a3, bq[t][cc][0], bq[t][cc][1]);
              mma_u8s8(*reinterpret_cast<int(*)[4]>(c23), e0, e1, e2, e3, bq[t][cc][0], bq[t][cc][1]);
            }
          }
          // head 4t + mt: limbs 0, 1 in tile t, limb 2 in column 2 mt + t of the last
          // tile; token rows k = 4tq + k: accumulators (0, 1) k 0, (2, 3) k 1,
          // (4, 5) k 2, (6, 7) k 3 (row grp / grp + 8 of c01 / c23)
#pragma unroll
          for (int t = 0; t < NT01; ++t) {
            float r[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float v01 = (float)(acc[t][2 * k] + 256 * acc[t][2 * k + 1]);   // |.| < 2^31
              const float tot = fmaf(65536.f, (float)acc[NT01][2 * k + t], v01);
              r[k] = ((sw[blk] >> k) & 1u) ? -INFINITY : tot * (fk[k] * dl[t]);
            }
            reinterpret_cast<float4 *>(un_f + (4 * t + mt) * S::LGP)[tq] = make_float4(r[0], r[1], r[2], r[3]);
          }
        }
      }
    } else if (s.kind == 1) {
      // ================= page V half: softmax of every head, value accumulation
      mbar_wait(&bar[st], par);
      const float *vs = reinterpret_cast<const float *>(B);
      const int32_t *vz = reinterpret_cast<const int32_t *>(B + (c.pg_vzero - c.pg_vscale));
      const uint32_t *vcw = reinterpret_cast<const uint32_t *>(B + (c.pg_vcodes - c.pg_vscale));
      __syncwarp();
      // logits of heads 4t + mt, tokens 4 (8 blk + mg) + k
      float lg[NT01][NB][4];
#pragma unroll
      for (int t = 0; t < NT01; ++t) {
#pragma unroll
        for (int blk = 0; blk < NB; ++blk) {
          const float4 r = reinterpret_cast<const float4 *>(un_f + (4 * t + mt) * S::LGP)[8 * blk + mg];
          lg[t][blk][0] = r.x; lg[t][blk][1] = r.y; lg[t][blk][2] = r.z; lg[t][blk][3] = r.w;
        }
      }
      __syncwarp();                                   // un is rewritten with W limbs below
      // V scales / zero points of the lane's tokens
      float vsv[NB][NG][4], vzv[NB][NG][4];
#pragma unroll
      for (int blk = 0; blk < NB; ++blk) {
        const int tq = 8 * blk + mg;
        if constexpr (NG == 1) {
          const float4 a = reinterpret_cast<const float4 *>(vs)[tq];
          const int4 b = reinterpret_cast<const int4 *>(vz)[tq];
          vsv[blk][0][0] = a.x; vsv[blk][0][1] = a.y; vsv[blk][0][2] = a.z; vsv[blk][0][3] = a.w;
          vzv[blk][0][0] = (float)b.x; vzv[blk][0][1] = (float)b.y; vzv[blk][0][2] = (float)b.z; vzv[blk][0][3] = (float)b.w;
        } else {
#pragma unroll
          for (int gi = 0; gi < NG; ++gi)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              vsv[blk][gi][k] = vs[(4 * tq + k) * NG + gi];
              vzv[blk][gi][k] = (float)vz[(4 * tq + k) * NG + gi];
            }
        }
      }
#pragma unroll
      for (int blk = 0; blk < NB; ++blk)
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
#pragma unroll
          for (int k = 0; k < 4; ++k) vsv[blk][gi][k] *= winv;
      bool live[NT01];
#pragma unroll
      for (int t = 0; t < NT01; ++t) {
        const int h = 4 * t + mt;
        float mloc = -INFINITY;
#pragma unroll
        for (int blk = 0; blk < NB; ++blk)
          mloc = fmaxf(mloc, fmaxf(fmaxf(lg[t][blk][0], lg[t][blk][1]), fmaxf(lg[t][blk][2], lg[t][blk][3])));
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, off));
        const float m_new = fmaxf(m_p[t], mloc);
        live[t] = m_new != -INFINITY;                 // uniform over the head's 8 lanes
        const float sc = live[t] ? ex2(m_p[t] - m_new) : 1.f;
        m_p[t] = m_new;
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb)
#pragma unroll
          for (int k = 0; k < 4; ++k) o_rot[t][cb][k] *= sc;
        float psum = 0.f;
        float zs[NG];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) zs[gi] = 0.f;
#pragma unroll
        for (int blk = 0; blk < NB; ++blk) {
          const int tq = 8 * blk + mg;
          float p[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) { p[k] = live[t] ? ex2(lg[t][blk][k] - m_new) : 0.f; psum += p[k]; }
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) {
            // W_t = rn(p_t s^V_t winv), signed 24-bit; zero-point term with the same W
            uint32_t W[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int wi = __float2int_rn(p[k] * vsv[blk][gi][k]);     // vsv = s^V winv
              W[k] = (uint32_t)wi + kQOff;
              zs[gi] = fmaf((float)wi, vzv[blk][gi][k], zs[gi]);
            }
            uint32_t *wl = un_u + ((gi * NH + h) * 3) * S::VLP + tq;
            wl[0] = prmt(prmt(W[0], W[1], 0x0040), prmt(W[2], W[3], 0x0040), 0x5410) ^ 0x80808080u;
            wl[S::VLP] = prmt(prmt(W[0], W[1], 0x0051), prmt(W[2], W[3], 0x0051), 0x5410) ^ 0x80808080u;
            wl[2 * S::VLP] = prmt(prmt(W[0], W[1], 0x0062), prmt(W[2], W[3], 0x0062), 0x5410) ^ 0x80808080u;
          }
        }
        l_p[t] = fmaf(l_p[t], sc, psum);
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) zl[t][gi] = fmaf(zl[t][gi], sc, dwu * zs[gi]);
      }
      __syncwarp();
      // value sums sum_t W_ht code_tc by warp MMA: rows = channels (row grp:
      // channel 4 cq + k0, grp + 8: 4 cq + k1, cq = 8 cb + grp), K = 32 tokens per
      // chunk, columns as in the K phase (limbs 0/1 of 4 heads per tile, limb 2)
      // B fragments (W limbs): the same for every channel block when NG == 1
      uint32_t bv[NG == 1 ? NT : 1][NG == 1 ? TC : 1][2];
      if constexpr (NG == 1) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int row = t < NT01 ? (4 * t + (mg >> 1)) * 3 + (mg & 1) : min((mg >> 1) + 4 * (mg & 1), NH - 1) * 3 + 2;
#pragma unroll
          for (int cc = 0; cc < TC; ++cc) {
            const uint2 b = *reinterpret_cast<const uint2 *>(un_u + row * S::VLP + 8 * cc + 2 * mt);
            bv[t][cc][0] = b.x;
            bv[t][cc][1] = b.y;
          }
        }
      }
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) {
        const int cq = 8 * cb + mg, gi = (32 * cb) / G;
        int acc[NT][8];
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[t][i] = 0;
#pragma unroll
        for (int cc = 0; cc < TC; ++cc) {
          const uint2 w = *reinterpret_cast<const uint2 *>(vcw + vword_idx(cq, 8 * cc + 2 * mt, CQ));
          const uint32_t a0 = fmask(w.x, 0), a1 = fmask(w.x, 1), a2 = fmask(w.y, 0), a3 = fmask(w.y, 1);
          const uint32_t e0 = fmask(w.x, 2), e1 = fmask(w.x, 3), e2 = fmask(w.y, 2), e3 = fmask(w.y, 3);
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            uint2 b;
            if constexpr (NG == 1) {
              b = make_uint2(bv[t][cc][0], bv[t][cc][1]);
            } else {
              const int row = t < NT01 ? (gi * NH + 4 * t + (mg >> 1)) * 3 + (mg & 1)
                                       : (gi * NH + min((mg >> 1) + 4 * (mg & 1), NH - 1)) * 3 + 2;
              b = *reinterpret_cast<const uint2 *>(un_u + row * S::VLP + 8 * cc + 2 * mt);
            }
            int *c01 = acc[t], *c23 = acc[t] + 4;
            mma_u8s8(*reinterpret_cast<int(*)[4]>(c01), a0, a1, a2, a3, b.x, b.y);
            mma_u8s8(*reinterpret_cast<int(*)[4]>(c23), e0, e1, e2, e3, b.x, b.y);
          }
        }
        const float fk[4] = {1.f, 0.25f, 0.0625f, 0.015625f};
#pragma unroll
        for (int t = 0; t < NT01; ++t) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float v01 = (float)(acc[t][2 * k] + 256 * acc[t][2 * k + 1]);   // |.| < 2^31
            const float tot = fmaf(65536.f, (float)acc[NT01][2 * k + t], v01);
            // channel 4 cq + k carried the factor 4^k; zero term: zl, at flush
            o_rot[t][cb][k] = fmaf(dwu * fk[k], tot, o_rot[t][cb][k]);
          }
        }
      }
    } else if (s.kind == 4) {
      mbar_wait(&bar[st], par);                       // empty unit marker (no data)
    } else {
      // ================= rows (rotated basis, one at a time)
      mbar_wait(&bar[st], par);
      const bool r16 = s.kind == 2;
      if (s.ring && app_k != nullptr) {
        const int tl = Lc - 1 - (lp.n_q + s.a);
        if (tl >= 0 && tl < s.n) {
          const int uu = cur_pu;
          const uint4 *sk = reinterpret_cast<const uint4 *>(app_k + (size_t)uu * D);
          const uint4 *svv = reinterpret_cast<const uint4 *>(app_v + (size_t)uu * D);
          uint8_t *Bw = B + (size_t)tl * 4 * D;
          uint4 *rrow = reinterpret_cast<uint4 *>(ring_row(c, uu, (Lc - 1) % c.slots));
          for (int i = lane; i < D / 8; i += 32) {
            const uint4 kv = sk[i], vv = svv[i];
            reinterpret_cast<uint4 *>(Bw)[i] = kv;
            reinterpret_cast<uint4 *>(Bw + 2 * D)[i] = vv;
            rrow[i] = kv;
            rrow[D / 8 + i] = vv;
          }
          if (lane == 0 && tsa && app_types != nullptr && app_types[uu] == 1)
            atomicOr(&c.bitmask[(size_t)uu * c.bm_words + (Lc - 1) / 32], 1u << ((Lc - 1) % 32));
          __syncwarp();
        }
      }
      const int nrows = s.ring ? min(s.n, Lc - lp.n_q - s.a) : s.n;
      for (int r = 0; r < nrows; ++r) {
        float k4[4], v4[4];
        if (r16) {                                    // 16-bit row (original basis) -> x . H
          const uint8_t *row = B + (size_t)r * 4 * D;
          const uint2 kw = *reinterpret_cast<const uint2 *>(row + 8 * vcq);
          const uint2 vw = *reinterpret_cast<const uint2 *>(row + 2 * D + 8 * vcq);
          cvt2<DT>(kw.x, k4[0], k4[1]); cvt2<DT>(kw.y, k4[2], k4[3]);
          cvt2<DT>(vw.x, v4[0], v4[1]); cvt2<DT>(vw.y, v4[2], v4[3]);
          auto fw = [&](float (&x)[4]) {
            { const float a = x[0], b = x[1]; x[0] = a + b; x[1] = a - b; }
            { const float a = x[2], b = x[3]; x[2] = a + b; x[3] = a - b; }
            { const float a = x[0], b = x[2]; x[0] = a + b; x[2] = a - b; }
            { const float a = x[1], b = x[3]; x[1] = a + b; x[3] = a - b; }
#pragma unroll
            for (int lm = 1; lm < CQ; lm <<= 1) {
              const bool upper = lane & lm;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float o2 = __shfl_xor_sync(0xffffffffu, x[k], lm);
                x[k] = upper ? o2 - x[k] : x[k] + o2;
              }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) x[k] *= rsd;
          };
          fw(k4);
          fw(v4);
        } else {                                      // 4-bit TSA text row (rotated, normalized)
          const uint8_t *e = B + (size_t)r * c.side_entry;
          const int gi = (4 * vcq) / G;
          const float sk = reinterpret_cast<const float *>(e)[gi];
          const float zk = (float)reinterpret_cast<const int32_t *>(e + 4 * NG)[gi];
          const float sv = reinterpret_cast<const float *>(e + 8 * NG)[gi];
          const float zv = (float)reinterpret_cast<const int32_t *>(e + 12 * NG)[gi];
          const uint32_t ck = *reinterpret_cast<const uint16_t *>(e + 16 * NG + 2 * vcq);
          const uint32_t cv = *reinterpret_cast<const uint16_t *>(e + 16 * NG + D / 2 + 2 * vcq);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            k4[k] = sk * ((float)((ck >> (4 * k)) & 15u) - zk);
            v4[k] = sv * ((float)((cv >> (4 * k)) & 15u) - zv);
          }
        }
        row_update(k4, v4, true);
      }
    }
    __syncwarp();
    rf = st;                                        // refill it at the loop top
    nrf = 1;
    if (++st == kLyStages) { st = 0; par ^= 1u; }
  }
  ly_exit(c, lp, lane, &cta_done);
}

template <int D, int G, int NH>
static size_t gq_smem(const DevCache &c) {
  return (size_t)kGqWarps * GqSmem<D, G, NH>::warp_bytes(ly_stage_bytes(c));
}

template <int D, int G, int DT, int NH>
static cudaError_t launch_gq(const DevCache &c, const LayerPlan &lp, const void *q, const void *k,
                             const void *v, const uint8_t *types, float *part, float *out,
                             uint32_t flags, cudaStream_t st) {
  const size_t smem = gq_smem<D, G, NH>(c);
  auto kern = c.kind == AKVQ_TSA ? k_decode_gqa<D, G, DT, NH, true> : k_decode_gqa<D, G, DT, NH, false>;
  {
    cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea == cudaSuccess)
      ea = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (ea != cudaSuccess) return ea;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((lp.W + kGqWarps - 1) / kGqWarps));
  cfg.blockDim = dim3(kGqWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c, lp, (const uint16_t *)q, (const uint16_t *)k,
                            (const uint16_t *)v, types, part, out, flags);
}

#ifndef AKVQ_GQ_MAXH
#define AKVQ_GQ_MAXH 8
#endif
int gqa_heads(int g) { return g <= 4 ? 4 : AKVQ_GQ_MAXH; }
int gqa_warps_per_cta() { return kGqWarps; }
int gqa_ctas_per_sm() { return AKVQ_GQ_CTAS; }
size_t gqa_record_floats(int d) { return (size_t)d + 4; }

cudaError_t launch_decode_gqa(const DevCache &c, int dtype16, const LayerPlan &lp, const void *q,
                              const void *k, const void *v, const uint8_t *types, float *part,
                              float *out, uint32_t flags, cudaStream_t st) {
  if (lp.T <= 0) return cudaSuccess;
  const int nh = gqa_heads(c.g);
#define AKVQ_GCASE(D_, G_)                                                                        \
  if (c.d == D_ && c.G == G_) {                                                                   \
    if (dtype16 == AKVQ_BF16)                                                                     \
      return nh == 4 ? launch_gq<D_, G_, AKVQ_BF16, 4>(c, lp, q, k, v, types, part, out, flags, st) \
                     : launch_gq<D_, G_, AKVQ_BF16, 8>(c, lp, q, k, v, types, part, out, flags, st); \
    return nh == 4 ? launch_gq<D_, G_, AKVQ_FP16, 4>(c, lp, q, k, v, types, part, out, flags, st)   \
                   : launch_gq<D_, G_, AKVQ_FP16, 8>(c, lp, q, k, v, types, part, out, flags, st);   \
  }
  AKVQ_GCASE(64, 32)
  AKVQ_GCASE(64, 64)
  AKVQ_GCASE(128, 32)
  AKVQ_GCASE(128, 64)
  AKVQ_GCASE(128, 128)
#undef AKVQ_GCASE
  return cudaErrorInvalidValue;
}

}  // namespace akvq
