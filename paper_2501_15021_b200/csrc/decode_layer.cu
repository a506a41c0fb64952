// decode_layer.cu -- AKVQ-VL single-query decode attention over one layer's
// packed cache on sm_100a, every tier in ONE persistent kernel:
//   2-bit pages      (K per channel, V per token; rotated basis)
//   16-bit ring rows (recent window) and PSA pivot rows,
//                    both in the ORIGINAL basis (R10)
//   4-bit TSA rows   (text tokens, R11; rotated basis)
// plus, for akvq_decode_step, the append of the new token (Eq. 2).
//
// Work list.  Every unit has the same host-built table of items (kernel
// parameter LayerPlan::tab): its P pages (two sub-loads each, K half: K meta +
// K codes; V half: V meta + V codes, never split across warps), Rc ring chunks (kRows rows) and Sc side
// splits, INTERLEAVED (the rows placed before page p are the first floor(p*NR/P)
// row items, NR = Rc + Sc), so every contiguous range of the flattened
// (unit-major) list has the same mix of ALU-heavy page work and memory-heavy
// row work.  Warp w of the persistent grid owns items [w*T/W, (w+1)*T/W) and
// streams their bytes through its own shared-memory stages with 1-D TMA bulk
// copies (cp.async.bulk + mbarrier); a side split (runtime entry count) may
// take several sub-loads.
//
// Arithmetic (profiles/r01_microbench_pipes.md):
//  pages, logits: q~ * s^K rounded once per page to a 16-bit fixed point Q_c
//    (two signed int8 limbs); sum_c Q_c code_tc for all G tokens is one warp-MMA
//    contraction (IMMA m16n8k32: A = LOP3-masked K tile words, rows = tokens;
//    B = the limbs, columns = 2 per head), exact in int32;
//    logit = delta (sum - sum_c Q_c z_c).  Per-token K: the same MMA, folded per
//    channel group with the token's scale and zero point.
//  pages, values: w_t = p_t s^V_t rounded to a 16-bit fixed point of the page's
//    largest weight (two uint8 limbs); sum_t W_t code_tc is the second warp-MMA
//    contraction (A = masked V tile words, rows = channels):
//    o'_c += dw (sum_t W_t code_tc - sum_t W_t z_t).
//  rows: lane = channel quad (8-byte slices, conflict-free LDS.64); per-row dot
//    products are reduced across lanes with a reduce-scatter.
// One online softmax (base 2) per (warp, unit) segment with two accumulators:
// o_rot (rotated basis: pages, 4-bit rows) and o_org (original basis: 16-bit
// rows).  Each segment writes one partial; the writer of a unit's last segment
// (per-unit ticket) merges them: log-sum-exp, out = (o_rot . H + o_org) / l.
#include <math.h>

#include <type_traits>

#include "decode_common.cuh"

namespace akvq {

constexpr int kLyWarps = 4;        // warps per CTA
#ifndef AKVQ_R16U
#define AKVQ_R16U 8
#endif
#ifndef AKVQ_R4U
#define AKVQ_R4U 2
#endif
#ifndef AKVQ_SIDE_RR
#define AKVQ_SIDE_RR 1             // side splits take round-robin sub-loads (A/B knob)
#endif
constexpr int kLimbCols = 4;
#ifndef AKVQ_LY_CTAS
#define AKVQ_LY_CTAS 4
#endif
__host__ __device__ constexpr int ly_ctas_per_sm(int nh) { return nh >= 4 ? 2 : (nh >= 2 ? 3 : AKVQ_LY_CTAS); }

// Per-warp shared memory (bytes):
//   stages [kLyStages][SB] | qh [NH][D] f32 (q~ = q.H_s) | limbs: K [NH][D/16][8]
//   u32 during a K half, V [NH][NG][G/16][8] u32 during a V half (same bytes) |
//   sub-load descriptors | barriers
template <int D, int G, int NH>
struct LySmem {
  static constexpr int NG = D / G;
  static __host__ __device__ size_t qh_off(size_t sb) { return kLyStages * sb; }
  // limbs: K [kLimbCols NH][D/4] u32, V [NG][kLimbCols NH][G/4] u32
  static constexpr size_t KL = (size_t)NH * kLimbCols * D, VL = (size_t)NH * NG * kLimbCols * G;
  static __host__ __device__ size_t kl_off(size_t sb) { return qh_off(sb) + NH * D * 4; }
  static __host__ __device__ size_t vl_off(size_t sb) { return kl_off(sb); }   // shared
  // page logits [NH][G] / page V sums [NH][D] (fp32, one at a time)
  static __host__ __device__ size_t lv_off(size_t sb) { return kl_off(sb) + (KL > VL ? KL : VL); }
  // [2][NH + 1][D] f32: per-limb-pair partial sums (even / odd MMA lanes; row NH
  // takes the stores of padded lanes, so the epilogue needs no branch), G <= D
  // rows are LP = D + 8 floats apart: the 4 MMA lanes of a fragment group (rows
  // even/odd x head/dummy) then store to distinct banks
  static constexpr int LP = D + 8;
  static __host__ __device__ size_t ds_off(size_t sb) { return lv_off(sb) + (size_t)2 * (NH + 1) * LP * 4; }
  static __host__ __device__ size_t bar_off(size_t sb) { return ds_off(sb) + kLyStages * 32; }
  static __host__ __device__ size_t warp_bytes(size_t sb) {
    return (bar_off(sb) + kLyStages * 8 + 127) / 128 * 128;
  }
};

template <int D, int G, int DT, int NH, bool TSA, int KM, bool DL>
__global__ void __launch_bounds__(kLyWarps * 32, ly_ctas_per_sm(NH))
    k_decode_layer(const __grid_constant__ DevCache c, const __grid_constant__ LayerPlan lp, const uint16_t *__restrict__ q,
                   const uint16_t *__restrict__ app_k, const uint16_t *__restrict__ app_v,
                   const uint8_t *__restrict__ app_types, float *__restrict__ part,
                   float *__restrict__ out, uint32_t flags) {
  using S = LySmem<D, G, NH>;
  constexpr bool KT = KM == 1;              // per-token K (AKVQ_K_PER_TOKEN)
  constexpr bool SO = KM == 2;              // profiling: TMA pipeline only (LayerPlan::stream_only)
  constexpr int NG = D / G;
  constexpr int CQ = D / 4, TQ = G / 4;     // channel quads, token quads
  constexpr int CG = D / 16, TG = G / 16;   // 4-quad groups (one LDS.128 of tile words)
  constexpr int KCS = 32 / TQ;              // page K phase: lanes per token quad
  constexpr int VTS = 32 / CQ;              // V phase / rows: lanes per channel quad
  constexpr int NV = kRows / VTS;           // rows per lane per 8-row group
  constexpr int BFLY = CQ / NV;             // lanes holding the same row total
  static_assert(TQ <= 32 && CQ <= 32 && CG % KCS == 0 && TG % VTS == 0, "page shape");
  static_assert(BFLY == 4, "row groups: lane bits >= 2 index the rows");
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ unsigned cta_done;                 // warps of this CTA done (ly_exit)
  if constexpr (DL) {                           // DEVICE_L: per-CTA exit count
    if (threadIdx.x == 0) cta_done = 0u;
    __syncthreads();
  }
  const size_t SB = ly_stage_bytes(c);
  uint8_t *wsm = smem + (size_t)warp * S::warp_bytes(SB);
  float *qh = reinterpret_cast<float *>(wsm + S::qh_off(SB));
  uint32_t *klimb = reinterpret_cast<uint32_t *>(wsm + S::kl_off(SB));
  uint32_t *vlimb = reinterpret_cast<uint32_t *>(wsm + S::vl_off(SB));
  uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + S::bar_off(SB));
  const uint32_t bar_s = smem_u32(bar), wsm_s = smem_u32(wsm);   // shared-window addresses

  // Programmatic dependent launch: q, k, v (and, after a flush or append, the
  // cache) come from the preceding grid.  When the host knows the preceding grid
  // does not write this cache (lp.prologue), the first cache sub-loads are
  // issued before griddepcontrol.wait, overlapping the previous layer's tail.
  if (!lp.prologue) {
    pdl_wait();
    pdl_launch_dependents();                    // the next layer's kernel may queue up
  }
  const int gw = blockIdx.x * kLyWarps + warp;
  if (gw >= lp.W) { if constexpr (DL) ly_exit(c, lp, lane, &cta_done); return; }
  const int ib = ly_first_item_p(&lp, gw);       // (one out-of-line copy: code size)
  const int ie = gw + 1 < lp.W ? ly_first_item_p(&lp, gw + 1) : lp.T;
  if (ib >= ie) { if constexpr (DL) ly_exit(c, lp, lane, &cta_done); return; }
  // this launch's token count, the new token included when it appends (DEVICE_L
  // launches have no prologue: the griddepcontrol.wait above has been passed)
  const int Lc = DL ? c.dstate->L + (lp.appends ? 1 : 0) : lp.L;
  constexpr bool tsa = TSA;                     // layer kind (Table I): TSA has 4-bit text rows
  // GQA (NEXT-3): a unit's g query heads are processed in HG groups of NH heads;
  // work items, partials and tickets are per virtual unit vu = u * HG + group
  const int HG = lp.hg;
  const float alpha_k = kLog2e / (float)D;     // (q.H_s) . K^ / d in log2 units
  const float alpha_o = kLog2e * c.inv_sqrt_d; // q.k / sqrt d in log2 units
  const uint32_t kbytes = c.pg_vscale, vbytes = c.page_bytes - c.pg_vscale;

  // ---- producer: every lane walks the same items (warp-uniform state, the
  // descriptors of the two stages stay in registers); lane 0 issues the TMA
  // sub-loads.  A page is two sub-loads (K half, V half); the V half is issued
  // from the pointer remembered with the K half.
  if (lane == 0) {
    for (int s = 0; s < kLyStages; ++s) mbar_init(&bar[s]);
    mbar_fence_init();
  }
  __syncwarp();
  int pu = ib / lp.per_u, pj = ib - (ib / lp.per_u) * lp.per_u, left = ie - ib, part_i = 0;
  int pphys = pu / HG, phg = pu - (pu / HG) * HG;   // physical unit / head group of pu
  const uint8_t *ubase = c.pages + (size_t)pphys * c.n_pages * c.page_bytes;   // pages of pphys
  int eu = -1;                                  // last (virtual) unit a sub-load was issued for
  const uint8_t *vsrc = nullptr;                // pending V half (issued next)
  uint2 vdesc = make_uint2(0u, 0u);
  // salient bits of a page's tokens, loaded with its K half (this lane's word:
  // tokens 32 (ktq >> 3) .. of the page, the lane's token quad is ktq)
  uint32_t pbits = 0u;
  const int pbw = (lane % (G / 4)) >> 3;
  auto produce = [&](int st) -> uint2 {
    const uint32_t dst = wsm_s + (uint32_t)st * (uint32_t)SB, bst = bar_s + 8u * st;
    if (vsrc != nullptr) {                      // V half of the page whose K half went last
      if (lane == 0) {
        mbar_expect_tx(bst, vbytes);
        bulk_g2s(dst, vsrc, vbytes, bst);
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
      if (kind == 0) {                            // page: K half now, V half next
        sb.kind = 0; sb.n = 0;
      } else if (kind == 2) {                     // ring chunk (rows n of it)
        sb.kind = 2; sb.ring = 1; sb.n = n;
        if constexpr (DL) {                       // chunks of the period past L: skip
          sb.n = min(n, Lc - lp.n_q - a);
          ok = sb.n > 0;
        }
      } else {                                    // side split a: entries [lo, hi), runtime count
        const int cnt = __ldg(c.side_cnt + pphys);
        // floor(a cnt / Sc) and floor((a + 1) cnt / Sc): fp32 estimate, corrected
        // (a cnt < 2^24: cnt <= capacity, a < Sc <= 8)
        auto fdiv = [&](int x) {
          int qd = __float2int_rz((float)x * lp.sc_inv);
          qd += (qd + 1) * lp.Sc <= x;
          qd -= qd * lp.Sc > x;
          return qd;
        };
        const int per = tsa ? kRows4 : kRows;
        sb.kind = tsa ? 3 : 2;
#if AKVQ_SIDE_RR
        // round-robin: split a takes the per-row sub-loads a, a + Sc, a + 2 Sc, ...
        // (full sub-loads whatever the runtime count; splits past it are empty)
        (void)fdiv;
        sb.a = (a + part_i * lp.Sc) * per;
        sb.n = min(per, cnt - sb.a);
#else
        const int lo = fdiv(a * cnt), hi = fdiv((a + 1) * cnt);
        sb.a = lo + part_i * per;
        sb.n = min(per, hi - sb.a);
#endif
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
            mbar_expect_tx(bst, kbytes);
            bulk_g2s(dst, pg, kbytes, bst);
          }
          pbits = __ldg(c.bitmask + (size_t)sb.pu * c.bm_words + (size_t)a * (G / 32) + pbw);
          if constexpr (KT) {                     // exact R (R26): the last page is partial;
            const int lim = lp.n_q - a * G - pbw * 32;   // its tokens >= n_q act as salient
            if (lim < 32) pbits |= lim <= 0 ? ~0u : (~0u << lim);
          }
          vsrc = pg + kbytes;
          LySub vb = sb;
          vb.kind = 1;
          vdesc = pack_sub(vb);
        } else if (sb.ring) {
          int s0 = lp.nq_mod + sb.a;              // ring slot of row n_q + a
          if (s0 >= c.slots) s0 -= c.slots;
          const int n1 = min(sb.n, c.slots - s0);
          const uint32_t rowb = 4 * D;
          if (lane == 0) {
            mbar_expect_tx(bst, (uint32_t)sb.n * rowb);
            bulk_g2s(dst, ring_row(c, sb.pu, s0), (uint32_t)n1 * rowb, bst);
            if (n1 < sb.n)
              bulk_g2s(dst + (uint32_t)n1 * rowb, ring_row(c, sb.pu, 0), (uint32_t)(sb.n - n1) * rowb, bst);
          }
        } else {
          const uint32_t eb = c.side_entry;
          if (lane == 0) {
            mbar_expect_tx(bst, (uint32_t)sb.n * eb);
            bulk_g2s(dst, side_ptr(c, sb.pu, sb.a), (uint32_t)sb.n * eb, bst);
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
        if (lane == 0) mbar_expect_tx(bst, 0u);
        break;
      }
      sb.kind = -1;
    }
    return pack_sub(sb);
  };
  // stage descriptors; both stages are primed by the loop's (single) producer
  // call site before the first consume (one inlined copy of produce)
  uint2 dsc0 = make_uint2(0u, 0u), dsc1 = make_uint2(0u, 0u);
  uint32_t bits0 = 0u, bits1 = 0u;
  static_assert(kLyStages == 2, "two stages: descriptors dsc0 / dsc1");

  // lane roles
  const int ktq = lane % TQ, kcs = lane / TQ;         // page K phase
  const int vcq = lane % CQ, vts = lane / CQ;         // page V phase and rows
  const int vgam = (4 * vcq) / G;                     // channel group of the lane's quad
  const int mg = lane >> 2, mt = lane & 3;            // page MMA: fragment group / thread in group
  // B column of the lane: head mg / 4, limb mg % 4 (the unused 4th column and
  // padded heads read a valid limb; their results are never used)
  const int mcol = [&] { const int m = min(mg, kLimbCols * NH - 1); return (m & 3) == 3 ? m - 1 : m; }();
  // MMA result columns 2 mt, 2 mt + 1 of this lane: head mt / 2; even mt holds
  // limbs 0 and 1, odd mt limb 2 (and the unused column)
  const int rhead = mt >> 1;
  const bool rodd = mt & 1;
  static_assert(kLimbCols * NH <= 8, "one MMA n-tile: at most 2 heads of 4 limb columns");
  uint32_t *qlimb = klimb;                            // [4 NH][CQ] Q limbs (page MMA layout)
  uint32_t *wlimb = vlimb;                            // [NG][4 NH][TQ] W limbs
  // page logits / V sums, split by limb pair: [2][NH][D] (row 0: limbs 0 + 256 x 1
  // from even MMA lanes, row 1: limb 2 from odd lanes; x 65536 when combined)
  float *lgs = reinterpret_cast<float *>(wsm + S::lv_off(SB));

  // per-unit segment state
  // l_run and zl are per-lane partials (each lane adds its own tokens / rows),
  // reduced across the warp once per segment in flush
  float m_run[NH], l_run[NH], o_rot[NH][4], o_org[NH][4], zl[NH][NG];
  float qk[NH][4], qt[NH][4], qsum[NH];               // q (orig) * alpha_o; q~ * alpha_k; sum
  // per-unit fixed points (per-channel K): Q_c = rn(q~_c s^K_c inv), inv =
  // kQMax / (max_c |q~_c| * umax.K), so |Q| <= kQMax on every page of the unit;
  // qinv = q~ * inv for the lane's channel quad; dA = alpha_k / inv.  V weights:
  // W_t = rn(p_t s^V_t winv) with winv = kQMax / umax.V (p <= 1), dw = 1 / winv.
  float qinv[NH][4], dAu[NH], winv = 0.f, dwu = 0.f;
  // per-token K (KT): this lane's delta and limb sums, fixed per unit
  float kt_d = 0.f, kt_s[2][NG];
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) { kt_s[0][gi] = 0.f; kt_s[1][gi] = 0.f; }
  float lg[NH][4];                                    // page logits of the lane's token quad
  int cur_u = -1, cur_pu = 0, cur_hg = 0;      // virtual unit, its physical unit and head group
  const int u_first = ib / lp.per_u;

  auto flush = [&](int u) {
    const size_t slot = (size_t)gw * lp.maxseg + (u - u_first);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int off = CQ; off < 32; off <<= 1) {
          o_rot[h][s] += __shfl_xor_sync(0xffffffffu, o_rot[h][s], off);
          o_org[h][s] += __shfl_xor_sync(0xffffffffu, o_org[h][s], off);
        }
      }
      // page zero-point terms: sum_t W_t z_t of every page (rescaled like o_rot),
      // subtracted once from every channel of its group
      float zg = 0.f;
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        const float z = warp_sum(zl[h][gi]);
        if (gi == vgam) zg = z;
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) o_rot[h][s] -= zg;
      l_run[h] = warp_sum(l_run[h]);
      float *rec = part + (slot * NH + h) * Rec<D>::R;
      if (vts == 0) {
        reinterpret_cast<float4 *>(rec)[vcq] = make_float4(o_org[h][0], o_org[h][1], o_org[h][2], o_org[h][3]);
        reinterpret_cast<float4 *>(rec + D)[vcq] = make_float4(o_rot[h][0], o_rot[h][1], o_rot[h][2], o_rot[h][3]);
      }
      if (lane == 0) { rec[2 * D] = m_run[h]; rec[2 * D + 1] = l_run[h]; }
    }
    const int w_lo = ly_warp_of(lp, u, 0), w_hi = ly_warp_of(lp, u, lp.per_u - 1);
    if (take_ticket(c, u, w_hi - w_lo + 1, lane)) {
      const int hg = u % HG, nh = min(NH, c.g - hg * NH);
      merge_layer_unit<D, NH>(c, lp, part, u, out + ((size_t)(u / HG) * c.g + hg * NH) * D, nh,
                              flags, lane);
      if (lane == 0) c.ticket[u] = 0u;
    }
  };

  // One group of n <= kRows rows (16-bit original-basis rows, or 4-bit TSA rows)
  // staged at shared address sb0 with the given pitch.  Lane (vcq, vts) handles
  // channels 4vcq..4vcq+3 of rows vts + VTS*i.  Rows n..kRows-1 of a partial
  // group were zero-filled by the caller (finite), their logits are masked.
  auto rows_group = [&](uint32_t sb0, uint32_t pitch, int n, auto r16_tag) {
    constexpr bool r16 = decltype(r16_tag)::value;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      float dot[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const uint32_t ra = sb0 + (uint32_t)(vts + VTS * i) * pitch;
        if (r16) {
          const uint2 v = lds64(ra + 8 * vcq);
          float a0, a1, a2, a3;
          cvt2<DT>(v.x, a0, a1);
          cvt2<DT>(v.y, a2, a3);
          float2 t2 = __fmul2_rn(make_float2(qk[h][0], qk[h][1]), make_float2(a0, a1));
          t2 = __ffma2_rn(make_float2(qk[h][2], qk[h][3]), make_float2(a2, a3), t2);
          dot[i] = t2.x + t2.y;
        } else {   // s_g (sum q~ code - z_g sum q~) over the lane's 4 channels
          const float sk = lds_f32(ra + 4 * vgam);
          const float zk = (float)lds_s32(ra + 4 * NG + 4 * vgam);
          const uint32_t cw = lds16(ra + 16 * NG + 2 * vcq);
          float a = qt[h][0] * (float)(cw & 15u);
          a = fmaf(qt[h][1], (float)((cw >> 4) & 15u), a);
          a = fmaf(qt[h][2], (float)((cw >> 8) & 15u), a);
          a = fmaf(qt[h][3], (float)(cw >> 12), a);
          dot[i] = sk * fmaf(-zk, qsum[h], a);
        }
      }
      int mine;
      float t = rs_reduce<NV, CQ>(dot, vcq, mine);
      t = (vts + VTS * mine) < n ? t : -INFINITY;
      // softmax over the group: lane bits 2..4 index the rows (bits 0, 1 replicate)
      float mx = t;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_run[h], mx);
      const float sc = ex2(m_run[h] - m_new);
      const float p = ex2(t - m_new);
      // one lane per row (vcq & 3 == 0) adds its row's p to the lane partial
      l_run[h] = fmaf(l_run[h], sc, (vcq & 3) == 0 ? p : 0.f);
      m_run[h] = m_new;
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) zl[h][gi] *= sc;
      if (r16) {
        float2 oa = __fmul2_rn(make_float2(o_org[h][0], o_org[h][1]), make_float2(sc, sc));
        float2 ob = __fmul2_rn(make_float2(o_org[h][2], o_org[h][3]), make_float2(sc, sc));
        AKVQ_UNROLL(AKVQ_R16U)                // 16-bit rows: code size knob
        for (int i = 0; i < NV; ++i) {
          const int row = vts + VTS * i;
          const float pr = __shfl_sync(0xffffffffu, p, (lane & (BFLY - 1)) | rs_enc<NV, CQ>(i) | (vts * CQ));
          const uint2 v = lds64(sb0 + (uint32_t)row * pitch + 2 * D + 8 * vcq);
          float a0, a1, a2, a3;
          cvt2<DT>(v.x, a0, a1);
          cvt2<DT>(v.y, a2, a3);
          oa = __ffma2_rn(make_float2(pr, pr), make_float2(a0, a1), oa);
          ob = __ffma2_rn(make_float2(pr, pr), make_float2(a2, a3), ob);
        }
        o_org[h][0] = oa.x; o_org[h][1] = oa.y; o_org[h][2] = ob.x; o_org[h][3] = ob.y;
#pragma unroll
        for (int k = 0; k < 4; ++k) o_rot[h][k] *= sc;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { o_rot[h][k] *= sc; o_org[h][k] *= sc; }
        AKVQ_UNROLL(AKVQ_R4U)                 // 4-bit rows (TSA only): code size knob
        for (int i = 0; i < NV; ++i) {
          const int row = vts + VTS * i;
          const float pr = __shfl_sync(0xffffffffu, p, (lane & (BFLY - 1)) | rs_enc<NV, CQ>(i) | (vts * CQ));
          const uint32_t ra = sb0 + (uint32_t)row * pitch;
          const float sv = lds_f32(ra + 8 * NG + 4 * vgam);
          const float zv = (float)lds_s32(ra + 12 * NG + 4 * vgam);
          const uint32_t cw = lds16(ra + 16 * NG + D / 2 + 2 * vcq);
          const float wt = pr * sv;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o_rot[h][k] = fmaf(wt, (float)((cw >> (4 * k)) & 15u) - zv, o_rot[h][k]);
        }
      }
    }
  };

  int st = 0;
  uint32_t par = 0;
  bool unit_fresh = false;                          // KT: q limbs of the new unit pending
  int rf = 0, nrf = kLyStages;                      // stages to (re)fill: both at first
  bool first = true;
  for (;;) {
#pragma unroll 1
    for (; nrf > 0; --nrf, rf ^= 1) {               // the only producer call site
      const uint2 d = produce(rf);
      if (rf) { dsc1 = d; bits1 = pbits; } else { dsc0 = d; bits0 = pbits; }
    }
    if (first) {
      first = false;
      if (lp.prologue) {                          // inputs from the preceding grid from here on
        pdl_wait();
        pdl_launch_dependents();
      }
      // host-L mode: keep the device copy current (a later DEVICE_L launch reads it)
      if constexpr (!DL)
        if (lp.appends && blockIdx.x == 0 && threadIdx.x == 0) c.dstate->L = lp.L;
    }
    const LySub s = unpack_sub(st ? dsc1 : dsc0);
    if constexpr (SO) {                             // profiling: pipeline only
      if (s.kind < 0) break;
      mbar_wait(bar_s + 8u * st, par);
      __syncwarp();
      rf = st;
      nrf = 1;
      if (++st == kLyStages) { st = 0; par ^= 1u; }
      continue;
    }
    uint8_t *B = wsm + (size_t)st * SB;
    if (s.kind < 0 || s.u != cur_u) {               // segment boundary (one flush site)
      if (cur_u >= 0) flush(cur_u);
      if (s.kind < 0) break;
      cur_u = s.u;
      unit_fresh = true;
      cur_pu = s.u / HG;
      cur_hg = s.u - cur_pu * HG;
      // q~ = q . H_s (unnormalized FWHT: in-register then shuffle butterflies)
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        constexpr int CPL = D / 32;
        float x[CPL];
        const uint16_t *qs = q + ((size_t)cur_pu * c.g + min(cur_hg * NH + h, c.g - 1)) * D + CPL * lane;
        if constexpr (CPL == 4) {
          const uint2 v = *reinterpret_cast<const uint2 *>(qs);
          cvt2<DT>(v.x, x[0], x[1]);
          cvt2<DT>(v.y, x[2], x[3]);
        } else {
          cvt2<DT>(*reinterpret_cast<const uint32_t *>(qs), x[0], x[1]);
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
        const uint2 v = *reinterpret_cast<const uint2 *>(
            q + ((size_t)cur_pu * c.g + min(cur_hg * NH + h, c.g - 1)) * D + 4 * vcq);
        cvt2<DT>(v.x, qk[h][0], qk[h][1]);
        cvt2<DT>(v.y, qk[h][2], qk[h][3]);
        const float4 t4 = reinterpret_cast<const float4 *>(qh + h * D)[vcq];
        qt[h][0] = t4.x * alpha_k; qt[h][1] = t4.y * alpha_k;
        qt[h][2] = t4.z * alpha_k; qt[h][3] = t4.w * alpha_k;
        qsum[h] = (qt[h][0] + qt[h][1]) + (qt[h][2] + qt[h][3]);
        if constexpr (!KT) {
          const float2 um = c.umax[cur_pu];
          const float M = warp_max(fmaxf(fmaxf(fabsf(t4.x), fabsf(t4.y)), fmaxf(fabsf(t4.z), fabsf(t4.w)))) * um.x;
          const float inv = M > 0.f ? __fdividef((float)kQMax, M) : 0.f;
          dAu[h] = alpha_k * M * (1.0f / (float)kQMax);
          qinv[h][0] = t4.x * inv; qinv[h][1] = t4.y * inv; qinv[h][2] = t4.z * inv; qinv[h][3] = t4.w * inv;
          winv = um.y > 0.f ? __fdividef((float)kQMax, um.y) : 0.f;
          dwu = um.y * (1.0f / (float)kQMax);
        } else {
          const float um_v = c.umax[cur_pu].y;
          winv = um_v > 0.f ? __fdividef((float)kQMax, um_v) : 0.f;
          dwu = um_v * (1.0f / (float)kQMax);
          qinv[h][0] = t4.x; qinv[h][1] = t4.y; qinv[h][2] = t4.z; qinv[h][3] = t4.w;   // q~ (KT)
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) { qk[h][k] *= alpha_o; o_rot[h][k] = 0.f; o_org[h][k] = 0.f; }
        m_run[h] = -INFINITY;
        l_run[h] = 0.f;
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) zl[h][gi] = 0.f;
      }
    }

    if constexpr (KT) {
      if (unit_fresh) {
        // ---- per-token K (NEXT-1): Q_c = rn(q~_c / delta) once per unit
        // (it does not depend on the page); the limb words replace q~ in qh (KT
        // reads q~ only here), the page loop reloads them as B fragments.
        // SQ_k,g = sum_{c in g} limb_k,c for the zero-point term.
        unit_fresh = false;
        __syncwarp();                            // every lane has read its q~ quad
        uint32_t *ql = reinterpret_cast<uint32_t *>(qh);
        float dT[NH], sqg[NH][2][NG];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const bool in = lane < CQ;
          const float am = in ? fmaxf(fmaxf(fabsf(qinv[h][0]), fabsf(qinv[h][1])),
                                      fmaxf(fabsf(qinv[h][2]), fabsf(qinv[h][3]))) : 0.f;
          const float M = warp_max(am);
          const float inv = M > 0.f ? __fdividef((float)kQMax, M) : 0.f;
          dT[h] = alpha_k * M * (1.0f / (float)kQMax);
          uint32_t x[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) x[b] = (uint32_t)__float2int_rn(in ? qinv[h][b] * inv : 0.f) + kQOff;
          int sq[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            sq[k] = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) sq[k] += (int)((x[b] >> (8 * k)) & 255u) - 128;
#pragma unroll
            for (int o = 1; o < G / 4 && o < 32; o <<= 1) sq[k] += __shfl_xor_sync(0xffffffffu, sq[k], o);
          }
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) {
            const int src = (gi * (G / 4)) & 31;
            const float s0 = (float)__shfl_sync(0xffffffffu, sq[0], src);
            const float s1 = (float)__shfl_sync(0xffffffffu, sq[1], src);
            const float s2 = (float)__shfl_sync(0xffffffffu, sq[2], src);
            sqg[h][0][gi] = rodd ? s2 : s0;
            sqg[h][1][gi] = rodd ? 0.f : s1;
          }
          __syncwarp();
          if (in) {
            ql[(4 * h) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0040), prmt(x[2], x[3], 0x0040), 0x5410) ^ 0x80808080u;
            ql[(4 * h + 1) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0051), prmt(x[2], x[3], 0x0051), 0x5410) ^ 0x80808080u;
            ql[(4 * h + 2) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0062), prmt(x[2], x[3], 0x0062), 0x5410) ^ 0x80808080u;
          }
        }
        const int hsel = min(rhead, NH - 1);
        kt_d = dT[0];
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) { kt_s[0][gi] = sqg[0][0][gi]; kt_s[1][gi] = sqg[0][1][gi]; }
#pragma unroll
        for (int h = 1; h < NH; ++h)
          if (hsel == h) {
            kt_d = dT[h];
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) { kt_s[0][gi] = sqg[h][0][gi]; kt_s[1][gi] = sqg[h][1][gi]; }
          }
        __syncwarp();
      }
    }

    if (s.kind == 0) {
      // ================= page K half: logits of the page's G tokens
      const uint32_t sbits = ((st ? bits1 : bits0) >> (4 * (ktq & 7))) & 15u;
      mbar_wait(bar_s + 8u * st, par);
      const float4 *ks4 = reinterpret_cast<const float4 *>(B + c.pg_kscale);
      const int4 *kz4 = reinterpret_cast<const int4 *>(B + c.pg_kzero);
      if constexpr (KT) {                      // per-token K variant (compile time)
        // ---- per-token K (NEXT-1): Q_c = rn(q~_c / delta) (once per unit),
        // logit_t = alpha delta sum_g s_tg sum_k 256^k (C_k,tg - z_tg SQ_k,g) with
        // C_k,tg = sum_{c in g} limb_k,c code_tc (the warp MMA, folded per
        // channel group: a 32-channel chunk lies in one group since G >= 32) and
        // SQ_k,g = sum_{c in g} limb_k,c
        const float *ksT = reinterpret_cast<const float *>(B + c.pg_kscale);    // [G][NG]
        const int32_t *kzT = reinterpret_cast<const int32_t *>(B + c.pg_kzero);
        constexpr int KC = D / 32, CPG = G / 32;     // chunks, chunks per channel group
        const uint32_t *ql = reinterpret_cast<const uint32_t *>(qh);   // q limbs (unit switch)
        uint32_t bq[KC][2];
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) {
          const uint2 b = *reinterpret_cast<const uint2 *>(ql + mcol * CQ + 8 * cc + 2 * mt);
          bq[cc][0] = b.x;
          bq[cc][1] = b.y;
        }
        const float dsel = kt_d;
        const float (&ssel)[2][NG] = kt_s;
        // even lanes: limbs 0 (x 1) and 1 (x 256); odd lanes: limb 2 (x 65536)
        const float wA = rodd ? 65536.f : 1.f, wB = rodd ? 0.f : 256.f;
        const uint32_t *kcw = reinterpret_cast<const uint32_t *>(B + c.pg_kcodes);
        AKVQ_UNROLL(AKVQ_KU)
        for (int blk = 0; blk < TQ / 8; ++blk) {
          const int tq = 8 * blk + mg;
          float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) {
            int c01[4] = {0, 0, 0, 0}, c23[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < CPG; ++j) {
              const int cc = gi * CPG + j;
              const uint2 w = *reinterpret_cast<const uint2 *>(kcw + kword_idx(8 * cc + 2 * mt, tq, TQ));
              mma_u8s8(c01, fmask(w.x, 0), fmask(w.x, 1), fmask(w.y, 0), fmask(w.y, 1), bq[cc][0], bq[cc][1]);
              mma_u8s8(c23, fmask(w.x, 2), fmask(w.x, 3), fmask(w.y, 2), fmask(w.y, 3), bq[cc][0], bq[cc][1]);
            }
            // token 4tq+0 (x1): c01[0..1]; 4tq+1 (x4): c01[2..3]; 4tq+2 (x16): c23[0..1]; 4tq+3 (x64): c23[2..3]
            const int ca[4] = {c01[0], c01[2], c23[0], c23[2]}, cb[4] = {c01[1], c01[3], c23[1], c23[3]};
            const float fk[4] = {1.f, 0.25f, 0.0625f, 0.015625f};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int mi = (4 * tq + k) * NG + gi;
              const float z = (float)kzT[mi];
              const float t = fmaf(wA, fmaf((float)ca[k], fk[k], -z * ssel[0][gi]),
                                   wB * fmaf((float)cb[k], fk[k], -z * ssel[1][gi]));
              part[k] = fmaf(ksT[mi], t, part[k]);
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) part[k] += __shfl_xor_sync(0xffffffffu, part[k], 1);
          if (!rodd && rhead < NH) {
            float4 r;
            r.x = part[0] * dsel; r.y = part[1] * dsel; r.z = part[2] * dsel; r.w = part[3] * dsel;
            reinterpret_cast<float4 *>(lgs + rhead * S::LP)[tq] = r;
          }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const float4 r = reinterpret_cast<const float4 *>(lgs + h * S::LP)[ktq];
          lg[h][0] = (sbits & 1u) ? -INFINITY : r.x;
          lg[h][1] = (sbits & 2u) ? -INFINITY : r.y;
          lg[h][2] = (sbits & 4u) ? -INFINITY : r.z;
          lg[h][3] = (sbits & 8u) ? -INFINITY : r.w;
        }
      } else {
      float dA[NH];
      int bA[NH][3];
      bool sat = false;                  // REDUX bias: a lane partial out of range
#pragma unroll
      for (int h = 0; h < NH; ++h) {      // Q_c = rn(q~_c s^K_c inv): lane = channel quad
        float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
        int4 zq = make_int4(0, 0, 0, 0);
        if (lane < CQ) { sv = ks4[lane]; zq = kz4[lane]; }
        uint32_t x[4];
        x[0] = (uint32_t)__float2int_rn(qinv[h][0] * sv.x) + kQOff;
        x[1] = (uint32_t)__float2int_rn(qinv[h][1] * sv.y) + kQOff;
        x[2] = (uint32_t)__float2int_rn(qinv[h][2] * sv.z) + kQOff;
        x[3] = (uint32_t)__float2int_rn(qinv[h][3] * sv.w) + kQOff;
        // zero-point bias B = sum_c Q_c z_c exactly (int64), split into limb
        // terms B = b0 + 256 b1 + 65536 b2 with b0, b1 in [0, 255] (the MMA
        // accumulators start at -4^k b_limb; |4^k b2| < 2^31 for any int32 z
        // with |z| < 2^14)
        long long bz = (long long)(int)(x[0] - kQOff) * zq.x + (long long)(int)(x[1] - kQOff) * zq.y +
                       (long long)(int)(x[2] - kQOff) * zq.z + (long long)(int)(x[3] - kQOff) * zq.w;
#if AKVQ_REDUX
        // two 32-bit REDUX sums: lane partial = hi 65536 + lo, lo in [0, 65535]
        // (sum < 2^21), hi saturated at +-2^26 (sum < 2^31); a saturated lane
        // sends the page to the fp32 path (its bias is beyond the MMA range anyway)
        {
          const long long hl = bz >> 16;
          const int hi = (int)(hl > (1LL << 26) ? (1LL << 26) : (hl < -(1LL << 26) ? -(1LL << 26) : hl));
          sat |= hi == (1 << 26) || hi == -(1 << 26);
          const unsigned slo = __reduce_add_sync(0xffffffffu, (unsigned)(bz & 0xffff));
          const int shi = __reduce_add_sync(0xffffffffu, hi);
          bA[h][0] = (int)(slo & 255u);
          bA[h][1] = (int)((slo >> 8) & 255u);
          bA[h][2] = shi + (int)(slo >> 16);
        }
#else
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bz += __shfl_xor_sync(0xffffffffu, bz, o);
        bA[h][0] = (int)(bz & 255);
        bA[h][1] = (int)((bz >> 8) & 255);
        bA[h][2] = (int)(bz >> 16);
#endif
        dA[h] = dAu[h];
        if (lane < CQ) {
          qlimb[(4 * h) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0040), prmt(x[2], x[3], 0x0040), 0x5410) ^ 0x80808080u;
          qlimb[(4 * h + 1) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0051), prmt(x[2], x[3], 0x0051), 0x5410) ^ 0x80808080u;
          qlimb[(4 * h + 2) * CQ + lane] = prmt(prmt(x[0], x[1], 0x0062), prmt(x[2], x[3], 0x0062), 0x5410) ^ 0x80808080u;
        }
      }
      __syncwarp();
      // Exactness needs |4^k b2| + |C| < 2^31, i.e. |b2| < 2^24 (zero points up to
      // ~1000 in magnitude).  A page beyond that (a near-constant channel with a
      // large offset: tiny range, huge zero point) takes the plain fp32 path:
      // logit_t = alpha_k sum_c q~_c s_c (code_tc - z_c), each (code - z) exact.
      bool slow = lp.exact_logits != 0 || __any_sync(0xffffffffu, sat);
#pragma unroll
      for (int h = 0; h < NH; ++h) slow |= bA[h][2] >= (1 << 24) || bA[h][2] <= -(1 << 24);
      if (slow) {
        const float *ksf = reinterpret_cast<const float *>(B + c.pg_kscale);
        const int32_t *kzf = reinterpret_cast<const int32_t *>(B + c.pg_kzero);
        const uint8_t *kcb = B + c.pg_kcodes;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int ch = 0; ch < D; ++ch) {
            const float qs = qh[h * D + ch] * ksf[ch];
            const float z = (float)kzf[ch];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              acc[k] = fmaf(qs, (float)kcode_at(kcb, 4 * ktq + k, ch, G) - z, acc[k]);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) lg[h][k] = ((sbits >> k) & 1u) ? -INFINITY : alpha_k * acc[k];
        }
      } else {
      // logits by warp MMA: rows = tokens (row grp: token 4 tq + k0, grp + 8:
      // 4 tq + k1, tq = 8 blk + grp), K = 32 channels per chunk, columns = Q limbs
      // (4 h + k).  The masked code word (code << 2k per byte) is the A fragment
      // of 4 channels of one token; rows carry the 4^k factor.  The accumulators
      // start at -4^k B_limb, so each limb column ends as the exact integer
      // 4^k (C_limb - B_limb); the limbs combine in fp32 (even lanes: limb 0 +
      // 256 limb 1, odd lanes: limb 2, x 65536 in the reader).
      constexpr int KC = D / 32;
      uint32_t bq[KC][2];
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) {
        const uint2 b = *reinterpret_cast<const uint2 *>(qlimb + mcol * CQ + 8 * cc + 2 * mt);
        bq[cc][0] = b.x;
        bq[cc][1] = b.y;
      }
      const int hsel = min(rhead, NH - 1);
      int ba = bA[0][0], bb = bA[0][1], b2 = bA[0][2];
#pragma unroll
      for (int h = 1; h < NH; ++h)
        if (hsel == h) { ba = bA[h][0]; bb = bA[h][1]; b2 = bA[h][2]; }
      if (rodd) { ba = b2; bb = 0; }
      const int wBi = rodd ? 0 : 256;
      float *lgw = lgs + ((rodd ? NH + 1 : 0) + min(rhead, NH)) * S::LP;
      const uint32_t *kcw = reinterpret_cast<const uint32_t *>(B + c.pg_kcodes);
      AKVQ_UNROLL(AKVQ_KU)
      for (int blk = 0; blk < TQ / 8; ++blk) {
        const int tq = 8 * blk + mg;
        int c01[4] = {-ba, -bb, -4 * ba, -4 * bb}, c23[4] = {-16 * ba, -16 * bb, -64 * ba, -64 * bb};
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) {
          const uint2 w = *reinterpret_cast<const uint2 *>(kcw + kword_idx(8 * cc + 2 * mt, tq, TQ));
          mma_u8s8(c01, fmask(w.x, 0), fmask(w.x, 1), fmask(w.y, 0), fmask(w.y, 1), bq[cc][0], bq[cc][1]);
          mma_u8s8(c23, fmask(w.x, 2), fmask(w.x, 3), fmask(w.y, 2), fmask(w.y, 3), bq[cc][0], bq[cc][1]);
        }
        // limb 0 + 256 limb 1 combined in int32 (|sum| < 2^30), one rounding like fmaf
        reinterpret_cast<float4 *>(lgw)[tq] =
              make_float4((float)(c01[0] + wBi * c01[1]), (float)(c01[2] + wBi * c01[3]),
                          (float)(c23[0] + wBi * c23[1]), (float)(c23[2] + wBi * c23[3]));
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float4 e = reinterpret_cast<const float4 *>(lgs + h * S::LP)[ktq];
        const float4 o = reinterpret_cast<const float4 *>(lgs + (NH + 1 + h) * S::LP)[ktq];
        const float d0 = dA[h], d1 = dA[h] * 0.25f, d2 = dA[h] * 0.0625f, d3 = dA[h] * 0.015625f;
        lg[h][0] = (sbits & 1u) ? -INFINITY : fmaf(65536.f * d0, o.x, d0 * e.x);
        lg[h][1] = (sbits & 2u) ? -INFINITY : fmaf(65536.f * d1, o.y, d1 * e.y);
        lg[h][2] = (sbits & 4u) ? -INFINITY : fmaf(65536.f * d2, o.z, d2 * e.z);
        lg[h][3] = (sbits & 8u) ? -INFINITY : fmaf(65536.f * d3, o.w, d3 * e.w);
      }
      }   // MMA path
      }   // per-channel K
    } else if (s.kind == 1) {
      // ================= page V half: softmax update, value accumulation
      mbar_wait(bar_s + 8u * st, par);
      const float *vs = reinterpret_cast<const float *>(B);
      const int32_t *vz = reinterpret_cast<const int32_t *>(B + (c.pg_vzero - c.pg_vscale));
      const uint4 *vc4 = reinterpret_cast<const uint4 *>(B + (c.pg_vcodes - c.pg_vscale));
      float dwv[NH][NG];
      bool live[NH];
      // the lane's 4 tokens' V scales / zero points (shared by the heads)
      float vsv[NG][4], vzv[NG][4];
      if constexpr (NG == 1) {
        const float4 a = reinterpret_cast<const float4 *>(vs)[ktq];
        const int4 b = reinterpret_cast<const int4 *>(vz)[ktq];
        vsv[0][0] = a.x; vsv[0][1] = a.y; vsv[0][2] = a.z; vsv[0][3] = a.w;
        vzv[0][0] = (float)b.x; vzv[0][1] = (float)b.y; vzv[0][2] = (float)b.z; vzv[0][3] = (float)b.w;
      } else {
#pragma unroll
        for (int gi = 0; gi < NG; ++gi)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            vsv[gi][k] = vs[(4 * ktq + k) * NG + gi];
            vzv[gi][k] = (float)vz[(4 * ktq + k) * NG + gi];
          }
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float mloc = warp_max_fast(fmaxf(fmaxf(lg[h][0], lg[h][1]), fmaxf(lg[h][2], lg[h][3])));
        const float m_new = fmaxf(m_run[h], mloc);
        live[h] = m_new != -INFINITY;                 // warp-uniform
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) dwv[h][gi] = 0.f;
        if (!live[h]) continue;
        const float sc = ex2(m_run[h] - m_new);
        m_run[h] = m_new;
#pragma unroll
        for (int k = 0; k < 4; ++k) { o_rot[h][k] *= sc; o_org[h][k] *= sc; }
        float pr[4], psum = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) { pr[k] = ex2(lg[h][k] - m_new); psum += pr[k]; }
        l_run[h] = fmaf(l_run[h], sc, kcs == 0 ? psum : 0.f);   // lane partial
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) {
          // W_t = rn(p_t s^V_t winv): |W| <= kQMax (p <= 1, |s^V| <= umax.V); signed
          // 24-bit fixed point (degenerate groups may store a negative scale, R8);
          // the zero-point term uses the same rounded weights
          uint32_t W[4];
          float zs = 0.f;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int wi = __float2int_rn(pr[k] * vsv[gi][k] * winv);
            W[k] = (uint32_t)wi + kQOff;
            zs = fmaf((float)wi, vzv[gi][k], zs);
          }
          dwv[h][gi] = dwu;
          zl[h][gi] = fmaf(zl[h][gi], sc, kcs == 0 ? dwu * zs : 0.f);   // lane partial
          if (kcs == 0) {
            uint32_t *wl = wlimb + (gi * kLimbCols * NH + kLimbCols * h) * TQ + ktq;
            wl[0] = prmt(prmt(W[0], W[1], 0x0040), prmt(W[2], W[3], 0x0040), 0x5410) ^ 0x80808080u;
            wl[TQ] = prmt(prmt(W[0], W[1], 0x0051), prmt(W[2], W[3], 0x0051), 0x5410) ^ 0x80808080u;
            wl[2 * TQ] = prmt(prmt(W[0], W[1], 0x0062), prmt(W[2], W[3], 0x0062), 0x5410) ^ 0x80808080u;
          }
        }
      }
      __syncwarp();
      // sum_t W_t code_tc by warp MMA: rows = channels (row grp: 4 cq + k0, grp + 8:
      // 4 cq + k1, cq = 8 cb + grp), K = 32 tokens per chunk, columns = W limbs
      // (2 h, 2 h + 1) of the chunk's channel group.  Integer sums go through
      // smem to the lane layout of o_rot (lane vcq: channels 4 vcq ..).
      constexpr int TC = G / 32;
      const uint32_t *vcw = reinterpret_cast<const uint32_t *>(vc4);
      const int wBv = rodd ? 0 : 256;
      float *lvw = lgs + ((rodd ? NH + 1 : 0) + min(rhead, NH)) * S::LP;
      AKVQ_UNROLL(AKVQ_VU)
      for (int cb = 0; cb < D / 32; ++cb) {
        const int cq = 8 * cb + mg, gi = (32 * cb) / G;
        int c01[4] = {0, 0, 0, 0}, c23[4] = {0, 0, 0, 0};
#pragma unroll
        for (int cc = 0; cc < TC; ++cc) {
          const uint2 b = *reinterpret_cast<const uint2 *>(wlimb + (gi * kLimbCols * NH + mcol) * TQ + 8 * cc + 2 * mt);
          const uint2 w = *reinterpret_cast<const uint2 *>(vcw + vword_idx(cq, 8 * cc + 2 * mt, CQ));
          mma_u8s8(c01, fmask(w.x, 0), fmask(w.x, 1), fmask(w.y, 0), fmask(w.y, 1), b.x, b.y);
          mma_u8s8(c23, fmask(w.x, 2), fmask(w.x, 3), fmask(w.y, 2), fmask(w.y, 3), b.x, b.y);
        }
        // per limb column: <= G tokens x 192 x 255 < 2^31 (exact); even lanes
        // store limb 0 + 256 limb 1, odd lanes limb 2 (x 65536 in the reader)
        reinterpret_cast<float4 *>(lvw)[cq] =
              make_float4((float)(c01[0] + wBv * c01[1]), (float)(c01[2] + wBv * c01[3]),
                          (float)(c23[0] + wBv * c23[1]), (float)(c23[2] + wBv * c23[3]));
      }
      __syncwarp();
      if (vts == 0) {
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          if (!live[h]) continue;
          float dw = dwv[h][0];
#pragma unroll
          for (int gi = 1; gi < NG; ++gi) if (gi == vgam) dw = dwv[h][gi];
          const float4 e = reinterpret_cast<const float4 *>(lgs + h * S::LP)[vcq];
          const float4 o = reinterpret_cast<const float4 *>(lgs + (NH + 1 + h) * S::LP)[vcq];
          // channel 4 vcq + k carried the factor 4^k; zero term: zl, subtracted at flush
          o_rot[h][0] = fmaf(dw, fmaf(65536.f, o.x, e.x), o_rot[h][0]);
          o_rot[h][1] = fmaf(dw * 0.25f, fmaf(65536.f, o.y, e.y), o_rot[h][1]);
          o_rot[h][2] = fmaf(dw * 0.0625f, fmaf(65536.f, o.z, e.z), o_rot[h][2]);
          o_rot[h][3] = fmaf(dw * 0.015625f, fmaf(65536.f, o.w, e.w), o_rot[h][3]);
        }
      }
    } else if (s.kind == 4) {
      mbar_wait(bar_s + 8u * st, par);                       // empty unit marker (no data)
    } else {
      // ================= rows: 16-bit (ring / PSA side, original basis) or
      //                   4-bit (TSA side, rotated basis), in groups of kRows
      mbar_wait(bar_s + 8u * st, par);
      const bool r16 = s.kind == 2;
      if (s.ring && app_k != nullptr) {
        // the newest token (Eq. 2): the stale ring slot was staged -- patch in
        // the caller's row, append it to the ring and set its TSA text bit
        const int tl = Lc - 1 - (lp.n_q + s.a);
        if (tl >= 0 && tl < s.n) {
          const int uu = cur_pu;                     // (every head group appends: benign, identical)
          const uint4 *sk = reinterpret_cast<const uint4 *>(app_k + (size_t)uu * D);
          const uint4 *sv = reinterpret_cast<const uint4 *>(app_v + (size_t)uu * D);
          uint8_t *Bw = B + (size_t)tl * 4 * D;
          uint4 *rrow = reinterpret_cast<uint4 *>(ring_row(c, uu, (Lc - 1) % c.slots));
          for (int i = lane; i < D / 8; i += 32) {
            const uint4 kv = sk[i], vv = sv[i];
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
      const uint32_t pitch = r16 ? 4u * D : (uint32_t)c.side_entry;
      const uint32_t sbase = smem_u32(B);
      // ring chunks planned for the whole flush period hold rows past L (DEVICE_L)
      const int nrows = s.ring ? min(s.n, Lc - lp.n_q - s.a) : s.n;
      for (int g0 = 0; g0 < nrows; g0 += kRows) {
        const int n = min(kRows, nrows - g0);
        const uint32_t sb0 = sbase + (uint32_t)g0 * pitch;
        if (n < kRows) {   // zero-fill the group's missing rows (finite, masked below)
          uint4 *z = reinterpret_cast<uint4 *>(B + (size_t)(g0 + n) * pitch);
          for (int i = lane; i < (int)((kRows - n) * pitch / 16); i += 32) z[i] = make_uint4(0, 0, 0, 0);
          __syncwarp();
        }
        if (!tsa || r16) rows_group(sb0, pitch, n, std::integral_constant<bool, true>());
        else if constexpr (tsa) rows_group(sb0, pitch, n, std::integral_constant<bool, false>());
      }
    }
    __syncwarp();                                   // every lane is done with stage st
    rf = st;                                        // refill it at the loop top
    nrf = 1;
    if (++st == kLyStages) { st = 0; par ^= 1u; }
  }
  if constexpr (DL) ly_exit(c, lp, lane, &cta_done);
}

template <int D, int G, int NH>
static size_t ly_smem(const DevCache &c) {
  return (size_t)kLyWarps * LySmem<D, G, NH>::warp_bytes(ly_stage_bytes(c));
}

template <int D, int G, int DT, int NH>
static cudaError_t launch_ly(const DevCache &c, const LayerPlan &lp, const void *q, const void *k,
                             const void *v, const uint8_t *types, float *part, float *out,
                             uint32_t flags, cudaStream_t st) {
  const size_t smem = ly_smem<D, G, NH>(c);
  const int km = c.k_axis == AKVQ_K_PER_TOKEN ? 1 : 0;
  auto kern = lp.dev_L
      ? (c.kind == AKVQ_TSA ? (km ? k_decode_layer<D, G, DT, NH, true, 1, true> : k_decode_layer<D, G, DT, NH, true, 0, true>)
                            : (km ? k_decode_layer<D, G, DT, NH, false, 1, true> : k_decode_layer<D, G, DT, NH, false, 0, true>))
      : (c.kind == AKVQ_TSA ? (km ? k_decode_layer<D, G, DT, NH, true, 1, false> : k_decode_layer<D, G, DT, NH, true, 0, false>)
                            : (km ? k_decode_layer<D, G, DT, NH, false, 1, false> : k_decode_layer<D, G, DT, NH, false, 0, false>));
  if (lp.stream_only) {                      // profiling variant: single-head MHA caches only
    if constexpr (NH == 1)
      kern = c.kind == AKVQ_TSA ? k_decode_layer<D, G, DT, NH, true, 2, false> : k_decode_layer<D, G, DT, NH, false, 2, false>;
    else
      return cudaErrorNotSupported;
  }
  {
    const cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((lp.W + kLyWarps - 1) / kLyWarps));
  cfg.blockDim = dim3(kLyWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap the previous tail
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c, lp, (const uint16_t *)q, (const uint16_t *)k,
                            (const uint16_t *)v, types, part, out, flags);
}

int layer_supported(int d, int G, int g) {
  return (d == 128 || d == 64) && G >= 32 && G <= d && g >= 1 && g <= 16;
}
// query heads per pass over a unit's cache: g itself for g <= 2 (k_decode_layer),
// else the single-pass GQA kernel's group of 4 or 8 (k_decode_gqa; g > 8 runs
// ceil(g / 8) groups)
int layer_uses_gqa(int g) { return g >= 3; }
int layer_group_heads(int g) { return g <= 2 ? g : gqa_heads(g); }
int layer_head_groups(int g) { return (g + layer_group_heads(g) - 1) / layer_group_heads(g); }
int layer_warps_per_cta() { return kLyWarps; }
int layer_ctas_per_sm(int nh) { return ly_ctas_per_sm(nh); }
int layer_rows_per_chunk() { return kRows; }
int layer_rows4_per_sub() { return kRows4; }

template <int D, int G, int DT>
static cudaError_t launch_ly_g(const DevCache &c, const LayerPlan &lp, const void *q, const void *k,
                               const void *v, const uint8_t *types, float *part, float *out,
                               uint32_t flags, cudaStream_t st) {
  const int nh = layer_group_heads(c.g);      // lp.hg = ceil(g / nh) groups per kv head
  if (nh == 1) return launch_ly<D, G, DT, 1>(c, lp, q, k, v, types, part, out, flags, st);
  if (nh == 2) return launch_ly<D, G, DT, 2>(c, lp, q, k, v, types, part, out, flags, st);
  return cudaErrorInvalidValue;               // 4 limb columns per head: <= 2 heads per n-tile
}

cudaError_t launch_decode_layer(const DevCache &c, int dtype16, const LayerPlan &lp, const void *q,
                                const void *k, const void *v, const uint8_t *types, float *part,
                                float *out, uint32_t flags, cudaStream_t st) {
  if (lp.T <= 0) return cudaSuccess;
#define AKVQ_LCASE(D_, G_)                                                                       \
  if (c.d == D_ && c.G == G_)                                                                    \
    return dtype16 == AKVQ_BF16                                                                  \
               ? launch_ly_g<D_, G_, AKVQ_BF16>(c, lp, q, k, v, types, part, out, flags, st)    \
               : launch_ly_g<D_, G_, AKVQ_FP16>(c, lp, q, k, v, types, part, out, flags, st);
  AKVQ_LCASE(64, 32)
  AKVQ_LCASE(64, 64)
  AKVQ_LCASE(128, 32)
  AKVQ_LCASE(128, 64)
  AKVQ_LCASE(128, 128)
#undef AKVQ_LCASE
  return cudaErrorInvalidValue;
}

}  // namespace akvq
