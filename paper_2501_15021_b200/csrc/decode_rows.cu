// decode_rows.cu -- decode attention over the non-2-bit rows of the AKVQ-VL
// cache on sm_100a: the 16-bit recent window (ring) and PSA pivots
// (side16), both in the ORIGINAL basis (R10), and TSA text rows
// (side4, 4-bit per token, rotated basis, R11).
//
// Persistent warps stream the flattened per-unit item list
//   [ring chunks of 16 tokens][side splits]
// with per-warp double-buffered 1-D TMA bulk copies (a ring chunk is 16
// contiguous slots, split in two copies where the ring wraps).  Each (warp,
// unit) segment keeps one online softmax with two accumulators: o_org (16-bit
// rows, original basis) and o_rot (4-bit rows, rotated basis), written as one
// partial for k_combine.
#include <math.h>

#include "decode_common.cuh"

namespace akvq {

constexpr int kRwWarps = 4;
constexpr int kRwStages = 2;
constexpr int kChunk = 16;             // tokens / side entries per item

template <int DT>
__device__ __forceinline__ void cvt2(uint32_t w, float &a, float &b) {
  if constexpr (DT == AKVQ_BF16) {
    a = __uint_as_float(w << 16);
    b = __uint_as_float(w & 0xffff0000u);
  } else {
    const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w));
    a = f.x;
    b = f.y;
  }
}

// Per-warp smem: stages (kChunk rows of 4d bytes), q (original, scaled) and
// q~ (rotated, unnormalized) per head, barriers.
template <int D, int NH>
struct RwSmem {
  static constexpr size_t stage = (size_t)kChunk * 4 * D;
  static constexpr size_t qo_off = kRwStages * stage;
  static constexpr size_t qh_off = qo_off + (size_t)NH * D * 4;
  static constexpr size_t bar_off = qh_off + (size_t)NH * D * 4;
  static constexpr size_t warp_bytes = (bar_off + kRwStages * 8 + 127) / 128 * 128;
};

template <int D, int G, int DT, int NH>
__global__ void __launch_bounds__(kRwWarps * 32)
    k_decode_rows(DevCache c, RowPlan rp, PagePlan pp, const uint16_t *__restrict__ q,
                  const uint16_t *__restrict__ app_k, const uint16_t *__restrict__ app_v,
                  const uint8_t *__restrict__ app_types, float *__restrict__ rw_part,
                  const float *__restrict__ pg_part, float *__restrict__ out, uint32_t flags) {
  using S = RwSmem<D, NH>;
  constexpr int NG = D / G;
  constexpr int KPR = D / 16;          // V phase: lanes per row (16 channels each)
  constexpr int NTG = 32 / KPR;        // V phase: token sub-groups
  constexpr int KHL = D / 2;           // K phase: channels per lane (2 lanes / row)
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t *wsm = smem + (size_t)warp * S::warp_bytes;
  float *qo = reinterpret_cast<float *>(wsm + S::qo_off);
  float *qh = reinterpret_cast<float *>(wsm + S::qh_off);
  uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + S::bar_off);

  pdl_wait();                     // q / k / v come from the preceding kernels
  pdl_launch_dependents();        // the page kernel may start filling idle SMs
  const int gw = blockIdx.x * kRwWarps + warp;
  if (gw >= (int)rp.W) return;
  const int ib = seg_begin((int)rp.T, (int)rp.W, gw), ie = seg_begin((int)rp.T, (int)rp.W, gw + 1);
  if (ib >= ie) return;
  const int per_u = rp.items_per_unit;
  const bool tsa = c.kind == AKVQ_TSA;
  const int n_ring = rp.L - rp.n_q;
  const float alpha_o = kLog2e * c.inv_sqrt_d;   // q.k / sqrt d in log2 units
  const float alpha_q = kLog2e / (float)D;       // (q.H_s).K^ / d

  if (lane == 0) {
    for (int s = 0; s < kRwStages; ++s) mbar_init(&bar[s]);
    mbar_fence_init();
  }
  __syncwarp();

  // item -> (unit, kind, first row, rows); side items are split by the device count
  struct Item { int u, kind, r0, n; };   // kind 0 ring, 1 side
  auto decode_item = [&](int it) {
    Item x;
    x.u = it / per_u;
    const int k = it - x.u * per_u;
    if (k < rp.n_ring_chunks) {
      x.kind = 0;
      x.r0 = k * kChunk;
      x.n = min(kChunk, n_ring - x.r0);
    } else {
      const int r = k - rp.n_ring_chunks;
      const int cnt = c.side_cnt[x.u];
      const int a = r * cnt / rp.n_side_splits;
      const int b = (r + 1) * cnt / rp.n_side_splits;
      x.kind = 1;
      x.r0 = a;
      x.n = b - a;
    }
    return x;
  };
  // A side split can exceed one chunk: it is processed as consecutive sub-chunks.
  // `issue` loads sub-chunk `sub` of item x into stage st.
  auto issue = [&](const Item &x, int sub, int st) {
    uint8_t *dst = wsm + (size_t)st * S::stage;
    const int r0 = x.r0 + sub * kChunk;
    const int n = min(kChunk, x.r0 + x.n - r0);
    if (n <= 0) return;
    if (x.kind == 0) {
      const int t0 = rp.n_q + r0;
      const int s0 = t0 % c.slots;
      const int n1 = min(n, c.slots - s0);
      const uint32_t rowb = 4 * D;
      mbar_expect_tx(&bar[st], (uint32_t)n * rowb);
      bulk_g2s(dst, ring_row(c, x.u, s0), (uint32_t)n1 * rowb, &bar[st]);
      if (n1 < n) bulk_g2s(dst + (size_t)n1 * rowb, ring_row(c, x.u, 0), (uint32_t)(n - n1) * rowb, &bar[st]);
    } else {
      const uint32_t eb = c.side_entry;
      mbar_expect_tx(&bar[st], (uint32_t)n * eb);
      bulk_g2s(dst, side_ptr(c, x.u, r0), (uint32_t)n * eb, &bar[st]);
    }
  };

  // flattened (item, sub-chunk) stream for the pipeline
  int it_cur = ib;
  int sub_cur = 0;
  Item x_cur = decode_item(ib);
  int it_nx = ib;           // producer cursor (lane 0 only uses it)
  int sub_nx = 0;
  Item x_nx = x_cur;
  auto advance = [&](int &it, int &sub, Item &x) {
    ++sub;
    if (sub * kChunk >= x.n) {
      sub = 0;
      ++it;
      if (it < ie) x = decode_item(it);
    }
  };
  // skip empty items at the producer start
  auto skip_empty = [&](int &it, int &sub, Item &x) {
    while (it < ie && x.n <= 0) {
      ++it;
      sub = 0;
      if (it < ie) x = decode_item(it);
    }
  };
  skip_empty(it_nx, sub_nx, x_nx);
  int n_issued = 0;
  if (lane == 0) {
    for (int s = 0; s < kRwStages && it_nx < ie; ++s) {
      issue(x_nx, sub_nx, s);
      ++n_issued;
      advance(it_nx, sub_nx, x_nx);
      skip_empty(it_nx, sub_nx, x_nx);
    }
  }
  n_issued = __shfl_sync(0xffffffffu, n_issued, 0);

  float m_run[NH], l_run[NH], o_org[NH][16], o_rot[NH][16], Zr[NH][NG];
  int cur_u = -1;
  const int u_first = ib / per_u;
  const int tq = lane >> 1, half = lane & 1;
  const int kw = lane % KPR, tg = lane / KPR;
  const int gam = (16 * kw) / G;

  auto flush = [&](int u) {
    const size_t slot = (size_t)gw * rp.maxseg + (u - u_first);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      float zg = Zr[h][0];
#pragma unroll
      for (int gi = 1; gi < NG; ++gi) if (gi == gam) zg = Zr[h][gi];
#pragma unroll
      for (int off = KPR; off < 32; off <<= 1) zg += __shfl_xor_sync(0xffffffffu, zg, off);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a = o_org[h][k], b = o_rot[h][k];
#pragma unroll
        for (int off = KPR; off < 32; off <<= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, off);
          b += __shfl_xor_sync(0xffffffffu, b, off);
        }
        o_org[h][k] = a;
        o_rot[h][k] = b - zg;
      }
      float *rec = rw_part + (slot * NH + h) * Rec<D>::R;
      if (tg == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          reinterpret_cast<float4 *>(rec + 16 * kw)[k] =
              make_float4(o_org[h][4 * k], o_org[h][4 * k + 1], o_org[h][4 * k + 2], o_org[h][4 * k + 3]);
          reinterpret_cast<float4 *>(rec + D + 16 * kw)[k] =
              make_float4(o_rot[h][4 * k], o_rot[h][4 * k + 1], o_rot[h][4 * k + 2], o_rot[h][4 * k + 3]);
        }
      }
      if (lane == 0) { rec[2 * D] = m_run[h]; rec[2 * D + 1] = l_run[h]; }
    }
    // without quantized pages nothing follows this kernel: merge here
    if (pp.T <= 0) {
      int w_lo, w_hi;
      seg_range((int)rp.T, (int)rp.W, rp.items_per_unit, u, w_lo, w_hi);
      if (take_ticket(c, u, (int)(w_hi - w_lo + 1), lane)) {
        merge_unit<D, NH>(c, pp, rp, pg_part, rw_part, u, out, flags, lane);
        if (lane == 0) c.ticket[u] = 0u;
      }
    }
  };

  skip_empty(it_cur, sub_cur, x_cur);
  for (int ci = 0; it_cur < ie; ++ci) {
    const int st = ci % kRwStages;
    const uint32_t par = (uint32_t)((ci / kRwStages) & 1);
    const Item x = x_cur;
    const int r0 = x.r0 + sub_cur * kChunk;
    const int n = min(kChunk, x.r0 + x.n - r0);
    if (x.u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      cur_u = x.u;
      for (int i = lane; i < NH * D; i += 32) {
        const float v = H16<DT>::to_f(q[(size_t)x.u * c.g * D + i]);
        qo[i] = v;                       // logits scaled by alpha_o after the dot
        qh[i] = v;
      }
      __syncwarp();
      if (tsa) {
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
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        m_run[h] = -INFINITY; l_run[h] = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) { o_org[h][k] = 0.f; o_rot[h][k] = 0.f; }
#pragma unroll
        for (int gi = 0; gi < NG; ++gi) Zr[h][gi] = 0.f;
      }
    }
    mbar_wait(&bar[st], par);
    if (rp.stream_only) {                             // profiling: pipeline only
      __syncwarp();
      if (lane == 0 && n_issued > 0 && it_nx < ie) {
        issue(x_nx, sub_nx, st);
        advance(it_nx, sub_nx, x_nx);
        skip_empty(it_nx, sub_nx, x_nx);
      }
      advance(it_cur, sub_cur, x_cur);
      skip_empty(it_cur, sub_cur, x_cur);
      continue;
    }
    const uint8_t *B = wsm + (size_t)st * S::stage;
    const bool rows16 = x.kind == 0 || !tsa;
    // the newest token (Eq. 2): attend to the caller's row -- the stale ring
    // slot was loaded -- and append it to the ring (and the TSA text bit)
    if (app_k != nullptr && x.kind == 0) {
      const int tl = rp.L - 1 - (rp.n_q + r0);
      if (tl >= 0 && tl < n) {
        const uint4 *sk = reinterpret_cast<const uint4 *>(app_k + (size_t)x.u * D);
        const uint4 *sv = reinterpret_cast<const uint4 *>(app_v + (size_t)x.u * D);
        uint8_t *Bw = wsm + (size_t)st * S::stage + (size_t)tl * 4 * D;
        uint4 *rr = reinterpret_cast<uint4 *>(ring_row(c, x.u, (rp.L - 1) % c.slots));
        for (int i = lane; i < D / 8; i += 32) {
          const uint4 kv = sk[i], vv = sv[i];
          reinterpret_cast<uint4 *>(Bw)[i] = kv;
          reinterpret_cast<uint4 *>(Bw + 2 * D)[i] = vv;
          rr[i] = kv;
          rr[D / 8 + i] = vv;
        }
        if (lane == 0 && tsa && app_types != nullptr && app_types[x.u] == 1)
          atomicOr(&c.bitmask[(size_t)x.u * c.bm_words + (rp.L - 1) / 32], 1u << ((rp.L - 1) % 32));
        __syncwarp();
      }
    }
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      // ---------------- K: logit of row tq (2 lanes per row, D/2 channels each)
      float dot = 0.f;
      if (tq < n) {
        if (rows16) {
          const uint4 *kr = reinterpret_cast<const uint4 *>(B + (size_t)tq * 4 * D + half * D);
          const float *qq = qo + h * D + half * KHL;
#pragma unroll
          for (int i = 0; i < KHL / 8; ++i) {
            const uint4 v = kr[i];
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float a, b;
              cvt2<DT>(wv[j], a, b);
              dot = fmaf(qq[8 * i + 2 * j], a, dot);
              dot = fmaf(qq[8 * i + 2 * j + 1], b, dot);
            }
          }
        } else {   // TSA 4-bit row: sum_g s_g (sum q~ code - z_g sum q~), rotated basis
          constexpr int NGL = KHL >= G ? KHL / G : 1;     // groups inside this lane's half
          const uint8_t *se = B + (size_t)tq * c.side_entry;
          const float *ks = reinterpret_cast<const float *>(se);
          const int32_t *kz = reinterpret_cast<const int32_t *>(se + 4 * NG);
          const uint32_t *cw = reinterpret_cast<const uint32_t *>(se + 16 * NG + half * (KHL / 2));
          const float *qq = qh + h * D + half * KHL;
          const int gbase = (half * KHL) / G;
          float A[NGL], Bs[NGL];
#pragma unroll
          for (int gl = 0; gl < NGL; ++gl) { A[gl] = 0.f; Bs[gl] = 0.f; }
#pragma unroll
          for (int w = 0; w < KHL / 8; ++w) {
            const uint32_t word = cw[w];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int gl = (8 * w + i) / G;
              A[gl] = fmaf(qq[8 * w + i], (float)((word >> (4 * i)) & 15u), A[gl]);
              Bs[gl] += qq[8 * w + i];
            }
          }
#pragma unroll
          for (int gl = 0; gl < NGL; ++gl)
            dot += ks[gbase + gl] * (A[gl] - (float)kz[gbase + gl] * Bs[gl]);
          dot *= alpha_q / alpha_o;                 // rescaled by alpha_o below
        }
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      const float lg = tq < n ? dot * alpha_o : -INFINITY;
      // ---------------- online softmax over the n rows
      float mx = lg;
#pragma unroll
      for (int off = 2; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_run[h], mx);
      if (m_new == -INFINITY) continue;
      const float sc = exp2f(m_run[h] - m_new);
      const float p = exp2f(lg - m_new);
      float ps = half == 0 ? p : 0.f;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
      l_run[h] = l_run[h] * sc + ps;
      m_run[h] = m_new;
#pragma unroll
      for (int k = 0; k < 16; ++k) { o_org[h][k] *= sc; o_rot[h][k] *= sc; }
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) Zr[h][gi] *= sc;
      // ---------------- V: lane (kw, tg) accumulates 16 channels over rows tg, tg+NTG, ...
#pragma unroll
      for (int r = 0; r < kChunk / NTG; ++r) {
        const int row = tg + NTG * r;
        const float pr = __shfl_sync(0xffffffffu, p, 2 * row);   // lane 2*row holds row's p
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
              cvt2<DT>(wv[j], a, b);
              o_org[h][8 * i + 2 * j] = fmaf(pr, a, o_org[h][8 * i + 2 * j]);
              o_org[h][8 * i + 2 * j + 1] = fmaf(pr, b, o_org[h][8 * i + 2 * j + 1]);
            }
          }
        } else {
          const uint8_t *se = B + (size_t)row * c.side_entry;
          float sv = reinterpret_cast<const float *>(se + 8 * NG)[0];
          float zv = (float)reinterpret_cast<const int32_t *>(se + 12 * NG)[0];
#pragma unroll
          for (int gi = 1; gi < NG; ++gi)
            if (gi == gam) {
              sv = reinterpret_cast<const float *>(se + 8 * NG)[gi];
              zv = (float)reinterpret_cast<const int32_t *>(se + 12 * NG)[gi];
            }
          const float w = pr * sv;
          const uint2 cv = *reinterpret_cast<const uint2 *>(se + 16 * NG + D / 2 + 8 * kw);
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const uint32_t word = k < 8 ? cv.x : cv.y;
            o_rot[h][k] = fmaf(w, (float)((word >> (4 * (k & 7))) & 15u), o_rot[h][k]);
          }
          // zero-point term once per row and group (lanes with tg == 0 keep it)
#pragma unroll
          for (int gi = 0; gi < NG; ++gi) if (gi == gam) Zr[h][gi] = fmaf(w, zv, Zr[h][gi]);
        }
      }
    }
    __syncwarp();
    // next sub-chunk / item
    if (lane == 0 && n_issued > 0) {
      if (it_nx < ie) {
        issue(x_nx, sub_nx, st);
        advance(it_nx, sub_nx, x_nx);
        skip_empty(it_nx, sub_nx, x_nx);
      }
    }
    advance(it_cur, sub_cur, x_cur);
    skip_empty(it_cur, sub_cur, x_cur);
  }
  if (cur_u >= 0 && !rp.stream_only) flush(cur_u);
}

template <int D, int NH>
static size_t rw_smem() { return (size_t)kRwWarps * RwSmem<D, NH>::warp_bytes; }

template <int D, int G, int DT, int NH>
static cudaError_t launch_rw(const DevCache &c, const RowPlan &rp, const PagePlan &pp, const void *q,
                             const void *k, const void *v, const uint8_t *types, float *rw_part,
                             const float *pg_part, float *out, uint32_t flags, cudaStream_t st) {
  const size_t smem = rw_smem<D, NH>();
  auto kern = k_decode_rows<D, G, DT, NH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int ctas = (int)((rp.W + kRwWarps - 1) / kRwWarps);
  kern<<<ctas, kRwWarps * 32, smem, st>>>(c, rp, pp, (const uint16_t *)q, (const uint16_t *)k,
                                          (const uint16_t *)v, types, rw_part, pg_part, out, flags);
  return cudaGetLastError();
}

template <int D, int G, int DT>
static cudaError_t launch_rw_g(const DevCache &c, const RowPlan &rp, const PagePlan &pp,
                               const void *q, const void *k, const void *v, const uint8_t *types,
                               float *rw_part, const float *pg_part, float *out, uint32_t flags,
                               cudaStream_t st) {
  if (c.g == 1) return launch_rw<D, G, DT, 1>(c, rp, pp, q, k, v, types, rw_part, pg_part, out, flags, st);
  if (c.g == 2) return launch_rw<D, G, DT, 2>(c, rp, pp, q, k, v, types, rw_part, pg_part, out, flags, st);
  return launch_rw<D, G, DT, 4>(c, rp, pp, q, k, v, types, rw_part, pg_part, out, flags, st);
}

int rows_chunk() { return kChunk; }
int rows_warps_per_cta() { return kRwWarps; }

cudaError_t launch_decode_rows(const DevCache &c, int dtype16, const RowPlan &rp, const PagePlan &pp,
                               const void *q, const void *k, const void *v, const uint8_t *types,
                               float *rw_part, const float *pg_part, float *out, uint32_t flags,
                               cudaStream_t st) {
  if (rp.T <= 0) return cudaSuccess;
#define AKVQ_RCASE(D_, G_)                                                                     \
  if (c.d == D_ && c.G == G_)                                                                  \
    return dtype16 == AKVQ_BF16                                                                \
               ? launch_rw_g<D_, G_, AKVQ_BF16>(c, rp, pp, q, k, v, types, rw_part, pg_part,  \
                                                out, flags, st)                                \
               : launch_rw_g<D_, G_, AKVQ_FP16>(c, rp, pp, q, k, v, types, rw_part, pg_part,  \
                                                out, flags, st);
  AKVQ_RCASE(64, 32)
  AKVQ_RCASE(64, 64)
  AKVQ_RCASE(128, 32)
  AKVQ_RCASE(128, 64)
  AKVQ_RCASE(128, 128)
#undef AKVQ_RCASE
  return cudaErrorInvalidValue;
}

}  // namespace akvq
