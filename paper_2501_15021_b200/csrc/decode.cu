// decode.cu -- single-query split-K decode attention straight from the packed
// AKVQ-VL cache (sm_100a), plus the split combine and the dequantized view.
//
//   logit_t = (q~ . K^_t) / sqrt(d)  with q~ = q.H            (Fig. 6)
//   o       = softmax(logit) . V^  then . H                    (Fig. 7, R4)
//
// 2-bit tokens (per-channel K, per-token V; Eqs. 3-4) are dequantized in
// registers; 16-bit ring / PSA-side rows are used in the original basis
// (q.k, sum p v; R10); TSA 4-bit side rows in the rotated basis.  Softmax is
// base-2 online softmax in fp32 per warp, merged per CTA, and merged across
// splits by k_combine (log-sum-exp), which also applies the output H.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace akvq {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;

enum SplitKind { kPage = 0, kRing = 1, kSide = 2 };

// Shared memory plan (floats): qh [g][D] (q.H_s), qo [g][D] (q * log2e/sqrt d),
// per warp: qs [g][D] (page-prescaled q), bias [g], lg [g][32] logits / probs,
// merge area [kWarps][g][D + 2].
template <int D>
struct Smem {
  static __host__ __device__ size_t floats(int g) {
    return (size_t)2 * g * D + (size_t)kWarps * (g * D + g + 32 * g) +
           (size_t)kWarps * g * (D + 2);
  }
};

template <int D, int G, int DT, int MAXG>
__global__ void __launch_bounds__(kThreads) k_decode_split(DevCache c, DecodePlan p,
                                                           const uint16_t *__restrict__ q,
                                                           float *__restrict__ ws_m,
                                                           float *__restrict__ ws_l,
                                                           float *__restrict__ ws_o) {
  constexpr int CL = D / 32;          // channels per lane in the V phase
  constexpr int NG = D / G;
  extern __shared__ float sm[];
  const int g = c.g;
  const int s = blockIdx.x, u = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float *qh = sm;
  float *qo = qh + g * D;
  float *wbase = qo + g * D + warp * (g * D + g + 32 * g);
  float *qs = wbase;
  float *bias = qs + g * D;
  float *lg = bias + g;
  float *mg = qo + g * D + kWarps * (g * D + g + 32 * g);   // merge area

  const float alpha_q = kLog2e / (float)D;                  // (q.H_s).K^ / d
  const float alpha_o = kLog2e * c.inv_sqrt_d;              // q.k / sqrt d

  // ---- q~ (unnormalized FWHT in smem) and scaled original q
  for (int i = tid; i < g * D; i += kThreads) {
    const float v = H16<DT>::to_f(q[(size_t)u * g * D + i]);
    qh[i] = v;
    qo[i] = v * alpha_o;
  }
  __syncthreads();
  for (int hs = 1; hs < D; hs <<= 1) {
    for (int idx = tid; idx < g * D / 2; idx += kThreads) {
      const int h = idx / (D / 2), k = idx % (D / 2);
      const int i = (k / hs) * 2 * hs + (k % hs);
      const float a = qh[h * D + i], b = qh[h * D + i + hs];
      qh[h * D + i] = a + b;
      qh[h * D + i + hs] = a - b;
    }
    __syncthreads();
  }

  // ---- split assignment
  int kind, n_items;            // items = 32-token chunks (pages/ring) or side chunks
  int item0 = 0;
  int side_n = 0, side0 = 0;
  if (s < p.n_page_splits) {
    kind = kPage;
    const int p0 = s * p.pages_per_split;
    const int p1 = min(p0 + p.pages_per_split, p.n_pages);
    item0 = p0 * (G / 32);
    n_items = (p1 - p0) * (G / 32);
    // exact R (R26): the last page is partial; chunks past n_q are skipped and
    // the tokens >= n_q of the last chunk are masked like salient ones
    n_items = min(n_items, (p.n_q + 31) / 32 - item0);
  } else if (s < p.n_page_splits + p.n_ring_splits) {
    kind = kRing;
    const int r = s - p.n_page_splits;
    item0 = p.n_q + r * p.ring_per_split;                  // first token
    const int t1 = min(item0 + p.ring_per_split, p.L);
    n_items = (t1 - item0 + 31) / 32;
  } else {
    kind = kSide;
    const int r = s - p.n_page_splits - p.n_ring_splits;
    const int cnt = c.side_cnt[u];            // device count; splits take equal shares
    side0 = (int)((long)r * cnt / p.n_side_splits);
    side_n = (int)((long)(r + 1) * cnt / p.n_side_splits) - side0;
    n_items = (side_n + 31) / 32;
  }

  float m[MAXG], l[MAXG], o[MAXG][CL];
#pragma unroll
  for (int h = 0; h < MAXG; ++h) {
    m[h] = -INFINITY; l[h] = 0.f;
#pragma unroll
    for (int k = 0; k < CL; ++k) o[h][k] = 0.f;
  }
  const int tq = lane >> 2, cq = lane & 3;   // K phase: 8 tokens x 4 channel quarters
  const uint32_t *bm = c.bitmask + (size_t)u * c.bm_words;

  for (int it = warp; it < n_items; it += kWarps) {
    float logit[MAXG];
    // ============ K phase: logits of up to 32 tokens, token i <-> lane i
    if (kind == kPage) {
      const int chunk = item0 + it;                        // global 32-token chunk
      const int pg = chunk / (G / 32);
      const int t0 = chunk * 32;                           // first token
      const uint8_t *P = page_ptr(c, u, pg);
      const float *ks = reinterpret_cast<const float *>(P + c.pg_kscale);
      const int32_t *kz = reinterpret_cast<const int32_t *>(P + c.pg_kzero);
      // per channel: prescale q~ by the page's K scale, bias = sum qs * zero;
      // per token (NEXT-1): q~ only, scale / zero applied per token below
      const bool kt = c.k_axis == AKVQ_K_PER_TOKEN;
      for (int h = 0; h < g; ++h) {
        float part = 0.f;
        for (int ch = lane; ch < D; ch += 32) {
          const float v = qh[h * D + ch] * (kt ? 1.f : ks[ch]) * alpha_q;
          qs[h * D + ch] = v;
          part += kt ? 0.f : v * (float)kz[ch];
        }
        part = warp_sum(part);
        if (lane == 0) bias[h] = part;
      }
      __syncwarp();
      const uint8_t *kc = P + c.pg_kcodes;
      const int tlb = t0 - pg * G;                         // first token in the page
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int ti = pass * 8 + tq;
        // the 4-token bytes of this token's channels (K tile layout, common.cuh)
        uint8_t by[D / 4];
#pragma unroll
        for (int k = 0; k < D / 4; ++k) {
          const int ch = cq * (D / 4) + k;
          by[k] = kc[4 * kword_idx(ch >> 2, (tlb + ti) >> 2, G / 4) + (ch & 3)];
        }
        const int sh = 2 * ((tlb + ti) & 3);
        for (int h = 0; h < g; ++h) {
          const float *qq = qs + h * D + cq * (D / 4);
          float dot = 0.f, qsum = 0.f;
#pragma unroll
          for (int k = 0; k < D / 4; ++k) {
            dot = fmaf(qq[k], (float)((by[k] >> sh) & 3u), dot);
            qsum += qq[k];
          }
          if (kt) {   // this lane's D/4 channels lie in one G-channel group
            const int mi = (tlb + ti) * NG + (cq * (D / 4)) / G;
            dot = ks[mi] * (dot - (float)kz[mi] * qsum);
          }
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          if (cq == 0) lg[h * 32 + ti] = dot - bias[h];
        }
      }
      __syncwarp();
      const bool sal = ((bm[t0 / 32] >> lane) & 1u) || t0 + lane >= p.n_q;
#pragma unroll
      for (int h = 0; h < MAXG; ++h)
        if (h < g) logit[h] = sal ? -INFINITY : lg[h * 32 + lane];
    } else if (kind == kRing || c.kind == AKVQ_PSA) {     // 16-bit rows, original basis
      int ntok;
      const uint16_t *krow_of_pass[4];
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int ti = pass * 8 + tq;
        if (kind == kRing) {
          const int tok = item0 + it * 32 + ti;
          krow_of_pass[pass] = tok < p.L ? ring_row(c, u, tok % c.slots) : nullptr;
        } else {
          const int e = it * 32 + ti;
          krow_of_pass[pass] = e < side_n ? reinterpret_cast<const uint16_t *>(side_ptr(c, u, side0 + e)) : nullptr;
        }
      }
      ntok = kind == kRing ? min(32, p.L - (item0 + it * 32)) : min(32, side_n - it * 32);
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int ti = pass * 8 + tq;
        float kx[D / 4];
        if (krow_of_pass[pass]) {
          const uint4 *src = reinterpret_cast<const uint4 *>(krow_of_pass[pass] + cq * (D / 4));
#pragma unroll
          for (int i = 0; i < D / 32; ++i) cvt8<DT>(src[i], kx + 8 * i);
        } else {
#pragma unroll
          for (int i = 0; i < D / 4; ++i) kx[i] = 0.f;
        }
        for (int h = 0; h < g; ++h) {
          const float *qq = qo + h * D + cq * (D / 4);
          float dot = 0.f;
#pragma unroll
          for (int i = 0; i < D / 4; ++i) dot = fmaf(qq[i], kx[i], dot);
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          if (cq == 0) lg[h * 32 + ti] = dot;
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < MAXG; ++h)
        if (h < g) logit[h] = lane < ntok ? lg[h * 32 + lane] : -INFINITY;
    } else {                                              // TSA 4-bit side rows
      const int ntok = min(32, side_n - it * 32);
#pragma unroll
      for (int pass = 0; pass < 4; ++pass) {
        const int ti = pass * 8 + tq;
        const int e = it * 32 + ti;
        const bool ok = e < side_n;
        const uint8_t *se = side_ptr(c, u, side0 + (ok ? e : 0));
        const int gi = (cq * (D / 4)) / G;
        const float sk = reinterpret_cast<const float *>(se)[gi];
        const float zk = (float)reinterpret_cast<const int32_t *>(se + 4 * NG)[gi];
        const uint32_t *cw = reinterpret_cast<const uint32_t *>(se + 16 * NG + cq * (D / 8));
        uint32_t wd[D / 32];
#pragma unroll
        for (int w = 0; w < D / 32; ++w) wd[w] = ok ? cw[w] : 0u;
        for (int h = 0; h < g; ++h) {
          const float *qq = qh + h * D + cq * (D / 4);
          float A = 0.f, B = 0.f;
#pragma unroll
          for (int w = 0; w < D / 32; ++w)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              A = fmaf(qq[8 * w + i], (float)((wd[w] >> (4 * i)) & 15u), A);
              B += qq[8 * w + i];
            }
          float dot = sk * alpha_q * (A - zk * B);
          dot += __shfl_xor_sync(0xffffffffu, dot, 1);
          dot += __shfl_xor_sync(0xffffffffu, dot, 2);
          if (cq == 0) lg[h * 32 + ti] = dot;
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < MAXG; ++h)
        if (h < g) logit[h] = lane < ntok ? lg[h * 32 + lane] : -INFINITY;
    }
    __syncwarp();

    // ============ online softmax (base 2), probabilities to lg
#pragma unroll
    for (int h = 0; h < MAXG; ++h) {
      if (h >= g) break;
      const float mx = warp_max(logit[h]);
      const float mn = fmaxf(m[h], mx);
      float pr = 0.f, sc = 1.f;
      if (mn != -INFINITY) {
        sc = exp2f(m[h] - mn);
        pr = exp2f(logit[h] - mn);
      }
      l[h] = l[h] * sc + warp_sum(pr);
      m[h] = mn;
#pragma unroll
      for (int k = 0; k < CL; ++k) o[h][k] *= sc;
      lg[h * 32 + lane] = pr;
    }
    __syncwarp();

    // ============ V phase: lane owns channels [lane*CL, lane*CL + CL)
    const int c0 = lane * CL;
    if (kind == kPage) {
      const int chunk = item0 + it;
      const int pg = chunk / (G / 32);
      const int tl0 = chunk * 32 - pg * G;                 // token offset in page
      const uint8_t *P = page_ptr(c, u, pg);
      const float *vs = reinterpret_cast<const float *>(P + c.pg_vscale);
      const int32_t *vz = reinterpret_cast<const int32_t *>(P + c.pg_vzero);
      const uint8_t *vc = P + c.pg_vcodes;
      const int gi = c0 / G;
      for (int i = 0; i < 32; ++i) {
        const int tl = tl0 + i;
        const uint32_t byte = vbyte_at(vc, tl, c0 / 4, D);
        const int sh = 2 * (c0 % 4);
        const float sv = vs[tl * NG + gi];
        const float zv = (float)vz[tl * NG + gi];
        float cf[CL];
#pragma unroll
        for (int k = 0; k < CL; ++k) cf[k] = (float)((byte >> (sh + 2 * k)) & 3u) - zv;
#pragma unroll
        for (int h = 0; h < MAXG; ++h) {
          if (h < g) {
            const float w = lg[h * 32 + i] * sv;
#pragma unroll
            for (int k = 0; k < CL; ++k) o[h][k] = fmaf(w, cf[k], o[h][k]);
          }
        }
      }
    } else if (kind == kRing || c.kind == AKVQ_PSA) {
      const int ntok = kind == kRing ? min(32, p.L - (item0 + it * 32)) : min(32, side_n - it * 32);
      for (int i = 0; i < ntok; ++i) {
        const uint16_t *vrow;
        if (kind == kRing) vrow = ring_row(c, u, (item0 + it * 32 + i) % c.slots) + D;
        else vrow = reinterpret_cast<const uint16_t *>(side_ptr(c, u, side0 + it * 32 + i)) + D;
        float vf[CL];
#pragma unroll
        for (int k = 0; k < CL; ++k) vf[k] = H16<DT>::to_f(vrow[c0 + k]);
#pragma unroll
        for (int h = 0; h < MAXG; ++h) {
          if (h < g) {
            const float w = lg[h * 32 + i];
#pragma unroll
            for (int k = 0; k < CL; ++k) o[h][k] = fmaf(w, vf[k], o[h][k]);
          }
        }
      }
    } else {
      const int ntok = min(32, side_n - it * 32);
      const int gi = c0 / G;
      for (int i = 0; i < ntok; ++i) {
        const uint8_t *se = side_ptr(c, u, side0 + it * 32 + i);
        const float sv = reinterpret_cast<const float *>(se + 8 * NG)[gi];
        const float zv = (float)reinterpret_cast<const int32_t *>(se + 12 * NG)[gi];
        const uint8_t *cv = se + 16 * NG + D / 2;
        float cf[CL];
#pragma unroll
        for (int k = 0; k < CL; ++k) {
          const int ch = c0 + k;
          cf[k] = (float)((cv[ch / 2] >> (4 * (ch & 1))) & 15u) - zv;
        }
#pragma unroll
        for (int h = 0; h < MAXG; ++h) {
          if (h < g) {
            const float w = lg[h * 32 + i] * sv;
#pragma unroll
            for (int k = 0; k < CL; ++k) o[h][k] = fmaf(w, cf[k], o[h][k]);
          }
        }
      }
    }
    __syncwarp();
  }

  // ---- merge the warps of this CTA, write the split partial
  float *mw = mg + warp * g * (D + 2);
#pragma unroll
  for (int h = 0; h < MAXG; ++h) {
    if (h >= g) break;
    if (lane == 0) { mw[h * (D + 2)] = m[h]; mw[h * (D + 2) + 1] = l[h]; }
#pragma unroll
    for (int k = 0; k < CL; ++k) mw[h * (D + 2) + 2 + lane * CL + k] = o[h][k];
  }
  __syncthreads();
  const size_t base = ((size_t)u * p.S + s) * g;
  for (int idx = tid; idx < g * D; idx += kThreads) {
    const int h = idx / D, ch = idx % D;
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, mg[(w * g + h) * (D + 2)]);
    float acc = 0.f, lsum = 0.f;
    if (M != -INFINITY) {
      for (int w = 0; w < kWarps; ++w) {
        const float mw_ = mg[(w * g + h) * (D + 2)];
        if (mw_ == -INFINITY) continue;
        const float f = exp2f(mw_ - M);
        acc += f * mg[(w * g + h) * (D + 2) + 2 + ch];
        lsum += f * mg[(w * g + h) * (D + 2) + 1];
      }
    }
    ws_o[(base + h) * D + ch] = acc;
    if (ch == 0) { ws_m[base + h] = M; ws_l[base + h] = lsum; }
  }
}

// Merge the splits of k_decode_split (log-sum-exp) and apply the output H
// (Fig. 7, R4).  Generic path (k_decode_fused merges in-kernel).
template <int D>
__global__ void __launch_bounds__(D) k_combine(DevCache c, DecodePlan p, const float *__restrict__ ws_m,
                                               const float *__restrict__ ws_l,
                                               const float *__restrict__ ws_o, float *__restrict__ out,
                                               uint32_t flags) {
  __shared__ float buf[D];
  const int u = blockIdx.x, ch = threadIdx.x, g = c.g;
  const bool side_rot = c.kind == AKVQ_TSA;
  for (int h = 0; h < g; ++h) {
    float M = -INFINITY;
    for (int s = 0; s < p.S; ++s) M = fmaxf(M, ws_m[((size_t)u * p.S + s) * g + h]);
    float rot = 0.f, org = 0.f, lsum = 0.f;
    for (int s = 0; s < p.S; ++s) {
      const size_t b = ((size_t)u * p.S + s) * g + h;
      const float ms = ws_m[b];
      if (ms == -INFINITY) continue;
      const float f = exp2f(ms - M);
      lsum += f * ws_l[b];
      const float v = f * ws_o[b * D + ch];
      const bool is_rot = s < p.n_page_splits ||
                          (s >= p.n_page_splits + p.n_ring_splits && side_rot);
      if (is_rot) rot += v; else org += v;
    }
    const bool out_rot = flags & AKVQ_OUT_ROTATED;
    buf[ch] = out_rot ? org : rot;          // the part that needs a basis change
    __syncthreads();
    for (int hs = 1; hs < D; hs <<= 1) {
      const int i = ch & ~hs;
      const float a = buf[i], b2 = buf[i | hs];
      const float v = (ch & hs) ? a - b2 : a + b2;
      __syncthreads();
      buf[ch] = v;
      __syncthreads();
    }
    const float tr = buf[ch] * c.inv_sqrt_d;
    const float res = out_rot ? rot + tr : tr + org;
    out[((size_t)u * g + h) * D + ch] = res / lsum;
    __syncthreads();
  }
}

template <int D, int G, int DT, int MAXG>
static cudaError_t launch_dec(const DevCache &c, const DecodePlan &p, const void *q, float *out,
                              void *ws, uint32_t flags, cudaStream_t st) {
  float *ws_m = reinterpret_cast<float *>(ws);
  float *ws_l = ws_m + (size_t)c.U * p.S * c.g;
  float *ws_o = ws_l + (size_t)c.U * p.S * c.g;
  const size_t smem = Smem<D>::floats(c.g) * sizeof(float);
  auto kern = k_decode_split<D, G, DT, MAXG>;
  {
    const cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ea != cudaSuccess) return ea;
  }
  dim3 grid(p.S, c.U);
  kern<<<grid, kThreads, smem, st>>>(c, p, (const uint16_t *)q, ws_m, ws_l, ws_o);
  k_combine<D><<<c.U, D, 0, st>>>(c, p, ws_m, ws_l, ws_o, out, flags);
  return cudaGetLastError();
}

template <int D, int G, int DT>
static cudaError_t launch_dec_g(const DevCache &c, const DecodePlan &p, const void *q, float *out,
                                void *ws, uint32_t flags, cudaStream_t st) {
  if (c.g <= 1) return launch_dec<D, G, DT, 1>(c, p, q, out, ws, flags, st);
  if (c.g <= 4) return launch_dec<D, G, DT, 4>(c, p, q, out, ws, flags, st);
  if (c.g <= 8) return launch_dec<D, G, DT, 8>(c, p, q, out, ws, flags, st);
  return launch_dec<D, G, DT, 16>(c, p, q, out, ws, flags, st);
}

cudaError_t launch_decode(const DevCache &c, int dtype16, const DecodePlan &p, const void *q,
                          float *out, void *ws, uint32_t flags, cudaStream_t st) {
#define AKVQ_DCASE(D_, G_)                                                                  \
  if (c.d == D_ && c.G == G_)                                                               \
    return dtype16 == AKVQ_BF16 ? launch_dec_g<D_, G_, AKVQ_BF16>(c, p, q, out, ws, flags, st) \
                                : launch_dec_g<D_, G_, AKVQ_FP16>(c, p, q, out, ws, flags, st);
  AKVQ_DCASE(64, 32)
  AKVQ_DCASE(64, 64)
  AKVQ_DCASE(128, 32)
  AKVQ_DCASE(128, 64)
  AKVQ_DCASE(128, 128)
#undef AKVQ_DCASE
  return cudaErrorInvalidValue;
}

// ===================================================================== view
// Dequantized view in the rotated normalized basis (R5).  One
// warp per (token, unit); 16-bit rows are rotated with an FWHT in smem.
template <int D, int DT>
__global__ void k_view(DevCache c, int L, int n_q, float *__restrict__ Ko, float *__restrict__ Vo) {
  __shared__ float row[2][D];
  const int t = blockIdx.x, u = blockIdx.y, lane = threadIdx.x;
  const int G = c.G, NG = c.ng;
  const uint32_t *bm = c.bitmask + (size_t)u * c.bm_words;
  const bool sal = (bm[t / 32] >> (t % 32)) & 1u;
  float *ko = Ko + ((size_t)u * L + t) * D;
  float *vo = Vo + ((size_t)u * L + t) * D;
  int e = 0;
  if (t < n_q && sal) {
    for (int w = 0; w < t / 32; ++w) e += __popc(bm[w]);
    e += __popc(bm[t / 32] & ((1u << (t % 32)) - 1u));
  }
  if (t >= n_q || (sal && c.kind == AKVQ_PSA)) {
    const uint16_t *kr = t >= n_q ? ring_row(c, u, t % c.slots)
                                  : reinterpret_cast<const uint16_t *>(side_ptr(c, u, e));
    for (int i = lane; i < D; i += 32) {
      row[0][i] = H16<DT>::to_f(kr[i]);
      row[1][i] = H16<DT>::to_f(kr[D + i]);
    }
    __syncwarp();
    for (int hs = 1; hs < D; hs <<= 1) {
      for (int k = lane; k < D; k += 32) {
        if (k & hs) continue;
        for (int r = 0; r < 2; ++r) {
          const float a = row[r][k], b = row[r][k + hs];
          row[r][k] = a + b;
          row[r][k + hs] = a - b;
        }
      }
      __syncwarp();
    }
    for (int i = lane; i < D; i += 32) {
      ko[i] = row[0][i] * c.inv_sqrt_d;
      vo[i] = row[1][i] * c.inv_sqrt_d;
    }
    return;
  }
  if (sal) {   // TSA 4-bit side entry
    const uint8_t *se = side_ptr(c, u, e);
    for (int i = lane; i < D; i += 32) {
      const int gi = i / G;
      const float sk = reinterpret_cast<const float *>(se)[gi];
      const int32_t zk = reinterpret_cast<const int32_t *>(se + 4 * NG)[gi];
      const float sv = reinterpret_cast<const float *>(se + 8 * NG)[gi];
      const int32_t zv = reinterpret_cast<const int32_t *>(se + 12 * NG)[gi];
      const int ck = (se[16 * NG + i / 2] >> (4 * (i & 1))) & 15;
      const int cv = (se[16 * NG + D / 2 + i / 2] >> (4 * (i & 1))) & 15;
      ko[i] = sk * (float)(ck - zk);
      vo[i] = sv * (float)(cv - zv);
    }
    return;
  }
  const int pg = t / G, tl = t % G;
  const uint8_t *P = page_ptr(c, u, pg);
  const float *ks = reinterpret_cast<const float *>(P + c.pg_kscale);
  const int32_t *kz = reinterpret_cast<const int32_t *>(P + c.pg_kzero);
  const float *vs = reinterpret_cast<const float *>(P + c.pg_vscale);
  const int32_t *vz = reinterpret_cast<const int32_t *>(P + c.pg_vzero);
  const uint8_t *kc = P + c.pg_kcodes;
  const uint8_t *vc = P + c.pg_vcodes;
  const bool kt = c.k_axis == AKVQ_K_PER_TOKEN;
  for (int i = lane; i < D; i += 32) {
    const int ck = (int)kcode_at(kc, tl, i, G);
    const int cv = (int)vcode_at(vc, tl, i, D);
    const int ki = kt ? tl * NG + i / G : i;         // per token [G][NG] | per channel [D]
    ko[i] = ks[ki] * (float)(ck - kz[ki]);
    vo[i] = vs[tl * NG + i / G] * (float)(cv - vz[tl * NG + i / G]);
  }
}

cudaError_t launch_view(const DevCache &c, int dtype16, int L, int n_q, float *K, float *V,
                        cudaStream_t st) {
  dim3 grid(L, c.U);
  if (c.d == 64) {
    if (dtype16 == AKVQ_BF16) k_view<64, AKVQ_BF16><<<grid, 32, 0, st>>>(c, L, n_q, K, V);
    else k_view<64, AKVQ_FP16><<<grid, 32, 0, st>>>(c, L, n_q, K, V);
  } else {
    if (dtype16 == AKVQ_BF16) k_view<128, AKVQ_BF16><<<grid, 32, 0, st>>>(c, L, n_q, K, V);
    else k_view<128, AKVQ_FP16><<<grid, 32, 0, st>>>(c, L, n_q, K, V);
  }
  return cudaGetLastError();
}

}  // namespace akvq
