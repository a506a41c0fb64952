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
// One CTA per (block j, unit u); thread t owns token j*G + t of the block.
//   1. row -> fp32 -> in-register FWHT (x.H_s, R5) -> smem for the K stats
//   2. thread ch: min/max of channel ch over the block's non-salient tokens,
//      Eqs. 5-6 -> K meta (per channel, R1)
//   3. thread t: K codes of its row, packed 4 per byte along channels
//   4. V row: FWHT, per-token stats over each G-channel group, codes, meta
//   5. salient tokens -> side table (PSA 16-bit originals; TSA 4-bit rotated)
// Source rows come from the prefill inputs or, for a flush, from the ring.
template <int D, int G, int DT>
__global__ void __launch_bounds__(G) k_quantize_blocks(DevCache c, QuantSrc src, int block0,
                                                       int last_block) {
  constexpr int P = D + 1;                   // smem pitch (conflict-free columns)
  constexpr int NG = D / G;
  extern __shared__ float xs[];              // [G][D+1]
  __shared__ float s_s[D], s_z[D];
  __shared__ int s_mode[D];
  __shared__ uint32_t s_bits[G / 32];
  __shared__ int s_base;

  const int u = blockIdx.y, j = block0 + blockIdx.x, t = threadIdx.x;
  const int tok = j * G + t;
  const uint32_t *bm = c.bitmask + (size_t)u * c.bm_words;
  if (t < G / 32) s_bits[t] = bm[j * (G / 32) + t];
  if (t == 0) s_base = 0;
  __syncthreads();
  {  // salient entries before this block -> first side slot of the block
    int cnt = 0;
    for (int w = t; w < j * (G / 32); w += G) cnt += __popc(bm[w]);
    if (cnt) atomicAdd(&s_base, cnt);
  }
  const bool sal = (s_bits[t >> 5] >> (t & 31)) & 1u;
  const size_t roff = (size_t)u * src.unit_stride +
                      (size_t)(src.ring_slots ? tok % src.ring_slots : tok) * src.tok_stride;
  const uint16_t *krow = src.K + roff;
  const uint16_t *vrow = src.V + roff;
  uint8_t *pg = page_ptr(c, u, j);
  const bool tsa = c.kind == AKVQ_TSA;

  // ---------------- K
  float x[D];
  load_row<D, DT>(krow, x);
  fwht_reg<D>(x);
#pragma unroll
  for (int i = 0; i < D; ++i) xs[t * P + i] = x[i];
  __syncthreads();
  for (int ch = t; ch < D; ch += G) {
    float mn = 0.f, mx = 0.f;
    bool any = false;
    for (int i = 0; i < G; ++i) {
      if ((s_bits[i >> 5] >> (i & 31)) & 1u) continue;
      const float v = xs[i * P + ch];
      if (!any) { mn = v; mx = v; any = true; }
      else { mn = fminf(mn, v); mx = fmaxf(mx, v); }
    }
    const QMeta m = q_meta(mn, mx, any, c.clip2, 3.f);
    s_s[ch] = m.s; s_z[ch] = m.zf; s_mode[ch] = m.mode;
    reinterpret_cast<float *>(pg + c.pg_kscale)[ch] = __fmul_rn(m.s, c.inv_sqrt_d);
    reinterpret_cast<int32_t *>(pg + c.pg_kzero)[ch] = zero_i32(m.zf);
  }
  __syncthreads();
  // codes staged as one byte each in smem (xs is dead now), then re-packed into
  // the page's 4x4-tile K words (common.cuh kword_idx) with coalesced stores
  uint8_t *cs8 = reinterpret_cast<uint8_t *>(xs);            // [G][D] K codes
  uint8_t *vb8 = cs8 + G * D;                                 // [G][D/4] V bytes
  {
#pragma unroll
    for (int w = 0; w < D / 4; ++w) {
      uint32_t word = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int ch = 4 * w + i;
        QMeta m; m.s = s_s[ch]; m.zf = s_z[ch]; m.mode = s_mode[ch];
        const uint32_t code = sal ? 0u : q_code(x[ch], m, 3.f);
        word |= code << (8 * i);
      }
      reinterpret_cast<uint32_t *>(cs8 + t * D)[w] = word;
    }
  }
  __syncthreads();
  {
    constexpr int TQ = G / 4;
    uint32_t *dst = reinterpret_cast<uint32_t *>(pg + c.pg_kcodes);
    for (int wi = t; wi < (D / 4) * TQ; wi += G) {      // word wi -> (cq, tq)
      const int cq = (wi & 3) + 4 * (wi / (4 * TQ)), tq = (wi / 4) % TQ;
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2)
          word |= (uint32_t)cs8[(4 * tq + s2) * D + 4 * cq + b] << (8 * b + 2 * s2);
      dst[wi] = word;
    }
  }
  // side slot of this token (ascending token order within the side table)
  const uint32_t below = (t & 31) ? (s_bits[t >> 5] & ((1u << (t & 31)) - 1u)) : 0u;
  int pos = s_base + __popc(below);
  for (int w = 0; w < (t >> 5); ++w) pos += __popc(s_bits[w]);
  uint8_t *se = sal ? side_ptr(c, u, pos) : nullptr;
  if (sal && tsa) {  // TSA text token: 4-bit per-token K groups, clip4 (R11)
    float *sk = reinterpret_cast<float *>(se);
    int32_t *zk = reinterpret_cast<int32_t *>(se + 4 * NG);
    uint8_t *ck = se + 16 * NG;
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      float mn = x[gi * G], mx = x[gi * G];
#pragma unroll
      for (int i = 1; i < G; ++i) { mn = fminf(mn, x[gi * G + i]); mx = fmaxf(mx, x[gi * G + i]); }
      const QMeta m = q_meta(mn, mx, true, c.clip4, 15.f);
      sk[gi] = __fmul_rn(m.s, c.inv_sqrt_d);
      zk[gi] = zero_i32(m.zf);
#pragma unroll
      for (int i = 0; i < G; i += 2) {
        const uint32_t lo = q_code(x[gi * G + i], m, 15.f), hi = q_code(x[gi * G + i + 1], m, 15.f);
        ck[(gi * G + i) / 2] = (uint8_t)(lo | (hi << 4));
      }
    }
  }

  // ---------------- V (per token over G-channel groups)
  load_row<D, DT>(vrow, x);
  fwht_reg<D>(x);
  {
    float *vs = reinterpret_cast<float *>(pg + c.pg_vscale) + (size_t)t * NG;
    int32_t *vz = reinterpret_cast<int32_t *>(pg + c.pg_vzero) + (size_t)t * NG;
    uint32_t wds[D / 16];
#pragma unroll
    for (int w = 0; w < D / 16; ++w) wds[w] = 0;
#pragma unroll
    for (int gi = 0; gi < NG; ++gi) {
      float mn = x[gi * G], mx = x[gi * G];
#pragma unroll
      for (int i = 1; i < G; ++i) { mn = fminf(mn, x[gi * G + i]); mx = fmaxf(mx, x[gi * G + i]); }
      QMeta m = q_meta(mn, mx, !sal, c.clip2, 3.f);
      vs[gi] = sal ? 0.f : __fmul_rn(m.s, c.inv_sqrt_d);
      vz[gi] = sal ? 0 : zero_i32(m.zf);
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int ch = gi * G + i;
        wds[ch / 16] |= (sal ? 0u : q_code(x[ch], m, 3.f)) << (2 * (ch % 16));
      }
    }
    // the token's S:146 bytes -> smem, re-packed below into 4x4-tile V words
#pragma unroll
    for (int w = 0; w < D / 16; ++w) reinterpret_cast<uint32_t *>(vb8 + t * (D / 4))[w] = wds[w];
  }
  __syncthreads();
  {
    constexpr int CQ = D / 4;
    uint32_t *dst = reinterpret_cast<uint32_t *>(pg + c.pg_vcodes);
    for (int wi = t; wi < CQ * (G / 4); wi += G) {      // word wi -> (cq, tq)
      const int tq = (wi & 3) + 4 * (wi / (4 * CQ)), cq = (wi / 4) % CQ;
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) word |= (uint32_t)vb8[(4 * tq + b) * (D / 4) + cq] << (8 * b);
      dst[wi] = word;
    }
  }
  if (sal) {
    c.side_idx[(size_t)u * c.side_cap + pos] = tok;
    if (tsa) {
      float *sv = reinterpret_cast<float *>(se + 8 * NG);
      int32_t *zv = reinterpret_cast<int32_t *>(se + 12 * NG);
      uint8_t *cv = se + 16 * NG + D / 2;
#pragma unroll
      for (int gi = 0; gi < NG; ++gi) {
        float mn = x[gi * G], mx = x[gi * G];
#pragma unroll
        for (int i = 1; i < G; ++i) { mn = fminf(mn, x[gi * G + i]); mx = fmaxf(mx, x[gi * G + i]); }
        const QMeta m = q_meta(mn, mx, true, c.clip4, 15.f);
        sv[gi] = __fmul_rn(m.s, c.inv_sqrt_d);
        zv[gi] = zero_i32(m.zf);
#pragma unroll
        for (int i = 0; i < G; i += 2) {
          const uint32_t lo = q_code(x[gi * G + i], m, 15.f), hi = q_code(x[gi * G + i + 1], m, 15.f);
          cv[(gi * G + i) / 2] = (uint8_t)(lo | (hi << 4));
        }
      }
    } else {  // PSA pivot: original 16-bit K and V rows (R10)
      uint4 *dk = reinterpret_cast<uint4 *>(se);
      const uint4 *sk = reinterpret_cast<const uint4 *>(krow);
      const uint4 *sv = reinterpret_cast<const uint4 *>(vrow);
#pragma unroll
      for (int i = 0; i < D / 8; ++i) { dk[i] = sk[i]; dk[D / 8 + i] = sv[i]; }
    }
  }
  if (j == last_block) {  // number of side entries after this block
    __syncthreads();
    if (t == 0) {
      int n = s_base;
      for (int w = 0; w < G / 32; ++w) n += __popc(s_bits[w]);
      c.side_cnt[u] = n;
    }
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
    cudaFuncSetAttribute(k_salient_psa, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int nt = L0 >= 8192 ? 1024 : (L0 >= 1024 ? 512 : 128);
    k_salient_psa<<<c.U, nt, smem, st>>>(c, colsum, L0, top_k);
  }
  return cudaGetLastError();
}

template <int D, int G, int DT>
static cudaError_t launch_q(const DevCache &c, const QuantSrc &src, int block0, int nblocks,
                            int last_block, cudaStream_t st) {
  const size_t smem = (size_t)G * (D + 1) * sizeof(float);
  auto kern = k_quantize_blocks<D, G, DT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid(nblocks, c.U);
  kern<<<grid, G, smem, st>>>(c, src, block0, last_block);
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

cudaError_t launch_ring_fill(const DevCache &c, const void *K, const void *V, int L0, int t0,
                             int t1, cudaStream_t st) {
  if (t1 <= t0) return cudaSuccess;
  const int n = (t1 - t0) * 2 * (c.d / 8);
  dim3 grid((n + 255) / 256, c.U);
  k_ring_fill<<<grid, 256, 0, st>>>(c, (const uint16_t *)K, (const uint16_t *)V, L0, t0, t1);
  return cudaGetLastError();
}

cudaError_t launch_append(const DevCache &c, const void *k, const void *v, const uint8_t *types,
                          int L, cudaStream_t st) {
  k_append<<<c.U, 2 * (c.d / 8), 0, st>>>(c, (const uint16_t *)k, (const uint16_t *)v, types, L);
  return cudaGetLastError();
}

}  // namespace akvq
