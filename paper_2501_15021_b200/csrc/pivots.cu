// pivots.cu -- massive-activation pivot detection (
// SURVEY NEXT-2) and the PSA salient bitmask from an explicit pivot list.
//
//   score(t) = max_c |residual[t][c]|                   k_pivot_scores
//   m = median of the scores (R22), pivots = score > tau * m ordered
//   (score desc, index asc), at most n_max, fallback [0]  k_pivot_select
//
// k_pivot_scores streams the residual (HBM-bound: hidden x 2 bytes per token),
// one warp per token, 16-byte loads; k_pivot_select is one CTA per residual
// row: exact medians by radix select over the order-preserving bit patterns of
// the non-negative fp32 scores, then n_max rounds of a block-wide arg-max.
#include "common.cuh"
#include "kernels.h"

namespace akvq {

constexpr int kPvScoreWarps = 8;
constexpr int kPvSelThreads = 1024;

template <int DT>
__global__ void __launch_bounds__(kPvScoreWarps * 32)
    k_pivot_scores(const uint16_t *__restrict__ res, int L0, int hidden, float *__restrict__ score) {
  const int row = blockIdx.y, lane = threadIdx.x & 31;
  const int t = blockIdx.x * kPvScoreWarps + (threadIdx.x >> 5);
  if (t >= L0) return;
  const uint16_t *x = res + ((size_t)row * L0 + t) * hidden;
  float mx = 0.f;
  if ((hidden & 7) == 0) {
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    for (int i = lane; i < hidden / 8; i += 32) {
      float v[8];
      cvt8<DT>(__ldg(x4 + i), v);
#pragma unroll
      for (int k = 0; k < 8; ++k) mx = fmaxf(mx, fabsf(v[k]));
    }
  } else {
    for (int i = lane; i < hidden; i += 32) mx = fmaxf(mx, fabsf(H16<DT>::to_f(x[i])));
  }
  mx = warp_max(mx);
  if (lane == 0) score[(size_t)row * L0 + t] = mx;
}

// k-th smallest (0-based) of n non-negative fp32 values in smem (uint order).
__device__ uint32_t radix_select(const float *s, int n, int k, uint32_t *hist) {
  const int tid = threadIdx.x;
  uint32_t prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
      const uint32_t b = __float_as_uint(s[i]);
      if ((b & mask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
    }
    __syncthreads();
    __shared__ uint32_t sel_bin, sel_k;
    if (tid == 0) {
      uint32_t acc = 0, bin = 0;
      for (; bin < 256; ++bin) {
        if (acc + hist[bin] > (uint32_t)k) break;
        acc += hist[bin];
      }
      sel_bin = bin;
      sel_k = (uint32_t)k - acc;
    }
    __syncthreads();
    prefix |= sel_bin << shift;
    mask |= 255u << shift;
    k = (int)sel_k;
    __syncthreads();
  }
  return prefix;
}

__device__ __forceinline__ uint64_t pv_key(float s, int t) {   // larger = earlier
  return ((uint64_t)__float_as_uint(s) << 32) | (uint32_t)(0xffffffffu - (uint32_t)t);
}

__global__ void __launch_bounds__(kPvSelThreads)
    k_pivot_select(const float *__restrict__ score, int L0, float tau, int n_max,
                   int32_t *__restrict__ pivots, int32_t *__restrict__ counts) {
  extern __shared__ float sc[];
  __shared__ uint32_t hist[256];
  __shared__ uint64_t red[32];
  __shared__ float s_thr;
  const int row = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  for (int t = tid; t < L0; t += nt) sc[t] = score[(size_t)row * L0 + t];
  __syncthreads();
  const uint32_t hi = radix_select(sc, L0, L0 / 2, hist);
  float m = __uint_as_float(hi);
  if ((L0 & 1) == 0) {
    const uint32_t lo = radix_select(sc, L0, L0 / 2 - 1, hist);
    m = __fmul_rn(__fadd_rn(__uint_as_float(lo), m), 0.5f);       // R22
  }
  if (tid == 0) s_thr = __fmul_rn(tau, m);
  __syncthreads();
  const float thr = s_thr;
  uint64_t prev = ~0ull;
  int n = 0;
  for (int r = 0; r < n_max; ++r) {
    uint64_t best = 0;
    for (int t = tid; t < L0; t += nt) {
      if (!(sc[t] > thr)) continue;
      const uint64_t key = pv_key(sc[t], t);
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
      if (tid == 0) red[0] = v;
    }
    __syncthreads();
    const uint64_t v = red[0];
    __syncthreads();
    if (v == 0) break;                               // no more tokens above the threshold
    if (tid == 0) pivots[(size_t)row * n_max + r] = (int)(0xffffffffu - (uint32_t)(v & 0xffffffffu));
    prev = v;
    ++n;
  }
  if (tid == 0) {
    if (n == 0) { pivots[(size_t)row * n_max] = 0; n = 1; }   // attention-sink fallback
    counts[row] = n;
  }
}

// PSA salient bitmask from pivot lists: unit u uses row u / units_per_row.
__global__ void k_salient_from_pivots(DevCache c, const int32_t *__restrict__ pivots,
                                      const int32_t *__restrict__ counts, int n_max,
                                      int units_per_row, int L0) {
  const int u = blockIdx.x, i = threadIdx.x;
  const int row = u / units_per_row;
  if (i >= counts[row] || i >= n_max) return;
  const int t = pivots[(size_t)row * n_max + i];
  if (t < 0 || t >= L0) return;
  atomicOr(&c.bitmask[(size_t)u * c.bm_words + t / 32], 1u << (t % 32));
}

cudaError_t launch_pivot_detect(const void *res, int n_rows, int L0, int hidden, int dtype16,
                                float tau, int n_max, float *score_ws, int32_t *pivots,
                                int32_t *counts, cudaStream_t st) {
  dim3 g1((L0 + kPvScoreWarps - 1) / kPvScoreWarps, n_rows);
  if (dtype16 == AKVQ_BF16)
    k_pivot_scores<AKVQ_BF16><<<g1, kPvScoreWarps * 32, 0, st>>>((const uint16_t *)res, L0, hidden, score_ws);
  else
    k_pivot_scores<AKVQ_FP16><<<g1, kPvScoreWarps * 32, 0, st>>>((const uint16_t *)res, L0, hidden, score_ws);
  const size_t smem = (size_t)L0 * sizeof(float);
  {
    const cudaError_t ea = cudaFuncSetAttribute(k_pivot_select, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (ea != cudaSuccess) return ea;
  }
  k_pivot_select<<<n_rows, kPvSelThreads, smem, st>>>(score_ws, L0, tau, n_max, pivots, counts);
  return cudaGetLastError();
}

cudaError_t launch_salient_from_pivots(const DevCache &c, const int32_t *pivots,
                                       const int32_t *counts, int n_max, int units_per_row,
                                       int L0, cudaStream_t st) {
  k_salient_from_pivots<<<c.U, 32, 0, st>>>(c, pivots, counts, n_max, units_per_row, L0);
  return cudaGetLastError();
}

}  // namespace akvq
