// decode_common.cuh -- pieces of the persistent decode kernel (k_decode_layer):
// TMA bulk / mbarrier / PDL wrappers, the partial-record layout, the
// (warp, unit) segment mapping and the per-unit merge (log-sum-exp over
// segments, output Walsh-Hadamard, Fig. 7 / R4).
#pragma once
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace akvq {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s));
  return r;
}
// Programmatic dependent launch (PDL) controls.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Partial record of one (warp, unit) segment, per head (floats, 16-byte aligned):
//   [o_org D][o_rot D][m][l][pad 2]
// o_org: sum p v over 16-bit rows (original basis); o_rot: sum p v^ over 2-bit
// pages and 4-bit rows (rotated, normalized basis); m, l: base-2 running max
// and sum of the segment's online softmax.
template <int D> struct Rec {
  static constexpr int R = 2 * D + 4;
};

// Cost-weighted segments of the layer plan (kernels.h LayerPlan): item i = (u, k)
// starts at cost u * cu + cpre[k]; warp(i) = floor(start * W / CT).  Products
// in 64 bits (CT * W may exceed 2^32 for long contexts and large batches).
__device__ __forceinline__ int ly_warp_of(const LayerPlan &lp, int u, int k) {
  const unsigned long long c = (unsigned long long)u * (unsigned)lp.cu + lp.cpre[k];
  return (int)((c * (unsigned)lp.W) / (unsigned long long)lp.CT);
}
// first cost owned by warp w: ceil(w CT / W)
__device__ __forceinline__ unsigned long long ly_first_cost(const LayerPlan &lp, int w) {
  return ((unsigned long long)w * (unsigned long long)lp.CT + (unsigned)lp.W - 1u) / (unsigned)lp.W;
}
// first item (flattened u * per_u + k) of warp w: the first start cost >= c0
__device__ __forceinline__ int ly_first_item(const LayerPlan &lp, int w) {
  const unsigned long long c0 = ly_first_cost(lp, w);
  int u = (int)(c0 / (unsigned)lp.cu);
  const int r = (int)(c0 - (unsigned long long)u * (unsigned)lp.cu);
  int lo = 0, hi = lp.per_u;                          // smallest k with cpre[k] >= r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (lp.cpre[mid] >= r) hi = mid; else lo = mid + 1;
  }
  if (lo == lp.per_u) { ++u; lo = 0; }
  return u * lp.per_u + lo;
}
// unit of warp w's first item (O(1): c0 falls in unit c0 / cu unless past its last start)
__device__ __forceinline__ int ly_first_unit(const LayerPlan &lp, int w) {
  const unsigned long long c0 = ly_first_cost(lp, w);
  const int u = (int)(c0 / (unsigned)lp.cu);
  return (int)(c0 - (unsigned long long)u * (unsigned)lp.cu) > (int)lp.cpre[lp.per_u - 1] ? u + 1 : u;
}

// Per-unit merge by one warp: log-sum-exp over all segments of unit u, then
// out = (o_rot . H + o_org) / l (or o_rot + o_org . H with AKVQ_OUT_ROTATED),
// H applied as an unnormalized FWHT times 1/sqrt d (Fig. 7, R4).  Partials are
// read with ld.global.cg (written by other SMs of this grid).  Lane j < #segs
// fetches segment j's (m, l) so the loads overlap.
template <int D, int NH>
__device__ __noinline__ void merge_layer_unit(const DevCache &c, const LayerPlan &lp, const float *part, int u,
                                 float *out_u, int nh, uint32_t flags, int lane) {
  constexpr int CPL = D / 32;
  const int w0 = ly_warp_of(lp, u, 0), w1 = ly_warp_of(lp, u, lp.per_u - 1);
  const int nseg = w1 - w0 + 1;
  const bool out_rot = flags & AKVQ_OUT_ROTATED;
  auto seg_rec = [&](int j, int h) -> const float * {
    const int w = w0 + j;
    const int slot = w * lp.maxseg + (u - ly_first_unit(lp, w));
    return part + ((size_t)slot * NH + h) * Rec<D>::R;
  };
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    if (h >= nh) break;                            // padded head of the last GQA group
    float M = -INFINITY;
    for (int b0 = 0; b0 < nseg; b0 += 32) {
      const float ms = b0 + lane < nseg ? __ldcg(seg_rec(b0 + lane, h) + 2 * D) : -INFINITY;
      M = fmaxf(M, warp_max(ms));
    }
    float rot[CPL], org[CPL], lsum = 0.f;
#pragma unroll
    for (int k = 0; k < CPL; ++k) { rot[k] = 0.f; org[k] = 0.f; }
    if (M != -INFINITY) {
      for (int b0 = 0; b0 < nseg; b0 += 32) {
        float f = 0.f, ls = 0.f;
        const float *rh = nullptr;
        if (b0 + lane < nseg) {
          rh = seg_rec(b0 + lane, h);
          const float ms = __ldcg(rh + 2 * D);
          ls = __ldcg(rh + 2 * D + 1);
          f = ms == -INFINITY ? 0.f : exp2f(ms - M);
        }
        lsum += warp_sum(f * ls);
        const int nb = min(32, nseg - b0);
        // 4 segments per round: their loads are independent and issue together
        // (segments with weight 0 -- empty softmax -- read a valid record, add 0)
        for (int j0 = 0; j0 < nb; j0 += 4) {
          float fj[4], vo[4][CPL], vr[4][CPL];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int j = min(j0 + jj, nb - 1);
            fj[jj] = j0 + jj < nb ? __shfl_sync(0xffffffffu, f, j) : 0.f;
            const unsigned long long pj =
                __shfl_sync(0xffffffffu, (unsigned long long)(uintptr_t)rh, j);
            const float *r = reinterpret_cast<const float *>((uintptr_t)pj);
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              vo[jj][k] = __ldcg(r + CPL * lane + k);
              vr[jj][k] = __ldcg(r + D + CPL * lane + k);
            }
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int k = 0; k < CPL; ++k) {
              if (fj[jj] != 0.f) {
                org[k] = fmaf(fj[jj], vo[jj][k], org[k]);
                rot[k] = fmaf(fj[jj], vr[jj][k], rot[k]);
              }
            }
        }
      }
    }
    float x[CPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) x[k] = out_rot ? org[k] : rot[k];
    // FWHT over D channels: lane holds channels CPL*lane .. CPL*lane + CPL - 1
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
    float *dst = out_u + (size_t)h * D + CPL * lane;
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const float tr = x[k] * c.inv_sqrt_d;
      dst[k] = (out_rot ? rot[k] + tr : tr + org[k]) * inv;
    }
  }
}

// Ticket: called by every warp that wrote a segment of unit u; returns true
// in exactly one warp (the last of `expected`), which then merges.
__device__ __forceinline__ bool take_ticket(const DevCache &c, int u, int expected, int lane) {
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atomicAdd(&c.ticket[u], 1u) == (unsigned)(expected - 1);
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) __threadfence();
  return last;
}

}  // namespace akvq
