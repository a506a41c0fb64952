// decode_common.cuh -- pieces of the persistent decode kernel (k_decode_layer):
// TMA bulk / mbarrier / PDL wrappers, the partial-record layout, the
// (warp, unit) segment mapping and the per-unit merge (log-sum-exp over
// segments, output Walsh-Hadamard, Fig. 7 / R4).
#pragma once
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace akvq {

// Single-instruction warp reductions (REDUX) for the per-page critical path;
// AKVQ_REDUX=0 builds the shuffle-tree versions (A/B).
#ifndef AKVQ_REDUX
#define AKVQ_REDUX 0
#endif
// max over the warp of a float: the order-preserving map of IEEE bits to
// signed integers (negative values: magnitude bits flipped) is an involution
__device__ __forceinline__ float warp_max_fast(float v) {
#if AKVQ_REDUX
  int i = __float_as_int(v);
  i ^= (i >> 31) & 0x7fffffff;
  i = __reduce_max_sync(0xffffffffu, i);
  i ^= (i >> 31) & 0x7fffffff;
  return __int_as_float(i);
#else
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
#endif
}


#ifndef AKVQ_LY_STAGES
#define AKVQ_LY_STAGES 2
#endif
constexpr int kLyStages = AKVQ_LY_STAGES;   // TMA stages per warp
constexpr int kRows = 8;           // 16-bit rows per ring chunk / side sub-load
constexpr int kRows4 = 32;         // 4-bit TSA rows per side sub-load
// unroll factors of the page MMA loops (K: token blocks, V: channel blocks)
#ifndef AKVQ_KU
#define AKVQ_KU 4
#endif
#ifndef AKVQ_VU
#define AKVQ_VU 4
#endif
#define AKVQ_PRAGMA(x) _Pragma(#x)
#define AKVQ_UNROLL(n) AKVQ_PRAGMA(unroll n)
// Page fixed points: signed 24-bit integers as three int8 limbs,
// relative to per-unit ranges (umax: the largest |K| / |V| scale of the unit's
// pages, maintained by the quantizer).
//  K: Q_c = rn(q~_c s^K_c kQMax / (max|q~| umax.K)), |Q| <= kQMax;
//  V: W_t = rn(p_t s^V_t kQMax / umax.V), |W| <= kQMax (p <= 1).
// X + kQOff lies in [0, 2^24); limb k = byte k of X + kQOff minus 128 (signed
// int8: byte ^ 0x80).  kQMax < 127 * 65793 leaves room for the few-ulp error of
// __fdividef and the products.  Each head owns 4 MMA B columns: limbs 0, 1, 2
// and one unused column (k_decode_layer; k_decode_gqa packs the limbs).
constexpr int kQMax = 8355700;
constexpr uint32_t kQOff = 0x808080u;

// stage bytes: max(page K half, page V half, kRows 16-bit rows, kRows4 side4 rows)
__host__ __device__ inline size_t ly_stage_bytes(const DevCache &c) {
  size_t a = c.pg_vscale, b = c.page_bytes - c.pg_vscale;
  size_t m = a > b ? a : b;
  const size_t r16 = (size_t)kRows * 4 * c.d;
  if (r16 > m) m = r16;
  if (c.kind == AKVQ_TSA) {
    const size_t r4 = (size_t)kRows4 * c.side_entry;
    if (r4 > m) m = r4;
  }
  return (m + 127) / 128 * 128;
}

// 2^x with the SFU's approximate ex2 (rel. error ~2^-22, flushes subnormal
// results to 0): softmax weights below 2^-126 of the running max are 0 anyway.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t fmask(uint32_t w, int s) { return w & (0x03030303u << (2 * s)); }

// Legacy warp MMA m16n8k32 (IMMA, int32 accumulate): A 16x32 u8 row-major, B
// 32x8 s8 / u8 column-major.  Fragments (lane = 4 * grp + tig): a0 / a1 hold
// rows grp / grp + 8, columns 4 tig .. 4 tig + 3; a2 / a3 the same rows,
// columns 16 + 4 tig ..; b0 / b1 rows 4 tig .. / 16 + 4 tig .. of column grp;
// c0, c1 row grp, columns 2 tig, 2 tig + 1; c2, c3 row grp + 8.
__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
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

// Sum v[NV] over the CQ lanes of a row group (lane bits below CQ): a reduce-
// scatter halves the values per step, then a butterfly finishes.  On return
// `mine` is the slot whose total this lane holds.
template <int NV, int CQ>
__device__ __forceinline__ float rs_reduce(float (&v)[NV], int cq, int &mine) {
  constexpr int L2 = NV == 8 ? 3 : (NV == 4 ? 2 : (NV == 2 ? 1 : 0));
  static_assert((1 << L2) == NV && (CQ >> L2) >= 1, "reduce shape");
  mine = 0;
#pragma unroll
  for (int step = 0; step < L2; ++step) {
    const int n = NV >> step, off = CQ >> (step + 1);
    const bool up = cq & off;
#pragma unroll
    for (int i = 0; i < n / 2; ++i) {
      const float send = up ? v[i] : v[i + n / 2];
      const float keep = up ? v[i + n / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    if (up) mine += n / 2;
  }
  float t = v[0];
#pragma unroll
  for (int off = CQ >> (L2 + 1); off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  return t;
}

// One sub-load of the pipeline: an item split into stage-sized pieces.  The
// producer lane records it in the warp's descriptor ring (one per stage).
struct LySub {
  int u, kind;   // u: (virtual) unit; kind: 0 page K half, 1 page V half, 2 16-bit rows, 3 4-bit rows,
                 // 4 empty unit marker (no data), -1 none
  int pu;        // physical unit (u / head groups), producer side only
  int a, n;      // page index | first row (ring offset from n_q / side entry) and row count
  int ring;      // 1 if ring rows
};
// descriptor as it travels from the producer lane to the warp: two words
//   x = u, y = (kind + 1) | ring << 3 | n << 4 (n < 64) | a << 10
__device__ __forceinline__ uint2 pack_sub(const LySub &s) {
  return make_uint2((uint32_t)s.u, (uint32_t)(s.kind + 1) | ((uint32_t)s.ring << 3) |
                                       ((uint32_t)s.n << 4) | ((uint32_t)s.a << 10));
}
__device__ __forceinline__ LySub unpack_sub(uint2 w) {
  LySub s;
  s.u = (int)w.x;
  s.kind = (int)(w.y & 7u) - 1;
  s.ring = (int)((w.y >> 3) & 1u);
  s.n = (int)((w.y >> 4) & 63u);
  s.a = (int)(w.y >> 10);
  return s;
}

__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// lane bits that encode slot m of rs_reduce<NV, CQ> (see there)
template <int NV, int CQ>
__device__ __forceinline__ constexpr int rs_enc(int m) {
  constexpr int L2 = NV == 8 ? 3 : (NV == 4 ? 2 : (NV == 2 ? 1 : 0));
  int e = 0;
  for (int j = 0; j < L2; ++j)
    if ((m >> (L2 - 1 - j)) & 1) e |= CQ >> (j + 1);
  return e;
}


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
// the same on precomputed shared-window addresses (no generic->shared conversion
// in the pipeline loop)
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
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
// out-of-line copy (the 64-bit divisions are large; called twice per warp)
static __device__ __noinline__ int ly_first_item_p(const LayerPlan *lp, int w) { return ly_first_item(*lp, w); }
// out-of-line: warps owning unit u's first and last items (segment flush)
static __device__ __noinline__ int2 ly_warp_span_p(const LayerPlan *lp, int u) {
  return make_int2(ly_warp_of(*lp, u, 0), ly_warp_of(*lp, u, lp->per_u - 1));
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

// End of a fused-step launch: every warp of the grid reports its exit; the last
// one advances the device token count L.  Every warp reads L right after its
// griddepcontrol.wait, before any warp can be the last to exit, so a launch sees
// the L of its own step; this keeps the launch parameters the same from step to
// step (CUDA-graph replay, AKVQ_OPT_DEVICE_L).
// The count is kept per CTA in shared memory (cta_done, zeroed before any warp
// can exit); the last warp of a CTA reports the CTA.  No fence is needed: a
// warp's L was loaded before its own exit, and the next launch sees the new L
// after griddepcontrol.wait (full completion of this grid).
__device__ __forceinline__ void ly_exit(const DevCache &c, const LayerPlan &lp, int lane,
                                        unsigned *cta_done) {
  if (!(lp.appends && lp.dev_L)) return;
  __syncwarp();
  if (lane == 0 && atomicAdd(cta_done, 1u) == (blockDim.x >> 5) - 1u &&
      atomicAdd(&c.dstate->done, 1u) == gridDim.x - 1u) {
    c.dstate->done = 0u;
    c.dstate->L += 1;
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
