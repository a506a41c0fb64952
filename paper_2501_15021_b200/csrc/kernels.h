// kernels.h -- host launchers of the libakvq.so kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace akvq {

struct DevCache;

// Source rows of a quantize launch: prefill inputs [U][L0][d] or the ring.
struct QuantSrc {
  const uint16_t *K, *V;
  size_t unit_stride;   // elements between units
  size_t tok_stride;    // elements between tokens (slots in ring mode)
  int ring_slots;       // 0: linear token index; >0: slot = token % ring_slots
};

// Fused decode plan (k_decode_fused): per unit, items [P pages][NR ring chunks]
// [NS side splits] with start costs k*cp, P*cp + r*cr, P*cp + NR*cr + s*cs;
// warp w of W owns the items whose start cost lies in [w*T/W, (w+1)*T/W),
// T = U * cost_unit.  Partials: W * maxseg slots.
struct FusedPlan {
  static constexpr int kRowChunk = 8;   // 16-bit / 4-bit rows per sub-load
  long long T, W;
  int cost_unit, P, NR, NS, cp, cr, cs, maxseg;
  int L, n_q;
  size_t stage_bytes;
};

// Decode split plan (host-computed, uniform across units).
struct DecodePlan {
  int L, n_q;
  int n_pages;           // quantized pages in use = n_q / G
  int pages_per_split, n_page_splits;
  int ring_per_split, n_ring_splits;
  int n_side_splits;     // side entries are shared equally among these splits
  int S;                 // total splits of k_decode_split (ring / side / fallback pages)
  int fused;             // 1: the whole decode runs in k_decode_fused
  FusedPlan fp;
};

cudaError_t launch_salient(const DevCache &c, const uint8_t *types, const float *colsum,
                           int L0, int top_k, cudaStream_t st);
cudaError_t launch_quantize_blocks(const DevCache &c, int dtype16, const QuantSrc &src,
                                   int block0, int nblocks, int last_block, cudaStream_t st);
cudaError_t launch_ring_fill(const DevCache &c, const void *K, const void *V, int L0, int t0,
                             int t1, cudaStream_t st);
cudaError_t launch_append(const DevCache &c, const void *k, const void *v,
                          const uint8_t *types, int L, cudaStream_t st);
cudaError_t launch_decode(const DevCache &c, int dtype16, const DecodePlan &p, const void *q,
                          float *out, void *ws, uint32_t flags, cudaStream_t st);
cudaError_t launch_decode_fused(const DevCache &c, int dtype16, const FusedPlan &fp, const void *q,
                                const void *k, const void *v, const uint8_t *types, float *part,
                                float *out, uint32_t flags, cudaStream_t st);
int fused_supported(int d, int G, int g);
int fused_warps_per_cta();
size_t fused_stage_bytes(int d, int G, size_t page_bytes, size_t pg_vscale, size_t side_entry);
size_t fused_smem_bytes(int d, int G, int g, size_t stage_bytes);
cudaError_t launch_view(const DevCache &c, int dtype16, int L, int n_q, float *K, float *V,
                        cudaStream_t st);

}  // namespace akvq
