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

// Persistent page-kernel plan: T = U * n_pages flattened (unit, page) items,
// W warps each owning items [w*T/W, (w+1)*T/W); a warp writes one partial per
// unit it touches into slot w*maxseg + (u - first unit of w).
struct PagePlan {
  long long T;
  long long W;
  int n_pages;
  int maxseg;
  int stream_only;      // AKVQ_OPT_STREAM_ONLY (profiling)
};

// Persistent row-kernel plan: per unit, n_ring_chunks items of 16 ring tokens
// then n_side_splits items sharing the unit's side entries; same segment /
// partial-slot scheme as PagePlan (partials hold o_org and o_rot).
struct RowPlan {
  long long T;
  long long W;
  int items_per_unit;
  int n_ring_chunks;
  int n_side_splits;
  int maxseg;
  int L, n_q;
  int stream_only;      // AKVQ_OPT_STREAM_ONLY (profiling)
};

// Decode split plan (host-computed, uniform across units).
struct DecodePlan {
  int L, n_q;
  int n_pages;           // quantized pages in use = n_q / G
  int pages_per_split, n_page_splits;
  int ring_per_split, n_ring_splits;
  int n_side_splits;     // side entries are shared equally among these splits
  int S;                 // total splits of k_decode_split (ring / side / fallback pages)
  int fast;              // 1: k_decode_rows then k_decode_pages (PDL), merged in-kernel
  PagePlan pp;
  RowPlan rp;
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
cudaError_t launch_decode_rows(const DevCache &c, int dtype16, const RowPlan &rp, const PagePlan &pp,
                               const void *q, const void *k, const void *v, const uint8_t *types,
                               float *rw_part, const float *pg_part, float *out, uint32_t flags,
                               cudaStream_t st);
cudaError_t launch_decode_pages(const DevCache &c, int dtype16, const PagePlan &pp,
                                const RowPlan &rp, const void *q, float *pg_part,
                                const float *rw_part, float *out, uint32_t flags, cudaStream_t st);
int pages_fast_supported(int d, int G, int g);
int pages_warps_per_cta();
int rows_chunk();
int rows_warps_per_cta();
cudaError_t launch_view(const DevCache &c, int dtype16, int L, int n_q, float *K, float *V,
                        cudaStream_t st);

}  // namespace akvq
