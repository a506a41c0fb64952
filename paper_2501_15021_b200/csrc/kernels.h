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

// Persistent layer-kernel plan (k_decode_layer): per unit, the item table tab
// (P pages as K/V halves, Rc ring chunks and Sc side splits, interleaved);
// T = U * per_u items; W warps, warp w owns items [w*T/W, (w+1)*T/W) and writes
// one partial per unit it touches into slot w*maxseg + (u - first unit of w).
// Item encoding: kind (bits 0-1: 0 page (K and V halves), 2 ring chunk,
// 3 side split) | rows (bits 2-7, ring chunk) | index (bits 8-31: page, first
// ring row relative to n_q, or side split).
#ifndef AKVQ_MAX_TAB
#define AKVQ_MAX_TAB 2048
#endif
constexpr int kLyMaxTab = AKVQ_MAX_TAB;
struct LayerPlan {
  int T, W;
  int per_u;
  int P, Rc, Sc;
  int hg;               // GQA head groups per unit (virtual units u * hg + group)
  int maxseg;
  int L, n_q, nq_mod;   // nq_mod = n_q % ring slots
  int stream_only;      // AKVQ_OPT_STREAM_ONLY (profiling)
  // cost-weighted split: item k of a unit starts at cost cpre[k] (cpre[per_u] =
  // cu, the unit's cost); CT = units * cu; warp w owns the items whose start cost
  // c satisfies floor(c W / CT) == w (64-bit products; host: CT / W >= max cost)
  int cu, CT;
  int exact_logits;     // AKVQ_OPT_EXACT_LOGITS (test hook): fp32 page logits
  float sc_inv;         // 1 / Sc (side-split bounds without an integer division)
  int dev_L;            // 1: take L from DevCache::dstate (plan covers the flush period)
  int appends;          // 1: this launch appends the new token (fused step)
  int prologue;         // 1: the preceding grid does not write this cache, so the
                        // first TMA sub-loads may be issued before griddepcontrol.wait
  uint32_t tab[kLyMaxTab];
  uint16_t cpre[kLyMaxTab + 1];
};

// Decode split plan (host-computed, uniform across units).
struct DecodePlan {
  int L, n_q;
  int n_pages;           // quantized pages in use = ceil(n_q / G) (exact R: last one partial)
  int pages_per_split, n_page_splits;
  int ring_per_split, n_ring_splits;
  int n_side_splits;     // side entries are shared equally among these splits
  int S;                 // total splits of k_decode_split (ring / side / fallback pages)
  int fast;              // 1: one k_decode_layer launch (all tiers, merged in-kernel)
  LayerPlan lp;
};

cudaError_t launch_salient(const DevCache &c, const uint8_t *types, const float *colsum,
                           int L0, int top_k, cudaStream_t st);
cudaError_t launch_quantize_blocks(const DevCache &c, int dtype16, const QuantSrc &src,
                                   int block0, int nblocks, int last_block, cudaStream_t st);
// exact residual window (R26): tokens [t0, t1) quantized one at a time
cudaError_t launch_quantize_tokens(const DevCache &c, int dtype16, const QuantSrc &src, int t0,
                                   int t1, cudaStream_t st);
cudaError_t launch_ring_fill(const DevCache &c, const void *K, const void *V, int L0, int t0,
                             int t1, cudaStream_t st);
cudaError_t launch_append(const DevCache &c, const void *k, const void *v,
                          const uint8_t *types, int L, cudaStream_t st);
cudaError_t launch_state_set(const DevCache &c, int L, cudaStream_t st);
cudaError_t launch_decode(const DevCache &c, int dtype16, const DecodePlan &p, const void *q,
                          float *out, void *ws, uint32_t flags, cudaStream_t st);
cudaError_t launch_decode_layer(const DevCache &c, int dtype16, const LayerPlan &lp, const void *q,
                                const void *k, const void *v, const uint8_t *types, float *part,
                                float *out, uint32_t flags, cudaStream_t st);
cudaError_t launch_decode_gqa(const DevCache &c, int dtype16, const LayerPlan &lp, const void *q,
                              const void *k, const void *v, const uint8_t *types, float *part,
                              float *out, uint32_t flags, cudaStream_t st);
int gqa_heads(int g);
int gqa_warps_per_cta();
int gqa_ctas_per_sm();
size_t gqa_record_floats(int d);
int layer_uses_gqa(int g);
int layer_supported(int d, int G, int g);
int layer_head_groups(int g);
int layer_group_heads(int g);
int layer_warps_per_cta();
int layer_ctas_per_sm(int g);
int layer_rows_per_chunk();
int layer_rows4_per_sub();
cudaError_t launch_pivot_detect(const void *res, int n_rows, int L0, int hidden, int dtype16,
                                float tau, int n_max, float *score_ws, int32_t *pivots,
                                int32_t *counts, cudaStream_t st);
cudaError_t launch_salient_from_pivots(const DevCache &c, const int32_t *pivots,
                                       const int32_t *counts, int n_max, int units_per_row,
                                       int L0, cudaStream_t st);
cudaError_t launch_view(const DevCache &c, int dtype16, int L, int n_q, float *K, float *V,
                        cudaStream_t st);

}  // namespace akvq
