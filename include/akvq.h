/*
 * akvq.h -- C ABI of libakvq.so, the B200 (sm_100a) hot path of AKVQ-VL
 * (arXiv 2501.15021): Walsh-Hadamard rotation, attention-aware saliency,
 * 2-bit group quantize-and-pack of one attention layer's KV cache, and
 * single-query decode attention that reads the packed cache directly.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n, BJ:n =
 * BASELINE.json line n; R1..R20 = DESIGN.md section 2 readings.
 *
 * Conventions shared by every call
 *  - Plain C types only.  Pointers named dev_* / K, V, q, out, ws, types,
 *    colsum are DEVICE pointers (cudaMalloc / torch CUDA storage) unless the
 *    comment says host.  akvq_config, akvq_cache and akvq_mem_report are
 *    HOST structs owned by the caller.
 *  - Every call is asynchronous on the caller's stream (akvq_stream_t is the
 *    CUDA runtime's cudaStream_t; NULL = legacy default stream).  The
 *    library never allocates device memory and never synchronizes; the
 *    caller owns every buffer.  Asynchronous faults surface at the caller's
 *    next synchronization.
 *  - Errors are returned, never thrown.  Argument/state errors are detected
 *    on the host BEFORE any work is enqueued and leave the cache unchanged.
 *    AKVQ_ECUDA reports cudaGetLastError() after a launch.
 *  - A cache is single-writer: calls on one cache must be
 *    ordered (same stream or explicit events).  Distinct caches are
 *    independent.  Sharding across GPUs is invisible to the library: each
 *    rank builds caches for its own unit range.
 *  - Units: u = b * n_kv_heads + h (b-major).  All per-unit arrays are
 *    row-major with the unit index outermost.
 */
#ifndef AKVQ_H
#define AKVQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st *akvq_stream_t;   /* == cudaStream_t */

typedef enum {
  AKVQ_OK = 0,
  AKVQ_EINVAL = 1,        /* bad argument: NULL pointer, non-power-of-two d/G,
                             clip outside (0,1], negative sizes */
  AKVQ_EUNSUPPORTED = 2,  /* valid per the paper but not built: d not in
                             {64,128}; G not in {32,64,128} or G > d; top_k > 32;
                             PSA prompt longer than AKVQ_MAX_PSA_PROMPT         */
  AKVQ_ECAPACITY = 3,     /* buffer/workspace too small, L0 > capacity,
                             append at L == capacity                            */
  AKVQ_ESTATE = 4,        /* prefill on a non-empty cache, decode or
                             view on an empty cache                             */
  AKVQ_ECUDA = 5          /* a CUDA launch failed (cudaGetLastError)            */
} akvq_status;

typedef enum { AKVQ_TSA = 0, AKVQ_PSA = 1 } akvq_kind;        /* Table I */
typedef enum { AKVQ_BF16 = 0, AKVQ_FP16 = 1 } akvq_dtype16;   /* R13 */
/* K quantization axis: per channel over G-token blocks (R1, BJ:5, graded) or
 * per token over G-channel groups (P:246 literally). */
typedef enum { AKVQ_K_PER_CHANNEL = 0, AKVQ_K_PER_TOKEN = 1 } akvq_k_axis;

/* decode flags */
#define AKVQ_OUT_ROTATED 1u     /* return o' = sum p V^ in the rotated basis
                                   (caller folded H into W_O, R4)      */

#define AKVQ_MAX_PSA_PROMPT 49152   /* PSA top-k keeps the prompt's scores in
                                       shared memory (192 KB)                 */

/* One layer's cache configuration.  Per-channel K / per-token V (R1). */
typedef struct {
  int32_t n_units;    /* U = batch x kv heads (>= 1)                          */
  int32_t q_per_kv;   /* g = query heads per kv head (GQA), 1..16      */
  int32_t head_dim;   /* d, 64 or 128 (power of two, Eq. 7)                   */
  int32_t group;      /* G: K token-block length = V channel-group length
                         (P:408), 32/64/128, G <= d                           */
  int32_t residual;   /* R: recent window kept 16-bit, >= 0    */
  int32_t capacity;   /* max tokens per unit (prompt + decode), >= 1          */
  int32_t top_k;      /* PSA pivots, 0..32; ignored for TSA           */
  int32_t kind;       /* akvq_kind                                            */
  int32_t dtype16;    /* akvq_dtype16 of K/V/q inputs and 16-bit tiers        */
  float clip2;        /* 2-bit clip ratio, (0,1], paper 0.8           */
  float clip4;        /* 4-bit clip ratio, (0,1], paper 1.0           */
  int32_t k_axis;     /* akvq_k_axis (0 = per channel, the graded default)    */
  int32_t paged;      /* 0: the pages live in the cache buffer; 1: in a caller-
                         owned page pool shared by any number of caches, found
                         through a block table (akvq_cache_attach_pages)      */
  int32_t exact_r;    /* per-token K only (k_axis 1, else EINVAL): 1 = exactly
                         the last R tokens stay 16-bit, n_q = max(0, L - R),
                         each token quantized on its own as it leaves the
                         window ("residual" R; DESIGN R26); 0 = whole
                         G-blocks leave the window (R9).  The last page is then
                         partly filled.  Not with AKVQ_OPT_DEVICE_L.          */
} akvq_config;

/* Byte layout of the caller's cache buffer (all offsets from its base;
 * every region 256-byte aligned).  cap = capacity rounded up to G;
 * n_pages = cap / G; ng = d / G; slots = R + G.
 *
 *  pages   [U][n_pages][page_bytes]        one page = one G-token block (not in
 *                                      the buffer when cfg.paged: page p of
 *                                      unit u is pool + block_table[u][p] *
 *                                      page_bytes, akvq_cache_attach_pages):
 *            +pg_kscale  f32 [d]     K scale per channel (normalized basis);
 *                                    per token: f32 [G][ng] (same bytes)
 *            +pg_kzero   i32 [d]     K zero point per channel; per token [G][ng]
 *            +pg_kcodes  u32 [G*d/16] K codes (2 bits each, G*d/4 bytes) as
 *                                    4x4 (token x channel) tile words: word
 *                                    ((cq>>2)*G/4 + tq)*4 + (cq&3), byte b =
 *                                    channel 4cq+b, bits 2s = token 4tq+s
 *            +pg_vscale  f32 [G][ng] V scale per token and channel group
 *            +pg_vzero   i32 [G][ng]
 *            +pg_vcodes  u32 [G*d/16] V codes as tile words: word
 *                                    ((tq>>2)*d/4 + cq)*4 + (tq&3), byte b =
 *                                    token 4tq+b's S:146 byte for channels
 *                                    4cq..4cq+3 (bits 2s = channel 4cq+s)
 *  ring    [U][slots][2][d] 16-bit     recent-window rows, ORIGINAL basis
 *                                      (R10); token t lives in slot t % slots
 *  bitmask [U][bitmask_words] u32      bit t = token t salient (R2, R11, R12)
 *  side_idx [U][side_cap] i32          token index of each side entry,
 *                                      ascending token order
 *  side_cnt [U] i32                    entries in use
 *  side    [U][side_cap][side_entry_bytes]
 *            PSA: K row, V row, 16-bit, ORIGINAL basis (R10)
 *            TSA: +0 kscale f32[ng], kzero i32[ng], vscale f32[ng],
 *                 vzero i32[ng], then K codes u8[d/2], V codes u8[d/2]
 *                 (4-bit, 2 per byte, low nibble first; clip4, R11)
 *  ticket  [U * hg] u32                merge tickets of the fused decode, one
 *                                      per unit and GQA head group hg (zeroed
 *                                      at init, self-resetting)
 *  state   i32 L, u32 counter          device copy of the token count L (kept by
 *                                      prefill, append and the fused decode) and
 *                                      the fused decode's launch-exit counter
 *  umax    [U] f32 x 2                 largest |K scale| and |V scale| of the
 *                                      unit's quantized pages (normalized
 *                                      basis; zeroed at init, raised by every
 *                                      quantize launch): the decode kernel's
 *                                      fixed-point ranges
 *  side_cap = top_k (PSA) or cap (TSA).
 */
typedef struct {
  uint64_t total_bytes;
  uint64_t pages_off, page_bytes;
  uint64_t pg_kscale, pg_kzero, pg_kcodes, pg_vscale, pg_vzero, pg_vcodes;
  uint64_t ring_off, ring_unit_bytes;
  uint64_t bitmask_off;
  uint64_t side_idx_off, side_cnt_off;
  uint64_t side_off, side_entry_bytes;
  uint64_t ticket_off;
  uint64_t umax_off;
  uint64_t state_off;
  int32_t cap, n_pages, slots, bitmask_words, side_cap, ng;
} akvq_layout;

/* Caller-owned handle.  L and n_q are host mirrors of the (uniform across
 * units) token count and quantized-region length n_q = G*floor(max(0,L-R)/G)
 * (R9; max(0, L-R) with cfg.exact_r, R26); the host needs them to schedule
 * flushes without device->host syncs. */
typedef struct {
  akvq_config cfg;
  akvq_layout lay;
  void *base;          /* device buffer of lay.total_bytes bytes              */
  int32_t L;
  int32_t n_q;
  int32_t sm_count;    /* filled at init, used to size decode grids           */
  int32_t options;     /* AKVQ_OPT_* bits, 0 by default (set after init)      */
  int32_t launches;    /* kernels enqueued by the last call on this cache
                          (host counter, for launch accounting in bench.py)  */
  uint64_t last_write; /* library launch sequence number of the last launch
                          that wrote this cache (host)                        */
  void *pool;          /* paged caches: device page pool (page_bytes each)    */
  const int32_t *block_table; /* paged caches: device [U][n_pages] i32, the
                          pool page of logical page p of unit u              */
} akvq_cache;

/* akvq_cache.options: route 2-bit pages through the generic split-K kernel
 * instead of the persistent dp4a page kernel (test hook for cross-checks). */
#define AKVQ_OPT_GENERIC_PAGES 1
/* Profiling hook: the fast decode kernel streams every byte it would read
 * (same TMA pipeline) but skips all arithmetic; outputs are garbage.  Used
 * only to measure the memory pipeline's ceiling (bench.py --stream-only).
 * A separate compile-time kernel variant, built for g == 1 caches only; with
 * g > 1 the decode call fails with AKVQ_ECUDA. */
#define AKVQ_OPT_STREAM_ONLY 2
/* Profiling hooks: skip the row kernel / the page kernel entirely (outputs are
 * garbage); used to attribute the decode time (bench.py --skip-rows/pages). */
#define AKVQ_OPT_SKIP_ROWS 4
#define AKVQ_OPT_SKIP_PAGES 8
/* Test hook: every 2-bit page's logits take the fast kernel's plain fp32 path
 * (the one a page with an out-of-range zero-point bias takes) instead of the
 * fixed-point MMA; results must match the oracle the same way. */
#define AKVQ_OPT_EXACT_LOGITS 16
/* Device-resident token count: the fused decode kernel takes L from the cache
 * buffer (state region) and advances it itself, and the item table covers every
 * L of the current flush period.  The launches of akvq_decode_step then have
 * the same parameters from one step to the next until the next block flush,
 * so a step can be captured in a CUDA graph and replayed (the host mirror is
 * brought up to date with akvq_cache_advance).  Needs the fast kernels (any
 * supported d, G, q_per_kv); the generic split kernels return EUNSUPPORTED. */
#define AKVQ_OPT_DEVICE_L 32

typedef struct {      /* memory_report, host arithmetic           */
  double bytes_fp16, bytes_int4, bytes_int2, bytes_overhead;
  double effective_bits_per_element, compression_ratio_vs_fp16;
  uint64_t allocated_bytes;
} akvq_mem_report;

/* ---------------------------------------------------------------- layout */
/* Layout of a cache for cfg.  Returns AKVQ_OK or the config error. */
akvq_status akvq_cache_layout(const akvq_config *cfg, akvq_layout *out);
/* Bytes the caller must provide for one cache; 0 if cfg is invalid. */
size_t akvq_cache_bytes(const akvq_config *cfg);

/* ---------------------------------------------------------------- init */
/* cache_new: validates cfg, records dev_buf, enqueues zeroing of
 * the bitmask and side counters on `stream`; L = n_q = 0.
 * Errors: EINVAL, EUNSUPPORTED, ECAPACITY (bytes < akvq_cache_bytes). */
akvq_status akvq_cache_init(akvq_cache *c, const akvq_config *cfg, void *dev_buf,
                            size_t bytes, akvq_stream_t stream);

/* Paged caches (cfg.paged = 1, a block table as in paged KV
 * caches): attach the caller's page pool and block table.  pool: device memory
 * of page_bytes-sized pages (any number, shared by caches); block_table: device
 * i32 [U][n_pages], entry (u, p) = index of the pool page holding logical page
 * p (tokens [pG, (p+1)G)) of unit u.  The caller owns both, fills the entries
 * of every page the cache will quantize before that happens (pages fill in
 * order: page p is written when n_q passes (p+1) G, or pG with cfg.exact_r,
 * whose first token zeroes the page), and never maps one pool
 * page to two live logical pages.  Host call; no work is enqueued.
 * Errors: EINVAL (NULL, or a cache that is not paged).  Every other call on a
 * paged cache without attached pages returns ESTATE. */
akvq_status akvq_cache_attach_pages(akvq_cache *c, void *pool, const int32_t *block_table);

/* ---------------------------------------------------------------- prefill */
/* prefill: for every unit, select salient
 * tokens (TSA: types[u][t] == 1; PSA: top-k of sum_j colsum[u][j][t]), then
 * rotate (x.H_s, R5) and quantize blocks [0, n_q) -- K per channel over each
 * G-token block, V per token over G-channel groups, 2 bits, clip2 -- with
 * salient tokens moved to the side table, and copy tokens [n_q, L0) into the
 * 16-bit ring.  Sets L = L0.
 *   K, V    device [U][L0][d] 16-bit (cfg.dtype16), post-RoPE
 *   types   device [U][L0] u8 (1 = text); required for TSA, may be NULL for PSA
 *   colsum  device [U][g][L0] f32 accumulated attention column sums;
 *           required for PSA, may be NULL for TSA
 * Errors: ESTATE (L != 0), ECAPACITY (L0 > capacity), EINVAL (NULL input the
 * layer kind needs, L0 < 0), EUNSUPPORTED (PSA with L0 > AKVQ_MAX_PSA_PROMPT). */
akvq_status akvq_rotate_quantize(akvq_cache *c, const void *K, const void *V,
                                 int32_t L0, const uint8_t *types,
                                 const float *colsum, akvq_stream_t stream);

/* ---------------------------------------------------------------- append */
/* append_decode (Eq. 2): store each unit's new row in
 * ring slot L % slots, mark it salient if TSA and types[u] == 1, L += 1; if
 * L - R - n_q >= G, quantize block [n_q, n_q + G) from the ring exactly as
 * prefill would and n_q += G.  cfg.exact_r: if L - R > n_q, quantize
 * token n_q alone from the ring (K and V per token, R26) and n_q += 1.
 *   k, v   device [U][d] 16-bit;  types device [U] u8 (NULL = all vision)
 * Errors: ECAPACITY (L == capacity; nothing changes). */
akvq_status akvq_append_token(akvq_cache *c, const void *k, const void *v,
                              const uint8_t *types, akvq_stream_t stream);

/* ---------------------------------------------------------------- decode */
/* Workspace (device bytes) akvq_decode_attention needs for this cache's
 * current L (grows with L; size it for capacity via the _max variant). */
size_t akvq_decode_workspace_bytes(const akvq_cache *c);
size_t akvq_decode_workspace_bytes_max(const akvq_cache *c);

/* Single-query decode attention over the whole cache (R17):
 *   out[u][j] = softmax_t(q~ . K^_t / sqrt d) . V^  then . H unless
 *   flags & AKVQ_OUT_ROTATED, with q~ = q[u][j] . H, K^/V^ the dequantized
 *   2-bit rows, 4-bit TSA side rows, and 16-bit ring / PSA side rows.
 *   q    device [U][g][d] 16-bit;   out device [U][g][d] f32
 *   ws   device scratch of >= akvq_decode_workspace_bytes(c) bytes
 * Errors: ESTATE (L == 0), ECAPACITY (ws too small), EINVAL (NULL). */
akvq_status akvq_decode_attention(const akvq_cache *c, const void *q, float *out,
                                  void *ws, size_t ws_bytes, uint32_t flags,
                                  akvq_stream_t stream);

/* One decode step = append (Eq. 2) + attention, fused into one launch when
 * no block flush is due (akvq_append_token + akvq_decode_attention otherwise;
 * results are identical).  k, v [U][d], types [U] (NULL = vision), q
 * [U][g][d] 16-bit; out [U][g][d] f32; ws >= akvq_decode_workspace_bytes_max.
 * Errors: ECAPACITY (L == capacity or ws too small; nothing changes), EINVAL. */
akvq_status akvq_decode_step(akvq_cache *c, const void *k, const void *v,
                             const uint8_t *types, const void *q, float *out,
                             void *ws, size_t ws_bytes, uint32_t flags,
                             akvq_stream_t stream);

/* ---------------------------------------------------------------- hooks */
/* Saliency only (classify_tokens): writes bitmask bits [0, L0).
 * Test hook; akvq_rotate_quantize calls the same kernel.  Cache must be
 * empty (ESTATE) and freshly initialised. */
akvq_status akvq_select_salient(akvq_cache *c, const uint8_t *types,
                                const float *colsum, int32_t L0,
                                akvq_stream_t stream);

/* ------------------------------------------------------------- NEXT-2 */
/* Massive-activation pivot detection (SPEC detect_pivot_tokens,
 * S:317-321; R22) for n_rows residual streams:
 *   score(t) = max_c |residual[r][t][c]|, m = median over t of score,
 *   pivots[r] = tokens with score > tau * m, ordered (score desc, index asc),
 *   at most n_max (1..32); none -> [0] (attention-sink fallback).
 *   residual  device [n_rows][L0][hidden] 16-bit (dtype16)
 *   score_ws  device f32 scratch of n_rows * L0 floats
 *   pivots    device i32 [n_rows][n_max] (entries >= counts[r] untouched)
 *   counts    device i32 [n_rows] (1..n_max)
 * Errors: EINVAL (NULL, sizes < 1, tau <= 0, n_max outside 1..32),
 *         EUNSUPPORTED (L0 > AKVQ_MAX_PSA_PROMPT). */
akvq_status akvq_detect_pivots(const void *residual, int32_t n_rows, int32_t L0, int32_t hidden,
                               int32_t dtype16, float tau, int32_t n_max, float *score_ws,
                               int32_t *pivots, int32_t *counts, akvq_stream_t stream);

/* PSA prefill with explicit pivots (NEXT-2): like akvq_rotate_quantize, but
 * the salient set of unit u is pivots[u / units_per_row][0 .. counts[...]) (the
 * pivot set of its batch row, R22) instead of the column-sum top-k.
 *   pivots, counts  device, as written by akvq_detect_pivots (stride n_max)
 * Errors: as akvq_rotate_quantize; EINVAL for a TSA cache, NULL pivot
 * arrays, units_per_row < 1 or n_max > top_k (side capacity). */
akvq_status akvq_rotate_quantize_pivots(akvq_cache *c, const void *K, const void *V, int32_t L0,
                                        const int32_t *pivots, const int32_t *counts,
                                        int32_t n_max, int32_t units_per_row,
                                        akvq_stream_t stream);

/* Host bookkeeping after CUDA-graph replays of akvq_decode_step under
 * AKVQ_OPT_DEVICE_L: L += steps (the device copy was advanced by the replayed
 * kernels).  Host arithmetic only.  Errors: EINVAL (steps < 0), ECAPACITY,
 * ESTATE (the steps would have crossed a block flush, which a replay does not
 * perform). */
akvq_status akvq_cache_advance(akvq_cache *c, int32_t steps);

/* dequantized_view: K^, V^ device f32 [U][L][d] in the rotated
 * normalized basis (R5).  Test hook.  Errors: ESTATE (L == 0). */
akvq_status akvq_dequantize_view(const akvq_cache *c, float *K, float *V,
                                 akvq_stream_t stream);

/* memory_report: host arithmetic over the current L, n_q and the
 * given number of side entries per unit (host value, <= n_q; the mean over
 * units if they differ).  -1 uses min(top_k, n_q) for PSA; a TSA cache must
 * pass its text-token count (read back from the side_cnt region): -1 is
 * EINVAL there, because the count lives on the device. */
akvq_status akvq_memory_report(const akvq_cache *c, int32_t side_entries,
                               akvq_mem_report *host_out);

const char *akvq_status_str(akvq_status s);
const char *akvq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AKVQ_H */
