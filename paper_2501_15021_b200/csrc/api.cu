// api.cu -- the C ABI of libakvq.so (include/akvq.h): argument validation,
// cache layout, host mirrors of L / n_q, decode split planning and launches.
// Every entry point is asynchronous on the caller's stream, allocates no
// device memory and never synchronizes.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "akvq.h"
#include "common.cuh"
#include "kernels.h"

using namespace akvq;

namespace {

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

akvq_status check_config(const akvq_config *f) {
  if (!f) return AKVQ_EINVAL;
  if (f->n_units < 1 || f->q_per_kv < 1 || f->residual < 0 || f->capacity < 1 ||
      f->top_k < 0 || !is_pow2(f->head_dim) || !is_pow2(f->group) ||
      !(f->clip2 > 0.f && f->clip2 <= 1.f) || !(f->clip4 > 0.f && f->clip4 <= 1.f) ||
      (f->kind != AKVQ_TSA && f->kind != AKVQ_PSA) ||
      (f->dtype16 != AKVQ_BF16 && f->dtype16 != AKVQ_FP16) ||
      (f->k_axis != AKVQ_K_PER_CHANNEL && f->k_axis != AKVQ_K_PER_TOKEN) ||
      (f->paged != 0 && f->paged != 1) || (f->exact_r != 0 && f->exact_r != 1) ||
      (f->exact_r && f->k_axis != AKVQ_K_PER_TOKEN))
    return AKVQ_EINVAL;
  if ((f->head_dim != 64 && f->head_dim != 128) || f->group < 32 || f->group > 128 ||
      f->group > f->head_dim || f->q_per_kv > 16 || f->top_k > 32)
    return AKVQ_EUNSUPPORTED;
  return AKVQ_OK;
}

DevCache make_dev(const akvq_cache *c) {
  const akvq_config &f = c->cfg;
  const akvq_layout &y = c->lay;
  uint8_t *b = static_cast<uint8_t *>(c->base);
  DevCache d;
  d.pages = f.paged ? static_cast<uint8_t *>(c->pool) : b + y.pages_off;
  d.btab = f.paged ? c->block_table : nullptr;
  d.ring = reinterpret_cast<uint16_t *>(b + y.ring_off);
  d.bitmask = reinterpret_cast<uint32_t *>(b + y.bitmask_off);
  d.side_idx = reinterpret_cast<int32_t *>(b + y.side_idx_off);
  d.side_cnt = reinterpret_cast<int32_t *>(b + y.side_cnt_off);
  d.side = b + y.side_off;
  d.ticket = reinterpret_cast<uint32_t *>(b + y.ticket_off);
  d.umax = reinterpret_cast<float2 *>(b + y.umax_off);
  d.dstate = reinterpret_cast<DevCache::State *>(b + y.state_off);
  d.page_bytes = (uint32_t)y.page_bytes;
  d.pg_kscale = (uint32_t)y.pg_kscale; d.pg_kzero = (uint32_t)y.pg_kzero;
  d.pg_kcodes = (uint32_t)y.pg_kcodes; d.pg_vscale = (uint32_t)y.pg_vscale;
  d.pg_vzero = (uint32_t)y.pg_vzero; d.pg_vcodes = (uint32_t)y.pg_vcodes;
  d.side_entry = (uint32_t)y.side_entry_bytes;
  d.n_pages = y.n_pages; d.slots = y.slots; d.bm_words = y.bitmask_words;
  d.side_cap = y.side_cap;
  d.U = f.n_units; d.g = f.q_per_kv; d.d = f.head_dim; d.G = f.group; d.R = f.residual;
  d.ng = y.ng; d.kind = f.kind; d.k_axis = f.k_axis;
  d.clip2 = f.clip2; d.clip4 = f.clip4;
  d.inv_sqrt_d = (float)(1.0 / sqrt((double)f.head_dim));
  return d;
}

akvq_status cuda_status(cudaError_t e) { return e == cudaSuccess ? AKVQ_OK : AKVQ_ECUDA; }

// Quantized-region length for L tokens: whole G-blocks (R9) or, with the exact
// residual window (R26), every token but the last R.
int nq_for(const akvq_config &f, int L) {
  if (L <= f.residual) return 0;
  return f.exact_r ? L - f.residual : (L - f.residual) / f.group * f.group;
}

// Ring rows of tokens [t0, t1) as a quantize source (flush / exact-R step).
QuantSrc ring_src(const DevCache &d) {
  QuantSrc src;
  src.K = d.ring;
  src.V = d.ring + d.d;
  src.unit_stride = (size_t)d.slots * 2 * d.d;
  src.tok_stride = (size_t)2 * d.d;
  src.ring_slots = d.slots;
  return src;
}

// Per-stream record of the library's last kernel launch on that stream and the
// cache buffer it wrote (NULL: it wrote no cache).  The decode kernel is
// launched with programmatic dependent launch, so it may start while the
// PRECEDING kernel of its stream is still running; it may therefore prefetch
// cache pages before griddepcontrol.wait only if that preceding kernel is known
// not to write this cache.  Kernels on other streams are ordered by the
// caller's events (full dependencies), so only the same stream matters.  An
// unknown stream (never seen, or evicted from the table) disables the prefetch.
std::atomic<unsigned long long> g_seq{0};
std::mutex g_stream_mu;
struct StreamLast {
  cudaStream_t s;
  const void *wrote;
  bool used;
};
StreamLast g_stream_last[64];
int g_stream_next = 0;

void note_launch(akvq_cache *c, cudaStream_t s, bool wrote) {
  if (wrote) c->last_write = g_seq.fetch_add(1) + 1;
  std::lock_guard<std::mutex> lk(g_stream_mu);
  for (auto &e : g_stream_last)
    if (e.used && e.s == s) { e.wrote = wrote ? c->base : nullptr; return; }
  StreamLast &e = g_stream_last[g_stream_next];
  g_stream_next = (g_stream_next + 1) % 64;
  e.s = s; e.wrote = wrote ? c->base : nullptr; e.used = true;
}
// true if the last library launch on s is known and did not write c
bool prefetch_safe(const akvq_cache *c, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_stream_mu);
  for (auto &e : g_stream_last)
    if (e.used && e.s == s) return e.wrote != c->base;
  return false;
}

// Persistent-grid sizes (CTAs per SM) of the two decode kernels; tuning
// overrides AKVQ_ROW_CTAS / AKVQ_PG_CTAS are read once (experiments only).
int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}
int min_items_per_warp() {
  static const int v = env_int("AKVQ_MIN_ITEMS", 4);
  return v < 1 ? 1 : v;
}
int pg_ctas_override() {
  static const int v = env_int("AKVQ_PG_CTAS", 0);
  return v;
}

// build_tab = false: sizes only (workspace queries), the item table is not filled
DecodePlan plan_decode(const akvq_cache *c, int L, int n_q, bool build_tab = true) {
  const akvq_config &f = c->cfg;
  DecodePlan p;
  p.L = L;
  p.n_q = n_q;
  p.n_pages = (n_q + f.group - 1) / f.group;         // exact R: the last page partial
  const int sms = c->sm_count > 0 ? c->sm_count : 148;
  const long target = 4L * sms;                       // CTAs to keep every SM busy
  long pps = ((long)f.n_units * p.n_pages + target - 1) / target;
  if (pps < 1) pps = 1;
  if (pps > p.n_pages) pps = p.n_pages > 0 ? p.n_pages : 1;
  p.pages_per_split = (int)pps;
  p.n_page_splits = p.n_pages > 0 ? (p.n_pages + (int)pps - 1) / (int)pps : 0;
  p.ring_per_split = 128;
  p.n_ring_splits = (L - n_q + p.ring_per_split - 1) / p.ring_per_split;
  if (f.kind == AKVQ_PSA) {
    p.n_side_splits = (f.top_k > 0 && n_q > 0) ? 1 : 0;
  } else {
    const int bound = n_q;                            // side entries <= n_q
    p.n_side_splits = bound > 0 ? (bound + 511) / 512 : 0;
    if (p.n_side_splits > 8) p.n_side_splits = 8;
  }
  // fast path: ONE persistent launch of k_decode_layer over every tier (pages,
  // ring, side rows interleaved per unit), the new token appended in-kernel;
  // the writer of each unit's last segment merges it and writes the output.
  p.fast = 0;
  memset(&p.lp, 0, offsetof(LayerPlan, tab));
  p.lp.per_u = 1;
  // (the single-pass GQA kernel has no per-token-K variant: the generic kernels
  // serve that combination)
  if (!(c->options & AKVQ_OPT_GENERIC_PAGES) &&
      layer_supported(f.head_dim, f.group, f.q_per_kv) &&
      !(layer_uses_gqa(f.q_per_kv) && f.k_axis == AKVQ_K_PER_TOKEN)) {
    p.fast = 1;
    LayerPlan &lp = p.lp;
    const int rows = layer_rows_per_chunk();
    lp.L = L;
    lp.n_q = n_q;
    lp.P = p.n_pages;
    lp.Rc = (L - n_q + rows - 1) / rows;
    lp.dev_L = (c->options & AKVQ_OPT_DEVICE_L) ? 1 : 0;
    if (lp.dev_L) {   // the ring chunks of the whole flush period: L - n_q <= R + G - 1
      const int span = f.residual + f.group - 1 > L - n_q ? f.residual + f.group - 1 : L - n_q;
      lp.Rc = (span + rows - 1) / rows;
    }
    if (f.kind == AKVQ_PSA) {
      lp.Sc = (f.top_k > 0 && n_q > 0) ? (f.top_k + rows - 1) / rows : 0;   // <= rows each
    } else {
#ifndef AKVQ_CSIDE_DIV
#define AKVQ_CSIDE_DIV 1024   // side splits of a TSA layer: one per 1024 tokens of n_q (measured, r02z3)
#endif
      lp.Sc = n_q > 0 ? (n_q + AKVQ_CSIDE_DIV - 1) / AKVQ_CSIDE_DIV : 0;    // text rows <= n_q
      if (lp.Sc > 8) lp.Sc = 8;
      // the GQA kernel takes its rows one at a time for all heads (~ a page's work
      // per dozen rows): many small splits keep the long text tiers balanced
      if (layer_uses_gqa(f.q_per_kv)) {
        lp.Sc = n_q > 0 ? (n_q + 63) / 64 : 0;
        if (lp.Sc > 512) lp.Sc = 512;
      }
    }
    if (c->options & AKVQ_OPT_SKIP_ROWS) lp.Rc = lp.Sc = 0;       // profiling hooks
    if (c->options & AKVQ_OPT_SKIP_PAGES) lp.P = 0;
    lp.per_u = lp.P + lp.Rc + lp.Sc;
    lp.sc_inv = lp.Sc > 0 ? 1.0f / (float)lp.Sc : 0.f;
    lp.nq_mod = n_q % c->lay.slots;
    if (lp.per_u > kLyMaxTab) {           // beyond the item table: generic kernels
      p.fast = 0;
      lp.per_u = 1;
    } else if (build_tab) {               // interleave rows between pages (Bresenham)
      const int NR = lp.Rc + lp.Sc, n_ring = lp.dev_L ? lp.Rc * rows : L - n_q;   // DEVICE_L: the period's span
      int k = 0, r = 0;
      auto row_item = [&](int ri) -> uint32_t {
        if (ri < lp.Rc) {
          const int a = ri * rows, n = n_ring - a < rows ? n_ring - a : rows;
          return 2u | ((uint32_t)n << 2) | ((uint32_t)a << 8);
        }
        return 3u | ((uint32_t)(ri - lp.Rc) << 8);
      };
      for (int pg = 0; pg < lp.P; ++pg) {
        const int thr = (int)((long long)pg * NR / lp.P);
        while (r < thr) lp.tab[k++] = row_item(r++);
        lp.tab[k++] = 0u | ((uint32_t)pg << 8);
      }
      while (r < NR) lp.tab[k++] = row_item(r++);
    }
    // item costs (relative time; profiles/r01_final_summary.md): a page (two 5 KB
    // sub-loads of MMA work), a ring chunk of 8 16-bit rows and a PSA side split,
    // a TSA side split (up to 32 4-bit rows each pass)
#ifndef AKVQ_CPAGE
#define AKVQ_CPAGE 7
#endif
#ifndef AKVQ_CROWS
#define AKVQ_CROWS 2
#endif
    const int c_page = AKVQ_CPAGE, c_rows = AKVQ_CROWS,
              c_side = f.kind == AKVQ_TSA ? (layer_uses_gqa(f.q_per_kv) ? 3 : 6) : 2;
    lp.cu = lp.P * c_page + lp.Rc * c_rows + lp.Sc * c_side;   // <= 2048 * 7 < 2^16
    if (build_tab && lp.per_u <= kLyMaxTab) {
      int acc = 0;
      lp.cpre[0] = 0;
      for (int j = 0; j < lp.per_u; ++j) {
        const uint32_t kd = lp.tab[j] & 3u;
        acc += kd == 0 ? c_page : (kd == 2 ? c_rows : c_side);
        lp.cpre[j + 1] = (uint16_t)acc;
      }
    }
    lp.hg = layer_head_groups(f.q_per_kv);
    if (p.fast && lp.per_u > 0) {
      const long long T = (long long)f.n_units * lp.hg * lp.per_u;
      const long long CT = (long long)f.n_units * lp.hg * lp.cu;
      const bool gq = layer_uses_gqa(f.q_per_kv);
      const int ctas = pg_ctas_override() > 0 ? pg_ctas_override()
                       : (gq ? gqa_ctas_per_sm() : layer_ctas_per_sm(layer_group_heads(f.q_per_kv)));
      const long long wmax = (long long)sms * ctas * (gq ? gqa_warps_per_cta() : layer_warps_per_cta());
      if (CT >= (1LL << 31) || T >= (1LL << 31)) {   // beyond the plan's 32-bit counters
        p.fast = 0;
        lp.per_u = 1;
        p.S = p.n_page_splits + p.n_ring_splits + p.n_side_splits;
        return p;
      }
      lp.T = (int)T;
      // at least min_items items per warp: fewer segments per unit to merge and
      // fewer tickets when the layer is small (W = T would give one item each)
      const long long wmin_items = (T + min_items_per_warp() - 1) / min_items_per_warp();
      long long W = wmin_items < wmax ? wmin_items : wmax;
      const int cmax = c_page > c_side ? c_page : c_side;
      if (W > CT / cmax) W = CT / cmax;                   // every warp gets >= 1 item
      lp.W = (int)(W < 1 ? 1 : W);
      lp.CT = (int)CT;
      // units one warp can touch: its cost share spans <= share / (cost of the
      // cheapest unit) + 2 units
      const long long share = (CT + lp.W - 1) / lp.W;
      lp.maxseg = (int)(share / (lp.cu > 0 ? lp.cu : 1) + 2);
    } else {
      lp.per_u = 1;
    }
    lp.stream_only = (c->options & AKVQ_OPT_STREAM_ONLY) ? 1 : 0;
    lp.exact_logits = (c->options & AKVQ_OPT_EXACT_LOGITS) ? 1 : 0;
    if (p.fast) p.n_page_splits = p.n_ring_splits = p.n_side_splits = 0;
  }
  p.S = p.n_page_splits + p.n_ring_splits + p.n_side_splits;
  return p;
}

size_t ws_bytes_for(const akvq_cache *c, const DecodePlan &p) {
  const size_t g = c->cfg.q_per_kv, d = c->cfg.head_dim;
  if (p.fast) {   // NH heads per record: [o_org][o_rot][m][l] (g <= 2) or [o_rot][m][l] (GQA)
    const size_t nh = (size_t)layer_group_heads((int)g);
    const size_t rec = layer_uses_gqa((int)g) ? gqa_record_floats((int)d) : 2 * d + 4;
    return (size_t)p.lp.W * p.lp.maxseg * nh * rec * sizeof(float);
  }
  return (size_t)c->cfg.n_units * p.S * g * (d + 2) * sizeof(float);
}

// Fast-path launch: one k_decode_layer (+ append when k != NULL).
akvq_status launch_fast(const akvq_cache *c, DecodePlan &p, const void *q, const void *k,
                        const void *v, const uint8_t *types, float *out, void *ws,
                        uint32_t flags, cudaStream_t s) {
  const DevCache d = make_dev(c);
  if (p.lp.T <= 0) return AKVQ_OK;                  // nothing to launch
  const_cast<akvq_cache *>(c)->launches += 1;
  // prologue prefetch: only if the preceding kernel of this stream does not
  // write this cache (the new row of a fused step is patched in after the wait)
  // (never under DEVICE_L: a replayed graph may run this launch right after the
  // same cache's previous step, whatever preceded it when it was recorded)
  p.lp.prologue = prefetch_safe(c, s) && !(c->options & (AKVQ_OPT_STREAM_ONLY | AKVQ_OPT_DEVICE_L)) ? 1 : 0;
  p.lp.appends = k != nullptr ? 1 : 0;
  const cudaError_t e =
      layer_uses_gqa(c->cfg.q_per_kv)
          ? launch_decode_gqa(d, c->cfg.dtype16, p.lp, q, k, v, types, static_cast<float *>(ws), out, flags, s)
          : launch_decode_layer(d, c->cfg.dtype16, p.lp, q, k, v, types, static_cast<float *>(ws), out, flags, s);
  // the fused step appends (writes the ring); a plain decode writes only its
  // self-resetting tickets, which no prologue reads
  note_launch(const_cast<akvq_cache *>(c), s, k != nullptr);
  return cuda_status(e);
}

}  // namespace

extern "C" {

akvq_status akvq_cache_layout(const akvq_config *f, akvq_layout *y) {
  const akvq_status st = check_config(f);
  if (st != AKVQ_OK) return st;
  if (!y) return AKVQ_EINVAL;
  memset(y, 0, sizeof(*y));
  const uint64_t U = f->n_units, d = f->head_dim, G = f->group;
  const uint64_t ng = d / G;
  y->cap = (int32_t)((f->capacity + G - 1) / G * G);
  y->n_pages = (int32_t)(y->cap / G);
  y->slots = (int32_t)(f->residual + G);
  y->bitmask_words = y->cap / 32;
  y->side_cap = f->kind == AKVQ_PSA ? f->top_k : y->cap;
  y->ng = (int32_t)ng;
  uint64_t o = 0;
  y->pg_kscale = o; o = align_up(o + 4 * d, 16);
  y->pg_kzero = o;  o = align_up(o + 4 * d, 16);
  y->pg_kcodes = o; o = align_up(o + G * d / 4, 16);
  y->pg_vscale = o; o = align_up(o + 4 * G * ng, 16);
  y->pg_vzero = o;  o = align_up(o + 4 * G * ng, 16);
  y->pg_vcodes = o; o = align_up(o + G * d / 4, 16);
  y->page_bytes = align_up(o, 128);
  uint64_t t = 0;
  y->pages_off = t;    t = align_up(t + (f->paged ? 0 : U * y->n_pages * y->page_bytes), 256);
  y->ring_unit_bytes = (uint64_t)y->slots * 2 * d * 2;
  y->ring_off = t;     t = align_up(t + U * y->ring_unit_bytes, 256);
  y->bitmask_off = t;  t = align_up(t + U * y->bitmask_words * 4, 256);
  y->side_idx_off = t; t = align_up(t + U * y->side_cap * 4, 256);
  y->side_cnt_off = t; t = align_up(t + U * 4, 256);
  y->side_entry_bytes = f->kind == AKVQ_PSA ? 4 * d : align_up(d + 16 * ng, 16);
  y->side_off = t;     t = align_up(t + U * y->side_cap * y->side_entry_bytes, 256);
  // one merge ticket per virtual unit of the decode kernel (unit x GQA head group)
  y->ticket_off = t;   t = align_up(t + U * (uint64_t)layer_head_groups(f->q_per_kv) * 4, 256);
  // per unit: the largest |K scale| and |V scale| stored so far (the decode
  // kernel's fixed-point ranges; maintained by the quantize kernel)
  y->umax_off = t;     t = align_up(t + U * 8, 256);
  // device token count L and the fused decode's launch-exit counter
  y->state_off = t;    t = align_up(t + 16, 256);
  y->total_bytes = t;
  return AKVQ_OK;
}

size_t akvq_cache_bytes(const akvq_config *f) {
  akvq_layout y;
  return akvq_cache_layout(f, &y) == AKVQ_OK ? (size_t)y.total_bytes : 0;
}

akvq_status akvq_cache_init(akvq_cache *c, const akvq_config *f, void *dev_buf, size_t bytes,
                            akvq_stream_t stream) {
  if (!c || !f || !dev_buf) return AKVQ_EINVAL;
  akvq_layout y;
  const akvq_status st = akvq_cache_layout(f, &y);
  if (st != AKVQ_OK) return st;
  if (bytes < y.total_bytes) return AKVQ_ECAPACITY;
  memset(c, 0, sizeof(*c));
  c->cfg = *f;
  c->lay = y;
  c->base = dev_buf;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  c->sm_count = sms;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t *b = static_cast<uint8_t *>(dev_buf);
  cudaError_t e = cudaMemsetAsync(b + y.bitmask_off, 0, (size_t)f->n_units * y.bitmask_words * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(b + y.side_cnt_off, 0, (size_t)f->n_units * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(b + y.ticket_off, 0, y.total_bytes - y.ticket_off, s);
  if (e == cudaSuccess && y.side_cap > 0)
    e = cudaMemsetAsync(b + y.side_idx_off, 0xff, (size_t)f->n_units * y.side_cap * 4, s);
  note_launch(c, s, true);
  return cuda_status(e);
}

akvq_status akvq_select_salient(akvq_cache *c, const uint8_t *types, const float *colsum,
                                int32_t L0, akvq_stream_t stream) {
  if (!c || !c->base || L0 < 0) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  if (c->L != 0) return AKVQ_ESTATE;
  if (L0 > c->cfg.capacity) return AKVQ_ECAPACITY;
  if (L0 == 0) return AKVQ_OK;
  if (c->cfg.kind == AKVQ_TSA && !types) return AKVQ_EINVAL;
  if (c->cfg.kind == AKVQ_PSA) {
    if (!colsum) return AKVQ_EINVAL;
    if (L0 > AKVQ_MAX_PSA_PROMPT) return AKVQ_EUNSUPPORTED;
  }
  const DevCache d = make_dev(c);
  note_launch(c, reinterpret_cast<cudaStream_t>(stream), true);
  return cuda_status(launch_salient(d, types, colsum, L0, c->cfg.top_k,
                                    reinterpret_cast<cudaStream_t>(stream)));
}

static akvq_status quantize_prompt(akvq_cache *c, const void *K, const void *V, int32_t L0,
                                   akvq_stream_t stream);

akvq_status akvq_rotate_quantize(akvq_cache *c, const void *K, const void *V, int32_t L0,
                                 const uint8_t *types, const float *colsum,
                                 akvq_stream_t stream) {
  if (!c || !c->base || L0 < 0) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  if (c->L != 0) return AKVQ_ESTATE;
  if (L0 > c->cfg.capacity) return AKVQ_ECAPACITY;
  if (L0 > 0 && (!K || !V)) return AKVQ_EINVAL;
  akvq_status st = akvq_select_salient(c, types, colsum, L0, stream);
  if (st != AKVQ_OK) return st;
  c->launches = (c->cfg.kind == AKVQ_TSA || c->cfg.top_k > 0) && L0 > 0 ? 1 : 0;
  return quantize_prompt(c, K, V, L0, stream);
}

akvq_status akvq_rotate_quantize_pivots(akvq_cache *c, const void *K, const void *V, int32_t L0,
                                        const int32_t *pivots, const int32_t *counts,
                                        int32_t n_max, int32_t units_per_row,
                                        akvq_stream_t stream) {
  if (!c || !c->base || L0 < 0 || !pivots || !counts || units_per_row < 1 || n_max < 1)
    return AKVQ_EINVAL;
  if (c->cfg.kind != AKVQ_PSA || n_max > c->cfg.top_k) return AKVQ_EINVAL;
  if (c->L != 0) return AKVQ_ESTATE;
  if (L0 > c->cfg.capacity) return AKVQ_ECAPACITY;
  if (L0 > 0 && (!K || !V)) return AKVQ_EINVAL;
  c->launches = 0;
  if (L0 > 0) {
    const DevCache d = make_dev(c);
    if (launch_salient_from_pivots(d, pivots, counts, n_max, units_per_row, L0,
                                   reinterpret_cast<cudaStream_t>(stream)) != cudaSuccess)
      return AKVQ_ECUDA;
    note_launch(c, reinterpret_cast<cudaStream_t>(stream), true);
    c->launches = 1;
  }
  return quantize_prompt(c, K, V, L0, stream);
}

akvq_status akvq_detect_pivots(const void *residual, int32_t n_rows, int32_t L0, int32_t hidden,
                               int32_t dtype16, float tau, int32_t n_max, float *score_ws,
                               int32_t *pivots, int32_t *counts, akvq_stream_t stream) {
  if (!residual || !score_ws || !pivots || !counts || n_rows < 1 || L0 < 1 || hidden < 1 ||
      !(tau > 0.f) || n_max < 1 || n_max > 32 ||
      (dtype16 != AKVQ_BF16 && dtype16 != AKVQ_FP16))
    return AKVQ_EINVAL;
  if (L0 > AKVQ_MAX_PSA_PROMPT) return AKVQ_EUNSUPPORTED;
  return cuda_status(launch_pivot_detect(residual, n_rows, L0, hidden, dtype16, tau, n_max,
                                         score_ws, pivots, counts,
                                         reinterpret_cast<cudaStream_t>(stream)));
}

static akvq_status quantize_prompt(akvq_cache *c, const void *K, const void *V, int32_t L0,
                                   akvq_stream_t stream) {
  const akvq_config &f = c->cfg;
  const int n_q = nq_for(f, L0);                     // R9 / R26
  const DevCache d = make_dev(c);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  QuantSrc src;
  src.K = static_cast<const uint16_t *>(K);
  src.V = static_cast<const uint16_t *>(V);
  src.unit_stride = (size_t)L0 * f.head_dim;
  src.tok_stride = f.head_dim;
  src.ring_slots = 0;
  const int nb = n_q / f.group;
  cudaError_t e = launch_quantize_blocks(d, f.dtype16, src, 0, nb, nb - 1, s);
  // exact R: the tokens of the partial last page, one at a time (R26)
  if (e == cudaSuccess) e = launch_quantize_tokens(d, f.dtype16, src, nb * f.group, n_q, s);
  if (e == cudaSuccess) e = launch_ring_fill(d, K, V, L0, n_q, L0, s);
  if (e == cudaSuccess) e = launch_state_set(d, L0, s);    // device copy of L
  c->launches += (nb > 0) + (n_q > nb * f.group) + (L0 > n_q) + 1;
  note_launch(c, s, true);
  if (e != cudaSuccess) return AKVQ_ECUDA;
  c->L = L0;
  c->n_q = n_q;
  return AKVQ_OK;
}

static akvq_status append_impl(akvq_cache *c, const void *k, const void *v, const uint8_t *types,
                        akvq_stream_t stream) {
  if (!c || !c->base || !k || !v) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  const akvq_config &f = c->cfg;
  if (c->L >= f.capacity) return AKVQ_ECAPACITY;
  const DevCache d = make_dev(c);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = launch_append(d, k, v, types, c->L, s);
  if (e != cudaSuccess) return AKVQ_ECUDA;
  c->launches += 1;
  note_launch(c, s, true);
  c->L += 1;
  if (f.exact_r && c->L - f.residual > c->n_q) {      // token n_q leaves the window (R26)
    e = launch_quantize_tokens(d, f.dtype16, ring_src(d), c->n_q, c->n_q + 1, s);
    if (e != cudaSuccess) return AKVQ_ECUDA;
    c->launches += 1;
    note_launch(c, s, true);
    c->n_q += 1;
  } else if (!f.exact_r && c->L - f.residual - c->n_q >= f.group) {   // block leaves the window (R9)
    const int j = c->n_q / f.group;
    e = launch_quantize_blocks(d, f.dtype16, ring_src(d), j, 1, j, s);
    if (e != cudaSuccess) return AKVQ_ECUDA;
    c->launches += 1;
    note_launch(c, s, true);
    c->n_q += f.group;
  }
  return AKVQ_OK;
}

akvq_status akvq_append_token(akvq_cache *c, const void *k, const void *v,
                              const uint8_t *types, akvq_stream_t stream) {
  if (c) c->launches = 0;
  return append_impl(c, k, v, types, stream);
}

size_t akvq_decode_workspace_bytes(const akvq_cache *c) {
  if (!c) return 0;
  return ws_bytes_for(c, plan_decode(c, c->L, c->n_q, false));
}

size_t akvq_decode_workspace_bytes_max(const akvq_cache *c) {
  if (!c) return 0;
  size_t best = 0;
  const akvq_config &f = c->cfg;
  for (int L = 1; L <= f.capacity; ++L) {     // plans are cheap; the size is not monotone in L
    const size_t b = ws_bytes_for(c, plan_decode(c, L, nq_for(f, L), false));
    if (b > best) best = b;
  }
  const size_t b = ws_bytes_for(c, plan_decode(c, f.capacity, nq_for(f, f.capacity), false));
  return b > best ? b : best;
}

static akvq_status decode_impl(const akvq_cache *c, const void *q, float *out, void *ws,
                        size_t ws_bytes, uint32_t flags, akvq_stream_t stream) {
  if (!c || !c->base || !q || !out || !ws) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  if (c->L == 0) return AKVQ_ESTATE;
  DecodePlan p = plan_decode(c, c->L, c->n_q);
  if (ws_bytes < ws_bytes_for(c, p)) return AKVQ_ECAPACITY;
  const DevCache d = make_dev(c);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if ((c->options & AKVQ_OPT_DEVICE_L) && c->cfg.exact_r) return AKVQ_EUNSUPPORTED;
  if (p.fast) return launch_fast(c, p, q, nullptr, nullptr, nullptr, out, ws, flags, s);
  if (c->options & AKVQ_OPT_DEVICE_L) return AKVQ_EUNSUPPORTED;   // generic kernels use the host L
  const_cast<akvq_cache *>(c)->launches += 2;         // split + combine
  const cudaError_t e = launch_decode(d, c->cfg.dtype16, p, q, out, ws, flags, s);
  note_launch(const_cast<akvq_cache *>(c), s, false);
  return cuda_status(e);
}

akvq_status akvq_decode_attention(const akvq_cache *c, const void *q, float *out, void *ws,
                                  size_t ws_bytes, uint32_t flags, akvq_stream_t stream) {
  if (c) const_cast<akvq_cache *>(c)->launches = 0;
  return decode_impl(c, q, out, ws, ws_bytes, flags, stream);
}

akvq_status akvq_decode_step(akvq_cache *c, const void *k, const void *v, const uint8_t *types,
                             const void *q, float *out, void *ws, size_t ws_bytes, uint32_t flags,
                             akvq_stream_t stream) {
  if (!c || !c->base || !k || !v || !q || !out || !ws) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  c->launches = 0;
  const akvq_config &f = c->cfg;
  if (c->L >= f.capacity) return AKVQ_ECAPACITY;
  const int L1 = c->L + 1;
  if ((c->options & AKVQ_OPT_DEVICE_L) && f.exact_r) return AKVQ_EUNSUPPORTED;
  // exact R (R26): token n_q leaves the window at this step; it is quantized
  // from the ring before the fused launch (it does not depend on the new token).
  // With R = 0 the leaving token IS the new one (not in the ring yet): that step
  // takes the unfused path (append, then quantize it from the ring, then decode).
  const bool ex0 = f.exact_r && f.residual == 0;
  const bool leave1 = f.exact_r && !ex0 && L1 - f.residual > c->n_q;
  const bool flush = (!f.exact_r && L1 - f.residual - c->n_q >= f.group) || ex0;
  DecodePlan p = plan_decode(c, L1, flush ? c->n_q + (ex0 ? 1 : f.group) : c->n_q + (leave1 ? 1 : 0));
  if (ws_bytes < ws_bytes_for(c, p)) return AKVQ_ECAPACITY;
  if (leave1) {
    const DevCache d = make_dev(c);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (launch_quantize_tokens(d, f.dtype16, ring_src(d), c->n_q, c->n_q + 1, s) != cudaSuccess)
      return AKVQ_ECUDA;
    note_launch(c, s, true);
    c->n_q += 1;
  }
  const int pre = leave1 ? 1 : 0;
  if (flush || !p.fast || p.lp.T <= 0) {   // flush step (every G tokens) or generic path
    akvq_status st = append_impl(c, k, v, types, stream);
    if (st != AKVQ_OK) return st;
    st = decode_impl(c, q, out, ws, ws_bytes, flags, stream);
    c->launches += pre;
    return st;
  }
  const akvq_status st = launch_fast(c, p, q, k, v, types, out, ws, flags,
                                     reinterpret_cast<cudaStream_t>(stream));
  if (st != AKVQ_OK) return st;
  c->launches += pre;
  c->L = L1;
  return AKVQ_OK;
}

akvq_status akvq_cache_attach_pages(akvq_cache *c, void *pool, const int32_t *block_table) {
  if (!c || !pool || !block_table || !c->cfg.paged) return AKVQ_EINVAL;
  c->pool = pool;
  c->block_table = block_table;
  return AKVQ_OK;
}

akvq_status akvq_cache_advance(akvq_cache *c, int32_t steps) {
  if (!c || steps < 0) return AKVQ_EINVAL;
  const akvq_config &f = c->cfg;
  if (c->L + steps > f.capacity) return AKVQ_ECAPACITY;
  // no block may have left the window in between (the replayed launches do not flush)
  if (c->L + steps - f.residual - c->n_q >= (f.exact_r ? 1 : f.group)) return AKVQ_ESTATE;
  c->L += steps;
  return AKVQ_OK;
}

akvq_status akvq_dequantize_view(const akvq_cache *c, float *K, float *V, akvq_stream_t stream) {
  if (!c || !c->base || !K || !V) return AKVQ_EINVAL;
  if (c->cfg.paged && !c->pool) return AKVQ_ESTATE;   // pages not attached
  if (c->L == 0) return AKVQ_ESTATE;
  const DevCache d = make_dev(c);
  return cuda_status(launch_view(d, c->cfg.dtype16, c->L, c->n_q, K, V,
                                 reinterpret_cast<cudaStream_t>(stream)));
}

// memory_report: bytes per tier over the current contents.
//  16-bit: ring tokens [n_q, L) and PSA side rows, 2 B/element;
//  4-bit : TSA side rows, 0.5 B/element + 8 B per group (scale, zero);
//  2-bit : the quantized region [n_q) minus side rows, 0.25 B/element;
//  overhead: K meta 8 B per channel per block, V meta 8 B per group per token.
// The 1-bit-per-token salient bitmask is not counted (allocated_bytes is).
akvq_status akvq_memory_report(const akvq_cache *c, int32_t side_entries, akvq_mem_report *r) {
  if (!c || !r) return AKVQ_EINVAL;
  const akvq_config &f = c->cfg;
  const double U = f.n_units, d = f.head_dim, G = f.group, ng = d / G;
  int se = side_entries;
  if (se < 0) {
    // PSA: the pivot count is bounded by top_k; TSA: the text-token count lives
    // on the device only (side_cnt region), so the caller must pass it
    if (f.kind != AKVQ_PSA) return AKVQ_EINVAL;
    se = f.top_k < c->n_q ? f.top_k : c->n_q;
  }
  if (se > c->n_q) return AKVQ_EINVAL;
  const double ring = (double)(c->L - c->n_q);
  const double quant = (double)c->n_q - se;
  memset(r, 0, sizeof(*r));
  r->bytes_fp16 = U * 2 * d * 2 * (ring + (f.kind == AKVQ_PSA ? se : 0));
  r->bytes_int4 = f.kind == AKVQ_TSA ? U * se * 2 * (d * 0.5 + 8 * ng) : 0;
  r->bytes_int2 = U * quant * 2 * d * 0.25;
  r->bytes_overhead = U * ((double)c->n_q / G * d * 8 + (double)c->n_q * ng * 8);
  const double total = r->bytes_fp16 + r->bytes_int4 + r->bytes_int2 + r->bytes_overhead;
  const double elems = U * (double)c->L * 2 * d;
  r->effective_bits_per_element = elems > 0 ? 8 * total / elems : 0;
  r->compression_ratio_vs_fp16 = elems > 0 ? 16.0 / r->effective_bits_per_element : 1.0;
  r->allocated_bytes = c->lay.total_bytes;
  return AKVQ_OK;
}

const char *akvq_status_str(akvq_status s) {
  switch (s) {
    case AKVQ_OK: return "ok";
    case AKVQ_EINVAL: return "invalid argument";
    case AKVQ_EUNSUPPORTED: return "unsupported configuration";
    case AKVQ_ECAPACITY: return "capacity exceeded";
    case AKVQ_ESTATE: return "invalid cache state";
    case AKVQ_ECUDA: return "CUDA launch error";
  }
  return "unknown status";
}

const char *akvq_version(void) { return "akvq-b200 0.1 (sm_100a)"; }

}  // extern "C"
