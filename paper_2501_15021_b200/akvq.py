"""Thin ctypes binding of libakvq.so (include/akvq.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA library; this module only turns
torch tensors into device pointers and the current torch stream into a
cudaStream_t.  There is no CPU fallback: if libakvq.so is missing or fails to
load, every call raises.  PyTorch is plumbing here (device memory, streams).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AKVQ_LIB") or os.path.join(_PKG, "libakvq.so")   # AKVQ_LIB: experiments only

AKVQ_OK, AKVQ_EINVAL, AKVQ_EUNSUPPORTED, AKVQ_ECAPACITY, AKVQ_ESTATE, AKVQ_ECUDA = range(6)
AKVQ_TSA, AKVQ_PSA = 0, 1
AKVQ_BF16, AKVQ_FP16 = 0, 1
AKVQ_OUT_ROTATED = 1
AKVQ_OPT_GENERIC_PAGES = 1
AKVQ_OPT_STREAM_ONLY = 2
AKVQ_OPT_SKIP_ROWS = 4
AKVQ_OPT_SKIP_PAGES = 8
AKVQ_OPT_EXACT_LOGITS = 16
AKVQ_OPT_DEVICE_L = 32
AKVQ_MAX_PSA_PROMPT = 49152

# every symbol include/akvq.h declares
EXPORTS = (
    "akvq_cache_layout", "akvq_cache_bytes", "akvq_cache_init", "akvq_rotate_quantize",
    "akvq_append_token", "akvq_decode_workspace_bytes", "akvq_decode_workspace_bytes_max",
    "akvq_decode_attention", "akvq_select_salient", "akvq_dequantize_view",
    "akvq_memory_report", "akvq_status_str", "akvq_version", "akvq_decode_step",
    "akvq_detect_pivots", "akvq_rotate_quantize_pivots", "akvq_cache_advance",
    "akvq_cache_attach_pages",
)


class AkvqError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_str(status)} (status {status})")


class akvq_config(C.Structure):
    _fields_ = [("n_units", C.c_int32), ("q_per_kv", C.c_int32), ("head_dim", C.c_int32),
                ("group", C.c_int32), ("residual", C.c_int32), ("capacity", C.c_int32),
                ("top_k", C.c_int32), ("kind", C.c_int32), ("dtype16", C.c_int32),
                ("clip2", C.c_float), ("clip4", C.c_float), ("k_axis", C.c_int32),
                ("paged", C.c_int32), ("exact_r", C.c_int32)]


class akvq_layout(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "total_bytes", "pages_off", "page_bytes", "pg_kscale", "pg_kzero", "pg_kcodes",
        "pg_vscale", "pg_vzero", "pg_vcodes", "ring_off", "ring_unit_bytes", "bitmask_off",
        "side_idx_off", "side_cnt_off", "side_off", "side_entry_bytes", "ticket_off", "umax_off",
        "state_off")] + [
        (n, C.c_int32) for n in ("cap", "n_pages", "slots", "bitmask_words", "side_cap", "ng")]


class akvq_cache(C.Structure):
    _fields_ = [("cfg", akvq_config), ("lay", akvq_layout), ("base", C.c_void_p),
                ("L", C.c_int32), ("n_q", C.c_int32), ("sm_count", C.c_int32),
                ("options", C.c_int32), ("launches", C.c_int32), ("last_write", C.c_uint64),
                ("pool", C.c_void_p), ("block_table", C.c_void_p)]


class akvq_mem_report(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "bytes_fp16", "bytes_int4", "bytes_int2", "bytes_overhead",
        "effective_bits_per_element", "compression_ratio_vs_fp16")] + [
        ("allocated_bytes", C.c_uint64)]


_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load libakvq.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libakvq.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2501_15021_b200.build` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        P, S = C.c_void_p, C.c_int
        L.akvq_cache_layout.argtypes = [C.POINTER(akvq_config), C.POINTER(akvq_layout)]
        L.akvq_cache_layout.restype = S
        L.akvq_cache_bytes.argtypes = [C.POINTER(akvq_config)]
        L.akvq_cache_bytes.restype = C.c_size_t
        L.akvq_cache_init.argtypes = [C.POINTER(akvq_cache), C.POINTER(akvq_config), P,
                                      C.c_size_t, P]
        L.akvq_cache_init.restype = S
        L.akvq_rotate_quantize.argtypes = [C.POINTER(akvq_cache), P, P, C.c_int32, P, P, P]
        L.akvq_rotate_quantize.restype = S
        L.akvq_append_token.argtypes = [C.POINTER(akvq_cache), P, P, P, P]
        L.akvq_append_token.restype = S
        L.akvq_decode_workspace_bytes.argtypes = [C.POINTER(akvq_cache)]
        L.akvq_decode_workspace_bytes.restype = C.c_size_t
        L.akvq_decode_workspace_bytes_max.argtypes = [C.POINTER(akvq_cache)]
        L.akvq_decode_workspace_bytes_max.restype = C.c_size_t
        L.akvq_decode_attention.argtypes = [C.POINTER(akvq_cache), P, P, P, C.c_size_t,
                                            C.c_uint32, P]
        L.akvq_decode_attention.restype = S
        L.akvq_decode_step.argtypes = [C.POINTER(akvq_cache), P, P, P, P, P, P, C.c_size_t,
                                       C.c_uint32, P]
        L.akvq_decode_step.restype = S
        L.akvq_select_salient.argtypes = [C.POINTER(akvq_cache), P, P, C.c_int32, P]
        L.akvq_select_salient.restype = S
        L.akvq_dequantize_view.argtypes = [C.POINTER(akvq_cache), P, P, P]
        L.akvq_dequantize_view.restype = S
        L.akvq_memory_report.argtypes = [C.POINTER(akvq_cache), C.c_int32,
                                         C.POINTER(akvq_mem_report)]
        L.akvq_memory_report.restype = S
        L.akvq_detect_pivots.argtypes = [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_float, C.c_int32, P, P, P, P]
        L.akvq_detect_pivots.restype = S
        L.akvq_rotate_quantize_pivots.argtypes = [C.POINTER(akvq_cache), P, P, C.c_int32, P, P,
                                                  C.c_int32, C.c_int32, P]
        L.akvq_rotate_quantize_pivots.restype = S
        L.akvq_cache_attach_pages.argtypes = [C.POINTER(akvq_cache), P, P]
        L.akvq_cache_attach_pages.restype = S
        L.akvq_cache_advance.argtypes = [C.POINTER(akvq_cache), C.c_int32]
        L.akvq_cache_advance.restype = S
        L.akvq_status_str.argtypes = [S]
        L.akvq_status_str.restype = C.c_char_p
        L.akvq_version.argtypes = []
        L.akvq_version.restype = C.c_char_p
        _lib = L
    return _lib


def status_str(st: int) -> str:
    return lib().akvq_status_str(st).decode()


def version() -> str:
    return lib().akvq_version().decode()


def _check(st: int, what: str):
    if st != AKVQ_OK:
        raise AkvqError(st, what)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libakvq takes device tensors")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return C.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_config(U, g, d, G, R, capacity, top_k, kind, dtype16=AKVQ_BF16, clip2=0.8,
                clip4=1.0, k_axis=0, paged=0, exact_r=0) -> akvq_config:
    return akvq_config(U, g, d, G, R, capacity, top_k, kind, dtype16, clip2, clip4, k_axis, paged,
                       exact_r)


# ----------------------------------------------------------------- C-ABI calls
def akvq_cache_layout(cfg: akvq_config) -> akvq_layout:
    y = akvq_layout()
    _check(lib().akvq_cache_layout(C.byref(cfg), C.byref(y)), "akvq_cache_layout")
    return y


def akvq_cache_bytes(cfg: akvq_config) -> int:
    return int(lib().akvq_cache_bytes(C.byref(cfg)))


def akvq_cache_init(cache: akvq_cache, cfg: akvq_config, buf: torch.Tensor, stream=None):
    _check(lib().akvq_cache_init(C.byref(cache), C.byref(cfg), _ptr(buf), buf.numel(),
                                 _stream(stream)), "akvq_cache_init")


def akvq_rotate_quantize(cache, K, V, L0, types=None, colsum=None, stream=None):
    _check(lib().akvq_rotate_quantize(C.byref(cache), _ptr(K), _ptr(V), int(L0), _ptr(types),
                                      _ptr(colsum), _stream(stream)), "akvq_rotate_quantize")


def akvq_append_token(cache, k, v, types=None, stream=None):
    _check(lib().akvq_append_token(C.byref(cache), _ptr(k), _ptr(v), _ptr(types),
                                   _stream(stream)), "akvq_append_token")


def akvq_decode_workspace_bytes(cache) -> int:
    return int(lib().akvq_decode_workspace_bytes(C.byref(cache)))


def akvq_decode_workspace_bytes_max(cache) -> int:
    return int(lib().akvq_decode_workspace_bytes_max(C.byref(cache)))


def akvq_decode_attention(cache, q, out, ws, flags=0, stream=None):
    _check(lib().akvq_decode_attention(C.byref(cache), _ptr(q), _ptr(out), _ptr(ws),
                                       ws.numel() * ws.element_size(), int(flags),
                                       _stream(stream)), "akvq_decode_attention")


def akvq_decode_step(cache, k, v, types, q, out, ws, flags=0, stream=None):
    _check(lib().akvq_decode_step(C.byref(cache), _ptr(k), _ptr(v), _ptr(types), _ptr(q),
                                  _ptr(out), _ptr(ws), ws.numel() * ws.element_size(), int(flags),
                                  _stream(stream)), "akvq_decode_step")


def akvq_select_salient(cache, types, colsum, L0, stream=None):
    _check(lib().akvq_select_salient(C.byref(cache), _ptr(types), _ptr(colsum), int(L0),
                                     _stream(stream)), "akvq_select_salient")


def akvq_detect_pivots(residual, dtype16, tau=50.0, n_max=15, stream=None):
    """residual [rows, L0, hidden] 16-bit CUDA tensor -> (pivots [rows, n_max] i32,
    counts [rows] i32) device tensors (NEXT-2)."""
    rows, L0, hidden = residual.shape
    dev = residual.device
    ws = torch.empty(rows * L0, dtype=torch.float32, device=dev)
    piv = torch.full((rows, n_max), -1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(rows, dtype=torch.int32, device=dev)
    _check(lib().akvq_detect_pivots(_ptr(residual), rows, L0, hidden, int(dtype16), float(tau),
                                    int(n_max), _ptr(ws), _ptr(piv), _ptr(cnt), _stream(stream)),
           "akvq_detect_pivots")
    return piv, cnt


def akvq_rotate_quantize_pivots(cache, K, V, L0, pivots, counts, units_per_row, stream=None):
    _check(lib().akvq_rotate_quantize_pivots(C.byref(cache), _ptr(K), _ptr(V), int(L0),
                                             _ptr(pivots), _ptr(counts), int(pivots.shape[1]),
                                             int(units_per_row), _stream(stream)),
           "akvq_rotate_quantize_pivots")


def akvq_cache_attach_pages(cache, pool: torch.Tensor, block_table: torch.Tensor):
    if block_table.dtype != torch.int32:
        raise ValueError("block_table must be int32")
    _check(lib().akvq_cache_attach_pages(C.byref(cache), _ptr(pool), _ptr(block_table)),
           "akvq_cache_attach_pages")


def akvq_cache_advance(cache, steps: int):
    _check(lib().akvq_cache_advance(C.byref(cache), int(steps)), "akvq_cache_advance")


def akvq_dequantize_view(cache, K, V, stream=None):
    _check(lib().akvq_dequantize_view(C.byref(cache), _ptr(K), _ptr(V), _stream(stream)),
           "akvq_dequantize_view")


def akvq_memory_report(cache, side_entries: int = -1) -> akvq_mem_report:
    r = akvq_mem_report()
    _check(lib().akvq_memory_report(C.byref(cache), int(side_entries), C.byref(r)),
           "akvq_memory_report")
    return r


# ----------------------------------------------------------------- convenience
class PagePool:
    """Device pool of cache pages shared by paged caches (akvq_config.paged = 1).
    Host-side free list; a page is page_bytes bytes (akvq_layout.page_bytes of
    the caches it serves, which must agree)."""

    def __init__(self, n_pages: int, page_bytes: int, device="cuda"):
        self.page_bytes = int(page_bytes)
        self.n_pages = int(n_pages)
        self.buf = torch.empty(self.n_pages * self.page_bytes, dtype=torch.uint8, device=device)
        self.free = list(range(self.n_pages))

    def alloc(self, n: int, shuffle_seed: Optional[int] = None):
        if n > len(self.free):
            raise RuntimeError(f"page pool exhausted ({n} > {len(self.free)} free)")
        if shuffle_seed is not None:           # scattered pages (tests)
            g = torch.Generator().manual_seed(shuffle_seed)
            perm = torch.randperm(len(self.free), generator=g).tolist()
            self.free = [self.free[i] for i in perm]
        out, self.free = self.free[:n], self.free[n:]
        return out

    def release(self, pages):
        self.free.extend(int(p) for p in pages)


class LayerCache:
    """One layer's packed cache in a torch-owned device buffer (pages in the
    buffer, or -- cfg.paged -- in a shared PagePool through a block table)."""

    def __init__(self, cfg: akvq_config, device="cuda", stream=None, options: int = 0,
                 pool: Optional[PagePool] = None, shuffle_seed: Optional[int] = None):
        self.cfg = cfg
        self.layout = akvq_cache_layout(cfg)
        self.buf = torch.empty(int(self.layout.total_bytes), dtype=torch.uint8, device=device)
        self.handle = akvq_cache()
        akvq_cache_init(self.handle, cfg, self.buf, stream)
        self.handle.options = options
        self.pool, self.pages = None, None
        if cfg.paged:
            if pool is None or pool.page_bytes != int(self.layout.page_bytes):
                raise ValueError("a paged cache needs a PagePool of its page size")
            n = cfg.n_units * int(self.layout.n_pages)
            self.pool, self.pages = pool, pool.alloc(n, shuffle_seed)
            self.block_table = torch.tensor(self.pages, dtype=torch.int32, device=device).view(
                cfg.n_units, int(self.layout.n_pages))
            akvq_cache_attach_pages(self.handle, pool.buf, self.block_table)
        self.ws = torch.empty(max(1, akvq_decode_workspace_bytes_max(self.handle)) // 4 + 1,
                              dtype=torch.float32, device=device)

    def release_pages(self):
        """Return a paged cache's pages to its pool (the cache is unusable after)."""
        if self.pool is not None and self.pages:
            self.pool.release(self.pages)
            self.pages = []

    @property
    def L(self) -> int:
        return self.handle.L

    @property
    def n_q(self) -> int:
        return self.handle.n_q

    def prefill(self, K, V, types=None, colsum=None, stream=None):
        akvq_rotate_quantize(self.handle, K, V, K.shape[1], types, colsum, stream)

    def prefill_pivots(self, K, V, pivots, counts, units_per_row, stream=None):
        akvq_rotate_quantize_pivots(self.handle, K, V, K.shape[1], pivots, counts,
                                    units_per_row, stream)

    def append(self, k, v, types=None, stream=None):
        akvq_append_token(self.handle, k, v, types, stream)

    def decode(self, q, out=None, flags=0, stream=None):
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        akvq_decode_attention(self.handle, q, out, self.ws, flags, stream)
        return out

    def step(self, k, v, q, types=None, out=None, flags=0, stream=None):
        """append (k, v) then attend with q, fused into one launch when possible"""
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        akvq_decode_step(self.handle, k, v, types, q, out, self.ws, flags, stream)
        return out

    @property
    def last_launches(self) -> int:
        """Kernels the library enqueued in the last call on this cache."""
        return self.handle.launches

    def view(self, stream=None):
        U, d = self.cfg.n_units, self.cfg.head_dim
        K = torch.empty((U, self.L, d), dtype=torch.float32, device=self.buf.device)
        V = torch.empty_like(K)
        akvq_dequantize_view(self.handle, K, V, stream)
        return K, V

    def side_counts(self) -> torch.Tensor:
        """Side-table entries per unit (device -> host read of the side_cnt region)."""
        y = self.layout
        return self.buf[y.side_cnt_off: y.side_cnt_off + 4 * self.cfg.n_units].view(
            torch.int32).cpu()

    def memory_report(self, side_entries: int = -1):
        """S:424-432.  For a TSA cache with side_entries = -1 the text-token
        count is read back from the device (a synchronizing copy)."""
        if side_entries < 0 and self.cfg.kind == AKVQ_TSA:
            side_entries = int(round(float(self.side_counts().double().mean())))
        return akvq_memory_report(self.handle, side_entries)
