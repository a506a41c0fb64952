"""CPU oracle of the AKVQ-VL hot path (arXiv 2501.15021) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2501_15021_b200``) never imports it, and this package never imports the
product path: the two share no code.

The arithmetic lives in ``akvq_oracle.c`` (plain C, fp64, explicit Walsh-Hadamard
matrix); this module only marshals numpy arrays through ctypes.

Parity status per function: every exported function is pinned
by ``tests/test_oracle_pins.py`` except the end-to-end attention *quality*
relative to the paper's accuracy tables (Tables II-III), which is
"parity unpinned" -- no model weights or MileBench data exist here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "akvq_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

TSA, PSA = 0, 1
BF16, FP16 = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain IEEE, no FMA contraction, OpenMP over units)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "akvq_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lm"]
        )
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("U", C.c_int), ("g", C.c_int), ("d", C.c_int), ("G", C.c_int),
                ("R", C.c_int), ("capacity", C.c_int), ("top_k", C.c_int),
                ("kind", C.c_int), ("dtype16", C.c_int), ("clip2", C.c_float),
                ("clip4", C.c_float), ("k_axis", C.c_int), ("decide64", C.c_int),
                ("exact_r", C.c_int)]


class _Export(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "kcodes", "vcodes", "kscale", "kzero", "vscale", "vzero", "kscale_raw",
        "vscale_raw", "kzpre", "vzpre", "kpre", "vpre", "salient", "side_index",
        "side_count", "side16", "side4", "side4_scale", "side4_zero", "side4_zpre",
        "side4_pre", "xs_k", "xs_v")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.c_void_p
        L.orc_hadamard.argtypes = [C.c_int, C.c_int, P]
        L.orc_rotate.argtypes = [C.c_int, C.c_int, P, P]
        L.orc_quantize_group.argtypes = [P, P, C.c_int, C.c_int, C.c_int, C.c_float,
                                         P, P, P, C.c_int]
        L.orc_quantize_group.restype = None
        L.orc_quantize_group64.argtypes = [P, P, C.c_int, C.c_int, C.c_float, P, P, P, P]
        L.orc_quantize_group64.restype = None
        L.orc_pack.argtypes = [P, C.c_int, C.c_int, P]
        L.orc_pack.restype = None
        L.orc_unpack.argtypes = [P, C.c_int, C.c_int, P]
        L.orc_unpack.restype = None
        L.orc_half_to_double.argtypes = [C.c_uint16, C.c_int]
        L.orc_half_to_double.restype = C.c_double
        L.orc_select_salient.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]
        L.orc_select_salient.restype = None
        L.orc_new.argtypes = [C.POINTER(_Cfg), C.POINTER(C.c_int)]
        L.orc_new.restype = P
        L.orc_free.argtypes = [P]
        L.orc_free.restype = None
        for f in ("orc_L", "orc_nq", "orc_cap_rounded", "orc_side_cap"):
            getattr(L, f).argtypes = [P]
        L.orc_nthreads.argtypes = []
        L.orc_prefill.argtypes = [P, P, P, C.c_int, P, P]
        L.orc_append.argtypes = [P, P, P, P]
        L.orc_decode.argtypes = [P, P, P, C.c_int, C.c_int, C.c_int]
        L.orc_view.argtypes = [P, P, P]
        L.orc_export.argtypes = [P, C.POINTER(_Export)]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def nthreads() -> int:
    return lib().orc_nthreads()


# ---------------------------------------------------------------- primitives
def detect_pivots(residual, dtype16: int, tau: float = 50.0, n_max: int = 15) -> np.ndarray:
    """Massive-activation pivots of one residual stream [L0, hidden] (uint16 bits)."""
    r = np.ascontiguousarray(residual, np.uint16)
    out = np.zeros(max(n_max, 1), np.int32)
    L = lib()
    L.orc_detect_pivots.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_float, C.c_int,
                                    C.c_void_p]
    n = L.orc_detect_pivots(r.shape[0], r.shape[1], _p(r), dtype16, float(tau), n_max, _p(out))
    return out[:n]


def hadamard(d: int, normalized: bool = True) -> np.ndarray:
    H = np.zeros((d, d), np.float64)
    if lib().orc_hadamard(d, int(normalized), _p(H)) != 0:
        raise ValueError("d must be a power of two")
    return H


def rotate(x, normalized: bool = True) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros_like(x)
    if lib().orc_rotate(x.shape[0], int(normalized), _p(x), _p(y)) != 0:
        raise ValueError("length must be a power of two")
    return y


def quantize_group(x, bits: int, clip: float, skip=None):
    """Eqs. 3,5,6 on one group; returns (scale_fp32, zero, codes)."""
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    sk = None if skip is None else np.ascontiguousarray(skip, np.uint8)
    s = np.zeros(1, np.float32)
    z = np.zeros(1, np.int32)
    codes = np.zeros(n, np.uint8)
    lib().orc_quantize_group(_p(x), _p(sk), n, 1, bits, float(clip), _p(s), _p(z),
                             _p(codes), 1)
    return float(s[0]), int(z[0]), codes


def quantize_group64(x, bits: int, clip: float, skip=None):
    """Eqs. 3,5,6 with fp64 decisions; returns (scale, zero, codes, zpre)."""
    x = np.ascontiguousarray(x, np.float64)
    n = x.shape[0]
    sk = None if skip is None else np.ascontiguousarray(skip, np.uint8)
    s = np.zeros(1, np.float64)
    z = np.zeros(1, np.int32)
    zp = np.zeros(1, np.float64)
    codes = np.zeros(n, np.uint8)
    lib().orc_quantize_group64(_p(x), _p(sk), n, bits, float(clip), _p(s), _p(z), _p(zp),
                               _p(codes))
    return float(s[0]), int(z[0]), codes, float(zp[0])


def pack(codes, bits: int) -> np.ndarray:
    codes = np.ascontiguousarray(codes, np.uint8)
    per = 8 // bits
    out = np.zeros((codes.shape[0] + per - 1) // per, np.uint8)
    lib().orc_pack(_p(codes), codes.shape[0], bits, _p(out))
    return out


def unpack(packed, n: int, bits: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, np.uint8)
    out = np.zeros(n, np.uint8)
    lib().orc_unpack(_p(packed), n, bits, _p(out))
    return out


def half_to_double(bits16: int, dtype16: int) -> float:
    return lib().orc_half_to_double(int(bits16), dtype16)


def select_salient(kind: int, types=None, colsum=None, top_k: int = 15) -> np.ndarray:
    """One unit.  types [L0] u8; colsum [g, L0] f32.  Returns salient [L0] u8."""
    if kind == TSA:
        types = np.ascontiguousarray(types, np.uint8)
        L0, g = types.shape[0], 1
    else:
        colsum = np.ascontiguousarray(colsum, np.float32)
        g, L0 = colsum.shape
    out = np.zeros(L0, np.uint8)
    lib().orc_select_salient(kind, g, L0, top_k, _p(types) if kind == TSA else None,
                             _p(colsum) if kind == PSA else None, _p(out))
    return out


# ---------------------------------------------------------------- the cache
@dataclass
class OracleConfig:
    U: int
    g: int
    d: int
    G: int
    R: int
    capacity: int
    top_k: int
    kind: int
    dtype16: int = BF16
    clip2: float = 0.8
    clip4: float = 1.0
    k_axis: int = 0          # 0 per channel (R1), 1 per token (NEXT-1)
    decide64: int = 1        # quantizer decisions in fp64; 0: fp32 (R6)
    exact_r: int = 0         # per-token K: exactly R tokens stay 16-bit (R26)


class OracleCache:
    """One layer's mixed-precision KV cache, computed plainly in fp64."""

    def __init__(self, cfg: OracleConfig):
        self.cfg = cfg
        c = _Cfg(cfg.U, cfg.g, cfg.d, cfg.G, cfg.R, cfg.capacity, cfg.top_k, cfg.kind,
                 cfg.dtype16, cfg.clip2, cfg.clip4, cfg.k_axis, cfg.decide64, cfg.exact_r)
        st = C.c_int(0)
        self._h = lib().orc_new(C.byref(c), C.byref(st))
        if not self._h:
            raise ValueError(f"oracle: invalid config (status {st.value})")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_free(self._h)
            self._h = None

    @property
    def L(self) -> int:
        return lib().orc_L(self._h)

    @property
    def nq(self) -> int:
        return lib().orc_nq(self._h)

    @property
    def cap(self) -> int:
        return lib().orc_cap_rounded(self._h)

    @property
    def side_cap(self) -> int:
        return lib().orc_side_cap(self._h)

    def prefill(self, K16, V16, types=None, colsum=None) -> int:
        """K16, V16: uint16 bit patterns [U, L0, d]; types [U, L0]; colsum [U, g, L0]."""
        K16 = np.ascontiguousarray(K16, np.uint16)
        V16 = np.ascontiguousarray(V16, np.uint16)
        ty = None if types is None else np.ascontiguousarray(types, np.uint8)
        cs = None if colsum is None else np.ascontiguousarray(colsum, np.float32)
        return lib().orc_prefill(self._h, _p(K16), _p(V16), K16.shape[1], _p(ty), _p(cs))

    def prefill_pivots(self, K16, V16, pivot_mask) -> int:
        """PSA prefill with an explicit pivot mask [U, L0] (NEXT-2)."""
        K16 = np.ascontiguousarray(K16, np.uint16)
        V16 = np.ascontiguousarray(V16, np.uint16)
        m = np.ascontiguousarray(pivot_mask, np.uint8)
        lib().orc_prefill_pivots.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                             C.c_void_p]
        return lib().orc_prefill_pivots(self._h, _p(K16), _p(V16), K16.shape[1], _p(m))

    def append(self, k16, v16, types=None) -> int:
        k16 = np.ascontiguousarray(k16, np.uint16)
        v16 = np.ascontiguousarray(v16, np.uint16)
        ty = None if types is None else np.ascontiguousarray(types, np.uint8)
        return lib().orc_append(self._h, _p(k16), _p(v16), _p(ty))

    def decode(self, q16, out_rotated: bool = False, units=None) -> np.ndarray:
        q16 = np.ascontiguousarray(q16, np.uint16)
        out = np.zeros(q16.shape, np.float64)
        lo, hi = (0, self.cfg.U) if units is None else units
        st = lib().orc_decode(self._h, _p(q16), _p(out), int(out_rotated), lo, hi)
        if st != 0:
            raise RuntimeError(f"oracle decode status {st}")
        return out

    def view(self):
        U, L, d = self.cfg.U, self.L, self.cfg.d
        K = np.zeros((U, L, d), np.float64)
        V = np.zeros((U, L, d), np.float64)
        lib().orc_view(self._h, _p(K), _p(V))
        return K, V

    def export(self, pre: bool = True) -> dict:
        """The packed state in the oracle's natural layout (akvq_oracle.h).  With
        pre=False the per-element pre-round arrays (kpre, vpre, side4_pre) are
        skipped (they are the size of the cache in fp64)."""
        cfg = self.cfg
        U, d, G, cap, sc = cfg.U, cfg.d, cfg.G, self.cap, self.side_cap
        ng = d // G
        scx = max(sc, 1)
        a = dict(
            kcodes=np.zeros((U, cap, d // 4), np.uint8),
            vcodes=np.zeros((U, cap, d // 4), np.uint8),
            kscale=np.zeros((U, cap // G, d), np.float64),
            kzero=np.zeros((U, cap // G, d), np.int32),
            vscale=np.zeros((U, cap, ng), np.float64),
            vzero=np.zeros((U, cap, ng), np.int32),
            kscale_raw=np.zeros((U, cap // G, d), np.float64),
            vscale_raw=np.zeros((U, cap, ng), np.float64),
            kzpre=np.zeros((U, cap // G, d), np.float64),
            vzpre=np.zeros((U, cap, ng), np.float64),
            salient=np.zeros((U, cap), np.uint8),
            side_index=np.zeros((U, scx), np.int32),
            side_count=np.zeros((U,), np.int32),
            side16=np.zeros((U, scx, 2, d), np.uint16),
            side4=np.zeros((U, scx, 2, d // 2), np.uint8),
            side4_scale=np.zeros((U, scx, 2, ng), np.float64),
            side4_zero=np.zeros((U, scx, 2, ng), np.int32),
            side4_zpre=np.zeros((U, scx, 2, ng), np.float64),
            xs_k=np.zeros((U, cap, d), np.float64),
            xs_v=np.zeros((U, cap, d), np.float64),
        )
        if pre:
            a["kpre"] = np.zeros((U, cap, d), np.float64)
            a["vpre"] = np.zeros((U, cap, d), np.float64)
            a["side4_pre"] = np.zeros((U, scx, 2, d), np.float64)
        ex = _Export(*[_p(a.get(n)) for n, _ in _Export._fields_])
        lib().orc_export(self._h, C.byref(ex))
        for k in ("side_index", "side16", "side4", "side4_scale", "side4_zero", "side4_zpre",
                  "side4_pre"):
            if k in a:
                a[k] = a[k][:, :sc]
        if cfg.k_axis == 1:      # per-token K meta: [U][cap][d/G] (same element count)
            for k in ("kscale", "kzero", "kscale_raw", "kzpre"):
                a[k] = a[k].reshape(U, cap, ng)
        return a
