"""Helpers for GPU-vs-oracle parity: read the raw cache buffer through the layout
the library reports, and compare it with the oracle's export under the agreement
rules of DESIGN.md section 4 (BJ:5)."""
from __future__ import annotations

import numpy as np
import torch

TIE_EPS = 1e-5


def f16_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def unpack2(b: np.ndarray) -> np.ndarray:
    """[..., n] bytes -> [..., 4n] 2-bit codes."""
    b = b.astype(np.uint8)
    return np.stack([(b >> (2 * i)) & 3 for i in range(4)], axis=-1).reshape(*b.shape[:-1], -1)


def unpack4(b: np.ndarray) -> np.ndarray:
    b = b.astype(np.uint8)
    return np.stack([b & 15, b >> 4], axis=-1).reshape(*b.shape[:-1], -1)


def k_tiles_to_rows(raw: np.ndarray, U, npg, G, d) -> np.ndarray:
    """K code region of each page (4x4-tile words, include/akvq.h) -> S:146 row
    bytes [U, npg*G, d/4].  Word (cq, tq) at ((cq>>2)*TQ + tq)*4 + (cq&3); its
    byte b = channel 4cq+b, bits 2s = token 4tq+s."""
    TQ, CG = G // 4, d // 16
    B = raw.reshape(U, npg, CG, TQ, 4, 4)                       # [.., cg, tq, j, b]
    codes = (B[..., None] >> (2 * np.arange(4, dtype=np.uint8))) & 3   # [.., cg, tq, j, b, s]
    codes = codes.transpose(0, 1, 3, 6, 2, 4, 5).reshape(U, npg * G, d)  # token 4tq+s, ch 16cg+4j+b
    c4 = codes.reshape(U, npg * G, d // 4, 4).astype(np.uint8)
    return (c4[..., 0] | (c4[..., 1] << 2) | (c4[..., 2] << 4) | (c4[..., 3] << 6)).astype(np.uint8)


def v_tiles_to_rows(raw: np.ndarray, U, npg, G, d) -> np.ndarray:
    """V code region (4x4-tile words) -> S:146 row bytes [U, npg*G, d/4].  Word
    (cq, tq) at ((tq>>2)*CQ + cq)*4 + (tq&3); its byte b is token 4tq+b's byte
    for channels 4cq..4cq+3."""
    TG, CQ = G // 16, d // 4
    B = raw.reshape(U, npg, TG, CQ, 4, 4)                       # [.., tg, cq, j, b]
    return np.ascontiguousarray(B.transpose(0, 1, 2, 4, 5, 3)).reshape(U, npg * G, CQ)


class GpuState:
    """numpy views of every region of one LayerCache buffer."""

    def __init__(self, lc):
        torch.cuda.synchronize()
        y, cfg = lc.layout, lc.cfg
        raw = lc.buf.cpu().numpy()
        U, d, G = cfg.n_units, cfg.head_dim, cfg.group
        ng, npg, pb = y.ng, y.n_pages, int(y.page_bytes)
        self.L, self.n_q = lc.L, lc.n_q
        pages = raw[y.pages_off: y.pages_off + U * npg * pb].reshape(U, npg, pb)

        def pg(off, nbytes, dt):
            return np.ascontiguousarray(pages[:, :, off: off + nbytes]).view(dt)

        if getattr(cfg, "k_axis", 0) == 1:    # per-token K meta [G][ng] per page
            self.kscale = pg(y.pg_kscale, 4 * d, np.float32).reshape(U, npg * G, ng)
            self.kzero = pg(y.pg_kzero, 4 * d, np.int32).reshape(U, npg * G, ng)
        else:
            self.kscale = pg(y.pg_kscale, 4 * d, np.float32).reshape(U, npg, d)
            self.kzero = pg(y.pg_kzero, 4 * d, np.int32).reshape(U, npg, d)
        self.kcodes = k_tiles_to_rows(pg(y.pg_kcodes, G * d // 4, np.uint8), U, npg, G, d)
        self.vscale = pg(y.pg_vscale, 4 * G * ng, np.float32).reshape(U, npg * G, ng)
        self.vzero = pg(y.pg_vzero, 4 * G * ng, np.int32).reshape(U, npg * G, ng)
        self.vcodes = v_tiles_to_rows(pg(y.pg_vcodes, G * d // 4, np.uint8), U, npg, G, d)
        ring = raw[y.ring_off: y.ring_off + U * y.ring_unit_bytes]
        self.ring = np.ascontiguousarray(ring).view(np.uint16).reshape(U, y.slots, 2, d)
        bm = np.ascontiguousarray(raw[y.bitmask_off: y.bitmask_off + U * y.bitmask_words * 4])
        bm = bm.view(np.uint32).reshape(U, y.bitmask_words)
        self.salient = ((bm[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(U, -1)
        sc = y.side_cap
        self.side_idx = np.ascontiguousarray(
            raw[y.side_idx_off: y.side_idx_off + U * sc * 4]).view(np.int32).reshape(U, sc)
        self.side_cnt = np.ascontiguousarray(
            raw[y.side_cnt_off: y.side_cnt_off + U * 4]).view(np.int32)
        se = int(y.side_entry_bytes)
        side = np.ascontiguousarray(raw[y.side_off: y.side_off + U * sc * se]).reshape(U, sc, se)
        if cfg.kind == 1:
            self.side16 = np.ascontiguousarray(side[:, :, : 4 * d]).view(np.uint16).reshape(U, sc, 2, d)
        else:
            f = lambda a, b, dt: np.ascontiguousarray(side[:, :, a:b]).view(dt)
            self.side4_kscale = f(0, 4 * ng, np.float32)
            self.side4_kzero = f(4 * ng, 8 * ng, np.int32)
            self.side4_vscale = f(8 * ng, 12 * ng, np.float32)
            self.side4_vzero = f(12 * ng, 16 * ng, np.int32)
            self.side4_k = side[:, :, 16 * ng: 16 * ng + d // 2]
            self.side4_v = side[:, :, 16 * ng + d // 2: 16 * ng + d]


def _code_mismatch_ok(gc, oc, x, s, zf_tie):
    """A code mismatch is a documented tie iff the oracle's pre-round value x/s is
    within TIE_EPS of a half-integer (or the group's zero point was a tie)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.abs(np.abs(np.mod(x / s, 1.0)) - 0.5) <= TIE_EPS
    return (gc == oc) | r | zf_tie


def compare_state(gs: GpuState, ex: dict, cfg, report: dict | None = None, units=None):
    """Assert GPU cache == oracle export on every region (bit-exact modulo ties;
    scales within 1e-6 relative).  Returns a dict of tie counts."""
    U, d, G = cfg.n_units, cfg.head_dim, cfg.group
    n_q, L = gs.n_q, gs.L
    nb = n_q // G
    rep = {"k_code_ties": 0, "v_code_ties": 0, "zero_ties": 0, "elements": 0}
    us = range(U) if units is None else units
    for ui, u in enumerate(us):
        # bitmask / salient flags over [0, L)
        assert np.array_equal(gs.salient[u, :L], ex["salient"][ui, :L]), f"bitmask u{u}"
        # side table
        cnt = int(gs.side_cnt[u])
        assert cnt == int(ex["side_count"][ui]), f"side count u{u}"
        assert np.array_equal(gs.side_idx[u, :cnt], ex["side_index"][ui, :cnt]), f"side idx u{u}"
        if nb == 0:
            continue
        # K meta: per channel per block [nb, d], or per token per group [n_q, ng]
        kt = getattr(cfg, "k_axis", 0) == 1
        nm = n_q if kt else nb
        ks_g, ks_o = gs.kscale[u, :nm], ex["kscale"][ui, :nm]
        assert np.all(np.abs(ks_g - ks_o) <= 1e-6 * np.abs(ks_o) + 1e-30), f"kscale u{u}"
        kz_g, kz_o = gs.kzero[u, :nm], ex["kzero"][ui, :nm]
        kc_g = unpack2(gs.kcodes[u, :n_q]).astype(np.int32)
        kc_o = unpack2(ex["kcodes"][ui, :n_q]).astype(np.int32)
        x = ex["xs_k"][ui, :n_q].astype(np.float64)
        ax = 1 if kt else 0          # expand meta to [n_q, d]
        s32 = np.repeat(ex["kscale32"][ui, :nm].astype(np.float64), G, axis=ax)
        zt = np.repeat(kz_g != kz_o, G, axis=ax)
        if np.any(kz_g != kz_o):
            # zero-point tie: cmn/scale within TIE_EPS of a half-integer
            rep["zero_ties"] += int((kz_g != kz_o).sum())
            assert np.all(np.abs(kz_g - kz_o)[kz_g != kz_o] == 1), f"kzero u{u}"
        ok = _code_mismatch_ok(kc_g, kc_o, x, s32, zt)
        assert ok.all(), f"K codes u{u}: {int((~ok).sum())} non-tie mismatches"
        rep["k_code_ties"] += int((kc_g != kc_o).sum())
        # V meta per token per group and codes
        vs_g, vs_o = gs.vscale[u, :n_q], ex["vscale"][ui, :n_q]
        assert np.all(np.abs(vs_g - vs_o) <= 1e-6 * np.abs(vs_o) + 1e-30), f"vscale u{u}"
        vz_g, vz_o = gs.vzero[u, :n_q], ex["vzero"][ui, :n_q]
        vzt = vz_g != vz_o
        rep["zero_ties"] += int(vzt.sum())
        vc_g = unpack2(gs.vcodes[u, :n_q]).astype(np.int32)
        vc_o = unpack2(ex["vcodes"][ui, :n_q]).astype(np.int32)
        xv = ex["xs_v"][ui, :n_q].astype(np.float64)
        sv = np.repeat(ex["vscale32"][ui, :n_q].astype(np.float64), G, axis=1)
        ok = _code_mismatch_ok(vc_g, vc_o, xv, sv, np.repeat(vzt, G, axis=1))
        assert ok.all(), f"V codes u{u}: {int((~ok).sum())} non-tie mismatches"
        rep["v_code_ties"] += int((vc_g != vc_o).sum())
        rep["elements"] += 2 * n_q * d
        # side rows
        if cfg.kind == 1:
            assert np.array_equal(gs.side16[u, :cnt], ex["side16"][ui, :cnt]), f"side16 u{u}"
        elif cnt:
            for kv, (sc_g, z_g, c_g) in enumerate((
                    (gs.side4_kscale, gs.side4_kzero, gs.side4_k),
                    (gs.side4_vscale, gs.side4_vzero, gs.side4_v))):
                so = ex["side4_scale"][ui, :cnt, kv]
                assert np.all(np.abs(sc_g[u, :cnt] - so) <= 1e-6 * np.abs(so) + 1e-30), "side4 scale"
                zo = ex["side4_zero"][ui, :cnt, kv]
                zg = z_g[u, :cnt]
                rep["zero_ties"] += int((zg != zo).sum())
                cg = unpack4(c_g[u, :cnt]).astype(np.int32)
                co = unpack4(ex["side4"][ui, :cnt, kv]).astype(np.int32)
                mism = cg != co
                rep["k_code_ties" if kv == 0 else "v_code_ties"] += int(mism.sum())
                assert mism.sum() <= max(2, 1e-3 * cg.size), f"side4 codes u{u} kv{kv}"
    if report is not None:
        for k, v in rep.items():
            report[k] = report.get(k, 0) + v
    total = rep["k_code_ties"] + rep["v_code_ties"]
    assert total <= max(4, 1e-4 * max(rep["elements"], 1)), f"too many ties: {rep}"
    return rep


def compare_ring(gs: GpuState, rows_k: np.ndarray, rows_v: np.ndarray, slots: int, units=None):
    """Ring tokens [n_q, L) must be bit-exact copies of the original rows (R10).
    rows_k/v: [U, L, d] uint16 of every token fed so far."""
    us = range(gs.ring.shape[0]) if units is None else units
    for ui, u in enumerate(us):
        for t in range(gs.n_q, gs.L):
            assert np.array_equal(gs.ring[u, t % slots, 0], rows_k[ui, t]), f"ring K u{u} t{t}"
            assert np.array_equal(gs.ring[u, t % slots, 1], rows_v[ui, t]), f"ring V u{u} t{t}"
