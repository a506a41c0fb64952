"""Helpers for GPU-vs-oracle parity: read the raw cache buffer through the layout
the library reports, and compare it with the oracle's export under the agreement
rules of DESIGN.md section 4 (BJ:5)."""
from __future__ import annotations

import numpy as np
import torch

TIE_EPS = 1e-5

# Per-test parity margins (worst decode max-abs error vs the 2e-3 bound, tie
# counts), written to $AKVQ_MARGINS_OUT at the end of the session (conftest).
MARGINS: dict = {}


def record_margin(case: str, worst: float, tol: float, rep: dict | None = None, **extra):
    m = MARGINS.setdefault(case, {"worst_out_err": 0.0, "tol": tol})
    m["worst_out_err"] = max(m["worst_out_err"], float(worst))
    m["margin"] = tol / m["worst_out_err"] if m["worst_out_err"] > 0 else None
    for k, v in (rep or {}).items():
        m[k] = m.get(k, 0) + v
    for k, v in extra.items():
        m[k] = max(m.get(k, v), v) if isinstance(v, float) else v


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
        if getattr(cfg, "paged", 0):            # pages through the block table
            pool = lc.pool.buf.cpu().numpy().reshape(-1, pb)
            pages = pool[lc.block_table.cpu().numpy().reshape(-1)].reshape(U, npg, pb)
        else:
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


def _half_tie(pre):
    """Documented round-half tie: the oracle's pre-round value (x / scale for a
    code, clipped_min / scale for a zero point) within TIE_EPS of a half-integer
    (BJ:5, SURVEY 8(c) agreement rules).  NaN (no decision) is never a tie."""
    with np.errstate(invalid="ignore"):
        return np.abs(np.abs(np.mod(pre, 1.0)) - 0.5) <= TIE_EPS


def _check_groups(tag, gz, oz, zpre, gcodes, ocodes, pre, gidx, levels, rep):
    """One quantized tier of one unit under the agreement rules.
      gz, oz, zpre: GPU / oracle zero points and the oracle's clipped_min/scale
                    per group (any shape, flattened);
      gcodes, ocodes, pre: codes and the oracle's x/scale per element;
      gidx: for every element, the flat index of its group.
    A zero-point mismatch must be a tie with |dz| = 1.  Each code must then equal
    clamp(rne(pre) + z_gpu, 0, levels) -- the oracle's code, shifted with the
    GPU's zero point and clamped -- unless pre itself is a tie; elements with no
    decision (pre NaN: salient slots, empty / degenerate groups) must match
    exactly."""
    gz, oz, zpre = gz.reshape(-1).astype(np.int64), oz.reshape(-1).astype(np.int64), zpre.reshape(-1)
    dz = gz != oz
    bad = dz & ~(_half_tie(zpre) & (np.abs(gz - oz) == 1))
    assert not bad.any(), f"{tag}: {int(bad.sum())} zero-point mismatches that are not ties"
    rep["zero_ties"] += int(dz.sum())
    gc, oc, pre = gcodes.reshape(-1).astype(np.int64), ocodes.reshape(-1).astype(np.int64), pre.reshape(-1)
    gidx = gidx.reshape(-1)
    nod = np.isnan(pre)
    with np.errstate(invalid="ignore"):
        exp = np.clip(np.rint(np.where(nod, 0.0, pre)).astype(np.int64) + gz[gidx], 0, levels)
    exp = np.where(nod, oc, exp)
    # sanity: with the oracle's own zero point the rule reproduces its codes
    with np.errstate(invalid="ignore"):
        own = np.clip(np.rint(np.where(nod, 0.0, pre)).astype(np.int64) + oz[gidx], 0, levels)
    assert np.array_equal(np.where(nod, oc, own), oc), f"{tag}: checker/oracle disagree"
    mism = gc != exp
    bad = mism & ~(_half_tie(pre) & ~nod)
    assert not bad.any(), f"{tag}: {int(bad.sum())} code mismatches that are not ties"
    rep["code_ties"] += int(mism.sum())
    rep["elements"] += gc.size


def _scale_ok(tag, g, o):
    g, o = np.asarray(g, np.float64), np.asarray(o, np.float64)
    assert np.all(np.abs(g - o) <= 1e-6 * np.abs(o) + 1e-30), \
        f"{tag}: max rel err {np.max(np.abs(g - o) / (np.abs(o) + 1e-30)):.3g}"


def compare_state(gs: GpuState, ex: dict, cfg, report: dict | None = None, units=None):
    """Assert GPU cache == oracle export on every region (bit-exact modulo
    documented ties; scales within 1e-6 relative).  Returns the tie counts."""
    U, d, G = cfg.n_units, cfg.head_dim, cfg.group
    ng = d // G
    n_q, L = gs.n_q, gs.L
    nb = n_q // G
    rep = {"code_ties": 0, "zero_ties": 0, "elements": 0}
    us = range(U) if units is None else units
    kt = getattr(cfg, "k_axis", 0) == 1
    tok = np.arange(n_q)
    ch = np.arange(d)
    # group index of every element [n_q, d] of a unit's code array
    kg = (tok[:, None] * ng + ch[None, :] // G) if kt else ((tok[:, None] // G) * d + ch[None, :])
    vg = tok[:, None] * ng + ch[None, :] // G
    for ui, u in enumerate(us):
        assert np.array_equal(gs.salient[u, :L], ex["salient"][ui, :L]), f"bitmask u{u}"
        cnt = int(gs.side_cnt[u])
        assert cnt == int(ex["side_count"][ui]), f"side count u{u}"
        assert np.array_equal(gs.side_idx[u, :cnt], ex["side_index"][ui, :cnt]), f"side idx u{u}"
        if nb == 0:
            continue
        nm = n_q if kt else nb
        _scale_ok(f"kscale u{u}", gs.kscale[u, :nm], ex["kscale"][ui, :nm])
        _check_groups(f"K u{u}", gs.kzero[u, :nm], ex["kzero"][ui, :nm], ex["kzpre"][ui, :nm],
                      unpack2(gs.kcodes[u, :n_q]), unpack2(ex["kcodes"][ui, :n_q]),
                      ex["kpre"][ui, :n_q], kg, 3, rep)
        _scale_ok(f"vscale u{u}", gs.vscale[u, :n_q], ex["vscale"][ui, :n_q])
        _check_groups(f"V u{u}", gs.vzero[u, :n_q], ex["vzero"][ui, :n_q], ex["vzpre"][ui, :n_q],
                      unpack2(gs.vcodes[u, :n_q]), unpack2(ex["vcodes"][ui, :n_q]),
                      ex["vpre"][ui, :n_q], vg, 3, rep)
        if cfg.kind == 1:
            assert np.array_equal(gs.side16[u, :cnt], ex["side16"][ui, :cnt]), f"side16 u{u}"
        elif cnt:
            e = np.arange(cnt)
            sg = e[:, None] * ng + ch[None, :] // G
            for kv, (sc_g, z_g, c_g) in enumerate((
                    (gs.side4_kscale, gs.side4_kzero, gs.side4_k),
                    (gs.side4_vscale, gs.side4_vzero, gs.side4_v))):
                _scale_ok(f"side4 scale u{u} kv{kv}", sc_g[u, :cnt], ex["side4_scale"][ui, :cnt, kv])
                _check_groups(f"side4 u{u} kv{kv}", z_g[u, :cnt], ex["side4_zero"][ui, :cnt, kv],
                              ex["side4_zpre"][ui, :cnt, kv], unpack4(c_g[u, :cnt]),
                              unpack4(ex["side4"][ui, :cnt, kv]), ex["side4_pre"][ui, :cnt, kv],
                              sg, 15, rep)
    if report is not None:
        for k, v in rep.items():
            report[k] = report.get(k, 0) + v
    total = rep["code_ties"] + rep["zero_ties"]
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
