"""CPU tests of the GPU-parity checker (tests/parity.py) itself: the oracle's
fp32-decision state stands in for the GPU state and is compared with the
fp64-decision export under the agreement rules (only documented ties may
differ), and planted defects -- a flipped code, a zero point off by one outside
a tie, a scale off by 1e-5, a wrong 4-bit code -- must be rejected."""
import types

import numpy as np
import pytest

import parity


def _bf16_bits(x):
    import torch
    t = torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _fake_gpu(e, oc, cfg_kind, k_axis=0):
    """GpuState look-alike built from an oracle export (fp32 decisions)."""
    g = types.SimpleNamespace()
    g.L, g.n_q = oc.L, oc.nq
    g.salient = e["salient"].copy()
    g.side_cnt = e["side_count"].copy()
    g.side_idx = e["side_index"].copy()
    g.kscale = e["kscale"].astype(np.float32)
    g.kzero = e["kzero"].copy()
    g.kcodes = e["kcodes"].copy()
    g.vscale = e["vscale"].astype(np.float32)
    g.vzero = e["vzero"].copy()
    g.vcodes = e["vcodes"].copy()
    if cfg_kind == 1:
        g.side16 = e["side16"].copy()
    else:
        g.side4_kscale = e["side4_scale"][:, :, 0].astype(np.float32)
        g.side4_vscale = e["side4_scale"][:, :, 1].astype(np.float32)
        g.side4_kzero = e["side4_zero"][:, :, 0].copy()
        g.side4_vzero = e["side4_zero"][:, :, 1].copy()
        g.side4_k = e["side4"][:, :, 0].copy()
        g.side4_v = e["side4"][:, :, 1].copy()
    return g


def _pair(orc, kind, k_axis=0, seed=3):
    rng = np.random.default_rng(seed)
    U, L0, d, G = 2, 260, 64, 32
    K = _bf16_bits(rng.normal(size=(U, L0, d)) * np.where(np.arange(d) == 4, 15, 1))
    V = _bf16_bits(rng.normal(size=(U, L0, d)))
    ty = (rng.random((U, L0)) < 0.3).astype(np.uint8)
    cs = rng.random((U, 1, L0)).astype(np.float32)
    out = []
    for d64 in (0, 1):
        c = orc.OracleCache(orc.OracleConfig(U, 1, d, G, 8, L0, 5, kind, orc.BF16, k_axis=k_axis,
                                             decide64=d64))
        assert c.prefill(K, V, types=ty, colsum=cs) == 0
        out.append((c, c.export()))
    cfg = types.SimpleNamespace(n_units=U, head_dim=d, group=G, kind=kind, k_axis=k_axis)
    return out, cfg


@pytest.mark.parametrize("kind,k_axis", [(1, 0), (0, 0), (1, 1)], ids=["PSA", "TSA", "PSA-ktok"])
def test_fp32_state_passes_against_fp64_oracle(orc, kind, k_axis):
    ((c32, e32), (c64, e64)), cfg = _pair(orc, kind, k_axis)
    rep = parity.compare_state(_fake_gpu(e32, c32, kind, k_axis), e64, cfg)
    assert rep["elements"] > 0
    # and bit-exact against the fp32-decision oracle itself
    rep2 = parity.compare_state(_fake_gpu(e32, c32, kind, k_axis), e32, cfg)
    assert rep2["code_ties"] == 0 and rep2["zero_ties"] == 0


def test_planted_defects_are_rejected(orc):
    ((c32, e32), (c64, e64)), cfg = _pair(orc, 0)
    nq = c64.nq
    # a code flipped on a non-salient element whose pre-round value is far from a tie
    g = _fake_gpu(e32, c32, 0)
    codes = parity.unpack2(g.vcodes[0, :nq])
    pre = e64["vpre"][0, :nq]
    ok = ~np.isnan(pre) & (np.abs(np.mod(pre, 1.0) - 0.5) > 0.1)
    t, c = np.argwhere(ok)[0]
    byte = g.vcodes[0, t, c // 4]
    g.vcodes[0, t, c // 4] = byte ^ (1 << (2 * (c % 4)))
    with pytest.raises(AssertionError, match="code mismatches"):
        parity.compare_state(g, e64, cfg)
    # a K zero point off by one where clipped_min/scale is not a tie
    g = _fake_gpu(e32, c32, 0)
    zp = e64["kzpre"][0, : nq // 32]
    j, ch = np.argwhere(~np.isnan(zp) & (np.abs(np.mod(zp, 1.0) - 0.5) > 0.1))[0]
    g.kzero[0, j, ch] += 1
    with pytest.raises(AssertionError, match="zero-point"):
        parity.compare_state(g, e64, cfg)
    # a V zero point off by one
    g = _fake_gpu(e32, c32, 0)
    zp = e64["vzpre"][0, :nq]
    t, gi = np.argwhere(~np.isnan(zp) & (np.abs(np.mod(zp, 1.0) - 0.5) > 0.1))[0]
    g.vzero[0, t, gi] -= 1
    with pytest.raises(AssertionError, match="zero-point"):
        parity.compare_state(g, e64, cfg)
    # a scale off by 1e-5 relative
    g = _fake_gpu(e32, c32, 0)
    g.vscale[1, 3, 0] *= 1 + 1e-5
    with pytest.raises(AssertionError, match="vscale"):
        parity.compare_state(g, e64, cfg)
    # a 4-bit side code changed (TSA text row)
    g = _fake_gpu(e32, c32, 0)
    pre4 = e64["side4_pre"][0, : int(e64["side_count"][0]), 0]
    e, c = np.argwhere(np.abs(np.mod(pre4, 1.0) - 0.5) > 0.1)[0]
    g.side4_k[0, e, c // 2] ^= (1 << (4 * (c % 2)))
    with pytest.raises(AssertionError, match="side4"):
        parity.compare_state(g, e64, cfg)
    # a 4-bit side zero point off by one
    g = _fake_gpu(e32, c32, 0)
    g.side4_vzero[1, 0, 0] += 1
    with pytest.raises(AssertionError, match="side4"):
        parity.compare_state(g, e64, cfg)


def test_zero_point_tie_shifts_the_group(orc):
    """A documented zero-point tie (cmn/scale on a half-integer): the GPU's zero
    differs by one and every code of the group is shifted by the same amount
    (except where it clamps) -- accepted; the unshifted codes are not."""
    # per-token V group with clipped_min / scale = -1.5 exactly: x = [-0.9375,
    # ... , 0.9375] symmetric -> cmn = -0.75 (clip 0.8), scale = 0.5, cmn/s = -1.5
    d = G = 4
    cfg = types.SimpleNamespace(n_units=1, head_dim=d, group=G, kind=1, k_axis=0)
    ex = {"salient": np.zeros((1, 4), np.uint8), "side_count": np.zeros(1, np.int32),
          "side_index": np.zeros((1, 0), np.int32), "side16": np.zeros((1, 0, 2, d), np.uint16)}
    pre = np.array([[-1.875, -0.625, 0.625, 1.875]] * 4)       # x / s for 4 tokens
    zpre = np.full((4, 1), -1.5)
    oz = np.full((4, 1), 2, np.int32)                          # -rne(-1.5) = 2
    oc = np.clip(np.rint(pre) + 2, 0, 3).astype(np.uint8)      # [0, 1, 3, 3]
    gz = oz - 1                                                # GPU rounded the tie down
    gc = np.clip(np.rint(pre) + 1, 0, 3).astype(np.uint8)      # shifted codes [0, 0, 2, 3]
    rep = {"code_ties": 0, "zero_ties": 0, "elements": 0}
    gidx = np.arange(4)[:, None] * 1 + np.zeros((1, d), int)
    parity._check_groups("V", gz, oz, zpre, gc, oc, pre, gidx, 3, rep)
    assert rep["zero_ties"] == 4
    with pytest.raises(AssertionError):
        parity._check_groups("V", gz, oz, zpre, oc, oc, pre, gidx, 3, dict(rep))
    del cfg, ex
