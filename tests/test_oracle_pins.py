"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something OTHER than itself: a value the
paper prints (Eq. 7), a SPEC worked example (tests/golden/spec_examples.json,
each with its citation), a closed form, an invariant, a library routine
(scipy.linalg.hadamard, torch SDPA in fp64) or brute force on tiny inputs.
A plausible mistake in the oracle -- a dropped term, a wrong sign or index, a
transposed operand, a mis-rounded code -- fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg
import torch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _spec():
    with open(os.path.join(GOLD, "spec_examples.json")) as f:
        return json.load(f)


def _f16_bits(x):
    return np.asarray(x, np.float16).view(np.uint16)


def _bf16_bits(x):
    t = torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


# ------------------------------------------------------------------ Eq. 7
def test_h1_and_h2_as_printed(orc):
    assert np.array_equal(orc.hadamard(1), np.array([[1.0]]))          # H_1 = [1]
    rows = [list(map(float, l.split())) for l in open(os.path.join(GOLD, "eq7_hadamard_h2.txt"))
            if l.strip() and not l.startswith("#")]
    H2 = np.array(rows) / math.sqrt(2.0)
    assert np.abs(orc.hadamard(2) - H2).max() <= 1e-15


@pytest.mark.parametrize("d", [2, 4, 8, 16, 32, 64, 128, 256, 512])
def test_hadamard_closed_form_and_library(orc, d):
    H = orc.hadamard(d)
    Hs = orc.hadamard(d, normalized=False)
    i = np.arange(d)
    pop = np.vectorize(lambda v: bin(int(v)).count("1"))(i[:, None] & i[None, :])
    closed = (-1.0) ** pop
    assert np.array_equal(Hs, closed)                                  # (-1)^popcount(i&j)
    assert np.array_equal(Hs, scipy.linalg.hadamard(d).astype(np.float64))
    assert np.abs(H * math.sqrt(d) - Hs).max() <= 1e-12
    assert np.abs(H @ H.T - np.eye(d)).max() <= 1e-12                  # H H^T = I
    assert np.abs(Hs @ Hs.T - d * np.eye(d)).max() <= 1e-9             # H_s H_s^T = d I (BJ:5)
    assert np.abs(H @ H - np.eye(d)).max() <= 1e-12                    # involution


def test_rotate_worked_examples(orc):
    # d = 4, x = [1,2,3,4]: x.H = [5, -1, -2, 0] (exact arithmetic).
    assert np.abs(orc.rotate([1, 2, 3, 4]) - [5, -1, -2, 0]).max() <= 1e-12
    ex = _spec()["fwht"][0]
    assert np.abs(orc.rotate(ex["x"]) * math.sqrt(2) - ex["y_times_sqrt_d"]).max() <= 1e-12
    for d in (8, 64, 128):                                             # one-hot
        for j in (0, d // 3, d - 1):
            e = np.zeros(d); e[j] = 3.5
            y = orc.rotate(e)
            assert np.abs(np.abs(y) - 3.5 / math.sqrt(d)).max() <= 1e-12


def test_rotation_invariants(orc):
    rng = np.random.default_rng(0)
    for d in (16, 64, 128):
        q, k = rng.normal(size=d), rng.normal(size=d)
        qt, kt = orc.rotate(q), orc.rotate(k)
        assert abs(np.dot(qt, kt) - np.dot(q, k)) <= 1e-10            # q~.k~ = q.k
        assert abs(np.linalg.norm(qt) - np.linalg.norm(q)) <= 1e-10   # energy
        assert np.abs(orc.rotate(qt) - q).max() <= 1e-12              # invertible
        # explicit matrix vs the library Hadamard
        assert np.abs(orc.rotate(q, normalized=False) - q @ scipy.linalg.hadamard(d)).max() <= 1e-9


def test_rotation_reduces_channel_outliers(orc):
    # Fig. 5 analogue: one-hot channel -> uniform; hot channels spread.
    rng = np.random.default_rng(1)
    d = 128
    X = rng.normal(size=(64, d)); X[:, [3, 17]] *= 20
    Y = np.stack([orc.rotate(x) for x in X])
    ratio = lambda T: np.abs(T).mean(0).max() / np.abs(T).mean(0).mean()
    assert ratio(Y) < ratio(X)


# ------------------------------------------------------------------ Eqs. 3-6
def test_quantizer_spec_examples(orc):
    for ex in _spec()["quantize"]:
        s, z, c = orc.quantize_group(ex["x"], ex["bits"], ex["clip"])
        assert s == pytest.approx(ex["scale"], rel=1e-7), ex["cite"]
        assert z == ex["zero"], ex["cite"]
        assert c.tolist() == ex["codes"], ex["cite"]


def test_clipped_range_via_scale(orc):
    # clipped range of [-10, 4] is (-10, 4) at 1.0 and (-8, 3.2) at 0.8;
    # Eq. 5 then gives scale = (max - min) / 3 for 2 bits.
    for ex in _spec()["clipped_range"]:
        s, z, _ = orc.quantize_group(ex["x"], 2, ex["clip"])
        assert s * 3 == pytest.approx(ex["max"] - ex["min"], rel=1e-6), ex["cite"]
        assert z == -round(ex["min"] / ((ex["max"] - ex["min"]) / 3))


def test_quantizer_hand_worked(orc):
    # on-grid: scale is a power of two, zero an integer -> exact reconstruction.
    x = [-0.5, 0, 0.5, 1, 1, -0.5, 0.5, 0]
    s, z, c = orc.quantize_group(x, 2, 1.0)
    assert (s, z, c.tolist()) == (0.5, 1, [0, 1, 2, 3, 3, 0, 2, 1])
    assert np.array_equal(s * (c.astype(np.float64) - z), np.asarray(x, np.float64))
    # clip 0.8, no ties: scale 32/15, zero 1 (cmn/scale = -1.125), codes [0,1,1,2,3].
    s, z, c = orc.quantize_group([-3, -1, 0.25, 2, 5], 2, 0.8)
    assert s == pytest.approx(32 / 15, rel=1e-6) and z == 1 and c.tolist() == [0, 1, 1, 2, 3]
    # a skipped (salient) element is excluded from the statistics and coded 0.
    s2, z2, c2 = orc.quantize_group([-3, -1, 100.0, 2, 5], 2, 0.8, skip=[0, 0, 1, 0, 0])
    assert (s2, z2) == (s, z) and c2.tolist() == [0, 1, 0, 2, 3]
    # all skipped: empty group -> (0, 0), codes 0.
    s3, z3, c3 = orc.quantize_group([1.0, 2.0], 2, 0.8, skip=[1, 1])
    assert (s3, z3, c3.tolist()) == (0.0, 0, [0, 0])


@pytest.mark.parametrize("bits,clip", [(2, 0.8), (2, 1.0), (4, 0.8), (4, 1.0)])
def test_quantizer_brute_force_and_bounds(orc, bits, clip):
    """brute-force nearest code, error <= scale/2, monotone."""
    rng = np.random.default_rng(bits * 10 + int(clip * 10))
    levels = (1 << bits) - 1
    for _ in range(300):
        x = rng.uniform(-1, 1, size=128).astype(np.float32) * rng.uniform(0.1, 10)
        s, z, c = orc.quantize_group(x, bits, clip)
        assert c.max() <= levels
        # brute force over every code q: argmin |x - s (q - z)|, ties -> even rounding
        # of x/s (checked by excluding exact half-way points, which random data avoids)
        grid = s * (np.arange(levels + 1)[None, :] - z)
        best = np.abs(x.astype(np.float64)[:, None] - grid).argmin(1)
        assert np.array_equal(best, c)
        xr = s * (c.astype(np.float64) - z)
        inclip = (x >= clip * x.min()) & (x <= clip * x.max())
        assert np.all(np.abs(x[inclip] - xr[inclip]) <= s / 2 + 1e-6)
        o = np.argsort(x, kind="stable")
        assert np.all(np.diff(c[o].astype(int)) >= 0)


def test_pack_examples_and_roundtrip(orc):
    for ex in _spec()["pack"]:
        assert orc.pack(ex["codes"], ex["bits"]).tolist() == ex["bytes"], ex["cite"]
    assert orc.pack([0, 1, 1, 2], 2).tolist() == [0x94]
    rng = np.random.default_rng(3)
    for bits in (2, 4):
        c = rng.integers(0, 1 << bits, size=1000).astype(np.uint8)
        assert np.array_equal(orc.unpack(orc.pack(c, bits), 1000, bits), c)


def test_half_decoding(orc):
    vals = np.array([0.0, 1.0, -2.5, 65504.0, 6.1e-5, 5.96e-8, -1e-3], np.float16)
    for v, b in zip(vals, vals.view(np.uint16)):
        assert orc.half_to_double(int(b), orc.FP16) == float(v)
    vb = np.array([1.0, -3.140625, 1e30, 1e-30], np.float32)
    for v, b in zip(torch.tensor(vb).to(torch.bfloat16).float().numpy(), _bf16_bits(vb)):
        assert orc.half_to_double(int(b), orc.BF16) == float(v)


# ------------------------------------------------------------------ saliency
def test_saliency_examples(orc):
    cs = np.array([[0.1, 0.3, 0.3, 0.2]], np.float32)
    assert np.flatnonzero(orc.select_salient(orc.PSA, colsum=cs, top_k=2)).tolist() == [1, 2]
    assert np.flatnonzero(orc.select_salient(orc.PSA, colsum=cs, top_k=1)).tolist() == [1]
    assert np.flatnonzero(orc.select_salient(orc.TSA, types=[1, 0, 0, 1])).tolist() == [0, 3]
    # g > 1: scores are summed over the query heads of the unit
    cs2 = np.array([[0.5, 0.0, 0.1], [0.0, 0.6, 0.1]], np.float32)
    assert np.flatnonzero(orc.select_salient(orc.PSA, colsum=cs2, top_k=1)).tolist() == [1]
    # k >= L0 selects everything
    assert orc.select_salient(orc.PSA, colsum=cs, top_k=9).tolist() == [1, 1, 1, 1]


def test_saliency_brute_force(orc):
    """The selected set is the unique k-subset whose members all precede every
    non-member in the order (score desc, index asc): checked over all subsets."""
    rng = np.random.default_rng(4)
    for trial in range(200):
        L0, k = 8, int(rng.integers(1, 5))
        sc = rng.integers(0, 4, size=(1, L0)).astype(np.float32)       # many ties
        got = set(np.flatnonzero(orc.select_salient(orc.PSA, colsum=sc, top_k=k)))
        wins = []
        for sub in itertools.combinations(range(L0), k):
            ok = all((sc[0, a] > sc[0, b]) or (sc[0, a] == sc[0, b] and a < b)
                     for a in sub for b in range(L0) if b not in sub)
            if ok:
                wins.append(set(sub))
        assert wins == [got]


# ------------------------------------------------------------------ the cache
def _cfg(orc, **kw):
    base = dict(U=1, g=1, d=4, G=4, R=0, capacity=16, top_k=1, kind=orc.PSA,
                dtype16=orc.FP16)
    base.update(kw)
    return orc.OracleConfig(**base)


def _rows_with_rotation(target):
    """fp16 rows K such that K.H_s = target exactly (H_s H_s = d I)."""
    target = np.asarray(target, np.float64)
    d = target.shape[-1]
    K = target @ scipy.linalg.hadamard(d) / d
    assert np.array_equal(K.astype(np.float16).astype(np.float64), K)
    return _f16_bits(K)


def test_per_channel_block_hand_worked(orc):
    """G = 4 tokens, d = 4, 2-bit, clip 1.0 (pre-rotated targets)."""
    # channel 0 = [0,1,2,3] -> (1,0,[0,1,2,3]); channel 1 = -1 const -> degenerate
    # (-1, 0, 1); channels 2,3 = 0 -> degenerate (0, 0, 1).
    Xs = np.array([[0, -1, 0, 0], [1, -1, 0, 0], [2, -1, 0, 0], [3, -1, 0, 0]], float)
    K = _rows_with_rotation(Xs)[None]
    for sal_tok in (None, 2):
        c = orc.OracleCache(_cfg(orc, clip2=1.0, kind=orc.PSA,
                                 top_k=0 if sal_tok is None else 1))
        cs = np.zeros((1, 1, 4), np.float32)
        if sal_tok is not None:
            cs[0, 0, sal_tok] = 1.0
        assert c.prefill(K, K, colsum=cs) == 0 and c.nq == 4
        e = c.export()
        assert np.allclose(e["kscale_raw"][0, 0], [1, -1, 0, 0]) and e["kzero"][0, 0].tolist() == [0] * 4
        kb = e["kcodes"][0, :4, 0].tolist()
        # byte of token t = code(ch0) | code(ch1) << 2 | code(ch2) << 4 | code(ch3) << 6
        exp = [t | (1 << 2) | (1 << 4) | (1 << 6) for t in range(4)]
        if sal_tok is not None:
            exp[sal_tok] = 0
            assert e["side_index"][0].tolist() == [sal_tok]
            assert np.array_equal(e["side16"][0, 0, 0], K[0, sal_tok])
        assert kb == exp
        # stored (normalized) scale = decision scale / sqrt(d)
        assert np.allclose(e["kscale"][0, 0], np.array([1, -1, 0, 0]) / 2)


def test_per_token_k_hand_worked(orc):
    """k_axis = 1 ("per-token"): K quantized per token over
    G-channel groups.  d = G = 4, 2-bit, clip 0.8, rotated targets chosen by hand.
      token 0: [0, 1, 2, 4] -> cmx 3.2, cmn 0, scale 3.2/3, zero 0,
               x/scale = [0, .9375, 1.875, 3.75] -> codes [0, 1, 2, 3]
      token 1: [-4, -2, 0, 2] -> cmx 1.6, cmn -3.2, scale 1.6, zero 2,
               x/scale = [-2.5?] avoided: [-4,-2,0,2]/1.6 = [-2.5, ...] is a tie,
               so token 1 = [-4, -1, 0, 3]: cmx 2.4, cmn -3.2, scale 5.6/3,
               cmn/scale = -12/7 -> zero 2, x/scale = [-15/7, -15/28, 0, 45/28]
               -> rne [-2, -1, 0, 2] + 2 -> codes [0, 1, 2, 3] (clamped 4 -> 3)
      tokens 2, 3: constant rows (degenerate: scale = the constant, zero 0, codes 1)
    The same rows with k_axis = 0 give per-channel meta instead (shape check)."""
    X = np.array([[0, 1, 2, 4], [-4, -1, 0, 3], [2, 2, 2, 2], [0, 0, 0, 0]], float)
    K = _rows_with_rotation(X)[None]
    c = orc.OracleCache(_cfg(orc, kind=orc.PSA, top_k=0, k_axis=1))
    assert c.prefill(K, K, colsum=np.zeros((1, 1, 4), np.float32)) == 0 and c.nq == 4
    e = c.export()
    assert e["kscale_raw"].shape == (1, c.cap, 1)
    s0, s1 = np.float32(np.float32(3.2) / np.float32(3.0)), np.float32(5.6) / np.float32(3.0)
    assert np.isclose(e["kscale_raw"][0, 0, 0], 3.2 / 3, rtol=1e-6)
    assert np.isclose(e["kscale_raw"][0, 1, 0], 5.6 / 3, rtol=1e-6)
    assert e["kscale_raw"][0, 2, 0] == 2.0 and e["kscale_raw"][0, 3, 0] == 0.0
    assert e["kzero"][0, :4, 0].tolist() == [0, 2, 0, 0]
    codes = orc.unpack(e["kcodes"][0, :4].reshape(-1), 16, 2).reshape(4, 4)
    assert codes.tolist() == [[0, 1, 2, 3], [0, 1, 2, 3], [1, 1, 1, 1], [1, 1, 1, 1]]
    # dequantized K (normalized basis) = scale/sqrt(d) * (code - zero)
    Kh, _ = c.view()
    assert np.allclose(Kh[0, 0], (3.2 / 3) / 2 * np.array([0, 1, 2, 3]), atol=1e-6)
    assert np.allclose(Kh[0, 1], (5.6 / 3) / 2 * (np.array([0, 1, 2, 3]) - 2), atol=1e-6)
    assert np.allclose(Kh[0, 2], 2.0 / 2 * 1) and np.allclose(Kh[0, 3], 0.0)
    del s0, s1


def test_per_token_k_bounds_and_library_sdpa(orc):
    """k_axis = 1 on random outlier data: every in-clip K element within scale/2
    of its dequantized value, and decode = library SDPA (torch,
    fp64) over the oracle's own dequantized view, un-rotated by scipy's H."""
    rng = np.random.default_rng(7)
    d, G, L0 = 64, 32, 80
    K = rng.standard_normal((2, L0, d)) * 2.0
    K[:, :, 5] *= 20.0
    V = rng.standard_normal((2, L0, d))
    cfg = _cfg(orc, U=2, d=d, G=G, R=8, capacity=96, top_k=3, k_axis=1)
    c = orc.OracleCache(cfg)
    cs = rng.random((2, 1, L0)).astype(np.float32)
    assert c.prefill(_f16_bits(K), _f16_bits(V), colsum=cs) == 0
    e = c.export()
    Kh, Vh = c.view()
    nq = c.nq
    xs = e["xs_k"][:, :nq] / np.sqrt(d)      # rotated, normalized
    sal = e["salient"][:, :nq].astype(bool)
    sc = np.repeat(e["kscale"][:, :nq], G, axis=-1)             # per token, per channel
    zf = np.repeat(e["kzero"][:, :nq], G, axis=-1).astype(np.float64)
    lo, hi = sc * (0 - zf), sc * (3 - zf)
    inclip = (xs >= np.minimum(lo, hi) - 1e-9) & (xs <= np.maximum(lo, hi) + 1e-9)
    err = np.abs(xs - Kh[:, :nq])
    ok = (err <= sc / 2 + 1e-9) | ~inclip
    assert ok[~sal].all()
    q = _f16_bits(rng.standard_normal((2, 1, d)))
    out = c.decode(q)
    H = scipy.linalg.hadamard(d) / np.sqrt(d)
    for u in range(2):
        qh = q[u].view(np.float16).astype(np.float64) @ H
        ref = _sdpa64(qh, Kh[u], Vh[u]) @ H
        assert np.abs(out[u] - ref).max() < 1e-9


def test_tier_rule_examples(orc):
    """S:332-333 tier examples, with G chosen so the block boundary equals L - R."""
    L, R, d, G = 300, 128, 4, 4
    rng = np.random.default_rng(5)
    K = _f16_bits(rng.normal(size=(1, L, d)))
    types = np.zeros((1, L), np.uint8); types[0, :100] = 1
    c = orc.OracleCache(_cfg(orc, R=R, capacity=L, kind=orc.TSA))
    assert c.prefill(K, K, types=types) == 0
    assert c.nq == 172                                                 # 172..299 16-bit
    e = c.export()
    assert e["side_count"][0] == 100 and e["side_index"][0, :100].tolist() == list(range(100))
    c2 = orc.OracleCache(_cfg(orc, R=R, capacity=L, kind=orc.PSA, top_k=2))
    cs = np.full((1, 1, L), 1e-3, np.float32); cs[0, 0, [0, 57]] = 0.5
    assert c2.prefill(K, K, colsum=cs) == 0
    e2 = c2.export()
    assert e2["side_index"][0].tolist() == [0, 57] and c2.nq == 172


def test_schedule_boundaries(orc):
    # tiny (BJ:7): n_q = 64 at L0 = 96 (G 32, R 8); flush at L = 104 -> 96.
    c = orc.OracleCache(_cfg(orc, d=64, G=32, R=8, capacity=120, top_k=4))
    rng = np.random.default_rng(6)
    K = _f16_bits(rng.normal(size=(1, 96, 64)))
    cs = rng.random((1, 1, 96)).astype(np.float32)
    assert c.prefill(K, K, colsum=cs) == 0 and c.nq == 64
    for L in range(97, 106):
        k = _f16_bits(rng.normal(size=(1, 64)))
        c.append(k, k)
        assert c.L == L and c.nq == (96 if L >= 104 else 64)
    # 7B (BJ:8): n_q = 512 at L0 = 671 (G 128, R 32); 640 at 672; next flush at 800.
    c = orc.OracleCache(_cfg(orc, d=128, G=128, R=32, capacity=801, top_k=15,
                             dtype16=orc.BF16))
    K = _bf16_bits(rng.normal(size=(1, 671, 128)))
    assert c.prefill(K, K, colsum=rng.random((1, 1, 671)).astype(np.float32)) == 0
    assert c.nq == 512
    k = _bf16_bits(rng.normal(size=(1, 128)))
    for L in range(672, 802):
        c.append(k, k)
        assert c.nq == (512 if L < 672 else 640 if L < 800 else 768)
    assert c.append(k, k) != 0 and c.L == 801                          # capacity error


def test_prefill_equals_incremental_append(orc):
    """prefill of T tokens == appending them one at a time (bit-exact)."""
    rng = np.random.default_rng(7)
    for kind in (orc.PSA, orc.TSA):
        L0, d = 200, 64
        K = _f16_bits(rng.normal(size=(2, L0, d)) * np.where(np.arange(d) == 5, 20, 1))
        V = _f16_bits(rng.normal(size=(2, L0, d)))
        types = (rng.random((2, L0)) < 0.3).astype(np.uint8)
        cfg = _cfg(orc, U=2, d=d, G=32, R=16, capacity=L0, kind=kind, top_k=3)
        a = orc.OracleCache(cfg)
        a.prefill(K, V, types=types, colsum=np.zeros((2, 1, L0), np.float32) + 1)
        b = orc.OracleCache(cfg)
        b.prefill(K[:, :0], V[:, :0], types=types[:, :0], colsum=np.zeros((2, 1, 0), np.float32))
        for t in range(L0):
            b.append(K[:, t], V[:, t], types[:, t])
        if kind == orc.PSA:            # pivots exist only for prompt tokens
            continue
        ea, eb = a.export(), b.export()
        assert a.nq == b.nq and a.L == b.L
        for key in ea:
            assert np.array_equal(ea[key], eb[key], equal_nan=ea[key].dtype.kind == "f"), key


def test_region_partition_and_view_bounds(orc):
    """Region partition, dequant error <= scale/2 (north_star), on-grid exact."""
    rng = np.random.default_rng(8)
    U, L0, d, G, R = 3, 150, 64, 32, 20
    K = _f16_bits(rng.normal(size=(U, L0, d)))
    V = _f16_bits(rng.normal(size=(U, L0, d)))
    cfg = _cfg(orc, U=U, d=d, G=G, R=R, capacity=L0, kind=orc.PSA, top_k=4, clip2=1.0)
    c = orc.OracleCache(cfg)
    c.prefill(K, V, colsum=rng.random((U, 1, L0)).astype(np.float32))
    e = c.export()
    Kh, Vh = c.view()
    H = scipy.linalg.hadamard(d) / math.sqrt(d)
    Kf = K.view(np.float16).astype(np.float64) @ H
    Vf = V.view(np.float16).astype(np.float64) @ H
    nq = c.nq
    assert nq == 128
    for u in range(U):
        sal = e["salient"][u, :L0].astype(bool)
        assert sal.sum() == 4 and e["side_count"][u] == (sal[:nq]).sum()
        # 16-bit tiers reproduce the input exactly (up to the fp64 rotation)
        exact = np.zeros(L0, bool); exact[nq:] = True; exact[:nq] |= sal[:nq]
        assert np.abs(Kh[u][exact] - Kf[u][exact]).max() <= 1e-12
        # 2-bit tier: |x - x'| <= scale/2 with clip 1.0 (every element in-clip)
        q = ~exact
        ks = np.repeat(e["kscale"][u, : nq // G], G, axis=0)[:nq]
        assert np.all(np.abs(Kh[u][q] - Kf[u][q]) <= ks[q[:nq]] / 2 * (1 + 1e-6) + 1e-12)
        vs = np.repeat(e["vscale"][u, :nq], G, axis=1)
        assert np.all(np.abs(Vh[u][q] - Vf[u][q]) <= vs[q[:nq]] / 2 * (1 + 1e-6) + 1e-12)
    # inputs on the quantization grid reconstruct exactly: two-level channels
    Xs = np.zeros((1, 32, 32)); Xs[0, :, :] = np.where(rng.random((32, 32)) < 0.5, 2.0, -1.0)
    Xs[0, 0, :] = 2.0; Xs[0, 1, :] = -1.0         # every channel sees both levels
    Kg = _rows_with_rotation(Xs)
    cg = orc.OracleCache(_cfg(orc, d=32, G=32, R=0, capacity=32, top_k=0, clip2=1.0))
    cg.prefill(Kg, Kg, colsum=np.zeros((1, 1, 32), np.float32))
    Kh, _ = cg.view()
    assert np.abs(Kh[0] - Xs[0] / math.sqrt(32)).max() <= 1e-12


def _sdpa64(q, K, V):
    return torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(q)[None, None], torch.tensor(K)[None, None], torch.tensor(V)[None, None]
    )[0, 0].numpy()


def test_decode_special_cases(orc):
    rng = np.random.default_rng(9)
    d = 64
    # single cached token -> output = v
    c = orc.OracleCache(_cfg(orc, d=d, G=32, R=8, capacity=8))
    k = _f16_bits(rng.normal(size=(1, 1, d))); v = _f16_bits(rng.normal(size=(1, 1, d)))
    c.prefill(k, v, colsum=np.ones((1, 1, 1), np.float32))
    q = _f16_bits(rng.normal(size=(1, 1, d)))
    out = c.decode(q)
    assert np.abs(out[0, 0] - v[0, 0].view(np.float16)).max() <= 1e-12
    # identical keys -> mean of values
    c = orc.OracleCache(_cfg(orc, d=d, G=32, R=8, capacity=8))
    K = np.repeat(k, 5, axis=1); V = _f16_bits(rng.normal(size=(1, 5, d)))
    c.prefill(K, V, colsum=np.ones((1, 1, 5), np.float32))
    assert np.abs(c.decode(q)[0, 0] - V[0].view(np.float16).astype(np.float64).mean(0)).max() <= 1e-12
    # 2-token closed form
    c = orc.OracleCache(_cfg(orc, d=d, G=32, R=8, capacity=8))
    K2 = _f16_bits(rng.normal(size=(1, 2, d))); V2 = _f16_bits(rng.normal(size=(1, 2, d)))
    c.prefill(K2, V2, colsum=np.ones((1, 1, 2), np.float32))
    qf = q[0, 0].view(np.float16).astype(np.float64)
    Kf, Vf = K2[0].view(np.float16).astype(np.float64), V2[0].view(np.float16).astype(np.float64)
    s = Kf @ qf / math.sqrt(d)
    p1 = 1.0 / (1.0 + math.exp(s[0] - s[1]))
    assert np.abs(c.decode(q)[0, 0] - ((1 - p1) * Vf[0] + p1 * Vf[1])).max() <= 1e-12


def test_decode_unquantized_matches_library_sdpa(orc):
    """R >= L: nothing is quantized -> output = SDPA on the original rows (torch fp64),
    which also pins the rotation equivalence q~.k~ = q.k and o = o'.H (Figs. 6-7)."""
    rng = np.random.default_rng(10)
    U, g, d, L0 = 2, 3, 64, 40
    K = _bf16_bits(rng.normal(size=(U, L0, d))); V = _bf16_bits(rng.normal(size=(U, L0, d)))
    c = orc.OracleCache(_cfg(orc, U=U, g=g, d=d, G=32, R=64, capacity=64, top_k=4,
                             dtype16=orc.BF16))
    c.prefill(K, V, colsum=rng.random((U, g, L0)).astype(np.float32))
    q = _bf16_bits(rng.normal(size=(U, g, d)))
    out = c.decode(q)
    f = lambda a: torch.tensor(a.view(np.int16)).view(torch.bfloat16).double().numpy()
    for u in range(U):
        ref = _sdpa64(f(q[u]), f(K[u]), f(V[u]))
        assert np.abs(out[u] - ref).max() <= 1e-12
    outr = c.decode(q, out_rotated=True)
    H = scipy.linalg.hadamard(d) / math.sqrt(d)
    assert np.abs(outr @ H - out).max() <= 1e-12


def test_decode_quantized_matches_library_sdpa_on_view(orc):
    """With quantization: decode == SDPA(q.H, view K^, view V^) . H, using scipy's H
    and torch's SDPA -- and outputs lie in the per-channel [min, max] of V^."""
    rng = np.random.default_rng(11)
    U, g, d, L0 = 2, 2, 64, 200
    K = _f16_bits(rng.normal(size=(U, L0, d)) * np.where(np.arange(d) % 17 == 3, 20, 1))
    V = _f16_bits(rng.normal(size=(U, L0, d)))
    types = (rng.random((U, L0)) < 0.2).astype(np.uint8)
    H = scipy.linalg.hadamard(d) / math.sqrt(d)
    for kind in (orc.PSA, orc.TSA):
        c = orc.OracleCache(_cfg(orc, U=U, g=g, d=d, G=32, R=24, capacity=L0, kind=kind,
                                 top_k=4))
        c.prefill(K, V, types=types, colsum=rng.random((U, g, L0)).astype(np.float32))
        q = _f16_bits(rng.normal(size=(U, g, d)))
        out = c.decode(q, out_rotated=True)
        Kh, Vh = c.view()
        for u in range(U):
            qt = q[u].view(np.float16).astype(np.float64) @ H
            ref = _sdpa64(qt, Kh[u], Vh[u])
            assert np.abs(out[u] - ref).max() <= 1e-12
            assert np.all(out[u] <= Vh[u].max(0) + 1e-12) and np.all(out[u] >= Vh[u].min(0) - 1e-12)


def test_decode_error_and_degenerate_states(orc):
    c = orc.OracleCache(_cfg(orc))
    with pytest.raises(RuntimeError):
        c.decode(np.zeros((1, 1, 4), np.uint16))                      # L == 0 -> ESTATE
    assert c.prefill(np.zeros((1, 17, 4), np.uint16), np.zeros((1, 17, 4), np.uint16),
                     colsum=np.zeros((1, 1, 17), np.float32)) != 0      # > capacity
    # all-zero cache: every group degenerate at 0, output 0
    c = orc.OracleCache(_cfg(orc, capacity=16))
    z = np.zeros((1, 16, 4), np.uint16)
    assert c.prefill(z, z, colsum=np.zeros((1, 1, 16), np.float32)) == 0
    assert np.array_equal(c.decode(np.zeros((1, 1, 4), np.uint16)), np.zeros((1, 1, 4)))
    with pytest.raises(ValueError):
        orc.OracleCache(_cfg(orc, d=6))


def test_codes_are_scale_invariant(orc):
    """Reading R5: Eqs. 3,5,6 are homogeneous in X, so quantizing x.H_s (exact sums of
    16-bit inputs) gives the codes of x.H = x.H_s/sqrt(d); only round-half ties can
    differ, and those are excluded here by construction (|frac - 1/2| > 1e-4)."""
    rng = np.random.default_rng(12)
    for _ in range(500):
        x = rng.normal(size=128).astype(np.float32)
        s1, z1, c1 = orc.quantize_group(x, 2, 0.8)
        xn = (x.astype(np.float64) / math.sqrt(128)).astype(np.float32)
        s2, z2, c2 = orc.quantize_group(xn, 2, 0.8)
        fr = np.abs(np.mod(x / s1, 1.0) - 0.5)
        frz = abs((0.8 * x.min() / s1) % 1.0 - 0.5)
        if fr.min() > 1e-4 and frz > 1e-4:
            assert z1 == z2 and np.array_equal(c1, c2)
            assert s2 == pytest.approx(s1 / math.sqrt(128), rel=1e-6)


# ----------------------------------------------------------------- NEXT-2 pivots
def _residual(rng, L0, hidden, inject=()):
    """|N(0,1)| background with injected massive activations."""
    x = np.abs(rng.standard_normal((L0, hidden)))
    for t, mag in inject:
        x[t, rng.integers(hidden)] = mag
    return _bf16_bits(x)


def test_detect_pivots_spec_examples(orc):
    """token 7 at 1000x over a unit-Gaussian background (tau 50) -> [7];
    all tokens identical -> fallback [0]; tokens 3 and 11 at 2000 and 1000 ->
    [3, 11] in descending-score order."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((32, 64))
    x[7] *= 1000.0
    assert orc.detect_pivots(_bf16_bits(x), orc.BF16, 50.0, 15).tolist() == [7]
    same = np.tile(rng.standard_normal((1, 64)), (20, 1))
    assert orc.detect_pivots(_bf16_bits(same), orc.BF16, 50.0, 15).tolist() == [0]
    r = _residual(rng, 40, 64, inject=[(11, 1000.0), (3, 2000.0)])
    assert orc.detect_pivots(r, orc.BF16, 50.0, 15).tolist() == [3, 11]
    # truncation to n_max keeps the largest
    assert orc.detect_pivots(r, orc.BF16, 50.0, 1).tolist() == [3]


def test_detect_pivots_median_and_invariants(orc):
    """The threshold is tau x median (numpy's median: the library routine, mean of
    the two middle values for even L0): a token just above / below it flips;
    scale invariance (power-of-two scale, exact in bf16); injection
    recovery for random background."""
    rng = np.random.default_rng(12)
    for L0 in (31, 32):                          # odd and even token counts
        base = np.full((L0, 8), 1.0)
        base[:, 0] = np.arange(1, L0 + 1, dtype=float)      # score(t) = t + 1
        med = float(np.median(np.arange(1, L0 + 1, dtype=float)))
        tau = 2.0
        # token 25 (above the median, so moving it up keeps the median): exactly
        # tau * median is not selected (strict >), one above is
        for val, want in ((tau * med, False), (tau * med + 1.0, True)):
            x = base.copy()
            x[25, 3] = val
            got = orc.detect_pivots(_bf16_bits(x), orc.BF16, tau, 15).tolist()
            assert got == ([25] if want else [0]), (L0, val, got)
    for _ in range(20):
        r = np.abs(rng.standard_normal((50, 32)))
        t = int(rng.integers(50))
        r[t, int(rng.integers(32))] = 50.0 * 10 * np.max(r)      # >= tau x 10
        bits = _bf16_bits(r)
        got = orc.detect_pivots(bits, orc.BF16, 50.0, 15).tolist()
        assert t in got
        r2 = bits.view(np.int16).astype(np.int32)
        scaled = torch.tensor(r, dtype=torch.float32).to(torch.bfloat16).float().numpy() * 4.0
        assert orc.detect_pivots(_bf16_bits(scaled), orc.BF16, 50.0, 15).tolist() == got
        del r2


def test_prefill_with_pivot_mask(orc):
    """A PSA prefill with an explicit pivot mask equals the colsum top-k prefill
    that selects the same tokens; more pivots than top_k is rejected."""
    rng = np.random.default_rng(13)
    U, d, G, L0 = 2, 64, 32, 72
    K = _bf16_bits(rng.standard_normal((U, L0, d))); V = _bf16_bits(rng.standard_normal((U, L0, d)))
    piv = [[0, 17, 40], [5, 33]]
    mask = np.zeros((U, L0), np.uint8)
    cs = np.zeros((U, 1, L0), np.float32)
    for u, ps in enumerate(piv):
        for i, t in enumerate(ps):
            mask[u, t] = 1
            cs[u, 0, t] = 10.0 - i
    cfg = _cfg(orc, U=U, d=d, G=G, R=8, capacity=80, top_k=3, dtype16=orc.BF16)
    a = orc.OracleCache(cfg); b = orc.OracleCache(cfg)
    assert a.prefill_pivots(K, V, mask) == 0
    cs[1, 0, 60] = 0.5                      # unit 1: top-3 = {5, 33, 60}; mask has 2 pivots
    assert b.prefill(K, V, colsum=cs) == 0
    ea, eb = a.export(), b.export()
    assert np.array_equal(ea["salient"][0], eb["salient"][0])
    assert np.array_equal(ea["kcodes"][0], eb["kcodes"][0])
    assert ea["salient"][1, :L0].nonzero()[0].tolist() == [5, 33]
    over = mask.copy(); over[0, 50] = 1; over[0, 51] = 1
    assert orc.OracleCache(cfg).prefill_pivots(K, V, over) == 1      # EINVAL



# ----------------------------------------------------------------- fp64 decisions
def test_quantizer_fp64_decisions_spec_and_hand_worked(orc):
    """The fp64-decision quantizer (the cache default) on the same
    pins as the fp32 one: SPEC examples S:131-133, the on-grid and clip-0.8
    hand-worked groups, salient skip, empty and degenerate groups."""
    for ex in _spec()["quantize"]:
        s, z, c, _ = orc.quantize_group64(ex["x"], ex["bits"], ex["clip"])
        assert s == pytest.approx(ex["scale"], rel=1e-7), ex["cite"]
        assert z == ex["zero"] and c.tolist() == ex["codes"], ex["cite"]
    x = [-0.5, 0, 0.5, 1, 1, -0.5, 0.5, 0]
    s, z, c, zp = orc.quantize_group64(x, 2, 1.0)
    assert (s, z, c.tolist(), zp) == (0.5, 1, [0, 1, 2, 3, 3, 0, 2, 1], -1.0)
    s, z, c, zp = orc.quantize_group64([-3, -1, 0.25, 2, 5], 2, 0.8)
    # clip is the fp32 constant 0.8f widened exactly (R3)
    c8 = float(np.float32(0.8))
    assert s == pytest.approx((5 * c8 + 3 * c8) / 3, rel=1e-15)
    assert zp == pytest.approx(-1.125, rel=1e-12) and z == 1 and c.tolist() == [0, 1, 1, 2, 3]
    s2, z2, c2, _ = orc.quantize_group64([-3, -1, 100.0, 2, 5], 2, 0.8, skip=[0, 0, 1, 0, 0])
    assert (s2, z2) == (s, z) and c2.tolist() == [0, 1, 0, 2, 3]
    s3, z3, c3, zp3 = orc.quantize_group64([1.0, 2.0], 2, 0.8, skip=[1, 1])
    assert (s3, z3, c3.tolist()) == (0.0, 0, [0, 0]) and math.isnan(zp3)
    s4, z4, c4, zp4 = orc.quantize_group64([5.0] * 4, 2, 0.8)       # degenerate
    assert (s4, z4, c4.tolist()) == (5.0, 0, [1, 1, 1, 1]) and math.isnan(zp4)


@pytest.mark.parametrize("bits,clip", [(2, 0.8), (2, 1.0), (4, 1.0)])
def test_quantizer_fp64_brute_force_and_bounds(orc, bits, clip):
    """fp64 decisions: brute-force nearest code, |x - x'| <= scale/2 for
    in-clip elements, monotone -- on fp64 inputs."""
    rng = np.random.default_rng(100 + bits)
    levels = (1 << bits) - 1
    c32 = float(np.float32(clip))
    for _ in range(300):
        x = rng.uniform(-1, 1, size=128) * rng.uniform(0.1, 10)
        s, z, c, zp = orc.quantize_group64(x, bits, clip)
        assert s == (c32 * x.max() - c32 * x.min()) / levels
        assert z == -round(c32 * x.min() / s) and zp == c32 * x.min() / s
        grid = s * (np.arange(levels + 1)[None, :] - z)
        assert np.array_equal(np.abs(x[:, None] - grid).argmin(1), c)
        xr = s * (c.astype(np.float64) - z)
        inclip = (x >= c32 * x.min()) & (x <= c32 * x.max())
        assert np.all(np.abs(x[inclip] - xr[inclip]) <= s / 2 * (1 + 1e-12))
        o = np.argsort(x, kind="stable")
        assert np.all(np.diff(c[o].astype(int)) >= 0)


def test_fp64_and_fp32_decision_modes_agree_except_ties(orc):
    """The two decision precisions of one cache (R6) give the same codes and zero
    points except documented round-half ties (pre-round value within 1e-5 of a
    half-integer in the fp64 mode), and scales within 1e-6 relative."""
    rng = np.random.default_rng(21)
    U, L0, d, G = 3, 300, 64, 32
    K = _bf16_bits(rng.normal(size=(U, L0, d)) * np.where(np.arange(d) == 9, 15, 1))
    V = _bf16_bits(rng.normal(size=(U, L0, d)))
    types = (rng.random((U, L0)) < 0.3).astype(np.uint8)
    cs = rng.random((U, 1, L0)).astype(np.float32)
    half = lambda a: np.abs(np.abs(np.mod(a, 1.0)) - 0.5) <= 1e-5
    for kind in (orc.PSA, orc.TSA):
        ex = []
        for d64 in (1, 0):
            c = orc.OracleCache(_cfg(orc, U=U, d=d, G=G, R=12, capacity=L0, kind=kind, top_k=5,
                                     dtype16=orc.BF16, decide64=d64))
            assert c.prefill(K, V, types=types, colsum=cs) == 0
            ex.append(c.export())
        e64, e32 = ex
        nq = c.nq
        for key, pre in (("kcodes", "kpre"), ("vcodes", "vpre")):
            a = orc.unpack(e64[key][:, :nq].reshape(-1), U * nq * d, 2)
            b = orc.unpack(e32[key][:, :nq].reshape(-1), U * nq * d, 2)
            tie = half(e64[pre][:, :nq].reshape(-1))
            assert np.all((a == b) | tie), key
        for key, zp in (("kzero", "kzpre"), ("vzero", "vzpre")):
            dz = e64[key] != e32[key]
            assert np.all(~dz | half(e64[zp])), key
        for key in ("kscale_raw", "vscale_raw", "side4_scale"):
            assert np.all(np.abs(e64[key] - e32[key]) <= 1e-6 * np.abs(e64[key]) + 1e-30), key
        if kind == orc.TSA:
            cnt = e64["side_count"]
            for u in range(U):
                a = orc.unpack(e64["side4"][u, :cnt[u]].reshape(-1), cnt[u] * 2 * d, 4)
                b = orc.unpack(e32["side4"][u, :cnt[u]].reshape(-1), cnt[u] * 2 * d, 4)
                tie = half(e64["side4_pre"][u, :cnt[u]].reshape(-1))
                assert np.all((a == b) | tie)


# ----------------------------------------------------------------- TSA 4-bit tier
def test_tsa_4bit_tier_hand_worked(orc):
    """TSA text tokens ("stored with 4-bit precision"; Eqs. 3-6 with
    clip 1.0): d = G = 4, rotated targets chosen by hand, tokens 0 and 2
    text (salient, 4-bit side rows), tokens 1 and 3 vision (2-bit block).
      K.H_s of token 0 = [-2, 1, 4, 7]: range 9 -> scale 9/15 = 0.6, cmn/scale =
        -10/3 -> zero 3; x/scale = [-10/3, 5/3, 20/3, 35/3] -> rne [-3, 2, 7, 12]
        + 3 -> codes [0, 5, 10, 15]; packed low nibble first: 0x50, 0xFA.
      K.H_s of token 2 = [-3, 0, 5, 12] (on the grid): scale 1, zero 3, codes
        [0, 3, 8, 15] -> 0x30, 0xF8; dequantizes exactly.
      V.H_s of tokens 0, 2 = [0, 3, 6, 9]: scale 0.6, zero 0, codes [0, 5, 10, 15].
    Stored scale = decision scale / sqrt(d) (R5); view = stored scale (code - zero)."""
    X = np.array([[-2, 1, 4, 7], [1, -1, 2, 0], [-3, 0, 5, 12], [0, 2, -2, 1]], float)
    Y = np.array([[0, 3, 6, 9], [1, 0, 0, -1], [0, 3, 6, 9], [2, 1, 0, 3]], float)
    K, V = _rows_with_rotation(X)[None], _rows_with_rotation(Y)[None]
    types = np.array([[1, 0, 1, 0]], np.uint8)
    for d64 in (1, 0):
        c = orc.OracleCache(_cfg(orc, kind=orc.TSA, clip4=1.0, decide64=d64))
        assert c.prefill(K, V, types=types) == 0 and c.nq == 4
        e = c.export()
        assert e["side_count"][0] == 2 and e["side_index"][0, :2].tolist() == [0, 2]
        assert e["side4"][0, 0, 0].tolist() == [0x50, 0xFA]           # K of token 0
        assert e["side4"][0, 1, 0].tolist() == [0x30, 0xF8]           # K of token 2
        assert e["side4"][0, 0, 1].tolist() == [0x50, 0xFA]           # V of token 0
        assert np.allclose(e["side4_scale"][0, 0, :, 0], [0.6 / 2, 0.6 / 2], rtol=1e-6)
        assert e["side4_scale"][0, 1, 0, 0] == 0.5                   # 1 / sqrt(4)
        assert e["side4_zero"][0, 0, :, 0].tolist() == [3, 0]
        assert e["side4_zero"][0, 1, 0, 0] == 3
        # the 2-bit region holds codes 0 and meta (0, 0) for the text tokens
        assert e["vscale"][0, [0, 2], 0].tolist() == [0.0, 0.0]
        codes = orc.unpack(e["kcodes"][0, :4].reshape(-1), 16, 2).reshape(4, 4)
        assert codes[0].tolist() == [0] * 4 and codes[2].tolist() == [0] * 4
        Kh, Vh = c.view()
        assert np.allclose(Kh[0, 0], 0.3 * (np.array([0, 5, 10, 15]) - 3), atol=1e-6)
        assert np.abs(Kh[0, 2] - X[2] / 2).max() <= 1e-6            # on the grid: exact
        assert np.abs(Vh[0, 0] - Y[0] / 2).max() <= 1e-6
        # |x - x'| <= scale / 2 on the 4-bit row (clip 1.0: every element in-clip)
        assert np.all(np.abs(Kh[0, 0] - X[0] / 2) <= 0.15 + 1e-6)


@pytest.mark.parametrize("d64", [1, 0])
def test_tsa_4bit_view_bounds_and_on_grid(orc, d64):
    """TSA layer on random outlier data: every 4-bit side element within scale/2
    of the exact rotated value x.H (clip 1.0); side rows on a
    power-of-two grid reconstruct exactly; 16-bit ring rows exact."""
    rng = np.random.default_rng(22)
    U, L0, d, G, R = 2, 160, 64, 32, 16
    K = rng.normal(size=(U, L0, d)); K[:, :, 7] *= 20
    V = rng.normal(size=(U, L0, d))
    types = (rng.random((U, L0)) < 0.4).astype(np.uint8)
    # unit 1, tokens 0..15: rows on a 4-bit grid (scale 0.25 after rotation,
    # integer zero point, codes 0 and 15 both present in every group)
    grid = rng.integers(0, 16, size=(16, d)).astype(float)
    grid[:, 0], grid[:, 1] = 0, 15
    grid[:, 32], grid[:, 33] = 0, 15
    Xg = 0.25 * (grid - 5)
    Kb, Vb = _f16_bits(K), _f16_bits(V)
    Kb[1, :16] = _rows_with_rotation(Xg)
    types[1, :16] = 1
    c = orc.OracleCache(_cfg(orc, U=U, d=d, G=G, R=R, capacity=L0, kind=orc.TSA, clip4=1.0,
                             decide64=d64))
    assert c.prefill(Kb, Vb, types=types) == 0
    e = c.export()
    Kh, Vh = c.view()
    H = scipy.linalg.hadamard(d) / math.sqrt(d)
    Kf = Kb.view(np.float16).astype(np.float64) @ H
    Vf = Vb.view(np.float16).astype(np.float64) @ H
    nq = c.nq
    for u in range(U):
        n = e["side_count"][u]
        idx = e["side_index"][u, :n]
        assert idx.tolist() == np.flatnonzero(types[u, :nq]).tolist()
        for kv, (Xh, Xf) in enumerate(((Kh, Kf), (Vh, Vf))):
            s = np.repeat(e["side4_scale"][u, :n, kv], G, axis=-1)
            assert np.all(np.abs(Xh[u, idx] - Xf[u, idx]) <= s / 2 * (1 + 1e-6) + 1e-12)
        assert np.abs(Kh[u, nq:] - Kf[u, nq:]).max() <= 1e-12
    assert np.abs(Kh[1, :16] - Xg / math.sqrt(d)).max() <= 1e-12


# --------------------------------------------- exact residual window (R26, NEXT-1)
def test_exact_r_schedule_and_window(orc):
    """Per-token K with an exact residual window ("per-token", R = the
    16-bit recent window of P:204; DESIGN R26): after prefill and after every
    append exactly min(L, R) tokens stay 16-bit, n_q = max(0, L - R); the view of
    the last R tokens is their original rows (16-bit tier, exact up to the fp64
    rotation), every older non-salient token is quantized (within scale/2 of its
    rotated row).  Invalid combinations are refused."""
    rng = np.random.default_rng(31)
    d, G, R = 64, 32, 8
    with pytest.raises(ValueError):
        orc.OracleCache(_cfg(orc, d=d, G=G, R=R, k_axis=0, exact_r=1))
    for kind, L0 in ((orc.PSA, 5), (orc.PSA, 45), (orc.TSA, 77)):
        cfg = _cfg(orc, U=2, d=d, G=G, R=R, capacity=L0 + 40, kind=kind, top_k=2,
                   k_axis=1, exact_r=1)
        c = orc.OracleCache(cfg)
        K = _f16_bits(rng.normal(size=(2, L0, d)))
        V = _f16_bits(rng.normal(size=(2, L0, d)))
        types = (rng.random((2, L0)) < 0.3).astype(np.uint8)
        assert c.prefill(K, V, types=types, colsum=rng.random((2, 1, L0)).astype(np.float32)) == 0
        assert c.nq == max(0, L0 - R)
        H = scipy.linalg.hadamard(d) / np.sqrt(d)
        ks, vs = [K], [V]
        for step in range(40):
            k = _f16_bits(rng.normal(size=(2, d)))
            v = _f16_bits(rng.normal(size=(2, d)))
            ks.append(k[:, None]); vs.append(v[:, None])
            assert c.append(k, v, np.ones(2, np.uint8)) == 0
            assert c.L == L0 + step + 1 and c.nq == max(0, c.L - R)
        Kh, Vh = c.view()
        e = c.export()
        Ko = np.concatenate(ks, 1).view(np.float16).astype(np.float64)
        Vo = np.concatenate(vs, 1).view(np.float16).astype(np.float64)
        assert np.abs(Kh[:, c.nq: c.L] - Ko[:, c.nq:] @ H).max() < 1e-12
        assert np.abs(Vh[:, c.nq: c.L] - Vo[:, c.nq:] @ H).max() < 1e-12
        sal = e["salient"][:, : c.L].astype(bool)
        xs = e["xs_k"][:, : c.nq] / np.sqrt(d)
        sc = np.repeat(e["kscale"][:, : c.nq], G, axis=-1)
        ok = np.abs(xs - Kh[:, : c.nq]) <= sc / 2 + 1e-9
        zf = np.repeat(e["kzero"][:, : c.nq], G, axis=-1).astype(np.float64)
        lo, hi = sc * (0 - zf), sc * (3 - zf)
        inclip = (xs >= np.minimum(lo, hi) - 1e-9) & (xs <= np.maximum(lo, hi) + 1e-9)
        assert (ok | ~inclip)[~sal[:, : c.nq]].all()
        assert c.L - c.nq == R


def test_exact_r_equals_block_schedule_per_token(orc):
    """Per-token quantization of a token depends only on its own row and salient
    flag, so the exact-R schedule (token by token, R26) and the block schedule
    (R9, quantize_block) must give identical codes, meta and side entries for
    every token both have quantized -- two independent code paths of the oracle
    checked against each other; plus prefill == incremental append under
    exact R."""
    rng = np.random.default_rng(32)
    d, G, R, L0, n_app = 64, 32, 8, 90, 37
    for kind in (orc.TSA, orc.PSA):
        K = _f16_bits(rng.normal(size=(2, L0 + n_app, d)) * np.where(np.arange(d) == 3, 15, 1))
        V = _f16_bits(rng.normal(size=(2, L0 + n_app, d)))
        types = (rng.random((2, L0 + n_app)) < 0.25).astype(np.uint8)
        cs = rng.random((2, 1, L0)).astype(np.float32)
        caches = []
        for ex in (1, 0):
            c = orc.OracleCache(_cfg(orc, U=2, d=d, G=G, R=R, capacity=L0 + n_app, kind=kind,
                                     top_k=3, k_axis=1, exact_r=ex))
            assert c.prefill(K[:, :L0], V[:, :L0], types=types[:, :L0], colsum=cs) == 0
            for t in range(L0, L0 + n_app):
                assert c.append(K[:, t], V[:, t], types[:, t]) == 0
            caches.append(c)
        a, b = caches                                    # exact, block
        assert a.nq == L0 + n_app - R and b.nq == (L0 + n_app - R) // G * G
        ea, eb = a.export(), b.export()
        n = b.nq
        for key in ("kcodes", "vcodes", "kscale_raw", "kzero", "vscale_raw", "vzero",
                    "kpre", "vpre"):
            assert np.array_equal(ea[key][:, :n], eb[key][:, :n],
                                  equal_nan=ea[key].dtype.kind == "f"), key
        cnt = eb["side_count"]
        assert np.all(ea["side_count"] >= cnt)
        for u in range(2):
            m = int(cnt[u])
            assert np.array_equal(ea["side_index"][u, :m], eb["side_index"][u, :m])
            if kind == orc.TSA:
                assert np.array_equal(ea["side4"][u, :m], eb["side4"][u, :m])
                assert np.array_equal(ea["side4_zero"][u, :m], eb["side4_zero"][u, :m])
        if kind == orc.TSA:                              # prefill == append (no pivots)
            c2 = orc.OracleCache(_cfg(orc, U=2, d=d, G=G, R=R, capacity=L0 + n_app, kind=kind,
                                      top_k=3, k_axis=1, exact_r=1))
            T = L0 + n_app
            assert c2.prefill(K, V, types=types, colsum=np.zeros((2, 1, T), np.float32)) == 0
            e2 = c2.export()
            assert c2.nq == a.nq
            for key in ea:
                assert np.array_equal(ea[key], e2[key], equal_nan=ea[key].dtype.kind == "f"), key
