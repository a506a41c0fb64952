"""GPU parity: libakvq.so (through the C ABI) vs the CPU oracle, element by element
on the same seeded inputs (-m gpu).  Agreement rules: DESIGN.md section 4 (BJ:5).

Sizes: the tiny config (BJ:7) and the 7B shape (BJ:8) in full; the sweep, video and
Qwen shapes (BJ:9-11) at full size on the GPU with sampled units checked against
the oracle (first, middle, last unit), in the launch configuration bench.py uses.
"""
import os

import numpy as np
import pytest
import torch

from parity import GpuState, compare_ring, compare_state, f16_bits, record_margin

pytestmark = pytest.mark.gpu

OUT_TOL = 2e-3


@pytest.fixture(scope="module")
def ak():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2501_15021_b200 import akvq
    akvq.lib()
    return akvq


@pytest.fixture(scope="module")
def sy():
    from paper_2501_15021_b200 import synth
    return synth


def _case_name():
    return os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0].split("::")[-1]


def _configs(ak, orc, w, layer, units_n, kind=None, cap=None, k_axis=0, decide64=1, exact_r=0):
    kind = w.kind(layer) if kind is None else kind
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    cap = w.capacity if cap is None else cap
    gcfg = ak.make_config(units_n, w.g, w.d, w.G, w.R, cap, w.top_k, kind, dt, w.clip2, w.clip4,
                          k_axis, exact_r=exact_r)
    ocfg = orc.OracleConfig(units_n, w.g, w.d, w.G, w.R, cap, w.top_k, kind,
                            orc.BF16 if dt == ak.AKVQ_BF16 else orc.FP16, w.clip2, w.clip4,
                            k_axis, decide64, exact_r)
    return gcfg, ocfg


def _run_case(ak, orc, sy, w, layer, kind=None, steps=4, units=None, check_every=1,
              flags=0, report=None, options=0, fused_step=None, k_axis=0,
              xf_layer=None, xf_decode=None, case=None, paged=None, exact_r=0):
    """Prefill + `steps` decode steps on the GPU for all units; the oracle runs the
    sampled `units` (default all) in BOTH decision precisions: fp64 (SURVEY 8(c),
    the contract) and fp32 (R6, the kernel's).  The cache state is compared with
    each after prefill and after every flush (bit-exact modulo documented ties),
    the outputs every `check_every` steps: within OUT_TOL of the fp32-decision
    oracle always, and of the fp64-decision oracle unless the state comparison
    found a documented tie (one tied code on a heavily attended token moves the
    output by up to scale * p).  xf_layer / xf_decode: input
    transforms (stress cases) applied identically to the GPU inputs and the
    oracle's sampled inputs.  Worst errors and tie counts go to parity.MARGINS."""
    U = w.U
    us = list(range(U)) if units is None else list(units)
    gcfg, _ = _configs(ak, orc, w, layer, U, kind, k_axis=k_axis, exact_r=exact_r)
    ocfgs = [_configs(ak, orc, w, layer, len(us), kind, k_axis=k_axis, decide64=d,
                      exact_r=exact_r)[1]
             for d in (1, 0)]
    rep64 = {} if report is None else report
    rep32 = {}
    dev = "cuda"
    inp = sy.layer_inputs(w, layer, device=dev)
    if xf_layer:
        inp = xf_layer(inp)
    if paged is not None:                 # pages scattered over a shared pool (NEXT-4)
        gcfg.paged = 1
        lc = ak.LayerCache(gcfg, options=options, pool=paged, shuffle_seed=layer + 17)
    else:
        lc = ak.LayerCache(gcfg, options=options)
    lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    inp_o = sy.layer_inputs(w, layer, units=us, device="cpu")
    if xf_layer:
        inp_o = xf_layer(inp_o)
    # the CPU-generated sampled units are the GPU's units (counter-based generator)
    assert torch.equal(inp_o["K"], inp["K"][us].cpu())
    assert torch.equal(inp_o["V"], inp["V"][us].cpu())
    ocs = [orc.OracleCache(c) for c in ocfgs]
    for oc in ocs:
        assert oc.prefill(f16_bits(inp_o["K"]), f16_bits(inp_o["V"]), inp_o["types"].numpy(),
                          inp_o["colsum"].numpy()) == 0
    oc = ocs[0]
    rows_k = [f16_bits(inp_o["K"])]
    rows_v = [f16_bits(inp_o["V"])]

    def check_state():
        gs = GpuState(lc)
        assert (gs.L, gs.n_q) == (oc.L, oc.nq)
        compare_state(gs, ocs[0].export(), gcfg, rep64, units=us)
        compare_state(gs, ocs[1].export(), gcfg, rep32, units=us)
        compare_ring(gs, np.concatenate(rows_k, 1), np.concatenate(rows_v, 1), gs.ring.shape[1], us)

    check_state()
    worst = [0.0, 0.0]
    name = case or _case_name()
    for step in range(steps):
        di = sy.decode_inputs(w, layer, step, device=dev)
        if xf_decode:
            di = xf_decode(di)
        nq_before = lc.n_q
        # alternate the fused append+decode call and the two separate calls
        if (step % 2 == 1) if fused_step is None else fused_step:
            out = lc.step(di["k"], di["v"], di["q"], di["types"], flags=flags)
        else:
            lc.append(di["k"], di["v"], di["types"])
            out = lc.decode(di["q"], flags=flags)
        do = sy.decode_inputs(w, layer, step, units=us, device="cpu")
        if xf_decode:
            do = xf_decode(do)
        for o in ocs:
            o.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
        rows_k.append(f16_bits(do["k"])[:, None])
        rows_v.append(f16_bits(do["v"])[:, None])
        assert (lc.L, lc.n_q) == (oc.L, oc.nq)
        if lc.n_q != nq_before:
            check_state()
        if step % check_every == 0 or step == steps - 1:
            got = out[us].double().cpu().numpy()
            errs = [float(np.abs(got - o.decode(f16_bits(do["q"]),
                                                out_rotated=bool(flags & ak.AKVQ_OUT_ROTATED))).max())
                    for o in ocs]
            worst = [max(a, b) for a, b in zip(worst, errs)]
            ties64 = rep64.get("code_ties", 0) + rep64.get("zero_ties", 0)
            record_margin(name, worst[1], OUT_TOL, None, worst_out_err_fp64_oracle=worst[0])
            assert errs[1] <= OUT_TOL, f"step {step}: max-abs {errs[1]} vs the fp32-decision oracle"
            assert errs[0] <= OUT_TOL or ties64 > 0, \
                f"step {step}: max-abs {errs[0]} vs the fp64-decision oracle with no tie"
    record_margin(name, worst[1], OUT_TOL, {k + "_fp64": v for k, v in rep64.items()},
                  **{k + "_fp32": v for k, v in rep32.items()})
    return lc, oc, worst[1]


# ----------------------------------------------------------------- tiny (BJ:7)
@pytest.mark.parametrize("options", [0, 1], ids=["layer-pages", "generic-pages"])
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
def test_tiny_prefill_decode_and_flush(ak, orc, sy, kind, options):
    """Quantize once, 4 decode steps, extended to 16 steps across the L = 104 flush."""
    w = sy.TINY
    lc, oc, worst = _run_case(ak, orc, sy, w, 0, kind=kind, steps=16, options=options)
    assert lc.L == 112 and lc.n_q == 96


def test_tiny_view_and_rotated_output(ak, orc, sy):
    w = sy.TINY
    lc, oc, _ = _run_case(ak, orc, sy, w, 0, kind=1, steps=9, flags=ak.AKVQ_OUT_ROTATED)
    K, V = lc.view()
    Ko, Vo = oc.view()
    for a, b in ((K, Ko), (V, Vo)):
        a = a.double().cpu().numpy()
        assert np.all(np.abs(a - b) <= 1e-6 * np.maximum(np.abs(b), np.abs(b).max(-1, keepdims=True)) + 1e-7)


# ----------------------------------------------------------------- 7B shape (BJ:8)
@pytest.mark.parametrize("options", [0, 1], ids=["layer-pages", "generic-pages"])
@pytest.mark.parametrize("layer", [0, 2], ids=["TSA-L0", "PSA-L2"])
def test_llava7b_layer_full(ak, orc, sy, layer, options):
    """All 32 units; decode across the L = 672 flush (n_q 512 -> 640)."""
    w = sy.LLAVA7B
    rep = {}
    lc, oc, worst = _run_case(ak, orc, sy, w, layer, steps=3, report=rep, options=options)
    assert lc.n_q == 640
    print("ties", rep, "worst", worst)


# ----------------------------------------------------------------- sampled, full size
@pytest.mark.parametrize("name,layer", [("sweep@b16", 2), ("video13b", 3), ("qwen_gqa", 5),
                                        ("qwen_gqa", 1), ("sweep@b64", 2), ("sweep@b64", 0)])
def test_full_size_sampled_units(ak, orc, sy, name, layer):
    """Full BJ sizes in bench.py's launch configuration (sweep@b64 is the bench
    workload), sampled units checked against the oracle."""
    w = sy.get(name)
    U = w.U
    _run_case(ak, orc, sy, w, layer, steps=2, units=[0, U // 3, U // 2, U - 1])


# ----------------------------------------------------------------- edge cases
def _mini(sy, **kw):
    base = dict(name="edge", n_layers=1, batch=1, hq=2, hkv=2, d=128, G=128, R=8, top_k=3,
                dtype="bf16", segments=((1, 20), (0, 200), (1, 30)), tsa_layers=(0,),
                n_outlier_ch=2, outlier_gain=15.0, pivots_random_vision=2, decode_steps=40)
    base.update(kw)
    return sy.Workload(**base)


@pytest.mark.parametrize("kw", [
    dict(),                                                         # TSA, ragged tail
    dict(tsa_layers=()),                                            # PSA
    dict(d=64, G=64, segments=((1, 7), (0, 100))),                  # d 64
    dict(G=32, segments=((0, 77),), R=0, tsa_layers=()),            # G 32, R 0, PSA
    dict(G=64, hq=14, hkv=2, segments=((1, 5), (0, 190)), tsa_layers=()),   # GQA g = 7
    dict(segments=((1, 5),), R=16, decode_steps=30),                # L0 < R: nothing quantized
    dict(segments=((1, 300),)),                                     # TSA all text: empty K groups
    dict(segments=((0, 136),), R=8, top_k=0, tsa_layers=()),        # L0 = G + R exactly, k = 0
    dict(top_k=32, segments=((0, 40),), R=0, G=32, d=64, tsa_layers=()),    # k = L0 > G
], ids=["tsa", "psa", "d64", "g32r0", "gqa7", "short", "alltext", "exact", "k32"])
def test_edge_cases(ak, orc, sy, kw):
    w = _mini(sy, **kw)
    _run_case(ak, orc, sy, w, 0, steps=w.decode_steps)


def test_empty_prefill_then_appends(ak, orc, sy):
    """append to an empty cache; prefill of 0 tokens then 150 appends."""
    w = _mini(sy, segments=((1, 1),), decode_steps=150)
    gcfg, ocfg = _configs(ak, orc, w, 0, w.U)
    lc = ak.LayerCache(gcfg)
    with pytest.raises(ak.AkvqError) as e:
        lc.decode(torch.zeros((w.U, w.g, w.d), dtype=torch.bfloat16, device="cuda"))
    assert e.value.status == ak.AKVQ_ESTATE
    oc = orc.OracleCache(ocfg)
    for step in range(150):
        di = sy.decode_inputs(w, 0, step, device="cuda")
        lc.append(di["k"], di["v"], di["types"])
        oc.append(f16_bits(di["k"]), f16_bits(di["v"]), di["types"].cpu().numpy())
        if step % 37 == 0 or step == 149:
            out = lc.decode(di["q"]).double().cpu().numpy()
            assert np.abs(out - oc.decode(f16_bits(di["q"]))).max() <= OUT_TOL
    compare_state(GpuState(lc), oc.export(), gcfg)


def test_degenerate_constant_rows(ak, orc):
    """Constant K/V rows -> degenerate groups (R8) reconstruct exactly."""
    U, d, G, L0 = 2, 128, 128, 300
    gcfg = ak.make_config(U, 1, d, G, 0, L0 + 4, 2, 1, ak.AKVQ_BF16)
    ocfg = orc.OracleConfig(U, 1, d, G, 0, L0 + 4, 2, 1, orc.BF16)
    K = torch.full((U, L0, d), 0.75, dtype=torch.bfloat16)
    K[:, :, 0] = 3.0                      # rotated rows are not constant, channels are
    V = torch.zeros((U, L0, d), dtype=torch.bfloat16)
    V[:, :, 5] = -2.0                     # rotated V rows = +-2/sqrt(d): two levels
    cs = torch.rand((U, 1, L0), generator=torch.Generator().manual_seed(0))
    lc = ak.LayerCache(gcfg)
    lc.prefill(K.cuda(), V.cuda(), None, cs.cuda())
    oc = orc.OracleCache(ocfg)
    oc.prefill(f16_bits(K), f16_bits(V), None, cs.numpy())
    compare_state(GpuState(lc), oc.export(), gcfg)
    q = torch.randn((U, 1, d), generator=torch.Generator().manual_seed(1)).to(torch.bfloat16)
    out = lc.decode(q.cuda()).double().cpu().numpy()
    assert np.abs(out - oc.decode(f16_bits(q))).max() <= OUT_TOL


def test_determinism_and_errors(ak, orc, sy):
    w = _mini(sy, tsa_layers=())
    gcfg, _ = _configs(ak, orc, w, 0, w.U)
    inp = sy.layer_inputs(w, 0, device="cuda")
    lc = ak.LayerCache(gcfg)
    lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    with pytest.raises(ak.AkvqError) as e:          # prefill on a non-empty cache
        lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    assert e.value.status == ak.AKVQ_ESTATE
    di = sy.decode_inputs(w, 0, 0, device="cuda")
    a = lc.decode(di["q"])
    b = lc.decode(di["q"])
    assert torch.equal(a, b)                         # bit-identical
    small = torch.empty(1, dtype=torch.float32, device="cuda")
    with pytest.raises(ak.AkvqError) as e:
        ak.akvq_decode_attention(lc.handle, di["q"], a, small)
    assert e.value.status == ak.AKVQ_ECAPACITY
    for _ in range(w.capacity - lc.L):
        lc.append(di["k"], di["v"], di["types"])
    with pytest.raises(ak.AkvqError) as e:
        lc.append(di["k"], di["v"], di["types"])
    assert e.value.status == ak.AKVQ_ECAPACITY


# ----------------------------------------------------------------- per-token K (NEXT-1)
@pytest.mark.parametrize("options", [0, 1], ids=["layer-pages", "generic-pages"])
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
def test_tiny_per_token_k(ak, orc, sy, kind, options):
    """k_axis = 1: codes, per-token K meta, view and decode vs the oracle,
    across a flush (tiny: L crosses 104 within 12 steps)."""
    lc, oc, _ = _run_case(ak, orc, sy, sy.TINY, 0, kind=kind, steps=12, options=options,
                          k_axis=1)
    K, V = lc.view()
    Ko, Vo = oc.view()
    for a, b in ((K, Ko), (V, Vo)):
        a = a.double().cpu().numpy()
        assert np.all(np.abs(a - b) <= 1e-6 * np.maximum(np.abs(b), np.abs(b).max(-1, keepdims=True)) + 1e-7)


@pytest.mark.parametrize("layer", [0, 2], ids=["TSA-L0", "PSA-L2"])
def test_llava7b_per_token_k(ak, orc, sy, layer):
    _run_case(ak, orc, sy, sy.LLAVA7B, layer, steps=3, units=[0, 13, 31], k_axis=1)


@pytest.mark.parametrize("name,layer", [("sweep@b16", 2), ("video13b", 3)])
def test_full_size_per_token_k_sampled(ak, orc, sy, name, layer):
    w = sy.get(name)
    _run_case(ak, orc, sy, w, layer, steps=2, units=[0, w.U // 2, w.U - 1], k_axis=1)



# ----------------------------------------------------------------- NEXT-2 pivots
@pytest.mark.parametrize("name", ["tiny", "llava7b", "sweep@b16", "video13b"])
def test_detect_pivots_parity(ak, orc, sy, name):
    """Massive-activation pivots (R22): GPU lists == oracle lists per
    batch row, bit for bit, and the planted pivots are recovered in order."""
    w = sy.get(name)
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    res = sy.residual_inputs(w, device="cuda")
    n_max = w.top_k
    piv, cnt = ak.akvq_detect_pivots(res, dt, 50.0, n_max)
    piv, cnt = piv.cpu().numpy(), cnt.cpu().numpy()
    od = orc.BF16 if dt == ak.AKVQ_BF16 else orc.FP16
    rows = sorted({0, w.batch // 2, w.batch - 1})
    for b in rows:
        ref = orc.detect_pivots(f16_bits(res[b]), od, 50.0, n_max)
        assert piv[b, :cnt[b]].tolist() == ref.tolist(), f"row {b}"
        assert ref.tolist()[: len(sy.pivot_positions(w, b))] == sy.pivot_positions(w, b)[:n_max]


def test_detect_pivots_fallback_and_errors(ak, orc):
    """No token above tau x median -> [0]; even and odd token counts; errors."""
    g = torch.Generator().manual_seed(5)
    for L0 in (33, 64):
        row = torch.randn(1, 1, 128, generator=g).to(torch.bfloat16)
        res = row.expand(2, L0, 128).contiguous().cuda()
        piv, cnt = ak.akvq_detect_pivots(res, ak.AKVQ_BF16, 50.0, 4)
        assert cnt.tolist() == [1, 1] and piv[:, 0].tolist() == [0, 0]
        noisy = torch.randn(2, L0, 128, generator=g).to(torch.bfloat16)
        noisy[1, L0 - 1, 7] = 900.0
        p2, c2 = ak.akvq_detect_pivots(noisy.cuda(), ak.AKVQ_BF16, 2.0, 8)
        for b in range(2):
            ref = orc.detect_pivots(f16_bits(noisy[b]), orc.BF16, 2.0, 8)
            assert p2[b, :int(c2[b])].tolist() == ref.tolist()
    with pytest.raises(ak.AkvqError):
        ak.akvq_detect_pivots(torch.zeros(1, 4, 8, dtype=torch.bfloat16, device="cuda"),
                              ak.AKVQ_BF16, 50.0, 33)


@pytest.mark.parametrize("name,layer", [("tiny", 0), ("llava7b", 2), ("sweep@b16", 2)])
def test_prefill_with_detected_pivots(ak, orc, sy, name, layer):
    """PSA prefill from the detected pivots (NEXT-2): cache state and decode
    outputs vs the oracle prefilled with the same pivot mask."""
    w = sy.get(name)
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    us = sorted({0, w.U // 2, w.U - 1})
    gcfg, _ = _configs(ak, orc, w, layer, w.U, kind=1)
    _, ocfg = _configs(ak, orc, w, layer, len(us), kind=1)
    res = sy.residual_inputs(w, device="cuda")
    piv, cnt = ak.akvq_detect_pivots(res, dt, 50.0, w.top_k)
    inp = sy.layer_inputs(w, layer, device="cuda")
    lc = ak.LayerCache(gcfg)
    lc.prefill_pivots(inp["K"], inp["V"], piv, cnt, w.hkv)
    mask = np.zeros((len(us), w.L0), np.uint8)
    pc, cc = piv.cpu().numpy(), cnt.cpu().numpy()
    for i, u in enumerate(us):
        b = u // w.hkv
        mask[i, pc[b, :cc[b]]] = 1
    oc = orc.OracleCache(ocfg)
    inp_o = sy.layer_inputs(w, layer, units=us, device="cpu")
    assert oc.prefill_pivots(f16_bits(inp_o["K"]), f16_bits(inp_o["V"]), mask) == 0
    compare_state(GpuState(lc), oc.export(), gcfg, None, units=us)
    for step in range(3):
        di = sy.decode_inputs(w, layer, step, device="cuda")
        out = lc.step(di["k"], di["v"], di["q"], di["types"])
        do = sy.decode_inputs(w, layer, step, units=us, device="cpu")
        oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
        ref = oc.decode(f16_bits(do["q"]))
        err = np.abs(out[us].double().cpu().numpy() - ref).max()
        assert err <= OUT_TOL, f"step {step}: {err}"


# ----------------------------------------------------------------- NEXT-3 GQA head groups
@pytest.mark.parametrize("g", [2, 3, 5, 7, 8, 16])
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
def test_gqa_head_groups(ak, orc, sy, g, kind):
    """q_per_kv > 1: g = 2 is one group of 2 heads (page MMA columns 0-3); for
    g > 2 the layer kernel runs ceil(g/2) head groups of 2
    (AKVQ_GQA_NH) per kv head (virtual units, a padded head in the last group
    for odd g); parity with
    the oracle over prefill, a flush and 12 decode steps (fused and split)."""
    import dataclasses
    w = dataclasses.replace(sy.TINY, name=f"tiny_g{g}", hq=4 * g, hkv=4)
    _run_case(ak, orc, sy, w, 0, kind=kind, steps=12)


def test_interleaved_layers_use_prologue(ak, orc, sy):
    """Two layer caches stepped alternately (as in a model): every decode launch
    follows a launch on the OTHER cache, so it streams its first pages before the
    PDL wait (LayerPlan.prologue); outputs must still match the oracle, across a
    flush, with fused and split steps."""
    w = sy.TINY
    caches, oracles = [], []
    for layer, kind in ((0, 1), (1, 0)):
        gcfg, ocfg = _configs(ak, orc, w, layer, w.U, kind)
        lc = ak.LayerCache(gcfg)
        inp = sy.layer_inputs(w, layer, device="cuda")
        lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
        oc = orc.OracleCache(ocfg)
        io = sy.layer_inputs(w, layer, device="cpu")
        oc.prefill(f16_bits(io["K"]), f16_bits(io["V"]), io["types"].numpy(), io["colsum"].numpy())
        caches.append(lc)
        oracles.append(oc)
    for step in range(12):
        for layer, (lc, oc) in enumerate(zip(caches, oracles)):
            di = sy.decode_inputs(w, layer, step, device="cuda")
            out = lc.step(di["k"], di["v"], di["q"], di["types"])
            do = sy.decode_inputs(w, layer, step, device="cpu")
            oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
            ref = oc.decode(f16_bits(do["q"]))
            err = np.abs(out.double().cpu().numpy() - ref).max()
            assert err <= OUT_TOL, f"layer {layer} step {step}: {err}"


# ----------------------------------------------------------------- stress (fixed point)
def _hadamard_row(d, j):
    i = np.arange(d)
    return torch.tensor((-1.0) ** np.vectorize(lambda v: bin(int(v)).count("1"))(i & j))


def _xf_q(scale):
    def f(di):
        di = dict(di)
        di["q"] = (di["q"].float() * scale).to(di["q"].dtype)      # exact: power of two
        return di
    return f


def _xf_v_channel(c, gain):
    def f(inp):
        inp = dict(inp)
        V = inp["V"].float()
        V[:, :, c] *= gain
        inp["V"] = V.to(inp["V"].dtype)
        return inp
    return f


def _xf_k_page_channel(j, amp, t0, t1):
    """Tokens [t0, t1) get amp * (row j of the +-1 Hadamard matrix) added to K, so
    in the rotated basis channel j of that page is ~amp * d, the page's fixed-point
    range is set by one channel."""
    def f(inp):
        inp = dict(inp)
        K = inp["K"].float()
        h = _hadamard_row(K.shape[-1], j).to(K.device, torch.float32)
        K[:, t0:t1, :] += amp * h
        inp["K"] = K.to(inp["K"].dtype)
        return inp
    return f


@pytest.mark.parametrize("stress", ["q8", "q16", "v100", "kpage"])
@pytest.mark.parametrize("layer", [2, 0], ids=["PSA-L2", "TSA-L0"])
def test_stress_fixed_point_sweep64(ak, orc, sy, stress, layer):
    """Large logit spreads (q x8, x16: peaky attention), a V channel x100 and a
    page whose rotated K range is dominated by one channel, at sweep@b64 in the
    bench launch configuration (U = 2048), sampled units vs the oracle.  These
    load the 16-bit fixed points of the page MMAs hardest."""
    w = sy.get("sweep@b64")
    kw = {"q8": dict(xf_decode=_xf_q(8.0)), "q16": dict(xf_decode=_xf_q(16.0)),
          "v100": dict(xf_layer=_xf_v_channel(5, 100.0)),
          "kpage": dict(xf_layer=_xf_k_page_channel(37, 8.0, 384, 512))}[stress]
    _run_case(ak, orc, sy, w, layer, steps=2, units=[0, w.U // 2, w.U - 1], **kw)


# ----------------------------------------------------------------- fixed-point edge cases
def _custom_case(ak, orc, K, V, cfg_kw, q, kind=1, strict64=True):
    """Prefill custom 16-bit K, V (torch, CPU) on the GPU and in both oracle
    modes; compare the state and the decode outputs for q."""
    U, L0, d = K.shape
    dt = ak.AKVQ_FP16 if K.dtype == torch.float16 else ak.AKVQ_BF16
    od = orc.FP16 if dt == ak.AKVQ_FP16 else orc.BF16
    G, R, top_k = cfg_kw["G"], cfg_kw["R"], cfg_kw["top_k"]
    cap = L0 + 4
    gcfg = ak.make_config(U, 1, d, G, R, cap, top_k, kind, dt)
    lc = ak.LayerCache(gcfg)
    g = torch.Generator().manual_seed(3)
    cs = torch.rand((U, 1, L0), generator=g)
    types = torch.zeros((U, L0), dtype=torch.uint8)
    lc.prefill(K.cuda(), V.cuda(), types.cuda(), cs.cuda())
    out = lc.decode(q.cuda()).double().cpu().numpy()
    errs = []
    for d64 in (1, 0):
        oc = orc.OracleCache(orc.OracleConfig(U, 1, d, G, R, cap, top_k, kind, od, decide64=d64))
        assert oc.prefill(f16_bits(K), f16_bits(V), types.numpy(), cs.numpy()) == 0
        if d64 and not strict64:
            # groups with a tiny clipped range next to a large offset: the fp32
            # rounding of clip*max and clip*min (R6) moves the scale by more than
            # 1e-6 relative; the state is checked against the fp32-decision oracle
            try:
                rep = compare_state(GpuState(lc), oc.export(), gcfg)
            except AssertionError as e:
                rep = {"code_ties": -1, "zero_ties": -1, "fp64_state": str(e)[:80]}
        else:
            rep = compare_state(GpuState(lc), oc.export(), gcfg)
        errs.append((float(np.abs(out - oc.decode(f16_bits(q))).max()), rep))
    return errs


def test_negative_degenerate_v_groups(ak, orc):
    """V rows v = c e_0 (c < 0) rotate to a constant negative row: every V group of
    those tokens is degenerate with a NEGATIVE scale (R8: scale = the constant).
    The signed 24-bit weights must carry them (an unsigned weight would drop them)."""
    U, L0, d = 2, 300, 128
    g = torch.Generator().manual_seed(11)
    K = torch.randn((U, L0, d), generator=g).to(torch.bfloat16)
    V = torch.randn((U, L0, d), generator=g)
    V[:, ::3, :] = 0.0
    V[:, ::3, 0] = -2.0                      # every third token: v = -2 e_0
    V = V.to(torch.bfloat16)
    q = torch.randn((U, 1, d), generator=g).to(torch.bfloat16)
    for (err, rep), name in zip(_custom_case(ak, orc, K, V, dict(G=128, R=8, top_k=2), q),
                                ("fp64", "fp32")):
        record_margin(f"test_negative_degenerate_v_groups[{name}]", err, OUT_TOL, rep)
        assert err <= OUT_TOL, (name, err)


def test_large_zero_points_exact_bias(ak, orc):
    """fp16 K rows = a fixed +-1024 pattern plus sparse one-ulp noise: every rotated
    K channel is a large offset with a small range, so the zero points reach tens
    of thousands and the exact page bias sum_c Q_c z_c (int64, folded into the MMA
    accumulators) is near its largest for 16-bit inputs."""
    U, L0, d = 2, 200, 128
    g = torch.Generator().manual_seed(12)
    sign = torch.where(torch.rand((1, 1, d), generator=g) < 0.5, -1.0, 1.0)
    K = (1024.0 * sign + (torch.rand((U, L0, d), generator=g) < 0.01).float()).to(torch.float16)
    V = torch.randn((U, L0, d), generator=g).to(torch.float16)
    q = (torch.randn((U, 1, d), generator=g) * 0.01).to(torch.float16)
    for (err, rep), name in zip(_custom_case(ak, orc, K, V, dict(G=32, R=8, top_k=2), q,
                                             strict64=False), ("fp64", "fp32")):
        record_margin(f"test_large_zero_points_exact_bias[{name}]", err, OUT_TOL,
                      {k: v for k, v in rep.items() if isinstance(v, int)})
        if name == "fp32":
            assert err <= OUT_TOL, (name, err)


@pytest.mark.parametrize("name,layer", [("tiny", 0), ("llava7b", 2), ("llava7b", 0)])
def test_exact_logit_path(ak, orc, sy, name, layer):
    """AKVQ_OPT_EXACT_LOGITS routes every page through the fp32 logit path that a
    page with an out-of-range zero-point bias takes (unreachable with ordinary
    16-bit inputs): parity as usual."""
    w = sy.get(name)
    units = None if name == "tiny" else [0, 17, 31]
    _run_case(ak, orc, sy, w, layer, steps=3, units=units, options=ak.AKVQ_OPT_EXACT_LOGITS)


# ----------------------------------------------------------------- NEXT-4: device L, graphs
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
@pytest.mark.parametrize("g", [1, 7])
def test_device_L_steps(ak, orc, sy, kind, g):
    """AKVQ_OPT_DEVICE_L: the fused kernel takes L from the cache buffer and the
    item table covers the flush period; stepping through two flushes matches the
    oracle exactly as the host-L mode does."""
    import dataclasses
    w = dataclasses.replace(sy.TINY, name=f"tinyg{g}", hq=4 * g, hkv=4, decode_steps=80)
    _run_case(ak, orc, sy, w, 0, kind=kind, steps=70, check_every=7,
              options=ak.AKVQ_OPT_DEVICE_L, fused_step=True)


@pytest.mark.parametrize("name,layer", [("tiny", 0), ("llava7b", 2), ("qwen_gqa", 3)])
def test_cuda_graph_replay(ak, orc, sy, name, layer):
    """A decode step captured once in a CUDA graph (AKVQ_OPT_DEVICE_L) and replayed
    for the following steps of the flush period, new q / k / v copied into the
    captured input buffers before each replay: outputs match the oracle step by
    step; the host mirror is then advanced with akvq_cache_advance."""
    w = sy.get(name)
    us = [0, w.U // 2, w.U - 1] if w.U > 4 else list(range(w.U))
    gcfg, _ = _configs(ak, orc, w, layer, w.U)
    _, ocfg = _configs(ak, orc, w, layer, len(us))
    lc = ak.LayerCache(gcfg, options=ak.AKVQ_OPT_DEVICE_L)
    inp = sy.layer_inputs(w, layer, device="cuda")
    lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    oc = orc.OracleCache(ocfg)
    io = sy.layer_inputs(w, layer, units=us, device="cpu")
    oc.prefill(f16_bits(io["K"]), f16_bits(io["V"]), io["types"].numpy(), io["colsum"].numpy())
    step0 = 0
    while w.R + w.G - 1 - (lc.L - lc.n_q) < 3:               # a flush is due: step past it
        di = sy.decode_inputs(w, layer, step0, device="cuda")
        lc.step(di["k"], di["v"], di["q"], di["types"])
        do = sy.decode_inputs(w, layer, step0, units=us, device="cpu")
        oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
        step0 += 1
    nsteps = min(12, w.R + w.G - 1 - (lc.L - lc.n_q))        # stay inside the flush period
    d0 = sy.decode_inputs(w, layer, 0, device="cuda")
    bq, bk, bv, bt = (d0["q"].clone(), d0["k"].clone(), d0["v"].clone(), d0["types"].clone())
    out = torch.empty(bq.shape, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            lc.step(bk, bv, bq, bt, out=out)                 # recorded, not run (host L += 1)
    torch.cuda.current_stream().wait_stream(s)
    L_host0 = lc.L - 1
    for step in range(step0, step0 + nsteps):
        di = sy.decode_inputs(w, layer, step, device="cuda")
        bq.copy_(di["q"]); bk.copy_(di["k"]); bv.copy_(di["v"]); bt.copy_(di["types"])
        graph.replay()
        do = sy.decode_inputs(w, layer, step, units=us, device="cpu")
        oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
        ref = oc.decode(f16_bits(do["q"]))
        err = np.abs(out[us].double().cpu().numpy() - ref).max()
        record_margin(_case_name(), err, OUT_TOL)
        assert err <= OUT_TOL, f"replay {step}: {err}"
    ak.akvq_cache_advance(lc.handle, nsteps - 1)
    assert lc.L == L_host0 + nsteps == oc.L
    compare_state(GpuState(lc), oc.export(), gcfg, units=us)
    # the next (non-replayed) step continues from the device state
    di = sy.decode_inputs(w, layer, step0 + nsteps, device="cuda")
    o2 = lc.step(di["k"], di["v"], di["q"], di["types"])
    do = sy.decode_inputs(w, layer, step0 + nsteps, units=us, device="cpu")
    oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
    assert np.abs(o2[us].double().cpu().numpy() - oc.decode(f16_bits(do["q"]))).max() <= OUT_TOL


@pytest.mark.parametrize("name,layer", [("tiny", 0), ("llava7b", 0), ("llava7b", 2), ("qwen_gqa", 3)])
def test_paged_block_table(ak, orc, sy, name, layer):
    """Paged caches (akvq_config.paged, NEXT-4): pages come from a shared pool in a
    shuffled order through the block table -- two caches share the pool (the
    second one reserves pages in between) and both match the oracle across a
    flush, fused and split steps alike."""
    w = sy.get(name)
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    cfg = ak.make_config(w.U, w.g, w.d, w.G, w.R, w.capacity, w.top_k, w.kind(layer), dt,
                         paged=1)
    y = ak.akvq_cache_layout(cfg)
    pool = ak.PagePool(2 * w.U * y.n_pages + 7, y.page_bytes)
    other = ak.LayerCache(cfg, pool=pool, shuffle_seed=3)        # interleaved owner
    units = None if w.U <= 32 else [0, w.U // 2, w.U - 1]
    steps = 16 if name == "tiny" else 3
    _run_case(ak, orc, sy, w, layer, steps=steps, units=units, paged=pool)
    other.release_pages()
    with pytest.raises(ak.AkvqError) as e:                      # not attached -> ESTATE
        c = ak.akvq_cache()
        ak.akvq_cache_init(c, cfg, torch.empty(y.total_bytes, dtype=torch.uint8, device="cuda"))
        ak.akvq_rotate_quantize(c, torch.zeros((w.U, 1, w.d), dtype=torch.bfloat16, device="cuda"),
                                torch.zeros((w.U, 1, w.d), dtype=torch.bfloat16, device="cuda"), 1)
    assert e.value.status == ak.AKVQ_ESTATE


# ------------------------------------------ per-token K, exact residual window (R26)
@pytest.mark.parametrize("options", [0, 1], ids=["layer-pages", "generic-pages"])
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
def test_tiny_exact_r(ak, orc, sy, kind, options):
    """exact_r = 1 (R26): n_q = L - R after every step, one token quantized
    as it leaves the window (partial last page), state and decode vs the oracle at
    every step across page boundaries; view vs the oracle's view."""
    lc, oc, _ = _run_case(ak, orc, sy, sy.TINY, 0, kind=kind, steps=16, options=options,
                          k_axis=1, exact_r=1)
    assert lc.n_q == lc.L - sy.TINY.R
    K, V = lc.view()
    Ko, Vo = oc.view()
    for a, b in ((K, Ko), (V, Vo)):
        a = a.double().cpu().numpy()
        assert np.all(np.abs(a - b) <= 1e-6 * np.maximum(np.abs(b), np.abs(b).max(-1, keepdims=True)) + 1e-7)


@pytest.mark.parametrize("R", [0, 1])
@pytest.mark.parametrize("kind", [1, 0], ids=["PSA", "TSA"])
def test_exact_r_small_window(ak, orc, sy, kind, R):
    """Exact R with R = 0 (the new token itself leaves the window at once: the
    fused step must append before quantizing it) and R = 1, fused and split
    calls alternating, state and outputs vs the oracle at every step."""
    import dataclasses
    w = dataclasses.replace(sy.TINY, name=f"tiny_er_r{R}", R=R)
    lc, oc, _ = _run_case(ak, orc, sy, w, 0, kind=kind, steps=16, k_axis=1, exact_r=1)
    assert lc.n_q == lc.L - R


@pytest.mark.parametrize("layer", [0, 2], ids=["TSA-L0", "PSA-L2"])
def test_llava7b_exact_r(ak, orc, sy, layer):
    _run_case(ak, orc, sy, sy.LLAVA7B, layer, steps=6, units=[0, 13, 31], k_axis=1, exact_r=1)


def test_full_size_exact_r_sampled(ak, orc, sy):
    w = sy.get("sweep@b16")
    _run_case(ak, orc, sy, w, 2, steps=3, units=[0, w.U // 2, w.U - 1], k_axis=1, exact_r=1)


@pytest.mark.parametrize("g", [2, 7])
def test_gqa_exact_r(ak, orc, sy, g):
    import dataclasses
    w = dataclasses.replace(sy.TINY, name=f"tiny_er_g{g}", hq=4 * g, hkv=4)
    _run_case(ak, orc, sy, w, 0, kind=0, steps=16, k_axis=1, exact_r=1)


def test_exact_r_errors(ak, sy):
    w = sy.TINY
    with pytest.raises(ak.AkvqError):     # exact R needs per-token K (EINVAL)
        ak.LayerCache(ak.make_config(w.U, w.g, w.d, w.G, w.R, w.capacity, w.top_k, 1,
                                     ak.AKVQ_BF16, k_axis=0, exact_r=1))


@pytest.mark.parametrize("g", [3, 7])
def test_gqa_per_token_k(ak, orc, sy, g):
    """Per-token K (NEXT-1) with g >= 3 query heads per kv head runs on the generic
    split kernels (the single-pass GQA kernel is per-channel only)."""
    import dataclasses
    w = dataclasses.replace(sy.TINY, name=f"tiny_kt_g{g}", hq=4 * g, hkv=4)
    _run_case(ak, orc, sy, w, 0, kind=1, steps=12, k_axis=1)


# ------------------------------------------------- sharding equivalence
_STATE_FIELDS = ("kscale", "kzero", "kcodes", "vscale", "vzero", "vcodes", "ring", "salient",
                 "side_idx", "side_cnt")
_SIDE_FIELDS = {1: ("side16",), 0: ("side4_kscale", "side4_kzero", "side4_vscale", "side4_vzero",
                                     "side4_k", "side4_v")}


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("layer", [2, 0], ids=["PSA-L2", "TSA-L0"])
def test_sharding_equivalence(ak, orc, sy, world, layer):
    """SURVEY 8(e) on one GPU: every rank's unit range (shard.unit_range, b-major
    batch x kv-head units) run as its own cache -- the per-rank shape a world-N
    job runs -- gives the same cache state bit for bit and the same outputs (within
    1e-5; the only difference is the item split across warps, i.e. the order of the
    segment merge) as the unsharded cache, across a flush; the first unit of every
    rank is also checked against the oracle (2e-3).  sweep@b16 shape (BJ:9)."""
    from paper_2501_15021_b200 import shard
    w = sy.get("sweep@b16")
    U = w.U
    steps = 4
    gcfg, _ = _configs(ak, orc, w, layer, U)
    inp = sy.layer_inputs(w, layer, device="cuda")
    full = ak.LayerCache(gcfg)
    full.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    shards = []
    for r in range(world):
        lo, hi = shard.unit_range(U, world, r)
        cfg_r, _ = _configs(ak, orc, w, layer, hi - lo)
        lc = ak.LayerCache(cfg_r)
        lc.prefill(inp["K"][lo:hi], inp["V"][lo:hi], inp["types"][lo:hi], inp["colsum"][lo:hi])
        shards.append((lo, hi, lc))
    firsts = [lo for lo, _, _ in shards]
    _, ocfg = _configs(ak, orc, w, layer, len(firsts))
    oc = orc.OracleCache(ocfg)
    io = sy.layer_inputs(w, layer, units=firsts, device="cpu")
    assert oc.prefill(f16_bits(io["K"]), f16_bits(io["V"]), io["types"].numpy(),
                      io["colsum"].numpy()) == 0

    def same_state():
        gs = GpuState(full)
        for lo, hi, lc in shards:
            s = GpuState(lc)
            assert (s.L, s.n_q) == (gs.L, gs.n_q)
            assert np.array_equal(gs.side_cnt[lo:hi], s.side_cnt)
            sc = int(s.side_cnt.max(initial=0))
            for f in _STATE_FIELDS + _SIDE_FIELDS[gcfg.kind]:
                a, b = getattr(gs, f)[lo:hi], getattr(s, f)
                # live regions only: pages / token rows below n_q, ring rows
                # [n_q, L), bits below L, side entries below the largest count
                n = {"kscale": s.n_q // w.G, "kzero": s.n_q // w.G, "ring": s.L - s.n_q,
                     "salient": s.L}.get(f, sc if f.startswith("side") and f != "side_cnt" else s.n_q)
                if f == "ring":                                   # slot of token t: t % slots
                    live = np.arange(s.n_q, s.L) % s.ring.shape[1]
                    a, b = a[:, live], b[:, live]
                elif f != "side_cnt":
                    a, b = a[:, :n], b[:, :n]
                if f.startswith("side") and f != "side_cnt":     # per-unit counts
                    keep = np.arange(n)[None, :] < s.side_cnt[:, None]
                    a, b = a[keep], b[keep]
                assert np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                                      np.ascontiguousarray(b).view(np.uint8)), f"{f} differs on [{lo},{hi})"

    same_state()
    # step past the next flush (n_q + G + R - L steps, Eq. 2 / R4 schedule)
    nq_start = full.n_q
    steps = max(steps, nq_start + w.G + w.R - full.L + 2)
    worst_shard, worst_orc = 0.0, 0.0
    for step in range(steps):
        di = sy.decode_inputs(w, layer, step, device="cuda")
        nq0 = full.n_q
        out = full.step(di["k"], di["v"], di["q"], di["types"]).clone()
        do = sy.decode_inputs(w, layer, step, units=firsts, device="cpu")
        oc.append(f16_bits(do["k"]), f16_bits(do["v"]), do["types"].numpy())
        ref = oc.decode(f16_bits(do["q"]))
        for j, (lo, hi, lc) in enumerate(shards):
            o = lc.step(di["k"][lo:hi], di["v"][lo:hi], di["q"][lo:hi], di["types"][lo:hi])
            worst_shard = max(worst_shard, float((o - out[lo:hi]).abs().max()))
            worst_orc = max(worst_orc, float(np.abs(o[0].double().cpu().numpy() - ref[j]).max()))
        if full.n_q != nq0:
            same_state()
    record_margin(_case_name(), worst_shard, 1e-5, None, worst_out_err_oracle=worst_orc)
    assert full.n_q > nq_start, "no flush exercised"
    assert worst_shard <= 1e-5, worst_shard
    assert worst_orc <= OUT_TOL, worst_orc
