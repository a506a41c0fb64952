"""Randomized operation sequences against the oracle (-m gpu; SPEC acceptance
criterion 8, and prefill == incremental append): >= 10^4 prefill /
append / decode / fused-step operations over many small caches with random
shapes (d, G, R, g, layer kind, K axis, exact residual window, DEVICE_L), every decode output compared
with the oracle (fp32-decision mode, where the kernel's codes agree bit for
bit) and the full cache state compared at the end of every cache's life and at
random points; a twin cache built by appends alone must equal the prefilled one."""
import os

import numpy as np
import pytest
import torch

from parity import GpuState, compare_state, f16_bits

pytestmark = pytest.mark.gpu
OUT_TOL = 2e-3


@pytest.fixture(scope="module")
def ak():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2501_15021_b200 import akvq
    akvq.lib()
    return akvq


def _rows(rng, n, U, d, dt, outlier):
    x = torch.from_numpy(rng.standard_normal((U, n, d))).float()
    x[..., outlier] *= 12.0
    return x.to(dt)


def test_random_operation_sequences(ak, orc):
    rng = np.random.default_rng(int(os.environ.get("AKVQ_RANDOM_SEED", "2501")))
    target = int(os.environ.get("AKVQ_RANDOM_OPS", "10000"))
    ops = states = caches = 0
    counts = {}
    while ops < target:
        d = int(rng.choice([64, 128]))
        G = int(rng.choice([g for g in (32, 64, 128) if g <= d]))
        R = int(rng.choice([0, 4, 16, 40]))
        g = int(rng.choice([1, 1, 2, 3, 7]))
        U = int(rng.integers(1, 4))
        kind = int(rng.integers(0, 2))
        k_axis = int(rng.integers(0, 2)) if g == 1 else 0
        top_k = int(rng.integers(0, 6))
        exact_r = int(rng.integers(0, 2)) if k_axis == 1 else 0      # R26
        dev_L = bool(rng.integers(0, 2)) and not exact_r
        fp16 = bool(rng.integers(0, 2))
        dt = torch.float16 if fp16 else torch.bfloat16
        cap = int(rng.integers(2 * G, 5 * G))
        L0 = int(rng.integers(0, cap // 2))
        gdt = ak.AKVQ_FP16 if fp16 else ak.AKVQ_BF16
        cfg = ak.make_config(U, g, d, G, R, cap, top_k, kind, gdt, 0.8, 1.0, k_axis,
                             exact_r=exact_r)
        lc = ak.LayerCache(cfg, options=ak.AKVQ_OPT_DEVICE_L if dev_L else 0)
        twin = ak.LayerCache(cfg)                              # built by appends only
        oc = orc.OracleCache(orc.OracleConfig(U, g, d, G, R, cap, top_k, kind,
                                              orc.FP16 if fp16 else orc.BF16, k_axis=k_axis,
                                              decide64=0, exact_r=exact_r))
        outl = int(rng.integers(0, d))
        K, V = _rows(rng, L0, U, d, dt, outl), _rows(rng, L0, U, d, dt, outl)
        types = torch.from_numpy((rng.random((U, L0)) < 0.3).astype(np.uint8))
        cs = torch.from_numpy(rng.random((U, g, L0)).astype(np.float32))
        lc.prefill(K.cuda(), V.cuda(), types.cuda(), cs.cuda() if kind == 1 else None)
        assert oc.prefill(f16_bits(K), f16_bits(V), types.numpy(), cs.numpy()) == 0
        # the twin: PSA pivots exist only for prompt tokens, so a twin is a TSA-only check
        use_twin = kind == 0 and L0 > 0
        if use_twin:
            twin.prefill(K[:, :0].cuda(), V[:, :0].cuda(), types[:, :0].cuda(), None)
            for t in range(L0):
                twin.append(K[:, t].contiguous().cuda(), V[:, t].contiguous().cuda(),
                            types[:, t].contiguous().cuda())
        caches += 1
        ops += 1
        while lc.L < cap and ops < target:
            op = rng.choice(["step", "step", "append", "decode"]) if lc.L > 0 else "append"
            counts[op] = counts.get(op, 0) + 1
            k = _rows(rng, 1, U, d, dt, outl)[:, 0]
            v = _rows(rng, 1, U, d, dt, outl)[:, 0]
            ty = torch.from_numpy((rng.random(U) < 0.5).astype(np.uint8))
            q = torch.from_numpy(rng.standard_normal((U, g, d)) * rng.choice([1, 4])).float().to(dt)
            if op in ("step", "append"):
                if op == "step":
                    out = lc.step(k.cuda(), v.cuda(), q.cuda(), ty.cuda())
                else:
                    lc.append(k.cuda(), v.cuda(), ty.cuda())
                if use_twin:
                    twin.append(k.cuda(), v.cuda(), ty.cuda())
                assert oc.append(f16_bits(k), f16_bits(v), ty.numpy()) == 0
            else:
                out = lc.decode(q.cuda())
            if op in ("step", "decode"):
                ref = oc.decode(f16_bits(q))
                err = np.abs(out.double().cpu().numpy() - ref).max()
                assert err <= OUT_TOL, (f"U {cfg.n_units} g {g} d {d} G {G} R {R} kind {kind} "
                                        f"k_axis {k_axis} exact_r {exact_r} dev_L {dev_L} op {op} "
                                        f"L {lc.L} n_q {lc.n_q} err {err}")
            assert (lc.L, lc.n_q) == (oc.L, oc.nq)
            ops += 1
            if rng.random() < 0.01:
                compare_state(GpuState(lc), oc.export(), cfg)
                states += 1
        if lc.L > 0:
            rep = compare_state(GpuState(lc), oc.export(), cfg)
            assert rep["code_ties"] + rep["zero_ties"] <= 2
            states += 1
        if use_twin and lc.L > 0:
            a, b = GpuState(lc), GpuState(twin)
            nq, L = a.n_q, a.L
            nm = nq if k_axis == 1 else nq // G
            assert (b.n_q, b.L) == (nq, L)
            for key, n in (("kcodes", nq), ("vcodes", nq), ("kscale", nm), ("kzero", nm),
                           ("vscale", nq), ("vzero", nq), ("salient", L)):
                assert np.array_equal(getattr(a, key)[:, :n], getattr(b, key)[:, :n]), key
            cnt = a.side_cnt
            assert np.array_equal(cnt, b.side_cnt)
            for u in range(U):
                assert np.array_equal(a.side_idx[u, :cnt[u]], b.side_idx[u, :cnt[u]])
                for t in range(nq, L):
                    assert np.array_equal(a.ring[u, t % a.ring.shape[1]], b.ring[u, t % b.ring.shape[1]])
        del lc, twin, oc
    print(f"random ops: {ops} operations over {caches} caches, {states} state comparisons, {counts}")
    assert ops >= target
