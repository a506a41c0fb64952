#!/usr/bin/env python3
"""Attention-output quality of the 2-bit cache (SURVEY NEXT-1 report).

For a workload's layer (synthetic LLaVA-shaped inputs with K outlier channels),
runs prefill + decode steps through libakvq.so for both K axes -- per channel
over G-token blocks (R1, graded) and per token over G-channel groups,
the latter also with the exact residual window (R26: exactly R 16-bit rows) --
and compares each decode output with plain unquantized attention computed in
fp64 by torch on the CPU over the same 16-bit rows (q.K^T/sqrt d, softmax, .V).
Reports cosine similarity and relative L2 error per layer kind (mean / min
over sampled units and steps).  Product path only (no oracle): this measures the
METHOD's approximation, not kernel parity (that is tests/test_gpu_parity.py).

WHT arms (the paper's "+ WHT" ablation row, Table III; motivation
P:305-308): "on" is the library as is.  "off" feeds every row already
multiplied by H (K.H, V.H, q.H): the library's own rotation then gives
K.H.H = K (H is an involution), so the cache quantizes the UNROTATED channels,
while attention is unchanged (H orthonormal); outputs are compared with plain
attention over the same fed rows.

    python tools/quality_report.py [--workload llava7b] [--steps 8] [--units 64]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_15021_b200 import akvq as ak, synth  # noqa: E402


def reference(Kall, Vall, q):
    """fp64 attention of q [n, g, d] over rows [n, L, d] (16-bit values widened)."""
    d = q.shape[-1]
    s = torch.einsum("ngd,nld->ngl", q, Kall) / d ** 0.5
    return torch.einsum("ngl,nld->ngd", torch.softmax(s, -1), Vall)


def run(w, layer, k_axis, steps, units, wht=True, exact_r=0):
    dt = ak.AKVQ_BF16 if w.dtype == "bf16" else ak.AKVQ_FP16
    cfg = ak.make_config(w.U, w.g, w.d, w.G, w.R, w.L0 + steps, w.top_k, w.kind(layer), dt,
                         w.clip2, w.clip4, k_axis, exact_r=exact_r)
    lc = ak.LayerCache(cfg)
    inp = synth.layer_inputs(w, layer, device="cuda")
    tdt = inp["K"].dtype
    if not wht:
        import scipy.linalg
        H = torch.tensor(scipy.linalg.hadamard(w.d) / w.d ** 0.5, dtype=torch.float32, device="cuda")
        pre = lambda x: (x.float() @ H).to(tdt)
        inp = dict(inp, K=pre(inp["K"]), V=pre(inp["V"]))
    else:
        pre = lambda x: x
    lc.prefill(inp["K"], inp["V"], inp["types"], inp["colsum"])
    Kall = inp["K"][units].double().cpu()
    Vall = inp["V"][units].double().cpu()
    cos, rel = [], []
    for s in range(steps):
        di = synth.decode_inputs(w, layer, s, device="cuda")
        di = dict(di, k=pre(di["k"]), v=pre(di["v"]), q=pre(di["q"]))
        out = lc.step(di["k"], di["v"], di["q"], di["types"])[units].double().cpu()
        Kall = torch.cat([Kall, di["k"][units].double().cpu()[:, None]], 1)
        Vall = torch.cat([Vall, di["v"][units].double().cpu()[:, None]], 1)
        ref = reference(Kall, Vall, di["q"][units].double().cpu())
        cos.append(torch.nn.functional.cosine_similarity(out.flatten(1), ref.flatten(1)))
        rel.append((out - ref).flatten(1).norm(dim=1) / ref.flatten(1).norm(dim=1))
    cos, rel = torch.cat(cos), torch.cat(rel)
    return {"cos_mean": float(cos.mean()), "cos_min": float(cos.min()),
            "rel_l2_mean": float(rel.mean()), "rel_l2_max": float(rel.max())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llava7b")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--units", type=int, default=64)
    a = ap.parse_args()
    w = synth.get(a.workload)
    units = torch.linspace(0, w.U - 1, min(a.units, w.U)).round().long().unique()
    psa = next(l for l in range(w.n_layers) if w.kind(l) == 1)
    tsa = next((l for l in range(w.n_layers) if w.kind(l) == 0), None)
    rows = []
    for layer in [l for l in (tsa, psa) if l is not None]:
        for wht in (True, False):
            for k_axis, ex, name in ((0, 0, "per-channel K (R1)"), (1, 0, "per-token K (P:246)"),
                                     (1, 1, "per-token K, exact R (R26)")):
                r = run(w, layer, k_axis, a.steps, units, wht, ex)
                r.update(layer=layer, kind="TSA" if w.kind(layer) == 0 else "PSA", k_axis=name,
                         wht="on" if wht else "off")
                rows.append(r)
                print(json.dumps(r), flush=True)
    print("\n| layer | kind | WHT | K axis | cos mean | cos min | rel L2 mean | rel L2 max |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['layer']} | {r['kind']} | {r['wht']} | {r['k_axis']} | {r['cos_mean']:.5f} | "
              f"{r['cos_min']:.5f} | {r['rel_l2_mean']:.4f} | {r['rel_l2_max']:.4f} |")


if __name__ == "__main__":
    main()
