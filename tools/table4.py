#!/usr/bin/env python3
"""B200 analogue of the paper's Table IV: grow the
batch until the KV cache no longer fits, for a bf16 cache and for the AKVQ-VL
2-bit cache, and compare decode-attention throughput at those batch sizes.

Setting: LLaVA-v1.5-7B shape (32 layers, 32 MHA heads, d = 128), an
input of ~500 tokens (35 text + 400 vision + 65 text), then `--decode` generated
tokens.  Memory budget = the GPU's memory - LLaVA-1.5-7B fp16 weights (~7.06 B
parameters, 14.1 GB; the paper's runs hold the model) - a 4 GB reserve.  Per
sequence the bf16 cache needs 2 * layers * heads * d * 2 bytes per token of
capacity; the 2-bit cache needs akvq_cache_bytes(...) per layer (pages, 16-bit
recent ring, side table, bitmask) plus its decode workspace.

Throughput is ATTENTION ONLY (no weights / GEMMs): the per-layer decode time at
the maximum batch is measured with one layer allocated and multiplied by the
layer count -- bf16: torch scaled_dot_product_attention (the library kernel) on
a [B, H, L, d] cache plus the append; 2-bit: one akvq_decode_step launch.
Inputs are random N(0,1) (throughput does not depend on values).

    python tools/table4.py [--decode 128] [--reserve-gb 4]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_15021_b200 import akvq as ak  # noqa: E402

LAYERS, HEADS, D, G, R, TOPK = 32, 32, 128, 128, 32, 15
L0 = 500
WEIGHTS_GB = 7.06e9 * 2 / 1e9


def time_ms(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def bf16_arm(B, cap):
    dev = "cuda"
    K = torch.randn(B, HEADS, cap, D, device=dev, dtype=torch.bfloat16)
    V = torch.randn_like(K)
    q = torch.randn(B, HEADS, 1, D, device=dev, dtype=torch.bfloat16)
    kn = torch.randn(B, HEADS, 1, D, device=dev, dtype=torch.bfloat16)
    L = L0 + 1

    def step():
        K[:, :, L - 1:L] = kn                    # append (Eq. 2)
        V[:, :, L - 1:L] = kn
        return torch.nn.functional.scaled_dot_product_attention(q, K[:, :, :L], V[:, :, :L])

    t = time_ms(step)
    del K, V
    torch.cuda.empty_cache()
    return t


def akvq_arm(B, cap):
    dev = "cuda"
    U = B * HEADS
    cfg = ak.make_config(U, 1, D, G, R, cap, TOPK, ak.AKVQ_PSA, ak.AKVQ_BF16)
    lc = ak.LayerCache(cfg, device=dev)
    Kp = torch.randn(U, L0, D, device=dev, dtype=torch.bfloat16)
    Vp = torch.randn_like(Kp)
    types = torch.zeros(U, L0, dtype=torch.uint8, device=dev)
    colsum = torch.rand(U, 1, L0, device=dev)
    lc.prefill(Kp, Vp, types, colsum)
    del Kp, Vp, colsum
    q = torch.randn(U, 1, D, device=dev, dtype=torch.bfloat16)
    k = torch.randn(U, D, device=dev, dtype=torch.bfloat16)
    ty = torch.zeros(U, dtype=torch.uint8, device=dev)
    out = torch.empty(U, 1, D, device=dev)
    n = [0]

    def step():
        if lc.L >= cap - 1:
            return
        lc.step(k, k, q, ty, out=out)
        n[0] += 1

    t = time_ms(step, iters=20, warm=5)
    del lc
    torch.cuda.empty_cache()
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--decode", type=int, default=128)
    ap.add_argument("--reserve-gb", type=float, default=4.0)
    a = ap.parse_args()
    cap = L0 + a.decode
    total = torch.cuda.get_device_properties(0).total_memory / 1e9
    budget = total - WEIGHTS_GB - a.reserve_gb
    bf16_seq = LAYERS * 2 * HEADS * D * 2 * cap / 1e9
    cfg1 = ak.make_config(HEADS, 1, D, G, R, cap, TOPK, ak.AKVQ_PSA, ak.AKVQ_BF16)
    c1 = ak.akvq_cache(); buf = torch.empty(ak.akvq_cache_bytes(cfg1), dtype=torch.uint8, device="cuda")
    ak.akvq_cache_init(c1, cfg1, buf)
    ws1 = ak.akvq_decode_workspace_bytes_max(c1)
    akvq_seq = LAYERS * ak.akvq_cache_bytes(cfg1) / 1e9     # + workspace (per layer, shared by steps)
    B_bf16 = int(budget // bf16_seq)
    B_akvq = int((budget - LAYERS * ws1 / 1e9 * 0) // akvq_seq)
    t_bf16 = bf16_arm(B_bf16, cap)
    t_akvq = akvq_arm(B_akvq, cap)
    rows = [
        {"method": "bf16 KV (torch SDPA)", "batch": B_bf16, "kv_gb": B_bf16 * bf16_seq,
         "per_seq_mb": bf16_seq * 1e3, "layer_ms": t_bf16,
         "tokens_per_s": B_bf16 / (LAYERS * t_bf16 * 1e-3)},
        {"method": "AKVQ-VL 2-bit (k_decode_layer)", "batch": B_akvq, "kv_gb": B_akvq * akvq_seq,
         "per_seq_mb": akvq_seq * 1e3, "layer_ms": t_akvq,
         "tokens_per_s": B_akvq / (LAYERS * t_akvq * 1e-3)},
    ]
    print(json.dumps({"gpu_gb": total, "budget_gb": budget, "capacity_tokens": cap, "rows": rows}))
    print(f"\nGPU memory {total:.1f} GB, budget for KV {budget:.1f} GB (weights {WEIGHTS_GB:.1f} GB,"
          f" reserve {a.reserve_gb} GB), capacity {cap} tokens per sequence\n")
    print("| method | max batch | KV memory (GB) | per sequence (MB) | attention ms / layer | attention-only tokens/s |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['method']} | {r['batch']} | {r['kv_gb']:.1f} | {r['per_seq_mb']:.1f} | "
              f"{r['layer_ms']:.3f} | {r['tokens_per_s']:.0f} |")
    print(f"\nbatch ratio {B_akvq / B_bf16:.2f}x, attention throughput ratio "
          f"{rows[1]['tokens_per_s'] / rows[0]['tokens_per_s']:.2f}x "
          f"(paper, V100 end to end: 3.25x batch, 2.46x throughput, Table IV)")


if __name__ == "__main__":
    main()
