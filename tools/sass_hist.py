#!/usr/bin/env python3
"""Static SASS opcode histogram of the hot kernels in libakvq.so (cuobjdump), as
checkable evidence of the instruction mix: warp MMA (IMMA), TMA bulk copies
(UBLKCP), mbarrier waits (SYNCS), programmatic-launch controls, shuffles.

    python tools/sass_hist.py [--lib paper_2501_15021_b200/libakvq.so] > profiles/r02/sass_opcodes.md
"""
import argparse
import collections
import re
import subprocess

KERNELS = [
    ("k_decode_layer<128,128,bf16,NH=1,PSA,per-channel>", "_ZN4akvq14k_decode_layerILi128ELi128ELi0ELi1ELb0ELi0ELb0EEEvNS_8DevCacheENS_9LayerPlanEPKtS4_S4_PKhPfS7_j"),
    ("k_decode_layer<128,128,bf16,NH=1,TSA,per-channel>", "_ZN4akvq14k_decode_layerILi128ELi128ELi0ELi1ELb1ELi0ELb0EEEvNS_8DevCacheENS_9LayerPlanEPKtS4_S4_PKhPfS7_j"),
    ("k_decode_gqa<128,128,bf16,NH=8,PSA>", "_ZN4akvq12k_decode_gqaILi128ELi128ELi0ELi8ELb0EEEvNS_8DevCacheENS_9LayerPlanEPKtS4_S4_PKhPfS7_j"),
    ("k_quantize_blocks<128,128,bf16,per-channel>", "_ZN4akvq17k_quantize_blocksILi128ELi128ELi0ELb0EEEvNS_8DevCacheENS_8QuantSrcEii"),
    ("k_quantize_tokens<128,128,bf16> (exact R, R26)", "_ZN4akvq17k_quantize_tokensILi128ELi128ELi0EEEvNS_8DevCacheENS_8QuantSrcEii"),
]
WATCH = ["IMMA", "HMMA", "UTCMMA", "UBLKCP", "UTMALDG", "SYNCS", "ACQBULK", "SHFL", "LOP3", "PRMT",
         "I2FP", "F2I", "MUFU", "FFMA", "FFMA2", "FMUL2", "LDS", "STS", "LDG", "STG", "ATOM", "RED",
         "BAR", "WARPSYNC", "BSSY", "BRA", "ELECT"]


def hist(lib, fn):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun", fn, lib],
                         capture_output=True, text=True).stdout
    ops = re.findall(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", out, re.M)
    return collections.Counter(ops), len(ops)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="paper_2501_15021_b200/libakvq.so")
    a = ap.parse_args()
    print("# SASS opcode histograms (static, `cuobjdump -sass`, sm_100a)\n")
    print("Static instruction counts per kernel (not execution counts); the dynamic mix is "
          "in the ncu captures.  Legacy warp MMA = IMMA.16832 (mma.sync m16n8k32 int8); "
          "TMA bulk copy = UBLKCP; mbarrier = SYNCS.*.\n")
    for name, fn in KERNELS:
        h, n = hist(a.lib, fn)
        if n == 0:
            continue
        print(f"## {name}\n\n{n} instructions.\n")
        print("| opcode | count |\n|---|---|")
        for op in WATCH:
            if h.get(op):
                print(f"| {op} | {h[op]} |")
        top = ", ".join(f"{k} {v}" for k, v in h.most_common(12))
        print(f"\nTop: {top}\n")


if __name__ == "__main__":
    main()
