#!/usr/bin/env python3
"""Build library variants of decode_layer.cu with -D flags for GPU A/B runs:
    python tools/build_variants.py NAME='-DX=1 -DY=2' ...  -> build_exp/lib_NAME.so
The other objects come from paper_2501_15021_b200/build/ (run build.py first)."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2501_15021_b200"))
import build as b  # noqa: E402


def one(spec):
    name, flags = spec.split("=", 1)
    out = os.path.join(ROOT, "build_exp", f"var_{name}")
    os.makedirs(out, exist_ok=True)
    objs = []
    qflag = "AKVQ_Q" in flags
    for s in b.SOURCES:
        o = os.path.join(b.BUILD, s.replace(".cu", ".o"))
        api_only = "AKVQ_C" in flags and "AKVQ_MAX_TAB" not in flags
        if (s == "decode_layer.cu" and not api_only and not qflag) or (s == "api.cu" and ("AKVQ_MAX_TAB" in flags or api_only)) \
                or (s == "decode_gqa.cu" and "AKVQ_GQ" in flags) or (s == "quantize.cu" and qflag):
            o = os.path.join(out, s.replace(".cu", ".o"))
            subprocess.run([b.NVCC, *b.FLAGS, *flags.split(), "-c", os.path.join(b.CSRC, s), "-o", o], check=True)
        objs.append(o)
    lib = os.path.join(ROOT, "build_exp", f"lib_{name}.so")
    subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                    "-cudart", "static"], check=True)
    return lib


if __name__ == "__main__":
    with cf.ThreadPoolExecutor(len(sys.argv) - 1) as ex:
        for lib in ex.map(one, sys.argv[1:]):
            print(lib)
