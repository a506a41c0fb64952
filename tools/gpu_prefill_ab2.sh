#!/bin/bash
# A/B of quantize-kernel variants: bash tools/gpu_prefill_ab2.sh ROUNDS lib1.so lib2.so ...
# (prefill = the 32-layer prompt quantization of bench.py's workload)
R=$1; shift; mkdir -p gpurun_out/ab
for r in $(seq $R); do for L in "$@"; do
  AKVQ_LIB=$PWD/$L timeout -k 10 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-strong-emulation $BENCH_ARGS > gpurun_out/ab/p.json 2> gpurun_out/ab/p.err
  python -c "import json; j=json.loads(open('gpurun_out/ab/p.json').read().strip().splitlines()[-1]); p=j['prefill']; print('$L'.ljust(24), round(p['ms_all_layers'],2), 'ms', round(p['frac'],3), round(j['roofline']['launch_ms']*1000,1), 'us')" || tail -3 gpurun_out/ab/p.err
done; done
