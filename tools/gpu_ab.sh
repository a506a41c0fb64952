#!/bin/bash
# A/B of library variants in one box session: bash tools/gpu_ab.sh ROUNDS lib1.so lib2.so ... (bench only)
R=$1; shift; mkdir -p gpurun_out/ab
for r in $(seq $R); do for L in "$@"; do
  AKVQ_LIB=$PWD/$L timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $BENCH_ARGS > gpurun_out/ab/b.json 2> gpurun_out/ab/b.err
  python -c "import json; j=json.loads(open('gpurun_out/ab/b.json').read().strip().splitlines()[-1]); print('$L'.ljust(24), round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -3 gpurun_out/ab/b.err
done; done
