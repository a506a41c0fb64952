#!/bin/bash
# A/B of library variants on one workload: bash tools/gpu_ab_w.sh WORKLOAD ROUNDS lib1.so lib2.so ...
W=$1; R=$2; shift 2; mkdir -p gpurun_out/ab
for r in $(seq $R); do for L in "$@"; do
  AKVQ_LIB=$PWD/$L timeout -k 10 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab/b.json 2> gpurun_out/ab/b.err
  python -c "import json; j=json.loads(open('gpurun_out/ab/b.json').read().strip().splitlines()[-1]); print('$W $L'.ljust(40), round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -3 gpurun_out/ab/b.err
done; done
