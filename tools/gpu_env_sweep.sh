#!/bin/bash
# env-knob sweep on one workload: bash tools/gpu_env_sweep.sh WORKLOAD "ENV1=a" "ENV1=b" ...
W=$1; shift; mkdir -p gpurun_out/ab
for e in "$@"; do
  env $e timeout -k 10 600 python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab/e.json 2> gpurun_out/ab/e.err
  python -c "import json; j=json.loads(open('gpurun_out/ab/e.json').read().strip().splitlines()[-1]); print('$W $e'.ljust(40), round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us')" || tail -3 gpurun_out/ab/e.err
done
