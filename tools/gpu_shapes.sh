#!/bin/bash
# Other-shape bench lines for profiles/r01_final_summary.md: bash tools/gpu_shapes.sh TAG
TAG=${1:-shapes}; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { n=$1; shift; timeout -k 10 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > $OUT/$n.json 2> $OUT/$n.err
  python -c "import json; j=json.loads(open('$OUT/$n.json').read().strip().splitlines()[-1]); print('$n'.ljust(16), round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -3 $OUT/$n.err; }
run sweep_b8 --workload sweep@b8
run sweep_b16 --workload sweep@b16
run sweep_b32 --workload sweep@b32
run llava7b --workload llava7b
run video13b --workload video13b
run qwen --workload qwen_gqa
run ktoken --k-axis token
run massive --pivots massive
run ktoken_exact --k-axis token-exact
