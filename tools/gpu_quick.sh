#!/bin/bash
# quick GPU iteration: parity tests, then bench variants. Usage: bash tools/gpu_quick.sh TAG [bench-args]
TAG=${1:-q}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
for opt in "" "--skip-rows" "--skip-pages" "--stream-only"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $opt "$@" > $OUT/bench$opt.json 2> $OUT/bench$opt.err
  python -c "import json,sys; j=json.loads(open('$OUT/bench$opt.json').read().strip().splitlines()[-1]); print('$opt', round(j['value']), round(j['ms_per_step'],3), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3), 'prefill_ms', round(j['prefill']['ms_all_layers'],1))" || tail -5 $OUT/bench$opt.err
done
