#!/bin/bash
# GPU iteration: parity tests (stop at first failure) then N bench runs. Usage: bash tools/gpu_tb.sh TAG [NRUNS] [extra bench args]
TAG=${1:-tb}; N=${2:-2}; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout -k 10 900 python -m pytest tests -m gpu -x -q --timeout 300 -o timeout_method=thread > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/tests.log
for i in $(seq $N); do
  timeout -k 10 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline "$@" > $OUT/b$i.json 2> $OUT/b$i.err
  python -c "import json; j=json.loads(open('$OUT/b$i.json').read().strip().splitlines()[-1]); print(round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3), j['e2e']['value'], j['clocks'])" || tail -5 $OUT/b$i.err
done
