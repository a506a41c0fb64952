#!/bin/bash
# quick GPU iteration: parity tests, then bench variants. Usage: bash tools/gpu_quick.sh TAG [notests]
TAG=${1:-q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$2" != "notests" ]; then
  timeout -k 10 900 python -m pytest tests -m gpu -x -q --timeout 300 -o timeout_method=thread > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/tests.log
fi
i=0
for opt in "" "--skip-rows" "--skip-pages" "--stream-only" "--skip-pages --stream-only" "--skip-rows --stream-only"; do
  i=$((i+1))
  timeout -k 10 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $opt > $OUT/bench$i.json 2> $OUT/bench$i.err
  python -c "import json,sys; j=json.loads(open('$OUT/bench$i.json').read().strip().splitlines()[-1]); print('$opt'.ljust(28), round(j['value']), round(j['ms_per_step'],3), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -5 $OUT/bench$i.err
done
