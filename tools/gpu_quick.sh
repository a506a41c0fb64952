#!/bin/bash
# Quick check on the box: a subset of GPU parity tests + a short bench line.
# Usage: bash tools/gpu_quick.sh TAG [pytest -k expression] [bench args...]
TAG=${1:-q}; K=${2:-"tiny or llava7b_layer_full or full_size_sampled or gqa_head_groups"}; shift; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > $OUT/tests.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/tests.log
timeout -k 10 600 python bench.py --no-cpu-baseline --steps 20 "$@" > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "import json;j=json.load(open('$OUT/bench.json'));print('tok/s %.0f  launch_us %.2f  frac %.4f' % (j['value'], 1e3*j['roofline']['launch_ms'], j['roofline']['frac']))"
