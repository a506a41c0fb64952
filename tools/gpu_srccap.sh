#!/bin/bash
# Full ncu capture with source counters of one launch: bash tools/gpu_srccap.sh TAG KREGEX SKIP [bench args]
TAG=$1; K=$2; SK=$3; shift 3
mkdir -p gpurun_out/$TAG
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SK -c 1 -o gpurun_out/$TAG/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-strong-emulation "$@" > gpurun_out/$TAG/ncu.log 2>&1; echo "ncu $TAG rc=$?"
ncu -i gpurun_out/$TAG/full.ncu-rep --page raw --csv > gpurun_out/$TAG/raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG/full.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/$TAG/src.csv 2>/dev/null
rm -f gpurun_out/$TAG/full.ncu-rep
