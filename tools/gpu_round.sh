#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + full capture.
# Usage (on the box): bash tools/gpu_round.sh TAG [what...]   what in {tests,smoke,bench,launches,full}
TAG=${1:-r01}; shift
WHAT=${@:-tests smoke bench launches full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
for w in $WHAT; do
  case $w in
    tests)  AKVQ_MARGINS_OUT=$OUT/parity_margins.json timeout -k 10 1800 python -m pytest tests -m gpu -q -rf --timeout 400 -o timeout_method=thread > $OUT/tests.log 2>&1; echo "tests rc=$?" ;;
    shapes) bash tools/gpu_shapes.sh $TAG/shapes ;;
    smoke)  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)  timeout -k 10 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json ;;
    launches) timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
               -k regex:"k_(decode|append|quantize|salient|ring|view|combine)" --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-strong-emulation > $OUT/ncu_launch.log 2>&1; echo "launches rc=$?" ;;
    full)   for k in ${KERNELS:-k_decode_layer}; do
              timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 200 -c 1 \
                -o $OUT/full_$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-strong-emulation > $OUT/ncu_full_$k.log 2>&1; echo "full $k rc=$?"; ncu -i $OUT/full_$k.ncu-rep --page raw --csv > $OUT/raw_$k.csv 2>/dev/null; ncu -i $OUT/full_$k.ncu-rep --page details --csv > $OUT/details_$k.csv 2>/dev/null; rm -f $OUT/full_$k.ncu-rep
            done ;;
  esac
done
