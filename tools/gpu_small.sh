#!/bin/bash
# Small-shape latency vs the per-warp item floor: bash tools/gpu_small.sh
mkdir -p gpurun_out/small
for wl in llava7b sweep@b8 sweep@b16; do for m in 1 2 4; do
  AKVQ_MIN_ITEMS=$m timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-strong-emulation > gpurun_out/small/b.json 2> gpurun_out/small/b.err
  python -c "import json; j=json.loads(open('gpurun_out/small/b.json').read().strip().splitlines()[-1]); print('$wl min_items=$m'.ljust(28), round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -3 gpurun_out/small/b.err
done; done
