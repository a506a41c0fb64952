#!/bin/bash
for mi in 1 4 8; do for wl in sweep@b8 sweep@b16 sweep@b64; do
  AKVQ_MIN_ITEMS=$mi timeout -k 10 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('min_items', $mi, '$wl', round(j['value']), round(j['roofline']['frac'],3), round(j['roofline']['launch_ms']*1000,1))"
done; done
