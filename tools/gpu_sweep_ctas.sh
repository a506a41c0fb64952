#!/bin/bash
OUT=gpurun_out/${1:-sw}; mkdir -p $OUT
for rc in 3 1 2; do for pc in 4 3; do
  AKVQ_ROW_CTAS=$rc AKVQ_PG_CTAS=$pc timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/b_$rc_$pc.json 2>/dev/null
  python -c "import json; j=json.loads(open('$OUT/b_$rc_$pc.json').read().strip().splitlines()[-1]); print('rows',$rc,'pages',$pc, round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))"
done; done
