#!/bin/bash
OUT=gpurun_out/${1:-sw2}; mkdir -p $OUT
for cfg in "4 1 4" "8 1 3" "8 1 4" "4 2 3" "16 1 3" "8 2 2"; do set -- $cfg
  AKVQ_ROW_WARPS=$1 AKVQ_ROW_CTAS=$2 AKVQ_PG_CTAS=$3 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/b.json 2>$OUT/b.err
  python -c "import json; j=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print('rowwarps',$1,'rowctas',$2,'pgctas',$3, round(j['value']), round(j['roofline']['launch_ms']*1000,1), 'us', round(j['roofline']['frac'],3))" || tail -3 $OUT/b.err
done
