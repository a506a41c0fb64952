#!/bin/bash
# Lightweight ncu of one k_decode_layer launch (after warm-up): duration, instruction
# count, issue activity, stall reasons.  Usage: bash tools/gpu_ncu_quick.sh TAG [bench args]
TAG=${1:-nq}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout -k 10 600 ncu --clock-control none ${KNB:+--kernel-name-base $KNB} -k regex:${KREGEX:-k_decode_layer} -s ${SKIP:-200} -c 1 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active,dram__bytes_read.sum,smsp__average_warp_latency_per_inst_issued.ratio,smsp__pcsamp_warps_issue_stalled_wait,smsp__pcsamp_warps_issue_stalled_short_scoreboard,smsp__pcsamp_warps_issue_stalled_long_scoreboard,smsp__pcsamp_warps_issue_stalled_selected,smsp__pcsamp_warps_issue_stalled_barrier,smsp__pcsamp_warps_issue_stalled_branch_resolving,smsp__pcsamp_warps_issue_stalled_math_pipe_throttle,smsp__pcsamp_warps_issue_stalled_not_selected,smsp__pcsamp_warps_issue_stalled_no_instructions,smsp__pcsamp_warps_issue_stalled_sleeping,smsp__pcsamp_warps_issue_stalled_membar,smsp__pcsamp_warps_issue_stalled_dispatch_stall,smsp__pcsamp_warps_issue_stalled_mio_throttle,smsp__pcsamp_warps_issue_stalled_lg_throttle,smsp__pcsamp_warps_issue_stalled_tex_throttle,smsp__pcsamp_warps_issue_stalled_drain,smsp__pcsamp_warps_issue_stalled_misc \
  --csv python bench.py --no-cpu-baseline --steps 3 --warmup 3 "$@" > $OUT/ncu.csv 2> $OUT/ncu.err
echo "ncu rc=$?"
python - "$OUT/ncu.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[h]; im = hdr.index("Metric Name"); iv = hdr.index("Metric Value")
vals = {}
for r in rows[h + 1:]:
    if len(r) == len(hdr):
        try: vals[r[im]] = float(r[iv].replace(',', ''))
        except ValueError: pass
st = {k.replace('smsp__pcsamp_warps_issue_stalled_', ''): v for k, v in vals.items() if 'stalled' in k}
tot = sum(st.values()) or 1
for k in ('gpu__time_duration.sum', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
          'sm__warps_active.avg.per_cycle_active', 'dram__bytes_read.sum', 'smsp__average_warp_latency_per_inst_issued.ratio'):
    print(f"{k:60s} {vals.get(k)}")
print("stalls:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01))
PY
