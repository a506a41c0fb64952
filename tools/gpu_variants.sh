mkdir -p gpurun_out/r01b
for opt in "--stream-only" "--skip-rows" "--skip-pages" "--stream-only --skip-rows" ""; do
  echo "== $opt" >> gpurun_out/r01b/variants.log
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $opt 2>&1 | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['value'], j['ms_per_step'], j['roofline']['launch_ms'], j['roofline']['frac'], j['gpu_launches'])" >> gpurun_out/r01b/variants.log 2>&1
done
bash tools/gpu_round.sh r01b launches
