mkdir -p gpurun_out/q1
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:k_quantize_blocks -s 4 -c 1 -o gpurun_out/q1/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-strong-emulation > gpurun_out/q1/ncu.log 2>&1; echo rc=$?
ncu -i gpurun_out/q1/full.ncu-rep --page raw --csv > gpurun_out/q1/raw.csv 2>/dev/null
ncu -i gpurun_out/q1/full.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/q1/src.csv 2>/dev/null
ncu -i gpurun_out/q1/full.ncu-rep --page source --csv --print-source cuda > gpurun_out/q1/src_cuda.csv 2>/dev/null
rm -f gpurun_out/q1/full.ncu-rep; ls -la gpurun_out/q1
