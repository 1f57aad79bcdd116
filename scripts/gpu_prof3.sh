CMD="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pcr|fwd_kernel|bwd_kernel" -s 4 -c 4 -o gpurun_out/prof3_${TAG:-v1} $CMD > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
