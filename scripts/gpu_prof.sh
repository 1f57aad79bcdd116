set -x
./scripts/fp64_peak > gpurun_out/fp64_peak.json 2>&1
CMD="python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|fft2d|bwd_kernel" -s 5 -c 5 -o gpurun_out/prof4_v1 $CMD > gpurun_out/ncu_full4.log 2>&1
echo finished
