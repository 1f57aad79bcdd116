CMD="python bench.py --config 5 --grid 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain5s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel|fft2d" -s 5 -c 5 -o gpurun_out/prof5s_v2 $CMD > gpurun_out/ncu5s.log 2>&1
tail -2 gpurun_out/ncu5s.log
