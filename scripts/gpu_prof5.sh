CMD="python bench.py --config 5 --grid 128 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain5s.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tfft_fwd|fft2d_rows|fft2d_cols" -s 4 -c 3 -o gpurun_out/prof5s_v5 $CMD > gpurun_out/ncu5s.log 2>&1
tail -2 gpurun_out/ncu5s.log
