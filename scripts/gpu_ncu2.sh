# ncu --set full on config 5: register-engine kernels, then the legacy time-FFT kernel (A/B)
CMD="python bench.py --config ${CFG:-5} --form correction --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
export PINT_TFFT_DB=0
$CMD > gpurun_out/plain_ncu.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tfft_reg|spatial2d" -s 3 -c 2 -o gpurun_out/prof_reg5b $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
PINT_LEGACY2D=1 $CMD > gpurun_out/plain_ncu2.log 2>&1 && PINT_LEGACY2D=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tfft_fwd|fft2d_rows" -s 2 -c 2 -o gpurun_out/prof_leg5 $CMD > gpurun_out/ncu_full2.log 2>&1
tail -1 gpurun_out/ncu_full2.log
