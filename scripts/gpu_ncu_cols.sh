# ncu --set full of the C pass (cols_pipe_kernel) on config 5, correction and direct form
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > gpurun_out/plain5.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cols_pipe" -s 1 -c 1 -o gpurun_out/prof_cols5 $CMD > gpurun_out/ncu5.log 2>&1
tail -1 gpurun_out/ncu5.log
python scripts/ncu_brief.py gpurun_out/prof_cols5.ncu-rep
