# ncu --set full of the four config-3 (1-D, N = 65536) kernels, plus a launch list
mkdir -p gpurun_out
CMD="python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd|pcr_|bwd_kernel" -s 4 -c 4 -o gpurun_out/prof_cfg3 $CMD > gpurun_out/ncu3.log 2>&1
tail -2 gpurun_out/ncu3.log
python scripts/ncu_brief.py gpurun_out/prof_cfg3.ncu-rep > gpurun_out/prof_cfg3_brief.txt 2>&1
cat gpurun_out/prof_cfg3_brief.txt
