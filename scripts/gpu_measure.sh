# Round measurement: full bench line (config 5), launch list, ncu --set full of the dominant kernel,
# plus bench lines for configs 3 and 4.
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cat gpurun_out/bench_full.json | head -c 400; echo
for c in 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2>> gpurun_out/bench_full.err; done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain_full.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${TOPK:-fft2d_cols}" -s 2 -c 1 -o gpurun_out/prof_cfg5_top $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
