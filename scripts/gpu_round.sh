# Round measurement (1 GPU): all GPU tests, bench lines (config 5 default incl. cpu_baseline/e2e,
# config 5 direct form, Hermitian mode both forms, configs 3 and 4), ncu launch list and ncu --set full
# of the dominant kernel, microbenchmarks.
set -x
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/gpu_tests_all.log 2>&1
tail -3 gpurun_out/gpu_tests_all.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --form direct --no-cpu-baseline > gpurun_out/bench_cfg5_direct.json 2>> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --hermitian --no-cpu-baseline > gpurun_out/bench_cfg5_herm.json 2>> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --form direct --hermitian --no-cpu-baseline > gpurun_out/bench_cfg5_direct_herm.json 2>> gpurun_out/bench_cfg5.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2>> gpurun_out/bench_cfg5.err; done
timeout 600 python bench.py --config 3 --hermitian --no-cpu-baseline > gpurun_out/bench_cfg3_herm.json 2>> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config 4 --hermitian --no-cpu-baseline > gpurun_out/bench_cfg4_herm.json 2>> gpurun_out/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>> gpurun_out/bench_cfg5.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > gpurun_out/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain_full.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${TOPK:-spatial2d}" -s 1 -c 1 -o gpurun_out/prof_cfg5_top $CMD > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
