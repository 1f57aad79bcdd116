# Round-2 measurement (1 GPU): default bench line (config 5, cpu_baseline, e2e, sequential), the
# other configs (1-2 with CUDA-graph replays), Hermitian + direct variants, ncu launch list.
set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
timeout 900 python bench.py > gpurun_out/r2/bench_cfg5.json 2> gpurun_out/r2/bench.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2/bench_cfg$c.json 2>> gpurun_out/r2/bench.err; done
timeout 600 python bench.py --form direct --no-cpu-baseline --no-sequential > gpurun_out/r2/bench_cfg5_direct.json 2>> gpurun_out/r2/bench.err
timeout 600 python bench.py --hermitian --no-cpu-baseline --no-sequential > gpurun_out/r2/bench_cfg5_herm.json 2>> gpurun_out/r2/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2/bench_reference.json 2>> gpurun_out/r2/bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > gpurun_out/r2/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_cfg5.csv $CMD > gpurun_out/r2/ncu_launch.log 2>&1
tail -3 gpurun_out/r2/bench.err
