# Round-2 (second session) measurement on 1 GPU: GPU test suite, bench lines for every config and
# variant, the default bench's ncu launch list, ncu --set full of the config-3 kernels
set -x
O=gpurun_out/r2b
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > $O/gpu_tests.log 2>&1
tail -5 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>> $O/bench.err; done
timeout 600 python bench.py --form direct --no-cpu-baseline --no-sequential > $O/bench_cfg5_direct.json 2>> $O/bench.err
timeout 600 python bench.py --hermitian --no-cpu-baseline --no-sequential > $O/bench_cfg5_herm.json 2>> $O/bench.err
timeout 600 python bench.py --config 3 --hermitian --no-cpu-baseline --no-sequential > $O/bench_cfg3_herm.json 2>> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>> $O/bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > $O/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_launch.log 2>&1
CMD3="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD3 > $O/plain_launch3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv $CMD3 > $O/ncu_launch3.log 2>&1
bash scripts/gpu_ncu_cfg3.sh > /dev/null 2>&1; cp gpurun_out/prof_cfg3_brief.txt $O/ncu_full_cfg3.txt
tail -3 $O/bench.err
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('roofline') or {}).get('frac'))" 2>/dev/null; done
