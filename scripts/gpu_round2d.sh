# Round-2 (fourth session) measurement on 1 GPU: smoke, GPU test suite, bench lines for every config
# and variant, the default bench's ncu launch list (configs 5 and 3), ncu --set full of the C pass
set -x
O=gpurun_out/r2d
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm --format=csv > $O/smi.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>> $O/bench.err; done
timeout 600 python bench.py --form direct --no-cpu-baseline --no-sequential > $O/bench_cfg5_direct.json 2>> $O/bench.err
timeout 600 python bench.py --hermitian --no-cpu-baseline --no-sequential > $O/bench_cfg5_herm.json 2>> $O/bench.err
timeout 600 python bench.py --hermitian --form direct --no-cpu-baseline --no-sequential > $O/bench_cfg5_herm_direct.json 2>> $O/bench.err
timeout 600 python bench.py --config 3 --hermitian --no-cpu-baseline --no-sequential > $O/bench_cfg3_herm.json 2>> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2>> $O/bench.err
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('roofline') or {}).get('frac'))" 2>/dev/null; done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > $O/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_launch.log 2>&1
CMD3="python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD3 > $O/plain_launch3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv $CMD3 > $O/ncu_launch3.log 2>&1
bash scripts/gpu_ncu_cols.sh > $O/ncu_full_cols5.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --timeout 1200 > $O/gpu_tests.log 2>&1
tail -5 $O/gpu_tests.log
tail -3 $O/bench.err
