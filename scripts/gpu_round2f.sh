# Round-2 (fourth session) final measurement after the TMA time tiles and the residual halo boxes:
# parity first, A/B of the inverse's reduce-add, bench lines, launch list (kernel names as launched),
# ncu --set full of the TMA-staged kernels and the C pass
set -x
O=gpurun_out/r2f
mkdir -p $O
export PYTHONPATH=$PWD
nvidia-smi --query-gpu=name,driver_version,memory.total,clocks.max.sm --format=csv > $O/smi.txt
timeout 600 python scripts/tfft_smoke.py > $O/tfft_smoke.txt 2>&1; tail -9 $O/tfft_smoke.txt
for v in "PINT_TFFT_BWD_TMA=0" "PINT_TFFT_BWD_TMA=1" "PINT_TFFT_BWD_TMA=0" "PINT_TFFT_BWD_TMA=1"; do
  for mode in "--config 5" "--config 4" "--form direct"; do
    tag=$(echo "$mode" | tr -d ' -')
    env $v PINT_LIBRARY=$PWD/paper_2103_12571_b200/libpint_exp.so timeout 600 python bench.py --allow-experiments $mode --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/ab_${v}_$tag.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/ab_${v}_$tag.json')); r=d['roofline']; print('$v $mode', round(d['ms_per_step'],3), {k: round(x,3) for k,x in r['per_kernel_ms'].items() if x > 0.1}, d['clocks']['sm_mhz'])" >> $O/ab_summary.txt 2>&1
  done
done
cat $O/ab_summary.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -k "sharded or direct or config5_plan or guards or windows or halo_boxes or parity or full_size_all" > $O/tests.log 2>&1; tail -3 $O/tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench.err
for c in 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_cfg$c.json 2>> $O/bench.err; done
timeout 600 python bench.py --form direct --no-cpu-baseline --no-sequential > $O/bench_cfg5_direct.json 2>> $O/bench.err
timeout 600 python bench.py --hermitian --form direct --no-cpu-baseline --no-sequential > $O/bench_cfg5_herm_direct.json 2>> $O/bench.err
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; print('$f', d.get('ms_per_step'), r.get('kernel'), r.get('frac'), (r.get('iteration') or {}).get('frac'), r.get('per_kernel_ms'))" 2>/dev/null; done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > $O/plain_launch.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv $CMD > $O/ncu_launch.log 2>&1
python scripts/launch_summary.py $O/launches_cfg5.csv | tail -8
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"residual2d|tfft_fwd_tma|tfft_bwd_tma|cols_pipe" -s 4 -c 4 -o $O/prof_tma5 $CMD > $O/ncu.log 2>&1
tail -1 $O/ncu.log
python scripts/ncu_brief.py $O/prof_tma5.ncu-rep > $O/ncu_full_cfg5.txt 2>&1
cat $O/ncu_full_cfg5.txt
rm -f $O/prof_tma5.ncu-rep
tail -3 $O/bench.err $O/err.log
