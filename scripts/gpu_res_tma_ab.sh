# A/B of the residual's TMA halo tile (interior blocks: one tensor box of u) against cp.async
# staging, experiments build; parity on the product build first
set -x
O=gpurun_out/res_tma
mkdir -p $O
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "parity or operators or forcing or config5_plan or sharded" > $O/tests.log 2>&1; tail -3 $O/tests.log
export PINT_LIBRARY=$PWD/paper_2103_12571_b200/libpint_exp.so
for v in "PINT_RES_TMA=0" "PINT_RES_TMA=1" "PINT_RES_TMA=0" "PINT_RES_TMA=1"; do
  for c in 5 4; do
    env $v timeout 600 python bench.py --allow-experiments --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/b_${v}_cfg$c.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/b_${v}_cfg$c.json')); r=d['roofline']; print('$v cfg$c', round(d['ms_per_step'],3), {k: round(x,3) for k,x in r['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
tail -5 $O/err.log
