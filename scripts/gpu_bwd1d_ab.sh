# A/B of the 1-D backward tile's TMA path (experiments build, PINT_BWD_TMA), config 3 and 2,
# with 1-D parity under the switch
set -x
O=gpurun_out/bwd1d
mkdir -p $O
export PYTHONPATH=$PWD
export PINT_LIBRARY=$PWD/paper_2103_12571_b200/libpint_exp.so
for v in "PINT_BWD_TMA=0" "PINT_BWD_TMA=1" "PINT_BWD_TMA=0" "PINT_BWD_TMA=1"; do
  for mode in "--config 3" "--config 3 --form direct"; do
    tag=$(echo "$mode" | tr -d ' -')
    env $v timeout 600 python bench.py --allow-experiments $mode --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/ab_${v}_$tag.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/ab_${v}_$tag.json')); r=d['roofline']; print('$v $mode', round(d['ms_per_step'],4), {k: round(x,4) for k,x in r['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
PINT_BWD_TMA=1 timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "(parity or operators or forcing or direct or sharded or guards) and not 2d" > $O/tests.log 2>&1; tail -3 $O/tests.log
tail -3 $O/err.log
