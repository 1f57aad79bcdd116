# A/B of the pipelined time transforms (TMA store / TMA reduce-add epilogues) against the
# one-tile-per-CTA kernels, experiments build (libpint_exp.so): parity first, then bench lines
set -x
O=gpurun_out/tfft_ab
mkdir -p $O
export PINT_LIBRARY=$PWD/paper_2103_12571_b200/libpint_exp.so
export PYTHONPATH=$PWD
PINT_TFFT_PIPE=1 timeout 600 python scripts/tfft_smoke.py > $O/smoke_pipe.txt 2>&1; cat $O/smoke_pipe.txt | tail -12
PINT_TFFT_PIPE=1 PINT_TFFT_PAIR=1 PINT_TFFT_PROMO=1 timeout 600 python scripts/tfft_smoke.py > $O/smoke_pipe_pair.txt 2>&1; cat $O/smoke_pipe_pair.txt | tail -12
for v in ${VARIANTS:-"PINT_TFFT_PIPE=0" "PINT_TFFT_PIPE=1" "PINT_TFFT_PIPE=1 PINT_TFFT_PAIR=1" "PINT_TFFT_PIPE=1 PINT_TFFT_PROMO=1" "PINT_TFFT_PIPE=1 PINT_TFFT_PAIR=1 PINT_TFFT_PROMO=1"}; do
  for c in 5 4; do
    tag=$(echo "$v" | tr ' =' '__')
    env $v timeout 600 python bench.py --allow-experiments --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/b_${tag}_cfg$c.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/b_${tag}_cfg$c.json')); r=d['roofline']; print('$v cfg$c', round(d['ms_per_step'],3), {k: round(x,3) for k,x in r['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
tail -5 $O/err.log
