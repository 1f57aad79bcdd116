# A/B of two builds of libpint.so on the same box (ab/libpint_base.so vs ab/libpint_new.so),
# alternating base/new twice on config 5 (and config 4), then the pipe-plan parity subset on new.
# Usage: AB_VARIANTS="base new base new" AB_K="pipe or hermitian" bash scripts/gpu_ab_lib.sh
set -x
O=gpurun_out/ab
mkdir -p $O
D=paper_2103_12571_b200
if [ -f scripts/rcp_check.cu ]; then nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o /tmp/rcp_check scripts/rcp_check.cu && /tmp/rcp_check > $O/rcp_check.txt 2>&1; cat $O/rcp_check.txt; fi
for v in ${AB_VARIANTS:-base new base new}; do
  cp $D/ab/libpint_$v.so $D/libpint.so
  for c in 5 4; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/b_${v}_cfg$c.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/b_${v}_cfg$c.json')); r=d['roofline']; print('$v cfg$c', round(d['ms_per_step'],3), {k: round(x,3) for k,x in r['per_kernel_ms'].items()}, d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
cp $D/ab/libpint_new.so $D/libpint.so
timeout 1800 python -m pytest tests -m gpu -q -x -k "${AB_K:-pipe or direct or hermitian}" > $O/tests.log 2>&1
tail -3 $O/tests.log
