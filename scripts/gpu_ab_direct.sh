# A/B of two builds (ab/libpint_base.so vs ab/libpint_new.so) on the direct form (complex and
# Hermitian) of config 5 and config 4, alternating; then direct-form / Hermitian parity on new
set -x
O=gpurun_out/ab_direct
mkdir -p $O
D=paper_2103_12571_b200
for v in base new base new; do
  cp $D/ab/libpint_$v.so $D/libpint.so
  for mode in "--form direct" "--form direct --hermitian" "--config 4 --form direct"; do
    tag=$(echo "$mode" | tr -d ' -')
    timeout 600 python bench.py $mode --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > $O/b_${v}_$tag.json 2>> $O/err.log
    python -c "import json; d=json.load(open('$O/b_${v}_$tag.json')); r=d['roofline']; print('$v $mode', round(d['ms_per_step'],3), {k: round(x,3) for k,x in r['per_kernel_ms'].items() if x > 0.1}, d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
  done
done
cat $O/summary.txt
cp $D/ab/libpint_new.so $D/libpint.so
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "direct or hermitian" > $O/tests.log 2>&1
tail -3 $O/tests.log
tail -3 $O/err.log
