# A/B loop: quick GPU parity tests, then bench lines for configs 4-5 under the env variants in $VARIANTS
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "${K:-not full_size_sampled}" > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for c in ${CFGS:-4 5}; do for f in ${FORMS:-correction direct}; do for v in ${VARIANTS:-X=0}; do
  env $v timeout 600 python bench.py --config $c --form $f --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench$c.json 2> gpurun_out/bench$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench$c.json')); r=d['roofline']
print($c, '$f', '$v', 'ms/iter %.3f'%d['ms_per_step'], 'iter frac %.3f'%r['iteration']['frac'], {k: round(v,3) for k,v in r['per_kernel_ms'].items()})
" || tail -5 gpurun_out/bench$c.err
done; done; done
