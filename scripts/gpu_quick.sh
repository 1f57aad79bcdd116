# quick loop: parity tests (not the full-size sampled ones) + bench configs 3-5 (device time only)

tail -3 gpurun_out/gpu_tests.log
for c in 3 4 5; do for f in ${FORMS:-correction}; do
  timeout 600 python bench.py --config $c --form $f --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench$c.json 2> gpurun_out/bench$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench$c.json')); r=d['roofline']
print($c, '$f', 'ms/iter %.3f'%d['ms_per_step'], 'iter frac %.3f'%r['iteration']['frac'], {k: round(v,3) for k,v in r['per_kernel_ms'].items()})
"
done; done
