timeout 1500 python -m pytest tests/test_gpu_hermitian.py tests/test_gpu_parity.py -m gpu -q --timeout 1200 > gpurun_out/gpu_herm.log 2>&1; tail -3 gpurun_out/gpu_herm.log
for f in correction direct; do for h in "" "--hermitian"; do
  timeout 600 python bench.py --config 5 --form $f $h --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']
print('$f', '$h', 'ms/iter %.3f'%d['ms_per_step'], {k: round(v,3) for k,v in r['per_kernel_ms'].items()})" || tail -3 gpurun_out/b.err
done; done
