# quick bench lines (per-kernel ms) for configs $CFGS with extra bench flags $FLAGS (e.g. "--hermitian")
for c in ${CFGS:-5 4}; do for f in ${FLAGS:-""}; do for fl in "" $f; do
  timeout 600 python bench.py --config $c $fl --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e --no-sequential > gpurun_out/q$c.json 2> gpurun_out/q$c.err
  python -c "
import json; d=json.load(open('gpurun_out/q$c.json')); r=d['roofline']
print($c, '$fl', 'ms %.3f'%d['ms_per_step'], {k: round(v,3) for k,v in r['per_kernel_ms'].items()})
" || tail -3 gpurun_out/q$c.err
done; done; done
