# Full GPU test suite + smoke on the product library
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/final/gpu_tests.log 2>&1
tail -5 gpurun_out/final/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -2 gpurun_out/final/smoke.log
timeout 600 python bench.py --hermitian --no-cpu-baseline --no-sequential > gpurun_out/final/bench_cfg5_herm.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/final/bench_cfg1.json 2>> gpurun_out/final/bench.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/final/bench_cfg2.json 2>> gpurun_out/final/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_reference.json 2>> gpurun_out/final/bench.err
tail -3 gpurun_out/final/bench.err
