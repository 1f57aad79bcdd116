mkdir -p gpurun_out/final1d
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "fuzz or full_size_all or boundary_1d or windows or test_gpu_parity or sequential or graph" > gpurun_out/final1d/tests.log 2>&1
tail -4 gpurun_out/final1d/tests.log
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/final1d/bench_cfg3.json 2> gpurun_out/final1d/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final1d/smoke.log 2>&1; tail -2 gpurun_out/final1d/smoke.log
