timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -k "${K:-not full_size_sampled}" > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
