# baseline of the restored state: fp64 FMA peak, quick GPU tests, bench configs 3-5 (both forms)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "not full_size_sampled" > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
FORMS="correction direct" bash scripts/gpu_quick.sh 2>&1 | grep -v "^$" | tail -8
