# HEAD verification on 1 GPU: quick bench lines for configs 5, 4, 3, then the GPU test suite
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
CFGS="${CFGS:-5 4 3}" bash scripts/gpu_quick.sh > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 ${K:+-k "$K"} > gpurun_out/gpu_tests.log 2>&1
tail -25 gpurun_out/gpu_tests.log
