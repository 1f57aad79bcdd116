# 1-D pipelined PCR: parity tests of every path through it, quick bench lines, ncu of config 3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hermitian.py tests/test_gpu_sharded.py tests/test_gpu_direct.py tests/test_gpu_forcing.py -m gpu -q -x --timeout 600 -k "pcr1d or two_pass or twopass or N16384" > gpurun_out/t_pcr1d.log 2>&1
tail -3 gpurun_out/t_pcr1d.log
CFGS="3" bash scripts/gpu_quick.sh
if [ -n "$FULL" ]; then timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x --timeout 800 -k "3 or 1d" > gpurun_out/t_full1d.log 2>&1; tail -3 gpurun_out/t_full1d.log; fi
if [ -n "$NCU" ]; then bash scripts/gpu_ncu_cfg3.sh > /dev/null 2>&1; grep -A15 pcr_ gpurun_out/prof_cfg3_brief.txt; fi
