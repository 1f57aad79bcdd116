# one compute-sanitizer tool per gpurun call (B200_PROFILING.md): TOOL=racecheck|synccheck|memcheck
mkdir -p gpurun_out
python scripts/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool ${TOOL:-racecheck} --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_${TOOL:-racecheck}.log 2>&1
echo rc=$?
tail -15 gpurun_out/san_${TOOL:-racecheck}.log
