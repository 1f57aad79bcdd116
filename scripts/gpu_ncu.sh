# ncu --set full of selected kernels (KREGEX) on config $CFG, after a plain run of the same command
CMD="python bench.py --config ${CFG:-5} --form ${FORM:-correction} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_ncu.log 2>&1 && timeout ${NCU_TIMEOUT:-1200} ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
