# Round-2 follow-up on 1 GPU: the new residual halo-box parity cases, then ncu --set full of the
# TMA-staged residual and time-transform kernels (config 5; DRAM bytes of the reduce-add update)
set -x
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "halo_boxes or bench_model" > $O/halo_tests.log 2>&1; tail -3 $O/halo_tests.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sequential"
$CMD > $O/plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"residual2d|tfft_fwd_tma|tfft_bwd_tma" -s 3 -c 3 -o $O/prof_tma5 $CMD > $O/ncu.log 2>&1
tail -1 $O/ncu.log
python scripts/ncu_brief.py $O/prof_tma5.ncu-rep > $O/ncu_full_tma_cfg5.txt 2>&1
cat $O/ncu_full_tma_cfg5.txt
rm -f $O/prof_tma5.ncu-rep
