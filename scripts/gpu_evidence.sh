# Full evidence for one config: bench line (with CPU baseline + e2e), launch list,
# and one ncu --set full capture of the fused kernels (DRAM traffic per launch).
CFG=${CFG:-papers}
set -x
python bench.py --config $CFG --steps ${STEPS:-10} --warmup 3 > gpurun_out/final_$CFG.json 2> gpurun_out/final_$CFG.err
tail -2 gpurun_out/final_$CFG.err
python scripts/bench_summary.py gpurun_out/final_$CFG.json
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
$CMD > gpurun_out/plain2_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_C:-400} --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_l_$CFG.log 2>&1
$CMD > gpurun_out/plain3_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fused_(fwd|bwd)|k_fused_w" -c 3 -o gpurun_out/full_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
tail -2 gpurun_out/ncu_full_$CFG.log
