# usage: CFG=papers bash scripts/gpu_prof.sh -- plain bench, then the ncu launch list of the same command
CFG=${CFG:-papers}
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_C:-300} --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_$CFG.log 2>&1
tail -2 gpurun_out/plain_$CFG.log | cut -c1-600
