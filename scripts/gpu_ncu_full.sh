# usage: CFG=papers KREGEX=k_fused bash scripts/gpu_ncu_full.sh  -- one --set full capture of the matching kernels
CFG=${CFG:-papers}
KREGEX=${KREGEX:-k_fused}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path ${BENCH_ARGS:-}"
$CMD > gpurun_out/plain_full_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c ${NCU_C:-2} -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
tail -3 gpurun_out/ncu_full_$CFG.log
