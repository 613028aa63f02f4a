# usage: CFGS="papers billion" [ENVS="A=1 B=2"] [BENCH_ARGS=..] bash scripts/cfg_bench.sh -- one bench line per config (no CPU baseline / e2e)
for cfg in ${CFGS:-papers}; do
  env ${ENVS:-TT_DUMMY=0} timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:---no-tensor-path} > gpurun_out/cb_${cfg}.json 2> gpurun_out/cb_${cfg}.err
  python scripts/bench_summary.py gpurun_out/cb_${cfg}.json
done
