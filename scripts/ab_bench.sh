# usage: VAR=TT_FWD8 VALS="0 1" CFG=papers [TESTS="pytest args"] bash scripts/ab_bench.sh
# A/B of an engine switch on one config: bench lines (no CPU baseline / e2e / tensor path) per value.
set -x
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -q -x 2>&1 | tail -5
fi
for cfg in ${CFG:-papers}; do
for v in ${VALS:-0 1}; do
  env $VAR=$v timeout 600 python bench.py --config $cfg --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:---no-tensor-path} > gpurun_out/ab_${cfg}_${VAR}_$v.json 2> gpurun_out/ab_${cfg}_${VAR}_$v.err
  python scripts/bench_summary.py gpurun_out/ab_${cfg}_${VAR}_$v.json
done
done
