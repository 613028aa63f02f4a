# usage: [PYTEST_ARGS=..] [BENCH_CONFIGS=".."] [BENCH_ARGS=".."] bash scripts/gpu_check.sh
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
for cfg in ${BENCH_CONFIGS:-small products papers}; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  tail -2 gpurun_out/bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/bench_$cfg.json
done
