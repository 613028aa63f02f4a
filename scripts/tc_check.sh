# usage: bash scripts/tc_check.sh -- tensor-core path parity + bench (papers, products)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tc" 2>&1 | tail -3
for cfg in ${CFGS:-papers products}; do
  timeout 300 python bench.py --config $cfg --path tc --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_tc_$cfg.json 2> gpurun_out/bench_tc_$cfg.err
  tail -3 gpurun_out/bench_tc_$cfg.err; python scripts/bench_summary.py gpurun_out/bench_tc_$cfg.json
done
