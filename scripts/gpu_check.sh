# usage: bash scripts/gpu_check.sh [pytest-args]  -- GPU tests then short benches
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
for cfg in ${BENCH_CONFIGS:-small products papers}; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  tail -3 gpurun_out/bench_$cfg.err
  cat gpurun_out/bench_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['path'], 'ms/step=%.3f'%d['ms_per_step'], 'Mrows/s=%.2f'%(d['value']/1e6), 'frac=%.3f'%d['roofline']['frac'], 'e2e=%.2f'%(d['e2e']['value']/1e6 if d['e2e'] else 0), 'cpu=', d['cpu_baseline'] and d['cpu_baseline']['value'])"
done
