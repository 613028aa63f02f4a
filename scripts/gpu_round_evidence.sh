# Round evidence in one call: bench lines (all BASELINE configs incl. the rank
# sweep, FFMA headline +
# tensor path), ncu launch lists (FFMA and tc paths at papers) and one
# --set full capture of the four GEMM kernels.  Summaries go to gpurun_out/ev_*.
set -x
for cfg in ${CFGS:-papers products small billion sweep8 sweep16 sweep32 sweep64 sweep128}; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/ev_bench_$cfg.json 2> gpurun_out/ev_bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/ev_bench_$cfg.json
done
for path in auto tc; do
  CMD="python bench.py --config papers --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path --path $path"
  $CMD > gpurun_out/ev_plain_$path.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches_$path.csv $CMD > gpurun_out/ev_ncu_$path.log 2>&1
  python scripts/ncu_summary.py gpurun_out/ev_launches_$path.csv > gpurun_out/ev_launches_$path.txt
done
for path in auto tc; do
  CMD="python bench.py --config papers --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path --path $path"
  ncu --set full --clock-control none --import-source on -k regex:"k_fused_fwd|k_fused_bwd|k_tc_fwd|k_tc_bwd|k_last_level|k_fused_w" -c 4 -o gpurun_out/ev_full_$path $CMD > gpurun_out/ev_ncu_full_$path.log 2>&1
  python scripts/ncu_stalls.py gpurun_out/ev_full_$path.ncu-rep > gpurun_out/ev_stalls_$path.txt
done
