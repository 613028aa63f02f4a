# Round-2 (second session) final evidence in one GPU call (outputs in gpurun_out/s2_*):
# pytest -m gpu first (log in gpurun_out/s2_pytest.log)
#  1. bench lines: papers and billion with the CPU baselines and e2e, the other
#     BASELINE configs, the rank sweep and the paper's Table-4 shapes without;
#     the reference arm (bench.py --impl reference) at papers;
#  2. ncu launch lists (--metrics gpu__time_duration.sum --clock-control none)
#     of the papers FFMA / tensor paths and billion;
#  3. one --set full capture of the main kernels (papers FFMA + tc, billion),
#     summarised by scripts/ncu_stalls.py.
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s2_pytest.log
for cfg in papers billion; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/s2_bench_$cfg.json 2> gpurun_out/s2_bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/s2_bench_$cfg.json
done
for cfg in products small sweep8 sweep16 sweep32 sweep64 sweep128 arxivT4_r32 papersT4_r64 productsT4_r32 productsT4_r64; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s2_bench_$cfg.json 2> gpurun_out/s2_bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/s2_bench_$cfg.json
done
timeout 900 python bench.py --impl reference --config papers --steps 3 --warmup 1 > gpurun_out/s2_ref_papers.json 2> gpurun_out/s2_ref_papers.err
cat gpurun_out/s2_ref_papers.json
for run in "papers auto" "papers tc" "billion auto" "sweep8 auto"; do
  set -- $run
  CMD="python bench.py --config $1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path --path $2"
  $CMD > gpurun_out/s2_plain_$1_$2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2_launches_$1_$2.csv $CMD > gpurun_out/s2_ncu_$1_$2.log 2>&1
  python scripts/ncu_summary.py gpurun_out/s2_launches_$1_$2.csv > gpurun_out/s2_launches_$1_$2.txt
done
for run in "papers auto k_fused_fwd8|k_fused_bwd|k_last_level|k_fused_w 4" "papers tc k_tc_fwd|k_tc_bwd3|k_fused_wdc 3" "billion auto k_fused_bwd_ws|k_fused_fwd8w<32,.16 2" "sweep8 auto k_lowrank_fwd|k_lowrank_bwd 2"; do
  set -- $run
  CMD="python bench.py --config $1 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path --path $2 --graph 0"
  ncu --set full --clock-control none --import-source on -k regex:"$3" -c $4 -o gpurun_out/s2_full_$1_$2 $CMD > gpurun_out/s2_ncu_full_$1_$2.log 2>&1
  python scripts/ncu_stalls.py gpurun_out/s2_full_$1_$2.ncu-rep > gpurun_out/s2_stalls_$1_$2.txt
  rm -f gpurun_out/s2_full_$1_$2.ncu-rep  # (gpurun brings back <= 64 MiB)
done
ls -la gpurun_out/ | grep s2_ | head -60
