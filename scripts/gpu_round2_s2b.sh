# Round 2 (second session) refresh after the forward's 4x k-loop unroll: bench lines for the
# configs that run k_fused_fwd8w, the papers / billion launch lists and a full capture of the
# papers forward (outputs in gpurun_out/s2b_*)
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2b_pytest.log
for cfg in papers billion; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/s2b_bench_$cfg.json 2> gpurun_out/s2b_bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/s2b_bench_$cfg.json
done
for cfg in products sweep32 sweep64 papersT4_r64; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s2b_bench_$cfg.json 2> gpurun_out/s2b_bench_$cfg.err
  python scripts/bench_summary.py gpurun_out/s2b_bench_$cfg.json
done
for cfg in papers billion; do
  CMD="python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path"
  $CMD > gpurun_out/s2b_plain_$cfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2b_launches_$cfg.csv $CMD > /dev/null 2>&1
  python scripts/ncu_summary.py gpurun_out/s2b_launches_$cfg.csv > gpurun_out/s2b_launches_$cfg.txt
done
CMD="python bench.py --config papers --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-tensor-path --graph 0"
ncu --set full --clock-control none --import-source on -k regex:"k_fused_fwd8w|k_fused_bwd" -c 2 -o gpurun_out/s2b_full_papers $CMD > gpurun_out/s2b_ncu_full.log 2>&1
python scripts/ncu_stalls.py gpurun_out/s2b_full_papers.ncu-rep > gpurun_out/s2b_stalls_papers.txt
rm -f gpurun_out/s2b_full_papers.ncu-rep
