for cfg in products billion sweep8 sweep64 small papers; do
 for fr in 1024 100000; do for br in 128 256; do
  TT_SPLIT_ROWS_FWD=$fr TT_SPLIT_ROWS_BWD=$br timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tensor-path > gpurun_out/sp_${cfg}_${fr}_${br}.json 2>/dev/null
  echo "$cfg fr=$fr br=$br $(python scripts/bench_summary.py gpurun_out/sp_${cfg}_${fr}_${br}.json | grep -o "ms/step=[0-9.]*\|phases=.*")"
 done; done
done
