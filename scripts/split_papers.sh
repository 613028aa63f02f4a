for sp in 1 2 3; do
 for fr in 1024 256; do
  TT_SPLIT=$sp TT_SPLIT_ROWS_FWD=$fr timeout 300 python bench.py --config papers --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tensor-path > gpurun_out/sp_p_$sp_$fr.json 2>/dev/null
  echo "split=$sp fwdrows=$fr $(python scripts/bench_summary.py gpurun_out/sp_p_$sp_$fr.json | grep -o "ms/step=[0-9.]*\|'fwd_main': [0-9.]*\|'bwd_main': [0-9.]*" | tr '\n' ' ')"
 done
done
