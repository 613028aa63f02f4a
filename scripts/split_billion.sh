for sp in 0 8 12 16; do
  TT_SPLIT=$sp timeout 300 python bench.py --config billion --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tensor-path > gpurun_out/sb_$sp.json 2>/dev/null
  echo "split=$sp $(python scripts/bench_summary.py gpurun_out/sb_$sp.json | grep -o "ms/step=[0-9.]*\|'fwd_main': [0-9.]*\|'bwd_main': [0-9.]*" | tr '\n' ' ')"
done
