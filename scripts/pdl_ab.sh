# A/B of programmatic dependent launch (default on): bench with PDL off and on (TT_PDL=0 vs 1)
for cfg in ${CFGS:-small products papers}; do
  for pdl in 0 1; do
    TT_PDL=$pdl timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-tensor-path > gpurun_out/pdl_${cfg}_$pdl.json 2>/dev/null
    echo "TT_PDL=$pdl $(python scripts/bench_summary.py gpurun_out/pdl_${cfg}_$pdl.json)"
  done
done
