for v in ${VARIANTS:-0 2 4 8 16 32 48 62}; do
  TT_TC_BVARIANT=$v timeout 300 python bench.py --config papers --path tc --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph 0 > gpurun_out/v$v.json 2>/dev/null
  echo "variant $v: $(python -c "import json;d=json.load(open('gpurun_out/v$v.json'));print(d['phases_ms_per_step']['bwd_main'])")"
done
