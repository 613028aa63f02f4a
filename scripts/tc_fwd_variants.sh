for v in ${VARIANTS:-0 2 4 8 12 6 10 14}; do
  TT_TC_VARIANT=$v timeout 300 python bench.py --config papers --path tc --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --graph 0 > gpurun_out/fv$v.json 2>/dev/null
  echo "fwd variant $v: $(python -c "import json;d=json.load(open('gpurun_out/fv$v.json'));print(d['phases_ms_per_step']['fwd_main'])")"
done
