# Functional smoke test of bench.py's N > 1 path on a 1-GPU box: gloo
# collectives (host-side, no kernel waits on another rank), ranks share cuda:0.
# Not a measurement.
for shard in owner position; do
  for n in 2 3; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
      bench.py --gpus $n --steps 2 --warmup 1 --config ${CFG:-products} --shard $shard --dist-backend gloo --no-cpu-baseline \
      > gpurun_out/dist_${shard}_$n.json 2> gpurun_out/dist_${shard}_$n.err
    echo "shard=$shard n=$n rc=$? $(python scripts/bench_summary.py gpurun_out/dist_${shard}_$n.json | cut -c1-160)"
    tail -3 gpurun_out/dist_${shard}_$n.err
  done
done
