set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config small --steps 5 --warmup 3 --path generic > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err; tail -3 gpurun_out/bench_small.err
cat gpurun_out/bench_small.json
timeout 600 python bench.py --config papers --steps 3 --warmup 3 --path generic --no-cpu-baseline > gpurun_out/bench_papers_gen.json 2> gpurun_out/bench_papers_gen.err; tail -3 gpurun_out/bench_papers_gen.err
cat gpurun_out/bench_papers_gen.json
