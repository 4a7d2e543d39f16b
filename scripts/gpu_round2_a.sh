set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_a.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_a.log
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_a.err
