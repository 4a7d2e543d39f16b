cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s1.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_s1.log
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_s1.json 2> gpurun_out/bench_s1.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_s1.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 7 -c 14 --csv \
  --log-file gpurun_out/launches_s1.csv python scripts/prof_step.py --steps 4 > gpurun_out/ncu_launch_s1.log 2>&1
echo "ncu rc=$?"
