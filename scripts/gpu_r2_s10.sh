cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s15.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_s15.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 7 -c 14 --csv \
  --log-file gpurun_out/launches_s15.csv python scripts/prof_step.py --steps 4 > gpurun_out/ncu_launch_s15.log 2>&1
python scripts/launches.py gpurun_out/launches_s15.csv
bash scripts/gpu_r2_ab.sh mb3
