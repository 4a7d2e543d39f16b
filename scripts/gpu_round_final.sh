# Final evidence capture of a round (one B200): GPU tests, bench + launch list + ncu full of the
# step kernels (scripts/profile_round.sh TAG), config-1 launch list.  (compute-sanitizer is closed on
# this GPU pool: runs under it have left GPUs needing a reset.)
# Summaries: scripts/summarize_profiles.py TAG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/gputest_$TAG.log
bash scripts/profile_round.sh $TAG; echo "profile_round rc=$?"
tail -2 gpurun_out/bench_$TAG.log | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 14 -c 18 --csv --log-file gpurun_out/launches_c1_$TAG.csv python scripts/prof_step.py --steps 6 --B 4 --k 4 --V 32000 --dtype f32 > /dev/null 2>&1
