# Round-2 evidence capture (one B200): tests, bench, launch lists, full ncu of the step kernels,
# microbenchmarks, compute-sanitizer.  Summaries: scripts/summarize_profiles.py r02.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_r02.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/gputest_r02.log
bash scripts/profile_round.sh r02; echo "profile_round rc=$?"
tail -2 gpurun_out/bench_r02.log | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 14 -c 18 --csv --log-file gpurun_out/launches_c1_r02.csv python scripts/prof_step.py --steps 6 --B 4 --k 4 --V 32000 --dtype f32 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 6 -c 20 --csv --log-file gpurun_out/launches_filtered_r02.csv python scripts/filtered_step.py --steps 5 > /dev/null 2>&1
(./scripts/micro/tma_ring; ./scripts/micro/cluster_occ 200 640; ./scripts/micro/cluster_occ 110 384) > gpurun_out/micro_r02.txt 2>&1
timeout 200 ./scripts/micro/ceil > gpurun_out/ceil_r02.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_workload.py > gpurun_out/sanitizer_${t}_r02.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitizer_r02.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|errors" gpurun_out/sanitizer_${t}_r02.log | tail -2 >> gpurun_out/sanitizer_r02.txt
done
cat gpurun_out/sanitizer_r02.txt
