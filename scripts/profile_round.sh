#!/bin/bash
# Round profile capture (run under gpurun, 1 GPU).  Produces in gpurun_out/:
#   launches_$TAG.csv      -- ncu launch list (gpu__time_duration.sum) of the bench command itself
#   prof_all_$TAG.ncu-rep  -- one `--set full` capture of each of the step's kernels
#   clocks_$TAG.csv        -- nvidia-smi clocks sampled during a plain bench run
#   bench_$TAG.log         -- that bench run's JSON line
# scripts/summarize_profiles.py then writes the committed summaries under profiles/$TAG/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 120 python scripts/prof_step.py --steps 3 > gpurun_out/hangcheck.log 2>&1 || { echo "hangcheck failed"; exit 3; }
timeout 300 python bench.py --steps 1000 --warmup 20 > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"sv_score_kernel|sv_score_cluster_kernel|sv_schedule_row_kernel|sv_rows_kernel|sv_decide_kernel|sv_resid_kernel|sv_find_kernel" -s 12 -c 6 \
  -o gpurun_out/prof_all_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_$TAG.log 2>&1
echo "profile rc=$?" >> gpurun_out/ncu_full_$TAG.log
