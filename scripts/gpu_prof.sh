#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_$TAG.csv python scripts/prof_step.py --steps 5 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_score_kernel -s 2 -c 1 -o gpurun_out/prof_score_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sv_rows_kernel|sv_sample_kernel" -s 4 -c 2 -o gpurun_out/prof_verify_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_v_$TAG.log 2>&1
