cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 120 python scripts/prof_step.py --steps 3 > gpurun_out/hangcheck.log 2>&1 || { echo "hangcheck failed"; exit 3; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 7 -c 14 --csv \
  --log-file gpurun_out/launches_c.csv python scripts/prof_step.py --steps 4 > gpurun_out/ncu_launch_c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"sv_score_kernel|sv_schedule_row_kernel|sv_rows_kernel|sv_decide_kernel|sv_resid_kernel|sv_find_kernel" -s 12 -c 6 \
  -o gpurun_out/prof_c -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_c.log 2>&1
echo "profile rc=$?"
