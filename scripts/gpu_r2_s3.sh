cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sv_score_ring_kernel" -s 2 -c 1 \
  -o gpurun_out/prof_ring_s3 -f python scripts/prof_step.py --steps 3 > gpurun_out/ncu_ring_s3.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_ring_s3.log
