cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py -x -q -p no:cacheprovider > gpurun_out/gputest_s7.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_s7.log
timeout 900 python scripts/k1_ab.py run r0 w1 w4 a12 a8 s4 > gpurun_out/ab_s7.jsonl 2> gpurun_out/ab_s7.err; echo "ab rc=$?"
cat gpurun_out/ab_s7.jsonl; tail -5 gpurun_out/ab_s7.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sv_score_ring_kernel" -s 2 -c 1 \
  -o gpurun_out/prof_ring_s7 -f python scripts/prof_step.py --steps 3 > gpurun_out/ncu_ring_s7.log 2>&1
echo "ncu rc=$?"
