cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s2.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/gputest_s2.log
timeout 900 python scripts/k1_ab.py run r0 p2 p4 lag96 u4s3 c12 > gpurun_out/ab_s2.jsonl 2> gpurun_out/ab_s2.err; echo "ab rc=$?"
cat gpurun_out/ab_s2.jsonl; tail -5 gpurun_out/ab_s2.err
