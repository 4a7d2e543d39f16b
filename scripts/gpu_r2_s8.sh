cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_s9.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest_s9.log
bash scripts/gpu_r2_ab.sh r0 l1 b5 u1k p2 p4
