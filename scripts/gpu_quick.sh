#!/bin/bash
# tests + smoke + short bench + one ncu capture of sv_score
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sv_score_kernel -s 2 -c 1 -o gpurun_out/prof_score_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_$TAG.log 2>&1
