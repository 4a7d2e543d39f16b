#!/bin/bash
# tests + smoke + short bench + one ncu capture of sv_score (short timeouts: a hang costs little)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-q}
timeout 120 python scripts/prof_step.py --steps 3 > gpurun_out/hangcheck.log 2>&1; echo "hangcheck rc=$?" >> gpurun_out/hangcheck.log
grep -q "rc=0" gpurun_out/hangcheck.log || exit 3
timeout 600 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 240 python bench.py --steps 300 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -z "$NO_NCU" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sv_score_kernel -s 2 -c 1 -o gpurun_out/prof_score_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
