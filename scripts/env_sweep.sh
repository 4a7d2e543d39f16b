#!/bin/bash
# Bench under several environment settings: SWEEP="A=1,B=2 A=3" -> gpurun_out/env_sweep.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
n=0
for combo in $SWEEP; do
  n=$((n+1))
  env $(echo "$combo" | tr ',' ' ') timeout 200 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/env_$n.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/env_$n.log').readline());print('$combo', 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step ms', round(d['ms_per_step'],4))" >> gpurun_out/env_sweep.txt 2>&1 || { echo "$combo FAILED"; tail -2 gpurun_out/env_$n.log; } >> gpurun_out/env_sweep.txt
done
