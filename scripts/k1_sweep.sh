#!/bin/bash
# K1 configuration sweep (SV_SCORE_CFG: CTAs/SM x loads in flight) -> gpurun_out/sweep.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in 0 1 2 3 4; do
  SV_SCORE_CFG=$cfg timeout 200 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/sweep_$cfg.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sweep_$cfg.log').readline());print('cfg $cfg', 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step ms', round(d['ms_per_step'],4))" >> gpurun_out/sweep.txt 2>&1 || tail -2 gpurun_out/sweep_$cfg.log >> gpurun_out/sweep.txt
done
