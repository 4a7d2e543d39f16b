#!/bin/bash
# K1 lag sweep (SV_SCORE_LAG rows between a chunk's two reads) -> gpurun_out/lag.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for lag in ${LAGS:-16 32 64 128 256}; do
  SV_SCORE_LAG=$lag timeout 200 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/lag_$lag.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/lag_$lag.log').readline());print('lag $lag', 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step ms', round(d['ms_per_step'],4))" >> gpurun_out/lag.txt 2>&1 || tail -2 gpurun_out/lag_$lag.log >> gpurun_out/lag.txt
done
