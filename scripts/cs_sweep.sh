#!/bin/bash
# K1 minimum chunks per row (SV_SCORE_MIN_CS) across configs -> gpurun_out/cs_sweep.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2 headline}; do for m in ${MINCS:-1 2 4 8}; do
  SV_SCORE_MIN_CS=$m timeout 200 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/cs_${c}_$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cs_${c}_$m.log').readline());print('$c min_cs $m graph step us', round(d['ms_per_step']*1000,1), 'eager', round(d['eager']['ms_per_step']*1000,1), 'K1', round(d['roofline']['avg_launch_ms']*1000,1))" >> gpurun_out/cs_sweep.txt 2>&1 || tail -2 gpurun_out/cs_${c}_$m.log >> gpurun_out/cs_sweep.txt
done; done
