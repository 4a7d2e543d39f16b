#!/bin/bash
# K1 configuration sweep: cluster budget x threads per CTA (bench K1 time)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "80 256" "80 512" "40 256" "40 512" "20 256"; do
  set -- $cfg
  SV_CHUNK_PAIR_KB=$1 SV_SCORE_THREADS=$2 timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/sweep_$1_$2.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/sweep_$1_$2.log').readline());print('$1 KB $2 thr', 'K1 ms', round(d['roofline']['avg_launch_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step ms', round(d['ms_per_step'],4))" >> gpurun_out/sweep.txt 2>&1 || tail -3 gpurun_out/sweep_$1_$2.log >> gpurun_out/sweep.txt
done
