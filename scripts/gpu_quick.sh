#!/bin/bash
# tests + smoke + short bench + ncu launch list of the step + optional --set full capture
#   NCU_K=<kernel regex> bash scripts/gpu_quick.sh TAG   (NO_NCU=1 skips the full capture)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-q}
timeout 120 python scripts/prof_step.py --steps 3 > gpurun_out/hangcheck.log 2>&1; echo "hangcheck rc=$?" >> gpurun_out/hangcheck.log
grep -q "rc=0" gpurun_out/hangcheck.log || exit 3
timeout 600 python -m pytest tests -m gpu -x -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 240 python bench.py --steps 300 --warmup 10 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python scripts/prof_step.py --steps 4 > gpurun_out/ncu_launch_$TAG.log 2>&1
if [ -z "$NO_NCU" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-sv_score_kernel}" -s 2 -c ${NCU_C:-1} -o gpurun_out/prof_$TAG -f python scripts/prof_step.py --steps 4 > gpurun_out/ncu_full_$TAG.log 2>&1
fi
if [ -n "$AB" ]; then  # A/B env experiments: AB="SV_PDL=0;SV_X=1"
IFS=';' read -ra VARS <<< "$AB"
for v in "${VARS[@]}"; do
  env $v timeout 200 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > "gpurun_out/bench_ab_${v//=/_}.log" 2>&1
done
fi
