# usage: gpu_launches_var.sh VARIANT...: ncu launch list (cold, serialized) of 4 headline steps per variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "$@"; do
  lib=paper_2509_24328_b200/variants/libsv_$v.so
  [ "$v" = product ] && lib=paper_2509_24328_b200/libsv.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 7 -c 14 --csv \
    --log-file gpurun_out/launches_$v.csv python scripts/prof_step.py --steps 4 --lib $lib > /dev/null 2>&1
  echo "== $v"; python scripts/launches.py gpurun_out/launches_$v.csv
done
