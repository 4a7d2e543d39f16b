# usage: gpu_prof_var.sh VARIANT OUTNAME [kernel-regex]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
lib=paper_2509_24328_b200/variants/libsv_$1.so
[ "$1" = product ] && lib=paper_2509_24328_b200/libsv.so
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${3:-sv_score_ring_kernel}" -s 2 -c 1 \
  -o gpurun_out/$2 -f python scripts/prof_step.py --steps 3 --lib $lib > gpurun_out/$2.log 2>&1
echo "ncu rc=$?"
