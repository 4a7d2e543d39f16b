set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_b.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/gputest_b.log
timeout 900 python scripts/k1_ab.py run sc152m4 sc152 m4 lag112 nt g3m4 > gpurun_out/ab_b.jsonl 2> gpurun_out/ab_b.err; echo "ab rc=$?"
cat gpurun_out/ab_b.jsonl; tail -3 gpurun_out/ab_b.err
