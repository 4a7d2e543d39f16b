cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python scripts/k1_ab.py run "$@" > gpurun_out/ab.jsonl 2> gpurun_out/ab.err; echo "ab rc=$?"
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['variant'].ljust(10), round(d['k1_us_mean'],1), round(d['eager_us'],1), round(d['graph_us'],1), d['diff_vs_product'] and d['diff_vs_product'].get('S'))
"; tail -3 gpurun_out/ab.err
