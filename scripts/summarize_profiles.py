"""Turn a round's raw ncu captures (gpurun_out/, scratch) into the committed summaries under
profiles/<tag>/ (see scripts/profile_round.sh):

  launches.csv        the ncu launch list of `bench.py` (name, duration) -- cold-cache, serialised
  launch_summary.md   per-kernel count / mean duration / share of the SV step
  ncu_full.csv        selected `--set full` metrics per captured kernel
  ncu_full.md         the same as a table, with DRAM traffic vs the algorithmic bytes
and profiles/sv_score_traffic.json (dram read+write bytes per sv_score launch), which bench.py
reports as roofline.traffic.

Usage: python scripts/summarize_profiles.py r01
"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = ("sv_score_kernel", "sv_score_cluster_kernel", "sv_schedule_row_kernel", "sv_greedy", "sv_rows_kernel", "sv_decide_kernel",
        "sv_resid_kernel", "sv_find_kernel", "sv_shard_p1_kernel", "sv_shard_p2_kernel", "sv_shard_finish_kernel")
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__cluster_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
]
TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TO_US = {"nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}


def short(name):
    for o in OURS:
        if o in name:
            return o
    return name.split("(")[0][-60:]


def launches(tag, out):
    path = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    recs = []
    for r in rows[hdr + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            recs.append((short(r[ik]), float(r[iv].replace(",", "")) * TO_US.get(r[iu], 1.0)))
    with open(os.path.join(out, "launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["launch", "kernel", "duration_us"])
        for i, (n, d) in enumerate(recs):
            w.writerow([i, n, f"{d:.3f}"])
    agg = OrderedDict()
    for n, d in recs:
        agg.setdefault(n, []).append(d)
    ours_total = sum(sum(v) / len(v) for n, v in agg.items() if n in OURS)
    lines = [f"# ncu launch list, round {tag}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 4 --warmup 3 "
             "--no-cpu-baseline` (cold-cache, serialised launches; compare shares, not absolutes).", "",
             "| kernel | launches | mean us | share of SV step |", "|---|---:|---:|---:|"]
    for n, v in agg.items():
        m = sum(v) / len(v)
        share = f"{100 * m / ours_total:.1f}%" if n in OURS else "-"
        lines.append(f"| {n} | {len(v)} | {m:.1f} | {share} |")
    lines += ["", f"Sum of per-kernel means over the SV step's kernels: {ours_total:.1f} us."]
    open(os.path.join(out, "launch_summary.md"), "w").write("\n".join(lines) + "\n")
    return agg


def full(tag, out):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_all_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    col = {n: i for i, n in enumerate(h)}
    table = []
    for r in rows[2:]:
        rec = OrderedDict(kernel=short(r[col["Kernel Name"]]))
        for m in METRICS:
            if m in col:
                v, u = r[col[m]].replace(",", ""), units[col[m]]
                try:
                    x = float(v)
                except ValueError:
                    rec[m] = v
                    continue
                if m.startswith("dram__bytes"):
                    x *= TO_BYTES.get(u, 1)
                elif m == "gpu__time_duration.sum":
                    x *= TO_US.get(u, 1.0)
                rec[m] = x
        table.append(rec)
    with open(os.path.join(out, "ncu_full.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(table[0].keys()))
        w.writeheader()
        w.writerows(table)
    lines = [f"# ncu --set full, round {tag}", "",
             "`ncu --set full --clock-control none --import-source on` of each SV kernel "
             "(scripts/profile_round.sh; headline workload B=80, k=8, V=152064, bf16).", "",
             "| kernel | us | DRAM read MB | DRAM write MB | DRAM % peak | SM % peak | warps active % | regs | grid | cluster |",
             "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
    for t in table:
        lines.append("| {} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {} | {} | {} |".format(
            t["kernel"], t.get("gpu__time_duration.sum", 0), t.get("dram__bytes_read.sum", 0) / 1e6,
            t.get("dram__bytes_write.sum", 0) / 1e6,
            t.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
            t.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0),
            t.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0),
            int(t.get("launch__registers_per_thread", 0)), int(t.get("launch__grid_size", 0)),
            int(t.get("launch__cluster_size", 0) or 0)))
    score = [t for t in table if t["kernel"] == "sv_score_kernel"]
    if score:
        t = score[0]
        traffic = t["dram__bytes_read.sum"] + t["dram__bytes_write.sum"]
        alg = 80 * 8 * 152064 * 2 * 2
        lines += ["", f"sv_score: algorithmic bytes per launch {alg / 1e6:.1f} MB (B*k*V*2 operands*2 B); "
                  f"DRAM read+write {traffic / 1e6:.1f} MB = {traffic / alg:.3f} x algorithmic."]
        json.dump({"round": tag, "kernel": "sv_score_kernel", "traffic_bytes_per_launch": traffic,
                   "dram_read_bytes": t["dram__bytes_read.sum"], "dram_write_bytes": t["dram__bytes_write.sum"],
                   "algorithmic_bytes_per_launch": alg, "source": f"profiles/{tag}/ncu_full.csv"},
                  open(os.path.join(ROOT, "profiles", "sv_score_traffic.json"), "w"), indent=1)
    open(os.path.join(out, "ncu_full.md"), "w").write("\n".join(lines) + "\n")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out = os.path.join(ROOT, "profiles", tag)
    os.makedirs(out, exist_ok=True)
    launches(tag, out)
    full(tag, out)
    b = os.path.join(ROOT, "gpurun_out", f"bench_{tag}.log")
    if os.path.exists(b):
        line = open(b).readline().strip()
        if line.startswith("{"):
            open(os.path.join(out, "bench.json"), "w").write(line + "\n")
    print(open(os.path.join(out, "launch_summary.md")).read())
    print(open(os.path.join(out, "ncu_full.md")).read())


if __name__ == "__main__":
    main()
