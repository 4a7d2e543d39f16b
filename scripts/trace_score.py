"""Debug: per-CTA phase timeline of sv_score (libsv_trace.so built by scripts/build_trace.sh)."""
import ctypes, os, sys, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_24328_b200 import _lib
_lib.load(os.path.join(ROOT, "paper_2509_24328_b200", "libsv_trace.so"))
import paper_2509_24328_b200 as sv, synth
B, k, V = 80, 8, 152064
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
D, C = (torch.from_numpy(t).view(torch.bfloat16).cuda() for t in (x["D"], x["C"]))
tok = torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile())
ncta = B * k * sv.cluster_size(V, torch.bfloat16)
tr = torch.zeros(ncta * 12, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sv_debug_set_trace.argtypes = [ctypes.c_void_p]
for it in range(3):
    lib.sv_debug_set_trace(tr.data_ptr() if it == 2 else None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); sv.sv_score(D, C, tok, 1.0, 1.0, prof); e1.record(); torch.cuda.synchronize()
    print("ms", e0.elapsed_time(e1))
t = tr.view(ncta, 12).cpu().numpy().astype(np.float64)
sub = t[:, [4, 8, 9, 10, 5]].copy()
t0 = t[:, 0].min()
t = (t[:, :8] - t0) / 1000.0
sub = (sub - t0) / 1000.0
print('merge sub-phases us (loads+max, shuffles, lam, sync):', np.round(np.diff(sub, axis=1).mean(0), 2))
names = ["tma", "passAB", "blockmerge", "clusterA", "merge", "phase2", "clusterB"]
d = np.diff(t, axis=1)
print("mean us per phase:", {n: round(float(d[:, j].mean()), 2) for j, n in enumerate(names)})
print("p90 us per phase:", {n: round(float(np.percentile(d[:, j], 90)), 2) for j, n in enumerate(names)})
life = t[:, 7] - t[:, 0]
print("lifetime mean", life.mean(), "start span", t[:, 0].max(), "end", t[:, 7].max())
order = np.argsort(t[:, 0])
for c in order[:: len(order) // 12]:
    print(c, np.round(t[c], 2))
