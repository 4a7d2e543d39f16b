"""Debug: per-CTA wave timeline of sv_score (libsv_trace.so built with -DSV_TRACE)."""
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
ws = sv.new_workspace(B, k, V, torch.bfloat16)
tr = torch.zeros(400 * 64 * 5, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.sv_debug_set_trace.argtypes = [ctypes.c_void_p]
for it in range(3):
    lib.sv_debug_set_trace(tr.data_ptr() if it == 2 else None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=ws); e1.record(); torch.cuda.synchronize()
    print("ms", e0.elapsed_time(e1))
t = tr.view(400, 64, 5).cpu().numpy().astype(np.float64)
valid = t[:, :, 0] > 0
t0 = t[valid][:, 0].min()
t = (t - t0) / 1000.0  # us
for c in (0, 1, 18, 100, 284):
    print("cta", c)
    for j in range(0, 46, 3):
        r = t[c, j]
        if r[0] <= 0: continue
        print(f"  wave {j:2d} start {r[0]:7.2f} tma {r[1]-r[0]:6.2f} p1 {r[2]-r[1]:6.2f} poll {r[3]-r[2]:6.2f} p2 {r[4]-r[3]:6.2f}")
d = t[:, 1:46, :]
m = d[:, :, 0] > 0
print("mean us: tma", np.mean((d[:,:,1]-d[:,:,0])[m]), "p1", np.mean((d[:,:,2]-d[:,:,1])[m]), "poll", np.mean((d[:,:,3]-d[:,:,2])[m]), "p2", np.mean((d[:,:,4]-d[:,:,3])[m]))
