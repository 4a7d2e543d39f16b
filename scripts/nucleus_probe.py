"""Launch list of the nucleus-only (Llama setting) filtered step at the headline size, for ncu:
ncu --metrics gpu__time_duration.sum --clock-control none python scripts/nucleus_probe.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402

B, k, V = int(os.environ.get("NB", 80)), 8, 152064
tau = float(os.environ.get("NTAU", 0.6))
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).cuda()
D, C, T = h(x["D"]), h(x["C"]), h(x["T"])
tok = torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile(), device="cuda")
L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
fws = sv.new_filter_workspace(B, k, "cuda")
if os.environ.get("NONLY"):  # two nucleus-only score calls (ncu: --launch-skip 1 -c 1 on sv_topk_kernel)
    for _ in range(2):
        sv.sv_score_filtered(D, C, tok, 0, 0.9, tau, tau, prof, fworkspace=fws)
    torch.cuda.synchronize()
    sys.exit(0)
for j in range(2):
    fs = sv.sv_score_filtered(D, C, tok, 0, 0.9, tau, tau, prof, fworkspace=fws)
    g = sv.sv_schedule(fs["p_hat"], L)["gamma"]
    r = sv.sd_verify_filtered(T, tok, g, fws, 0, 0.9, tau, 1, j, D=D)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
fs = sv.sv_score_filtered(D, C, tok, 0, 0.9, tau, tau, prof, fworkspace=fws)
e1.record()
torch.cuda.synchronize()
print("score ms", e0.elapsed_time(e1), "status nonzero", int((fs["status"] != 0).sum()))
# how many rows are wide: nucleus size from the oracle-free GPU outputs is not exposed; estimate
# from the filtered lists' wide flag in the workspace (FList layout: n, st, ..., wide at byte 400)
ws = fws.view(torch.int32)
rec = 440 // 4  # sizeof(FList)
nl = B * k
wd = ws[: nl * rec].view(nl, rec)[:, 400 // 4]
print("wide draft rows", int(wd.sum()), "of", nl)
# kernel-only timing of the score launch in several modes
for (tk, tp, tt) in ((20, 0.8, tau), (32, 0.9, tau), (0, 0.9, 0.3), (0, 0.9, tau), (0, 0.9, 1.0)):
    for _ in range(2):
        sv.sv_score_filtered(D, C, tok, tk, tp, tt, tt, prof, fworkspace=fws)
    e0.record()
    for _ in range(5):
        sv.sv_score_filtered(D, C, tok, tk, tp, tt, tt, prof, fworkspace=fws)
    e1.record()
    torch.cuda.synchronize()
    wd = ws[: nl * rec].view(nl, rec)[:, 400 // 4]
    print(f"top_k {tk} top_p {tp} tau {tt}: score {e0.elapsed_time(e1) / 5:.3f} ms, wide draft rows "
          f"{int(wd.sum()) if tk == 0 else 0}")
