"""Minimal driver for ncu: the filtered step (Qwen settings: top_k 20, top_p 0.8, tau 0.7, P L737-740)
at the headline size, a few times.  --nucleus: the Llama setting (top_k 0, top_p 0.9, tau 0.6)."""
import argparse, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv, synth
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--nucleus", action="store_true")
a = ap.parse_args()
B, k, V = 80, 8, 152064
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
h = lambda t: torch.from_numpy(np.ascontiguousarray(t)).view(torch.bfloat16).cuda()
D, C, T = h(x["D"]), h(x["C"]), h(x["T"])
tok = torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile(), device="cuda")
L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
fws = sv.new_filter_workspace(B, k, "cuda")
tk, tp, tau = (0, 0.9, 0.6) if a.nucleus else (20, 0.8, 0.7)
for j in range(a.steps):
    fs = sv.sv_score_filtered(D, C, tok, tk, tp, tau, tau, prof, fworkspace=fws)
    g = sv.sv_schedule(fs["p_hat"], L)["gamma"]
    r = sv.sd_verify_filtered(T, tok, g, fws, tk, tp, tau, 1, j, D=D if a.nucleus else None)
torch.cuda.synchronize()
print("ok")
