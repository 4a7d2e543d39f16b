"""Minimal driver for ncu: builds the headline workload and runs a few pipeline steps."""
import os, sys, argparse
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv, synth
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--B", type=int, default=80); ap.add_argument("--k", type=int, default=8)
ap.add_argument("--V", type=int, default=152064); ap.add_argument("--dtype", default="bf16")
ap.add_argument("--force", type=int, default=None)
ap.add_argument("--lib", default=None, help="variant library (scripts/k1_ab.py build)")
a = ap.parse_args()
if a.lib:
    from paper_2509_24328_b200 import _lib
    _lib._lib = None
    _lib.load(a.lib)
x = synth.make_inputs(a.B, a.k, a.V, a.dtype, seed=0x5EED)
conv = (lambda t: torch.from_numpy(t).view(torch.bfloat16).cuda()) if a.dtype == "bf16" else (lambda t: torch.from_numpy(t).cuda())
D, C, T = conv(x["D"]), conv(x["C"]), conv(x["T"]); tok = torch.from_numpy(x["tok"]).cuda()
prof = sv.Profile.from_dict(synth.load_profile())
L = torch.tensor(synth.latency_table(a.k + 2), dtype=torch.float64, device="cuda")
pipe = sv.Pipeline(a.B, a.k, a.V, D.dtype, prof, L)
for j in range(a.steps):
    pipe.run(D, C, T, tok, seed=1, offset=j, force_gamma=a.force)
torch.cuda.synchronize()
print("gamma", pipe.sched_out["gamma"].tolist())
