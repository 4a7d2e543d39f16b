#!/usr/bin/env python3
"""Experiment: K1 time vs the device's persisting-L2 limit (cudaLimitPersistingL2CacheSize), which
bounds how many lines the `evict_last` policy of pass 1 may keep.  On the GPU:
    python scripts/l2persist_ab.py"""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

B, k, V = 80, 8, 152064
dev = torch.device("cuda")
torch.zeros(1, device=dev)
err, mx = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err2, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
print(json.dumps({"max_persisting_l2": mx, "l2": l2}), flush=True)
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
h = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16)
sets = [(h(x["D"]).to(dev), h(x["C"]).to(dev), torch.from_numpy(x["tok"]).to(dev)) for _ in range(2)]
prof = sv.Profile.from_dict(synth.load_profile())
ws = sv.new_workspace(B, k, V, torch.bfloat16)
out = None
st = torch.cuda.current_stream()
for lim in (0, 16 << 20, 32 << 20, 64 << 20, 96 << 20, mx):
    lim = min(lim, mx)
    print(rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, lim), file=sys.stderr)
    for j in range(6):
        D, C, tok = sets[j & 1]
        out = sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=ws, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
    for j in range(60):
        D, C, tok = sets[j & 1]
        ev[j][0].record(st)
        sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=ws, out=out)
        ev[j][1].record(st)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    print(json.dumps({"persisting_l2_MB": lim / 2 ** 20, "k1_us_mean": sum(t) / len(t) * 1e3,
                      "k1_us_median": t[len(t) // 2] * 1e3}), flush=True)
