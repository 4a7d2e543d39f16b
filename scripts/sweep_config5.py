"""BASELINE config 5 measurement: scored positions/s over B = 4..80, k in {2, 4, 8} at
V = 128256 bf16 with swept alignment, one GPU (CUDA events, 2 rotating input sets per point,
SV-scheduled step = sv_score -> sv_schedule -> sd_verify).  Writes one JSON line per point."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402

V = 128256
prof = sv.Profile.from_dict(synth.load_profile())
for k in (2, 4, 8):
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    for B in (4, 8, 16, 32, 48, 64, 80):
        x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED + 97 * 5, alignment="sweep")
        conv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).cuda()  # noqa: E731
        sets = [(conv(x["D"]), conv(x["C"]), conv(x["T"]), torch.from_numpy(x["tok"]).cuda()) for _ in range(2)]
        pipe = sv.Pipeline(B, k, V, torch.bfloat16, prof, L)
        for j in range(10):
            pipe.run(*sets[j & 1], seed=1, offset=j)
        torch.cuda.synchronize()
        steps = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for j in range(steps):
            pipe.run(*sets[j & 1], seed=1, offset=10 + j)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        g = pipe.sched_out["gamma"].cpu().numpy()
        print(json.dumps({"config": "5", "B": B, "k": k, "V": V, "ms_per_step": ms,
                          "positions_per_s": B * k / (ms * 1e-3), "mean_gamma": float(g.mean()),
                          "input_MB_per_set": (2 * B * k + B * (k + 1)) * V * 2 / 1e6}), flush=True)
