#!/usr/bin/env python3
"""How the L2 flush between graph replays shapes the small-config step times (on the GPU):
    python scripts/flush_ab.py
modes: rw = a 256 MB read-modify-write (bench.py's flush), rw+r = the same followed by a 256 MB
read of a second buffer (evicts the flush's dirty lines: the step then starts with a clean L2
holding none of its inputs), none = no flush (small inputs stay L2-resident)."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda", 0)
prof = sv.Profile.from_dict(synth.load_profile(), device=dev)
f1 = torch.empty(64 << 20, dtype=torch.float32, device=dev)
f2 = torch.ones(64 << 20, dtype=torch.float32, device=dev)
sink = torch.empty(1, dtype=torch.float32, device=dev)
for (pn, B, k, V, dt) in [("tiny", 1, 1, 64, "f32"), ("c1", 4, 4, 32000, "f32"), ("c2", 32, 8, 32000, "bf16")]:
    x = synth.make_inputs(B, k, V, dt, seed=0x5EED)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(dev)) if dt == "bf16" \
        else (lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev))
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device=dev)
    gp = sv.GraphPipeline(B, k, V, tdt, prof, L, device=dev, seed=1, offset0=0)
    for d, s in zip((gp.D, gp.C, gp.T), (x["D"], x["C"], x["T"])):
        d.copy_(conv(s))
    gp.tok.copy_(torch.from_numpy(x["tok"]).to(dev))
    gp.capture()
    res = {}
    for mode in ("rw", "rw+r", "none"):
        for _ in range(5):
            gp.replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
        for j in range(40):
            if mode != "none":
                f1.add_(1)
            if mode == "rw+r":
                torch.amax(f2, dim=0, out=sink.view(()))
            ev[j][0].record()
            gp.replay()
            ev[j][1].record()
        torch.cuda.synchronize()
        res[mode] = round(sum(a.elapsed_time(b) for a, b in ev) / 40 * 1e3, 1)
    print(json.dumps({"point": pn, "us_per_step": res}), flush=True)
