#!/usr/bin/env python3
"""A/B of build variants on the small / mid BASELINE configs through the graph path (bench.py's
graph_point: per-replay events, L2 flushed before every replay).  On the GPU:
    python scripts/config_ab.py product notail ...   (variants: scripts/k1_ab.py build NAME DEF=VAL)"""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402
from paper_2509_24328_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
peak = bench.measured_peaks()[0]
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
prof = sv.Profile.from_dict(synth.load_profile(), device=dev)


def inputs(B, k, V, dt, seed, alignment="mix"):
    x = synth.make_inputs(B, k, V, dt, seed=seed, alignment=alignment)
    conv = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(dev)) if dt == "bf16" \
        else (lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev))
    return conv(x["D"]), conv(x["C"]), conv(x["T"]), torch.from_numpy(x["tok"]).to(dev)


points = [("tiny", 1, 1, 64, "f32"), ("c1", 4, 4, 32000, "f32"), ("c2", 32, 8, 32000, "bf16"), ("B4k8", 4, 8, 128256, "bf16"),
          ("B16k8", 16, 8, 128256, "bf16"), ("B32k8", 32, 8, 128256, "bf16"), ("B80k8", 80, 8, 128256, "bf16"),
          ("head", 80, 8, 152064, "bf16")]
for name in sys.argv[1:]:
    _lib._lib = None
    _lib.load(_lib.LIB_PATH if name == "product" else
              os.path.join(ROOT, "paper_2509_24328_b200", "variants", f"libsv_{name}.so"))
    res = {}
    for (pn, B, k, V, dt) in points:
        D, C, T, tok = inputs(B, k, V, dt, 0x5EED)
        tdt, elem = (torch.bfloat16, 2) if dt == "bf16" else (torch.float32, 4)
        r = bench.graph_point(sv, torch, dev, D, C, T, tok, B, k, V, tdt, elem, prof, 40, 5, flush, peak)
        res[pn] = round(r["ms_per_step"] * 1e3, 1)
        del D, C, T, tok
    print(json.dumps({"variant": name, "us_per_step": res}), flush=True)
