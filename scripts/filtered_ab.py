#!/usr/bin/env python3
"""A/B of libsv variants on the filtered step (NEXT-2) at the headline size (on the GPU):
    python scripts/filtered_ab.py product NAME ...   (variants: scripts/k1_ab.py build NAME DEF=VAL)
Per variant: mean CUDA-event time of sv_score_filtered, and of the whole filtered step
(score, schedule, sd_verify_filtered), Qwen (top_k 20, top_p 0.8, tau 0.7) and Llama
nucleus-only (top_k 0, top_p 0.9, tau 0.6) settings; outputs compared bitwise with the first."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2509_24328_b200 as sv  # noqa: E402
import synth  # noqa: E402
from paper_2509_24328_b200 import _lib  # noqa: E402

B, k, V = 80, 8, 152064
x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
h = lambda t: torch.from_numpy(np.ascontiguousarray(t)).view(torch.bfloat16).cuda()  # noqa: E731
D, C, T = h(x["D"]), h(x["C"]), h(x["T"])
tok = torch.from_numpy(x["tok"]).cuda()
L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
ref = {}
for name in sys.argv[1:]:
    _lib._lib = None
    _lib.load(_lib.LIB_PATH if name == "product" else
              os.path.join(ROOT, "paper_2509_24328_b200", "variants", f"libsv_{name}.so"))
    prof = sv.Profile.from_dict(synth.load_profile(), device="cuda")
    fws = sv.new_filter_workspace(B, k, "cuda")
    res = {"variant": name}
    for tag, (tk, tp, tau) in (("qwen", (20, 0.8, 0.7)), ("nucleus", (0, 0.9, 0.6))):
        Dn = D if tk == 0 else None
        for _ in range(3):
            fs = sv.sv_score_filtered(D, C, tok, tk, tp, tau, tau, prof, fworkspace=fws)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        for _ in range(20):
            fs = sv.sv_score_filtered(D, C, tok, tk, tp, tau, tau, prof, fworkspace=fws)
        e[1].record()
        for j in range(20):
            fs = sv.sv_score_filtered(D, C, tok, tk, tp, tau, tau, prof, fworkspace=fws)
            g = sv.sv_schedule(fs["p_hat"], L)["gamma"]
            r = sv.sd_verify_filtered(T, tok, g, fws, tk, tp, tau, 1, j, D=Dn)
        e[2].record()
        torch.cuda.synchronize()
        res[tag + "_score_ms"] = round(e[0].elapsed_time(e[1]) / 20, 4)
        res[tag + "_step_ms"] = round(e[1].elapsed_time(e[2]) / 20, 4)
        out = [fs[n].cpu().numpy() for n in ("S", "A", "KL", "p_hat", "status")] + \
              [r[n].cpu().numpy() for n in ("n_accept", "out_tok", "status")]
        if tag in ref:
            res[tag + "_same"] = all(np.array_equal(a, b, equal_nan=True) for a, b in zip(out, ref[tag]))
        else:
            ref[tag] = out
    print(json.dumps(res), flush=True)
