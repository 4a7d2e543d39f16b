#!/usr/bin/env python3
"""A/B timing of build-time variants of libsv (experiments only; the product ships one build).

    python scripts/k1_ab.py build NAME DEF=VAL ...   # here: build variants/libsv_NAME.so
    python scripts/k1_ab.py run [NAME ...]           # on the GPU: time each variant (+ the product)

Per variant, at the headline (B=80, k=8, V=152064 bf16, two rotating input sets > L2): the mean
CUDA-event time of sv_score alone (K1 + K1e), of the eager step and of the graph-replayed step.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2509_24328_b200", "variants")


def build(name, defs):
    from paper_2509_24328_b200 import build as b
    os.makedirs(VDIR, exist_ok=True)
    print(b.build(defines=defs, out=os.path.join(VDIR, f"libsv_{name}.so")))


def run(names, steps=60, B=80, k=8, V=152064):
    import numpy as np
    import torch

    import paper_2509_24328_b200 as sv
    import synth
    from paper_2509_24328_b200 import _lib
    x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
    dev = torch.device("cuda")

    def h(a):
        return torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16)
    sets = [(h(x["D"]).to(dev), h(x["C"]).to(dev), h(x["T"]).to(dev), torch.from_numpy(x["tok"]).to(dev))
            for _ in range(2)]
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    ref = None
    for name in ["product"] + list(names):
        _lib._lib = None
        _lib.load(_lib.LIB_PATH if name == "product" else os.path.join(VDIR, f"libsv_{name}.so"))
        pipe = sv.Pipeline(B, k, V, torch.bfloat16, prof, L)
        for j in range(6):
            D, C, T, tok = sets[j & 1]
            pipe.run(D, C, T, tok, seed=1, offset=j)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for j in range(steps):
            D, C, T, tok = sets[j & 1]
            ev[j][0].record(st)
            sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=pipe.workspace, out=pipe.score_out)
            ev[j][1].record(st)
        torch.cuda.synchronize()
        k1 = sorted(a.elapsed_time(b) for a, b in ev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for j in range(steps):
            D, C, T, tok = sets[j & 1]
            pipe.run(D, C, T, tok, seed=1, offset=j)
        e1.record(st)
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / steps
        # sd_verify alone (K4..K5b) on the last step's gamma, rotating input sets
        sc, gam = pipe.score_out, pipe.sched_out["gamma"]
        e0.record(st)
        for j in range(steps):
            D, C, T, tok = sets[j & 1]
            sv.sd_verify(D, T, tok, gam, sc["draft_m"], sc["draft_l"], sc["draft_ptok"], 1.0, 1.0, 1, j,
                         workspace=pipe.workspace, out=pipe.ver_out)
        e1.record(st)
        torch.cuda.synchronize()
        verify = e0.elapsed_time(e1) / steps
        vout = (pipe.ver_out["n_accept"].clone(), pipe.ver_out["out_tok"].clone())
        gps = []
        for si in range(2):
            gp = sv.GraphPipeline(B, k, V, torch.bfloat16, prof, L, seed=1, offset0=si)
            for dst, src in zip((gp.D, gp.C, gp.T, gp.tok), sets[si]):
                dst.copy_(src)
            gps.append(gp.capture())
        for j in range(4):
            gps[j & 1].replay()
        torch.cuda.synchronize()
        e0.record(st)
        for j in range(steps):
            gps[j & 1].replay()
        e1.record(st)
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / steps
        out = {n: v.clone() for n, v in pipe.score_out.items()}
        diff = None
        if ref is not None:
            diff = {n: float((out[n] - ref[n]).abs().nan_to_num(0).max()) for n in ("S", "A", "KL", "draft_l")}
            diff["p_hat_eq"] = bool(torch.equal(out["p_hat"], ref["p_hat"]))
            diff["n_accept_eq"] = bool(torch.equal(vout[0], vref[0]))
            diff["out_tok_mismatch"] = int((vout[1] != vref[1]).sum())
        else:
            ref, vref = out, vout
        k1_mean = sum(k1) / len(k1)
        print(json.dumps({"variant": name, "k1_us_mean": k1_mean * 1e3, "k1_us_median": k1[len(k1) // 2] * 1e3,
                          "k1_frac": 2 * B * k * V * 2 / (k1_mean * 1e-3) / 1e9 / 6545.0,
                          "eager_us": eager * 1e3, "verify_us": verify * 1e3, "graph_us": graph * 1e3, "diff_vs_product": diff}), flush=True)
        del gps, pipe


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2], sys.argv[3:])
    else:
        run(sys.argv[2:])
