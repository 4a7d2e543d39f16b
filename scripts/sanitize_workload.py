import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np, torch, synth, sv_helpers as H
import paper_2509_24328_b200 as sv
from paper_2509_24328_b200.shard import VocabShardedPipeline, run_vocab_sharded_lockstep
prof = sv.Profile.from_dict(synth.load_profile())
for (B, k, V, dt) in [(3, 4, 3001, "bf16"), (2, 3, 1001, "f32")]:
    x = synth.make_inputs(B, k, V, dt, seed=1)
    D, C, T, tok = H.to_torch(x)
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    pipe = sv.Pipeline(B, k, V, D.dtype, prof, L)
    pipe.run(D, C, T, tok, seed=1, offset=0)
    sv.sv_score_schedule(D, C, tok, L, 1.0, 1.0, prof, workspace=pipe.workspace)
    gs = sv.sv_score_filtered(D, C, tok, 20, 0.8, 0.7, 0.7, prof)
    sv.sd_verify_filtered(T, tok, pipe.sched_out["gamma"], gs["fworkspace"], 20, 0.8, 0.7, 1, 0)
    gs = sv.sv_score_filtered(D, C, tok, 0, 0.9, 1.0, 1.0, prof)  # nucleus-only: wide rows at tau 1
    sv.sd_verify_filtered(T, tok, pipe.sched_out["gamma"], gs["fworkspace"], 0, 0.9, 1.0, 1, 0, D=D)
    g = pipe.sched_out["gamma"]
    gn = g.cpu().numpy()
    rows = torch.cat([T[b, : gn[b] + 1] for b in range(B)])
    rp = torch.tensor(np.concatenate([[0], np.cumsum(gn + 1)[:-1]]), dtype=torch.int64, device="cuda")
    sv.sd_verify_ragged(D, rows, rp, tok, g, pipe.score_out["draft_m"], pipe.score_out["draft_l"], pipe.score_out["draft_ptok"])
    sv.sv_profile_build(pipe.score_out["S"].nan_to_num(0), pipe.score_out["A"].nan_to_num(0), pipe.ver_out["accept_ratio"].nan_to_num(0), 5, 4, 10)
    G = 3 if V % 3 == 0 else 1
    VL = V // G
    pipes = [VocabShardedPipeline(B, k, V, G, r, D.dtype, prof, L) for r in range(G)]
    sl = lambda t, r: t[:, :, r * VL:(r + 1) * VL]
    run_vocab_sharded_lockstep(pipes, [sl(D, r) for r in range(G)], [sl(C, r) for r in range(G)], [sl(T, r) for r in range(G)], tok, 1, 0)
    Lg = torch.tensor(synth.latency_table(B * (k + 1) + 1), dtype=torch.float64, device="cuda")
    sv.sv_schedule(pipe.score_out["p_hat"], Lg, sv.SV_SCHED_BATCH_GREEDY)
# wide nucleus of ~4600 tokens (geometric row): the radix fallback of the cut search
import math
r, V = 0.9995, 20000
xg = torch.tensor([[[j * math.log(r) for j in range(V)]] * 2] * 2, dtype=torch.float32, device="cuda")
tg = torch.zeros((2, 2), dtype=torch.int32, device="cuda")
gsw = sv.sv_score_filtered(xg, xg, tg, 0, 0.9, 1.0, 1.0)
T3 = torch.cat([xg, xg[:, :1]], dim=1).contiguous()
sv.sd_verify_filtered(T3, tg, torch.tensor([2, 1], dtype=torch.int32, device="cuda"), gsw["fworkspace"], 0, 0.9, 1.0,
                      1, 0, D=xg)
# the three K1 variants (chosen by launch shape): K1c resident (the small cases above),
# K1c with global re-reads (D + C 41 MB, more than one wave) and the ticket kernel (D + C 82 MB)
for (B, k, V) in [(40, 8, 32000), (80, 8, 32000)]:
    x = synth.make_inputs(B, k, V, "bf16", seed=2)
    D, C, T, tok = H.to_torch(x)
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    sv.Pipeline(B, k, V, D.dtype, prof, L).run(D, C, T, tok, seed=1, offset=0)
torch.cuda.synchronize()
print("sanitizer workload done")
