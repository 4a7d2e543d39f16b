import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle, synth, sv_helpers as H
import paper_2509_24328_b200 as sv
from oracle import profile as oprof
pd_ = synth.load_profile()
for (B,k,V,dt) in [(4,4,32000,"f32"),(32,8,32000,"bf16"),(2,8,152064,"bf16")]:
    x = synth.make_inputs(B,k,V,dt,seed=42)
    D,C,T,tok = H.to_torch(x)
    prof = sv.Profile.from_dict(pd_)
    gs = H.gpu_np(sv.sv_score(D,C,tok,1.0,1.0,prof)); torch.cuda.synchronize()
    Dd,Cd,Td = H.oracle_inputs(x)
    rs = oracle.score(Dd,Cd,x["tok"],1.0,1.0,pd_)
    print(B,k,V,dt, "status", gs["status"].ravel()[:8], rs["status"].ravel()[:8])
    for n in ("S","A","KL","draft_ptok"):
        r = rs["pd_tok" if n=="draft_ptok" else n]
        err = np.abs(gs[n]-r)/np.maximum(np.abs(r),1e-30)
        print(n, "max rel err", np.nanmax(err), "gpu", gs[n].ravel()[:4], "orc", r.ravel()[:4])
    print("phat gpu", gs["p_hat"].ravel()[:8]); print("phat orc", rs["p_hat"].ravel()[:8])
    sb_g=[oprof.bin_of(pd_["s_edges"],v) for v in gs["S"].ravel()[:8]]; sb_r=[oprof.bin_of(pd_["s_edges"],v) for v in rs["S"].ravel()[:8]]
    ab_g=[oprof.bin_of(pd_["a_edges"],v) for v in gs["A"].ravel()[:8]]; ab_r=[oprof.bin_of(pd_["a_edges"],v) for v in rs["A"].ravel()[:8]]
    print("bins", sb_g, sb_r, ab_g, ab_r)
    print("dm", gs["draft_m"].ravel()[:4], Dd.max(-1).ravel()[:4])
    l = np.exp(Dd - Dd.max(-1, keepdims=True)).sum(-1)
    print("dl rel", np.max(np.abs(gs["draft_l"]-l)/l))
