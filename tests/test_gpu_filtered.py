"""NEXT-2: the SV path under sampling filters (temperature -> top_k -> top_p ->
renormalise on draft, companion and target; S L73-81, L183, L238; P L731-743 Table 5) against
the fp64 filtered oracle (oracle/filtered.py) on the same inputs.  Draft tokens are drawn from
the FILTERED draft distribution, as a filtered drafter would.  Continuous outputs within the
north_star tolerance; integer decisions exact unless the oracle's margin is inside the 1e-6 tie
band (logged)."""
import numpy as np
import pytest

import oracle
import synth
import sv_helpers as H
from oracle.filtered import filter_dist, score_filtered, verify_filtered

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2509_24328_b200 as sv
    sv.load_library()
    return sv


@pytest.mark.parametrize("B,k,V,dtype,top_k,top_p,tau", [
    (8, 4, 32000, "bf16", 20, 0.8, 0.7),    # Qwen settings (Table 5)
    (3, 8, 152064, "bf16", 20, 0.8, 0.7),   # headline vocabulary
    (6, 3, 1001, "f32", 5, 0.9, 1.0),
    (4, 4, 4096, "bf16", 32, 1.0, 0.6),     # top-k only
    (3, 2, 50, "f32", 1, 1.0, 1.0),         # greedy
])
def test_filtered_parity(sv, B, k, V, dtype, top_k, top_p, tau):
    x = synth.make_inputs(B, k, V, dtype, seed=99 + V + top_k)
    Dd, Cd, Td = H.oracle_inputs(x)
    rng = np.random.default_rng(V + k)
    tok = np.zeros((B, k), dtype=np.int32)
    for b in range(B):
        for i in range(k):
            p, _ = filter_dist(Dd[b, i], tau, top_k, top_p)
            tok[b, i] = rng.choice(V, p=p / p.sum())
    D, C, T, _ = H.to_torch(x)
    tk = torch.from_numpy(tok).cuda()
    pd = synth.load_profile()
    prof = sv.Profile.from_dict(pd)
    gs = sv.sv_score_filtered(D, C, tk, top_k, top_p, tau, tau, prof)
    torch.cuda.synchronize()
    rs = score_filtered(Dd, Cd, tok, tau, tau, top_k, top_p)
    g = {n: gs[n].cpu().numpy() for n in ("S", "A", "KL", "p_hat", "draft_ptok", "status")}
    assert np.array_equal(g["status"], rs["status"])
    ok = rs["status"] == 0
    for n in ("S", "A", "KL"):
        assert H.close(g[n][ok], rs[n][ok]).all(), (n, g[n][ok], rs[n][ok])
    assert H.close(g["draft_ptok"], rs["pd_tok"]).all()
    for idx in zip(*np.nonzero(ok)):
        want = oracle.lookup(pd["s_edges"], pd["a_edges"], pd["cells"], float(g["S"][idx]), float(g["A"][idx]))
        assert np.float32(want) == g["p_hat"][idx]
    gam = rng.integers(0, k + 1, B).astype(np.int32)
    gv = sv.sd_verify_filtered(T, tk, torch.from_numpy(gam).cuda(), gs["fworkspace"], top_k, top_p, tau, seed=5,
                               offset=2)
    torch.cuda.synchronize()
    gv = {n: v.cpu().numpy() for n, v in gv.items()}
    rv = verify_filtered(Dd, Td, tok, gam, tau, tau, top_k, top_p, 5, 2)
    tie = rv["margin"] < 1e-6
    assert np.array_equal(gv["n_accept"][~tie], rv["n_accept"][~tie])
    assert np.array_equal(gv["out_tok"][~tie], rv["out_tok"][~tie])
    assert H.close(gv["resid_mass"][~tie], rv["resid_mass"][~tie]).all()
    r_ok = ~np.isnan(rv["accept_ratio"])
    assert np.array_equal(np.isnan(gv["accept_ratio"]), ~r_ok)
    assert H.close(gv["accept_ratio"][r_ok], rv["accept_ratio"][r_ok]).all()
    print("ties:", int(tie.sum()))


def test_filtered_unsupported_nucleus_only(sv):
    B, k, V = 2, 2, 64
    x = synth.make_inputs(B, k, V, "f32", seed=1)
    D, C, T, tok = H.to_torch(x)
    with pytest.raises(sv.SvError):
        sv.sv_score_filtered(D, C, tok, 0, 0.9)
