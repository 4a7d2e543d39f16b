"""sv_step (the whole step in one cluster launch): every output must equal sv_score ->
sv_schedule(PER_ROW) -> sd_verify_ragged on the same inputs bit for bit (the same device code runs
every phase, DESIGN §5 "fused small-batch step"), and the oracle at BASELINE config 1."""
import numpy as np
import pytest

import oracle
import synth
import sv_helpers as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sv():
    import paper_2509_24328_b200 as sv
    sv.load_library()
    return sv


def _eq(a, b):
    a, b = a.cpu().numpy(), b.cpu().numpy()
    return np.array_equal(np.nan_to_num(a, nan=7.0), np.nan_to_num(b, nan=7.0))


def _three_calls(sv, D, C, T, tok, prof, L, tau, seed, offset, seq_base):
    B, k, V = D.shape
    sc = sv.sv_score(D, C, tok, tau[0], tau[1], prof)
    sh = sv.sv_schedule(sc["p_hat"], L)
    rowptr = torch.arange(B, dtype=torch.int64, device="cuda") * (k + 1)
    ver = sv.sd_verify_ragged(D, T.reshape(-1, V), rowptr, tok, sh["gamma"], sc["draft_m"], sc["draft_l"],
                              sc["draft_ptok"], tau[0], tau[2], seed, offset, None, seq_base)
    return sc, sh, ver


@pytest.mark.parametrize("B,k,V,dtype,bad", [
    (4, 4, 32000, "f32", False),     # BASELINE config 1
    (2, 8, 152064, "bf16", False),   # the headline vocabulary
    (5, 16, 1001, "f32", False),     # k = 16: a 16-CTA cluster; unaligned rows
    (3, 3, 4099, "bf16", True),      # unaligned, with a NaN draft row and a bad token
    (64, 8, 128256, "bf16", False),  # B k = 512, the largest shape sv_step takes
    (1, 1, 16, "f32", False),
])
def test_step_matches_three_calls(sv, B, k, V, dtype, bad):
    x = synth.make_inputs(B, k, V, dtype, seed=9000 + V + k)
    D, C, T, tok = H.to_torch(x)
    if bad:
        D[0, 1, 5] = float("nan")
        tok[B - 1, 0] = -1
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    tau = (1.0, 0.8, 1.2)
    rowptr = torch.arange(B, dtype=torch.int64, device="cuda") * (k + 1)
    off = torch.tensor([7], dtype=torch.int64, device="cuda")
    r = sv.sv_step(D, C, T.reshape(-1, V), rowptr, tok, L, prof, tau, 1, 31, 0, off, 5)
    assert r is not None
    sc, sh, ver = r
    rsc, rsh, rver = _three_calls(sv, D, C, T, tok, prof, L, tau, 31, 7, 5)
    torch.cuda.synchronize()
    for got, ref in ((sc, rsc), (sh, rsh), (ver, rver)):
        for n in ref:
            assert _eq(got[n], ref[n]), n


def test_step_declines_large_batches(sv):
    B, k, V = 80, 8, 256
    x = synth.make_inputs(B, k, V, "bf16", seed=1)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    rowptr = torch.arange(B, dtype=torch.int64, device="cuda") * (k + 1)
    assert sv.sv_step(D, C, T.reshape(-1, V), rowptr, tok, L, prof) is None  # B k = 640 > 512


def test_step_vs_oracle_config1(sv):
    B, k, V = 4, 4, 32000
    x = synth.make_inputs(B, k, V, "f32", seed=42)
    D, C, T, tok = H.to_torch(x)
    prof_dict = synth.load_profile()
    prof = sv.Profile.from_dict(prof_dict)
    lat = synth.latency_table(k + 2)
    L = torch.tensor(lat, dtype=torch.float64, device="cuda")
    rowptr = torch.arange(B, dtype=torch.int64, device="cuda") * (k + 1)
    sc, sh, ver = sv.sv_step(D, C, T.reshape(-1, V), rowptr, tok, L, prof, (1.0, 1.0, 1.0), 1, 7, 3)
    torch.cuda.synchronize()
    Dd, Cd, Td = H.oracle_inputs(x)
    rep = H.ParityReport()
    H.compare_score(H.gpu_np(sc), oracle.score(Dd, Cd, x["tok"], 1.0, 1.0, prof_dict), prof_dict, rep)
    gam = sh["gamma"].cpu().numpy()
    rs = oracle.schedule(sc["p_hat"].cpu().numpy().astype(np.float64), lat)
    assert np.array_equal(gam, rs["gamma"])
    H.compare_verify(H.gpu_np(ver), oracle.verify(Dd, Td, x["tok"], gam, 1.0, 1.0, 7, 3, 0), rep,
                     H.oracle_rerun(Dd, Td, x["tok"], gam, 1.0, 1.0, 7, 3, 0))
    print("ties:", rep.ties)


def test_graph_pipeline_step_matches_three_call_graph(sv):
    """GraphPipeline replays through sv_step equal the three-call graph, replay by replay."""
    B, k, V = 16, 8, 128256
    x = synth.make_inputs(B, k, V, "bf16", seed=88)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    gps = []
    for use in (True, False):
        gp = sv.GraphPipeline(B, k, V, torch.bfloat16, prof, L, seed=3, offset0=100, use_step=use)
        for dst, src in zip((gp.D, gp.C, gp.T, gp.tok), (D, C, T, tok)):
            dst.copy_(src)
        gps.append(gp.capture())
    for j in range(3):
        a = {n: v.clone() for n, v in gps[0].replay().items()}
        b = {n: v.clone() for n, v in gps[1].replay().items()}
        torch.cuda.synchronize()
        for n in a:
            assert _eq(a[n], b[n]), (j, n)
