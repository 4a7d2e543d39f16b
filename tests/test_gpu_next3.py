"""NEXT-3: compacted (ragged) target layout and the whole step captured in a CUDA
graph.  Both are pure re-plumbing of the same kernels, so the pins are bitwise: the ragged call
equals sd_verify on the equivalent dense target, and graph replay j equals an eager step with
Philox offset offset0 + j (P L266 for the compaction; DESIGN R12 for the offset contract)."""
import numpy as np
import pytest

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


@pytest.mark.parametrize("B,k,V,dtype", [(8, 8, 32000, "bf16"), (5, 4, 32003, "bf16"), (4, 3, 1001, "f32"),
                                         (6, 8, 152064, "bf16")])
def test_ragged_target_matches_dense(sv, B, k, V, dtype):
    x = synth.make_inputs(B, k, V, dtype, seed=4242 + V)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    sc = sv.sv_score(D, C, tok, 1.0, 1.0, prof)
    gam = sv.sv_schedule(sc["p_hat"], L)["gamma"]
    gam[0] = k  # exercise the bonus row k and gamma = 0 too
    gam[-1] = 0
    dense = sv.sd_verify(D, T, tok, gam, sc["draft_m"], sc["draft_l"], sc["draft_ptok"], 1.0, 1.0, 11, 3, 0)
    g = gam.cpu().numpy()
    rows = torch.cat([T[b, : g[b] + 1] for b in range(B)])  # compacted: only the verified rows exist
    rowptr = torch.tensor(np.concatenate([[0], np.cumsum(g + 1)[:-1]]), dtype=torch.int64, device="cuda")
    rag = sv.sd_verify_ragged(D, rows, rowptr, tok, gam, sc["draft_m"], sc["draft_l"], sc["draft_ptok"], 1.0, 1.0,
                              11, 3)
    for n in dense:
        assert _eq(dense[n], rag[n]), n


def test_graph_replay_matches_eager(sv):
    B, k, V = 16, 8, 32000
    x = synth.make_inputs(B, k, V, "bf16", seed=77)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    gp = sv.GraphPipeline(B, k, V, torch.bfloat16, prof, L, seed=5, offset0=10)
    gp.D.copy_(D)
    gp.C.copy_(C)
    gp.T.copy_(T)
    gp.tok.copy_(tok)
    gp.capture()
    eager = sv.Pipeline(B, k, V, torch.bfloat16, prof, L)
    for j in range(3):
        out = {n: v.clone() for n, v in gp.replay().items()}
        ref = eager.run(D, C, T, tok, seed=5, offset=10 + j)
        torch.cuda.synchronize()
        for n in ref:
            assert _eq(out[n], ref[n]), (j, n)
    assert int(gp.offset.item()) == 13


@pytest.mark.parametrize("B,k,V,dtype", [(80, 8, 32000, "bf16"), (1, 1, 4096, "f32"), (5, 16, 1001, "f32"),
                                         (3, 8, 152064, "bf16")])
def test_score_schedule_fused_matches_separate(sv, B, k, V, dtype):
    """sv_score_schedule (K3 folded into K1's last row epilogue) == sv_score + sv_schedule, bitwise."""
    x = synth.make_inputs(B, k, V, dtype, seed=808 + V + k)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    ws = sv.new_workspace(B, k, V, D.dtype)
    sc = sv.sv_score(D, C, tok, 1.0, 1.0, prof, workspace=ws)
    sh = sv.sv_schedule(sc["p_hat"], L)
    fc, fh = sv.sv_score_schedule(D, C, tok, L, 1.0, 1.0, prof, workspace=ws)
    torch.cuda.synchronize()
    for n in sc:
        if sc[n] is not None:
            assert _eq(sc[n], fc[n]), n
    for n in sh:
        assert _eq(sh[n], fh[n]), n
    # a bad latency entry: every sequence flagged, as the separate kernel does
    Lbad = L.clone()
    Lbad[2] = -1.0
    sh = sv.sv_schedule(sc["p_hat"], Lbad)
    fc, fh = sv.sv_score_schedule(D, C, tok, Lbad, 1.0, 1.0, prof, workspace=ws)
    torch.cuda.synchronize()
    for n in sh:
        assert _eq(sh[n], fh[n]), n


def test_graph_replay_headline_size(sv):
    """The bench's headline launch configuration (GraphPipeline: sv_score, sv_schedule,
    sd_verify_ragged in one graph) at B=80, k=8, V=152064 bf16 equals the eager pipeline
    bitwise (which test_gpu_parity checks against the oracle at this size)."""
    B, k, V = 80, 8, 152064
    x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(synth.load_profile())
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    gp = sv.GraphPipeline(B, k, V, torch.bfloat16, prof, L, seed=0xC0FFEE, offset0=4)
    gp.D.copy_(D)
    gp.C.copy_(C)
    gp.T.copy_(T)
    gp.tok.copy_(tok)
    gp.capture()
    out = {n: v.clone() for n, v in gp.replay().items()}
    ref = sv.Pipeline(B, k, V, torch.bfloat16, prof, L).run(D, C, T, tok, seed=0xC0FFEE, offset=4)
    torch.cuda.synchronize()
    for n in ref:
        assert _eq(out[n], ref[n]), n
