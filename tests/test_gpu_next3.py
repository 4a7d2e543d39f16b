"""NEXT-3: compacted (ragged) target layout and the whole step captured in a CUDA
graph.  Both are pure re-plumbing of the same kernels, so the pins are bitwise: the ragged call
equals sd_verify on the equivalent dense target, and graph replay j equals an eager step with
Philox offset offset0 + j (P L266 for the compaction; DESIGN R12 for the offset contract)."""
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
    # and the ragged call itself against the oracle (P L266 compaction changes no arithmetic)
    torch.cuda.synchronize()
    Dd, _, Td = H.oracle_inputs(x)
    rv = oracle.verify(Dd, Td, x["tok"], g, 1.0, 1.0, 11, 3, 0)
    rep = H.ParityReport()
    H.compare_verify(H.gpu_np(rag), rv, rep, H.oracle_rerun(Dd, Td, x["tok"], g, 1.0, 1.0, 11, 3, 0))
    print("ties:", rep.ties)


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


def _graph_vs_oracle(sv, B, k, V, dtype, seed_in, offset0, replays, seq_base=0):
    """The bench's timed path -- GraphPipeline (sv_score, sv_schedule, sd_verify_ragged with a
    device-side Philox offset, offset += 1, one CUDA graph) -- replayed `replays` times and every
    replay compared with the oracle on ALL sequences: score and schedule stage-wise, verify at
    offset0 + j (R12: replay j draws the uniforms of offset0 + j)."""
    x = synth.make_inputs(B, k, V, dtype, seed=seed_in, seq_ids=np.arange(seq_base, seq_base + B))
    D, C, T, tok = H.to_torch(x)
    prof_dict = synth.load_profile()
    prof = sv.Profile.from_dict(prof_dict)
    Lh = synth.latency_table(k + 2)
    L = torch.tensor(Lh, dtype=torch.float64, device="cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    gp = sv.GraphPipeline(B, k, V, tdt, prof, L, seed=0xC0FFEE, offset0=offset0, seq_base=seq_base)
    gp.D.copy_(D)
    gp.C.copy_(C)
    gp.T.copy_(T)
    gp.tok.copy_(tok)
    gp.capture()
    outs = []
    for _ in range(replays):
        gv = {n: v.clone() for n, v in gp.replay().items()}
        gs = {n: v.clone() for n, v in gp.pipe.score_out.items()}
        gh = {n: v.clone() for n, v in gp.pipe.sched_out.items()}
        outs.append((gs, gh, gv))
    torch.cuda.synchronize()
    assert int(gp.offset.item()) == offset0 + replays
    del gp, D, C, T
    Dd, Cd, Td = H.oracle_inputs(x)
    rs = oracle.score(Dd, Cd, x["tok"], 1.0, 1.0, prof_dict)
    rep = H.ParityReport()
    for j, (gs, gh, gv) in enumerate(outs):
        gs, gh, gv = H.gpu_np(gs), H.gpu_np(gh), H.gpu_np(gv)
        H.compare_score(gs, rs, prof_dict, rep)
        rh = oracle.schedule(gs["p_hat"].astype(np.float64), Lh)
        assert np.array_equal(gh["gamma"], rh["gamma"])
        assert np.array_equal(gh["exp_accept"], rh["exp_accept"].astype(np.float32))
        gam = gh["gamma"]
        off = offset0 + j
        rv = oracle.verify(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, off, seq_base)
        H.compare_verify(gv, rv, rep, H.oracle_rerun(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, off, seq_base))
    return rep


def test_graph_replay_headline_size_vs_oracle(sv):
    """BASELINE config 3 at full size (B=80, k=8, V=152064 bf16), the exact launch configuration
    bench.py times, three consecutive replays, all 80 sequences against the oracle."""
    rep = _graph_vs_oracle(sv, 80, 8, 152064, "bf16", 0x5EED, offset0=4, replays=3)
    print("ties:", rep.ties)


@pytest.mark.parametrize("B,k,V,dtype,seq_base", [(4, 4, 32000, "f32", 0), (32, 8, 32000, "bf16", 0),
                                                  (40, 8, 152064, "bf16", 40)])
def test_graph_replay_configs_vs_oracle(sv, B, k, V, dtype, seq_base):
    """Configs 1 and 2 and one rank's half of config 3 at world size 2 (seq_base = 40) through
    the graph path, three replays each, against the oracle."""
    rep = _graph_vs_oracle(sv, B, k, V, dtype, 0x5EED + V + B, offset0=7, replays=3, seq_base=seq_base)
    print("ties:", rep.ties)
