"""GPU parity of the vocab-sharded staging (BASELINE config 4; include/sv.h
"Vocab-sharded staging").  One GPU simulates G ranks: each rank's pipeline sees a column slice
[r V/G, (r+1) V/G) of the same logits, the exchanges are concatenations and the token
all-reduce a max (paper_2509_24328_b200.shard.run_vocab_sharded_lockstep).  Every rank must
produce identical outputs, and they must match the fp64 oracle stage by stage with the same
tolerances / tie bands as the unsharded path."""
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


def run_sharded(sv, x, G, prof_dict, seed=0xC0FFEE, offset=5, seq_base=0):
    from paper_2509_24328_b200.shard import VocabShardedPipeline, run_vocab_sharded_lockstep
    B, k, V = x["B"], x["k"], x["V"]
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(prof_dict)
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    VL = V // G
    pipes = [VocabShardedPipeline(B, k, V, G, r, D.dtype, prof, L) for r in range(G)]
    sl = lambda t, r: t[:, :, r * VL:(r + 1) * VL]  # noqa: E731  (column views, vocabulary contiguous)
    outs = run_vocab_sharded_lockstep(pipes, [sl(D, r) for r in range(G)], [sl(C, r) for r in range(G)],
                                      [sl(T, r) for r in range(G)], tok, seed, offset, seq_base)
    torch.cuda.synchronize()
    return pipes, outs


@pytest.mark.parametrize("B,k,V,dtype,G", [
    (4, 4, 32000, "f32", 2),
    (8, 8, 32000, "bf16", 4),
    (3, 8, 152064, "bf16", 8),   # config 4: Qwen vocabulary over 8 ranks
    (5, 3, 3000, "bf16", 3),
])
def test_vocab_sharded_matches_oracle(sv, B, k, V, dtype, G):
    prof_dict = synth.load_profile()
    x = synth.make_inputs(B, k, V, dtype, seed=777 + V + G)
    pipes, outs = run_sharded(sv, x, G, prof_dict)
    # identical on every rank
    s0 = H.gpu_np(pipes[0].score_out)
    for p in pipes[1:]:
        sp = H.gpu_np(p.score_out)
        for n in s0:
            assert np.array_equal(np.nan_to_num(s0[n], nan=7.0), np.nan_to_num(sp[n], nan=7.0)), n
        assert torch.equal(p.sched_out["gamma"], pipes[0].sched_out["gamma"])
        for n in ("n_accept", "out_tok", "accept_ratio", "resid_mass", "status"):
            a, b = outs[0][n].cpu().numpy(), p.ver_out[n].cpu().numpy()
            assert np.array_equal(np.nan_to_num(a, nan=7.0), np.nan_to_num(b, nan=7.0)), n
    # vs the oracle, stage by stage
    rep = H.ParityReport()
    Dd, Cd, Td = H.oracle_inputs(x)
    H.compare_score(s0, oracle.score(Dd, Cd, x["tok"], 1.0, 1.0, prof_dict), prof_dict, rep)
    gam = pipes[0].sched_out["gamma"].cpu().numpy()
    rh = oracle.schedule(s0["p_hat"].astype(np.float64), synth.latency_table(k + 2))
    assert np.array_equal(gam, rh["gamma"])
    gv = H.gpu_np(outs[0])
    H.compare_verify(gv, oracle.verify(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, 5, 0), rep,
                     H.oracle_rerun(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, 5, 0))
    print("ties:", rep.ties)


def test_vocab_sharded_forced_gamma_and_bonus(sv):
    """gamma = k everywhere (identical rows -> every token accepted -> bonus sample of row k)."""
    prof_dict = synth.load_profile()
    B, k, V, G = 3, 4, 4096, 4
    x = synth.make_inputs(B, k, V, "bf16", seed=31)
    x["D"] = x["T"][:, :k].copy()
    x["C"] = x["T"][:, :k].copy()
    pipes, outs = run_sharded(sv, x, G, prof_dict)
    gv = H.gpu_np(outs[0])
    gam = pipes[0].sched_out["gamma"].cpu().numpy()
    assert np.array_equal(gv["n_accept"], gam)  # identical rows: every verified token accepted
    Dd, Cd, Td = H.oracle_inputs(x)
    rep = H.ParityReport()
    H.compare_verify(gv, oracle.verify(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, 5, 0), rep,
                     H.oracle_rerun(Dd, Td, x["tok"], gam, 1.0, 1.0, 0xC0FFEE, 5, 0))
