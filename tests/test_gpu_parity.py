"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs, stage by stage.  Each stage is fed the GPU's own upstream outputs,
so a logged tie upstream cannot cascade.  All tests need a B200 (-m gpu)."""
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


@pytest.fixture(scope="module")
def prof_dict():
    return synth.load_profile()


def run_case(sv, prof_dict, x, tau=(1.0, 1.0, 1.0), seed=0xC0FFEE, offset=3, seq_base=0, gamma=None, report=None):
    """Full pipeline on GPU + stage-wise oracle comparison; returns (gpu dicts, report)."""
    rep = report or H.ParityReport()
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(prof_dict)
    L = torch.tensor(synth.latency_table(x["k"] + 2), dtype=torch.float64, device="cuda")
    gs = sv.sv_score(D, C, tok, tau[0], tau[1], prof)
    if gamma is None:
        gh = sv.sv_schedule(gs["p_hat"], L)
        gam = gh["gamma"]
    else:
        gam = torch.as_tensor(np.asarray(gamma, dtype=np.int32), device="cuda")
        gh = None
    gv = sv.sd_verify(D, T, tok, gam, gs["draft_m"], gs["draft_l"], gs["draft_ptok"], tau[0], tau[2],
                      seed, offset, seq_base)
    torch.cuda.synchronize()
    gs, gv = H.gpu_np(gs), H.gpu_np(gv)
    Dd, Cd, Td = H.oracle_inputs(x)
    rs = oracle.score(Dd, Cd, x["tok"], tau[0], tau[1], prof_dict)
    H.compare_score(gs, rs, prof_dict, rep)
    if gh is not None:
        gh = H.gpu_np(gh)
        rh = oracle.schedule(gs["p_hat"].astype(np.float64), synth.latency_table(x["k"] + 2))
        assert np.array_equal(gh["gamma"], rh["gamma"])  # bit-exact given the same p_hat
        assert np.array_equal(gh["exp_accept"], rh["exp_accept"].astype(np.float32))
        assert np.array_equal(gh["goodput"], rh["goodput"].astype(np.float32))
        gam_np = gh["gamma"]
    else:
        gam_np = np.asarray(gamma, dtype=np.int32)
    rv = oracle.verify(Dd, Td, x["tok"], gam_np, tau[0], tau[2], seed, offset, seq_base)
    H.compare_verify(gv, rv, rep, H.oracle_rerun(Dd, Td, x["tok"], gam_np, tau[0], tau[2], seed, offset, seq_base))
    return gs, gv, gam_np, rep


# ----------------------------------------------------------------- configs
@pytest.mark.parametrize("B,k,V,dtype", [
    (4, 4, 32000, "f32"),     # BASELINE config 1
    (32, 8, 32000, "bf16"),   # BASELINE config 2
    (6, 5, 32003, "bf16"),    # ragged tail, unaligned rows
    (5, 3, 1001, "f32"),      # unaligned fp32 rows
    (3, 16, 4096, "bf16"),    # k = 16
    (7, 1, 2, "f32"),         # V = 2
    (5, 2, 13, "bf16"),       # tiny V, odd
    (2, 8, 152064, "bf16"),   # headline vocabulary
    (3, 4, 128256, "bf16"),   # sweep vocabulary
    (2, 2, 70000, "f32"),     # fp32 at cluster 4
])
def test_pipeline_parity(sv, prof_dict, B, k, V, dtype):
    x = synth.make_inputs(B, k, V, dtype, seed=1234 + V + k)
    *_, rep = run_case(sv, prof_dict, x)
    print("ties:", rep.ties)


def test_temperature(sv, prof_dict):
    x = synth.make_inputs(8, 5, 5000, "bf16", seed=77, tau_d=0.7)
    run_case(sv, prof_dict, x, tau=(0.7, 0.6, 0.8))


@pytest.mark.parametrize("g", [0, "k", "mixed"])
def test_forced_gamma(sv, prof_dict, g):
    x = synth.make_inputs(12, 6, 20000, "bf16", seed=5)
    gam = {0: np.zeros(12), "k": np.full(12, 6), "mixed": np.arange(12) % 7}[g]
    run_case(sv, prof_dict, x, gamma=gam)


def test_identical_rows_accept_all(sv, prof_dict):
    # P L159 / north_star: identical distributions -> S = 1, A = 1, KL = 0 and N = gamma
    x = synth.make_inputs(4, 4, 3000, "bf16", seed=9)
    x["C"] = x["D"].copy()
    x["T"][:, :4] = x["D"]
    gs, gv, gam, _ = run_case(sv, prof_dict, x, gamma=np.full(4, 4))
    assert np.allclose(gs["S"], 1.0, atol=2e-6) and np.all(gs["A"] == 1.0) and np.all(gs["KL"] == 0.0)
    assert np.array_equal(gv["n_accept"], gam)


def test_disjoint_supports(sv, prof_dict):
    # disjoint supports -> S = 0, A = 0 (P L159); target disjoint from the draft -> N = 0
    B, k, V = 3, 2, 64
    D = np.full((B, k, V), -np.inf, np.float32)
    C = np.full((B, k, V), -np.inf, np.float32)
    T = np.full((B, k + 1, V), -np.inf, np.float32)
    rng = np.random.default_rng(3)
    D[..., :32] = rng.normal(0, 1, (B, k, 32))
    C[..., 32:] = rng.normal(0, 1, (B, k, 32))
    T[..., 32:] = rng.normal(0, 1, (B, k + 1, 32))
    tok = rng.integers(0, 32, (B, k)).astype(np.int32)
    x = {"D": D, "C": C, "T": T, "tok": tok, "dtype": "f32", "B": B, "k": k, "V": V}
    gs, gv, _, _ = run_case(sv, prof_dict, x, gamma=np.full(B, k))
    assert np.all(gs["S"] == 0) and np.all(gs["A"] == 0) and np.all(np.isinf(gs["KL"]))
    assert np.all(gv["n_accept"] == 0) and np.all(gv["out_tok"] >= 32)


def test_data_errors(sv, prof_dict):
    x = synth.make_inputs(6, 3, 2048, "f32", seed=11)
    x["D"][0, 1, 7] = np.nan              # NaN draft logit
    x["C"][1, 0, :] = -np.inf             # all -inf companion row
    x["tok"][2, 2] = 5000                 # token out of range
    x["D"][3, 0, x["tok"][3, 0]] = -np.inf  # p_d(t) = 0
    x["T"][4, 1, 3] = np.inf              # +inf target logit
    gs, gv, _, _ = run_case(sv, prof_dict, x, gamma=np.full(6, 3))
    assert gs["status"][0, 1] & oracle.ROW_NAN and gs["status"][1, 0] & oracle.ROW_ALL_NEG_INF
    assert gs["status"][2, 2] & oracle.ROW_BAD_TOKEN and gs["status"][3, 0] & oracle.ROW_DRAFT_ZERO
    assert gv["status"][4] & oracle.ROW_NAN and gv["out_tok"][4] == -1


def test_bad_gamma(sv, prof_dict):
    x = synth.make_inputs(3, 4, 1000, "bf16", seed=12)
    _, gv, _, _ = run_case(sv, prof_dict, x, gamma=np.array([-1, 5, 2]))
    assert gv["status"][0] & oracle.ROW_BAD_GAMMA and gv["status"][1] & oracle.ROW_BAD_GAMMA
    assert gv["status"][2] == 0


def test_determinism_and_batch_split(sv, prof_dict):
    # identical inputs -> identical bits; a sub-batch with seq_base = its first id gives the
    # same results as the full batch (independent of the GPU count)
    x = synth.make_inputs(10, 4, 40000, "bf16", seed=21)
    a = run_case(sv, prof_dict, x)
    b = run_case(sv, prof_dict, x)
    for k_ in ("S", "A", "KL", "p_hat", "draft_l"):
        assert np.array_equal(a[0][k_], b[0][k_], equal_nan=True)
    for k_ in ("n_accept", "out_tok", "resid_mass"):
        assert np.array_equal(a[1][k_], b[1][k_], equal_nan=True)
    sub = {kk: (v[4:10] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == 10 else v)
           for kk, v in x.items()}
    sub["B"] = 6
    c = run_case(sv, prof_dict, sub, seq_base=4)
    for k_ in ("S", "A", "KL", "p_hat"):
        assert np.array_equal(a[0][k_][4:], c[0][k_], equal_nan=True)
    for k_ in ("n_accept", "out_tok", "resid_mass"):
        assert np.array_equal(a[1][k_][4:], c[1][k_], equal_nan=True)


@pytest.mark.parametrize("B,k,V,parts", [
    (80, 8, 32000, ((0, 40), (40, 42), (77, 80))),
    (8, 8, 300000, ((0, 1), (3, 6))),   # cs = 8: the widest K1c cluster (8 CTAs) vs the ticket kernel
])
def test_k1_variants_bit_identical(sv, prof_dict, B, k, V, parts):
    """sv_score picks its K1 kernel by launch shape: at V = 32000 bf16 the whole batch
    B = 80 (D + C 82 MB) runs the ticket kernel, B = 40 (41 MB, more than one wave) K1c with
    cluster-exchanged partials, B = 2 K1c with shared-memory resident chunks; at V = 300000 (cs =
    8 chunks per row) B = 8 runs the ticket kernel and its sub-batches K1c.  All share the chunking
    and every reduction order, so the rows of a sub-batch must match the full batch bit for bit
    (the batch-sharded multi-GPU layout relies on it)."""
    x = synth.make_inputs(B, k, V, "bf16", seed=33)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(prof_dict)
    keys = ("S", "A", "KL", "p_hat", "draft_m", "draft_l", "draft_ptok", "status")
    full = H.gpu_np(sv.sv_score(D, C, tok, 1.0, 1.0, prof))
    for lo, hi in parts:
        part = H.gpu_np(sv.sv_score(D[lo:hi].contiguous(), C[lo:hi].contiguous(), tok[lo:hi].contiguous(), 1.0, 1.0,
                                    prof))
        for k_ in keys:
            assert np.array_equal(full[k_][lo:hi], part[k_], equal_nan=True), (lo, hi, k_)
    # and the full batch against the oracle on sampled sequences
    rep = H.ParityReport()
    idx = np.array(sorted({0, B // 2 - 1, B // 2, B - 1}))
    Dd, Cd, _ = H.oracle_inputs({**x, "D": x["D"][idx], "C": x["C"][idx], "T": x["T"][idx]})
    rs = oracle.score(Dd, Cd, x["tok"][idx], 1.0, 1.0, prof_dict)
    H.compare_score({k_: full[k_][idx] for k_ in full}, rs, prof_dict, rep)


def test_broadcast_losslessness(sv):
    # S L156, L521: the emitted first token follows P_t (chi^2 / TV < 0.005 over 10^6 trials),
    # and P(accept) = sum min(p_d, p_t); stride_b = 0 broadcast rows, fresh t ~ p_d per trial
    rng = np.random.default_rng(31)
    n, V = 1_000_000, 6
    for trial in range(3):
        pd = rng.dirichlet(np.ones(V))
        pt = rng.dirichlet(np.ones(V))
        D = torch.tensor(np.log(pd), dtype=torch.float32, device="cuda").view(1, 1, V).expand(n, 1, V)
        T = torch.tensor(np.log(pt), dtype=torch.float32, device="cuda").view(1, 1, V).expand(n, 2, V)
        tok = torch.as_tensor(rng.choice(V, size=(n, 1), p=pd).astype(np.int32), device="cuda")
        gs = sv.sv_score(D, D, tok)
        gam = torch.ones(n, dtype=torch.int32, device="cuda")
        gv = sv.sd_verify(D, T, tok, gam, gs["draft_m"], gs["draft_l"], gs["draft_ptok"], seed=trial, offset=0)
        acc = (gv["n_accept"] == 1).cpu().numpy()
        emitted = np.where(acc, tok[:, 0].cpu().numpy(), gv["out_tok"].cpu().numpy())
        freq = np.bincount(emitted, minlength=V) / n
        assert np.abs(freq - pt).sum() / 2 < 0.005
        alpha = np.minimum(pd, pt).sum()
        assert abs(acc.mean() - alpha) < 5 * np.sqrt(alpha * (1 - alpha) / n)


def test_batch_greedy_matches_oracle(sv):
    rng = np.random.default_rng(41)
    for B, k in [(2, 2), (5, 4), (80, 8), (300, 16)]:
        ph = rng.random((B, k)).astype(np.float32) ** 0.5
        L = synth.latency_table(B * (k + 1) + 1, base=4.0 * B, knee=B * 2, slope=1.0)
        g = sv.sv_schedule(torch.as_tensor(ph, device="cuda"), torch.as_tensor(L, device="cuda"),
                           mode=sv.SV_SCHED_BATCH_GREEDY)
        torch.cuda.synchronize()
        r = oracle.batch_greedy(ph.astype(np.float64), L)
        assert np.array_equal(g["gamma"].cpu().numpy(), r["gamma"])
        assert np.array_equal(g["exp_accept"].cpu().numpy(), r["exp_accept"].astype(np.float32))
    # S L410 hand trace
    g = sv.sv_schedule(torch.tensor([[0.9, 0.9], [0.8, 0.8]], device="cuda"),
                       torch.as_tensor(synth.latency_table(10), device="cuda"), mode=sv.SV_SCHED_BATCH_GREEDY)
    assert g["gamma"].tolist() == [2, 1]


def test_headline_full_size_sampled(sv, prof_dict):
    """BASELINE config 3 at full size in the bench's launch configuration; the oracle checks a
    sample of sequences one by one (each sequence is independent given seq_base)."""
    B, k, V = 80, 8, 152064
    x = synth.make_inputs(B, k, V, "bf16", seed=0x5EED)
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(prof_dict)
    L = torch.tensor(synth.latency_table(k + 2), dtype=torch.float64, device="cuda")
    pipe = sv.Pipeline(B, k, V, torch.bfloat16, prof, L)
    gv = H.gpu_np(pipe.run(D, C, T, tok, seed=0xC0FFEE, offset=1))
    gs = H.gpu_np(pipe.score_out)
    gam = pipe.sched_out["gamma"].cpu().numpy()
    rep = H.ParityReport()
    for b in (0, 13, 41, 79):
        sub = {kk: (v[b:b + 1] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == B else v)
               for kk, v in x.items()}
        Dd, Cd, Td = H.oracle_inputs(sub)
        rs = oracle.score(Dd, Cd, sub["tok"], 1.0, 1.0, prof_dict)
        H.compare_score({kk: v[b:b + 1] for kk, v in gs.items()}, rs, prof_dict, rep)
        rv = oracle.verify(Dd, Td, sub["tok"], gam[b:b + 1], 1.0, 1.0, 0xC0FFEE, 1, b)
        H.compare_verify({kk: v[b:b + 1] for kk, v in gv.items()}, rv, rep,
                         H.oracle_rerun(Dd, Td, sub["tok"], gam[b:b + 1], 1.0, 1.0, 0xC0FFEE, 1, b))
    print("ties:", rep.ties)


@pytest.mark.parametrize("B,k", [(4, 2), (12, 4), (6, 8)])
def test_config5_sweep_points(sv, prof_dict, B, k):
    """BASELINE config 5: V = 128256 bf16, k in {2, 4, 8}, alignment swept so the per-sequence
    acceptance spans ~0.1..0.9 (synth 'sweep' amplitudes)."""
    x = synth.make_inputs(B, k, 128256, "bf16", seed=5000 + B * k, alignment="sweep")
    *_, rep = run_case(sv, prof_dict, x)
    print("ties:", rep.ties)


@pytest.mark.parametrize("B,k,V,dtype", [
    (1, 1, 1_000_003, "bf16"),   # one very long row: 25 chunk tasks, 489 K4 splits, ragged tail
    (512, 16, 256, "bf16"),      # many short rows at the k limit (8192 positions)
    (1, 16, 33, "f32"),          # k = 16 with V barely above a unit
])
def test_extreme_shapes(sv, prof_dict, B, k, V, dtype):
    x = synth.make_inputs(B, k, V, dtype, seed=31337 + V)
    *_, rep = run_case(sv, prof_dict, x)
    print("ties:", rep.ties)


def test_golden_convention_vector_gpu(sv):
    """SURVEY §8(c)'s golden convention vector (tests/golden/convention_vector.json) through the
    CUDA path: every printed value within its 6-decimal rounding, integer decisions exact."""
    g, x, Lh = H.load_golden()
    e, st = g["expected"], g["setup"]
    D, C, T, tok = H.to_torch(x)
    prof = sv.Profile.from_dict(st["profile"])
    L = torch.tensor(Lh, dtype=torch.float64, device="cuda")
    gs = sv.sv_score(D, C, tok, 1.0, 1.0, prof)
    gh = sv.sv_schedule(gs["p_hat"], L)
    gv = sv.sd_verify(D, T, tok, gh["gamma"], gs["draft_m"], gs["draft_l"], gs["draft_ptok"], 1.0, 1.0,
                      st["seed"], st["offset"], st["seq_base"])
    torch.cuda.synchronize()
    gs, gh, gv = H.gpu_np(gs), H.gpu_np(gh), H.gpu_np(gv)
    tol = 6e-7
    for n in ("S", "A", "KL"):
        assert np.allclose(gs[n], e[n], rtol=0, atol=tol), (n, gs[n])
    assert np.array_equal(gs["p_hat"], np.array(e["p_hat"], dtype=np.float32))
    assert gh["gamma"].tolist() == e["gamma"]
    want_ratio = np.array([[np.nan if v is None else v for v in row] for row in e["accept_ratio"]])
    assert np.allclose(gv["accept_ratio"], want_ratio, rtol=0, atol=tol, equal_nan=True)
    assert gv["n_accept"].tolist() == e["n_accept"] and gv["out_tok"].tolist() == e["out_tok"]
    assert np.allclose(gv["resid_mass"], e["resid_mass"], rtol=0, atol=tol)


def test_schedule_literal_goodput_plus_one_0(sv):
    """R2's literal reading g_j = E_j / L[j] (plus_one = 0) on the GPU: bit-exact with the oracle,
    including the S L392 chain where it moves gamma from 2 to 3."""
    rng = np.random.default_rng(19)
    ph = np.concatenate([np.array([[0.9, 0.9, 0.2, 0.2, 0.2, 0.0, 0.0, 0.0]], dtype=np.float32),
                         (rng.random((300, 8)) ** rng.uniform(0.2, 3, (300, 1))).astype(np.float32)])
    for Lh in (np.array([10.0 + n for n in range(10)]), synth.latency_table(10),
               np.cumsum(rng.random(10) + 0.05)):
        g = sv.sv_schedule(torch.as_tensor(ph, device="cuda"), torch.as_tensor(Lh, device="cuda"), plus_one=0)
        torch.cuda.synchronize()
        r = oracle.schedule(ph.astype(np.float64), Lh, plus_one=0)
        assert np.array_equal(g["gamma"].cpu().numpy(), r["gamma"])
        assert np.array_equal(g["exp_accept"].cpu().numpy(), r["exp_accept"].astype(np.float32))
        assert np.array_equal(g["goodput"].cpu().numpy(), r["goodput"].astype(np.float32))
    g = sv.sv_schedule(torch.as_tensor(ph[:1], device="cuda"),
                       torch.as_tensor(np.array([10.0 + n for n in range(10)]), device="cuda"), plus_one=0)
    assert int(g["gamma"][0]) == 3


def test_schedule_phat_out_of_range_and_bad_latency(sv):
    """R22: p_hat outside [0, 1] is used as 0 and flagged PHAT_BAD, in both schedule modes; the
    batch-greedy mode flags every sequence BAD_LATENCY when a reachable latency is not positive."""
    ph = np.array([[0.9, 1.5, 0.9], [0.5, -0.25, 0.5], [0.0, 1.0, 0.7], [np.nan, 0.5, 0.5]], dtype=np.float32)
    Lh = synth.latency_table(5)
    g = sv.sv_schedule(torch.as_tensor(ph, device="cuda"), torch.as_tensor(Lh, device="cuda"))
    r = oracle.schedule(ph.astype(np.float64), Lh)
    assert np.array_equal(g["gamma"].cpu().numpy(), r["gamma"])
    assert np.array_equal(g["status"].cpu().numpy(), r["status"])
    assert (g["status"].cpu().numpy() & oracle.ROW_PHAT_BAD).tolist() == [16, 16, 0, 16]
    Lg = synth.latency_table(4 * 4 + 1, base=4.0, knee=8, slope=0.5)
    g = sv.sv_schedule(torch.as_tensor(ph, device="cuda"), torch.as_tensor(Lg, device="cuda"),
                       mode=sv.SV_SCHED_BATCH_GREEDY)
    rg = oracle.batch_greedy(ph.astype(np.float64), Lg)
    assert np.array_equal(g["gamma"].cpu().numpy(), rg["gamma"])
    assert (g["status"].cpu().numpy() & oracle.ROW_PHAT_BAD).tolist() == [16, 16, 0, 16]
    Lg[6] = -1.0
    g = sv.sv_schedule(torch.as_tensor(ph, device="cuda"), torch.as_tensor(Lg, device="cuda"),
                       mode=sv.SV_SCHED_BATCH_GREEDY)
    rg = oracle.batch_greedy(ph.astype(np.float64), Lg)
    assert np.array_equal(g["gamma"].cpu().numpy(), rg["gamma"]) and rg["gamma"].tolist() == [0, 0, 0, 0]
    assert np.all(g["status"].cpu().numpy() == oracle.ROW_BAD_LATENCY)
