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
                               offset=2, D=D)
    torch.cuda.synchronize()
    gv = {n: v.cpu().numpy() for n, v in gv.items()}
    rv = verify_filtered(Dd, Td, tok, gam, tau, tau, top_k, top_p, 5, 2)
    tie = rv["margin"] < 1e-6
    assert np.array_equal(gv["n_accept"][~tie], rv["n_accept"][~tie])
    assert np.array_equal(gv["out_tok"][~tie], rv["out_tok"][~tie])
    assert H.close(gv["resid_mass"][~tie], rv["resid_mass"][~tie]).all()
    assert np.array_equal((gv["status"][~tie] & 32) != 0, rv["resid_zero"][~tie])  # R10 flag
    r_ok = ~np.isnan(rv["accept_ratio"])
    assert np.array_equal(np.isnan(gv["accept_ratio"]), ~r_ok)
    assert H.close(gv["accept_ratio"][r_ok], rv["accept_ratio"][r_ok]).all()
    print("ties:", int(tie.sum()))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_filtered_nan_rows(sv, dtype):
    """R18 in the filtered path: a NaN of either sign or +inf in a draft or companion row flags
    SV_ROW_NAN (1) for that position; -inf is a legal mask; clean rows stay clean."""
    V = 1000
    rng = np.random.default_rng(7)
    x = rng.standard_normal((1, 4, V)).astype(np.float32)
    c = x + 0.1 * rng.standard_normal((1, 4, V)).astype(np.float32)
    bits = x.view(np.uint32)
    bits[0, 0, 17] = 0xFFC00000  # -NaN in draft row 0
    cb = c.view(np.uint32)
    cb[0, 1, 400] = 0x7F800000   # +inf in companion row 1
    bits[0, 2, 999] = 0x7FC00000  # +NaN in draft row 2
    x[0, 3, 5] = -np.inf          # a masked logit in row 3 (legal)
    tok = np.argmax(np.where(np.isfinite(x), x, -np.inf), axis=-1).astype(np.int32)
    if dtype == "bf16":
        D = torch.from_numpy(synth.f32_to_bf16_bits(x).astype(np.int16)).view(torch.bfloat16).cuda()
        C = torch.from_numpy(synth.f32_to_bf16_bits(c).astype(np.int16)).view(torch.bfloat16).cuda()
    else:
        D, C = torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda()
    g = sv.sv_score_filtered(D, C, torch.from_numpy(tok).cuda(), 20, 0.8, 0.7, 0.7,
                             sv.Profile.from_dict(synth.load_profile()))
    st = g["status"].cpu().numpy()[0]
    assert (st[0] & 1) and (st[1] & 1) and (st[2] & 1), st
    assert st[3] == 0, st


def test_filtered_bad_configs(sv):
    B, k, V = 2, 2, 64
    x = synth.make_inputs(B, k, V, "f32", seed=1)
    D, C, T, tok = H.to_torch(x)
    for top_k, top_p in ((33, 0.9), (0, 1.0), (20, 0.0)):
        with pytest.raises(sv.SvError):
            sv.sv_score_filtered(D, C, tok, top_k, top_p)


def _cut_margin(x, tau, top_p):
    """Distance of the oracle's sequential cumulative to top_p at the nucleus cut (the last two
    prefix sums): inside ~1e-6 the GPU's normaliser rounding may move the cut by one token."""
    _, keep = filter_dist(x, tau, 0, top_p)
    y = np.asarray(x, dtype=np.float64) / tau
    order = np.lexsort((np.arange(y.size), -y))
    p = np.exp(y[order] - y[order[0]])
    p = p / p.sum()
    c = np.cumsum(p)
    n = len(keep)
    return min(abs(c[n - 1] - top_p), abs(c[n - 2] - top_p) if n > 1 else 1.0)


@pytest.mark.parametrize("V,dtype,tau", [(32000, "f32", 0.6), (32000, "bf16", 0.6), (4096, "bf16", 1.0),
                                         (32000, "f32", 1.0), (152064, "bf16", 1.0),
                                         (1001, "f32", 2.0), (4099, "bf16", 1.5)])  # unaligned rows
def test_nucleus_only_llama_setting(sv, V, dtype, tau):
    """top_k = 0, top_p = 0.9 (P L739-740, Llama) over the FULL distribution, any nucleus size:
    <= 32 tokens as lists, larger nuclei in threshold form (mass-weighted radix select, full-row
    scoring) -- every row against the filtered oracle."""
    B, k = (6, 4) if V < 100000 else (2, 3)
    x = synth.make_inputs(B, k, V, dtype, seed=4321 + V)
    Dd, Cd, Td = H.oracle_inputs(x)
    rng = np.random.default_rng(V)
    tok = np.zeros((B, k), dtype=np.int32)
    big = np.zeros((B, k), dtype=bool)
    tie = np.zeros((B, k), dtype=bool)
    for b in range(B):
        for i in range(k):
            p, keep_d = filter_dist(Dd[b, i], tau, 0, 0.9)
            _, keep_c = filter_dist(Cd[b, i], tau, 0, 0.9)
            big[b, i] = len(keep_d) > 32 or len(keep_c) > 32
            tie[b, i] = min(_cut_margin(Dd[b, i], tau, 0.9), _cut_margin(Cd[b, i], tau, 0.9)) < 1e-6
            tok[b, i] = rng.choice(V, p=p / p.sum())
    D, C, T, _ = H.to_torch(x)
    tk = torch.from_numpy(tok).cuda()
    pd = synth.load_profile()
    gs = sv.sv_score_filtered(D, C, tk, 0, 0.9, tau, tau, sv.Profile.from_dict(pd))
    torch.cuda.synchronize()
    g = {n: gs[n].cpu().numpy() for n in ("S", "A", "KL", "status", "draft_ptok")}
    rs = score_filtered(Dd, Cd, tok, tau, tau, 0, 0.9)
    assert np.array_equal(g["status"], rs["status"])
    ok = (rs["status"] == 0) & ~tie
    for n in ("S", "A", "KL"):
        assert H.close(g[n][ok], rs[n][ok]).all(), (n, g[n][ok], rs[n][ok])
    assert H.close(g["draft_ptok"][ok], rs["pd_tok"][ok]).all()
    print("rows with a nucleus > 32:", int(big.sum()), "of", big.size, "cut ties:", int(tie.sum()))


@pytest.mark.parametrize("V,dtype,tau", [(4096, "bf16", 1.0), (32000, "f32", 1.0), (32000, "bf16", 0.8),
                                         (32000, "f32", 3.0),   # nuclei of thousands: radix fallback
                                         (1001, "f32", 2.0)])   # unaligned rows
def test_nucleus_wide_verify(sv, V, dtype, tau):
    """sd_verify_filtered, nucleus-only, with nuclei wider than 32 tokens on draft and target rows:
    accept tests in threshold form and the full-row residual / bonus sample against the oracle;
    without the draft logits the sequences that need a wide draft row are flagged 256."""
    B, k = (24 if tau >= 3.0 else 8), 4  # flat rows: more sequences, most land near a tie
    x = synth.make_inputs(B, k, V, dtype, seed=97 + V)
    Dd, Cd, Td = H.oracle_inputs(x)
    rng = np.random.default_rng(V + 1)
    tok = np.zeros((B, k), dtype=np.int32)
    wide_d = np.zeros((B, k), dtype=bool)
    wide_t = np.zeros((B, k + 1), dtype=bool)
    tie = np.zeros(B, dtype=bool)
    for b in range(B):
        for i in range(k):
            p, keep = filter_dist(Dd[b, i], tau, 0, 0.9)
            wide_d[b, i] = len(keep) > 32
            tie[b] |= _cut_margin(Dd[b, i], tau, 0.9) < 1e-6
            tok[b, i] = rng.choice(V, p=p / p.sum())
        for i in range(k + 1):
            wide_t[b, i] = len(filter_dist(Td[b, i], tau, 0, 0.9)[1]) > 32
            tie[b] |= _cut_margin(Td[b, i], tau, 0.9) < 1e-6
    assert wide_d.any() and wide_t.any()
    print("largest draft nucleus:", max(len(filter_dist(Dd[b, i], tau, 0, 0.9)[1]) for b in range(B) for i in range(k)))
    D, C, T, _ = H.to_torch(x)
    tk = torch.from_numpy(tok).cuda()
    gs = sv.sv_score_filtered(D, C, tk, 0, 0.9, tau, tau, sv.Profile.from_dict(synth.load_profile()))
    gam = rng.integers(0, k + 1, B).astype(np.int32)
    gam[0], gam[1] = k, 0
    gg = torch.from_numpy(gam).cuda()
    gv = sv.sd_verify_filtered(T, tk, gg, gs["fworkspace"], 0, 0.9, tau, seed=9, offset=1, D=D)
    torch.cuda.synchronize()
    gv = {n: v.cpu().numpy() for n, v in gv.items()}
    rv = verify_filtered(Dd, Td, tok, gam, tau, tau, 0, 0.9, 9, 1)
    tie |= rv["margin"] < 1e-6
    assert (gv["status"][~tie] == 0).all()
    assert np.array_equal(gv["n_accept"][~tie], rv["n_accept"][~tie])
    assert np.array_equal(gv["out_tok"][~tie], rv["out_tok"][~tie])
    assert H.close(gv["resid_mass"][~tie], rv["resid_mass"][~tie]).all()
    r_ok = ~np.isnan(rv["accept_ratio"]) & ~tie[:, None]
    assert H.close(gv["accept_ratio"][r_ok], rv["accept_ratio"][r_ok]).all()
    wide_seq = np.array([wide_t[b, rv["n_accept"][b]] or (rv["n_accept"][b] < gam[b] and wide_d[b, rv["n_accept"][b]])
                         for b in range(B)])
    print("sequences sampled in threshold form:", int(wide_seq.sum()), "of", B, "ties:", int(tie.sum()))
    # without the draft logits: a sequence whose draft row 0 is wide and gamma >= 1 cannot be tested
    nv = sv.sd_verify_filtered(T, tk, gg, gs["fworkspace"], 0, 0.9, tau, seed=9, offset=1)
    torch.cuda.synchronize()
    nst = nv["status"].cpu().numpy()
    need = (gam >= 1) & wide_d[:, 0]
    assert ((nst[need] & 256) != 0).all()
    no_wide = np.array([not wide_d[b, :gam[b]].any() for b in range(B)])
    assert ((nst[no_wide] & 256) == 0).all()


def test_nucleus_only_verify(sv):
    """sd_verify_filtered with top_k = 0 (nucleus), Llama temperature: every row's nucleus is
    small here, so the whole verification must match the filtered oracle."""
    B, k, V, tau = 6, 4, 32000, 0.6
    x = synth.make_inputs(B, k, V, "f32", seed=777)
    Dd, Cd, Td = H.oracle_inputs(x)
    rng = np.random.default_rng(3)
    tok = np.zeros((B, k), dtype=np.int32)
    for b in range(B):
        for i in range(k):
            p, _ = filter_dist(Dd[b, i], tau, 0, 0.9)
            tok[b, i] = rng.choice(V, p=p / p.sum())
    for b in range(B):
        for i in range(k + 1):
            assert len(filter_dist(Td[b, i], tau, 0, 0.9)[1]) <= 32
    D, C, T, _ = H.to_torch(x)
    tk = torch.from_numpy(tok).cuda()
    gs = sv.sv_score_filtered(D, C, tk, 0, 0.9, tau, tau, sv.Profile.from_dict(synth.load_profile()))
    gam = np.full(B, k, dtype=np.int32)
    gv = sv.sd_verify_filtered(T, tk, torch.from_numpy(gam).cuda(), gs["fworkspace"], 0, 0.9, tau, seed=9, offset=1, D=D)
    torch.cuda.synchronize()
    gv = {n: v.cpu().numpy() for n, v in gv.items()}
    rv = verify_filtered(Dd, Td, tok, gam, tau, tau, 0, 0.9, 9, 1)
    tie = rv["margin"] < 1e-6
    assert np.array_equal(gv["n_accept"][~tie], rv["n_accept"][~tie])
    assert np.array_equal(gv["out_tok"][~tie], rv["out_tok"][~tie])
    assert H.close(gv["resid_mass"][~tie], rv["resid_mass"][~tie]).all()
    assert np.array_equal((gv["status"][~tie] & 32) != 0, rv["resid_zero"][~tie])  # R10 flag


@pytest.mark.parametrize("r,V,tp", [(0.995, 5000, 0.9),      # 460 tokens: candidate sort
                                    (0.9995, 20000, 0.9),    # 4604 tokens: radix fallback
                                    (0.99, 3000, 0.99999)])  # top_p + margin > 1: radix fallback
def test_nucleus_wide_closed_form(sv, r, V, tp):
    """Geometric rows p_j ∝ r^j on a shuffled vocabulary (fp32 logits): nucleus size
    ceil(log(1 - top_p (1 - r^V)) / log r) > 32, so the GPU holds them in threshold form; with
    draft = companion, S = 1, A = 1, KL = 0 and p'_d(t) = r^j (1 - r) / (1 - r^n) for the token of
    rank j; a token outside the nucleus is DRAFT_ZERO."""
    import math
    n = math.ceil(math.log(1 - tp * (1 - r ** V)) / math.log(r))
    rng = np.random.default_rng(3)
    B, k = 2, 3
    perm = [rng.permutation(V) for _ in range(B * k)]
    x = np.empty((B, k, V), dtype=np.float32)
    for j in range(B * k):
        x[j // k, j % k, perm[j]] = (np.arange(V) * math.log(r)).astype(np.float32)
    ranks = np.array([[3, n - 5, 0], [n + 5, 17, n - 6]])  # clear of the cut (fp32 logits move it by ~1e-7)
    tok = np.array([[perm[b * k + i][ranks[b, i]] for i in range(k)] for b in range(B)], dtype=np.int32)
    D = torch.from_numpy(x).cuda()
    gs = sv.sv_score_filtered(D, D, torch.from_numpy(tok).cuda(), 0, tp, 1.0, 1.0)
    torch.cuda.synchronize()
    g = {n_: gs[n_].cpu().numpy() for n_ in ("S", "A", "KL", "draft_ptok", "status")}
    xs = x.astype(np.float64)
    for b in range(B):
        for i in range(k):
            if ranks[b, i] >= n:
                assert g["status"][b, i] == 8
                continue
            assert g["status"][b, i] == 0
            assert abs(g["S"][b, i] - 1.0) < 1e-6 and g["A"][b, i] == 1.0 and abs(g["KL"][b, i]) < 1e-6
            # the fp32-rounded logits make p_j slightly off the closed form: compare with it at 1e-5
            j = ranks[b, i]
            want = math.exp(xs[b, i, perm[b * k + i][j]]) * (1 - r) / (1 - r ** n)
            assert abs(g["draft_ptok"][b, i] - want) <= 1e-5 * want


def test_nucleus_wide_deterministic(sv):
    """The wide-nucleus path is bitwise reproducible (integer fixed-point histograms, sorted
    candidate bands, fixed-order sums): two runs of score + verify give identical outputs."""
    B, k, V, tau = 6, 4, 32000, 1.5
    x = synth.make_inputs(B, k, V, "bf16", seed=2024)
    D, C, T, tok = H.to_torch(x)
    gam = torch.full((B,), k, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(2):
        gs = sv.sv_score_filtered(D, C, tok, 0, 0.9, tau, tau)
        gv = sv.sd_verify_filtered(T, tok, gam, gs["fworkspace"], 0, 0.9, tau, seed=3, offset=7, D=D)
        torch.cuda.synchronize()
        outs.append({**{n: gs[n].cpu().numpy() for n in ("S", "A", "KL", "draft_ptok", "status")},
                     **{n: v.cpu().numpy() for n, v in gv.items()}})
    for n in outs[0]:
        assert np.array_equal(outs[0][n], outs[1][n], equal_nan=True) if outs[0][n].dtype.kind == "f" \
            else np.array_equal(outs[0][n], outs[1][n]), n
