"""Pins of the fp64 oracle against what the paper, SPEC's hand-derived examples,
closed forms, invariants, library routines and brute force fix (-m "not gpu").

Each test names its source: P Lnnn = PAPER.md line, S Lnnn = SPEC.md line.
None of the expected values comes from the CUDA path.
"""
import itertools
import math

import numpy as np
import pytest
import scipy.stats

import oracle
from oracle import profile as oprof

# ----------------------------------------------------------------- Philox KAT
# Random123 known-answer vectors for philox4x32_10 (Salmon et al., SC'11,
# distributed as kat_vectors with Random123): (ctr, key) -> output.
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_kat(ctr, key, want):
    assert tuple(int(w) for w in oracle.philox4x32_10(ctr, key)) == want


def test_u24_and_counter_layout():
    # U24(w) = (w >> 8) / 2^24 (DESIGN R12): exact dyadic rational.
    assert oracle.u24(0x6627E8D5) == 0x6627E8 / 2**24
    assert oracle.u24(0xFFFFFFFF) == 1 - 2**-24
    # position 0 of sequence 0 with seed 0, offset 0 uses ctr = key = 0 -> KAT vector 1
    u, us = oracle.uniforms(0, 0, 0, 0)
    assert u == 0x6627E8 / 2**24 and us == 0xE169C5 / 2**24
    # counter words: (i, g, lo(offset), hi(offset)); key: (lo(seed), hi(seed))
    u2, _ = oracle.uniforms(0xA4093822 | (0x299F31D0 << 32), 0x13198A2E | (0x03707344 << 32),
                            0x85A308D3, 0x243F6A88)
    assert u2 == (0xD16CFE09 >> 8) / 2**24


# -------------------------------------------------------------------- softmax
def test_softmax_uniform_and_two_token():
    p, st = oracle.softmax(np.full(7, 3.25))
    assert st == 0 and np.allclose(p, 1 / 7, rtol=0, atol=1e-16)
    for d, tau in [(0.0, 1.0), (1.5, 1.0), (-4.0, 0.7), (30.0, 2.0)]:
        p, _ = oracle.softmax([d, 0.0], tau)
        want = 1.0 / (1.0 + math.exp(-d / tau))  # logistic closed form
        assert abs(p[0] - want) < 1e-15 and abs(p.sum() - 1) < 1e-15


def test_softmax_masks_and_errors():
    p, st = oracle.softmax([0.0, -np.inf, 1.0])
    assert st == 0 and p[1] == 0.0 and abs(p.sum() - 1) < 1e-15
    assert oracle.softmax([-np.inf, -np.inf])[1] == oracle.ROW_ALL_NEG_INF
    assert oracle.softmax([0.0, np.nan])[1] == oracle.ROW_NAN
    assert oracle.softmax([0.0, np.inf])[1] == oracle.ROW_NAN


def test_softmax_matches_scipy():
    rng = np.random.default_rng(1)
    x = rng.normal(0, 3, 1000)
    p, _ = oracle.softmax(x, 0.7)
    assert np.allclose(p, scipy.special.softmax(x / 0.7), rtol=1e-13, atol=0)


# ------------------------------------------------------------ indicators S, A
def _score1(pd, pc, t, **kw):
    with np.errstate(divide="ignore"):
        D = np.log(np.asarray(pd, dtype=np.float64))[None, None]
        C = np.log(np.asarray(pc, dtype=np.float64))[None, None]
    r = oracle.score(D, C, [[t]], **kw)
    return {k: v[0, 0] for k, v in r.items()}


def test_spec_indicator_example():
    # S L220: P_d=[.5,.3,.2], P_c=[.2,.5,.3], t_d=0 -> s = .2+.3+.2 = .7, a = min(1,.2/.5) = .4
    r = _score1([0.5, 0.3, 0.2], [0.2, 0.5, 0.3], 0)
    assert abs(r["S"] - 0.7) < 1e-12 and abs(r["A"] - 0.4) < 1e-12
    assert abs(r["TV"] - 0.3) < 1e-12


def test_identical_and_disjoint():
    # S L219: P_d = P_c -> (1, 1); north_star: identical -> zero divergence
    rng = np.random.default_rng(2)
    x = rng.normal(0, 2, (1, 1, 500))
    r = oracle.score(x, x.copy(), [[7]])
    assert abs(r["S"][0, 0] - 1) < 1e-12 and r["A"][0, 0] == 1.0 and r["KL"][0, 0] == 0.0
    # S L221: disjoint supports -> s = 0, a = 0 (and KL = +inf)
    D = np.array([[[0.0, 0.0, -np.inf, -np.inf]]])
    C = np.array([[[-np.inf, -np.inf, 0.0, 1.0]]])
    r = oracle.score(D, C, [[1]])
    assert r["S"][0, 0] == 0.0 and r["A"][0, 0] == 0.0 and r["KL"][0, 0] == math.inf


def test_spec_divergence_example():
    # S L230: P=[.5,.5], Q=[.9,.1] -> 1 - (.5 + .1) = .4
    assert abs((1 - oracle.overlap([0.5, 0.5], [0.9, 0.1])) - 0.4) < 1e-15


def test_overlap_identities():
    rng = np.random.default_rng(3)
    for _ in range(50):
        V = int(rng.integers(2, 300))
        pd = rng.dirichlet(np.full(V, 0.3))
        pc = rng.dirichlet(np.full(V, 0.3))
        s = oracle.overlap(pd, pc)
        # S L233: 1 - sum min = 0.5 * L1
        assert abs((1 - s) - 0.5 * np.abs(pd - pc).sum()) < 1e-12
        # S L234: permutation invariance
        perm = rng.permutation(V)
        assert abs(oracle.overlap(pd[perm], pc[perm]) - s) < 1e-12
        # symmetric (S L225)
        assert abs(oracle.overlap(pc, pd) - s) < 1e-15


def test_a_is_one_when_companion_dominates():
    # S L235: A = 1 whenever P_c(t_d) >= P_d(t_d)
    r = _score1([0.1, 0.6, 0.3], [0.4, 0.3, 0.3], 0)
    assert r["A"] == 1.0
    r = _score1([0.1, 0.6, 0.3], [0.4, 0.3, 0.3], 1)
    assert abs(r["A"] - 0.5) < 1e-12


def test_kl_two_point_closed_form():
    """KL between two-point distributions (north_star KL, direction R6: expectation under the
    draft).  Bernoulli closed form: KL(Ber(1/2) || Ber(1/4)) = 1/2 ln(1/2 / 1/4) + 1/2 ln(1/2 /
    3/4) = 1/2 ln(4/3); the reverse direction KL(Ber(1/4) || Ber(1/2)) = 3/4 ln 3 - ln 2.  Both
    through oracle.score on logits (softmax included): draft [0, 0], companion [0, ln 3]."""
    D = np.array([[[0.0, 0.0]]])
    C = np.array([[[0.0, math.log(3.0)]]])
    r = oracle.score(D, C, [[0]])
    assert abs(r["KL"][0, 0] - 0.5 * math.log(4.0 / 3.0)) < 1e-15
    r = oracle.score(C, D, [[0]])  # swapped roles: the other direction
    assert abs(r["KL"][0, 0] - (0.75 * math.log(3.0) - math.log(2.0))) < 1e-15
    # p_c = 0 where p_d > 0 -> +inf
    r = oracle.score(D, np.array([[[0.0, -np.inf]]]), [[0]])
    assert np.isinf(r["KL"][0, 0]) and r["KL"][0, 0] > 0


def test_kl_against_scipy_gibbs_pinsker():
    rng = np.random.default_rng(4)
    for _ in range(50):
        V = int(rng.integers(2, 200))
        pd = rng.dirichlet(np.full(V, 0.5))
        pc = rng.dirichlet(np.full(V, 0.5))
        k = oracle.kl(pd, pc)
        assert abs(k - scipy.stats.entropy(pd, pc)) < 1e-10 * max(1, k)  # library routine
        tv = 1 - oracle.overlap(pd, pc)
        assert k >= 0 and k >= 2 * tv * tv - 1e-12  # Gibbs, Pinsker


# ------------------------------------------------------------------- lookup
def test_lookup_spec_examples():
    se = [0.0, 0.3, 0.6, 1.0]
    ae = [0.0, 0.5, 1.0]
    cells = np.arange(6, dtype=float).reshape(3, 2) / 10
    # S L299: inside a populated cell -> that cell's mean
    assert oracle.lookup(se, ae, cells, 0.45, 0.7) == cells[1, 1]
    # S L300: above the max edge -> clamped to the last bin; below min -> first bin
    assert oracle.lookup(se, ae, cells, 1.7, 0.2) == cells[2, 0]
    assert oracle.lookup(se, ae, cells, -0.5, 9.0) == cells[0, 1]
    # right-closed bins (e_j, e_j+1] (DESIGN R9): a value on an interior edge belongs below it
    assert oracle.bin_index(se, 0.3) == 0 and oracle.bin_index(se, 0.30000001) == 1
    assert oracle.bin_index(se, 0.0) == 0 and oracle.bin_index(se, 1.0) == 2
    # S L324: piecewise constant
    assert oracle.lookup(se, ae, cells, 0.31, 0.51) == oracle.lookup(se, ae, cells, 0.59, 0.99)


def test_adaptive_edges_and_profile_fallbacks():
    # S L281: samples 1..100, 10 bins -> edges at every 10th order statistic
    e = oprof.adaptive_edges(np.arange(1, 101), 10)
    assert list(e) == [1] + list(range(10, 100, 10)) + [100]
    # each right-closed bin then holds exactly 10 samples
    counts = np.bincount([oprof.bin_of(e, v) for v in range(1, 101)])
    assert list(counts) == [10] * 10
    # S L282-283: constant samples / one bin -> single bin
    assert len(oprof.adaptive_edges([0.5] * 20, 10)) - 1 == 1
    assert len(oprof.adaptive_edges(np.arange(5.0), 1)) - 1 == 1
    # S L290: single record -> 1x1 profile with mean p
    p = oprof.build_profile([0.3], [0.4], [0.77], 5, 5)
    assert np.array(p["cells"]).shape == (1, 1) and p["cells"][0][0] == 0.77
    # S L291: two s-clusters, 2 s-bins -> each cell mean = its cluster mean
    s = [0.1, 0.12, 0.11, 0.9, 0.91, 0.92]
    a = [0.5] * 6
    x = [0.2, 0.3, 0.4, 0.8, 0.9, 1.0]
    p = oprof.build_profile(s, a, x, 2, 1)
    assert np.allclose(np.array(p["cells"])[:, 0], [0.3, 0.9])
    # S L301: empty cell -> s-row marginal mean (built by hand: 2x2 with one empty cell)
    s = [0.1, 0.2, 0.3, 0.7, 0.8, 0.9]
    a = [0.7, 0.8, 0.9, 0.1, 0.2, 0.3]
    x = [0.2, 0.4, 0.6, 0.5, 0.6, 0.7]
    p = oprof.build_profile(s, a, x, 2, 2)
    c = np.array(p["cells"])
    assert p["counts"] == [[0, 3], [3, 0]]
    assert abs(c[0, 0] - 0.4) < 1e-15 and abs(c[1, 1] - 0.6) < 1e-15


def test_info_gain_structure():
    # S L308-310, S L322-323: conditioning never increases plug-in entropy; X constant -> 0
    rng = np.random.default_rng(5)
    x = rng.random(4000)
    sb = rng.integers(0, 5, 4000)
    ab = rng.integers(0, 4, 4000)
    r = oprof.info_gain(x, sb, ab)
    assert r["h_x_sa"] <= min(r["h_x_s"], r["h_x_a"]) + 1e-12 <= r["h_x"] + 2e-12
    assert r["i_x_sa"] >= 0
    assert oprof.info_gain(np.full(10, 0.5), sb[:10], ab[:10])["h_x"] == 0
    # X a deterministic function of the (S,A) cell -> H(X|S,A) = 0
    sb2 = np.array([0, 0, 1, 1] * 10)
    ab2 = np.array([0, 1, 0, 1] * 10)
    x2 = (sb2 * 2 + ab2) / 4 + 0.05
    r2 = oprof.info_gain(x2, sb2, ab2)
    assert r2["h_x_sa"] == 0 and abs(r2["i_x_sa"] - 2.0) < 1e-12


# ------------------------------------------------------------ P_gamma(N), E
def test_p_gamma_n_spec_example():
    # S L372: gamma=2, p=[.5,.5] -> P(N=0)=.5, P(N=1)=.25, P(N=2)=.25
    assert [oracle.p_gamma_n([0.5, 0.5], 2, n) for n in range(3)] == [0.5, 0.25, 0.25]
    # S L373: all p=1 -> P(N=gamma) = 1
    assert [oracle.p_gamma_n([1.0] * 4, 4, n) for n in range(5)] == [0, 0, 0, 0, 1]
    assert math.isnan(oracle.p_gamma_n([0.5], 1, 2))  # S L370: n > gamma is an error


def test_expected_accepted_examples():
    assert oracle.expected_def([0.5, 0.5], 2) == 0.75  # S L381
    assert oracle.expected_def([1.0] * 5, 5) == 5.0  # S L382
    assert oracle.expected_def([0.3, 0.9], 0) == 0.0


def _brute_force_E(chain, gamma):
    """Enumerate all 2^gamma accept/reject patterns; N = number of leading accepts."""
    e = 0.0
    for pattern in itertools.product([0, 1], repeat=gamma):
        pr = 1.0
        for i, acc in enumerate(pattern):
            pr *= chain[i] if acc else 1 - chain[i]
        n = 0
        while n < gamma and pattern[n]:
            n += 1
        e += n * pr
    return e


def test_expected_bruteforce_and_total_probability():
    # S L383, L520: E matches 2^gamma enumeration within 1e-12; sum_n P = 1 (S L374)
    rng = np.random.default_rng(6)
    for _ in range(300):
        k = int(rng.integers(1, 11))
        chain = rng.random(k)
        pref = oracle.expected_prefix(chain)
        for g in range(k + 1):
            bf = _brute_force_E(chain, g)
            assert abs(oracle.expected_def(chain, g) - bf) < 1e-12
            assert abs(pref[g] - bf) < 1e-12
            assert abs(sum(oracle.p_gamma_n(chain, g, n) for n in range(g + 1)) - 1) < 1e-12


def test_leviathan_closed_form():
    # constant alpha: E + 1 = (1 - alpha^(gamma+1)) / (1 - alpha) (Leviathan et al., cited P L29)
    for alpha in (0.1, 0.5, 0.8, 0.95):
        pref = oracle.expected_prefix([alpha] * 12)
        for g in range(13):
            assert abs(pref[g] + 1 - (1 - alpha ** (g + 1)) / (1 - alpha)) < 1e-12


# ------------------------------------------------------------------ schedule
def _lat(base, knee, slope, n_max):
    return np.array([base + slope * max(0, n - knee) for n in range(n_max + 1)], dtype=np.float64)


def test_goodput_spec_examples():
    L = _lat(10, 0, 1, 8)
    # S L390: gamma = 0 -> 1 / latency(1)
    assert oracle.goodputs([0.9], L)[0] == 1 / L[1]
    # S L392 hand enumeration: p=[.9,.9,.2,.2,.2], base 10, knee 0, slope 1
    g = oracle.goodputs([0.9, 0.9, 0.2, 0.2, 0.2], L)
    by_hand = [1 / 11, 1.9 / 12, 2.71 / 13, 2.872 / 14, 2.9044 / 15, 2.91088 / 16]
    assert np.allclose(g, by_hand, rtol=0, atol=1e-12)
    r = oracle.schedule(np.array([[0.9, 0.9, 0.2, 0.2, 0.2]]), L)
    assert r["gamma"][0] == 2 and abs(r["exp_accept"][0] - 1.71) < 1e-12
    # S L391: constant latency, p = .9 -> strictly increasing -> gamma* = k (S L399)
    assert oracle.schedule(np.full((1, 6), 0.9), np.full(9, 3.0))["gamma"][0] == 6
    # S L400: strictly decreasing goodput -> gamma* = 0
    assert oracle.schedule(np.full((1, 6), 0.01), _lat(1, 0, 1, 8))["gamma"][0] == 0


def test_schedule_ties_and_exhaustive():
    # exact tie g0 == g1 -> smallest gamma (S L396): p1 = 0 with flat latency
    L = _lat(4, 2, 1, 8)
    assert oracle.schedule(np.array([[0.0, 0.9]]), L)["gamma"][0] == 0
    # exhaustive argmax over gamma with E from brute force (S L383, L520)
    rng = np.random.default_rng(7)
    for _ in range(200):
        k = int(rng.integers(1, 9))
        chain = rng.random(k)
        Lr = np.cumsum(rng.random(k + 3) + 0.05)
        g_bf = [(_brute_force_E(chain, g) + 1) / Lr[g + 1] for g in range(k + 1)]
        r = oracle.schedule(chain[None], Lr)
        assert g_bf[r["gamma"][0]] >= max(g_bf) - 1e-12


def test_first_decline_equals_argmax_under_convex_latency():
    # P L239 claim, S L401 / L522: 10^4 random chains, convex piecewise-linear L
    rng = np.random.default_rng(8)
    for _ in range(10_000):
        k = int(rng.integers(1, 17))
        chain = rng.random(k) ** rng.uniform(0.2, 3)
        L = _lat(rng.uniform(0.5, 10), int(rng.integers(0, 6)), rng.uniform(0, 3), k + 2)
        assert oracle.first_decline(chain, L) == oracle.schedule(chain[None], L)["gamma"][0]


def test_goodput_literal_reading_plus_one_0():
    """R2's literal reading of P L211 ("expected number of accepted tokens divided by
    verification latency"): g_j = E_j / L[j].  Hand enumeration of the S L392 chain
    p=[.9,.9,.2,.2,.2] with L[n] = 10 + n: E = 0, .9, 1.71, 1.872, 1.9044, 1.91088, so
    g = 0/10, .9/11, 1.71/12, 1.872/13, 1.9044/14, 1.91088/15 and the maximum moves from
    gamma = 2 (plus_one = 1, S L392) to gamma = 3."""
    L = _lat(10, 0, 1, 8)
    chain = [0.9, 0.9, 0.2, 0.2, 0.2]
    g = oracle.goodputs(chain, L, plus_one=0)
    by_hand = [0 / 10, 0.9 / 11, 1.71 / 12, 1.872 / 13, 1.9044 / 14, 1.91088 / 15]
    assert np.allclose(g, by_hand, rtol=0, atol=1e-12)
    r = oracle.schedule(np.array([chain]), L, plus_one=0)
    assert r["gamma"][0] == 3 and abs(r["exp_accept"][0] - 1.872) < 1e-12
    assert abs(r["goodput"][0] - 1.872 / 13) < 1e-12
    # gamma = 0 scores 0 under the literal reading: an all-zero chain ties everywhere -> 0 (S L396)
    assert oracle.schedule(np.zeros((1, 4)), L, plus_one=0)["gamma"][0] == 0
    # constant acceptance alpha, flat latency: E_j = alpha (1 - alpha^j) / (1 - alpha) (Leviathan's
    # closed form minus the bonus token) is increasing, so gamma* = k
    r = oracle.schedule(np.full((1, 7), 0.5), np.full(9, 2.0), plus_one=0)
    assert r["gamma"][0] == 7 and abs(r["exp_accept"][0] - 0.5 * (1 - 0.5 ** 7) / 0.5) < 1e-15
    # exhaustive argmax with brute-force E (2^gamma enumeration, S L383) under the literal reading
    rng = np.random.default_rng(17)
    for _ in range(200):
        k = int(rng.integers(1, 9))
        chain = rng.random(k)
        Lr = np.cumsum(rng.random(k + 3) + 0.05)
        g_bf = [_brute_force_E(chain, j) / Lr[j] for j in range(k + 1)]
        gam = oracle.schedule(chain[None], Lr, plus_one=0)["gamma"][0]
        assert g_bf[gam] >= max(g_bf) - 1e-12


def test_schedule_bad_inputs():
    r = oracle.schedule(np.array([[np.nan, 0.5]]), _lat(4, 2, 1, 4))
    assert r["status"][0] & oracle.ROW_PHAT_BAD
    # R22: p_hat is an acceptance probability (P L176); outside [0, 1] it is used as 0 and flagged
    for bad in (1.5, -0.25, np.inf):
        r = oracle.schedule(np.array([[0.9, bad, 0.9]]), np.full(6, 2.0))
        assert r["status"][0] & oracle.ROW_PHAT_BAD
        assert r["gamma"][0] == 1 and r["exp_accept"][0] == 0.9  # the chain stops at the bad entry
    r = oracle.schedule(np.array([[0.0, 1.0]]), np.full(4, 2.0))
    assert r["status"][0] == 0  # the end points are probabilities
    r = oracle.schedule(np.array([[0.5, 0.5]]), np.array([0.0, 1.0, -1.0, 1.0]))
    assert r["status"][0] & oracle.ROW_BAD_LATENCY and r["gamma"][0] == 0


# ------------------------------------------------------------- batch greedy
def test_batch_greedy_spec_trace():
    # S L410 (hand trace): [.9,.9] & [.8,.8], base 4, knee 2, slope 1 -> adds (q0,.9), (q0,.81),
    # (q1,.8), rejects (q1,.64): gamma = (2, 1), goodput = (2 + .9 + .81 + .8) / 7
    r = oracle.batch_greedy(np.array([[0.9, 0.9], [0.8, 0.8]]), _lat(4, 2, 1, 10))
    assert list(r["gamma"]) == [2, 1]
    assert abs(r["goodput"] - 4.51 / 7) < 1e-12


def test_batch_greedy_bad_inputs():
    # a non-positive / non-finite reachable latency: gamma = 0 everywhere, goodput NaN
    L = _lat(4, 2, 1, 10)
    L[5] = 0.0
    r = oracle.batch_greedy(np.array([[0.9, 0.9], [0.8, 0.8]]), L)
    assert list(r["gamma"]) == [0, 0] and np.isnan(r["goodput"])
    # R22: p_hat outside [0, 1] counts as 0 -> that query never gains a token
    r = oracle.batch_greedy(np.array([[1.5, 0.9], [0.8, 0.8]]), _lat(4, 2, 1, 10))
    assert r["gamma"][0] == 0


def test_batch_greedy_consistency_properties():
    rng = np.random.default_rng(9)
    for _ in range(200):
        k = int(rng.integers(1, 9))
        chain = rng.random(k)
        L = _lat(rng.uniform(1, 10), int(rng.integers(0, 4)), rng.uniform(0.1, 2), k + 3)
        # S L408: a single query gives the same gamma as optimal_gamma when goodput is
        # unimodal (first-decline == argmax under convex L; ties resolved identically)
        assert oracle.batch_greedy(chain[None], L)["gamma"][0] == oracle.first_decline(chain, L)
    # S L409: dominant chain first; constant latency region wide enough
    r = oracle.batch_greedy(np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 0.0]]), np.full(20, 5.0))
    assert list(r["gamma"]) == [3, 0]


# ------------------------------------------------------------------- verify
def _verify_pair(pd, pt, n, seed=11, rng=None, gamma=1, offset=0):
    """n independent single-position verifies of a fixed (P_d, P_t) pair with a fresh
    draft token t ~ P_d per trial (S L156, L521)."""
    rng = rng or np.random.default_rng(seed)
    V = len(pd)
    with np.errstate(divide="ignore"):
        ld, lt = np.log(pd), np.log(pt)
    D = np.ascontiguousarray(np.broadcast_to(ld, (n, 1, V)))
    T = np.ascontiguousarray(np.broadcast_to(lt, (n, 2, V)))
    tok = rng.choice(V, size=(n, 1), p=pd)
    r = oracle.verify(D, T, tok, np.full(n, gamma), seed=seed, offset=offset)
    return r, tok


def test_ratio_ge_one_always_accepts():
    # S L154: P_t(t_i) >= P_d(t_i) for all i -> N = gamma
    rng = np.random.default_rng(10)
    B, k, V = 64, 5, 50
    D = rng.normal(0, 2, (B, k, V))
    T = np.concatenate([D, rng.normal(0, 2, (B, 1, V))], axis=1)
    tok = rng.integers(0, V, (B, k))
    gam = rng.integers(0, k + 1, B)
    r = oracle.verify(D, T, tok, gam, seed=3)
    assert np.array_equal(r["n_accept"], gam)
    assert np.all(r["accept_ratio"][np.arange(k)[None] < gam[:, None]] == 1.0)


def test_disjoint_rejects_and_residual_is_target():
    # disjoint supports -> p_t(t) = 0 -> N = 0; residual = P_t (S L163)
    D = np.array([[[0.0, 0.0, -np.inf, -np.inf]]])
    T = np.array([[[-np.inf, -np.inf, 5.0, -np.inf], [0.0, 0.0, 0.0, 0.0]]])
    r = oracle.verify(D, T, [[1]], [1])
    assert r["n_accept"][0] == 0 and r["out_tok"][0] == 2 and abs(r["resid_mass"][0] - 1) < 1e-15


def test_spec_residual_examples():
    # S L164: P_t=[.6,.4], P_d=[.2,.8] -> residual [1, 0]: every rejection emits token 0
    r, tok = _verify_pair(np.array([0.2, 0.8]), np.array([0.6, 0.4]), 20000)
    rej = r["n_accept"] == 0
    assert rej.any() and np.all(r["out_tok"][rej] == 0)
    assert np.allclose(r["resid_mass"][rej], 0.4, atol=1e-12)
    # S L163: P_t=[1,0], P_d=[0,1] -> always reject, always token 0
    r, _ = _verify_pair(np.array([0.0, 1.0]), np.array([1.0, 0.0]), 1000)
    assert np.all(r["n_accept"] == 0) and np.all(r["out_tok"] == 0)


def test_gamma_zero_is_target_sampling():
    # S L155: gamma = 0 -> N = 0 and the token ~ P_t
    pt = np.array([0.1, 0.2, 0.3, 0.4])
    r, _ = _verify_pair(np.array([0.25] * 4), pt, 200000, gamma=0)
    assert np.all(r["n_accept"] == 0)
    freq = np.bincount(r["out_tok"], minlength=4) / r["out_tok"].size
    assert np.abs(freq - pt).sum() / 2 < 0.005


def test_survey_golden_convention_vector():
    """SURVEY §8(c) golden convention vector (tests/golden/convention_vector.json; values from an
    independent scratch implementation of the conventions, printed to 6 decimals) through the
    whole oracle pipeline: score -> schedule -> verify, and the Philox words it draws."""
    import sv_helpers as H
    g, x, L = H.load_golden()
    e, st = g["expected"], g["setup"]
    prof = st["profile"]
    D, C, T = (x[n].astype(np.float64) for n in ("D", "C", "T"))
    rs = oracle.score(D, C, x["tok"], 1.0, 1.0, prof)
    tol = 6e-7
    for n in ("S", "A", "KL"):
        assert np.allclose(rs[n], e[n], rtol=0, atol=tol), (n, rs[n])
    assert np.array_equal(rs["p_hat"], np.array(e["p_hat"]))
    for b in range(3):
        assert np.allclose(oracle.goodputs(rs["p_hat"][b], L), e["goodputs"][b], rtol=0, atol=tol)
    rh = oracle.schedule(rs["p_hat"], L)
    assert list(rh["gamma"]) == e["gamma"]
    for b in range(3):
        for i, u in enumerate(e["u_w0"][b]):
            assert abs(oracle.uniforms(0, 0, b, i)[0] - u) < tol
    rv = oracle.verify(D, T, x["tok"], rh["gamma"], 1.0, 1.0, st["seed"], st["offset"], st["seq_base"])
    want_ratio = np.array([[np.nan if v is None else v for v in row] for row in e["accept_ratio"]])
    assert np.allclose(rv["accept_ratio"], want_ratio, rtol=0, atol=tol, equal_nan=True)
    assert list(rv["n_accept"]) == e["n_accept"] and list(rv["out_tok"]) == e["out_tok"]
    assert np.allclose(rv["resid_mass"], e["resid_mass"], rtol=0, atol=tol)
    for b in range(3):
        assert abs(oracle.uniforms(0, 0, b, int(rv["n_accept"][b]))[1] - e["u_s"][b]) < tol


def test_verify_forced_n_and_crossing_neighbours():
    """The tie-reporting outputs of oracle.verify: n_force = the oracle's own N reproduces the run;
    the crossing neighbours are the positive-residual entries around the token (S L82-90, R11)."""
    rng = np.random.default_rng(23)
    B, k, V = 6, 4, 50
    D = rng.normal(0, 1, (B, k, V))
    T = rng.normal(0, 1.5, (B, k + 1, V))
    T[:, :k] += D
    tok = rng.integers(0, V, (B, k))
    gam = np.full(B, k)
    r0 = oracle.verify(D, T, tok, gam, seed=3, offset=9)
    r1 = oracle.verify(D, T, tok, gam, seed=3, offset=9, n_force=r0["n_accept"])
    for n in ("n_accept", "out_tok", "resid_mass"):
        assert np.array_equal(r0[n], r1[n])
    for b in range(B):
        N, t = int(r0["n_accept"][b]), int(r0["out_tok"][b])
        pt, _ = oracle.softmax(T[b, N])
        r = np.maximum(0.0, pt - oracle.softmax(D[b, N])[0]) if N < k else pt
        pos = np.nonzero(r > 0)[0]
        j = int(np.searchsorted(pos, t))
        assert pos[j] == t
        assert r0["tok_prev"][b] == (pos[j - 1] if j > 0 else -1)
        assert r0["tok_next"][b] == (pos[j + 1] if j + 1 < pos.size else -1)
        # margins: distances of u_s Z to the cumulative sums at the token and just before it
        _, us = oracle.uniforms(3, 9, b, N)
        cum = np.cumsum(r)
        assert abs(r0["sample_margin_hi"][b] - abs(cum[t] - us * cum[-1])) < 1e-12
        # forcing N = 0 samples the residual of row 0 (gamma = k > 0)
        rf = oracle.verify(D[b:b + 1], T[b:b + 1], tok[b:b + 1], gam[b:b + 1], seed=3, offset=9, seq_base=b,
                           n_force=[0])
        assert rf["n_accept"][0] == 0
        pt0, _ = oracle.softmax(T[b, 0])
        r_0 = np.maximum(0.0, pt0 - oracle.softmax(D[b, 0])[0])
        assert abs(rf["resid_mass"][0] - r_0.sum()) < 1e-12
        assert np.isfinite(r0["accept_margins"][b, : max(1, min(N + 1, k))]).all()


def test_hand_derived_convention_vector():
    # Closed-form check of the counter layout + accept rule + residual inverse CDF:
    # D row = [2,1,0,-1], T row = [1,2,0,-1], token 0, seed = offset = 0, b = i = 0.
    # ratio = e^1/e^2 = e^-1 < u = U24(0x6627e8d5) -> reject at N = 0;
    # both rows share the normaliser, so the residual is nonzero only at v = 1 with
    # Z = (e^2 - e^1) / (e^2 + e^1 + 1 + e^-1); u_s = U24(0xe169c58d) -> token 1.
    D = np.array([[[2.0, 1.0, 0.0, -1.0]]])
    T = np.array([[[1.0, 2.0, 0.0, -1.0], [0.0, 0.0, 0.0, 0.0]]])
    r = oracle.verify(D, T, [[0]], [1])
    e = math.e
    assert r["n_accept"][0] == 0 and r["out_tok"][0] == 1
    assert abs(r["accept_ratio"][0, 0] - 1 / e) < 1e-15
    assert abs(r["resid_mass"][0] - (e * e - e) / (e * e + e + 1 + 1 / e)) < 1e-15


@pytest.mark.parametrize("pair", range(20))
def test_losslessness_monte_carlo(pair):
    # S L156, L177, L521: emitted token ~ P_t, TV < 0.005 over 10^6 trials on a 5-token vocab;
    # and P(accept) = sum_v min(P_d, P_t) (north_star "expected acceptance equals sum min").
    rng = np.random.default_rng(1000 + pair)
    V = 5
    pd = rng.dirichlet(np.ones(V))
    pt = rng.dirichlet(np.ones(V))
    n = 1_000_000
    r, tok = _verify_pair(pd, pt, n, seed=pair, rng=rng)
    acc = r["n_accept"] == 1
    # emitted first token: the draft token if accepted, else the residual sample
    emitted = np.where(acc, tok[:, 0], r["out_tok"])
    freq = np.bincount(emitted, minlength=V) / n
    assert np.abs(freq - pt).sum() / 2 < 0.005
    chi2 = ((np.bincount(emitted, minlength=V) - n * pt) ** 2 / (n * pt)).sum()
    assert scipy.stats.chi2.sf(chi2, V - 1) > 1e-4
    alpha = np.minimum(pd, pt).sum()
    assert abs(acc.mean() - alpha) < 5 * math.sqrt(alpha * (1 - alpha) / n) + 1e-9


def test_verify_bad_inputs():
    D = np.zeros((2, 2, 3))
    T = np.zeros((2, 3, 3))
    T[1, 0, 1] = np.nan
    r = oracle.verify(D, T, [[0, 1], [0, 1]], [2, 2])
    assert r["status"][0] == 0 and r["status"][1] & oracle.ROW_NAN and r["out_tok"][1] == -1
    r = oracle.verify(D, T[:, :, :], [[0, 5], [0, 0]], [2, 3])
    assert r["status"][0] & oracle.ROW_BAD_TOKEN and r["status"][1] & oracle.ROW_BAD_GAMMA


# ----------------------------------------------------------------- NEXT-2: sampling filters
def test_filter_spec_examples():
    """S L79-81: [.7,.2,.1] with top_k = 1 -> [1,0,0]; [.5,.3,.2] with top_p = .8 keeps the
    first two -> [.625,.375,0].  The literal top_p = 0.8 sits exactly on the cumulative 0.5+0.3
    (a rounding tie in fp64), so the pin uses 0.79 (keeps two) and 0.81 (keeps three)."""
    from oracle.filtered import filter_dist
    p, keep = filter_dist(np.log([0.7, 0.2, 0.1]), top_k=1)
    assert np.array_equal(p, [1.0, 0.0, 0.0]) and list(keep) == [0]
    p, _ = filter_dist(np.log([0.5, 0.3, 0.2]), top_p=0.79)
    assert np.allclose(p, [0.625, 0.375, 0.0], rtol=0, atol=1e-15)
    p, _ = filter_dist(np.log([0.5, 0.3, 0.2]), top_p=0.81)
    assert np.allclose(p, [0.5, 0.3, 0.2], rtol=0, atol=1e-15)


def test_filter_sample_zero_residual_falls_back_to_target():
    """R10 (S L152 asserts the zero residual unreachable; it is reachable through rounding only):
    a zero residual mass samples p_t of the same row and is flagged; otherwise the residual is
    max(0, p_t - p_d) (S L157-165) and the bonus samples p_t."""
    from oracle.filtered import sample_filtered
    pt = np.array([0.0, 0.25, 0.0, 0.75])
    # p_d = p_t -> r = 0 everywhere: the draw is inverse-CDF over p_t (cum .25, 1.0)
    assert sample_filtered(pt, pt.copy(), 0.2)[::3] == (1, True)
    tok, z, _, rz = sample_filtered(pt, pt.copy(), 0.5)
    assert (tok, z, rz) == (3, 1.0, True)
    # ordinary residual: p_d = one-hot at 1 -> r = [0, 0, 0, .75], Z = .75
    tok, z, _, rz = sample_filtered(pt, np.array([0.0, 1.0, 0.0, 0.0]), 0.99)
    assert (tok, z, rz) == (3, 0.75, False)
    # bonus (no draft): plain p_t
    assert sample_filtered(pt, None, 0.1)[0] == 1


def test_filter_identity_idempotence_support():
    """Identity config = plain softmax (S L78) and idempotent; every config shrinks the support
    (S L196-197: "idempotent for identity config and monotone-support-shrinking otherwise");
    top-k alone is idempotent; top_k ties go to the lower index (DESIGN R21)."""
    import oracle
    from oracle.filtered import filter_dist
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.normal(0, 3, 50)
        p, _ = filter_dist(x, 0.7)
        ref, _ = oracle.softmax(x, 0.7)
        assert np.allclose(p, ref, rtol=1e-13, atol=1e-16)
        for k, tp in ((20, 0.8), (0, 0.9), (5, 1.0), (1, 0.5)):
            q, keep = filter_dist(x, 0.7, k, tp)
            assert abs(q.sum() - 1.0) < 1e-12 and np.all(q >= 0)
            assert np.count_nonzero(q) <= (k if k else 50) and np.count_nonzero(q) == len(keep)
            xf = np.where(q > 0, np.log(np.where(q > 0, q, 1.0)), -np.inf)
            q2, _ = filter_dist(xf, 1.0, k, tp)
            assert np.all((q2 > 0) <= (q > 0)) and np.all((q > 0) <= (p > 0))  # support shrinks
            if tp == 1.0:
                assert np.allclose(q, q2, rtol=1e-12, atol=1e-15)  # top-k alone: idempotent
    # ties: equal logits -> the lower indices are kept
    q, keep = filter_dist(np.array([1.0, 3.0, 3.0, 3.0, 0.0]), 1.0, 2)
    assert list(keep) == [1, 2] and q[3] == 0.0


def test_filter_wide_nucleus_closed_form():
    """A nucleus of hundreds of tokens (the case the GPU holds in threshold form): geometric
    probabilities p_j ∝ r^j on a shuffled vocabulary; the cumulative of the sorted prefix is
    (1 - r^n) / (1 - r^V), so the nucleus size is the closed form ceil(log(1 - top_p (1 - r^V)) / log r)
    and the kept mass renormalises to p_j (1 - r) / (1 - r^n)."""
    from oracle.filtered import filter_dist
    rng = np.random.default_rng(17)
    for r, V, tp in ((0.995, 5000, 0.9), (0.98, 3000, 0.8), (0.9993, 20000, 0.95)):
        n_exact = math.log(1 - tp * (1 - r ** V)) / math.log(r)
        assert abs(n_exact - round(n_exact)) > 1e-6  # not a rounding tie
        n = math.ceil(n_exact)
        perm = rng.permutation(V)
        x = np.empty(V)
        x[perm] = np.arange(V) * math.log(r)  # rank j sits at vocabulary index perm[j]
        q, keep = filter_dist(x, 1.0, 0, tp)
        assert len(keep) == n > 32
        assert list(keep) == list(perm[:n])
        want = r ** np.arange(n) * (1 - r) / (1 - r ** n)
        assert np.allclose(q[perm[:n]], want, rtol=1e-10, atol=0)
        assert np.count_nonzero(q) == n


def test_filter_score_identities():
    """Filtered S / A / KL keep the unfiltered identities (S L233-235): identical rows -> S = 1,
    A = 1, KL = 0; S = 1 - TV; A = 1 whenever p'_c(t) >= p'_d(t)."""
    from oracle.filtered import filter_dist, score_filtered
    rng = np.random.default_rng(9)
    D = rng.normal(0, 2, (2, 3, 40))
    C = D + rng.normal(0, 0.7, D.shape)
    tok = np.zeros((2, 3), dtype=np.int32)
    for b in range(2):
        for i in range(3):
            tok[b, i] = int(np.argmax(filter_dist(D[b, i], 1.0, 8, 0.9)[0]))
    r = score_filtered(D, D, tok, 1.0, 1.0, 8, 0.9)
    assert np.allclose(r["S"], 1.0) and np.allclose(r["A"], 1.0) and np.allclose(r["KL"], 0.0)
    r = score_filtered(D, C, tok, 1.0, 1.0, 8, 0.9)
    for b in range(2):
        for i in range(3):
            pd, _ = filter_dist(D[b, i], 1.0, 8, 0.9)
            pc, _ = filter_dist(C[b, i], 1.0, 8, 0.9)
            assert abs(r["S"][b, i] - (1 - 0.5 * np.abs(pd - pc).sum())) < 1e-12
            if pc[tok[b, i]] >= pd[tok[b, i]]:
                assert r["A"][b, i] == 1.0


def test_filter_losslessness_monte_carlo():
    """Under filters the emitted token still follows the FILTERED target (S L156, L183):
    t ~ p'_d per trial, verify_filtered with gamma = 1, chi-square over 20,000 trials."""
    from scipy import stats
    from oracle.filtered import filter_dist, verify_filtered
    import oracle
    rng = np.random.default_rng(13)
    V = 7
    xd = rng.normal(0, 1.5, V)
    xt = rng.normal(0, 1.5, V)
    pd, _ = filter_dist(xd, 1.0, 5, 0.95)
    pt, _ = filter_dist(xt, 1.0, 5, 0.95)
    D = xd.reshape(1, 1, V)
    T = np.stack([xt, xt]).reshape(1, 2, V)
    n = 20000
    counts = np.zeros(V)
    cdf = np.cumsum(pd)
    for j in range(n):
        u = oracle.uniforms(77, j, 0, 1)[0]  # an independent stream for the draft token
        t = int(np.searchsorted(cdf, u, side="right"))
        t = min(t, V - 1)
        while pd[t] == 0.0:
            t -= 1
        r = verify_filtered(D, T, np.array([[t]]), np.array([1]), 1.0, 1.0, 5, 0.95, 11, j)
        counts[r["out_tok"][0] if r["n_accept"][0] == 0 else t] += 1
    m = pt > 0
    assert counts[~m].sum() == 0
    chi = stats.chisquare(counts[m], pt[m] * n)
    assert chi.pvalue > 1e-4, chi
