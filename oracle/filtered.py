"""Sampling filters before S / A / accept (NEXT-2) -- TEST INFRASTRUCTURE ONLY.

Plain numpy fp64, row by row, following SPEC's filter operator and the paper's sampling
settings:
  filter_dist     S L73-81 (apply_sampling_filters): temperature -> top_k -> top_p ->
                  renormalise; P L731-743 Table 5 (Qwen: top_k 20, top_p 0.8, tau 0.7;
                  Llama: top_p 0.9, tau 0.6).  Readings (DESIGN R21): top_k keeps the k largest
                  logits, ties to the LOWER vocabulary index; top_p keeps the shortest prefix of
                  the top-k distribution (sorted by probability desc, index asc) whose sequential
                  fp64 cumulative mass is >= top_p (S L81: [.5,.3,.2], 0.8 -> first two).
  score_filtered  S, A, KL over the filtered draft / companion (S L238: "S is computed over the
                  SAME filtered distributions used for drafting"; P L159)
  verify_filtered the standard SD test and residual / bonus sample over the filtered draft /
                  target (S L183: filters on BOTH draft and target before the ratio), Philox
                  uniforms and the inverse-CDF convention of the unfiltered oracle (R11, R12).
Only ``tests/`` use this module.  Parity unpinned beyond the pins in
tests/test_oracle_pins.py::test_filter_* (SPEC examples, identity, idempotence, support shrink,
losslessness under filters).
"""
from __future__ import annotations

import math

import numpy as np

from . import uniforms


def filter_dist(x, tau: float = 1.0, top_k: int = 0, top_p: float = 1.0):
    """Filtered distribution of one logit row (S L73-81).  Returns (p [V] fp64, kept indices in
    kept order).  top_k = 0 means no top-k; top_p = 1 means no top-p."""
    x = np.asarray(x, dtype=np.float64)
    V = x.size
    y = x / tau
    order = np.lexsort((np.arange(V), -y))  # probability desc, index asc
    kk = V if top_k <= 0 else min(top_k, V)
    keep = order[:kk]
    p = np.exp(y[keep] - y[keep[0]])
    tot = 0.0
    for v in p:  # sequential sum (the GPU's order)
        tot += v
    p = p / tot
    if top_p < 1.0:
        c = 0.0
        n = kk
        for j in range(kk):
            c += p[j]
            if c >= top_p:
                n = j + 1
                break
        keep = keep[:n]
        s = 0.0
        for v in p[:n]:
            s += v
        p = p[:n] / s
    full = np.zeros(V)
    full[keep] = p
    return full, keep


def score_filtered(D, C, tok, tau_d, tau_c, top_k, top_p, profile=None):
    """S = sum_v min(p'_d, p'_c), A = min(1, p'_c(t)/p'_d(t)), KL(p'_d || p'_c) per (b, i)."""
    B, k, V = D.shape
    S = np.zeros((B, k))
    A = np.zeros((B, k))
    KL = np.zeros((B, k))
    pdt = np.zeros((B, k))
    st = np.zeros((B, k), dtype=np.int32)
    for b in range(B):
        for i in range(k):
            pd, _ = filter_dist(D[b, i], tau_d, top_k, top_p)
            pc, _ = filter_dist(C[b, i], tau_c, top_k, top_p)
            t = int(tok[b, i])
            S[b, i] = np.minimum(pd, pc).sum()
            pdt[b, i] = pd[t]
            if pd[t] == 0.0:
                st[b, i] = 8  # DRAFT_ZERO
                A[b, i] = np.nan
                KL[b, i] = np.nan
                continue
            A[b, i] = min(1.0, pc[t] / pd[t])
            m = pd > 0
            KL[b, i] = math.inf if np.any(pc[m] == 0) else float((pd[m] * np.log(pd[m] / pc[m])).sum())
    out = {"S": S, "A": A, "KL": KL, "pd_tok": pdt, "status": st}
    if profile is not None:
        from . import lookup
        out["p_hat"] = np.array([[lookup(profile["s_edges"], profile["a_edges"], profile["cells"], S[b, i], A[b, i])
                                  if st[b, i] == 0 else 0.0 for i in range(k)] for b in range(B)])
    return out


def verify_filtered(D, T, tok, gamma, tau_d, tau_t, top_k, top_p, seed, offset, seq_base=0):
    """Accept t_i iff u_i < p'_t(t_i)/p'_d(t_i); residual max(0, p'_t - p'_d) at the first
    rejection, else the bonus p'_t of row gamma; token = smallest j (vocab order) with
    cum_j > u_s Z, fallback = last positive entry (R11)."""
    B, k, V = D.shape
    n_acc = np.zeros(B, dtype=np.int32)
    out = np.full(B, -1, dtype=np.int32)
    Z = np.zeros(B)
    ratio = np.full((B, k), np.nan)
    margin = np.full(B, np.inf)
    resid_zero = np.zeros(B, dtype=bool)
    for b in range(B):
        g = int(gamma[b])
        N = g
        for i in range(g):
            pd, _ = filter_dist(D[b, i], tau_d, top_k, top_p)
            pt, _ = filter_dist(T[b, i], tau_t, top_k, top_p)
            t = int(tok[b, i])
            r = pt[t] / pd[t]
            ratio[b, i] = min(1.0, r)
            u, _ = uniforms(seed, offset, seq_base + b, i)
            margin[b] = min(margin[b], abs(u - r))
            if not u < r:
                N = i
                break
        n_acc[b] = N
        pt, _ = filter_dist(T[b, N], tau_t, top_k, top_p)
        pd = filter_dist(D[b, N], tau_d, top_k, top_p)[0] if N < g else None
        _, us = uniforms(seed, offset, seq_base + b, N)
        tokn, z, mg, rz = sample_filtered(pt, pd, us)
        Z[b] = z
        margin[b] = min(margin[b], mg)
        resid_zero[b] = rz
        out[b] = tokn
    return {"n_accept": n_acc, "out_tok": out, "resid_mass": Z, "accept_ratio": ratio, "margin": margin,
            "resid_zero": resid_zero}


def sample_filtered(pt, pd, us):
    """The correction / bonus draw over full-length filtered distributions (S L151, L157-165):
    r = max(0, p_t - p_d) (residual, pd given) or p_t (bonus, pd None); Z = sum r in vocabulary
    order; token = smallest j with cumulative > u_s Z (R11), fallback the last positive entry.
    A zero residual mass (reachable through rounding only) samples p_t instead and is flagged
    (R10, S L152).  Returns (token, Z, margin to the crossing, resid_zero)."""
    r = pt if pd is None else np.maximum(0.0, pt - pd)
    z = 0.0
    for v in r:
        z += v
    resid_zero = False
    if pd is not None and not z > 0.0:
        resid_zero = True
        r = pt
        z = 0.0
        for v in r:
            z += v
    th = us * z
    cum = 0.0
    for j in range(r.size):
        if r[j] <= 0.0:
            continue
        cum += r[j]
        if cum > th:
            return j, z, abs(cum - th), resid_zero
    return int(np.nonzero(r > 0)[0][-1]), z, np.inf, resid_zero
