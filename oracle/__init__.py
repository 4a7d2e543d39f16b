"""fp64 CPU oracle for the SV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2509_24328_b200`` never imports it, and the two share no code: the
arithmetic lives in ``sv_oracle.c`` (plain C, fp64, ``-ffp-contract=off``),
this module only marshals numpy arrays through ctypes.

Each wrapper names the passage it follows (``P Lnnn`` = PAPER.md line, ``S Lnnn``
= SPEC.md line, ``R n`` = reading n in DESIGN.md §3).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sv_oracle.c")
_LIB = os.path.join(_HERE, "libsv_oracle.so")

ROW_NAN = 1
ROW_ALL_NEG_INF = 2
ROW_BAD_TOKEN = 4
ROW_DRAFT_ZERO = 8
ROW_PHAT_BAD = 16
ROW_RESID_ZERO = 32
ROW_BAD_GAMMA = 64
ROW_BAD_LATENCY = 128


def build(force: bool = False) -> str:
    """Compile sv_oracle.c with gcc (fp64, no FMA contraction, OpenMP over rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-Wall",
             "-shared", "-fPIC", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, i32, i64, u64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        P = ctypes.c_void_p
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_u24.argtypes = [ctypes.c_uint32]
        _lib.oracle_u24.restype = d
        _lib.oracle_uniforms.argtypes = [u64, u64, i64, i32, P, P]
        _lib.oracle_softmax.argtypes = [P, i64, d, P]
        _lib.oracle_softmax.restype = ctypes.c_int
        _lib.oracle_overlap.argtypes = [P, P, i64]
        _lib.oracle_overlap.restype = d
        _lib.oracle_kl.argtypes = [P, P, i64]
        _lib.oracle_kl.restype = d
        _lib.oracle_bin_index.argtypes = [P, i32, d]
        _lib.oracle_bin_index.restype = ctypes.c_int
        _lib.oracle_lookup.argtypes = [P, i32, P, i32, P, d, d]
        _lib.oracle_lookup.restype = d
        _lib.oracle_score.argtypes = [P, P, P, i32, i32, i64, d, d, P, i32, P, i32, P,
                                      P, P, P, P, P, P, P, i32]
        _lib.oracle_p_gamma_n.argtypes = [P, i32, i32]
        _lib.oracle_p_gamma_n.restype = d
        _lib.oracle_expected_def.argtypes = [P, i32]
        _lib.oracle_expected_def.restype = d
        _lib.oracle_expected_prefix.argtypes = [P, i32, P]
        _lib.oracle_goodputs.argtypes = [P, i32, P, i32, P]
        _lib.oracle_schedule.argtypes = [P, i32, i32, P, i32, i32, P, P, P, P]
        _lib.oracle_first_decline.argtypes = [P, i32, P, i32]
        _lib.oracle_first_decline.restype = i32
        _lib.oracle_batch_greedy.argtypes = [P, i32, i32, P, i32, P, P]
        _lib.oracle_batch_greedy.restype = d
        _lib.oracle_verify.argtypes = [P, P, P, P, i32, i32, i64, d, d, u64, u64, i64,
                                       P, P, P, P, P, P, P, i32, P, P, P]
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------- RNG
def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 block (Salmon et al. SC'11; reading R12)."""
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def u24(w: int) -> float:
    return lib().oracle_u24(ctypes.c_uint32(w))


def uniforms(seed: int, offset: int, g: int, i: int) -> tuple[float, float]:
    """(u, u_s) of draft position i of global sequence g (reading R12)."""
    u = ctypes.c_double()
    us = ctypes.c_double()
    lib().oracle_uniforms(seed, offset, g, i, ctypes.byref(u), ctypes.byref(us))
    return u.value, us.value


# --------------------------------------------------------------------- a1 - a3
def softmax(x, tau: float = 1.0) -> tuple[np.ndarray, int]:
    """p = softmax(x / tau) in fp64 (P L159; tau P L739-740)."""
    x = _f64(x)
    p = np.empty_like(x)
    st = lib().oracle_softmax(_p(x), x.size, tau, _p(p))
    return p, st


def overlap(pd, pc) -> float:
    """S = sum_v min(P_d, P_c) (P L159)."""
    pd, pc = _f64(pd), _f64(pc)
    return lib().oracle_overlap(_p(pd), _p(pc), pd.size)


def kl(pd, pc) -> float:
    """KL(P_d || P_c) (north_star; reading R6)."""
    pd, pc = _f64(pd), _f64(pc)
    return lib().oracle_kl(_p(pd), _p(pc), pd.size)


def bin_index(edges, value: float) -> int:
    e = _f64(edges)
    return lib().oracle_bin_index(_p(e), e.size - 1, value)


def lookup(s_edges, a_edges, cells, s: float, a: float) -> float:
    """P(T_i | S, A) from the adaptive-binned profile (P L176; S L293-301; R9)."""
    se, ae, c = _f64(s_edges), _f64(a_edges), _f64(cells)
    return lib().oracle_lookup(_p(se), se.size - 1, _p(ae), ae.size - 1, _p(c), s, a)


def score(D, C, tok, tau_d=1.0, tau_c=1.0, profile=None, nthreads=None) -> dict:
    """Steps a1-a3 for [B,k,V] draft/companion logits (P L159, L164, L176)."""
    D, C = _f64(D), _f64(C)
    B, k, V = D.shape
    tok = _i32(tok).reshape(B, k)
    if profile is None:
        profile = {"s_edges": [0.0, 1.0], "a_edges": [0.0, 1.0], "cells": [[0.5]]}
    se, ae = _f64(profile["s_edges"]), _f64(profile["a_edges"])
    cells = _f64(profile["cells"]).reshape(-1)
    out = {n: np.empty((B, k)) for n in ("S", "A", "KL", "TV", "p_hat", "pd_tok")}
    st = np.empty((B, k), dtype=np.int32)
    lib().oracle_score(_p(D), _p(C), _p(tok), B, k, V, tau_d, tau_c,
                       _p(se), se.size - 1, _p(ae), ae.size - 1, _p(cells),
                       _p(out["S"]), _p(out["A"]), _p(out["KL"]), _p(out["TV"]),
                       _p(out["p_hat"]), _p(out["pd_tok"]), _p(st),
                       nthreads or default_threads())
    out["status"] = st
    return out


# -------------------------------------------------------------------------- a4
def p_gamma_n(chain, gamma: int, n: int) -> float:
    """P_gamma(N = n), literal piecewise formula (P L224-228)."""
    c = _f64(chain)
    return lib().oracle_p_gamma_n(_p(c), gamma, n)


def expected_def(chain, gamma: int) -> float:
    """E(N | gamma) = sum_i i * P_gamma(N = i) (P L231-234)."""
    c = _f64(chain)
    return lib().oracle_expected_def(_p(c), gamma)


def expected_prefix(chain) -> np.ndarray:
    """E_j for j = 0..k via the prefix-product identity (S L378)."""
    c = _f64(chain)
    e = np.empty(c.size + 1)
    lib().oracle_expected_prefix(_p(c), c.size, _p(e))
    return e


def goodputs(chain, L, plus_one: int = 1) -> np.ndarray:
    """g_j for j = 0..k (P L211, L236; R2)."""
    c, Lv = _f64(chain), _f64(L)
    g = np.empty(c.size + 1)
    lib().oracle_goodputs(_p(c), c.size, _p(Lv), plus_one, _p(g))
    return g


def schedule(p_hat, L, plus_one: int = 1) -> dict:
    """Per-row gamma = smallest argmax of goodput (P L236-239; S L396; R4)."""
    ph = _f64(p_hat)
    B, k = ph.shape
    Lv = _f64(L)
    gamma = np.empty(B, dtype=np.int32)
    E = np.empty(B)
    g = np.empty(B)
    st = np.empty(B, dtype=np.int32)
    lib().oracle_schedule(_p(ph), B, k, _p(Lv), Lv.size, plus_one, _p(gamma), _p(E), _p(g), _p(st))
    return {"gamma": gamma, "exp_accept": E, "goodput": g, "status": st}


def first_decline(chain, L, plus_one: int = 1) -> int:
    """The paper's incremental search (P L239)."""
    c, Lv = _f64(chain), _f64(L)
    return lib().oracle_first_decline(_p(c), c.size, _p(Lv), plus_one)


def batch_greedy(p_hat, L) -> dict:
    """NEXT-1 batch greedy (P L247-252; S L402-417; R16, R17)."""
    ph = _f64(p_hat)
    B, k = ph.shape
    Lv = _f64(L)
    gamma = np.empty(B, dtype=np.int32)
    E = np.empty(B)
    G = lib().oracle_batch_greedy(_p(ph), B, k, _p(Lv), Lv.size, _p(gamma), _p(E))
    return {"gamma": gamma, "exp_accept": E, "goodput": G}


# --------------------------------------------------------------------- a5 + a6
def verify(D, T, tok, gamma, tau_d=1.0, tau_t=1.0, seed=0, offset=0, seq_base=0, nthreads=None,
           n_force=None) -> dict:
    """Standard SD verification + residual / bonus inverse-CDF sample
    (P L29; S L148-165, L82-90; R1, R10-R13).

    Tie reporting (north_star: decisions within 1e-6 of their threshold are logged):
    ``accept_margins[b, i]`` = |u_i - ratio_i| of every test performed; ``sample_margin_hi`` =
    |cum_{j*} - u_s Z| and ``sample_margin_lo`` = |cum_{j*-1} - u_s Z| with ``tok_next`` /
    ``tok_prev`` the positive-residual neighbours a perturbed sampler would pick instead.
    ``n_force[b] >= 0`` replaces the first rejection by a given N (stage-wise comparison of the
    sampling step after a logged accept tie); ratios and margins are still those of the tests."""
    D, T = _f64(D), _f64(T)
    B, k, V = D.shape
    assert T.shape == (B, k + 1, V)
    tok = _i32(tok).reshape(B, k)
    gamma = _i32(gamma).reshape(B)
    nf = None if n_force is None else _i32(n_force).reshape(B)
    n_acc = np.empty(B, dtype=np.int32)
    out_tok = np.empty(B, dtype=np.int32)
    ratio = np.empty((B, k))
    Z = np.empty(B)
    st = np.empty(B, dtype=np.int32)
    margins = np.empty((B, 3))
    ea = np.empty((B, k))
    am = np.empty((B, k))
    nbr = np.empty((B, 2), dtype=np.int32)
    lib().oracle_verify(_p(D), _p(T), _p(tok), _p(gamma), B, k, V, tau_d, tau_t,
                        ctypes.c_uint64(seed), ctypes.c_uint64(offset), seq_base,
                        _p(n_acc), _p(out_tok), _p(ratio), _p(Z), _p(st), _p(margins), _p(ea),
                        nthreads or default_threads(), _p(nf) if nf is not None else None, _p(am), _p(nbr))
    return {"n_accept": n_acc, "out_tok": out_tok, "accept_ratio": ratio, "resid_mass": Z,
            "status": st, "accept_margin": margins[:, 2], "accept_margins": am,
            "sample_margin": np.minimum(margins[:, 0], margins[:, 1]),
            "sample_margin_hi": margins[:, 0], "sample_margin_lo": margins[:, 1],
            "tok_prev": nbr[:, 0], "tok_next": nbr[:, 1], "exp_accept_true": ea}
