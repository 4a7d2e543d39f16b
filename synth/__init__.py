"""Seeded synthetic inputs for the SV hot path (shared by tests, bench and the oracle-side
scripts).  This module holds NONE of the method's arithmetic: no softmax, no overlap, no
schedule, no rejection test.  It only draws logits, draft tokens (Gumbel-max on the draft
logits, i.e. t ~ softmax(x_d / tau) without evaluating a softmax) and the fixed inputs
(latency table, profile file).

Recipe (SURVEY §8(d) "Synthetic inputs"), per sequence b, seeded by
numpy PCG64 with the seed sequence [seed, b] so any subset of sequences can be regenerated
independently of B and of the GPU count:
  z     ~ 2 N(0,1) over V, plus `head` entries boosted by U(h0-4, h0+1), h0 = ln(e^2 V)
          (LLM-like: a few head tokens carrying 10-60% of the mass over a long tail)
  x_t   = z + a_b eta_t,  x_d = z + a_b eta_d,  x_c = z + a_b exp(sigma_c N) eta_c
          (a_b sets the draft/target alignment, hence the acceptance rate)
  rows  : D, C have k rows (positions 0..k-1), T has k+1 rows (row k = bonus row)
  dtype : rounded to bf16 (round-to-nearest-even) or kept fp32
  tokens: t_i = argmax(x_d/tau_d + Gumbel) (resampled if x_d[t] is > 46 tau below the max)
"""
from __future__ import annotations

import json
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
PROFILE_PATH = os.path.join(_HERE, "profile_20x15.json")

# alignment amplitudes: ~0.95 ... ~0.05 acceptance at V = 32000..152064
ALIGN_MIX = (0.1, 0.3, 0.6, 1.0, 1.5, 2.5)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (round-to-nearest-even), returned as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def latency_table(n_max: int, base: float = 4.0, knee: int = 2, slope: float = 1.0) -> np.ndarray:
    """L[n] = base + slope * max(0, n - knee) for n = 0..n_max (fp64; DESIGN R3: base 4, knee 2,
    slope 1 = SPEC S L410's model).  n counts target positions (gamma + 1)."""
    return np.array([base + slope * max(0, n - knee) for n in range(n_max + 1)], dtype=np.float64)


def load_profile(path: str = PROFILE_PATH) -> dict:
    """The (S, A) profile as the fp32 table the C ABI consumes (sv_profile is fp32): edges and
    cells are rounded to float32 once here, so the oracle and the GPU see identical values."""
    with open(path) as f:
        prof = json.load(f)
    for key in ("s_edges", "a_edges", "cells"):
        prof[key] = np.asarray(prof[key], dtype=np.float32).astype(np.float64).tolist()
    return prof


def amplitudes(B: int, seed: int, alignment="mix") -> np.ndarray:
    rng = np.random.default_rng([seed, 0xA11])
    if alignment == "mix":
        return rng.choice(np.asarray(ALIGN_MIX), size=B)
    if alignment == "sweep":  # evenly spread over the mix, per sequence
        return np.asarray(ALIGN_MIX)[np.arange(B) % len(ALIGN_MIX)]
    return np.full(B, float(alignment))


def _gen_sequence(seed, b, k, V, a, dtype, tau_d, sigma_c, head):
    rng = np.random.default_rng([seed, b])
    h0 = math.log(math.e ** 2 * V)
    z = rng.standard_normal((k + 1, V), dtype=np.float32)
    z *= 2.0
    idx = rng.integers(0, V, (k + 1, head))
    boost = rng.uniform(h0 - 4.0, h0 + 1.0, (k + 1, head)).astype(np.float32)
    np.add.at(z, (np.arange(k + 1)[:, None], idx), boost)
    xt = z + np.float32(a) * rng.standard_normal((k + 1, V), dtype=np.float32)
    xd = z[:k] + np.float32(a) * rng.standard_normal((k, V), dtype=np.float32)
    fac = np.exp(sigma_c * rng.standard_normal((k, 1))).astype(np.float32)
    xc = z[:k] + np.float32(a) * fac * rng.standard_normal((k, V), dtype=np.float32)
    if dtype == "bf16":
        xd, xc, xt = f32_to_bf16_bits(xd), f32_to_bf16_bits(xc), f32_to_bf16_bits(xt)
        xd_val = bf16_bits_to_f32(xd)
    else:
        xd_val = xd
    tok = np.empty(k, dtype=np.int32)
    for i in range(k):
        y = xd_val[i].astype(np.float64) / tau_d
        ymax = y.max()
        while True:
            g = -np.log(-np.log(rng.random(V)))
            t = int(np.argmax(y + g))
            if y[t] - ymax > -46.0:  # p_d(t) > ~1e-20 (DESIGN R14)
                break
        tok[i] = t
    return xd, xc, xt, tok


def make_inputs(B: int, k: int, V: int, dtype: str = "bf16", seed: int = 0x5EED, alignment="mix",
                tau_d: float = 1.0, sigma_c: float = 0.5, head: int = 8, seq_ids=None,
                threads: int | None = None) -> dict:
    """Draft D [B,k,V], companion C [B,k,V], target T [B,k+1,V] logits (uint16 bf16 bits or
    float32) and draft tokens [B,k].  `seq_ids` selects which global sequences to draw
    (default 0..B-1); sequence g is identical whatever else is generated."""
    assert dtype in ("bf16", "f32")
    seq_ids = np.arange(B) if seq_ids is None else np.asarray(seq_ids)
    amp_all = amplitudes(int(seq_ids.max()) + 1, seed, alignment)
    store = np.uint16 if dtype == "bf16" else np.float32
    D = np.empty((len(seq_ids), k, V), dtype=store)
    C = np.empty((len(seq_ids), k, V), dtype=store)
    T = np.empty((len(seq_ids), k + 1, V), dtype=store)
    tok = np.empty((len(seq_ids), k), dtype=np.int32)

    def work(j):
        g = int(seq_ids[j])
        D[j], C[j], T[j], tok[j] = _gen_sequence(seed, g, k, V, amp_all[g], dtype, tau_d, sigma_c, head)

    with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(len(seq_ids))))
    return {"D": D, "C": C, "T": T, "tok": tok, "dtype": dtype, "amp": amp_all[seq_ids],
            "B": len(seq_ids), "k": k, "V": V}


def to_f64(x: np.ndarray, dtype: str) -> np.ndarray:
    """Exact widening of stored logits to float64 (for the oracle)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(x).astype(np.float64)
    return np.asarray(x, dtype=np.float32).astype(np.float64)
