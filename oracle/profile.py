"""Offline (S, A) acceptance profile -- TEST / OFFLINE INFRASTRUCTURE ONLY (NEXT-4, CPU form).

Plain numpy, fp64, following SPEC's profiler module step by step:
  adaptive_edges   S L275-283 (P L176 "adaptive binning, ensuring each bin contains a
                   similar number of observations")
  build_profile    S L284-292 (P L176 "compute the average token acceptance probability
                   for each bin combination"); empty-cell fallbacks of S L296 are
                   pre-filled so that the GPU does a pure table lookup (DESIGN R9)
  info_gain        S L302-310 (P L150-152 I(X;Y) = H(X) - H(X|Y); Table 2 P L347-368)

Only ``scripts/build_profile.py`` and ``tests/`` use this module.
"""
from __future__ import annotations

import math

import numpy as np


def adaptive_edges(samples, n_bins: int) -> np.ndarray:
    """Equal-frequency edges: interior edge j (1..n_bins-1) is the ceil(j*n/n_bins)-th
    order statistic (S L281: samples 1..100, 10 bins -> every 10th order statistic),
    first edge = min, last edge = max; duplicates collapsed (S L278)."""
    x = np.sort(np.asarray(samples, dtype=np.float64))
    n = x.size
    assert n >= 1 and n_bins >= 1
    edges = [x[0]]
    for j in range(1, n_bins):
        e = x[int(math.ceil(j * n / n_bins)) - 1]
        if e > edges[-1]:
            edges.append(e)
    if x[-1] > edges[-1] or len(edges) == 1:
        edges.append(x[-1])
    return np.asarray(edges, dtype=np.float64)


def bin_of(edges, value: float) -> int:
    """Right-closed bins (e_j, e_{j+1}], first bin [e_0, e_1]; clamp (DESIGN R9)."""
    idx = 0
    for j in range(1, len(edges) - 1):
        if edges[j] < value:
            idx = j
    return idx


def build_profile(s, a, x, n_s_bins: int = 20, n_a_bins: int = 15) -> dict:
    """Cell means of the true acceptance probability X over adaptive (S, A) bins.
    Empty cell -> its S-row mean -> global mean (S L296), pre-filled."""
    s = np.asarray(s, dtype=np.float64)
    a = np.asarray(a, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    se = adaptive_edges(s, n_s_bins)
    ae = adaptive_edges(a, n_a_bins)
    ns, na = len(se) - 1, len(ae) - 1
    cnt = np.zeros((ns, na))
    tot = np.zeros((ns, na))
    for sv, av, xv in zip(s, a, x):
        i, j = bin_of(se, sv), bin_of(ae, av)
        cnt[i, j] += 1
        tot[i, j] += xv
    gmean = float(x.mean())
    cells = np.empty((ns, na))
    for i in range(ns):
        row_n = cnt[i].sum()
        row_mean = tot[i].sum() / row_n if row_n > 0 else gmean
        for j in range(na):
            cells[i, j] = tot[i, j] / cnt[i, j] if cnt[i, j] > 0 else row_mean
    return {"s_edges": se.tolist(), "a_edges": ae.tolist(), "cells": cells.tolist(),
            "counts": cnt.astype(int).tolist(), "global_mean": gmean}


def _entropy(counts) -> float:
    c = np.asarray(counts, dtype=np.float64)
    c = c[c > 0]
    p = c / c.sum()
    return float(-(p * np.log2(p)).sum())


def info_gain(x, s_bin, a_bin, x_bins: int = 10) -> dict:
    """Plug-in H(X), H(X|S), H(X|A), H(X|S,A), I(X;S,A) in bits (S L302-310, Table 2 layout);
    X discretised into x_bins equal-width bins on [0, 1] (S L328)."""
    x = np.asarray(x, dtype=np.float64)
    xb = np.minimum((x * x_bins).astype(int), x_bins - 1)
    sb = np.asarray(s_bin)
    ab = np.asarray(a_bin)

    def cond(keys):
        h = 0.0
        n = len(x)
        for key in np.unique(keys):
            sel = keys == key
            h += sel.sum() / n * _entropy(np.bincount(xb[sel], minlength=x_bins))
        return h

    hx = _entropy(np.bincount(xb, minlength=x_bins))
    sa = sb.astype(np.int64) * 100000 + ab.astype(np.int64)
    hs, ha, hsa = cond(sb), cond(ab), cond(sa)
    return {"h_x": hx, "h_x_s": hs, "h_x_a": ha, "h_x_sa": hsa, "i_x_sa": hx - hsa}
