#!/usr/bin/env python3
"""Build the benchmark (S, A) -> acceptance profile from a synthetic profiling run.

Calls ONLY oracle/ (fp64 CPU) and synth/ (input generator): the paper's offline step
(P L176: "perform a profiling run of speculative decoding using these discretized
variables and compute the average token acceptance probability for each bin
combination"), with SPEC's adaptive binning (S L275-292) and 20 x 15 bins (S L331).

Records per position: S, A (draft vs companion, P L159) and X = min(1, P_t(t)/P_d(t)),
the true acceptance probability (P L150; S L260), obtained as the oracle's A-indicator
of the (draft, target) pair.  Output: synth/profile_20x15.json (edges, cells, counts,
global mean, Table-2-layout information-gain report of the run).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import profile as oprof  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--positions", type=int, default=65536)
    ap.add_argument("--V", type=int, default=32000)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--seed", type=int, default=0xB0F1)
    ap.add_argument("--out", default=synth.PROFILE_PATH)
    args = ap.parse_args()
    k, V = args.k, args.V
    n_seq = args.positions // k
    S, A, X = [], [], []
    chunk = 256
    for s0 in range(0, n_seq, chunk):
        ids = np.arange(s0, min(n_seq, s0 + chunk))
        x = synth.make_inputs(len(ids), k, V, "bf16", seed=args.seed, seq_ids=ids)
        D = synth.to_f64(x["D"], "bf16")
        C = synth.to_f64(x["C"], "bf16")
        T = synth.to_f64(x["T"], "bf16")
        r = oracle.score(D, C, x["tok"])
        xr = oracle.score(D, T[:, :k], x["tok"])["A"]
        ok = (r["status"] == 0)
        S.append(r["S"][ok]); A.append(r["A"][ok]); X.append(xr[ok])
        print(f"  {s0 + len(ids)}/{n_seq} sequences", file=sys.stderr)
    S, A, X = np.concatenate(S), np.concatenate(A), np.concatenate(X)
    prof = oprof.build_profile(S, A, X, 20, 15)
    sb = [oprof.bin_of(prof["s_edges"], v) for v in S]
    ab = [oprof.bin_of(prof["a_edges"], v) for v in A]
    prof["info_gain_adaptive"] = oprof.info_gain(X, np.array(sb), np.array(ab))
    prof["meta"] = {"generator": "synth.make_inputs", "seed": args.seed, "V": V, "k": k, "dtype": "bf16",
                    "n_records": int(S.size), "script": "scripts/build_profile.py (oracle/ only)",
                    "cells_layout": "[s_bin][a_bin], right-closed bins, fallbacks pre-filled (S L296)"}
    with open(args.out, "w") as f:
        json.dump(prof, f, indent=1)
    print(json.dumps(prof["info_gain_adaptive"]), file=sys.stderr)


if __name__ == "__main__":
    main()
