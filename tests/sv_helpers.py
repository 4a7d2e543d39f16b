"""Shared test helpers: upload synthetic inputs, run the CUDA path and the oracle on the
same bytes, and compare stage by stage (DESIGN.md §6 tolerances and tie bands)."""
from __future__ import annotations

import numpy as np

import oracle
import synth

# north_star: continuous outputs within 1e-4 relative / 1e-6 absolute
RTOL, ATOL = 1e-4, 1e-6
# ties logged, not failed, within this distance of a decision threshold (north_star: 1e-6)
TIE = 1e-6


def to_torch(x: dict, device="cuda"):
    import torch
    if x["dtype"] == "bf16":
        conv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.bfloat16).to(device)  # noqa: E731
    else:
        conv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
    return conv(x["D"]), conv(x["C"]), conv(x["T"]), torch.from_numpy(x["tok"]).to(device)


def oracle_inputs(x: dict):
    return synth.to_f64(x["D"], x["dtype"]), synth.to_f64(x["C"], x["dtype"]), synth.to_f64(x["T"], x["dtype"])


def close(gpu, ref, rtol=RTOL, atol=ATOL):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    both_nan = np.isnan(gpu) & np.isnan(ref)
    both_inf = np.isinf(gpu) & np.isinf(ref) & (np.sign(gpu) == np.sign(ref))
    with np.errstate(invalid="ignore"):
        ok = np.abs(gpu - ref) <= atol + rtol * np.abs(ref)
    return ok | both_nan | both_inf


def bin_ties(values, edges, tie=TIE):
    e = np.asarray(edges, dtype=np.float64)[1:-1]
    v = np.asarray(values, dtype=np.float64)
    if e.size == 0:
        return np.zeros(v.shape, dtype=bool)
    with np.errstate(invalid="ignore"):
        return (np.abs(v[..., None] - e) < tie).any(-1)


class ParityReport:
    def __init__(self):
        self.ties = []

    def log(self, what, idx, margin):
        self.ties.append((what, idx, margin))


def compare_score(gs: dict, rs: dict, profile: dict | None, rep: ParityReport):
    """sv_score outputs vs oracle.score on the same inputs."""
    st_g, st_r = gs["status"], rs["status"]
    assert np.array_equal(st_g != 0, st_r != 0), f"status mismatch {np.argwhere((st_g != 0) != (st_r != 0))[:5]}"
    ok = st_r == 0
    for name in ("S", "A", "KL"):
        good = close(gs[name][ok], rs[name][ok])
        assert good.all(), f"{name} mismatch: gpu {gs[name][ok][~good][:5]} oracle {rs[name][ok][~good][:5]}"
    assert close(gs["draft_ptok"][ok], rs["pd_tok"][ok]).all()
    if profile is not None:
        # stage-wise: GPU p_hat equals the profile cell of ITS OWN fp32 (S, A) exactly
        for idx in zip(*np.nonzero(ok)):
            want = oracle.lookup(profile["s_edges"], profile["a_edges"], profile["cells"],
                                 float(gs["S"][idx]), float(gs["A"][idx]))
            assert np.float32(want) == gs["p_hat"][idx], (idx, want, gs["p_hat"][idx])
        # vs the oracle's own p_hat: equal unless S or A sits within TIE of a bin edge
        diff = ok & (gs["p_hat"].astype(np.float64) != rs["p_hat"])
        tie = bin_ties(rs["S"], profile["s_edges"]) | bin_ties(rs["A"], profile["a_edges"])
        for idx in zip(*np.nonzero(diff)):
            assert tie[idx], f"p_hat mismatch outside the tie band at {idx}"
            rep.log("bin", idx, 0.0)
        assert np.all(gs["p_hat"][~ok] == 0)


def compare_verify(gv: dict, rv: dict, rep: ParityReport, rerun=None):
    """sd_verify outputs vs oracle.verify given the same gamma.

    Integer decisions must be bit-exact unless the oracle's own decision is a tie (north_star:
    within 1e-6 of its threshold), judged where the decisions part:
      * n_accept: the first position where exactly one side rejected must have
        |u_i - ratio_i| < TIE; the sampling stage is then compared on the GPU's N by re-running
        the oracle with n_force = N_gpu (``rerun(b, N) -> oracle.verify dict for sequence b``);
      * out_tok: the GPU token must be the oracle's positive-residual neighbour on the side the
        margin allows (tok_next with |cum_{j*} - u_s Z| < TIE, or tok_prev with
        |cum_{j*-1} - u_s Z| < TIE)."""
    err_g, err_r = gv["status"] & ~32, rv["status"] & ~32  # bit 32 (RESID_ZERO) is not an error
    assert np.array_equal(err_g != 0, err_r != 0), \
        f"status mismatch gpu {err_g[err_g != err_r][:5]} oracle {err_r[err_g != err_r][:5]}"
    ok = err_r == 0
    assert close(gv["accept_ratio"][ok], rv["accept_ratio"][ok]).all(), "accept ratio mismatch"
    for b in np.nonzero(ok)[0]:
        ref = rv
        rb = b
        ng, nr = int(gv["n_accept"][b]), int(rv["n_accept"][b])
        if ng != nr:
            j = min(ng, nr)  # the first test whose outcome differs
            m = rv["accept_margins"][b, j]
            assert m < TIE, f"seq {b}: n_accept {ng} vs oracle {nr}, margin {m} at position {j}"
            rep.log("accept", int(b), float(m))
            assert rerun is not None, f"seq {b}: accept tie but no stage-wise rerun available"
            ref, rb = rerun(int(b), ng), 0  # the sampling stage on the GPU's own N
            assert (ref["status"][0] & ~32) == 0
        assert close(gv["resid_mass"][b], ref["resid_mass"][rb]), \
            f"seq {b}: residual mass {gv['resid_mass'][b]} vs oracle {ref['resid_mass'][rb]}"
        tg, tr = int(gv["out_tok"][b]), int(ref["out_tok"][rb])
        if tg != tr:
            hi, lo = ref["sample_margin_hi"][rb], ref["sample_margin_lo"][rb]
            nxt, prv = int(ref["tok_next"][rb]), int(ref["tok_prev"][rb])
            assert (tg == nxt and hi < TIE) or (tg == prv and lo < TIE), \
                f"seq {b}: token {tg} vs oracle {tr} (neighbours {prv}/{nxt}, margins lo {lo} hi {hi})"
            rep.log("sample", int(b), float(min(hi, lo)))
    bad = ~ok
    assert np.all(gv["n_accept"][bad] == 0) and np.all(gv["out_tok"][bad] == -1)


def oracle_rerun(Dd, Td, tok, gamma, tau_d, tau_t, seed, offset, seq_base):
    """rerun(b, N) for compare_verify: oracle.verify of sequence b alone with N forced."""
    def rerun(b, N):
        sl = slice(b, b + 1)
        return oracle.verify(Dd[sl], Td[sl], np.asarray(tok)[sl], np.asarray(gamma)[sl], tau_d, tau_t, seed,
                             offset, seq_base + b, n_force=[N])
    return rerun


def load_golden(name="convention_vector"):
    """tests/golden/<name>.json: logits as fp32 arrays ("-inf" strings decoded), plus the setup
    and expected blocks as they are stored."""
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name + ".json")) as f:
        g = json.load(f)
    st = g["setup"]

    def arr(v):
        return np.array([[[(-np.inf if e == "-inf" else e) for e in row] for row in seq] for seq in v],
                        dtype=np.float32)
    x = {"D": arr(st["D"]), "C": arr(st["C"]), "T": arr(st["T"]), "tok": np.array(st["tok"], dtype=np.int32),
         "dtype": "f32", "B": st["B"], "k": st["k"], "V": st["V"]}
    L = np.array([4.0 + max(0, n - 2) for n in range(st["k"] + 2)])
    return g, x, L


def gpu_np(d: dict) -> dict:
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in d.items()}
