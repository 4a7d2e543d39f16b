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


def compare_verify(gv: dict, rv: dict, rep: ParityReport):
    """sd_verify outputs vs oracle.verify given the same gamma."""
    err_g, err_r = gv["status"] & ~32, rv["status"] & ~32  # bit 32 (RESID_ZERO) is not an error
    assert np.array_equal(err_g != 0, err_r != 0), \
        f"status mismatch gpu {err_g[err_g != err_r][:5]} oracle {err_r[err_g != err_r][:5]}"
    ok = err_r == 0
    assert close(gv["accept_ratio"][ok], rv["accept_ratio"][ok]).all(), "accept ratio mismatch"
    assert close(gv["resid_mass"][ok], rv["resid_mass"][ok]).all(), "residual mass mismatch"
    for b in np.nonzero(ok)[0]:
        if gv["n_accept"][b] != rv["n_accept"][b]:
            m = rv["accept_margin"][b]
            assert m < TIE, f"seq {b}: n_accept {gv['n_accept'][b]} vs oracle {rv['n_accept'][b]}, margin {m}"
            rep.log("accept", int(b), float(m))
            continue
        if gv["out_tok"][b] != rv["out_tok"][b]:
            m = rv["sample_margin"][b]
            assert m < TIE, f"seq {b}: token {gv['out_tok'][b]} vs oracle {rv['out_tok'][b]}, margin {m}"
            rep.log("sample", int(b), float(m))
    bad = ~ok
    assert np.all(gv["n_accept"][bad] == 0) and np.all(gv["out_tok"][bad] == -1)


def gpu_np(d: dict) -> dict:
    return {k: (v.cpu().numpy() if v is not None else None) for k, v in d.items()}
