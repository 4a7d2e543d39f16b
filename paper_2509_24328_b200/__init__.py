"""paper_2509_24328_b200 -- B200-native hot path of Speculative Verification (arxiv 2509.24328).

Thin torch-facing wrappers with the names of the C ABI (include/sv.h):
    sv_score    steps a1-a3  (softmax normalisers, S / A / KL, profiled p_hat)   P L159-176
    sv_schedule step a4      (goodput-maximising verification length)           P L207-252
    sd_verify   steps a5-a6  (rejection test + residual / bonus sample)          P L29; S L148-165
and `Pipeline`, which owns preallocated outputs and runs the three calls back to back on
one stream (optionally captured in a CUDA graph).  PyTorch supplies device memory and
streams only.  No CPU fallback exists: the compute calls raise without libsv.so / a GPU.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (ROW_ALL_NEG_INF, ROW_BAD_GAMMA, ROW_BAD_LATENCY, ROW_BAD_TOKEN, ROW_DRAFT_ZERO,  # noqa: F401
                   ROW_NAN, ROW_PHAT_BAD, ROW_RESID_ZERO, SV_SCHED_BATCH_GREEDY, SV_SCHED_PER_ROW, SvError)

__all__ = ["sv_score", "sv_score_schedule", "sv_schedule", "sd_verify", "sd_verify_ragged", "workspace_bytes", "Profile",
           "Pipeline", "GraphPipeline", "sv_profile_build", "sv_score_filtered", "sd_verify_filtered", "load_library"]


def load_library():
    return _lib.load()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SV_BF16
    if t.dtype == torch.float32:
        return _lib.SV_F32
    raise SvError(f"unsupported logits dtype {t.dtype}")


def _logits(t: torch.Tensor) -> _lib.SvLogits:
    if not t.is_cuda:
        raise SvError("logits must be CUDA tensors (no CPU fallback)")
    if t.dim() != 3 or t.stride(2) != 1:
        raise SvError("logits must be [B, rows, V] with the vocabulary dimension contiguous")
    return _lib.SvLogits(t.data_ptr(), _dtype_code(t), 0, t.stride(0), t.stride(1))


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise SvError("all tensors passed to libsv must live on the GPU")
    if not t.is_contiguous():
        raise SvError("tensor must be contiguous")
    return t.data_ptr()


def _req(t, name: str, dtype: torch.dtype, shape: tuple, device=None):
    """Argument contract of the C ABI that the C side cannot see (element type and extent)."""
    if t is None:
        raise SvError(f"{name} is required")
    if t.dtype != dtype:
        raise SvError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise SvError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise SvError(f"{name} must live on {device}, got {t.device}")
    return t


def _out(o: dict, name: str, shape, dtype, dev):
    if name in o and o[name] is not None:
        return _req(o[name], f"out[{name!r}]", dtype, shape, dev)
    return torch.empty(shape, dtype=dtype, device=dev)


def _same_logits(ref, t, name: str, shape):
    if t.dtype != ref.dtype:
        raise SvError(f"{name} must have the draft's dtype {ref.dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise SvError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.device != ref.device:
        raise SvError(f"{name} must live on {ref.device}")


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def workspace_bytes(B: int, k: int, V: int, dtype: torch.dtype) -> int:
    code = _lib.SV_BF16 if dtype == torch.bfloat16 else _lib.SV_F32
    return int(_lib.load().sv_workspace_bytes(B, k, V, code))


class Profile:
    """Device copy of an (S, A) -> p_hat profile (edges + cells, fp32)."""

    def __init__(self, s_edges, a_edges, cells, device="cuda"):
        self.s_edges = torch.as_tensor(s_edges, dtype=torch.float32, device=device).contiguous()
        self.a_edges = torch.as_tensor(a_edges, dtype=torch.float32, device=device).contiguous()
        self.cells = torch.as_tensor(cells, dtype=torch.float32, device=device).reshape(-1).contiguous()
        self.n_s = self.s_edges.numel() - 1
        self.n_a = self.a_edges.numel() - 1
        assert self.cells.numel() == self.n_s * self.n_a
        self.c = _lib.SvProfile(self.s_edges.data_ptr(), self.n_s, self.n_a, self.a_edges.data_ptr(),
                                self.cells.data_ptr())

    @classmethod
    def from_dict(cls, d: dict, device="cuda"):
        return cls(d["s_edges"], d["a_edges"], d["cells"], device)


def new_workspace(B: int, k: int, V: int, dtype: torch.dtype, device="cuda") -> torch.Tensor:
    """Workspace for sv_score / sd_verify: zero-filled once (the library keeps its counters
    zeroed at the end of every call), reusable across calls on one stream."""
    return torch.zeros(max(16, workspace_bytes(B, k, V, dtype)), dtype=torch.uint8, device=device)


def sv_score(D, C, tok, tau_d=1.0, tau_c=1.0, profile: Profile | None = None, workspace=None, out=None,
             stream=None) -> dict:
    """Steps a1-a3 (P L159, L164, L176) through the C ABI `sv_score`."""
    B, k, V = D.shape
    dev = D.device
    _same_logits(D, C, "C", (B, k, V))
    _req(tok, "tok", torch.int32, (B, k), dev)
    if workspace is None:
        workspace = new_workspace(B, k, V, D.dtype, D.device)
    o = out or {}
    res = {n: _out(o, n, (B, k), torch.float32, dev) for n in ("S", "A", "KL", "p_hat", "draft_m", "draft_l",
                                                                 "draft_ptok")}
    res["status"] = _out(o, "status", (B, k), torch.int32, dev)
    if profile is None:
        res["p_hat"] = None
    st = _lib.load().sv_score(
        ctypes.byref(_logits(D)), ctypes.byref(_logits(C)), _ptr(tok), B, k, V, float(tau_d), float(tau_c),
        ctypes.byref(profile.c) if profile is not None else None,
        _ptr(res["S"]), _ptr(res["A"]), _ptr(res["KL"]), _ptr(res["p_hat"]), _ptr(res["draft_m"]),
        _ptr(res["draft_l"]), _ptr(res["draft_ptok"]), _ptr(res["status"]), workspace.data_ptr(), workspace.numel(),
        _stream(stream))
    _lib.check(st, "sv_score")
    return res


def sv_score_schedule(D, C, tok, latency, tau_d=1.0, tau_c=1.0, profile: Profile | None = None, plus_one=1,
                      workspace=None, out=None, sched_out=None, stream=None) -> tuple[dict, dict]:
    """Steps a1-a4 in one launch (C ABI `sv_score_schedule`): sv_score, and the last row epilogue
    of each sequence runs the per-row schedule.  Bit-identical to sv_score + sv_schedule."""
    B, k, V = D.shape
    dev = D.device
    if profile is None:
        raise SvError("sv_score_schedule needs a profile (p_hat drives the schedule)")
    _same_logits(D, C, "C", (B, k, V))
    _req(tok, "tok", torch.int32, (B, k), dev)
    _req(latency, "latency", torch.float64, (latency.numel(),), dev)
    if workspace is None:
        workspace = new_workspace(B, k, V, D.dtype, dev)
    o = out or {}
    res = {n: _out(o, n, (B, k), torch.float32, dev) for n in ("S", "A", "KL", "p_hat", "draft_m", "draft_l",
                                                                 "draft_ptok")}
    res["status"] = _out(o, "status", (B, k), torch.int32, dev)
    so = sched_out or {}
    sch = {"gamma": _out(so, "gamma", (B,), torch.int32, dev),
           "exp_accept": _out(so, "exp_accept", (B,), torch.float32, dev),
           "goodput": _out(so, "goodput", (B,), torch.float32, dev),
           "status": _out(so, "status", (B,), torch.int32, dev)}
    st = _lib.load().sv_score_schedule(
        ctypes.byref(_logits(D)), ctypes.byref(_logits(C)), _ptr(tok), B, k, V, float(tau_d), float(tau_c),
        ctypes.byref(profile.c), _ptr(res["S"]), _ptr(res["A"]), _ptr(res["KL"]), _ptr(res["p_hat"]),
        _ptr(res["draft_m"]), _ptr(res["draft_l"]), _ptr(res["draft_ptok"]), _ptr(res["status"]), _ptr(latency),
        latency.numel(), int(plus_one), _ptr(sch["gamma"]), _ptr(sch["exp_accept"]), _ptr(sch["goodput"]),
        _ptr(sch["status"]), workspace.data_ptr(), workspace.numel(), _stream(stream))
    _lib.check(st, "sv_score_schedule")
    return res, sch


def sv_schedule(p_hat, latency, mode=SV_SCHED_PER_ROW, plus_one=1, out=None, stream=None) -> dict:
    """Step a4 (P L207-252) through the C ABI `sv_schedule`; latency is a CUDA fp64 tensor."""
    B, k = p_hat.shape
    dev = p_hat.device
    _req(p_hat, "p_hat", torch.float32, (B, k))
    _req(latency, "latency", torch.float64, (latency.numel(),), dev)
    o = out or {}
    res = {"gamma": _out(o, "gamma", (B,), torch.int32, dev),
           "exp_accept": _out(o, "exp_accept", (B,), torch.float32, dev),
           "goodput": _out(o, "goodput", (B,), torch.float32, dev),
           "status": _out(o, "status", (B,), torch.int32, dev)}
    st = _lib.load().sv_schedule(_ptr(p_hat), B, k, _ptr(latency), latency.numel(), mode, plus_one,
                                 _ptr(res["gamma"]), _ptr(res["exp_accept"]), _ptr(res["goodput"]),
                                 _ptr(res["status"]), None, 0, _stream(stream))
    _lib.check(st, "sv_schedule")
    return res


def _verify_args(B, k, dev, tok, gamma, draft_m, draft_l, draft_ptok):
    _req(tok, "tok", torch.int32, (B, k), dev)
    _req(gamma, "gamma", torch.int32, (B,), dev)
    for n, t in (("draft_m", draft_m), ("draft_l", draft_l), ("draft_ptok", draft_ptok)):
        _req(t, n, torch.float32, (B, k), dev)


def _verify_out(o: dict, B, k, dev) -> dict:
    return {"n_accept": _out(o, "n_accept", (B,), torch.int32, dev),
            "out_tok": _out(o, "out_tok", (B,), torch.int32, dev),
            "accept_ratio": _out(o, "accept_ratio", (B, k), torch.float32, dev),
            "resid_mass": _out(o, "resid_mass", (B,), torch.float32, dev),
            "status": _out(o, "status", (B,), torch.int32, dev)}


def sd_verify(D, T, tok, gamma, draft_m, draft_l, draft_ptok, tau_d=1.0, tau_t=1.0, seed=0, offset=0,
              seq_base=0, workspace=None, out=None, stream=None) -> dict:
    """Steps a5-a6 (P L29; S L148-165) through the C ABI `sd_verify`."""
    B, k, V = D.shape
    dev = D.device
    _same_logits(D, T, "T", (B, k + 1, V))
    _verify_args(B, k, dev, tok, gamma, draft_m, draft_l, draft_ptok)
    res = _verify_out(out or {}, B, k, dev)
    if workspace is None:
        workspace = new_workspace(B, k, V, D.dtype, dev)
    st = _lib.load().sd_verify(
        ctypes.byref(_logits(D)), ctypes.byref(_logits(T)), _ptr(tok), _ptr(gamma), _ptr(draft_m), _ptr(draft_l),
        _ptr(draft_ptok), B, k, V, float(tau_d), float(tau_t), ctypes.c_uint64(seed), ctypes.c_uint64(offset),
        int(seq_base), _ptr(res["n_accept"]), _ptr(res["out_tok"]), _ptr(res["accept_ratio"]), _ptr(res["resid_mass"]),
        _ptr(res["status"]), workspace.data_ptr(), workspace.numel(), _stream(stream))
    _lib.check(st, "sd_verify")
    return res


def sd_verify_ragged(D, T_rows, t_rowptr, tok, gamma, draft_m, draft_l, draft_ptok, tau_d=1.0, tau_t=1.0, seed=0,
                     offset=0, offset_dev=None, seq_base=0, workspace=None, out=None, stream=None) -> dict:
    """Steps a5-a6 over a compacted target `T_rows` [R, V] (NEXT-3, P L266) through the C ABI
    `sd_verify_ragged`; `t_rowptr` [B] int64 = first row of each sequence.  `offset_dev` (a CUDA
    uint64/int64 scalar tensor) makes the Philox offset a device value (CUDA-graph replays)."""
    B, k, V = D.shape
    dev = D.device
    if T_rows.dim() != 2 or T_rows.stride(1) != 1 or T_rows.dtype != D.dtype or T_rows.shape[1] != V:
        raise SvError("ragged target must be [rows, V] with the vocabulary contiguous and the draft's dtype")
    _req(t_rowptr, "t_rowptr", torch.int64, (B,), dev)
    if offset_dev is not None and (offset_dev.dtype not in (torch.int64, torch.uint64) or offset_dev.numel() != 1):
        raise SvError("offset_dev must be a one-element int64 / uint64 CUDA tensor")
    _verify_args(B, k, dev, tok, gamma, draft_m, draft_l, draft_ptok)
    if not T_rows.is_cuda or T_rows.device != dev:
        raise SvError(f"ragged target must be a CUDA tensor on {dev}")
    res = _verify_out(out or {}, B, k, dev)
    if workspace is None:
        workspace = new_workspace(B, k, V, D.dtype, dev)
    st = _lib.load().sd_verify_ragged(
        ctypes.byref(_logits(D)), T_rows.data_ptr(), T_rows.stride(0), _ptr(t_rowptr), _ptr(tok), _ptr(gamma),
        _ptr(draft_m), _ptr(draft_l), _ptr(draft_ptok), B, k, V, float(tau_d), float(tau_t), ctypes.c_uint64(seed),
        ctypes.c_uint64(offset), _ptr(offset_dev), int(seq_base), _ptr(res["n_accept"]), _ptr(res["out_tok"]),
        _ptr(res["accept_ratio"]), _ptr(res["resid_mass"]), _ptr(res["status"]), workspace.data_ptr(),
        workspace.numel(), _stream(stream))
    _lib.check(st, "sd_verify_ragged")
    return res


def new_filter_workspace(B: int, k: int, device="cuda") -> torch.Tensor:
    return torch.empty(max(16, int(_lib.load().sv_filter_workspace_bytes(B, k))), dtype=torch.uint8, device=device)


def sv_score_filtered(D, C, tok, top_k=20, top_p=0.8, tau_d=1.0, tau_c=1.0, profile: Profile | None = None,
                      fworkspace=None, stream=None) -> dict:
    """Steps a1-a3 over the filtered distributions (NEXT-2; S L73-81, L238) through the C ABI
    `sv_score_filtered`.  Keep `fworkspace` for `sd_verify_filtered` (it holds the draft lists)."""
    B, k, V = D.shape
    dev = D.device
    _same_logits(D, C, "C", (B, k, V))
    _req(tok, "tok", torch.int32, (B, k), dev)
    fworkspace = fworkspace if fworkspace is not None else new_filter_workspace(B, k, dev)
    res = {n: torch.empty((B, k), dtype=torch.float32, device=dev) for n in ("S", "A", "KL", "p_hat", "draft_ptok")}
    res["status"] = torch.empty((B, k), dtype=torch.int32, device=dev)
    if profile is None:
        res["p_hat"] = None
    f = _lib.SvFilter(int(top_k), float(top_p))
    st = _lib.load().sv_score_filtered(
        ctypes.byref(_logits(D)), ctypes.byref(_logits(C)), _ptr(tok), B, k, V, float(tau_d), float(tau_c),
        ctypes.byref(f), ctypes.byref(profile.c) if profile is not None else None, _ptr(res["S"]), _ptr(res["A"]),
        _ptr(res["KL"]), _ptr(res["p_hat"]), _ptr(res["draft_ptok"]), _ptr(res["status"]), fworkspace.data_ptr(),
        fworkspace.numel(), _stream(stream))
    _lib.check(st, "sv_score_filtered")
    res["fworkspace"] = fworkspace
    return res


def sd_verify_filtered(T, tok, gamma, fworkspace, top_k=20, top_p=0.8, tau_t=1.0, seed=0, offset=0, seq_base=0,
                       stream=None, D=None) -> dict:
    """Steps a5-a6 over the filtered distributions (NEXT-2; S L183) through `sd_verify_filtered`.
    `D` (the draft logits given to `sv_score_filtered`) is needed only when a draft nucleus may
    exceed 32 tokens (top_k = 0)."""
    B, k1, V = T.shape
    k = k1 - 1
    dev = T.device
    _req(tok, "tok", torch.int32, (B, k), dev)
    _req(gamma, "gamma", torch.int32, (B,), dev)
    if D is not None:
        _same_logits(T, D, "D", (B, k, V))
    res = {"n_accept": torch.empty(B, dtype=torch.int32, device=dev),
           "out_tok": torch.empty(B, dtype=torch.int32, device=dev),
           "accept_ratio": torch.empty((B, k), dtype=torch.float32, device=dev),
           "resid_mass": torch.empty(B, dtype=torch.float32, device=dev),
           "status": torch.empty(B, dtype=torch.int32, device=dev)}
    f = _lib.SvFilter(int(top_k), float(top_p))
    st = _lib.load().sd_verify_filtered(
        ctypes.byref(_logits(T)), ctypes.byref(_logits(D)) if D is not None else None, _ptr(tok), _ptr(gamma), B, k, V,
        float(tau_t), ctypes.byref(f), ctypes.c_uint64(seed),
        ctypes.c_uint64(offset), int(seq_base), _ptr(res["n_accept"]), _ptr(res["out_tok"]), _ptr(res["accept_ratio"]),
        _ptr(res["resid_mass"]), _ptr(res["status"]), fworkspace.data_ptr(), fworkspace.numel(), _stream(stream))
    _lib.check(st, "sd_verify_filtered")
    return res


def sv_profile_build(S, A, X, n_s_bins=20, n_a_bins=15, x_bins=10, stream=None) -> dict:
    """NEXT-4 (P L176; S L275-310): the offline (S, A) -> acceptance profile of N records and the
    Table-2 information-gain report, through the C ABI `sv_profile_build`."""
    S, A, X = (t.reshape(-1).contiguous().float() for t in (S, A, X))
    N = S.numel()
    dev = S.device
    ws = torch.empty(int(_lib.load().sv_profile_workspace_bytes(N, n_s_bins, n_a_bins, x_bins)) or 16,
                     dtype=torch.uint8, device=dev)
    se = torch.empty(n_s_bins + 1, dtype=torch.float32, device=dev)
    ae = torch.empty(n_a_bins + 1, dtype=torch.float32, device=dev)
    nb = torch.empty(2, dtype=torch.int32, device=dev)
    cells = torch.empty(n_s_bins * n_a_bins, dtype=torch.float64, device=dev)
    counts = torch.empty(n_s_bins * n_a_bins, dtype=torch.int32, device=dev)
    info = torch.empty(5, dtype=torch.float64, device=dev)
    st = _lib.load().sv_profile_build(_ptr(S), _ptr(A), _ptr(X), N, n_s_bins, n_a_bins, x_bins, _ptr(se), _ptr(ae),
                                      _ptr(nb), _ptr(cells), _ptr(counts), _ptr(info), ws.data_ptr(), ws.numel(),
                                      _stream(stream))
    _lib.check(st, "sv_profile_build")
    ns, na = (int(v) for v in nb.tolist())
    return {"s_edges": se[: ns + 1], "a_edges": ae[: na + 1], "cells": cells[: ns * na].view(ns, na),
            "counts": counts[: ns * na].view(ns, na), "n_s": ns, "n_a": na,
            "info": dict(zip(("h_x", "h_x_s", "h_x_a", "h_x_sa", "i_x_sa"), info.tolist()))}


class GraphPipeline:
    """The whole step (sv_score -> sv_schedule -> sd_verify) captured once in a CUDA graph
    (NEXT-3): inputs are copied into fixed device buffers, the Philox offset lives on the device
    and advances by one per replay inside the graph, so replay j draws the same uniforms as an
    eager step with offset = offset0 + j."""

    def __init__(self, B, k, V, dtype, profile: Profile, latency: torch.Tensor, tau=(1.0, 1.0, 1.0),
                 mode=SV_SCHED_PER_ROW, device="cuda", seed=0, offset0=0, seq_base=0):
        self.pipe = Pipeline(B, k, V, dtype, profile, latency, tau, mode, device)
        self.B, self.k, self.V = B, k, V
        self.D = torch.empty((B, k, V), dtype=dtype, device=device)
        self.C = torch.empty((B, k, V), dtype=dtype, device=device)
        self.T = torch.empty((B, k + 1, V), dtype=dtype, device=device)
        self.tok = torch.empty((B, k), dtype=torch.int32, device=device)
        self.offset = torch.full((1,), offset0, dtype=torch.int64, device=device)
        self.rowptr = (torch.arange(B, dtype=torch.int64, device=device) * (k + 1)).contiguous()
        self.seed, self.seq_base = seed, seq_base
        self.graph = None

    def _step(self, stream):
        p = self.pipe
        if p.mode == SV_SCHED_PER_ROW and p.fused:
            sc, sh = sv_score_schedule(self.D, self.C, self.tok, p.latency, p.tau_d, p.tau_c, p.profile,
                                       workspace=p.workspace, out=p.score_out, sched_out=p.sched_out, stream=stream)
        else:
            sc = sv_score(self.D, self.C, self.tok, p.tau_d, p.tau_c, p.profile, workspace=p.workspace,
                          out=p.score_out, stream=stream)
            sh = sv_schedule(sc["p_hat"], p.latency, p.mode, 1, out=p.sched_out, stream=stream)
        r = sd_verify_ragged(self.D, self.T.view(-1, self.V), self.rowptr, self.tok, sh["gamma"], sc["draft_m"],
                             sc["draft_l"], sc["draft_ptok"], p.tau_d, p.tau_t, self.seed, 0, self.offset,
                             self.seq_base, workspace=p.workspace, out=p.ver_out, stream=stream)
        self.offset.add_(1)
        return r

    def capture(self):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm the launch paths once outside the graph, then restore
            off = self.offset.clone()
            self._step(s)
            self.offset.copy_(off)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = self._step(torch.cuda.current_stream())
        return self

    def replay(self):
        self.graph.replay()
        return self.out


class Pipeline:
    """sv_score -> sv_schedule -> sd_verify on one stream with preallocated outputs.

    `force_gamma` (int) replaces the schedule by a constant gamma (full SD verification:
    the fixed-bytes roofline variant of SURVEY §8(d))."""

    def __init__(self, B, k, V, dtype, profile: Profile, latency: torch.Tensor, tau=(1.0, 1.0, 1.0),
                 mode=SV_SCHED_PER_ROW, device="cuda", fused=False):
        self.B, self.k, self.V, self.dtype = B, k, V, dtype
        self.profile, self.latency, self.mode = profile, latency, mode
        self.tau_d, self.tau_c, self.tau_t = tau
        f32 = dict(dtype=torch.float32, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        self.score_out = {n: torch.empty((B, k), **f32) for n in
                          ("S", "A", "KL", "p_hat", "draft_m", "draft_l", "draft_ptok")}
        self.score_out["status"] = torch.empty((B, k), **i32)
        self.sched_out = {"gamma": torch.empty(B, **i32), "exp_accept": torch.empty(B, **f32),
                          "goodput": torch.empty(B, **f32), "status": torch.empty(B, **i32)}
        self.ver_out = {"n_accept": torch.empty(B, **i32), "out_tok": torch.empty(B, **i32),
                        "accept_ratio": torch.empty((B, k), **f32), "resid_mass": torch.empty(B, **f32),
                        "status": torch.empty(B, **i32)}
        self.workspace = new_workspace(B, k, V, dtype, device)
        self.forced_gamma = torch.empty(B, **i32)
        self._forced = None
        # sv_score_schedule (K3 folded into K1's last row epilogue) measured ~1.5 us SLOWER per step
        # than sv_score + a PDL-overlapped sv_schedule at every config; fused=True opts in
        self.fused = bool(fused)

    def run(self, D, C, T, tok, seed=0, offset=0, seq_base=0, force_gamma=None, stream=None):
        if force_gamma is None and self.mode == SV_SCHED_PER_ROW and self.fused:
            sc, sh = sv_score_schedule(D, C, tok, self.latency, self.tau_d, self.tau_c, self.profile,
                                       workspace=self.workspace, out=self.score_out, sched_out=self.sched_out,
                                       stream=stream)
            return sd_verify(D, T, tok, sh["gamma"], sc["draft_m"], sc["draft_l"], sc["draft_ptok"], self.tau_d,
                             self.tau_t, seed, offset, seq_base, workspace=self.workspace, out=self.ver_out,
                             stream=stream)
        sc = sv_score(D, C, tok, self.tau_d, self.tau_c, self.profile, workspace=self.workspace, out=self.score_out,
                      stream=stream)
        if force_gamma is None:
            sh = sv_schedule(sc["p_hat"], self.latency, self.mode, 1, out=self.sched_out, stream=stream)
            gamma = sh["gamma"]
        else:
            if self._forced != int(force_gamma):  # filled once, outside any timed loop
                self.forced_gamma.fill_(int(force_gamma))
                self._forced = int(force_gamma)
            gamma = self.forced_gamma
        return sd_verify(D, T, tok, gamma, sc["draft_m"], sc["draft_l"], sc["draft_ptok"], self.tau_d, self.tau_t,
                         seed, offset, seq_base, workspace=self.workspace, out=self.ver_out, stream=stream)
