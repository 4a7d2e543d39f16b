"""Batch sharding of the SV hot path across ranks.

The sequence is the unit that shards: rank r of `world` owns the contiguous global sequences
[begin, end) and passes `seq_base = begin` to `sd_verify`, so the Philox counter -- and hence
every output -- is identical to a single-GPU run over the global batch.  There is no data-path
collective; `gather_rows` is only for checking / reporting outside any timed region.
"""
from __future__ import annotations

import torch


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of `total` sequences: [floor(r*T/W), floor((r+1)*T/W))."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    return (rank * total) // world, ((rank + 1) * total) // world


def weak_range(per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns `per_rank` sequences of a global batch of per_rank*world."""
    return rank * per_rank, (rank + 1) * per_rank


def gather_rows(x: torch.Tensor, total: int, group=None) -> torch.Tensor | None:
    """Gather per-rank row blocks (first dim = this rank's sequences) to rank 0 in global order.
    Works with any torch.distributed backend (gloo on CPU, NCCL on GPU)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    m = max(sizes)
    pad = torch.zeros((m,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


# ---------------------------------------------------------------------------------------------
# Vocab-sharded staging (BASELINE config 4; include/sv.h "Vocab-sharded staging").
# Thin wrappers with the C-ABI names (argument marshalling only) and `VocabShardedPipeline`,
# which runs score -> schedule -> verify for one rank's column slice and performs the
# exchanges with a pluggable communicator: `TorchComm` (torch.distributed all_gather_into_tensor
# / all_reduce(MAX), NCCL over NVLink on GPUs) or, for single-process checks, a driver that
# steps G pipelines in lock step (tests/test_gpu_shard.py).

import ctypes  # noqa: E402

from . import _lib  # noqa: E402


def _sv():
    from . import _dtype_code, _logits, _ptr, _stream  # late: avoid an import cycle
    return _dtype_code, _logits, _ptr, _stream


def xch_bytes(stage: int, B: int, k: int, V_local: int, dtype: torch.dtype) -> int:
    code = _lib.SV_BF16 if dtype == torch.bfloat16 else _lib.SV_F32
    n = int(_lib.load().sv_shard_xch_bytes(stage, B, k, V_local, code))
    if n == 0:
        raise _lib.SvError("unsupported vocab-sharded shape")
    return n


class TorchComm:
    """Exchanges over a torch.distributed process group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> None:
        self.dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce_max(self, t: torch.Tensor) -> None:
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)


class VocabShardedPipeline:
    """One rank of the vocab-sharded SV step: this rank holds columns [v_begin, v_begin + V_local)
    of the draft / companion / target logits ([B, k(+1), V_local] views, vocabulary contiguous)."""

    def __init__(self, B, k, V, G, rank, dtype, profile, latency, tau=(1.0, 1.0, 1.0), device="cuda"):
        from . import new_workspace
        if V % G:
            raise _lib.SvError("vocab-sharded staging needs V divisible by the rank count")
        self.B, self.k, self.V, self.G, self.rank, self.dtype = B, k, V, G, rank, dtype
        self.V_local = V // G
        self.v_begin = rank * self.V_local
        self.profile, self.latency = profile, latency
        self.tau_d, self.tau_c, self.tau_t = tau
        self.code = _lib.SV_BF16 if dtype == torch.bfloat16 else _lib.SV_F32
        u8 = dict(dtype=torch.uint8, device=device)
        self.xch = [torch.zeros(xch_bytes(s, B, k, self.V_local, dtype), **u8) for s in range(4)]
        self.xch_all = [torch.zeros(G * x.numel(), **u8) for x in self.xch]
        self.workspace = new_workspace(B, k, self.V_local, dtype, device)
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

    # --- the six stages (each only enqueues kernels on `stream`) ---
    def score_p1(self, Dl, Cl, tok, stream=None):
        _, L, P, S = _sv()
        _lib.check(_lib.load().sv_shard_score_p1(
            ctypes.byref(L(Dl)), ctypes.byref(L(Cl)), P(tok), self.B, self.k, self.V_local, self.v_begin,
            float(self.tau_d), float(self.tau_c), self.xch[0].data_ptr(), S(stream)), "sv_shard_score_p1")

    def score_p2(self, Dl, Cl, tok, stream=None):
        _, L, P, S = _sv()
        _lib.check(_lib.load().sv_shard_score_p2(
            ctypes.byref(L(Dl)), ctypes.byref(L(Cl)), P(tok), self.B, self.k, self.V_local, float(self.tau_d),
            float(self.tau_c), self.xch_all[0].data_ptr(), self.G, self.xch[1].data_ptr(), S(stream)),
            "sv_shard_score_p2")

    def score_finish(self, tok, stream=None):
        _, _, P, S = _sv()
        o = self.score_out
        _lib.check(_lib.load().sv_shard_score_finish(
            P(tok), self.B, self.k, self.V, self.V_local, self.code, float(self.tau_d), float(self.tau_c),
            ctypes.byref(self.profile.c), self.xch_all[0].data_ptr(), self.xch_all[1].data_ptr(), self.G,
            P(o["S"]), P(o["A"]), P(o["KL"]), P(o["p_hat"]), P(o["draft_m"]), P(o["draft_l"]), P(o["draft_ptok"]),
            P(o["status"]), S(stream)), "sv_shard_score_finish")

    def schedule(self, stream=None):
        from . import sv_schedule
        return sv_schedule(self.score_out["p_hat"], self.latency, out=self.sched_out, stream=stream)["gamma"]

    def verify_p1(self, Tl, tok, gamma, stream=None):
        _, L, P, S = _sv()
        _lib.check(_lib.load().sv_shard_verify_p1(
            ctypes.byref(L(Tl)), P(tok), P(gamma), self.B, self.k, self.V_local, self.v_begin, float(self.tau_t),
            self.xch[2].data_ptr(), S(stream)), "sv_shard_verify_p1")

    def verify_p2(self, Dl, Tl, tok, gamma, seed, offset, seq_base=0, stream=None):
        _, L, P, S = _sv()
        so, vo = self.score_out, self.ver_out
        _lib.check(_lib.load().sv_shard_verify_p2(
            ctypes.byref(L(Dl)), ctypes.byref(L(Tl)), P(tok), P(gamma), P(so["draft_m"]), P(so["draft_l"]),
            P(so["draft_ptok"]), self.B, self.k, self.V, self.V_local, float(self.tau_d), float(self.tau_t),
            ctypes.c_uint64(seed), ctypes.c_uint64(offset), int(seq_base), self.xch_all[2].data_ptr(), self.G,
            P(vo["n_accept"]), P(vo["accept_ratio"]), self.xch[3].data_ptr(), self.workspace.data_ptr(),
            self.workspace.numel(), S(stream)), "sv_shard_verify_p2")

    def verify_finish(self, Dl, Tl, stream=None):
        _, L, P, S = _sv()
        vo = self.ver_out
        _lib.check(_lib.load().sv_shard_verify_finish(
            ctypes.byref(L(Dl)), ctypes.byref(L(Tl)), self.B, self.k, self.V_local, self.v_begin, float(self.tau_d),
            float(self.tau_t), self.xch_all[3].data_ptr(), self.G, self.rank, P(vo["out_tok"]), P(vo["resid_mass"]),
            P(vo["status"]), self.workspace.data_ptr(), self.workspace.numel(), S(stream)), "sv_shard_verify_finish")

    def run(self, comm, Dl, Cl, Tl, tok, seed=0, offset=0, seq_base=0, stream=None):
        """The whole step on this rank: 4 all-gathers of the stage blocks + 1 all-reduce(MAX).
        Kernels and collectives go to ONE stream: `stream` is made current for the step, so the
        process group's collectives are ordered after the kernels that produce their inputs."""
        if stream is not None:
            with torch.cuda.stream(stream):
                return self.run(comm, Dl, Cl, Tl, tok, seed, offset, seq_base, None)
        self.score_p1(Dl, Cl, tok, stream)
        comm.all_gather(self.xch_all[0], self.xch[0])
        self.score_p2(Dl, Cl, tok, stream)
        comm.all_gather(self.xch_all[1], self.xch[1])
        self.score_finish(tok, stream)
        gamma = self.schedule(stream)
        self.verify_p1(Tl, tok, gamma, stream)
        comm.all_gather(self.xch_all[2], self.xch[2])
        self.verify_p2(Dl, Tl, tok, gamma, seed, offset, seq_base, stream)
        comm.all_gather(self.xch_all[3], self.xch[3])
        self.verify_finish(Dl, Tl, stream)
        comm.all_reduce_max(self.ver_out["out_tok"])
        return self.ver_out


def run_vocab_sharded_lockstep(pipes, Ds, Cs, Ts, tok, seed=0, offset=0, seq_base=0):
    """Single-process driver: G pipelines (one per simulated rank, column slices on one GPU)
    stepped in lock step; gathers are concatenations, the token all-reduce a max."""
    def gather(stage):
        full = torch.cat([p.xch[stage] for p in pipes])
        for p in pipes:
            p.xch_all[stage].copy_(full)
    for p, D, C in zip(pipes, Ds, Cs):
        p.score_p1(D, C, tok)
    gather(0)
    for p, D, C in zip(pipes, Ds, Cs):
        p.score_p2(D, C, tok)
    gather(1)
    gammas = []
    for p in pipes:
        p.score_finish(tok)
        gammas.append(p.schedule())
    for p, T, g in zip(pipes, Ts, gammas):
        p.verify_p1(T, tok, g)
    gather(2)
    for p, D, T, g in zip(pipes, Ds, Ts, gammas):
        p.verify_p2(D, T, tok, g, seed, offset, seq_base)
    gather(3)
    for p, D, T in zip(pipes, Ds, Ts):
        p.verify_finish(D, T)
    tokmax = torch.stack([p.ver_out["out_tok"] for p in pipes]).max(dim=0).values
    for p in pipes:
        p.ver_out["out_tok"].copy_(tokmax)
    return [p.ver_out for p in pipes]
