"""Vocab-sharded staging on CPU (gloo, world_size 2 and 3): the exchange contract the GPU
staging implements (include/sv.h "Vocab-sharded staging") -- per-rank softmax
partials merged in rank order, accept tests identical on every rank, per-rank residual masses,
the two-level inverse CDF on the owner rank and the all-reduce(MAX) of the token -- run through
paper_2509_24328_b200.shard.TorchComm with fp64 numpy staging on each rank's column slice, and
checked against the unsharded fp64 oracle.  (The kernels themselves are pinned on the GPU by
tests/test_gpu_shard.py.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _staged_verify(comm, Dl, Tl, tok, gamma, v_begin, seed, offset):
    """One rank's fp64 staging of steps a5-a6 over its columns (numpy only, no kernels)."""
    import oracle
    B, k, VL = Dl.shape
    G = comm.world

    def gather(x):
        x = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).reshape(-1)
        out = torch.empty(G * x.numel(), dtype=torch.float64)
        comm.all_gather(out, x)
        return out.numpy().reshape((G,) + tuple(x.shape))

    def norm(X):  # rank-local (m, l) partials -> merged (M, L) in rank order
        m = X.max(-1)
        l = np.exp(X - m[..., None]).sum(-1)
        g = gather(np.stack([m, l], -1)).reshape((G,) + m.shape + (2,))
        M = g[..., 0].max(0)
        L = np.zeros_like(M)
        for r in range(G):
            L += g[r, ..., 1] * np.exp(g[r, ..., 0] - M)
        return M, L

    Md, Ld = norm(Dl)
    Mt, Lt = norm(Tl)
    loc = tok - v_begin
    own = (loc >= 0) & (loc < VL)
    bi, ii = np.nonzero(own)
    xd = np.full(tok.shape, -np.inf)
    xt = np.full(tok.shape, -np.inf)
    xd[bi, ii] = Dl[bi, ii, loc[bi, ii]]
    xt[bi, ii] = Tl[bi, ii, loc[bi, ii]]
    xd, xt = gather(xd).reshape((G,) + tok.shape).max(0), gather(xt).reshape((G,) + tok.shape).max(0)
    n_acc = np.zeros(B, dtype=np.int32)
    mode = np.zeros(B, dtype=np.int32)
    us = np.zeros(B)
    for b in range(B):
        N = gamma[b]
        for i in range(gamma[b]):
            pt = np.exp(xt[b, i] - Mt[b, i]) / Lt[b, i]
            pd = np.exp(xd[b, i] - Md[b, i]) / Ld[b, i]
            if not oracle.uniforms(seed, offset, b, i)[0] < pt / pd:
                N = i
                break
        n_acc[b] = N
        mode[b] = N < gamma[b]
        us[b] = oracle.uniforms(seed, offset, b, N)[1]
    r = np.zeros((B, VL))
    for b in range(B):
        N = n_acc[b]
        pt = np.exp(Tl[b, N] - Mt[b, N]) / Lt[b, N]
        r[b] = np.maximum(0.0, pt - np.exp(Dl[b, N] - Md[b, N]) / Ld[b, N]) if mode[b] else pt
    Zr = gather(r.sum(-1)).reshape(G, B)  # per-rank masses
    tok_out = np.full(B, -1, dtype=np.int32)
    for b in range(B):
        theta = us[b] * Zr[:, b].sum()
        pre = np.concatenate([[0.0], np.cumsum(Zr[:, b])])
        owner = int(np.searchsorted(pre[1:], theta, side="right"))
        owner = min(owner, G - 1)
        if owner == comm.rank:
            c = pre[owner] + np.cumsum(r[b])
            j = int(np.argmax(c > theta)) if (c > theta).any() else int(np.nonzero(r[b] > 0)[0][-1])
            tok_out[b] = v_begin + j
    t = torch.from_numpy(tok_out)
    comm.all_reduce_max(t)
    return n_acc, t.numpy()


def _worker(rank, world, port, out_path):
    import synth
    from paper_2509_24328_b200.shard import TorchComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    B, k, V = 6, 3, 60 * world
    x = synth.make_inputs(B, k, V, "f32", seed=41)
    D, T = synth.to_f64(x["D"], "f32"), synth.to_f64(x["T"], "f32")
    VL = V // world
    gamma = np.array([0, 1, 2, 3, 3, 2], dtype=np.int32)
    n_acc, tok = _staged_verify(comm, D[:, :, rank * VL:(rank + 1) * VL], T[:, :, rank * VL:(rank + 1) * VL],
                                x["tok"], gamma, rank * VL, seed=9, offset=4)
    if rank == 0:
        np.savez(out_path, n_acc=n_acc, tok=tok)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_vocab_sharded_staging_gloo_matches_oracle(tmp_path, world):
    import oracle
    import synth
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    B, k, V = 6, 3, 60 * world
    x = synth.make_inputs(B, k, V, "f32", seed=41)
    D, T = synth.to_f64(x["D"], "f32"), synth.to_f64(x["T"], "f32")
    gamma = np.array([0, 1, 2, 3, 3, 2], dtype=np.int32)
    ref = oracle.verify(D, T, x["tok"], gamma, seed=9, offset=4, seq_base=0, nthreads=1)
    assert np.array_equal(got["n_acc"], ref["n_accept"])
    tie = ref["sample_margin"] < 1e-9
    assert np.array_equal(got["tok"][~tie], ref["out_tok"][~tie])
