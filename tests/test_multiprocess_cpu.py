"""Multi-process host logic of the batch-sharded path on CPU (gloo, world_size 2): shard
ranges, seq_base and the gather reproduce the single-process result bit for bit.  The device
kernels are not run here (no GPU); each rank evaluates its shard with the fp64 oracle, which
follows the same Philox counter convention (DESIGN R12), so this pins the sharding contract
the GPU path relies on (the GPU side is pinned by test_gpu_parity.test_determinism_and_batch_split)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_24328_b200.shard import gather_rows, shard_range, weak_range


def test_shard_ranges_cover():
    for total in (0, 1, 7, 80, 81):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
    assert weak_range(80, 3) == (240, 320)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import oracle
    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, k, V = 6, 3, 257
    b0, b1 = shard_range(B, world, rank)
    x = synth.make_inputs(b1 - b0, k, V, "f32", seed=99, seq_ids=np.arange(b0, b1))
    D, T = synth.to_f64(x["D"], "f32"), synth.to_f64(x["T"], "f32")
    gam = np.full(b1 - b0, k, dtype=np.int32)
    r = oracle.verify(D, T, x["tok"], gam, seed=5, offset=7, seq_base=b0, nthreads=1)
    mine = torch.from_numpy(np.stack([r["n_accept"], r["out_tok"]], axis=1).astype(np.int64))
    full = gather_rows(mine, B)
    if rank == 0:
        torch.save(full, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_batch_sharded_gloo_matches_single_process(tmp_path):
    import oracle
    import synth
    out = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = torch.load(out)
    B, k, V = 6, 3, 257
    x = synth.make_inputs(B, k, V, "f32", seed=99)
    r = oracle.verify(synth.to_f64(x["D"], "f32"), synth.to_f64(x["T"], "f32"), x["tok"], np.full(B, k, np.int32),
                      seed=5, offset=7, seq_base=0, nthreads=1)
    want = np.stack([r["n_accept"], r["out_tok"]], axis=1)
    assert np.array_equal(got.numpy(), want)
