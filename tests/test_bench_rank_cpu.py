"""bench.py's multi-GPU rank logic on CPU (gloo, world size 2 and 3): the strong-scaling split of
the global batch of 80 (BASELINE config 3), seq_base, the max-over-ranks timing and the gather
of per-sequence outputs -- the same functions bench.py runs under torchrun with NCCL.  Each rank
evaluates its shard with the fp64 oracle (no GPU here); gathered outputs must equal one process
over the whole batch bit for bit (the Philox counter carries the global sequence id, R12)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

B_GLOBAL, K, V = 80, 3, 129


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _outputs(b0, b1):
    import oracle
    import synth
    x = synth.make_inputs(b1 - b0, K, V, "f32", seed=0x5EED, seq_ids=np.arange(b0, b1))
    Dd, Cd, Td = (synth.to_f64(x[n], "f32") for n in ("D", "C", "T"))
    rs = oracle.score(Dd, Cd, x["tok"], 1.0, 1.0, synth.load_profile(), nthreads=1)
    rh = oracle.schedule(rs["p_hat"], synth.latency_table(K + 2))
    rv = oracle.verify(Dd, Td, x["tok"], rh["gamma"], 1.0, 1.0, 0xC0FFEE, 11, b0, nthreads=1)
    return {"gamma": torch.from_numpy(rh["gamma"].astype(np.int64)),
            "n_accept": torch.from_numpy(rv["n_accept"].astype(np.int64)),
            "out_tok": torch.from_numpy(rv["out_tok"].astype(np.int64)),
            "p_hat": torch.from_numpy(rs["p_hat"])}


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench
    r, w = bench.init_dist("gloo")
    assert (r, w) == (rank, world) and dist.get_backend() == "gloo"
    b0, b1 = bench.rank_plan(B_GLOBAL, w, r, "strong")
    mine = _outputs(b0, b1)
    slowest = bench.max_over_ranks(float(10 + rank))  # a per-rank "time"
    got = bench.gather_outputs(mine, B_GLOBAL)
    if rank == 0:
        torch.save({"got": got, "slowest": slowest, "spans": [bench.rank_plan(B_GLOBAL, w, q) for q in range(w)]},
                   out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_bench_strong_split_gloo_matches_world_1(tmp_path, world):
    import bench
    out = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = torch.load(out)
    assert res["slowest"] == 10.0 + world - 1
    spans = res["spans"]
    assert spans[0][0] == 0 and spans[-1][1] == B_GLOBAL and all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    want = _outputs(0, B_GLOBAL)
    for n, v in want.items():
        assert torch.equal(res["got"][n], v), n
    # world 1: the same helpers are identities (no process group)
    assert bench.rank_plan(B_GLOBAL, 1, 0) == (0, B_GLOBAL) and bench.max_over_ranks(3.5) == 3.5
    assert bench.rank_plan(B_GLOBAL, world, world - 1, "weak") == ((world - 1) * 80, world * 80)
