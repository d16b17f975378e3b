"""World-size-2 `gloo` test of the column-sharded multi-rank path (CPU only).

Each rank multiplies its column block of B with the CPU checker (the product
kernel is covered by tests/test_gpu_parity.py::test_strided_column_shards_
bitwise_equal); the blocks are gathered and must equal the single-shot C bit
for bit, and the max-over-ranks timing reduction must pick the slowest rank —
the two pieces of logic bench.py relies on for N > 1.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_14469_b200.shard import column_shards, gather_columns, weak_block


def test_column_shards_partition():
    for n, w in [(8000, 1), (8000, 2), (8000, 3), (8000, 8), (130, 4), (64, 8), (0, 2), (32768, 8)]:
        sh = column_shards(n, w)
        assert len(sh) == w
        assert sh[0][0] == 0 and sh[-1][1] == n
        for (a, b), (c, _) in zip(sh, sh[1:]):
            assert b == c and a <= b
        for lo, _ in sh:
            assert lo % 64 == 0 or lo == n
    assert weak_block(8000, 3) == (24000, 32000)
    with pytest.raises(ValueError):
        column_shards(10, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle
        O = Oracle()
        rng = np.random.default_rng(7)
        m, k, n = 96, 80, 200
        a = np.where(rng.random((m, k)) < 0.1, 1.0 - rng.random((m, k)), 0.0).astype(np.float32)
        b = (1.0 - rng.random((k, n))).astype(np.float32)
        g = O.dense_to_gcoo(a, 4)
        lo, hi = column_shards(n, world)[rank]
        c_loc, _ = O.spdm(g, np.ascontiguousarray(b[:, lo:hi]), 64, fma=True)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, c_loc))
        # the optional C gather (point to point onto rank 0) reassembles the same bits
        gathered = gather_columns(torch.from_numpy(c_loc), column_shards(n, world), root=0)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            full, _ = O.spdm(g, b, 64, fma=True)
            c = np.concatenate([p[2] for p in sorted(parts, key=lambda x: x[0])], axis=1)
            q.put((bool(np.array_equal(c, full)) and bool(np.array_equal(gathered.numpy(), full)),
                   float(t.item())))
        else:
            assert gathered is None
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_column_shards_bitwise_equal():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    same, tmax = q.get(timeout=5)
    assert same
    assert tmax == 2.0
