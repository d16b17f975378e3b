"""World-size-2 runs of the PRODUCT's column-sharded path on one GPU (gloo
for the plumbing: the driver's boxes give this suite a single GPU).

* each rank multiplies its column shard of B with the CUDA kernel
  (spdm_gcoo_dev on a strided view), the shards are gathered onto rank 0 with
  shard.gather_columns and must equal the oracle's single-shot C bit for bit;
* bench.strong_scaling (the configs[4] block of every SCALE line) runs end to
  end at a reduced n: A built on rank 0 and broadcast, per-rank shard timing,
  t1 on rank 0, sampled-row parity against the 1-GPU product, the C gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q, mode):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch.distributed as dist
    import paper_2005_14469_b200 as G
    from paper_2005_14469_b200.shard import column_shards, gather_columns
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    try:
        if mode == "shards":
            dist.init_process_group("gloo", rank=rank, world_size=world)
            from oracle import Oracle
            O = Oracle()
            rng = np.random.default_rng(7)
            m, k, n = 4000, 4000, 2048  # each 1024-column shard is a 0.66 GFLOP product: the TMEM kernel
            a = np.where(rng.random((m, k)) < 0.02, 1.0 - rng.random((m, k)), 0.0).astype(np.float32)
            b = (1.0 - rng.random((k, n))).astype(np.float32)
            dg = G.dense_to_gcoo_dev(torch.from_numpy(a).to(dev), 4)
            lo, hi = column_shards(n, world)[rank]
            dB = torch.from_numpy(b).to(dev)
            dC = torch.empty((m, hi - lo), dtype=torch.float32, device=dev)
            G.spdm_gcoo_dev(dg, dB[:, lo:hi], dC)   # the product kernel on a strided shard
            torch.cuda.synchronize()
            kern = G.last_kernel()
            full = gather_columns(dC.cpu(), column_shards(n, world), root=0)
            if rank == 0:
                ref, _ = O.spdm(O.dense_to_gcoo(a, 4), b, 64, fma=True)
                q.put((bool(np.array_equal(full.numpy(), ref)), kern))
            else:
                assert full is None
            dist.destroy_process_group()
        else:
            import bench
            D = bench.Dist(world, rank, dev, ndev=1)  # two ranks, one GPU -> gloo
            flush = torch.empty(1 << 20, dtype=torch.float32, device=dev)
            stream = torch.cuda.Stream(device=dev)
            out = bench.strong_scaling(G, D, dev, stream, flush, steps=2, warmup=1, n=4096)
            if rank == 0:
                q.put(out)
            D.barrier()
            D.dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put(("error", rank, repr(e)))
        raise


def _run(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = q.get(timeout=5)
    assert all(p.exitcode == 0 for p in procs), res
    return res


def test_two_rank_product_shards_bitwise_equal(cuda):
    same, kern = _run("shards")
    assert same
    assert kern.startswith("tacc"), kern


def test_two_rank_strong_scaling_block(cuda):
    out = _run("strong")
    assert isinstance(out, dict), out
    assert out["parity_sampled_rows_equal_1gpu"] is True
    assert out["c_gather"]["equals_1gpu"] is True
    assert out["shards"] == [[0, 2048], [2048, 4096]]
    assert out["t1_ms"] > 0 and out["tN_ms"] > 0 and out["speedup"] > 0
