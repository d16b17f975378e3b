"""A few small launches of every kernel family for compute-sanitizer
(memcheck / racecheck): the TMEM multiply (two-entry, three-entry, fp64
records, a two-class split), the row-tile kernel, the planner/constructors and
the baselines (row-split CSR, ungrouped COO with an unsorted input, dense
GEMM).  Checks C against the one-shot row-tile result so a sanitizer run is
also a parity run.

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    dev = torch.device("cuda")
    m, k, n = 1100, 1300, 640
    for dens, kern in ((0.01, "tacc28_k200"), (0.05, "tacc28_k160"), (0.004, "tacc_v4_k216"), (0.3, "tacc28_k64")):
        a = np.where(rng.random((m, k)) < dens, 1 - rng.random((m, k)), 0).astype(np.float32)
        b = (1 - rng.random((k, n))).astype(np.float32)
        d = G.dense_to_gcoo_dev(torch.from_numpy(a).to(dev), 4)
        c1 = torch.empty((m, n), device=dev)
        c2 = torch.empty((m, n), device=dev)
        G.force_kernel(kern)
        G.spdm_gcoo_dev(d, torch.from_numpy(b).to(dev), c1)
        G.force_kernel("rowtile")
        G.spdm_gcoo_dev(d, torch.from_numpy(b).to(dev), c2)
        G.force_kernel("auto")
        torch.cuda.synchronize()
        assert torch.equal(c1, c2), kern
        # baselines on the same operands
        r, cc = np.nonzero(a)
        v = a[r, cc]
        rp = np.concatenate([[0], np.cumsum(np.count_nonzero(a, axis=1))]).astype(np.int64)
        assert np.array_equal(G.spdm_csr(m, k, v, cc, rp, b), c2.cpu().numpy())
        perm = rng.permutation(r.size)
        G.spdm_coo(m, k, v[perm], r[perm], cc[perm], b)
        G.gemm_dense_blocked(a[:200, :300].copy(), b[:300, :100].copy())
    # two-class split (above the small-product gate, so the TMEM kernels run)
    ms, ks = 2000, 2000
    a = np.where(rng.random((ms, ks)) < 0.004, 1 - rng.random((ms, ks)), 0).astype(np.float32)
    a[::97] = (1 - rng.random((len(a[::97]), ks))).astype(np.float32)
    b = (1 - rng.random((ks, 4096))).astype(np.float32)
    d = G.dense_to_gcoo_dev(torch.from_numpy(a).to(dev), 4)
    c1 = torch.empty((ms, 4096), device=dev)
    c2 = torch.empty((ms, 4096), device=dev)
    G.force_split("always")
    G.spdm_gcoo_dev(d, torch.from_numpy(b).to(dev), c1)
    split = G.last_split()
    G.force_split("auto")
    G.force_kernel("rowtile")
    G.spdm_gcoo_dev(d, torch.from_numpy(b).to(dev), c2)
    G.force_kernel("auto")
    torch.cuda.synchronize()
    assert split and torch.equal(c1, c2)
    # fp64 TMEM kernel
    a = np.where(rng.random((m, k)) < 0.02, 1 - rng.random((m, k)), 0)
    b = 1 - rng.random((k, n))
    d = G.dense_to_gcoo_dev(torch.from_numpy(a).to(dev), 4)
    c1 = torch.empty((m, n), device=dev, dtype=torch.float64)
    G.force_kernel("tacc28_f64_k160")
    G.spdm_gcoo_dev(d, torch.from_numpy(b).to(dev), c1)
    G.force_kernel("auto")
    torch.cuda.synchronize()
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
