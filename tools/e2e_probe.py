"""e2e host-API probe: raw pinned H2D/D2H bandwidth and the pipelined
spdm_gcoo time for several strip counts (n=8000, s=0.99)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

n = 8000
x = torch.empty(n * n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n * n, dtype=torch.float32, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, "GB/s", round(5 * x.numel() * 4 / (time.perf_counter() - t) / 1e9, 1))
a = G.generate_uniform_sparse(n, 0.99, 1)
b = G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))
g = G.dense_to_gcoo(a, 4)
pin = lambda arr: (lambda t_: (t_.numpy().__setitem__(Ellipsis, arr), t_.numpy())[1])(
    torch.empty(arr.shape, dtype=getattr(torch, str(arr.dtype)), pin_memory=True))
gp = G.GcooMatrix(g.rows_dim, g.cols_dim, g.p, pin(g.values), pin(g.row_idx), pin(g.col_idx), pin(g.g_idxes),
                  pin(g.nnz_per_group))
bp = pin(b)
cp = pin(np.empty((n, n), np.float32))
for strips in [int(x) for x in os.environ.get("STRIPS", "1 8 12 16 24 32 64").split()]:
    G.lib().gcoo_debug_pipeline_strips(strips)
    G.spdm_gcoo(gp, bp, out=cp)
    ts = []
    for _ in range(7):
        t = time.perf_counter()
        G.spdm_gcoo(gp, bp, out=cp)
        ts.append(time.perf_counter() - t)
    print("strips", strips, "median ms", round(sorted(ts)[3] * 1e3, 3))
