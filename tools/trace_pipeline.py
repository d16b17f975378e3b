"""Timeline of one host-pointer spdm_gcoo call (n=8000, s=0.99) with
GCOO_TRACE_PIPELINE=1: per strip, when its H2D copy, multiply and D2H copy end."""
import os
import sys

os.environ["GCOO_TRACE_PIPELINE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

n = 8000
a = G.generate_uniform_sparse(n, 0.99, 1)
b = G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))
g = G.dense_to_gcoo(a, 4)


def pin(arr):
    t_ = torch.empty(arr.shape, dtype=getattr(torch, str(arr.dtype)), pin_memory=True)
    t_.numpy()[...] = arr
    return t_.numpy()


gp = G.GcooMatrix(g.rows_dim, g.cols_dim, g.p, pin(g.values), pin(g.row_idx), pin(g.col_idx), pin(g.g_idxes),
                  pin(g.nnz_per_group))
bp, cp = pin(b), pin(np.empty((n, n), np.float32))
for _ in range(3):
    G.spdm_gcoo(gp, bp, out=cp)
