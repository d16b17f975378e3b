"""Run one spdm launch configuration for ncu (no timing printed: profiler runs are not bench numbers).

    python tools/prof_one.py --s 0.99 --kernel tacc_v4 --launches 2
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8000)
ap.add_argument("--s", type=float, default=0.99)
ap.add_argument("--kernel", default="auto")
ap.add_argument("--launches", type=int, default=2)
args = ap.parse_args()
n = args.n
b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).cuda()
d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, args.s, 1)).cuda(), 4)
c = torch.empty((n, n), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
G.force_kernel(args.kernel)
for _ in range(args.launches):
    G.spdm_gcoo_dev(d, b, c)
torch.cuda.synchronize()
print("done", args)
