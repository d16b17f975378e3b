"""Run one spdm launch configuration for ncu (no timing printed: profiler runs are not bench numbers).

    python tools/prof_one.py --s 0.99 --kernel tacc28_k200 --launches 2 [--powerlaw] [--n 8000]
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
ap.add_argument("--powerlaw", action="store_true")
args = ap.parse_args()
n = args.n if not (args.powerlaw and args.n == 8000) else 16384  # configs[3] is n=16384
if args.powerlaw:
    v, r, c = G.generate_powerlaw_coo(n, args.s, 1.0, 1)
    d = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).cuda(), torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda(), 4)
    b = 1.0 - torch.rand((n, n), device="cuda")
else:
    b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).cuda()
    d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, args.s, 1)).cuda(), 4)
c = torch.empty((n, n), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
G.force_kernel(args.kernel)
for _ in range(args.launches):
    G.spdm_gcoo_dev(d, b, c)
torch.cuda.synchronize()
print("done", args)
