"""Run the panel kernel from a debug build (tools/libgcoo_cuda_debug.so) on a
failing shape; the kernel printf's the first malformed staged entry."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G
G.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgcoo_cuda_debug.so")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
s = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
kern = sys.argv[3] if len(sys.argv) > 3 else "panel_tall"
b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).cuda()
d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, s, 1)).cuda(), 4)
c = torch.empty((n, n), dtype=torch.float32, device="cuda")
G.force_kernel(kern)
G.spdm_gcoo_dev(d, b, c)
torch.cuda.synchronize()
print("ok")
