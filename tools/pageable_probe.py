"""e2e through the host API with PAGEABLE numpy buffers (the C++ drop-in's
std::vector case): n=8000, s=0.99, median of 7 calls after 2 warm-ups, and a
bit-exact check against the pinned-buffer call.  Pool size via
GCOO_HOST_THREADS (read once per process), strip count via STRIPS
(gcoo_debug_pipeline_strips), so run once per setting."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

n = 8000
a = G.generate_uniform_sparse(n, 0.99, 1)
b = G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))
g = G.dense_to_gcoo(a, 4)
c = np.empty((n, n), np.float32)
if os.environ.get("STRIPS"):
    G.lib().gcoo_debug_pipeline_strips(int(os.environ["STRIPS"]))
for _ in range(2):
    G.spdm_gcoo(g, b, out=c)
ts = []
for _ in range(7):
    t = time.perf_counter()
    G.spdm_gcoo(g, b, out=c)
    ts.append(time.perf_counter() - t)
c_pin = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy()
b_pin = torch.empty((n, n), dtype=torch.float32, pin_memory=True).numpy()
b_pin[...] = b
G.spdm_gcoo(g, b_pin, out=c_pin)
ms = sorted(ts)[3] * 1e3
print(json.dumps({"threads": os.environ.get("GCOO_HOST_THREADS", "default"), "strips": os.environ.get("STRIPS", "default"), "pageable_ms": round(ms, 3),
                  "gflops": round(2 * g.nnz() * n / ms / 1e6, 1), "all_ms": [round(x * 1e3, 2) for x in ts],
                  "bitwise_equal_pinned": bool(np.array_equal(c, c_pin))}), flush=True)
