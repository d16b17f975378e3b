"""Per-step device times of the bench step (planner + multiply, n=8000,
s=0.99, L2 flushed between steps) — for spotting outliers and A/B runs
(e.g. GCOO_NO_PDL=1)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

n, s = int(os.environ.get("N", 8000)), float(os.environ.get("S", 0.99))
a = G.generate_uniform_sparse(n, s, 1)
b = G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))
dg = G.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
dB = torch.from_numpy(b).cuda()
dC = torch.empty((n, n), device="cuda")
flush = torch.empty(64 << 20, device="cuda")
st = torch.cuda.Stream()
timing = os.environ.get("KT", "0") == "1"
with torch.cuda.stream(st):
    for _ in range(3):
        flush.zero_()
        G.spdm_gcoo_dev(dg, dB, dC, stream=st)
    torch.cuda.synchronize()
    G.kernel_timing(timing)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    if os.environ.get("SLEEP"):
        torch.cuda._sleep(int(2e6))  # ~1 ms: the host queues ahead of the device
    import time
    cpu = []
    for e0, e1 in ev:
        t0 = time.perf_counter()
        flush.zero_()
        e0.record(st)
        G.spdm_gcoo_dev(dg, dB, dC, stream=st)
        e1.record(st)
        cpu.append(round((time.perf_counter() - t0) * 1e3, 3))
    torch.cuda.synchronize()
    G.kernel_timing(False)
print("pdl_off" if os.environ.get("GCOO_NO_PDL") else "pdl_on", "kt" if timing else "",
      [round(e0.elapsed_time(e1), 4) for e0, e1 in ev], "cpu ms", cpu[:5])
