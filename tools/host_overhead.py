"""Host-side cost of one multiply call (the time the CPU needs to enqueue it).

The device is held busy by a long torch.cuda._sleep so that every call below
only enqueues work; wall time per call = host overhead (ctypes, planner
buffer allocation, tensor-map encode, ~10 kernel launches).  If it exceeds the
device time of a step, back-to-back calls become host-bound.

    python tools/host_overhead.py [--n 8000] [--s 0.99] [--calls 50]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--s", type=float, default=0.99)
    ap.add_argument("--calls", type=int, default=20)
    args = ap.parse_args()
    n, dev = args.n, torch.device("cuda")
    d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, args.s, 1)).to(dev), 4)
    b = torch.rand((n, n), device=dev)
    c = torch.empty((n, n), device=dev)
    st = torch.cuda.Stream()
    plan = G.SpdmPlan(d, stream=st)
    for _ in range(3):
        G.spdm_gcoo_dev(d, b, c, stream=st)
        plan.run(b, c, stream=st)
    torch.cuda.synchronize()

    def per_call(fn):
        with torch.cuda.stream(st):
            torch.cuda._sleep(int(2e8))  # ~0.1 s of device time: every call below only enqueues
            t0 = time.perf_counter()
            for _ in range(args.calls):
                fn()
            t1 = time.perf_counter()
        torch.cuda.synchronize()
        return (t1 - t0) / args.calls * 1e6

    x = torch.empty(1 << 20, device=dev)
    # each probe in its own sleep window, well below the launch-queue depth
    out = {"n": n, "s": args.s, "calls": args.calls}
    for name, fn in (("spdm_gcoo_dev_us", lambda: G.spdm_gcoo_dev(d, b, c, stream=st)),
                     ("plan_run_us", lambda: plan.run(b, c, stream=st)),
                     ("torch_zero_us", lambda: x.zero_())):
        out[name] = round(min(per_call(fn) for _ in range(3)), 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
