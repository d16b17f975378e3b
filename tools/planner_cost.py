"""Planner cost (step with planning minus the multiply with a reused plan) as
the GCOO group size p grows, and on configs[3] (power-law, two-class split).

    python tools/planner_cost.py [--n 8000] [--s 0.99] [--p 4 16 64 256 1024]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def med(fn, st, flush, reps):
    with torch.cuda.stream(st):
        for _ in range(2):
            fn()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        torch.cuda._sleep(int(1e7))
        for e0, e1 in evs:
            flush.zero_()
            e0.record(st)
            fn()
            e1.record(st)
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--s", type=float, default=0.99)
    ap.add_argument("--p", type=int, nargs="+", default=[4, 16, 64, 256, 1024])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--powerlaw", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda")
    st = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    n = 16384 if args.powerlaw and args.n == 8000 else args.n
    if args.powerlaw:
        v, r, c = G.generate_powerlaw_coo(n, args.s, 1.0, 1)
        b = 1.0 - torch.rand((n, n), device=dev)
    else:
        a = torch.from_numpy(G.generate_uniform_sparse(n, args.s, 1)).to(dev)
        b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).to(dev)
    out_c = torch.empty((n, n), dtype=torch.float32, device=dev)
    ref = None
    for p in args.p:
        if args.powerlaw:
            d = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                  torch.from_numpy(c).to(dev), p)
        else:
            d = G.dense_to_gcoo_dev(a, p)
        step = med(lambda: G.spdm_gcoo_dev(d, b, out_c, G.ExecConfig(p=p), stream=st), st, flush, args.reps)
        res = out_c.clone()
        plan = G.SpdmPlan(d, stream=st)
        mult = med(lambda: plan.run(b, out_c, stream=st), st, flush, args.reps)
        plan.close()
        same = None if ref is None else bool(torch.equal(res, ref))
        ref = res if ref is None else ref
        print(json.dumps({"n": n, "s": args.s, "powerlaw": args.powerlaw, "p": p, "step_ms": round(step, 4),
                          "multiply_ms": round(mult, 4), "planner_ms": round(step - mult, 4),
                          "kernel": G.last_kernel(), "C_equal_p_first": same}), flush=True)


if __name__ == "__main__":
    main()
