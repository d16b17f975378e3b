"""Time every fp32 multiply kernel variant on the n=8000 benchmark inputs.

    python tools/kernel_sweep.py [--n 8000] [--s 0.9 0.99 0.995] [--kernels ...]

Kernel-only CUDA-event times (L2 flushed before each launch), one JSON line per
(kernel, sparsity), plus a bit-exactness check of each variant's C against the
first variant's.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--s", type=float, nargs="+", default=[0.9, 0.99, 0.995])
    ap.add_argument("--kernels", nargs="+", default=["auto", "tacc28_k200", "tacc28_k192", "tacc28_k160", "tacc28_k128",
                                                       "tacc28_k96", "tacc28_k64", "tacc_v4_k216", "rowtile"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--powerlaw", action="store_true", help="BASELINE configs[3]: power-law A (n=16384 default)")
    args = ap.parse_args()
    if args.powerlaw and args.n == 8000:
        args.n = 16384
    n = args.n
    dev = torch.device("cuda")
    if args.powerlaw:
        b = 1.0 - torch.rand((n, n), device=dev, dtype=torch.float32, generator=torch.Generator(device=dev).manual_seed(1))
    else:
        b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).to(dev)
    c = torch.empty((n, n), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()
    for s in args.s:
        if args.powerlaw:
            v, r, cc = G.generate_powerlaw_coo(n, s, 1.0, 1)
            d = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                  torch.from_numpy(cc).to(dev), 4)
        else:
            d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, s, 1)).to(dev), 4)
        torch.cuda.synchronize()
        ref = None
        for kname in args.kernels:
            G.force_kernel(kname)
            with torch.cuda.stream(st):
                for _ in range(3):
                    G.spdm_gcoo_dev(d, b, c, stream=st)
                def reps(kernel_events):
                    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                           for _ in range(args.reps)]
                    G.kernel_timing(kernel_events)
                    torch.cuda._sleep(int(1e7))  # host queues the reps ahead of the device
                    for e0, e1 in evs:  # back to back (no host sync between reps), L2 flushed before each
                        flush.zero_()
                        e0.record(st)
                        G.spdm_gcoo_dev(d, b, c, stream=st)
                        e1.record(st)
                    torch.cuda.synchronize()
                    out = [e0.elapsed_time(e1) for e0, e1 in evs], G.kernel_time()
                    G.kernel_timing(False)
                    return out

                # step times without the kernel-timing events (they sit inside the
                # planner -> multiply PDL chain), the multiply's own time from a second pass
                ts, _ = reps(False)
                _, (k_ms, k_n) = reps(True)
            out = c.clone()
            same = None if ref is None else bool(torch.equal(out, ref))
            if ref is None:
                ref = out
            ms = float(np.median(ts))
            fl = 2.0 * d.nnz() * n
            print(json.dumps({"s": s, "kernel": kname, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 3),
                              "min_ms": round(min(ts), 4), "kernel_ms": round(k_ms / max(k_n, 1), 4), "bitwise_equal_first": same, "all_ms": [round(t, 3) for t in ts]}), flush=True)
        G.force_kernel("auto")


if __name__ == "__main__":
    main()
