"""Step and kernel times of the TMEM multiply with one CTA per tile against one
persistent CTA per SM walking the tiles (gcoo_debug_persistent), n=8000
reference inputs and configs[3]; C compared bit for bit between the modes.

    python tools/persist_ab.py [--s 0.9 0.99 ...] [--powerlaw]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def timed(d, b, c, st, flush, reps, events):
    with torch.cuda.stream(st):
        for _ in range(3):
            G.spdm_gcoo_dev(d, b, c, stream=st)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        G.kernel_timing(events)
        torch.cuda._sleep(int(1e7))
        for e0, e1 in evs:
            flush.zero_()
            e0.record(st)
            G.spdm_gcoo_dev(d, b, c, stream=st)
            e1.record(st)
    torch.cuda.synchronize()
    k_ms, k_n = G.kernel_time()
    G.kernel_timing(False)
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in evs])), k_ms / max(k_n, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--s", type=float, nargs="+", default=[0.9, 0.95, 0.98, 0.99, 0.995, 0.998, 0.999])
    ap.add_argument("--powerlaw", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    n = 16384 if args.powerlaw and args.n == 8000 else args.n
    dev = torch.device("cuda")
    st = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    if args.powerlaw:
        b = 1.0 - torch.rand((n, n), device=dev)
    else:
        b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).to(dev)
    c = torch.empty((n, n), dtype=torch.float32, device=dev)
    for s in args.s:
        if args.powerlaw:
            v, r, cc = G.generate_powerlaw_coo(n, s, 1.0, 1)
            d = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                  torch.from_numpy(cc).to(dev), 4)
        else:
            d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, s, 1)).to(dev), 4)
        out = {"n": n, "s": s, "powerlaw": args.powerlaw}
        ref = None
        for mode in ("per_tile", "persistent", "per_tile", "persistent"):
            G.persistent(mode == "persistent")
            ms, _ = timed(d, b, c, st, flush, args.reps, False)
            _, kms = timed(d, b, c, st, flush, max(5, args.reps // 4), True)
            out.setdefault(mode + "_ms", []).append(round(ms, 4))
            out.setdefault(mode + "_kernel_ms", []).append(round(kms, 4))
            if ref is None:
                ref = c.clone()
            else:
                out[mode + "_bit_equal"] = bool(torch.equal(c, ref))
        G.persistent(False)
        out["kernel"] = G.last_kernel()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
