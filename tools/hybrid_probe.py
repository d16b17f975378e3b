"""Would a two-class (heavy rows / light rows) split help configs[3]?  Times
the power-law product's heavy rows and light rows as two separate products
(compacted row sets, each with its own configuration), one after the other and
concurrently on two streams, against the one-shot product.

    python tools/hybrid_probe.py [--heavy 504] [--kh tacc28_k96] [--kl auto]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def timed(fn, reps=5, flush=None):
    evs = []
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--heavy", type=int, nargs="+", default=[504])
    ap.add_argument("--kh", nargs="+", default=["tacc28_k96"])
    ap.add_argument("--kl", nargs="+", default=["auto"])
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda")
    v, r, c = G.generate_powerlaw_coo(n, 0.99, 1.0, 1)
    deg = np.bincount(r, minlength=n)
    order = np.argsort(-deg, kind="stable")
    b = 1.0 - torch.rand((n, n), device=dev)
    flush = torch.empty(64 << 20, device=dev)
    full = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                             torch.from_numpy(c).to(dev), 4)
    cfull = torch.empty((n, n), device=dev)
    t_full = timed(lambda: G.spdm_gcoo_dev(full, b, cfull), flush=flush)
    print(json.dumps({"one_shot_ms": round(t_full, 3), "kernel": G.last_kernel()}), flush=True)
    for H in args.heavy:
        heavy_rows = np.sort(order[:H])
        is_h = np.zeros(n, bool)
        is_h[heavy_rows] = True
        newidx = np.empty(n, np.int64)
        newidx[heavy_rows] = np.arange(H)
        light_rows = np.sort(order[H:])
        newidx[light_rows] = np.arange(n - H)

        def sub(mask, rows_count):
            sel = mask[r]
            rr = newidx[r[sel]].astype(np.int32)
            o = np.lexsort((c[sel], rr))
            return G.coo_to_gcoo_dev(rows_count, n, torch.from_numpy(v[sel][o]).to(dev), torch.from_numpy(rr[o]).to(dev),
                                     torch.from_numpy(c[sel][o]).to(dev), 4)
        gh, gl = sub(is_h, H), sub(~is_h, n - H)
        ch = torch.empty((H, n), device=dev)
        cl = torch.empty((n - H, n), device=dev)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        for kh in args.kh:
            for kl in args.kl:
                def both_seq():
                    G.force_kernel(kh)
                    G.spdm_gcoo_dev(gh, b, ch)
                    G.force_kernel(kl)
                    G.spdm_gcoo_dev(gl, b, cl)

                def both_conc():
                    ev = torch.cuda.Event()
                    ev.record()
                    s1.wait_event(ev)
                    s2.wait_event(ev)
                    G.force_kernel(kh)
                    G.spdm_gcoo_dev(gh, b, ch, stream=s1)
                    G.force_kernel(kl)
                    G.spdm_gcoo_dev(gl, b, cl, stream=s2)
                    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
                    e1.record(s1)
                    e2.record(s2)
                    torch.cuda.current_stream().wait_event(e1)
                    torch.cuda.current_stream().wait_event(e2)
                G.force_kernel(kh)
                th = timed(lambda: G.spdm_gcoo_dev(gh, b, ch), flush=flush)
                G.force_kernel(kl)
                tl = timed(lambda: G.spdm_gcoo_dev(gl, b, cl), flush=flush)
                ts = timed(both_seq, flush=flush)
                tc = timed(both_conc, flush=flush)
                G.force_kernel("auto")
                # parity of the split against the one-shot product
                same = bool(torch.equal(cfull[torch.from_numpy(heavy_rows).to(dev)], ch)) and \
                    bool(torch.equal(cfull[torch.from_numpy(light_rows).to(dev)], cl))
                print(json.dumps({"H": H, "heavy_nnz": int(deg[heavy_rows].sum()), "kh": kh, "kl": kl,
                                  "heavy_ms": round(th, 3), "light_ms": round(tl, 3), "seq_ms": round(ts, 3),
                                  "concurrent_ms": round(tc, 3), "bitwise_equal_one_shot": same}), flush=True)


if __name__ == "__main__":
    main()
