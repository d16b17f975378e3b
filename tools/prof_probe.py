"""Cycle accounting of the TMEM multiply kernel (a GCOO_PROF=1 measurement
build, never the product): where consumer warps spend their chunk loop —
waiting for a stage (full barrier) vs consuming records — and how long the
producer waits for stage releases.

    python tools/prof_probe.py [--s 0.99 0.995] [--powerlaw] [--kernel auto]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANT = os.environ.get("GCOO_PROF_LIB", os.path.join(ROOT, "tools", "_abl", "libgcoo_prof.so"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=float, nargs="+", default=[0.99, 0.995])
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--kernel", nargs="+", default=["auto"])
    ap.add_argument("--powerlaw", action="store_true")
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--persistent", action="store_true", help="one persistent CTA per SM (even A)")
    args = ap.parse_args()
    if args.build:
        from paper_2005_14469_b200 import build
        os.makedirs(os.path.dirname(VARIANT), exist_ok=True)
        build.build(out=VARIANT, defines=["GCOO_PROF=1"])
        return
    os.environ["GCOO_LIB"] = VARIANT
    import torch
    import paper_2005_14469_b200 as G
    L = G.lib()
    if args.persistent:
        G.persistent(True)
    L.gcoo_debug_prof.restype = C.c_int
    L.gcoo_debug_prof.argtypes = [C.c_void_p, C.c_int]
    buf = (C.c_ulonglong * 12)()
    n = args.n if not args.powerlaw or args.n != 8000 else 16384
    dev = torch.device("cuda")
    if args.powerlaw:
        b = 1.0 - torch.rand((n, n), device=dev)
    else:
        b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).to(dev)
    c = torch.empty((n, n), device=dev)
    for s in args.s:
        if args.powerlaw:
            v, r, cc = G.generate_powerlaw_coo(n, s, 1.0, 1)
            d = G.coo_to_gcoo_dev(n, n, torch.from_numpy(v).to(dev), torch.from_numpy(r).to(dev),
                                  torch.from_numpy(cc).to(dev), 4)
        else:
            d = G.dense_to_gcoo_dev(torch.from_numpy(G.generate_uniform_sparse(n, s, 1)).to(dev), 4)
        for k in args.kernel:
            G.force_kernel(k)
            G.spdm_gcoo_dev(d, b, c)
            L.gcoo_debug_prof(buf, 1)
            G.spdm_gcoo_dev(d, b, c)
            torch.cuda.synchronize()
            L.gcoo_debug_prof(buf, 1)
            w, tot, epi, pw, ptot, warps, recs, swaps, hcyc, hwarps, mx, _ = list(buf)
            print(json.dumps({"s": s, "n": n, "powerlaw": args.powerlaw, "kernel": G.last_kernel(),
                              "consumer_wait_frac": round(w / max(tot, 1), 4),
                              "consumer_loop_cycles_per_warp": round(tot / max(warps, 1)),
                              "epilogue_frac": round(epi / max(tot + epi, 1), 4),
                              "producer_wait_frac": round(pw / max(ptot, 1), 4),
                              "records": recs, "swaps": swaps, "consumer_warps": warps,
                              "heavy_rb_warps": hwarps, "heavy_rb_loop_cycles_per_warp": round(hcyc / max(hwarps, 1)),
                              "light_loop_cycles_per_warp": round((tot - hcyc) / max(warps - hwarps, 1)),
                              "max_loop_cycles": mx}), flush=True)
        G.force_kernel("auto")


if __name__ == "__main__":
    main()
