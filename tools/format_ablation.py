"""The paper's format ablation on the B200: GCOO against the
reference's own comparison kernels — row-split CSR (kernels.hpp:163-184),
ungrouped COO (kernels.hpp:193-232) and the dense blocked GEMM
(kernels.hpp:107-155) — each as this repository's sm_100a kernel, with
cuSPARSE CSR SpMM and cuBLAS SGEMM (TF32 off) beside them as library
yardsticks.  n=8000 reference inputs (bench.hpp:168-174), CUDA-event times per
call with the L2 flushed before each, one JSON line per sparsity; the four own
kernels' C are compared bit for bit (every one runs each C element's chain in
ascending column order, so they must agree exactly).

    python tools/format_ablation.py [--n 8000] [--s 0.9 0.99 ...] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def timed(fn, reps, flush, st):
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
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8000)
    ap.add_argument("--s", type=float, nargs="+", default=[0.9, 0.95, 0.98, 0.99, 0.995, 0.999])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda")
    st = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(1, n, 0xB))).to(dev)
    c = torch.empty((n, n), dtype=torch.float32, device=dev)
    torch.backends.cuda.matmul.allow_tf32 = False
    dense_ms = None
    for s in args.s:
        a_host = G.generate_uniform_sparse(n, s, 1)
        a = torch.from_numpy(a_host).to(dev)
        r, cc = np.nonzero(a_host)  # row-major: each row's entries in column order
        vals = torch.from_numpy(a_host[r, cc]).to(dev)
        rows = torch.from_numpy(r.astype(np.int32)).to(dev)
        cols = torch.from_numpy(cc.astype(np.int32)).to(dev)
        rp = torch.from_numpy(np.concatenate([[0], np.cumsum(np.count_nonzero(a_host, axis=1))]).astype(np.int64)).to(dev)
        d = G.dense_to_gcoo_dev(a, 4)
        nnz = d.nnz()
        fl = 2.0 * nnz * n
        out = {}
        res = {}
        out["gcoo_ms"] = timed(lambda: G.spdm_gcoo_dev(d, b, c, stream=st), args.reps, flush, st)
        res["gcoo"] = c.clone()
        out["csr_rowsplit_ms"] = timed(lambda: G.spdm_csr_dev(n, n, vals, cols, rp, b, c, stream=st), args.reps, flush, st)
        res["csr"] = c.clone()
        out["coo_ungrouped_ms"] = timed(lambda: G.spdm_coo_dev(n, n, vals, rows, cols, b, c, stream=st), args.reps, flush,
                                        st)
        res["coo"] = c.clone()
        if dense_ms is None:  # the dense baselines do the same work at every sparsity
            dense_ms = timed(lambda: G.gemm_dense_dev(a, b, c, stream=st), max(2, args.reps // 2), flush, st)
            res["dense"] = c.clone()
            same_dense = bool(torch.equal(res["dense"], res["gcoo"]))
            sgemm_ms = timed(lambda: torch.mm(a, b, out=c), args.reps, flush, st)
        out["dense_gemm_ms"] = dense_ms
        out["cublas_sgemm_ms"] = sgemm_ms
        acsr = a.to_sparse_csr()
        out["cusparse_csr_ms"] = timed(lambda: c.copy_(torch.sparse.mm(acsr, b)), args.reps, flush, st)
        cs = torch.sparse.mm(acsr, b)
        rel = float(((cs - res["gcoo"]).abs() / res["gcoo"].abs().clamp_min(1e-30)).max())
        line = {"n": n, "s": s, "nnz": nnz, **{k: round(v, 4) for k, v in out.items()},
                "gcoo_tflops": round(fl / out["gcoo_ms"] / 1e9, 3),
                "speedup_vs_csr_rowsplit": round(out["csr_rowsplit_ms"] / out["gcoo_ms"], 2),
                "speedup_vs_coo_ungrouped": round(out["coo_ungrouped_ms"] / out["gcoo_ms"], 2),
                "speedup_vs_dense_gemm": round(dense_ms / out["gcoo_ms"], 2),
                "speedup_vs_cusparse": round(out["cusparse_csr_ms"] / out["gcoo_ms"], 2),
                "speedup_vs_cublas": round(sgemm_ms / out["gcoo_ms"], 2),
                "csr_bit_equal_gcoo": bool(torch.equal(res["csr"], res["gcoo"])),
                "coo_bit_equal_gcoo": bool(torch.equal(res["coo"], res["gcoo"])),
                "dense_bit_equal_gcoo": same_dense if s == args.s[0] else None,
                "cusparse_max_rel": rel}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
