"""BASELINE configs[2]: sparsity sweep at n = 2000..14000, uniform random A
(the reference's sweep() seeds, bench.hpp:216-231, bit-identical inputs), and
the crossover against dense-equivalent FLOPs — the smallest sparsity at which
the GCOO multiply beats a dense FP32 GEMM of the same shape
(crossover_search, bench.hpp:272-299).  The dense yardstick is cuBLAS SGEMM
with TF32 off (torch.mm); the paper's sparse yardstick is cuSPARSE CSR SpMM
(torch.sparse.mm on a CSR tensor, the timed region includes copying its
output into a preallocated C).  Both are measurement only, never on the
product path.

    python tools/sweep_crossover.py > profiles/rNN_sweep_crossover.jsonl

One JSON line per (n, s): step time (planner + multiply, device-resident, L2
flushed before every launch), kernel-only time, GFLOPS (2*nnz*N), EO time
(dense -> GCOO on the GPU), dense SGEMM time; then one line per n with the
crossover sparsity.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402


def realized_sparsity(n, s):
    return 1.0 - round((1.0 - s) * n * n) / float(n * n)


def timed(fn, reps, flush, st):
    with torch.cuda.stream(st):
        for _ in range(2):
            flush.zero_()
            fn()
        torch.cuda.synchronize()
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
    ap.add_argument("--sizes", type=int, nargs="+", default=[2000, 4000, 8000, 14000])
    ap.add_argument("--s", type=float, nargs="+", default=[0.8, 0.9, 0.95, 0.98, 0.99, 0.995, 0.999])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda")
    st = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for n in args.sizes:
        dense_ms = None
        cross = None
        for s in args.s:
            rs = realized_sparsity(n, s)
            a_seed = G.derive_seed(args.seed, n, int(round((1.0 - rs) * n * n)))
            a = torch.from_numpy(G.generate_uniform_sparse(n, s, a_seed)).to(dev)
            b = torch.from_numpy(G.generate_uniform_sparse(n, 0.0, G.derive_seed(a_seed, n, 0xB))).to(dev)
            c = torch.empty((n, n), dtype=torch.float32, device=dev)
            torch.cuda.synchronize()
            eo_ms = timed(lambda: G.dense_to_gcoo_dev(a, 4, stream=st), 3, flush, st)
            d = G.dense_to_gcoo_dev(a, 4)
            torch.cuda.synchronize()
            G.kernel_timing(True)
            ms = timed(lambda: G.spdm_gcoo_dev(d, b, c, stream=st), args.reps, flush, st)
            k_ms, k_n = G.kernel_time()
            G.kernel_timing(False)
            # the paper's comparison: cuSPARSE CSR SpMM (torch.sparse.mm on a CSR
            # tensor) on the same operands — a yardstick, never the product path
            csr = a.to_sparse_csr()
            cc = torch.empty_like(c)
            try:
                cusparse_ms = timed(lambda: cc.copy_(torch.sparse.mm(csr, b)), args.reps, flush, st)
                same = bool(torch.allclose(cc, c, rtol=1e-5, atol=1e-6))
            except RuntimeError as e:  # noqa: F841
                cusparse_ms, same = None, None
            del csr, cc
            if dense_ms is None:  # the dense time does not depend on the values
                cd = torch.empty_like(c)
                dense_ms = timed(lambda: torch.mm(a, b, out=cd), args.reps, flush, st)
                del cd
            nnz = d.nnz()
            fl = 2.0 * nnz * n
            row = {"n": n, "s": s, "realized_s": rs, "nnz": nnz, "ms": round(ms, 4),
                   "kernel_ms": round(k_ms / max(k_n, 1), 4), "gflops": round(fl / ms / 1e6, 1),
                   "eo_ms": round(eo_ms, 4), "dense_sgemm_ms": round(dense_ms, 4),
                   "dense_sgemm_tflops": round(2.0 * n ** 3 / dense_ms / 1e9, 2),
                   "speedup_vs_dense": round(dense_ms / ms, 3),
                   "cusparse_csr_ms": None if cusparse_ms is None else round(cusparse_ms, 4),
                   "speedup_vs_cusparse": None if cusparse_ms is None else round(cusparse_ms / ms, 3),
                   "cusparse_matches_1e-5": same}
            print(json.dumps(row), flush=True)
            if cross is None and ms < dense_ms:
                cross = s
            del a, b, c, d
            torch.cuda.empty_cache()
        print(json.dumps({"n": n, "crossover_s": cross, "dense_sgemm_ms": round(dense_ms, 4),
                          "rule": "smallest s on the grid with GCOO step < dense SGEMM (crossover_search)"}),
              flush=True)


if __name__ == "__main__":
    main()
