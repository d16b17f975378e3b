"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

    python tests/golden/make_golden.py

Runs the unmodified reference library (oracle/_ref/libgcoo_ref{,_fma}.so,
compiled from /root/reference/proj by oracle/Makefile) on:

* small.npz   — the paper's 4x4 example and small seeded random cases: dense
  A and B, the GCOO arrays for several p, C in both numeric flavours and the
  KernelStats for several b;
* hashes.json — the benchmark configurations (square_benchmark(seed=1)
  inputs, bench.hpp:168-174): FNV-1a-32 of the GCOO arrays and of C (both
  flavours), C[0], C[last], the double checksum of C and KernelStats at
  p=4, b=64.

Fixtures are committed; /root/reference is not needed to run the tests.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Oracle, Reference, build  # noqa: E402


def example4x4() -> np.ndarray:
    # tests/common.hpp:107-117 (the paper's worked example)
    a = np.zeros((4, 4), np.float32)
    a[0, 0], a[0, 3], a[1, 1], a[2, 0], a[3, 2], a[3, 3] = 7, 8, 10, 9, 6, 3
    return a


def small_cases(R: Reference, RF: Reference):
    rng = np.random.default_rng(20050144)
    out = {}
    cases = [("ex4x4", example4x4(), np.eye(4, dtype=np.float32))]
    for i in range(12):
        m, k, n = (int(x) for x in rng.integers(1, 97, size=3))
        dens = float(rng.choice([0.0, 0.05, 0.2, 0.5, 1.0]))
        a = np.where(rng.random((m, k)) < dens, 1.0 - rng.random((m, k)), 0.0).astype(np.float32)
        b = (1.0 - rng.random((k, n))).astype(np.float32)
        cases.append((f"r{i}", a, b))
    for name, a, b in cases:
        out[f"{name}.A"] = a
        out[f"{name}.B"] = b
        for p in (1, 2, 4, 8, 64):
            g = R.dense_to_gcoo(a, p)
            for f in ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group"):
                out[f"{name}.p{p}.{f}"] = getattr(g, f)
        g4 = R.dense_to_gcoo(a, 4)
        c_mad, _ = R.spdm(g4, b, 64)
        c_fma, _ = RF.spdm(g4, b, 64)
        out[f"{name}.C_mad"] = c_mad
        out[f"{name}.C_fma"] = c_fma
        for bb in (1, 4, 64, 256):
            _, st = R.spdm(g4, b, bb)
            out[f"{name}.stats_b{bb}"] = np.array(st, np.uint64)
    return out


def big_hashes(O: Oracle, R: Reference, RF: Reference):
    res = {}
    for n, s in [(512, 0.95), (4000, 0.95), (8000, 0.99), (8000, 0.995), (8000, 0.9)]:
        t0 = time.time()
        a = R.uniform_sparse(n, s, 1)
        b = R.uniform_sparse(n, 0.0, R.derive_seed(1, n, 0xB))
        ent = {"n": n, "s": s, "seed": 1, "b_seed": R.derive_seed(1, n, 0xB),
               "A_fnv": O.fnv(a), "B_fnv": O.fnv(b)}
        for p in (4, 64) if n == 8000 and s == 0.99 else (4,):
            g = R.dense_to_gcoo(a, p)
            ent[f"p{p}"] = {f: O.fnv(getattr(g, f)) for f in ("values", "row_idx", "col_idx", "g_idxes",
                                                              "nnz_per_group")}
            ent[f"p{p}"].update(nnz=g.nnz, groups=g.groups, max_group_nnz=int(g.nnz_per_group.max()))
        g = R.dense_to_gcoo(a, 4)
        c, st = R.spdm(g, b, 64)
        ent["C_mad"] = {"fnv": O.fnv(c), "c0": float(c.flat[0]), "clast": float(c.flat[-1]),
                        "checksum": float(c.astype(np.float64).sum())}
        ent["stats_p4_b64"] = list(st)
        cf, _ = RF.spdm(g, b, 64)
        ent["C_fma"] = {"fnv": O.fnv(cf), "c0": float(cf.flat[0]), "clast": float(cf.flat[-1]),
                        "checksum": float(cf.astype(np.float64).sum())}
        ent["mad_vs_fma_max_rel"] = float(np.max(np.abs(c.astype(np.float64) - cf) / (np.abs(cf) + 1e-30)))
        res[f"n{n}_s{s}"] = ent
        print(f"n={n} s={s} done in {time.time() - t0:.1f}s", flush=True)
    return res


def main():
    build()
    O, R, RF = Oracle(), Reference(False), Reference(True)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **small_cases(R, RF))
    with open(os.path.join(HERE, "hashes.json"), "w") as f:
        json.dump(big_hashes(O, R, RF), f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
