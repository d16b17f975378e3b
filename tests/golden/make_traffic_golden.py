"""Regenerate tests/golden/traffic.json from the REFERENCE's traffic model
(model_gcoo_traffic / model_csr_traffic, traffic.cpp:43-197, through
oracle/_ref/libgcoo_ref.so) on the benchmark patterns:
square_benchmark(seed=1) A at n=512 s=0.95 and n=8000 s=0.99, p=4, b=64,
both cache modes, N = n.

    python tests/golden/make_traffic_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference  # noqa: E402


def main():
    R = Reference(False)
    out = {}
    for n, s in ((512, 0.95), (8000, 0.99)):
        a = R.uniform_sparse(n, s, 1)
        rows, cols = np.nonzero(a)
        ent = {}
        for kind in ("gcoo", "csr"):
            for mode in ("cold", "infinite_l2"):
                ent[f"{kind}_{mode}"] = R.model_traffic(rows, cols, n, n, n, 4, 64, mode == "infinite_l2",
                                                        kind == "csr")
        out[f"n{n}_s{s}"] = ent
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
