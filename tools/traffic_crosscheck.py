"""Predicted vs measured memory traffic of the multiply.

For the n=8000 benchmark patterns (square_benchmark(seed=1)) this prints one
JSON line per sparsity with three predictions and the ncu measurement:

* paper model  — the reference's model_gcoo_traffic (traffic.cpp:43-137),
  infinite_l2, at the paper's kernel parameters p=4, b=64, evaluated on the
  GPU (gcoo_model_traffic_dev); transactions x 128 B.  n_dm is the DRAM
  prediction; n_l2 + n_dm the L2 -> SM prediction; n_shm + tex the on-chip
  (staging + reuse window) traffic — the paper's argument that GCOO moves
  traffic from DRAM/L2 into shared memory.
* tiling model — the same model at THIS kernel's tiling (p = rows per CTA
  rounded to a power of two, b = CTA strip width W), i.e. what the paper's
  model says once the group is a whole CTA row block.
* kernel model — this kernel's own traffic: DRAM = compulsory bytes; L2 -> SM
  = B tiles (CTAs x k x W x 4) + the record stream once per column tile;
  shared-memory wavefronts = B reads (4 per entry and column tile) + record
  loads (1 per record) + TMA tile writes (bytes / 128).
* measured — ncu (profiles/r0X_ncu_*.json, `--set full` of the same launch).

    python tools/traffic_crosscheck.py profiles/r01_ncu_tacc28_s0.9.json \
        profiles/r01_ncu_tacc28_s0.99.json profiles/r01_ncu_tacc28_s0.995.json
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_14469_b200 as G  # noqa: E402

N = 8000


def tiling(kernel_name):
    """RB, W, KC of the profiled kernel from its template arguments
    (TaccCfg<V, KC, STAGES, CAP, NW>: RB = NW * (512 / (NW/4) & ~7) / V; TileCfg: RB = 15 * 64 / V)."""
    import re
    m = re.search(r"TaccCfg<(\d+), (\d+), \d+, \d+(?:, (\d+))?(?:, (\d+))?(?:, \w+)?>", kernel_name)
    if m:
        v, kc, nw, epr = int(m.group(1)), int(m.group(2)), int(m.group(3) or 16), int(m.group(4) or 2)
        tcols = (512 // (nw // 4)) & ~7
        return dict(RB=nw * (tcols // v), W=32 * v, KC=kc, EPR=epr, NW=nw)
    m = re.search(r"TileCfg<(\d+), (\d+),", kernel_name)
    v, kc = int(m.group(1)), int(m.group(2))
    return dict(RB=15 * (64 // v), W=32 * v, KC=kc, EPR=3, NW=15)


def pow2_at_least(x):
    p = 1
    while p < x:
        p *= 2
    return p


def main():
    meas = {}
    for path in sys.argv[1:]:
        with open(path) as f:
            m = json.load(f)
        s = float(path.rsplit("_s", 1)[1].rsplit(".json", 1)[0])
        meas[s] = (m["kernel"], m, os.path.basename(path))
    for s in sorted(meas):
        kname, m, src = meas[s]
        t = tiling(kname)
        a = torch.from_numpy(G.generate_uniform_sparse(N, s, 1)).cuda()
        d = G.dense_to_gcoo_dev(a, 4)
        nnz = d.nnz()
        paper = G.model_traffic_dev(d, N, G.ExecConfig(p=4, b=64), infinite_l2=True)
        dp = G.dense_to_gcoo_dev(a, pow2_at_least(t["RB"]))
        tmodel = G.model_traffic_dev(dp, N, G.ExecConfig(p=dp.p, b=t["W"]), infinite_l2=True)
        del a, dp
        # this kernel's records, counted exactly: three-entry records hold up to
        # three entries of one row per chunk; two-entry records hold any two
        # consecutive entries of a warp's stream (identity placement: row j of a
        # row block belongs to warp j % NW), i.e. ceil(entries / 2) per warp and chunk
        rows = d.row_idx.long()
        cols = d.col_idx.long()
        nch = (N + t["KC"] - 1) // t["KC"]
        if t["EPR"] == 2:
            unit = (rows // t["RB"]) * t["NW"] + (rows % t["RB"]) % t["NW"]
            key = unit * nch + cols // t["KC"]
        else:
            key = rows * nch + cols // t["KC"]
        per_run = torch.bincount(key)
        records = int(((per_run + t["EPR"] - 1) // t["EPR"]).sum())
        col_tiles = (N + t["W"] - 1) // t["W"]
        row_blocks = (N + t["RB"] - 1) // t["RB"]
        b_tiles = row_blocks * col_tiles * N * t["W"] * 4
        rec_bytes = records * 16 * col_tiles
        compulsory = 12 * nnz + 16 * ((N + 3) // 4) + 4 * N * N + 4 * N * N
        wavefronts = nnz * col_tiles * 4 + records * col_tiles + (b_tiles + rec_bytes) / 128
        row = {
            "n": N, "s": s, "nnz": nnz, "kernel": kname[:60], "tiling": t, "ncu": src,
            "paper_model_p4_b64": {"dram_bytes": paper["n_dm"] * 128, "l2_to_sm_bytes": (paper["n_dm"] + paper["n_l2"]) * 128,
                                   "onchip_bytes": (paper["n_shm"] + paper["tex_l1_trans"]) * 4,
                                   "share": {k: round(paper[k] / max(1, sum(paper[x] for x in ("n_dm", "n_l2", "n_shm", "tex_l1_trans"))), 4)
                                             for k in ("n_dm", "n_l2", "n_shm", "tex_l1_trans")}},
            "tiling_model": {"p": pow2_at_least(t["RB"]), "b": t["W"], "dram_bytes": tmodel["n_dm"] * 128,
                             "l2_to_sm_bytes": (tmodel["n_dm"] + tmodel["n_l2"]) * 128},
            "kernel_model": {"dram_bytes": compulsory, "l2_to_sm_bytes": b_tiles + rec_bytes,
                             "smem_wavefronts": int(wavefronts), "records": records},
            "measured": {"dram_bytes": m["dram_read_bytes"] + m["dram_write_bytes"],
                         "l2_to_sm_bytes": m["l2_read_bytes_from_sm"], "smem_wavefronts": m["smem_wavefronts"],
                         "smem_wavefront_pct": m["smem_wavefront_pct"], "duration_s": m["duration_s"]},
        }
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
