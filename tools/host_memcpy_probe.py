"""Host memcpy roof for the pageable e2e leg: 256 MiB pageable -> pinned copies
(what the staging ring's pack does) with 1..N threads, as JSON lines.  The
pageable call moves B (256 MB) in and C (256 MB) out through such copies."""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

N = 64 << 20  # floats: 256 MiB
src = np.random.default_rng(1).random(N, dtype=np.float32)
dst_pin = torch.empty(N, dtype=torch.float32, pin_memory=True).numpy()
dst_page = np.empty(N, np.float32)
dst_page[...] = 0
for name, dst in (("pageable->pinned", dst_pin), ("pageable->pageable", dst_page)):
    for nt in (1, 2, 4, 8, 16, os.cpu_count()):
        parts = np.array_split(np.arange(N), nt)
        bounds = [(p[0], p[-1] + 1) for p in parts]

        def cp(b):
            np.copyto(dst[b[0]:b[1]], src[b[0]:b[1]])

        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(cp, bounds))
            ts = []
            for _ in range(5):
                t = time.perf_counter()
                list(ex.map(cp, bounds))
                ts.append(time.perf_counter() - t)
        best = min(ts)
        print(json.dumps({"copy": name, "threads": nt, "gb_s": round(N * 4 / best / 1e9, 2),
                          "ms_256MiB": round(best * 1e3, 2)}), flush=True)
