"""PCIe ceilings for the host-pointer path (n=8000 fp32 B/C, 256 MB each):
one-way and concurrent H2D+D2H bandwidth, contiguous and 2-D strided (the
column strips the pipeline copies), timed with CUDA events.  Prints JSON lines.

    python tools/pcie_probe.py > profiles/rNN_pcie_probe.jsonl
"""
import json

import torch

n = 8000
NB = n * n * 4
x = torch.empty(n * n, dtype=torch.float32, pin_memory=True)
y = torch.empty(n * n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n * n, dtype=torch.float32, device="cuda")
e = torch.empty(n * n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    t0.record(cur)
    for _ in range(reps):
        fn()
    # join both side streams into the current one
    ev1, ev2 = torch.cuda.Event(), torch.cuda.Event()
    ev1.record(s1)
    ev2.record(s2)
    cur.wait_event(ev1)
    cur.wait_event(ev2)
    t1.record(cur)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        y.copy_(e, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, nbytes in (("h2d", h2d, NB), ("d2h", d2h, NB), ("h2d+d2h", both, 2 * NB)):
    ms = timed(fn)
    print(json.dumps({"probe": name, "bytes": nbytes, "ms": round(ms, 3), "gb_s": round(nbytes / ms / 1e6, 1)}))

# 2-D strided strips through cudaMemcpy2DAsync, exactly as the pipeline copies
import ctypes
import os

import nvidia.cuda_runtime as _rt

rt = ctypes.CDLL(os.path.join(_rt.__path__[0], "lib", "libcudart.so.12"))
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H2D, D2H = 1, 2
for W in (128, 256, 512, 1024, 2048):
    ds = torch.empty((n, W), device="cuda")
    es = torch.empty((n, W), device="cuda")
    nstrip = n // W

    def cp2d(dst, dpitch, src, spitch, kind, stream):
        r = rt.cudaMemcpy2DAsync(dst, dpitch, src, spitch, W * 4, n, kind, stream.cuda_stream)
        assert r == 0, r

    def h2d_s():
        for j in range(nstrip):
            cp2d(ds.data_ptr(), W * 4, x.data_ptr() + 4 * j * W, n * 4, H2D, s1)

    def both_s():
        for j in range(nstrip):
            cp2d(ds.data_ptr(), W * 4, x.data_ptr() + 4 * j * W, n * 4, H2D, s1)
            cp2d(y.data_ptr() + 4 * j * W, n * 4, es.data_ptr(), W * 4, D2H, s2)

    nb = nstrip * n * W * 4
    ms = timed(h2d_s, 3)
    print(json.dumps({"probe": "h2d_2d", "W": W, "bytes": nb, "ms": round(ms, 3), "gb_s": round(nb / ms / 1e6, 1)}))
    ms = timed(both_s, 3)
    print(json.dumps({"probe": "h2d+d2h_2d", "W": W, "bytes": 2 * nb, "ms": round(ms, 3),
                      "gb_s": round(2 * nb / ms / 1e6, 1)}))
