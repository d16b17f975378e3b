"""Build libgcoo_cuda.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_2005_14469_b200.build [--force]

The shared library lands in paper_2005_14469_b200/lib/ so that it travels to
the GPU box with the repository snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libgcoo_cuda.so")
SOURCES = ["capi.cu", "host_gen.cpp", "host_mtx.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _inputs() -> list[str]:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".cpp", ".h"))]
    files.append(os.path.join(ROOT, "include", "gcoo_capi.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """out/defines: variant builds for measurements (e.g. ablations), never the product."""
    if out is None and not force and up_to_date():
        return LIB
    lib_path = out or LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    cmd = [
        _nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v", "-shared",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC,
        *["-D" + d for d in defines],
        "-o", lib_path + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES],
    ]
    # nvcc picks the host compiler from PATH; make sure it is the system gcc
    env = dict(os.environ)
    env.pop("CXX", None)
    env.pop("CC", None)
    res = subprocess.run(cmd, capture_output=True, text=True, env=env)
    log = lib_path + ".log" if out else os.path.join(LIB_DIR, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed (see %s):\n%s" % (log, res.stderr[-4000:]))
    os.replace(lib_path + ".tmp", lib_path)
    if verbose:
        print(res.stderr)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
