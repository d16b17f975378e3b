"""ctypes front-end for the CPU checker (TEST INFRASTRUCTURE ONLY).

Two back-ends, both built by ``oracle/Makefile``:

* ``Oracle``    — ``oracle/_build/libgcoo_oracle.so``, the plain-C restatement
  (``gcoo_oracle.c``; every function cites the reference file:line it follows).
* ``Reference`` — ``oracle/_ref/libgcoo_ref{,_fma}.so``, the unmodified reference
  library compiled from ``/root/reference/proj`` (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package; the CUDA
product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libgcoo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgcoo_ref.so")
REF_FMA_SO = os.path.join(HERE, "_ref", "libgcoo_ref_fma.so")

_i64, _i32, _u64, _dbl, _vp = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_void_p


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; the reference when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(_vp)


def _n(x) -> int:
    """nnz/groups as attribute (oracle Gcoo) or method (product GcooMatrix)."""
    return int(x() if callable(x) else x)


@dataclass
class Gcoo:
    """Host GCOO arrays with the reference's field names (matrix.hpp:176-245)."""
    rows_dim: int
    cols_dim: int
    p: int
    values: np.ndarray
    row_idx: np.ndarray
    col_idx: np.ndarray
    g_idxes: np.ndarray
    nnz_per_group: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    @property
    def groups(self) -> int:
        return int(self.g_idxes.size)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64, _u64]
        L.orc_uniform_sparse_f32.restype = _i64
        L.orc_uniform_sparse_f32.argtypes = [_i64, _dbl, _u64, _vp]
        L.orc_uniform_sparse_f64.restype = _i64
        L.orc_uniform_sparse_f64.argtypes = [_i64, _dbl, _u64, _vp]
        L.orc_uniform_sparse_coo_f32.restype = _i64
        L.orc_uniform_sparse_coo_f32.argtypes = [_i64, _dbl, _u64, _vp, _vp, _vp, _i64]
        L.orc_powerlaw_coo_f32.restype = _i64
        L.orc_powerlaw_coo_f32.argtypes = [_i64, _dbl, _dbl, _u64, _vp, _vp, _vp, _i64]
        L.orc_realized_nnz.restype = _i64
        L.orc_realized_nnz.argtypes = [_i64, _dbl]
        for t in ("f32", "f64"):
            f = getattr(L, f"orc_dense_to_gcoo_{t}")
            f.restype = _i64
            f.argtypes = [_i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp]
            f = getattr(L, f"orc_spdm_gcoo_{t}")
            f.restype = None
            f.argtypes = [_i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int]
        L.orc_coo_to_gcoo_f32.restype = C.c_int
        L.orc_coo_to_gcoo_f32.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
        L.orc_gcoo_validate.restype = C.c_int
        L.orc_gcoo_validate.argtypes = [_i64, _i64, _i32, _i64, _vp, _vp, _i64, _vp, _vp]
        L.orc_gcoo_stats.restype = None
        L.orc_gcoo_stats.argtypes = [_i64, _i32, _i64, _vp, _vp, _vp, _vp]
        L.orc_spdm_gcoo_rows_f32.restype = None
        L.orc_spdm_gcoo_rows_f32.argtypes = [_i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, C.c_int]
        L.orc_fnv1a32.restype = C.c_uint32
        L.orc_fnv1a32.argtypes = [_vp, _i64]
        for t in ("f32", "f64"):
            for name, args in (("orc_spdm_csr_", [_i64, _i64, _vp, _vp, _vp, _vp, _vp, C.c_int]),
                               ("orc_spdm_coo_", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, C.c_int]),
                               ("orc_gemm_dense_", [_i64, _i64, _i64, _vp, _vp, _vp, C.c_int])):
                f = getattr(L, name + t)
                f.restype = None
                f.argtypes = args

    # -- inputs -------------------------------------------------------------
    def derive_seed(self, base: int, a: int, b: int = 0) -> int:
        return int(self.lib.orc_derive_seed(base, a, b))

    def uniform_sparse(self, n: int, s: float, seed: int, dtype=np.float32) -> np.ndarray:
        out = np.empty((n, n), dtype=dtype)
        f = self.lib.orc_uniform_sparse_f32 if dtype == np.float32 else self.lib.orc_uniform_sparse_f64
        f(n, s, seed, _p(out))
        return out

    def uniform_sparse_coo(self, n: int, s: float, seed: int):
        nnz = int(self.lib.orc_realized_nnz(n, s))
        v = np.empty(nnz, np.float32); r = np.empty(nnz, np.int32); c = np.empty(nnz, np.int32)
        got = self.lib.orc_uniform_sparse_coo_f32(n, s, seed, _p(v), _p(r), _p(c), nnz)
        assert got == nnz
        return v, r, c

    def powerlaw_coo(self, n: int, s: float, alpha: float, seed: int):
        nnz = int(self.lib.orc_realized_nnz(n, s))
        v = np.empty(nnz, np.float32); r = np.empty(nnz, np.int32); c = np.empty(nnz, np.int32)
        got = self.lib.orc_powerlaw_coo_f32(n, s, alpha, seed, _p(v), _p(r), _p(c), nnz)
        assert got == nnz, got
        return v, r, c

    # -- construction -------------------------------------------------------
    def dense_to_gcoo(self, a: np.ndarray, p: int) -> Gcoo:
        m, k = a.shape
        a = np.ascontiguousarray(a)
        cap = int(np.count_nonzero(a))
        g = -(-m // p) if p > 0 else 0
        vals = np.empty(cap, a.dtype); rows = np.empty(cap, np.int32); cols = np.empty(cap, np.int32)
        gi = np.empty(max(g, 1), np.int64); gn = np.empty(max(g, 1), np.int64)
        f = self.lib.orc_dense_to_gcoo_f32 if a.dtype == np.float32 else self.lib.orc_dense_to_gcoo_f64
        nnz = f(m, k, _p(a), p, _p(vals), _p(rows), _p(cols), _p(gi), _p(gn))
        if nnz < 0:
            raise ValueError("dense_to_gcoo: p must be a power of two")
        return Gcoo(m, k, p, vals, rows, cols, gi[:g], gn[:g])

    def coo_to_gcoo(self, m, k, vals, rows, cols, p) -> Gcoo:
        nnz = vals.size
        g = -(-m // p) if p > 0 else 1
        ov = np.empty(nnz, np.float32); orr = np.empty(nnz, np.int32); oc = np.empty(nnz, np.int32)
        gi = np.empty(max(g, 1), np.int64); gn = np.empty(max(g, 1), np.int64)
        bad = C.c_int64(-1)
        rc = self.lib.orc_coo_to_gcoo_f32(m, k, nnz, _p(vals), _p(rows), _p(cols), p, _p(ov), _p(orr), _p(oc),
                                          _p(gi), _p(gn), C.byref(bad))
        if rc == -1:
            raise ValueError("coo_to_gcoo: p must be a power of two")
        if rc == -2:
            raise ValueError(f"CooMatrix: invalid entry {bad.value}")
        return Gcoo(m, k, p, ov, orr, oc, gi[:g], gn[:g])

    def validate(self, g: Gcoo) -> int:
        return int(self.lib.orc_gcoo_validate(g.rows_dim, g.cols_dim, g.p, g.nnz, _p(g.row_idx), _p(g.col_idx),
                                              g.groups, _p(g.g_idxes), _p(g.nnz_per_group)))

    # -- multiply -----------------------------------------------------------
    def spdm(self, g: Gcoo, B: np.ndarray, b: int = 64, fma: bool = True):
        k, n = B.shape
        Cm = np.empty((g.rows_dim, n), dtype=B.dtype)
        st = (_u64 * 4)()
        f = self.lib.orc_spdm_gcoo_f32 if B.dtype == np.float32 else self.lib.orc_spdm_gcoo_f64
        f(g.rows_dim, k, n, g.p, b, _p(g.values), _p(g.row_idx), _p(g.col_idx), _p(g.g_idxes),
          _p(g.nnz_per_group), _p(np.ascontiguousarray(B)), _p(Cm), st, int(fma))
        return Cm, tuple(int(x) for x in st)

    def spdm_rows(self, g: Gcoo, B: np.ndarray, r0: int, r1: int, b: int = 64, fma: bool = True) -> np.ndarray:
        k, n = B.shape
        Cm = np.zeros((g.rows_dim, n), dtype=np.float32)
        self.lib.orc_spdm_gcoo_rows_f32(g.rows_dim, n, g.p, b, _p(g.values), _p(g.row_idx), _p(g.col_idx),
                                        _p(g.g_idxes), _p(g.nnz_per_group), _p(np.ascontiguousarray(B)),
                                        _p(Cm), r0, r1, int(fma))
        return Cm

    def stats(self, g: Gcoo, n: int, b: int):
        st = (_u64 * 4)()
        self.lib.orc_gcoo_stats(n, b, g.groups, _p(g.col_idx), _p(g.g_idxes), _p(g.nnz_per_group), st)
        return tuple(int(x) for x in st)

    # -- the reference's comparison kernels (kernels.hpp:107-232) ----------
    def spdm_csr(self, m: int, vals, cols, row_ptr, B: np.ndarray, fma: bool = True) -> np.ndarray:
        """Row-split CSR: each row's chain in CSR order (kernels.hpp:163-184)."""
        B = np.ascontiguousarray(B)
        vals = np.ascontiguousarray(vals, dtype=B.dtype)
        Cm = np.empty((m, B.shape[1]), dtype=B.dtype)
        f = self.lib.orc_spdm_csr_f32 if B.dtype == np.float32 else self.lib.orc_spdm_csr_f64
        f(m, B.shape[1], _p(vals), _p(np.ascontiguousarray(cols, dtype=np.int32)),
          _p(np.ascontiguousarray(row_ptr, dtype=np.int64)), _p(B), _p(Cm), int(fma))
        return Cm

    def spdm_coo(self, m: int, vals, rows, cols, B: np.ndarray, fma: bool = True) -> np.ndarray:
        """Ungrouped COO: each row's chain in entry order (kernels.hpp:193-232)."""
        B = np.ascontiguousarray(B)
        vals = np.ascontiguousarray(vals, dtype=B.dtype)
        Cm = np.empty((m, B.shape[1]), dtype=B.dtype)
        f = self.lib.orc_spdm_coo_f32 if B.dtype == np.float32 else self.lib.orc_spdm_coo_f64
        f(m, B.shape[1], vals.size, _p(vals), _p(np.ascontiguousarray(rows, dtype=np.int32)),
          _p(np.ascontiguousarray(cols, dtype=np.int32)), _p(B), _p(Cm), int(fma))
        return Cm

    def gemm_dense(self, A: np.ndarray, B: np.ndarray, fma: bool = True) -> np.ndarray:
        """gemm_dense_blocked: l-ascending chain per element (kernels.hpp:107-155)."""
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B, dtype=A.dtype)
        Cm = np.empty((A.shape[0], B.shape[1]), dtype=A.dtype)
        f = self.lib.orc_gemm_dense_f32 if A.dtype == np.float32 else self.lib.orc_gemm_dense_f64
        f(A.shape[0], A.shape[1], B.shape[1], _p(A), _p(B), _p(Cm), int(fma))
        return Cm

    def fnv(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        return "%08x" % self.lib.orc_fnv1a32(_p(a), a.nbytes)


class Reference:
    """The reference library itself (fma=False: as shipped; fma=True: -mfma)."""

    def __init__(self, fma: bool = False):
        path = REF_FMA_SO if fma else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build with make -C oracle while /root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _u64, _u64]
        L.ref_uniform_sparse_f32.restype = C.c_int
        L.ref_uniform_sparse_f32.argtypes = [_i64, _dbl, _u64, _vp]
        L.ref_uniform_sparse_f64.restype = C.c_int
        L.ref_uniform_sparse_f64.argtypes = [_i64, _dbl, _u64, _vp]
        for t in ("f32", "f64"):
            f = getattr(L, f"ref_dense_to_gcoo_{t}")
            f.restype = _i64
            f.argtypes = [_i64, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp]
            f = getattr(L, f"ref_spdm_gcoo_{t}")
            f.restype = C.c_int
            f.argtypes = [_i64, _i64, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                          C.c_int, _vp, _i64]
            f = getattr(L, f"ref_gemm_oracle_{t}")
            f.restype = C.c_int
            f.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp]
        L.ref_coo_to_gcoo_f32.restype = C.c_int
        L.ref_coo_to_gcoo_f32.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp]
        L.ref_run_benchmark_gcoo_f32.restype = C.c_int
        L.ref_run_benchmark_gcoo_f32.argtypes = [_i64, _vp, _vp, _i32, _i32, C.c_int, C.c_int, C.c_int, _vp]
        L.ref_time_spdm_gcoo_f32.restype = C.c_int
        L.ref_time_spdm_gcoo_f32.argtypes = [_i64, _i64, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp,
                                             _vp, C.c_int, C.c_int, C.c_int, _vp]

    TRAFFIC_FIELDS = ("n_dm", "n_l2", "n_shm", "tex_l1_trans", "flops", "b_element_loads", "b_element_reused",
                      "staged_entries", "b_load_transactions", "sparse_transactions", "store_transactions")

    def model_traffic(self, rows, cols, m, k, n, p=4, b=64, infinite_l2=False, csr=False):
        """The reference's model_gcoo_traffic / model_csr_traffic -> dict of the 11 counters."""
        L = self.lib
        L.ref_model_traffic.restype = C.c_int
        L.ref_model_traffic.argtypes = [C.c_int, _i64, _vp, _vp, _i64, _i64, _i64, _i32, _i32, C.c_int, _vp]
        r = np.ascontiguousarray(rows, dtype=np.int32)
        c = np.ascontiguousarray(cols, dtype=np.int32)
        out = np.zeros(11, np.uint64)
        self._check(L.ref_model_traffic(1 if csr else 0, r.size, r.ctypes.data, c.ctypes.data, m, k, n, p, b,
                                        1 if infinite_l2 else 0, out.ctypes.data))
        return dict(zip(self.TRAFFIC_FIELDS, (int(x) for x in out)))

    def read_mtx(self, path: str, dtype=np.float32):
        """read_matrix_market<T> (io.hpp:66-85).  Returns ("dense", array) or
        ("coo", rows_dim, cols_dim, values, row_idx, col_idx); a ParseError comes
        back as ("error", line, message), other failures raise."""
        t = "f32" if np.dtype(dtype) == np.float32 else "f64"
        rd, fe = getattr(self.lib, f"ref_mtx_read_{t}"), getattr(self.lib, f"ref_mtx_fetch_{t}")
        rd.restype, rd.argtypes = C.c_int, [C.c_char_p, _vp]
        fe.restype, fe.argtypes = None, [_vp, _vp, _vp]
        info = np.zeros(5, np.int64)
        rc = rd(os.fsencode(path), info.ctypes.data)
        if rc == 3:
            return ("error", int(info[4]), self.lib.ref_last_error().decode())
        self._check(rc)
        dense, m, k, cnt = (int(x) for x in info[:4])
        if dense:
            out = np.empty((m, k), dtype=dtype)
            fe(out.ctypes.data, None, None)
            return ("dense", out)
        v, r, c = np.empty(cnt, dtype=dtype), np.empty(cnt, np.int32), np.empty(cnt, np.int32)
        fe(v.ctypes.data, r.ctypes.data, c.ctypes.data)
        return ("coo", m, k, v, r, c)

    def write_mtx(self, path: str, a=None, coo=None):
        """write_matrix_market (io.hpp:87-109): dense `a`, or coo=(m, k, values, row_idx, col_idx)."""
        if a is not None:
            a = np.ascontiguousarray(a)
            t = "f32" if a.dtype == np.float32 else "f64"
            f = getattr(self.lib, f"ref_mtx_write_dense_{t}")
            f.restype, f.argtypes = C.c_int, [C.c_char_p, _i64, _i64, _vp]
            self._check(f(os.fsencode(path), a.shape[0], a.shape[1], a.ctypes.data))
            return
        m, k, v, r, c = coo
        v = np.ascontiguousarray(v)
        r = np.ascontiguousarray(r, dtype=np.int32)
        c = np.ascontiguousarray(c, dtype=np.int32)
        t = "f32" if v.dtype == np.float32 else "f64"
        f = getattr(self.lib, f"ref_mtx_write_coo_{t}")
        f.restype, f.argtypes = C.c_int, [C.c_char_p, _i64, _i64, _i64, _vp, _vp, _vp]
        self._check(f(os.fsencode(path), m, k, v.size, v.ctypes.data, r.ctypes.data, c.ctypes.data))

    def _check(self, rc: int):
        if rc == 1:
            raise ValueError(self.lib.ref_last_error().decode())
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def uniform_sparse(self, n, s, seed, dtype=np.float32):
        out = np.empty((n, n), dtype=dtype)
        f = self.lib.ref_uniform_sparse_f32 if dtype == np.float32 else self.lib.ref_uniform_sparse_f64
        self._check(f(n, s, seed, _p(out)))
        return out

    def derive_seed(self, base, a, b=0):
        return int(self.lib.ref_derive_seed(base, a, b))

    def dense_to_gcoo(self, a: np.ndarray, p: int) -> Gcoo:
        m, k = a.shape
        a = np.ascontiguousarray(a)
        f = self.lib.ref_dense_to_gcoo_f32 if a.dtype == np.float32 else self.lib.ref_dense_to_gcoo_f64
        nnz = f(m, k, _p(a), p, None, None, None, None, None)
        if nnz < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        g = -(-m // p)
        vals = np.empty(nnz, a.dtype); rows = np.empty(nnz, np.int32); cols = np.empty(nnz, np.int32)
        gi = np.empty(g, np.int64); gn = np.empty(g, np.int64)
        f(m, k, _p(a), p, _p(vals), _p(rows), _p(cols), _p(gi), _p(gn))
        return Gcoo(m, k, p, vals, rows, cols, gi, gn)

    def coo_to_gcoo(self, m, k, vals, rows, cols, p) -> Gcoo:
        nnz = vals.size
        g = -(-m // p) if p > 0 else 1
        ov = np.empty(nnz, np.float32); orr = np.empty(nnz, np.int32); oc = np.empty(nnz, np.int32)
        gi = np.empty(max(g, 1), np.int64); gn = np.empty(max(g, 1), np.int64)
        self._check(self.lib.ref_coo_to_gcoo_f32(m, k, nnz, _p(vals), _p(rows), _p(cols), p, _p(ov), _p(orr),
                                                 _p(oc), _p(gi), _p(gn)))
        return Gcoo(m, k, p, ov, orr, oc, gi[:g], gn[:g])

    def spdm(self, g: Gcoo, B: np.ndarray, b: int = 64, workers: int = 0, tile_order=None):
        k, n = B.shape
        Cm = np.empty((g.rows_dim, n), dtype=B.dtype)
        st = (_u64 * 4)()
        f = self.lib.ref_spdm_gcoo_f32 if B.dtype == np.float32 else self.lib.ref_spdm_gcoo_f64
        to = None if tile_order is None else np.ascontiguousarray(tile_order, dtype=np.int64)
        self._check(f(g.rows_dim, k, n, g.p, b, _n(g.nnz), _p(g.values), _p(g.row_idx), _p(g.col_idx), _n(g.groups),
                      _p(g.g_idxes), _p(g.nnz_per_group), _p(np.ascontiguousarray(B)), _p(Cm), st, workers,
                      _p(to), 0 if to is None else to.size))
        return Cm, tuple(int(x) for x in st)

    def spdm_csr(self, m, k, vals, cols, row_ptr, B, p=4, b=64, workers=0):
        B = np.ascontiguousarray(B)
        Cm = np.empty((m, B.shape[1]), dtype=B.dtype)
        f = self.lib.ref_spdm_csr_f32 if B.dtype == np.float32 else self.lib.ref_spdm_csr_f64
        f.restype = C.c_int
        f.argtypes = [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, C.c_int]
        vals = np.ascontiguousarray(vals, dtype=B.dtype)
        self._check(f(_n(m), _n(k), _n(B.shape[1]), _n(vals.size), _p(vals),
                      _p(np.ascontiguousarray(cols, dtype=np.int32)), _p(np.ascontiguousarray(row_ptr, dtype=np.int64)),
                      _p(B), _p(Cm), p, b, workers))
        return Cm

    def spdm_coo(self, m, k, vals, rows, cols, B, p=4, b=64, workers=0):
        B = np.ascontiguousarray(B)
        Cm = np.empty((m, B.shape[1]), dtype=B.dtype)
        f = self.lib.ref_spdm_coo_f32 if B.dtype == np.float32 else self.lib.ref_spdm_coo_f64
        f.restype = C.c_int
        f.argtypes = [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, C.c_int]
        vals = np.ascontiguousarray(vals, dtype=B.dtype)
        self._check(f(_n(m), _n(k), _n(B.shape[1]), _n(vals.size), _p(vals),
                      _p(np.ascontiguousarray(rows, dtype=np.int32)), _p(np.ascontiguousarray(cols, dtype=np.int32)),
                      _p(B), _p(Cm), p, b, workers))
        return Cm

    def gemm_dense(self, A, B, p=4, b=64, workers=0):
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B, dtype=A.dtype)
        Cm = np.empty((A.shape[0], B.shape[1]), dtype=A.dtype)
        f = self.lib.ref_gemm_dense_f32 if A.dtype == np.float32 else self.lib.ref_gemm_dense_f64
        f.restype = C.c_int
        f.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _i32, C.c_int]
        self._check(f(_n(A.shape[0]), _n(A.shape[1]), _n(B.shape[1]), _p(A), _p(B), _p(Cm), p, b, workers))
        return Cm

    def gemm_oracle(self, A: np.ndarray, B: np.ndarray) -> np.ndarray:
        m, k = A.shape
        n = B.shape[1]
        Cm = np.empty((m, n), dtype=A.dtype)
        f = self.lib.ref_gemm_oracle_f32 if A.dtype == np.float32 else self.lib.ref_gemm_oracle_f64
        self._check(f(m, k, n, _p(np.ascontiguousarray(A)), _p(np.ascontiguousarray(B)), _p(Cm)))
        return Cm

    def run_benchmark_gcoo(self, A: np.ndarray, B: np.ndarray, p=4, b=64, workers=0, warmup=1, reps=5):
        out = (_dbl * 5)()
        self._check(self.lib.ref_run_benchmark_gcoo_f32(A.shape[0], _p(A), _p(B), p, b, workers, warmup, reps, out))
        return dict(eo_s=out[0], kc_s=out[1], gflops=out[2], workers=int(out[3]), nnz=int(out[4]))

    def time_spdm(self, g: Gcoo, B: np.ndarray, b=64, workers=0, warmup=1, reps=5):
        out = (_dbl * 2)()
        k, n = B.shape
        self._check(self.lib.ref_time_spdm_gcoo_f32(g.rows_dim, k, n, g.p, b, g.nnz, _p(g.values), _p(g.row_idx),
                                                    _p(g.col_idx), g.groups, _p(g.g_idxes), _p(g.nnz_per_group),
                                                    _p(np.ascontiguousarray(B)), workers, warmup, reps, out))
        return dict(kc_s=out[0], workers=int(out[1]))


def have_reference() -> bool:
    return os.path.exists(REF_SO) and os.path.exists(REF_FMA_SO)


# --------------------------------------------------------- traffic model --
def _trans(elems: int) -> int:
    """traffic.cpp:16-18 — 32-element coalesced transactions."""
    return -(-elems // 32)


def model_traffic(rows, cols, m, k, n, p=4, b=64, infinite_l2=False, csr=False) -> dict:
    """Plain-Python restatement of model_gcoo_traffic (traffic.cpp:43-137) and
    model_csr_traffic (:140-197): the same loops over groups/rows, strips and
    runs, for small patterns (the checker of the device model)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    rep = dict(n_dm=0, n_l2=0, n_shm=0, tex_l1_trans=0, flops=0)
    det = dict(b_element_loads=0, b_element_reused=0, staged_entries=0, b_load_transactions=0,
               sparse_transactions=0, store_transactions=0)
    if csr:
        segs = -(-n // 32)
        touched = set()
        rep["n_dm"] += _trans(m + 1)                      # :162-163
        det["sparse_transactions"] += _trans(m + 1)
        by_row = [[] for _ in range(m)]
        for r, c in zip(rows.tolist(), cols.tolist()):
            by_row[r].append(c)
        for r in range(m):
            cs = sorted(by_row[r])
            if cs:                                        # :168-173
                sp = _trans(2 * len(cs))
                det["sparse_transactions"] += sp
                rep["n_dm"] += sp
            for c in cs:                                  # :175-191
                det["b_element_loads"] += n
                det["b_load_transactions"] += segs
                if infinite_l2:
                    for s_ in range(segs):
                        if (c, s_) in touched:
                            rep["n_l2"] += 1
                        else:
                            rep["n_dm"] += 1
                            touched.add((c, s_))
                else:
                    rep["n_dm"] += segs
            rep["n_dm"] += segs                           # :194-196
            det["store_transactions"] += segs
            rep["flops"] += 2 * len(cs) * n
        return {**rep, **det}
    groups = -(-m // p)
    strips = -(-n // b)
    gcols = [[] for _ in range(groups)]
    for r, c in zip(rows.tolist(), cols.tolist()):
        gcols[r // p].append(c)
    touched = set()
    for gi in range(groups):
        cs = sorted(gcols[gi])
        nnz_g = len(cs)
        h = min(p, m - gi * p)
        runs = []                                         # :81-91 runs never cross a chunk of b entries
        for chunk in range(0, nnz_g, b):
            blk = cs[chunk:chunk + b]
            e = 0
            while e < len(blk):
                ln = 1
                while e + ln < len(blk) and blk[e + ln] == blk[e]:
                    ln += 1
                runs.append((blk[e], ln))
                e += ln
        for sj in range(strips):
            w = min(b, n - sj * b)
            if nnz_g > 0:                                 # :96-108
                rep["n_shm"] += 2 * nnz_g
                det["staged_entries"] += nnz_g
                sp = _trans(3 * nnz_g)
                det["sparse_transactions"] += sp
                if infinite_l2 and sj > 0:
                    rep["n_l2"] += sp
                else:
                    rep["n_dm"] += sp
            for col, ln in runs:                          # :111-128
                bt = _trans(w)
                det["b_load_transactions"] += bt
                det["b_element_loads"] += w
                det["b_element_reused"] += (ln - 1) * w
                rep["tex_l1_trans"] += (ln - 1) * w
                if infinite_l2:
                    if (col, sj) in touched:
                        rep["n_l2"] += bt
                    else:
                        rep["n_dm"] += bt
                        touched.add((col, sj))
                else:
                    rep["n_dm"] += bt
            st = _trans(h * w)                            # :131-133
            det["store_transactions"] += st
            rep["n_dm"] += st
            rep["flops"] += 2 * nnz_g * w
    return {**rep, **det}
