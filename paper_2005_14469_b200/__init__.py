"""B200-native GCOOSpDM (arXiv 2005.14469): Python host mirror of the reference API.

The product is ``lib/libgcoo_cuda.so`` (hand-written sm_100a CUDA behind the C
ABI in ``include/gcoo_capi.h``).  This module binds that ABI with ctypes and
mirrors the reference's C++ names and semantics (``proj/include/gcoo``):

==========================  =========================================
reference (C++)             here
==========================  =========================================
``GcooMatrix<T>``           :class:`GcooMatrix` (same fields)
``ExecConfig``              :class:`ExecConfig` (p, b, workers)
``KernelStats``             :class:`KernelStats`
``TimingBreakdown``         :class:`TimingBreakdown`
``dense_to_gcoo``           :func:`dense_to_gcoo`
``coo_to_gcoo``             :func:`coo_to_gcoo`
(new) CSR entry             :func:`csr_to_gcoo`
``spdm_gcoo`` (2 overloads) :func:`spdm_gcoo`
``spdm_gcoo_auto``          :func:`spdm_gcoo_auto`
``generate_uniform_sparse`` :func:`generate_uniform_sparse`
``derive_seed``             :func:`derive_seed`
==========================  =========================================

``std::invalid_argument`` surfaces as :class:`ValueError`, CUDA failures as
:class:`RuntimeError`, allocation failures as :class:`MemoryError` — raised at
the same points the reference throws.  There is no CPU fallback: without the
built library or a GPU every compute call raises.

Device-resident variants (``*_dev``) take torch CUDA tensors and a stream and
are what bench.py times.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GCOO_LIB") or os.path.join(PKG, "lib", "libgcoo_cuda.so")

_i64, _i32, _u64, _dbl, _vp, _int = C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_void_p, C.c_int

GCOO_OK, GCOO_EINVAL, GCOO_ECUDA, GCOO_ENOMEM = 0, 1, 2, 3
FLAVOR_FMA, FLAVOR_MUL_ADD = 0, 1


class _Stats(C.Structure):
    _fields_ = [("flops", _u64), ("b_loads_total", _u64), ("b_loads_reused", _u64), ("staging_fills", _u64)]


_lib = None


def _sig(L, name, res, args):
    # test / measurement hooks may be absent from a measurement variant's
    # library (GCOO_LIB); every other entry point is required
    if name.startswith("gcoo_debug_") and os.environ.get("GCOO_LIB") and not hasattr(L, name):
        return
    f = getattr(L, name)
    f.restype = res
    f.argtypes = args


def lib():
    """Load libgcoo_cuda.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2005_14469_b200.build`")
    L = C.CDLL(LIB_PATH)
    _sig(L, "gcoo_abi_version", _int, [])
    _sig(L, "gcoo_last_error", C.c_char_p, [])
    _sig(L, "gcoo_device_count", _int, [C.POINTER(_int)])
    _sig(L, "gcoo_set_device", _int, [_int])
    _sig(L, "gcoo_launch_count", _u64, [])
    _sig(L, "gcoo_stream_sync", _int, [_vp])
    spdm_args = [_i64, _i64, _i64, _i32, _i32, _i32, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                 C.POINTER(_Stats), _vp, _i64]
    _sig(L, "gcoo_spdm_f32", _int, spdm_args)
    _sig(L, "gcoo_spdm_f64", _int, spdm_args)
    for t in ("f32", "f64"):
        _sig(L, f"gcoo_spdm_auto_{t}", _int, [_i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, C.POINTER(_Stats),
                                                C.POINTER(_dbl), C.POINTER(_dbl)])
    dev_args = [_i64, _i64, _i64, _i32, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _i64,
                C.POINTER(_Stats), _int, _vp]
    _sig(L, "gcoo_spdm_f32_dev", _int, dev_args)
    _sig(L, "gcoo_spdm_f64_dev", _int, dev_args)
    _sig(L, "gcoo_stats_dev", _int, [_i64, _i64, _i32, _i32, _i64, _vp, _vp, _i64, _vp, C.POINTER(_Stats), _vp])
    _sig(L, "gcoo_model_traffic_dev", _int, [_int, _i64, _i64, _i64, _i32, _i32, _i64, _vp, _vp, _i64, _vp, _vp,
                                              _int, C.POINTER(_Traffic), C.POINTER(_TrafficDetail), _vp])
    coo_args = [_i64, _i64, _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
    _sig(L, "gcoo_coo_to_gcoo_f32", _int, coo_args)
    _sig(L, "gcoo_coo_to_gcoo_f64", _int, coo_args)
    _sig(L, "gcoo_coo_to_gcoo_f32_dev", _int, coo_args + [_vp])
    _sig(L, "gcoo_coo_to_gcoo_f64_dev", _int, coo_args + [_vp])
    _sig(L, "gcoo_csr_to_gcoo_f32_dev", _int, coo_args + [_vp])
    _sig(L, "gcoo_csr_to_gcoo_f64_dev", _int, coo_args + [_vp])
    _sig(L, "gcoo_csr_to_gcoo_f32", _int, coo_args)
    _sig(L, "gcoo_csr_to_gcoo_f64", _int, coo_args)
    dense_args = [_i64, _i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp, _vp, C.POINTER(_i64)]
    _sig(L, "gcoo_dense_to_gcoo_f32", _int, dense_args)
    _sig(L, "gcoo_dense_to_gcoo_f64", _int, dense_args)
    _sig(L, "gcoo_dense_to_gcoo_f32_dev", _int, dense_args + [_vp])
    _sig(L, "gcoo_dense_to_gcoo_f64_dev", _int, dense_args + [_vp])
    for t in ("f32", "f64"):
        _sig(L, f"gcoo_spdm_csr_{t}", _int, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp])
        _sig(L, f"gcoo_spdm_csr_{t}_dev", _int, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int, _vp])
        _sig(L, f"gcoo_spdm_coo_{t}", _int, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp])
        _sig(L, f"gcoo_spdm_coo_{t}_dev", _int, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _int, _vp])
        _sig(L, f"gcoo_gemm_dense_{t}", _int, [_i64, _i64, _i64, _vp, _vp, _vp])
        _sig(L, f"gcoo_gemm_dense_{t}_dev", _int, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp])
    _sig(L, "gcoo_generate_uniform_sparse_f32", _int, [_i64, _dbl, _u64, _vp])
    _sig(L, "gcoo_generate_uniform_sparse_coo_f32", _int, [_i64, _dbl, _u64, _i64, _vp, _vp, _vp, C.POINTER(_i64)])
    _sig(L, "gcoo_generate_powerlaw_coo_f32", _int, [_i64, _dbl, _dbl, _u64, _i64, _vp, _vp, _vp, C.POINTER(_i64)])
    _sig(L, "gcoo_derive_seed", _u64, [_u64, _u64, _u64])
    _sig(L, "gcoo_debug_force_kernel", _int, [_int])
    _sig(L, "gcoo_debug_last_kernel", _int, [])
    _sig(L, "gcoo_debug_last_split", _int, [])
    _sig(L, "gcoo_debug_force_split", _int, [_int])
    _sig(L, "gcoo_debug_seg_planner", _int, [_int])
    _sig(L, "gcoo_debug_persistent", _int, [_int])
    _sig(L, "gcoo_plan_create_f32_dev", _int, [_i64, _i64, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _int,
                                                C.POINTER(_vp), _vp])
    _sig(L, "gcoo_plan_spdm_f32_dev", _int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp])
    _sig(L, "gcoo_plan_create_f64_dev", _int, [_i64, _i64, _i32, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _int,
                                                C.POINTER(_vp), _vp])
    _sig(L, "gcoo_plan_spdm_f64_dev", _int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp])
    _sig(L, "gcoo_plan_destroy", _int, [_vp])
    _sig(L, "gcoo_debug_kernel_timing", _int, [_int])
    _sig(L, "gcoo_debug_pipeline_strips", _int, [_int])
    _sig(L, "gcoo_debug_host_staging", _int, [_int])
    _sig(L, "gcoo_debug_kernel_time", _int, [C.POINTER(_dbl), C.POINTER(_i64)])
    _lib = L
    return L


def _check(rc: int):
    if rc == GCOO_OK:
        return
    msg = (lib().gcoo_last_error() or b"").decode()
    if rc == GCOO_EINVAL:
        raise ValueError(msg)
    if rc == GCOO_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _p(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(_vp)
    return C.c_void_p(a.data_ptr())  # torch tensor


def device_count() -> int:
    c = _int(0)
    lib().gcoo_device_count(C.byref(c))
    return int(c.value)


def set_device(device: int) -> None:
    _check(lib().gcoo_set_device(device))


KERNELS = {"auto": -1, "rowtile": 0, "tacc28_k192": 11, "tacc28_k160": 12,
           "tacc28_k128": 13, "tacc28_k96": 14, "tacc28_k64": 15, "tacc28_k200": 16, "tacc_v4_k216": 17, "tacc28_k176": 18,
           "tacc28_f64_k160": 20, "tacc28_f64_k96": 21, "tacc28_f64_k64": 22}


def force_kernel(which: str = "auto") -> None:
    """Test/benchmark hook: pin the fp32 multiply kernel (auto = heuristic)."""
    lib().gcoo_debug_force_kernel(KERNELS[which])


def last_kernel() -> str:
    """Test hook: the multiply kernel this thread's latest call ran (a KERNELS name)."""
    k = int(lib().gcoo_debug_last_kernel())
    return next((name for name, v in KERNELS.items() if v == k and name != "auto"), str(k))


def host_staging(on: bool = True) -> None:
    """Test hook: pageable host buffers through the library's pinned staging
    ring (default) or through the driver's own staging (off)."""
    lib().gcoo_debug_host_staging(1 if on else 0)


def last_split() -> bool:
    """Test hook: whether this thread's latest multiply ran as a two-class
    (heavy rows / light rows) split."""
    return bool(lib().gcoo_debug_last_split())


def force_split(mode: str = "auto") -> None:
    """Test hook: the two-class split of skewed matrices ("auto", "never",
    "always" = whenever the rows form two degree classes)."""
    lib().gcoo_debug_force_split({"auto": -1, "never": 0, "always": 1}[mode])


def persistent(on: bool = True) -> None:
    """Test / measurement hook: the TMEM multiply as one persistent CTA per SM
    walking the tiles, or one CTA per tile."""
    lib().gcoo_debug_persistent(1 if on else 0)


def seg_planner(on: bool = True) -> None:
    """Test hook: build even-A plans with the segment planner (default) or the
    general count / size / header / fill chain."""
    lib().gcoo_debug_seg_planner(1 if on else 0)


def kernel_timing(enable: bool = True) -> None:
    """Benchmark hook: record CUDA events around every multiply-kernel launch
    (planner kernels excluded); enable=True starts a fresh record."""
    _check(lib().gcoo_debug_kernel_timing(1 if enable else 0))


def kernel_time():
    """(total ms, launches) of the multiply kernels recorded since kernel_timing(True)."""
    t, n = _dbl(0.0), _i64(0)
    _check(lib().gcoo_debug_kernel_time(C.byref(t), C.byref(n)))
    return float(t.value), int(n.value)


def launch_count() -> int:
    """Kernels this process launched through the library (bench: gpu_launches)."""
    return int(lib().gcoo_launch_count())


# ---------------------------------------------------------------- types ----
@dataclass
class ExecConfig:
    """kernels.hpp:27-37.  workers is accepted and ignored on the GPU."""
    p: int = 4
    b: int = 64
    workers: int = 0

    def validate(self) -> None:
        if not (_pow2(self.p) and _pow2(self.b)):
            raise ValueError("ExecConfig: p and b must be powers of two")
        if self.workers < 0:
            raise ValueError("ExecConfig: workers must be >= 0")


@dataclass
class KernelStats:
    """kernels.hpp:52-65."""
    flops: int = 0
    b_loads_total: int = 0
    b_loads_reused: int = 0
    staging_fills: int = 0

    @classmethod
    def _from(cls, s: _Stats) -> "KernelStats":
        return cls(int(s.flops), int(s.b_loads_total), int(s.b_loads_reused), int(s.staging_fills))

    def __iadd__(self, o: "KernelStats"):
        self.flops += o.flops
        self.b_loads_total += o.b_loads_total
        self.b_loads_reused += o.b_loads_reused
        self.staging_fills += o.staging_fills
        return self


@dataclass
class TimingBreakdown:
    """kernels.hpp:69-72."""
    eo_seconds: float = 0.0
    kc_seconds: float = 0.0


def _pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


@dataclass
class GcooMatrix:
    """GcooMatrix<T> (matrix.hpp:176-245): p-row bands, per-band COO slices in
    (col,row) order, int32 coordinates, int64 group offsets and counts."""
    rows_dim: int
    cols_dim: int
    p: int
    values: np.ndarray
    row_idx: np.ndarray
    col_idx: np.ndarray
    g_idxes: np.ndarray
    nnz_per_group: np.ndarray

    def nnz(self) -> int:
        return int(self.values.size)

    def groups(self) -> int:
        return int(self.g_idxes.size)

    @property
    def dtype(self):
        return self.values.dtype

    def validate(self) -> None:
        """GcooMatrix::validate (matrix.hpp:206-244), vectorised on the host."""
        m, k, p = self.rows_dim, self.cols_dim, self.p
        if m < 1 or k < 1:
            raise ValueError("GcooMatrix: dimensions must be >= 1")
        if not _pow2(p):
            raise ValueError("GcooMatrix: p must be a power of two")
        g = -(-m // p)
        if self.groups() != g or self.nnz_per_group.size != g:
            raise ValueError(f"GcooMatrix: expected {g} groups")
        n = self.nnz()
        if self.row_idx.size != n or self.col_idx.size != n:
            raise ValueError("GcooMatrix: array lengths differ")
        gn = self.nnz_per_group.astype(np.int64)
        if np.any(gn < 0):
            raise ValueError("GcooMatrix: negative group size")
        off = np.concatenate([[0], np.cumsum(gn)[:-1]]) if g else np.zeros(0, np.int64)
        if not np.array_equal(off, self.g_idxes):
            raise ValueError("GcooMatrix: g_idxes inconsistent with group sizes")
        if gn.sum() != n:
            raise ValueError("GcooMatrix: group sizes do not cover all entries")
        grp = np.repeat(np.arange(g, dtype=np.int64), gn)
        r = self.row_idx.astype(np.int64)
        c = self.col_idx.astype(np.int64)
        if np.any(r // p != grp) or np.any(r >= m) or np.any(r < 0):
            raise ValueError("GcooMatrix: row outside its group band")
        if np.any(c < 0) or np.any(c >= k):
            raise ValueError("GcooMatrix: column out of range")
        if n > 1:
            same = grp[1:] == grp[:-1]
            ok = (c[:-1] < c[1:]) | ((c[:-1] == c[1:]) & (r[:-1] < r[1:]))
            if np.any(same & ~ok):
                raise ValueError("GcooMatrix: group entries not in (col,row) order (or duplicate)")


def _dense_check(a: np.ndarray) -> np.ndarray:
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("DenseMatrix: dimensions must be >= 1")
    if a.dtype not in (np.float32, np.float64):
        raise TypeError("DenseMatrix: float32 or float64 required")
    return np.ascontiguousarray(a)


# ---------------------------------------------------------- construction ---
def dense_to_gcoo(a: np.ndarray, p: int) -> GcooMatrix:
    """dense_to_gcoo (matrix.hpp:306-353) on the GPU."""
    a = _dense_check(a)
    m, k = a.shape
    L = lib()
    f = L.gcoo_dense_to_gcoo_f32 if a.dtype == np.float32 else L.gcoo_dense_to_gcoo_f64
    nnz = _i64(0)
    _check(f(m, k, p, _p(a), 0, None, None, None, None, None, C.byref(nnz)))
    n = int(nnz.value)
    g = -(-m // p)
    vals = np.empty(n, a.dtype)
    rows = np.empty(n, np.int32)
    cols = np.empty(n, np.int32)
    gi = np.empty(g, np.int64)
    gn = np.empty(g, np.int64)
    _check(f(m, k, p, _p(a), n, _p(vals), _p(rows), _p(cols), _p(gi), _p(gn), C.byref(nnz)))
    return GcooMatrix(m, k, p, vals, rows, cols, gi, gn)


def coo_to_gcoo(rows_dim: int, cols_dim: int, values: np.ndarray, row_idx: np.ndarray, col_idx: np.ndarray,
                p: int) -> GcooMatrix:
    """coo_to_gcoo (matrix.hpp:366-405) on the GPU; validates the COO like
    CooMatrix::validate (:95-115)."""
    values = np.ascontiguousarray(values)
    row_idx = np.ascontiguousarray(row_idx, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    if rows_dim < 1 or cols_dim < 1:
        raise ValueError("CooMatrix: dimensions must be >= 1")
    if not (values.size == row_idx.size == col_idx.size):
        raise ValueError("CooMatrix: array lengths differ")
    n = values.size
    g = -(-rows_dim // p) if _pow2(p) else 0
    ov = np.empty(n, values.dtype)
    orr = np.empty(n, np.int32)
    oc = np.empty(n, np.int32)
    gi = np.empty(max(g, 1), np.int64)
    gn = np.empty(max(g, 1), np.int64)
    L = lib()
    f = L.gcoo_coo_to_gcoo_f32 if values.dtype == np.float32 else L.gcoo_coo_to_gcoo_f64
    _check(f(rows_dim, cols_dim, p, n, _p(values), _p(row_idx), _p(col_idx), _p(ov), _p(orr), _p(oc), _p(gi),
             _p(gn)))
    return GcooMatrix(rows_dim, cols_dim, p, ov, orr, oc, gi[:g], gn[:g])


def csr_to_gcoo(rows_dim: int, cols_dim: int, values: np.ndarray, col_idx: np.ndarray, row_ptr: np.ndarray,
                p: int) -> GcooMatrix:
    """CSR -> GCOO (new entry point; CSR validated like CsrMatrix::validate)."""
    values = np.ascontiguousarray(values)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    if rows_dim < 1 or cols_dim < 1:
        raise ValueError("CsrMatrix: dimensions must be >= 1")
    if values.size != col_idx.size:
        raise ValueError("CsrMatrix: array lengths differ")
    if row_ptr.size != rows_dim + 1:
        raise ValueError("CsrMatrix: row_ptr must have rows_dim+1 entries")
    n = values.size
    g = -(-rows_dim // p) if _pow2(p) else 0
    ov = np.empty(n, values.dtype)
    orr = np.empty(n, np.int32)
    oc = np.empty(n, np.int32)
    gi = np.empty(max(g, 1), np.int64)
    gn = np.empty(max(g, 1), np.int64)
    L = lib()
    f = L.gcoo_csr_to_gcoo_f32 if values.dtype == np.float32 else L.gcoo_csr_to_gcoo_f64
    _check(f(rows_dim, cols_dim, p, n, _p(values), _p(col_idx), _p(row_ptr), _p(ov), _p(orr), _p(oc), _p(gi),
             _p(gn)))
    return GcooMatrix(rows_dim, cols_dim, p, ov, orr, oc, gi[:g], gn[:g])


# -------------------------------------------------------------- multiply ---
def spdm_gcoo(a: GcooMatrix, b: np.ndarray, cfg: Optional[ExecConfig] = None,
              tile_order: Optional[Sequence[int]] = None, stats: Optional[KernelStats] = None,
              out: Optional[np.ndarray] = None) -> np.ndarray:
    """spdm_gcoo (kernels.hpp:334-348): C = A_gcoo * B on the GPU.

    ``tile_order`` is the second overload's span (must have
    groups*ceil(n/b) entries).  When ``stats`` is given it is filled with the
    KernelStats for ``cfg.b``.  ``out`` (optional, e.g. pinned host memory)
    receives C instead of a fresh array."""
    cfg = cfg or ExecConfig()
    if b.ndim != 2:
        raise ValueError("DenseMatrix: 2-D operand required")
    b = np.ascontiguousarray(b, dtype=a.values.dtype)
    k_b, n = b.shape
    if out is not None:
        if out.shape != (a.rows_dim, n) or out.dtype != a.values.dtype or not out.flags.c_contiguous:
            raise ValueError("spdm_gcoo: out has the wrong shape/dtype/layout")
        c = out
    else:
        c = np.empty((a.rows_dim, n), dtype=a.values.dtype)
    to = None if tile_order is None else np.ascontiguousarray(np.asarray(tile_order, dtype=np.int64))
    st = _Stats()
    L = lib()
    f = L.gcoo_spdm_f32 if a.values.dtype == np.float32 else L.gcoo_spdm_f64
    _check(f(a.rows_dim, a.cols_dim, n, a.p, cfg.p, cfg.b, k_b, a.nnz(), _p(a.values), _p(a.row_idx),
             _p(a.col_idx), a.groups(), _p(a.g_idxes), _p(a.nnz_per_group), _p(b), _p(c),
             C.byref(st) if stats is not None else None, _p(to), 0 if to is None else to.size))
    if stats is not None:
        s = KernelStats._from(st)
        stats.flops, stats.b_loads_total, stats.b_loads_reused, stats.staging_fills = (
            s.flops, s.b_loads_total, s.b_loads_reused, s.staging_fills)
    return c


def spdm_gcoo_auto(a: np.ndarray, b: np.ndarray, cfg: Optional[ExecConfig] = None,
                   timing: Optional[TimingBreakdown] = None, stats: Optional[KernelStats] = None) -> np.ndarray:
    """spdm_gcoo_auto (kernels.hpp:353-367): EO = dense_to_gcoo, KC = spdm_gcoo,
    with the GCOO kept on the device between them (gcoo_spdm_auto_*): only A,
    B and C cross PCIe."""
    cfg = cfg or ExecConfig()
    cfg.validate()
    a = _dense_check(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    if b.ndim != 2 or b.shape[0] != a.shape[1]:
        raise ValueError("spdm_gcoo: inner dimensions differ")
    c = np.empty((a.shape[0], b.shape[1]), a.dtype)
    st, eo, kc = _Stats(), _dbl(0.0), _dbl(0.0)
    _check(getattr(lib(), f"gcoo_spdm_auto_{_sfx(a.dtype)}")(a.shape[0], a.shape[1], b.shape[1], cfg.p, cfg.b, _p(a),
                                                             _p(b), _p(c), C.byref(st) if stats is not None else None,
                                                             C.byref(eo), C.byref(kc)))
    if timing is not None:
        timing.eo_seconds, timing.kc_seconds = float(eo.value), float(kc.value)
    if stats is not None:
        s = KernelStats._from(st)
        stats.flops, stats.b_loads_total, stats.b_loads_reused, stats.staging_fills = (
            s.flops, s.b_loads_total, s.b_loads_reused, s.staging_fills)
    return c


# ------------------------------------------- baselines ---
def _sfx(dtype) -> str:
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise TypeError("float32 or float64 required")


def spdm_csr(rows_dim: int, cols_dim: int, values: np.ndarray, col_idx: np.ndarray, row_ptr: np.ndarray,
             b: np.ndarray, cfg: Optional[ExecConfig] = None) -> np.ndarray:
    """spdm_csr (kernels.hpp:163-184) on the GPU: row-split, each row's chain in
    CSR order (no grouping or staging — the paper's CSR baseline)."""
    (cfg or ExecConfig()).validate()
    b = np.ascontiguousarray(b)
    if b.ndim != 2 or b.shape[0] != cols_dim:
        raise ValueError("spdm_csr: inner dimensions differ")
    values = np.ascontiguousarray(values, dtype=b.dtype)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    if row_ptr.size != rows_dim + 1 or col_idx.size != values.size:
        raise ValueError("spdm_csr: inconsistent CSR arrays")
    c = np.empty((rows_dim, b.shape[1]), b.dtype)
    _check(getattr(lib(), f"gcoo_spdm_csr_{_sfx(b.dtype)}")(rows_dim, cols_dim, b.shape[1], values.size, _p(values),
                                                            _p(col_idx), _p(row_ptr), _p(b), _p(c)))
    return c


def spdm_coo(rows_dim: int, cols_dim: int, values: np.ndarray, row_idx: np.ndarray, col_idx: np.ndarray,
             b: np.ndarray, cfg: Optional[ExecConfig] = None) -> np.ndarray:
    """spdm_coo (kernels.hpp:193-232) on the GPU: any entry order (each row's
    chain in array order), the ungrouped ablation of GCOO."""
    (cfg or ExecConfig()).validate()
    b = np.ascontiguousarray(b)
    if b.ndim != 2 or b.shape[0] != cols_dim:
        raise ValueError("spdm_coo: inner dimensions differ")
    values = np.ascontiguousarray(values, dtype=b.dtype)
    row_idx = np.ascontiguousarray(row_idx, dtype=np.int32)
    col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
    if not (values.size == row_idx.size == col_idx.size):
        raise ValueError("spdm_coo: inconsistent COO arrays")
    c = np.empty((rows_dim, b.shape[1]), b.dtype)
    _check(getattr(lib(), f"gcoo_spdm_coo_{_sfx(b.dtype)}")(rows_dim, cols_dim, b.shape[1], values.size, _p(values),
                                                            _p(row_idx), _p(col_idx), _p(b), _p(c)))
    return c


def gemm_dense_blocked(a: np.ndarray, b: np.ndarray, cfg: Optional[ExecConfig] = None) -> np.ndarray:
    """gemm_dense_blocked (kernels.hpp:107-155) on the GPU: every element summed
    over l ascending (the dense crossover baseline)."""
    (cfg or ExecConfig()).validate()
    a = _dense_check(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    if b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError("gemm_dense_blocked: inner dimensions differ")
    c = np.empty((a.shape[0], b.shape[1]), a.dtype)
    _check(getattr(lib(), f"gcoo_gemm_dense_{_sfx(a.dtype)}")(a.shape[0], a.shape[1], b.shape[1], _p(a), _p(b),
                                                              _p(c)))
    return c


def spdm_csr_dev(rows_dim: int, cols_dim: int, values, col_idx, row_ptr, b, c, flavor: int = FLAVOR_FMA,
                 stream=None) -> None:
    """Stream-ordered spdm_csr on device tensors (b: k x n, c: m x n, unit column stride)."""
    import torch
    values = _dev_array("values", values, (torch.float32, torch.float64))
    col_idx = _dev_array("col_idx", col_idx, (torch.int32,))
    row_ptr = _dev_array("row_ptr", row_ptr, (torch.int64,))
    _check_dense_pair(values.dtype, b, c, rows_dim, cols_dim)
    f = getattr(lib(), f"gcoo_spdm_csr_{'f64' if values.dtype == torch.float64 else 'f32'}_dev")
    _check(f(rows_dim, cols_dim, b.shape[1], values.numel(), _p(values), _p(col_idx), _p(row_ptr), _p(b), b.stride(0),
             _p(c), c.stride(0), flavor, _stream_ptr(stream)))


def spdm_coo_dev(rows_dim: int, cols_dim: int, values, row_idx, col_idx, b, c, flavor: int = FLAVOR_FMA,
                 stream=None) -> None:
    """Stream-ordered spdm_coo on device tensors (any entry order)."""
    import torch
    values = _dev_array("values", values, (torch.float32, torch.float64))
    row_idx = _dev_array("row_idx", row_idx, (torch.int32,))
    col_idx = _dev_array("col_idx", col_idx, (torch.int32,))
    _check_dense_pair(values.dtype, b, c, rows_dim, cols_dim)
    f = getattr(lib(), f"gcoo_spdm_coo_{'f64' if values.dtype == torch.float64 else 'f32'}_dev")
    _check(f(rows_dim, cols_dim, b.shape[1], values.numel(), _p(values), _p(row_idx), _p(col_idx), _p(b), b.stride(0),
             _p(c), c.stride(0), flavor, _stream_ptr(stream)))


def gemm_dense_dev(a, b, c, flavor: int = FLAVOR_FMA, stream=None) -> None:
    """Stream-ordered gemm_dense_blocked on device tensors."""
    import torch
    a = _dev_array("A", a, (torch.float32, torch.float64))
    if a.dim() != 2:
        raise ValueError("gemm_dense_blocked: A must be 2-D")
    _check_dense_pair(a.dtype, b, c, a.shape[0], a.shape[1])
    f = getattr(lib(), f"gcoo_gemm_dense_{'f64' if a.dtype == torch.float64 else 'f32'}_dev")
    _check(f(a.shape[0], a.shape[1], b.shape[1], _p(a), a.stride(0), _p(b), b.stride(0), _p(c), c.stride(0), flavor,
             _stream_ptr(stream)))


def _check_dense_pair(dtype, b, c, m: int, k: int) -> None:
    for name, t in (("B", b), ("C", c)):
        if t.dim() != 2 or t.dtype != dtype or not t.is_cuda or t.stride(1) != 1:
            raise ValueError(f"{name}: 2-D CUDA tensor of the operands' dtype with unit column stride required")
    if b.shape[0] != k or c.shape[0] != m or c.shape[1] != b.shape[1]:
        raise ValueError("inner dimensions differ / C has the wrong shape")


# ------------------------------------------------------ device-resident ----
@dataclass
class DeviceGcoo:
    """GCOO arrays resident in HBM (torch tensors on one CUDA device)."""
    rows_dim: int
    cols_dim: int
    p: int
    values: "object"
    row_idx: "object"
    col_idx: "object"
    g_idxes: "object"
    nnz_per_group: "object"

    @classmethod
    def from_host(cls, g: GcooMatrix, device="cuda") -> "DeviceGcoo":
        import torch
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(device)
        return cls(g.rows_dim, g.cols_dim, g.p, t(g.values), t(g.row_idx), t(g.col_idx), t(g.g_idxes),
                   t(g.nnz_per_group))

    def nnz(self) -> int:
        return int(self.values.numel())

    def groups(self) -> int:
        return int(self.g_idxes.numel())

    def to_host(self) -> GcooMatrix:
        h = lambda x: x.cpu().numpy()
        return GcooMatrix(self.rows_dim, self.cols_dim, self.p, h(self.values), h(self.row_idx),
                          h(self.col_idx), h(self.g_idxes), h(self.nnz_per_group))


class _Traffic(C.Structure):
    _fields_ = [(f, _u64) for f in ("n_dm", "n_l2", "n_shm", "tex_l1_trans", "flops")]


class _TrafficDetail(C.Structure):
    _fields_ = [(f, _u64) for f in ("b_element_loads", "b_element_reused", "staged_entries",
                                     "b_load_transactions", "sparse_transactions", "store_transactions")]


def model_traffic_dev(a: "DeviceGcoo", n: int, cfg: Optional["ExecConfig"] = None, infinite_l2: bool = False,
                      csr: bool = False, stream=None) -> dict:
    """The reference's model_gcoo_traffic (csr=False) / model_csr_traffic
    (csr=True) (traffic.cpp:43-197) of A's pattern times a dense k x n
    operand, evaluated on the GPU: TrafficReport + TrafficDetail counters as
    one dict (exact, equal to the reference's).  cfg.p must be A's p."""
    cfg = cfg or ExecConfig(p=a.p)
    if cfg.p != a.p:
        raise ValueError("traffic model: matrix grouped with a different p")
    r, d = _Traffic(), _TrafficDetail()
    _check(lib().gcoo_model_traffic_dev(1 if csr else 0, a.rows_dim, a.cols_dim, n, a.p, cfg.b, a.nnz(),
                                         _p(a.row_idx), _p(a.col_idx), a.groups(), _p(a.g_idxes),
                                         _p(a.nnz_per_group), 1 if infinite_l2 else 0, C.byref(r), C.byref(d),
                                         _stream_ptr(stream)))
    return {**{f: int(getattr(r, f)) for f, _ in _Traffic._fields_},
            **{f: int(getattr(d, f)) for f, _ in _TrafficDetail._fields_}}


# RooflineModel profiles (traffic.cpp:226-233) plus this pool's B200, measured:
# FP32 FFMA peak (tools/microbench, profiles/r01_microbench.json) and HBM copy
# bandwidth (MEASURED_PEAKS.json).
ROOFLINE_PROFILES = {
    "gtx980": (4.981e12, 224e9),
    "titanx": (10.97e12, 433e9),
    "p100": (9.5e12, 732e9),
    "b200": (72.47e12, 6524.3e9),  # = gcoo_roofline_b200 (include/gcoo/roofline_b200.hpp)
}


def operational_intensity(rep: dict, bytes_per_transaction: int = 128) -> float:
    """operational_intensity (traffic.cpp:201-208): flops per DRAM byte."""
    if rep["flops"] == 0:
        return 0.0
    if rep["n_dm"] == 0 or bytes_per_transaction <= 0:
        raise ValueError("operational_intensity: undefined without DRAM traffic")
    return rep["flops"] / (rep["n_dm"] * bytes_per_transaction)


def roofline_throughput(r: float, profile: str = "b200") -> float:
    """roofline_throughput (traffic.cpp:210-213): min(peak, r * bandwidth), FLOP/s."""
    if r < 0:
        raise ValueError("roofline_throughput: negative intensity")
    peak, bw = ROOFLINE_PROFILES[profile.lower()]
    return min(peak, r * bw)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def _check_device_gcoo(a: "DeviceGcoo") -> None:
    """A's device arrays: one CUDA device, contiguous, fp32/fp64 values, int32
    coordinates, int64 group arrays — anything else would be read as garbage
    by the C ABI, so it is rejected here."""
    import torch
    if a.values.dtype not in (torch.float32, torch.float64):
        raise ValueError("DeviceGcoo: values must be float32 or float64")
    for name, t, dt in (("values", a.values, a.values.dtype), ("row_idx", a.row_idx, torch.int32),
                        ("col_idx", a.col_idx, torch.int32), ("g_idxes", a.g_idxes, torch.int64),
                        ("nnz_per_group", a.nnz_per_group, torch.int64)):
        if t.dtype != dt:
            raise ValueError(f"DeviceGcoo: {name} must be {dt}")
        if not t.is_cuda or t.device != a.values.device:
            raise ValueError(f"DeviceGcoo: {name} must live on the values' CUDA device")
        if not t.is_contiguous():
            raise ValueError(f"DeviceGcoo: {name} must be contiguous")


def _check_operands(a: "DeviceGcoo", b, c) -> None:
    """B (k x n) and C (m x n): A's dtype and device, 2-D, unit column stride."""
    _check_device_gcoo(a)
    for name, t in (("B", b), ("C", c)):
        if t.dim() != 2:
            raise ValueError(f"spdm_gcoo_dev: {name} must be 2-D")
        if t.dtype != a.values.dtype:
            raise ValueError(f"spdm_gcoo_dev: {name} dtype {t.dtype} differs from A's {a.values.dtype}")
        if t.device != a.values.device:
            raise ValueError(f"spdm_gcoo_dev: {name} is not on A's device")
        if t.stride(1) != 1:
            raise ValueError("spdm_gcoo_dev: B and C need unit column stride")


def spdm_gcoo_dev(a: DeviceGcoo, b, c, cfg: Optional[ExecConfig] = None, flavor: int = FLAVOR_FMA,
                  stream=None, stats: Optional[KernelStats] = None) -> None:
    """Stream-ordered C = A * B on device tensors (b: k x n, c: m x n; a
    column shard may be a strided view with unit column stride)."""
    import torch
    cfg = cfg or ExecConfig(p=a.p)
    n = b.shape[1]
    _check_operands(a, b, c)
    if b.shape[0] != a.cols_dim:
        raise ValueError("spdm_gcoo: inner dimensions differ")
    if cfg.p != a.p:
        raise ValueError("spdm_gcoo: matrix grouped with a different p")
    if c.shape[0] != a.rows_dim or c.shape[1] != n:
        raise ValueError("spdm_gcoo_dev: C has the wrong shape")
    st = _Stats()
    L = lib()
    f = L.gcoo_spdm_f32_dev if a.values.dtype == torch.float32 else L.gcoo_spdm_f64_dev
    _check(f(a.rows_dim, a.cols_dim, n, a.p, cfg.b, a.nnz(), _p(a.values), _p(a.row_idx), _p(a.col_idx),
             a.groups(), _p(a.g_idxes), _p(a.nnz_per_group), _p(b), b.stride(0), _p(c), c.stride(0),
             C.byref(st) if stats is not None else None, flavor, _stream_ptr(stream)))
    if stats is not None:
        s = KernelStats._from(st)
        stats.flops, stats.b_loads_total, stats.b_loads_reused, stats.staging_fills = (
            s.flops, s.b_loads_total, s.b_loads_reused, s.staging_fills)


class SpdmPlan:
    """Plan / execute split (C ABI gcoo_plan_*): the multiply's record stream
    built once from a DeviceGcoo (fp32 or fp64), then `run(b, c)` per dense operand —
    the same bits as spdm_gcoo_dev without the ~35 us planner per call.  Keeps
    a reference to A's tensors; close() (or garbage collection) frees it."""

    def __init__(self, a: "DeviceGcoo", flavor: int = FLAVOR_FMA, stream=None):
        import torch
        self.a = a
        self._h = _vp()
        _check_device_gcoo(a)
        self._f64 = a.values.dtype == torch.float64
        create = lib().gcoo_plan_create_f64_dev if self._f64 else lib().gcoo_plan_create_f32_dev
        _check(create(a.rows_dim, a.cols_dim, a.p, a.nnz(), _p(a.values), _p(a.row_idx), _p(a.col_idx), a.groups(),
                      _p(a.g_idxes), _p(a.nnz_per_group), flavor, C.byref(self._h), _stream_ptr(stream)))

    def run(self, b, c, stream=None) -> None:
        import torch
        _check_operands(self.a, b, c)
        if b.shape[0] != self.a.cols_dim or c.shape[0] != self.a.rows_dim or c.shape[1] != b.shape[1]:
            raise ValueError("spdm_gcoo: operand shapes do not match the plan's A")
        if self._h is None:
            raise ValueError("SpdmPlan: closed")
        if (b.dtype == torch.float64) != self._f64 or c.dtype != b.dtype:
            raise ValueError("SpdmPlan: operand dtype differs from the plan's")
        run = lib().gcoo_plan_spdm_f64_dev if self._f64 else lib().gcoo_plan_spdm_f32_dev
        _check(run(self._h, b.shape[1], _p(b), b.stride(0), _p(c), c.stride(0), _stream_ptr(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and _lib is not None:
            lib().gcoo_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def _dev_array(name: str, t, dtypes):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype not in dtypes:
        raise ValueError(f"{name} must be one of {dtypes}, got {t.dtype}")
    return t.contiguous()


def coo_to_gcoo_dev(rows_dim: int, cols_dim: int, values, row_idx, col_idx, p: int, stream=None) -> DeviceGcoo:
    """coo_to_gcoo (matrix.hpp:366-405) on device arrays (fp32 or fp64 values,
    int32 coordinates, one device); validated like CooMatrix::validate."""
    import torch
    values = _dev_array("values", values, (torch.float32, torch.float64))
    row_idx = _dev_array("row_idx", row_idx, (torch.int32,))
    col_idx = _dev_array("col_idx", col_idx, (torch.int32,))
    if not (values.numel() == row_idx.numel() == col_idx.numel()):
        raise ValueError("CooMatrix: array lengths differ")
    if row_idx.device != values.device or col_idx.device != values.device:
        raise ValueError("coo_to_gcoo_dev: arrays on different devices")
    n = values.numel()
    g = -(-rows_dim // p) if _pow2(p) else 1
    dev = values.device
    ov = torch.empty(n, dtype=values.dtype, device=dev)
    orr = torch.empty(n, dtype=torch.int32, device=dev)
    oc = torch.empty(n, dtype=torch.int32, device=dev)
    gi = torch.empty(g, dtype=torch.int64, device=dev)
    gn = torch.empty(g, dtype=torch.int64, device=dev)
    sp = _stream_ptr(stream)
    L = lib()
    f = L.gcoo_coo_to_gcoo_f64_dev if values.dtype == torch.float64 else L.gcoo_coo_to_gcoo_f32_dev
    _check(f(rows_dim, cols_dim, p, n, _p(values), _p(row_idx), _p(col_idx), _p(ov), _p(orr), _p(oc), _p(gi),
             _p(gn), sp))
    # setup routine: finish before the arrays are handed to other streams
    _check(L.gcoo_stream_sync(sp))
    return DeviceGcoo(rows_dim, cols_dim, p, ov, orr, oc, gi, gn)


def csr_to_gcoo_dev(rows_dim: int, cols_dim: int, values, col_idx, row_ptr, p: int, stream=None) -> DeviceGcoo:
    """CSR -> GCOO on device arrays (int64 row_ptr[rows_dim+1], int32 columns);
    validated like CsrMatrix::validate (matrix.hpp:122-165)."""
    import torch
    values = _dev_array("values", values, (torch.float32, torch.float64))
    col_idx = _dev_array("col_idx", col_idx, (torch.int32,))
    row_ptr = _dev_array("row_ptr", row_ptr, (torch.int64,))
    if values.numel() != col_idx.numel():
        raise ValueError("CsrMatrix: array lengths differ")
    if row_ptr.numel() != rows_dim + 1:
        raise ValueError("CsrMatrix: row_ptr must have rows_dim+1 entries")
    n = values.numel()
    g = -(-rows_dim // p) if _pow2(p) else 1
    dev = values.device
    ov = torch.empty(n, dtype=values.dtype, device=dev)
    orr = torch.empty(n, dtype=torch.int32, device=dev)
    oc = torch.empty(n, dtype=torch.int32, device=dev)
    gi = torch.empty(g, dtype=torch.int64, device=dev)
    gn = torch.empty(g, dtype=torch.int64, device=dev)
    sp = _stream_ptr(stream)
    L = lib()
    f = L.gcoo_csr_to_gcoo_f64_dev if values.dtype == torch.float64 else L.gcoo_csr_to_gcoo_f32_dev
    _check(f(rows_dim, cols_dim, p, n, _p(values), _p(col_idx), _p(row_ptr), _p(ov), _p(orr), _p(oc), _p(gi),
             _p(gn), sp))
    _check(L.gcoo_stream_sync(sp))
    return DeviceGcoo(rows_dim, cols_dim, p, ov, orr, oc, gi, gn)


def dense_to_gcoo_dev(a, p: int, stream=None) -> DeviceGcoo:
    """dense_to_gcoo (matrix.hpp:306-353) on a device matrix (fp32 or fp64)."""
    import torch
    a = _dev_array("A", a, (torch.float32, torch.float64))
    if a.dim() != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("DenseMatrix: dimensions must be >= 1")
    m, k = a.shape
    dev = a.device
    if not _pow2(p):
        raise ValueError("dense_to_gcoo: p must be a power of two")
    g = -(-m // p)
    gi = torch.empty(g, dtype=torch.int64, device=dev)
    gn = torch.empty(g, dtype=torch.int64, device=dev)
    nnz = _i64(0)
    L = lib()
    f = L.gcoo_dense_to_gcoo_f64_dev if a.dtype == torch.float64 else L.gcoo_dense_to_gcoo_f32_dev
    sp = _stream_ptr(stream)
    _check(f(m, k, p, _p(a), 0, None, None, None, _p(gi), _p(gn), C.byref(nnz), sp))
    n = int(nnz.value)
    ov = torch.empty(n, dtype=a.dtype, device=dev)
    orr = torch.empty(n, dtype=torch.int32, device=dev)
    oc = torch.empty(n, dtype=torch.int32, device=dev)
    _check(f(m, k, p, _p(a), n, _p(ov), _p(orr), _p(oc), _p(gi), _p(gn), C.byref(nnz), sp))
    # setup routine: finish before the arrays are handed to other streams
    _check(L.gcoo_stream_sync(sp))
    return DeviceGcoo(m, k, p, ov, orr, oc, gi, gn)


# ------------------------------------------------------- synthetic inputs ---
def derive_seed(base: int, salt_a: int, salt_b: int = 0) -> int:
    return int(lib().gcoo_derive_seed(base, salt_a, salt_b))


def generate_uniform_sparse(n: int, s: float, seed: int) -> np.ndarray:
    """generate_uniform_sparse<float> (io.hpp:129-145), bit-identical."""
    out = np.empty((n, n), np.float32)
    _check(lib().gcoo_generate_uniform_sparse_f32(n, s, seed, _p(out)))
    return out


def generate_uniform_sparse_coo(n: int, s: float, seed: int):
    """Same sample as generate_uniform_sparse, as row-major COO arrays."""
    nnz = _i64(0)
    L = lib()
    _check(L.gcoo_generate_uniform_sparse_coo_f32(n, s, seed, 0, None, None, None, C.byref(nnz)))
    k = int(nnz.value)
    v = np.empty(k, np.float32)
    r = np.empty(k, np.int32)
    c = np.empty(k, np.int32)
    _check(L.gcoo_generate_uniform_sparse_coo_f32(n, s, seed, k, _p(v), _p(r), _p(c), C.byref(nnz)))
    return v, r, c


def generate_powerlaw_coo(n: int, s: float, alpha: float, seed: int):
    nnz = _i64(0)
    L = lib()
    _check(L.gcoo_generate_powerlaw_coo_f32(n, s, alpha, seed, 0, None, None, None, C.byref(nnz)))
    k = int(nnz.value)
    v = np.empty(k, np.float32)
    r = np.empty(k, np.int32)
    c = np.empty(k, np.int32)
    _check(L.gcoo_generate_powerlaw_coo_f32(n, s, alpha, seed, k, _p(v), _p(r), _p(c), C.byref(nnz)))
    return v, r, c


__all__ = [
    "ExecConfig", "KernelStats", "TimingBreakdown", "GcooMatrix", "DeviceGcoo", "dense_to_gcoo", "coo_to_gcoo",
    "csr_to_gcoo", "spdm_gcoo", "spdm_gcoo_auto", "spdm_gcoo_dev", "coo_to_gcoo_dev", "csr_to_gcoo_dev",
    "dense_to_gcoo_dev", "SpdmPlan", "spdm_csr", "spdm_coo", "gemm_dense_blocked", "spdm_csr_dev", "spdm_coo_dev",
    "gemm_dense_dev",
    "derive_seed", "generate_uniform_sparse", "generate_uniform_sparse_coo", "generate_powerlaw_coo",
    "device_count", "set_device", "launch_count", "lib", "FLAVOR_FMA", "FLAVOR_MUL_ADD",
    "read_matrix_market", "write_matrix_market", "read_matrix_market_gcoo_dev", "CooMatrix", "ParseError",
]

# MatrixMarket I/O (io.hpp:21-109), as in the reference's gcoo namespace
from .mmio import CooMatrix, ParseError, read_matrix_market, read_matrix_market_gcoo_dev, write_matrix_market  # noqa: E402
