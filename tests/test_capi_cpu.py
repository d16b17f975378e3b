"""CPU-side checks of the product boundary (no device work).

* libgcoo_cuda.so loads and exports every symbol include/gcoo_capi.h declares;
* the harness generators are bit-identical to the oracle's (and hence to the
  reference's) streams;
* argument validation raises the reference's exception class before any
  device work (kernels.hpp:32-36, :244-254; matrix.hpp:308-309);
* the Python GcooMatrix.validate mirrors GcooMatrix::validate
  (test_matrix.cpp:78-102).
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "gcoo_capi.h")).read()
    return sorted(set(re.findall(r"\b(gcoo_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(gcoo):
    lib = ctypes.CDLL(gcoo.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert gcoo.lib().gcoo_abi_version() == 1


def test_generators_match_oracle(gcoo, oracle):
    for n, s, seed in [(1, 0.0, 1), (33, 0.5, 2), (64, 0.99, 3), (200, 0.9, 4), (90, 0.3, 5)]:
        assert np.array_equal(gcoo.generate_uniform_sparse(n, s, seed), oracle.uniform_sparse(n, s, seed))
        v, r, c = gcoo.generate_uniform_sparse_coo(n, s, seed)
        v2, r2, c2 = oracle.uniform_sparse_coo(n, s, seed)
        assert np.array_equal(v, v2) and np.array_equal(r, r2) and np.array_equal(c, c2)
        assert gcoo.derive_seed(seed, n, 0xB) == oracle.derive_seed(seed, n, 0xB)
    v, r, c = gcoo.generate_powerlaw_coo(777, 0.98, 1.0, 3)
    v2, r2, c2 = oracle.powerlaw_coo(777, 0.98, 1.0, 3)
    assert np.array_equal(v, v2) and np.array_equal(r, r2) and np.array_equal(c, c2)


def test_generator_matches_golden_hash(gcoo, oracle, golden_hashes):
    ent = golden_hashes["n512_s0.95"]
    assert oracle.fnv(gcoo.generate_uniform_sparse(512, 0.95, 1)) == ent["A_fnv"]
    assert gcoo.derive_seed(1, 512, 0xB) == ent["b_seed"]


def _small_gcoo(gcoo, oracle):
    a = np.zeros((4, 4), np.float32)
    a[0, 0], a[0, 3], a[1, 1], a[2, 0], a[3, 2], a[3, 3] = 7, 8, 10, 9, 6, 3
    g = oracle.dense_to_gcoo(a, 2)
    return gcoo.GcooMatrix(4, 4, 2, g.values, g.row_idx, g.col_idx, g.g_idxes, g.nnz_per_group)


def test_spdm_validation_raises_before_device_work(gcoo, oracle):
    # test_kernels.cpp:185-198 — only the exception TYPE is part of the contract
    g = _small_gcoo(gcoo, oracle)
    eye4 = np.eye(4, dtype=np.float32)
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo(g, eye4, gcoo.ExecConfig())  # p=4 vs grouped with p=2
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo(g, np.eye(5, dtype=np.float32), gcoo.ExecConfig(p=2))
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo(g, eye4, gcoo.ExecConfig(p=2, b=3))
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo(g, eye4, gcoo.ExecConfig(p=2), tile_order=[0, 1, 2])
    with pytest.raises(ValueError):
        gcoo.ExecConfig(p=3).validate()


def test_dense_to_gcoo_pow2_rejected_before_device_work(gcoo):
    a = np.eye(4, dtype=np.float32)
    for p in (3, 0, -2, 6):
        with pytest.raises(ValueError):
            gcoo.dense_to_gcoo(a, p)


def test_host_gcoo_validate(gcoo, oracle):
    G = gcoo.GcooMatrix
    _small_gcoo(gcoo, oracle).validate()
    i32 = lambda *x: np.array(x, np.int32)
    i64 = lambda *x: np.array(x, np.int64)
    f32 = lambda *x: np.array(x, np.float32)
    bad = [
        G(4, 4, 2, f32(1), i32(0), i32(0), i64(0, 2), i64(1, 0)),  # inconsistent offsets
        G(4, 4, 2, f32(1), i32(3), i32(0), i64(0, 1), i64(1, 0)),  # row outside band
        G(4, 4, 2, f32(1, 2), i32(0, 1), i32(3, 0), i64(0, 2), i64(2, 0)),  # (row,col) order
        G(4, 4, 3, f32(1), i32(0), i32(0), i64(0, 1), i64(1, 0)),  # p not pow2
    ]
    for g in bad:
        with pytest.raises(ValueError):
            g.validate()


def test_no_oracle_in_product():
    """The product package must never import or link the checker."""
    pkg = os.path.join(ROOT, "paper_2005_14469_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "gcoo_oracle" not in txt and "libgcoo_ref" not in txt, f


def test_roofline_profiles(gcoo):
    """RooflineModel profiles + helpers (traffic.cpp:201-233) with the measured b200 entry."""
    rep = {"flops": 1000, "n_dm": 10}
    assert gcoo.operational_intensity(rep, 128) == 1000 / 1280
    assert gcoo.roofline_throughput(1.0, "P100") == 732e9  # bandwidth-bound (traffic.cpp:210-213)
    assert gcoo.roofline_throughput(1e6, "b200") == gcoo.ROOFLINE_PROFILES["b200"][0]
