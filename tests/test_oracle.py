"""Pin the CPU oracle (oracle/gcoo_oracle.c) before trusting it.

* against the reference's own known-answer tests (test_matrix.cpp:49-68,
  test_kernels.cpp:91-123) restated here;
* against the golden fixtures generated from the reference (tests/golden);
* against the reference library itself (oracle/_ref), on seeded random cases,
  when it is built (always in the build container; the prebuilt .so also
  travels to the GPU box).
"""
import numpy as np
import pytest

FIELDS = ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group")


def example4x4():
    a = np.zeros((4, 4), np.float32)
    a[0, 0], a[0, 3], a[1, 1], a[2, 0], a[3, 2], a[3, 3] = 7, 8, 10, 9, 6, 3
    return a


def test_gcoo_4x4_p2_known_answer(oracle):
    # test_matrix.cpp:49-58
    g = oracle.dense_to_gcoo(example4x4(), 2)
    assert g.groups == 2
    assert g.g_idxes.tolist() == [0, 3]
    assert g.nnz_per_group.tolist() == [3, 3]
    assert g.values.tolist() == [7, 10, 8, 9, 6, 3]
    assert g.row_idx.tolist() == [0, 1, 0, 2, 3, 3]
    assert g.col_idx.tolist() == [0, 1, 3, 0, 2, 3]
    assert oracle.validate(g) == 0


def test_empty_leading_group(oracle):
    # test_matrix.cpp:60-68
    a = np.zeros((5, 5), np.float32)
    a[4, :] = 1
    g = oracle.dense_to_gcoo(a, 4)
    assert g.nnz_per_group.tolist() == [0, 5]
    assert g.g_idxes.tolist() == [0, 0]
    assert (g.row_idx == 4).all()


def test_pow2_rejected(oracle):
    for p in (3, 0, -2, 6):
        with pytest.raises(ValueError):
            oracle.dense_to_gcoo(example4x4(), p)


def test_identity_and_flops(oracle):
    # test_kernels.cpp:91-101
    g = oracle.dense_to_gcoo(example4x4(), 2)
    c, st = oracle.spdm(g, np.eye(4, dtype=np.float32), b=4)
    assert np.array_equal(c, example4x4())
    assert st[0] == 48


def test_reuse_accounting_hand_traced(oracle):
    # test_kernels.cpp:103-123
    a = np.zeros((4, 4), np.float32)
    a[0, 1], a[1, 1] = 2, 5
    g = oracle.dense_to_gcoo(a, 2)
    c, st = oracle.spdm(g, np.eye(4, dtype=np.float32), b=4)
    assert st == (16, 4, 4, 2)  # flops, total, reused, staging
    assert c[0, 1] == 2 and c[1, 1] == 5 and np.count_nonzero(c) == 2


def test_stats_identities(oracle):
    # test_kernels.cpp:125-155: total + reused == flops/2; diagonal => reused 0
    rng = np.random.default_rng(41)
    for _ in range(20):
        m, k, n = rng.integers(1, 129, size=3)
        p, b = 1 << int(rng.integers(0, 5)), 1 << int(rng.integers(0, 7))
        a = np.where(rng.random((m, k)) < 0.15, 1 - rng.random((m, k)), 0).astype(np.float32)
        g = oracle.dense_to_gcoo(a, p)
        _, st = oracle.spdm(g, np.ones((k, n), np.float32), b=b)
        assert st[1] + st[2] == st[0] // 2
        assert oracle.stats(g, int(n), b) == st
    for n in (1, 2, 5, 16, 64, 129):
        g = oracle.dense_to_gcoo(np.eye(n, dtype=np.float32) * 1.5, 4)
        _, st = oracle.spdm(g, np.ones((n, n), np.float32), b=64)
        assert st[2] == 0


def test_oracle_vs_golden_small(oracle, golden_small):
    names = sorted({k.split(".")[0] for k in golden_small})
    assert len(names) >= 10
    for name in names:
        a, b = golden_small[f"{name}.A"], golden_small[f"{name}.B"]
        for p in (1, 2, 4, 8, 64):
            g = oracle.dense_to_gcoo(a, p)
            for f in FIELDS:
                assert np.array_equal(getattr(g, f), golden_small[f"{name}.p{p}.{f}"]), (name, p, f)
        g = oracle.dense_to_gcoo(a, 4)
        c_mad, _ = oracle.spdm(g, b, 64, fma=False)
        c_fma, _ = oracle.spdm(g, b, 64, fma=True)
        assert np.array_equal(c_mad, golden_small[f"{name}.C_mad"]), name
        assert np.array_equal(c_fma, golden_small[f"{name}.C_fma"]), name
        for bb in (1, 4, 64, 256):
            assert oracle.stats(g, b.shape[1], bb) == tuple(int(x) for x in golden_small[f"{name}.stats_b{bb}"])


def test_oracle_vs_golden_hashes_n512(oracle, golden_hashes):
    ent = golden_hashes["n512_s0.95"]
    a = oracle.uniform_sparse(512, 0.95, 1)
    b = oracle.uniform_sparse(512, 0.0, oracle.derive_seed(1, 512, 0xB))
    assert oracle.derive_seed(1, 512, 0xB) == ent["b_seed"]
    assert oracle.fnv(a) == ent["A_fnv"] and oracle.fnv(b) == ent["B_fnv"]
    g = oracle.dense_to_gcoo(a, 4)
    for f in FIELDS:
        assert oracle.fnv(getattr(g, f)) == ent["p4"][f]
    c, st = oracle.spdm(g, b, 64, fma=False)
    assert oracle.fnv(c) == ent["C_mad"]["fnv"]
    assert list(st) == ent["stats_p4_b64"]
    c, _ = oracle.spdm(g, b, 64, fma=True)
    assert oracle.fnv(c) == ent["C_fma"]["fnv"]


def test_survey_appendix_b_gcoo_hashes(oracle, golden_hashes):
    # SURVEY.md Appendix B GCOO hashes agree with the regenerated fixtures
    assert golden_hashes["n512_s0.95"]["p4"]["values"] == "406a99aa"
    assert golden_hashes["n8000_s0.99"]["p4"]["col_idx"] == "88e5c32e"
    assert golden_hashes["n8000_s0.99"]["p64"]["values"] == "794f5406"
    assert golden_hashes["n8000_s0.99"]["stats_p4_b64"] == [10240000000, 5045760000, 74240000, 80000000]


def test_coo_to_gcoo_matches_dense(oracle):
    rng = np.random.default_rng(19)
    for _ in range(30):
        m, k = rng.integers(1, 41, size=2)
        a = np.where(rng.random((m, k)) < 0.25, 1 - rng.random((m, k)), 0).astype(np.float32)
        p = 1 << int(rng.integers(0, 6))
        r, c = np.nonzero(a)
        g1 = oracle.dense_to_gcoo(a, p)
        g2 = oracle.coo_to_gcoo(int(m), int(k), a[r, c], r.astype(np.int32), c.astype(np.int32), p)
        for f in FIELDS:
            assert np.array_equal(getattr(g1, f), getattr(g2, f))


def test_coo_validation(oracle):
    with pytest.raises(ValueError):  # duplicate
        oracle.coo_to_gcoo(2, 2, np.ones(2, np.float32), np.array([0, 0], np.int32), np.array([1, 1], np.int32), 2)
    with pytest.raises(ValueError):  # out of range
        oracle.coo_to_gcoo(2, 2, np.ones(1, np.float32), np.array([0], np.int32), np.array([5], np.int32), 2)


# --------------------------------------------- against the reference .so ---
def test_generators_vs_reference(oracle, reference):
    R, _ = reference
    for n, s, seed in [(1, 0.0, 1), (7, 0.5, 2), (64, 0.99, 3), (300, 0.9, 4), (129, 0.2, 5), (50, 1.0, 6)]:
        assert np.array_equal(oracle.uniform_sparse(n, s, seed), R.uniform_sparse(n, s, seed))
        assert oracle.derive_seed(seed, n, 0xB) == R.derive_seed(seed, n, 0xB)
    assert np.array_equal(oracle.uniform_sparse(40, 0.3, 9, np.float64), R.uniform_sparse(40, 0.3, 9, np.float64))


def test_construction_vs_reference(oracle, reference):
    R, _ = reference
    rng = np.random.default_rng(7)
    for _ in range(25):
        m, k = (int(x) for x in rng.integers(1, 120, size=2))
        a = np.where(rng.random((m, k)) < rng.random() * 0.5, 1 - rng.random((m, k)), 0).astype(np.float32)
        p = 1 << int(rng.integers(0, 8))
        gr, go = R.dense_to_gcoo(a, p), oracle.dense_to_gcoo(a, p)
        for f in FIELDS:
            assert np.array_equal(getattr(gr, f), getattr(go, f))
        r, c = np.nonzero(a)
        gc = R.coo_to_gcoo(m, k, a[r, c], r.astype(np.int32), c.astype(np.int32), p)
        for f in FIELDS:
            assert np.array_equal(getattr(gc, f), getattr(go, f))


def test_spdm_both_flavours_vs_reference(oracle, reference):
    R, RF = reference
    rng = np.random.default_rng(43)
    for _ in range(20):
        m, k, n = (int(x) for x in rng.integers(1, 200, size=3))
        p, b = 1 << int(rng.integers(0, 6)), 1 << int(rng.integers(0, 8))
        a = np.where(rng.random((m, k)) < rng.random() * 0.4, 1 - rng.random((m, k)), 0).astype(np.float32)
        bm = (1 - rng.random((k, n))).astype(np.float32)
        g = oracle.dense_to_gcoo(a, p)
        c_o, st_o = oracle.spdm(g, bm, b, fma=False)
        c_r, st_r = R.spdm(g, bm, b)
        assert np.array_equal(c_o, c_r) and st_o == st_r
        c_of, _ = oracle.spdm(g, bm, b, fma=True)
        c_rf, _ = RF.spdm(g, bm, b)
        assert np.array_equal(c_of, c_rf)
        # the reference's own gate against gemm_oracle (acceptance.cpp:90)
        ref = R.gemm_oracle(a, bm).astype(np.float64)
        assert np.max(np.abs(c_of - ref) / (np.abs(ref) + 1e-30)) <= 1e-5


def test_spdm_f64_vs_reference(oracle, reference):
    R, RF = reference
    rng = np.random.default_rng(5)
    a = np.where(rng.random((70, 50)) < 0.3, 1 - rng.random((70, 50)), 0)
    bm = 1 - rng.random((50, 33))
    g = oracle.dense_to_gcoo(a, 4)
    assert np.array_equal(oracle.spdm(g, bm, 16, fma=False)[0], R.spdm(g, bm, 16)[0])
    assert np.array_equal(oracle.spdm(g, bm, 16, fma=True)[0], RF.spdm(g, bm, 16)[0])


def test_powerlaw_generator_shape(oracle):
    v, r, c = oracle.powerlaw_coo(1024, 0.99, 1.0, 11)
    assert v.size == round(1024 * 1024 * 0.01)
    deg = np.bincount(r, minlength=1024)
    assert deg.max() > 20 * np.median(deg[deg > 0])  # skewed
    key = r.astype(np.int64) * 1024 + c
    assert np.all(np.diff(key) > 0)  # strictly row-major, no duplicates
    assert np.all((v > 0) & (v <= 1))


# ----------------------------------------------------------- traffic model --
def _traffic_golden():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "traffic.json")) as f:
        return json.load(f)


def test_traffic_restatement_matches_golden(oracle):
    """oracle.model_traffic (plain-Python restatement of traffic.cpp:43-197)
    against the reference's own counts on square_benchmark(512, 0.95)."""
    from oracle import model_traffic
    a = oracle.uniform_sparse(512, 0.95, 1)
    rows, cols = np.nonzero(a)
    gold = _traffic_golden()["n512_s0.95"]
    for kind in ("gcoo", "csr"):
        for mode in ("cold", "infinite_l2"):
            got = model_traffic(rows, cols, 512, 512, 512, 4, 64, mode == "infinite_l2", kind == "csr")
            assert got == gold[f"{kind}_{mode}"], (kind, mode)


def test_traffic_restatement_vs_reference_random(reference):
    """Ragged shapes, p and b extremes, empty groups: restatement == reference."""
    from oracle import model_traffic
    R, _ = reference
    rng = np.random.default_rng(17)
    for m, k, n, p, b, d in [(37, 29, 70, 4, 8, 0.2), (64, 64, 64, 1, 1, 0.1), (50, 80, 33, 8, 64, 0.3),
                             (9, 9, 1, 2, 2, 0.5), (100, 7, 129, 64, 4, 0.05), (5, 300, 31, 2, 128, 0.0)]:
        rows, cols = np.nonzero(rng.random((m, k)) < d)
        for inf in (False, True):
            for csr in (False, True):
                assert model_traffic(rows, cols, m, k, n, p, b, inf, csr) == \
                    R.model_traffic(rows, cols, m, k, n, p, b, inf, csr), (m, k, n, p, b, inf, csr)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_baseline_restatements_match_reference(oracle, reference, dtype):
    """The plain-C restatements of the reference's comparison kernels —
    spdm_csr (kernels.hpp:163-184), spdm_coo in any entry order with
    duplicates (:193-232), gemm_dense_blocked (:107-155) — equal the compiled
    reference bit for bit, as shipped (mul+add) and built -mfma, for several
    (p, b, workers) (the reference's result must not depend on them)."""
    R, RF = reference
    rng = np.random.default_rng(5 if dtype == np.float32 else 6)
    for trial in range(8):
        m, k, n = (int(x) for x in rng.integers(1, 120, size=3))
        a = np.where(rng.random((m, k)) < 0.15, 1.0 - rng.random((m, k)), 0.0).astype(dtype)
        b = (1.0 - rng.random((k, n))).astype(dtype)
        r, c = np.nonzero(a)
        v = a[r, c]
        rp = np.concatenate([[0], np.cumsum(np.count_nonzero(a, axis=1))]).astype(np.int64)
        perm = rng.permutation(r.size)
        dup = rng.integers(0, max(r.size, 1), size=min(4, r.size))
        rr, cc, vv = (np.concatenate([x[perm], x[dup]]) for x in (r, c, v))
        p, bw, w = 1 << int(rng.integers(0, 5)), 1 << int(rng.integers(0, 8)), int(rng.integers(0, 4))
        for fma, Rx in ((False, R), (True, RF)):
            assert np.array_equal(oracle.spdm_csr(m, v, c, rp, b, fma), Rx.spdm_csr(m, k, v, c, rp, b, p, bw, w))
            assert np.array_equal(oracle.spdm_coo(m, vv, rr, cc, b, fma), Rx.spdm_coo(m, k, vv, rr, cc, b, p, bw, w))
            assert np.array_equal(oracle.gemm_dense(a, b, fma), Rx.gemm_dense(a, b, p, bw, w))
