"""GPU parity of the reference's comparison kernels: the
B200 row-split CSR SpDM, the ungrouped-COO ablation and the dense GEMM, each
against the oracle's restatement of the reference (pinned to the compiled
reference in tests/test_oracle.py) — bit-exact in both numeric flavours."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_dense(rng, m, k, density, dtype=np.float32):
    return np.where(rng.random((m, k)) < density, 1.0 - rng.random((m, k)), 0.0).astype(dtype)


def csr_of(a):
    r, c = np.nonzero(a)
    rp = np.concatenate([[0], np.cumsum(np.count_nonzero(a, axis=1))]).astype(np.int64)
    return a[r, c], r.astype(np.int32), c.astype(np.int32), rp


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_csr_coo_dense_random_shapes_bit_exact(gcoo, cuda, oracle, dtype):
    rng = np.random.default_rng(100 if dtype == np.float32 else 101)
    for m, k, n, d in [(1, 1, 1, 1.0), (37, 29, 70, 0.2), (300, 200, 132, 0.02), (513, 129, 67, 0.3),
                       (64, 700, 256, 0.01), (100, 100, 5, 0.0), (1025, 333, 130, 0.05)]:
        a = rand_dense(rng, m, k, d, dtype)
        b = rand_dense(rng, k, n, 1.0, dtype)
        v, r, c, rp = csr_of(a)
        assert np.array_equal(gcoo.spdm_csr(m, k, v, c, rp, b), oracle.spdm_csr(m, v, c, rp, b, True)), (m, k, n)
        assert np.array_equal(gcoo.spdm_coo(m, k, v, r, c, b), oracle.spdm_coo(m, v, r, c, b, True)), (m, k, n)
        assert np.array_equal(gcoo.gemm_dense_blocked(a, b), oracle.gemm_dense(a, b, True)), (m, k, n)


def test_unsorted_csr_and_shuffled_duplicated_coo(gcoo, cuda, oracle):
    """The reference accepts any column order inside a CSR row and any COO
    entry order with duplicates; C follows that order (not column order)."""
    rng = np.random.default_rng(7)
    m, k, n = 700, 900, 260
    a = rand_dense(rng, m, k, 0.03)
    b = rand_dense(rng, k, n, 1.0)
    v, r, c, rp = csr_of(a)
    # shuffle columns inside every row
    v2, c2 = v.copy(), c.copy()
    for i in range(m):
        sl = slice(rp[i], rp[i + 1])
        p = rng.permutation(rp[i + 1] - rp[i])
        v2[sl], c2[sl] = v[sl][p], c[sl][p]
    assert np.array_equal(gcoo.spdm_csr(m, k, v2, c2, rp, b), oracle.spdm_csr(m, v2, c2, rp, b, True))
    perm = rng.permutation(r.size)
    dup = rng.integers(0, r.size, size=500)
    rr, cc, vv = (np.concatenate([x[perm], x[dup]]) for x in (r, c, v))
    assert np.array_equal(gcoo.spdm_coo(m, k, vv, rr, cc, b), oracle.spdm_coo(m, vv, rr, cc, b, True))


def test_device_variants_flavours_and_strided_shards(gcoo, cuda, oracle):
    import torch
    rng = np.random.default_rng(8)
    m, k, n = 900, 1100, 390
    a = rand_dense(rng, m, k, 0.02)
    b = rand_dense(rng, k, n, 1.0)
    v, r, c, rp = csr_of(a)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    dB = T(b)
    for flavor, fma in ((gcoo.FLAVOR_FMA, True), (gcoo.FLAVOR_MUL_ADD, False)):
        for j0, j1 in ((0, n), (3, 200), (128, 390)):  # unaligned and aligned column shards
            want_csr = oracle.spdm_csr(m, v, c, rp, np.ascontiguousarray(b[:, j0:j1]), fma)
            ct = torch.empty((m, n), device="cuda")
            gcoo.spdm_csr_dev(m, k, T(v), T(c), T(rp), dB[:, j0:j1], ct[:, j0:j1], flavor=flavor)
            torch.cuda.synchronize()
            assert np.array_equal(ct[:, j0:j1].cpu().numpy(), want_csr), (flavor, j0, j1)
            gcoo.spdm_coo_dev(m, k, T(v), T(r), T(c), dB[:, j0:j1], ct[:, j0:j1], flavor=flavor)
            torch.cuda.synchronize()
            assert np.array_equal(ct[:, j0:j1].cpu().numpy(), want_csr), (flavor, j0, j1)
        cd = torch.empty((m, n), device="cuda")
        gcoo.gemm_dense_dev(T(a), dB, cd, flavor=flavor)
        torch.cuda.synchronize()
        assert np.array_equal(cd.cpu().numpy(), oracle.gemm_dense(a, b, fma))


def test_baselines_reject_out_of_range(gcoo, cuda):
    b = np.ones((3, 4), np.float32)
    with pytest.raises(ValueError):
        gcoo.spdm_csr(2, 3, np.ones(2, np.float32), np.array([0, 7]), np.array([0, 1, 2]), b)
    with pytest.raises(ValueError):
        gcoo.spdm_csr(2, 3, np.ones(2, np.float32), np.array([0, 1]), np.array([0, 3, 2]), b)
    with pytest.raises(ValueError):
        gcoo.spdm_coo(2, 3, np.ones(2, np.float32), np.array([0, 2]), np.array([0, 1]), b)
    with pytest.raises(ValueError):
        gcoo.spdm_coo(2, 3, np.ones(1, np.float32), np.array([0]), np.array([0]), np.ones((4, 4), np.float32))


@pytest.mark.slow
def test_full_size_csr_equals_gcoo_n8000(gcoo, cuda, oracle):
    """configs[1] inputs: the row-split CSR kernel (sorted columns) and the
    GCOO path compute the same chain, so C is bitwise equal; sampled rows of
    the COO ablation too, and all against the oracle on sampled rows."""
    import torch
    n = 8000
    a = gcoo.generate_uniform_sparse(n, 0.99, 1)
    bm = gcoo.generate_uniform_sparse(n, 0.0, gcoo.derive_seed(1, n, 0xB))
    v, r, c, rp = csr_of(a)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    dB = T(bm)
    c1 = torch.empty((n, n), device="cuda")
    c2 = torch.empty_like(c1)
    c3 = torch.empty_like(c1)
    gcoo.spdm_csr_dev(n, n, T(v), T(c), T(rp), dB, c1)
    gcoo.spdm_coo_dev(n, n, T(v), T(r), T(c), dB, c2)
    gcoo.spdm_gcoo_dev(gcoo.dense_to_gcoo_dev(T(a), 4), dB, c3)
    torch.cuda.synchronize()
    assert torch.equal(c1, c3) and torch.equal(c2, c3)
    g = oracle.dense_to_gcoo(a, 4)
    for r0 in (0, 3992, 7992):
        want = oracle.spdm_rows(g, bm, r0, r0 + 8, fma=True)[r0:r0 + 8]
        assert c1[r0:r0 + 8].cpu().numpy().tobytes() == want.tobytes()
