"""GPU parity: the CUDA product, called through the C ABI, against the oracle.

Bars (BASELINE.json north star): GCOO arrays bit-exact; C bit-exact against
the reference's accumulation order with FMA contraction (the oracle's fma
flavour == reference built -mfma), and bit-exact against the as-shipped
mul+add reference through the MUL_ADD flavour; max relative error <= 1e-5
(fp32) / 1e-12 (fp64) against gemm_oracle-style double accumulation
(acceptance.cpp:90).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
FIELDS = ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group")


def rand_dense(rng, m, k, density, dtype=np.float32):
    return np.where(rng.random((m, k)) < density, 1.0 - rng.random((m, k)), 0.0).astype(dtype)


def to_prod(G, g):
    return G.GcooMatrix(g.rows_dim, g.cols_dim, g.p, g.values, g.row_idx, g.col_idx, g.g_idxes, g.nnz_per_group)


def max_rel(x, ref):
    ref = ref.astype(np.float64)
    return float(np.max(np.abs(x.astype(np.float64) - ref) / (np.abs(ref) + 1e-30))) if ref.size else 0.0


# ------------------------------------------------------------ multiply -----
def test_example_identity_and_flops(gcoo, cuda, oracle):
    # test_kernels.cpp:91-101
    a = np.zeros((4, 4), np.float32)
    a[0, 0], a[0, 3], a[1, 1], a[2, 0], a[3, 2], a[3, 3] = 7, 8, 10, 9, 6, 3
    g = gcoo.dense_to_gcoo(a, 2)
    st = gcoo.KernelStats()
    c = gcoo.spdm_gcoo(g, np.eye(4, dtype=np.float32), gcoo.ExecConfig(p=2, b=4), stats=st)
    assert np.array_equal(c, a)
    assert st.flops == 48


def test_reuse_accounting_hand_traced(gcoo, cuda):
    # test_kernels.cpp:103-123
    a = np.zeros((4, 4), np.float32)
    a[0, 1], a[1, 1] = 2, 5
    st = gcoo.KernelStats()
    c = gcoo.spdm_gcoo(gcoo.dense_to_gcoo(a, 2), np.eye(4, dtype=np.float32), gcoo.ExecConfig(p=2, b=4), stats=st)
    assert (st.b_loads_total, st.b_loads_reused, st.staging_fills, st.flops) == (4, 4, 2, 16)
    assert c[0, 1] == 2 and c[1, 1] == 5 and np.count_nonzero(c) == 2


def test_golden_small_cases(gcoo, cuda, golden_small):
    names = sorted({k.split(".")[0] for k in golden_small})
    for name in names:
        a, b = golden_small[f"{name}.A"], golden_small[f"{name}.B"]
        for p in (1, 2, 4, 8, 64):
            g = gcoo.dense_to_gcoo(a, p)
            for f in FIELDS:
                assert np.array_equal(getattr(g, f), golden_small[f"{name}.p{p}.{f}"]), (name, p, f)
        g = gcoo.dense_to_gcoo(a, 4)
        for bb in (1, 4, 64, 256):
            st = gcoo.KernelStats()
            c = gcoo.spdm_gcoo(g, b, gcoo.ExecConfig(p=4, b=bb), stats=st)
            assert np.array_equal(c, golden_small[f"{name}.C_fma"]), name
            assert (st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills) == tuple(
                int(x) for x in golden_small[f"{name}.stats_b{bb}"]), (name, bb)


def test_mul_add_flavour_bit_exact_vs_shipped_reference(gcoo, cuda, golden_small):
    import torch
    for name in sorted({k.split(".")[0] for k in golden_small}):
        a, b = golden_small[f"{name}.A"], golden_small[f"{name}.B"]
        d = gcoo.DeviceGcoo.from_host(gcoo.dense_to_gcoo(a, 4))
        bt = torch.from_numpy(b).cuda()
        ct = torch.empty((a.shape[0], b.shape[1]), dtype=torch.float32, device="cuda")
        gcoo.spdm_gcoo_dev(d, bt, ct, gcoo.ExecConfig(p=4), flavor=gcoo.FLAVOR_MUL_ADD)
        torch.cuda.synchronize()
        assert np.array_equal(ct.cpu().numpy(), golden_small[f"{name}.C_mad"]), name


@pytest.mark.parametrize("seed", range(6))
def test_random_shapes_bit_exact(gcoo, cuda, oracle, seed):
    # test_kernels.cpp:157-183 distributions, plus wider p and odd n
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        m, k, n = (int(x) for x in rng.integers(1, 260, size=3))
        p = 1 << int(rng.integers(0, 7))
        b = 1 << int(rng.integers(0, 8))
        a = rand_dense(rng, m, k, float(rng.random() * 0.4))
        bm = rand_dense(rng, k, n, 0.95)
        go = oracle.dense_to_gcoo(a, p)
        c_ref, st_ref = oracle.spdm(go, bm, b, fma=True)
        st = gcoo.KernelStats()
        c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p, b=b), stats=st)
        assert np.array_equal(c, c_ref), (m, k, n, p, b)
        assert (st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills) == st_ref
        c_mad, _ = oracle.spdm(go, bm, b, fma=False)
        assert max_rel(c, c_mad) <= 1e-5


_TACC_FP32 = ["tacc28_k192", "tacc28_k160", "tacc28_k128", "tacc28_k96", "tacc28_k64", "tacc28_k200",
              "tacc_v4_k216", "tacc28_k176", "auto"]


@pytest.mark.parametrize("kernel,planner", [("rowtile", "none")] +
                         [(k, pl) for pl in ("segment", "general", "persistent") for k in _TACC_FP32])
def test_each_fp32_kernel_bit_exact(gcoo, cuda, oracle, kernel, planner):
    """Every fp32 kernel variant, on shapes that hit its edges (m not a multiple
    of the row block, k not a multiple of the chunk, n not a multiple of the
    strip, empty rows/tiles, every p the variant supports), with its record
    stream built by the segment planner (even A, the default) and by the
    general count / header / fill chain."""
    rng = np.random.default_rng(sorted(gcoo.KERNELS).index(kernel))
    gcoo.force_kernel(kernel)
    gcoo.seg_planner(planner != "general")  # the row-tile kernel has no planner
    gcoo.persistent(planner == "persistent")  # one persistent CTA per SM walking the tiles (default) or one per tile
    try:
        for m, k, n, p, dens in [(1, 1, 4, 1, 1.0), (300, 200, 132, 4, 0.02), (777, 1000, 256, 1, 0.01),
                                 (513, 129, 68, 16, 0.2), (1030, 333, 200, 8, 0.05), (64, 4000, 512, 2, 0.003),
                                 (2000, 700, 196, 32, 0.01), (100, 100, 1024, 4, 0.0)]:
            a = rand_dense(rng, m, k, dens)
            bm = rand_dense(rng, k, n, 1.0)
            go = oracle.dense_to_gcoo(a, p)
            c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
            c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p))
            assert np.array_equal(c, c_ref), (kernel, m, k, n, p)
    finally:
        gcoo.force_kernel("auto")
        gcoo.seg_planner(True)
        gcoo.persistent(True)


def test_segment_planner_group_sizes_and_row_spread(gcoo, cuda, oracle):
    """The segment planner across group sizes p = 1 .. 4096 (groups spanning
    several row blocks when p > RB), three-entry and fp64 records, and the
    narrow-strip row spreading (rows per block < RB): bit-exact against the
    oracle and equal to the general planner's C."""
    import torch
    rng = np.random.default_rng(91)
    cases = [("tacc28_k200", np.float32, 0.01), ("tacc28_k128", np.float32, 0.08), ("tacc_v4_k216", np.float32, 0.002),
             ("tacc28_f64_k160", np.float64, 0.01)]
    try:
        for kernel, dt, dens in cases:
            gcoo.force_kernel(kernel)
            m, k, n = 2100, 1700, 260 if dt == np.float32 else 130
            a = rand_dense(rng, m, k, dens, dt)
            bm = rand_dense(rng, k, n, 1.0, dt)
            for p in (1, 2, 8, 64, 512, 4096):
                go = oracle.dense_to_gcoo(a, p)
                c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
                for seg in (True, False):
                    gcoo.seg_planner(seg)
                    c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p))
                    assert np.array_equal(c, c_ref), (kernel, p, seg)
            # device path on a narrow strip: one column tile, rows spread over more row blocks
            go = oracle.dense_to_gcoo(a, 4)
            d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
            bn = bm[:, :64].copy()
            c_ref, _ = oracle.spdm(go, bn, 64, fma=True)
            cd = torch.empty((m, 64), dtype=torch.from_numpy(bn).dtype, device="cuda")
            gcoo.spdm_gcoo_dev(d, torch.from_numpy(bn).cuda(), cd)
            assert np.array_equal(cd.cpu().numpy(), c_ref), kernel
    finally:
        gcoo.force_kernel("auto")
        gcoo.seg_planner(True)


def test_f64(gcoo, cuda, oracle):
    rng = np.random.default_rng(77)
    for _ in range(6):
        m, k, n = (int(x) for x in rng.integers(1, 150, size=3))
        p = 1 << int(rng.integers(0, 6))
        a = rand_dense(rng, m, k, 0.2, np.float64)
        bm = rand_dense(rng, k, n, 1.0, np.float64)
        g = gcoo.dense_to_gcoo(a, p)
        go = oracle.dense_to_gcoo(a, p)
        for f in FIELDS:
            assert np.array_equal(getattr(g, f), getattr(go, f))
        c = gcoo.spdm_gcoo(g, bm, gcoo.ExecConfig(p=p))
        c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
        assert np.array_equal(c, c_ref)
        exact = a.astype(np.longdouble) @ bm.astype(np.longdouble)
        assert max_rel(c, exact) <= 1e-12


@pytest.mark.parametrize("kernel", ["tacc28_f64_k160", "tacc28_f64_k96", "tacc28_f64_k64", "auto"])
def test_f64_tmem_kernels_bit_exact(gcoo, cuda, oracle, kernel):
    """fp64 through the TMEM kernels (two 32-bit cells per double, one entry
    per record): edge shapes and p values, bit-exact against the oracle's
    double FMA chain; "auto" on a product large enough to take them."""
    rng = np.random.default_rng(53)
    gcoo.force_kernel(kernel)
    try:
        shapes = [(1, 1, 2, 1, 1.0), (300, 200, 132, 4, 0.02), (777, 1000, 256, 1, 0.01), (513, 129, 68, 16, 0.2),
                  (64, 4000, 512, 2, 0.003), (100, 100, 1024, 4, 0.0)]
        if kernel == "auto":
            shapes = [(3000, 2000, 512, 4, 0.05), (2000, 3000, 640, 8, 0.005)]
        for m, k, n, p, dens in shapes:
            a = rand_dense(rng, m, k, dens, np.float64)
            bm = rand_dense(rng, k, n, 1.0, np.float64)
            go = oracle.dense_to_gcoo(a, p)
            c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
            c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p))
            assert np.array_equal(c, c_ref), (kernel, m, k, n, p)
    finally:
        gcoo.force_kernel("auto")


def test_empty_and_full_operands(gcoo, cuda, oracle):
    # test_kernels.cpp:254-264
    ones = np.ones((16, 16), np.float32)
    c = gcoo.spdm_gcoo(gcoo.dense_to_gcoo(np.zeros((16, 16), np.float32), 4), ones)
    assert np.array_equal(c, np.zeros((16, 16), np.float32))
    full = rand_dense(np.random.default_rng(61), 16, 16, 1.0)
    c = gcoo.spdm_gcoo(gcoo.dense_to_gcoo(full, 4), ones)
    assert np.array_equal(c, oracle.spdm(oracle.dense_to_gcoo(full, 4), ones, 64, True)[0])
    # 1x1 and single-row / single-column shapes
    for m, k, n in [(1, 1, 1), (1, 7, 1), (9, 1, 5), (1, 300, 3)]:
        a = rand_dense(np.random.default_rng(m * 100 + n), m, k, 0.7)
        bm = rand_dense(np.random.default_rng(k), k, n, 1.0)
        go = oracle.dense_to_gcoo(a, 4)
        assert np.array_equal(gcoo.spdm_gcoo(to_prod(gcoo, go), bm), oracle.spdm(go, bm, 64, True)[0])


def test_tile_order_permutation_and_list(gcoo, cuda, oracle, reference):
    # test_kernels.cpp:200-234 (shuffled tile list gives identical bits)
    R, RF = reference
    rng = np.random.default_rng(53)
    a = rand_dense(rng, 257, 129, 0.1)
    bm = rand_dense(rng, 129, 193, 1.0)
    g = gcoo.dense_to_gcoo(a, 4)
    cfg = gcoo.ExecConfig()
    tiles = g.groups() * -(-193 // cfg.b)
    c1 = gcoo.spdm_gcoo(g, bm, cfg)
    order = rng.permutation(tiles)
    assert np.array_equal(c1, gcoo.spdm_gcoo(g, bm, cfg, tile_order=order))
    # a non-permutation list: the reference leaves unlisted tiles at 0 and
    # counts duplicates twice — reproduce that exactly
    lst = rng.integers(0, tiles, size=tiles)
    st = gcoo.KernelStats()
    c2 = gcoo.spdm_gcoo(g, bm, cfg, tile_order=lst, stats=st)
    cr, st_r = RF.spdm(g, bm, cfg.b, tile_order=lst)
    assert np.array_equal(c2, cr)
    assert (st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills) == st_r


def test_determinism(gcoo, cuda):
    rng = np.random.default_rng(9)
    a = rand_dense(rng, 300, 400, 0.05)
    bm = rand_dense(rng, 400, 260, 1.0)
    g = gcoo.dense_to_gcoo(a, 4)
    c0 = gcoo.spdm_gcoo(g, bm)
    for _ in range(3):
        assert np.array_equal(c0, gcoo.spdm_gcoo(g, bm))


def test_concurrent_host_calls_are_independent(gcoo, cuda, oracle):
    """The C ABI is re-entrant (per-thread stream, thread-local error string):
    host threads calling spdm_gcoo / coo_to_gcoo at once (ctypes drops the GIL)
    each get their own bit-exact result, including the pipelined size and an
    error raised on one thread while the others compute."""
    import threading
    rng = np.random.default_rng(41)
    cases = []
    for i, (m, k, n, d) in enumerate([(700, 900, 320, 0.01), (2048, 2048, 2048, 0.004), (513, 129, 68, 0.2),
                                      (1000, 3000, 512, 0.002), (4096, 4096, 2304, 0.002), (64, 64, 64, 0.5)]):
        a = rand_dense(rng, m, k, d)
        bm = rand_dense(rng, k, n, 1.0)
        go = oracle.dense_to_gcoo(a, 4)
        cases.append((a, bm, go, oracle.spdm(go, bm, 64, fma=True)[0]))
    out, errs = [None] * len(cases), []

    def work(i):
        try:
            a, bm, go, _ = cases[i]
            for _ in range(3):
                g = gcoo.dense_to_gcoo(a, 4)
                out[i] = gcoo.spdm_gcoo(g, bm)
            if i == 0:
                with pytest.raises(ValueError):
                    gcoo.spdm_gcoo(g, bm[:-1].copy())  # inner-dimension mismatch on this thread only
        except Exception as e:  # noqa: BLE001
            errs.append((i, repr(e)))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(cases))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for (a, bm, go, c_ref), c in zip(cases, out):
        assert np.array_equal(c, c_ref)


@pytest.mark.parametrize("p", [128, 1024])
def test_large_group_size_bit_exact(gcoo, cuda, oracle, p):
    """Large p: a group spans several row blocks and a chunk's range inside a
    group slice holds hundreds of entries (the planner ranks them one warp per
    range); C bit-exact against the oracle, the multiply on a TMEM kernel."""
    rng = np.random.default_rng(p)
    m, k, n = 2600, 3000, 4096  # above the small-product gate: the TMEM kernel runs
    a = rand_dense(rng, m, k, 0.01)
    bm = rand_dense(rng, k, n, 1.0)
    go = oracle.dense_to_gcoo(a, p)
    c_ref, st_ref = oracle.spdm(go, bm, 64, fma=True)
    st = gcoo.KernelStats()
    c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p), stats=st)
    assert np.array_equal(c, c_ref)
    assert (st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills) == st_ref
    assert gcoo.last_kernel().startswith("tacc")

@pytest.mark.parametrize("n,s", [(2000, 0.8), (2000, 0.999), (4000, 0.95), (14000, 0.99), (14000, 0.9)])
def test_configs2_sweep_points_vs_oracle(gcoo, cuda, oracle, n, s):
    """BASELINE configs[2] (the sparsity sweep at n = 2000..14000, inputs from
    the reference's sweep seeds as tools/sweep_crossover.py makes them): the
    GPU's dense -> GCOO (K3) and multiply on device tensors, against the
    oracle — GCOO arrays bit-exact, C bit-exact on sampled row blocks (the
    oracle's row-range multiply keeps each row's chain)."""
    import torch
    dens = round(n * n * (1.0 - s)) / (n * n)  # the reference's realised sparsity (bench.cpp:67-74)
    a_seed = gcoo.derive_seed(1, n, int(round(dens * n * n)))
    a = gcoo.generate_uniform_sparse(n, s, a_seed)
    b = gcoo.generate_uniform_sparse(n, 0.0, gcoo.derive_seed(a_seed, n, 0xB))
    d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
    c = torch.empty((n, n), dtype=torch.float32, device="cuda")
    gcoo.spdm_gcoo_dev(d, torch.from_numpy(b).cuda(), c)
    torch.cuda.synchronize()
    go = oracle.dense_to_gcoo(a, 4)
    g = d.to_host()
    for f in ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group"):
        assert np.array_equal(getattr(g, f), getattr(go, f)), f
    rows = 16 if n > 4000 else 64
    for r0 in (0, n // 2 - rows // 2, n - rows):
        c_ref = oracle.spdm_rows(go, b, r0, r0 + rows)
        assert np.array_equal(c[r0:r0 + rows].cpu().numpy(), c_ref[r0:r0 + rows]), (n, s, r0)

def test_plan_execute_split_bit_exact(gcoo, cuda, oracle):
    """gcoo_plan_*: one plan, many multiplies (different B widths, a strided
    column shard, an unaligned shard that needs another kernel class) — every
    result equals the one-shot device call bit for bit."""
    import torch
    rng = np.random.default_rng(43)
    for m, k, d in [(3000, 2500, 0.01), (777, 1000, 0.05), (5000, 5000, 0.002)]:
        a = rand_dense(rng, m, k, d)
        dg = gcoo.DeviceGcoo.from_host(gcoo.dense_to_gcoo(a, 4))
        plan = gcoo.SpdmPlan(dg)
        bfull = torch.from_numpy(rand_dense(rng, k, 1030, 1.0)).cuda()
        for n0, n1 in [(0, 512), (0, 1030), (128, 640), (3, 515)]:
            b = bfull[:, n0:n1]
            c1 = torch.empty((m, n1 - n0), device="cuda")
            c2 = torch.empty_like(c1)
            plan.run(b, c1)
            gcoo.spdm_gcoo_dev(dg, b, c2)
            torch.cuda.synchronize()
            assert torch.equal(c1, c2), (m, k, n0, n1)
        plan.close()
    with pytest.raises(ValueError):
        plan.run(bfull, torch.empty((5000, 1030), device="cuda"))
    # fp64 plans
    a = rand_dense(rng, 2000, 1500, 0.02, np.float64)
    dg = gcoo.DeviceGcoo.from_host(gcoo.dense_to_gcoo(a, 4))
    plan = gcoo.SpdmPlan(dg)
    b = torch.from_numpy(rand_dense(rng, 1500, 640, 1.0, np.float64)).cuda()
    c1 = torch.empty((2000, 640), device="cuda", dtype=torch.float64)
    c2 = torch.empty_like(c1)
    plan.run(b, c1)
    gcoo.spdm_gcoo_dev(dg, b, c2)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    with pytest.raises(ValueError):
        plan.run(b.float(), c1.float())
    plan.close()


def test_plan_run_is_one_launch(gcoo, cuda):
    """A reused plan issues exactly one multiply kernel per run, at every size
    class (the plan is chosen without the per-call small-product gate), and
    the planner runs once at create time."""
    import torch
    rng = np.random.default_rng(44)
    for m, k, n, d in [(8000, 8000, 512, 0.01), (600, 500, 64, 0.05), (3000, 3000, 8, 0.002)]:
        a = rand_dense(rng, m, k, d)
        dg = gcoo.DeviceGcoo.from_host(gcoo.dense_to_gcoo(a, 4))
        plan = gcoo.SpdmPlan(dg)
        b = torch.from_numpy(rand_dense(rng, k, n, 1.0)).cuda()
        c1 = torch.empty((m, n), device="cuda")
        c2 = torch.empty_like(c1)
        plan.run(b, c1)
        l0 = gcoo.launch_count()
        plan.run(b, c1)
        assert gcoo.launch_count() - l0 == 1, (m, k, n)
        gcoo.spdm_gcoo_dev(dg, b, c2)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2)
        plan.close()


def test_hypersparse_routes_and_empty_chunks(gcoo, cuda, oracle):
    """Hypersparse A (a few entries per row block and chunk): auto takes the
    row-tile kernel; a forced TMEM kernel skips the B tiles of empty chunks —
    both bit-exact, including entirely empty row blocks."""
    rng = np.random.default_rng(45)
    for m, k, n, nnz in [(6000, 7000, 256, 300), (3000, 9000, 132, 40), (1100, 20000, 512, 2000)]:
        flat = np.sort(rng.choice(m * k, nnz, replace=False))
        a = np.zeros((m, k), np.float32)
        a.flat[flat] = (1.0 - rng.random(nnz)).astype(np.float32)
        bm = rand_dense(rng, k, n, 1.0)
        go = oracle.dense_to_gcoo(a, 4)
        c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
        for kern in ("auto", "tacc28_k200", "tacc_v4_k216", "tacc28_k64"):
            gcoo.force_kernel(kern)
            try:
                c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=4))
            finally:
                gcoo.force_kernel("auto")
            assert np.array_equal(c, c_ref), (m, k, n, nnz, kern)


def test_device_api_rejects_mismatched_operands(gcoo, cuda):
    """The Python device API checks dtypes, devices and layouts before the C
    ABI reads the pointers (an fp64 B with an fp32 A must not be multiplied)."""
    import torch
    rng = np.random.default_rng(46)
    a = rand_dense(rng, 64, 48, 0.2)
    dg = gcoo.DeviceGcoo.from_host(gcoo.dense_to_gcoo(a, 4))
    b32 = torch.ones((48, 16), device="cuda")
    c32 = torch.empty((64, 16), device="cuda")
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo_dev(dg, b32.double(), c32)
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo_dev(dg, b32, c32.double())
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo_dev(dg, b32.t().contiguous().t(), c32)
    with pytest.raises(ValueError):
        gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda().half(), 4)
    r, c = np.nonzero(a)
    with pytest.raises(ValueError):  # int64 coordinates
        gcoo.coo_to_gcoo_dev(64, 48, torch.from_numpy(a[r, c]).cuda(), torch.from_numpy(r).cuda(),
                             torch.from_numpy(c).cuda(), 4)
    bad = gcoo.DeviceGcoo(dg.rows_dim, dg.cols_dim, dg.p, dg.values, dg.row_idx.long(), dg.col_idx, dg.g_idxes,
                          dg.nnz_per_group)
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo_dev(bad, b32, c32)


def test_strided_column_shards_bitwise_equal(gcoo, cuda, oracle):
    """Column sharding (the multi-GPU decomposition) is bitwise invisible."""
    import torch
    rng = np.random.default_rng(3)
    a = rand_dense(rng, 500, 300, 0.03)
    bm = rand_dense(rng, 300, 640, 1.0)
    go = oracle.dense_to_gcoo(a, 4)
    ref, _ = oracle.spdm(go, bm, 64, True)
    d = gcoo.DeviceGcoo.from_host(to_prod(gcoo, go))
    bt = torch.from_numpy(bm).cuda()
    for shards in (1, 2, 4, 5, 8):
        ct = torch.zeros((500, 640), dtype=torch.float32, device="cuda")
        bounds = np.linspace(0, 640, shards + 1).astype(int)
        for j0, j1 in zip(bounds[:-1], bounds[1:]):
            gcoo.spdm_gcoo_dev(d, bt[:, j0:j1], ct[:, j0:j1])
        torch.cuda.synchronize()
        assert np.array_equal(ct.cpu().numpy(), ref), shards


# -------------------------------------------------------- construction -----
@pytest.mark.parametrize("seed", range(4))
def test_construction_bit_exact(gcoo, cuda, oracle, seed):
    rng = np.random.default_rng(seed)
    for _ in range(8):
        m, k = (int(x) for x in rng.integers(1, 300, size=2))
        p = 1 << int(rng.integers(0, 9))
        a = rand_dense(rng, m, k, float(rng.random() * 0.5))
        go = oracle.dense_to_gcoo(a, p)
        g1 = gcoo.dense_to_gcoo(a, p)
        r, c = np.nonzero(a)
        g2 = gcoo.coo_to_gcoo(m, k, a[r, c], r.astype(np.int32), c.astype(np.int32), p)
        rp = np.concatenate([[0], np.cumsum(np.count_nonzero(a, axis=1))]).astype(np.int64)
        g3 = gcoo.csr_to_gcoo(m, k, a[r, c], c.astype(np.int32), rp, p)
        for g in (g1, g2, g3):
            for f in FIELDS:
                assert np.array_equal(getattr(g, f), getattr(go, f)), (m, k, p, f)
            g.validate()


def test_coo_validation_errors(gcoo, cuda):
    # test_matrix.cpp:78-87
    with pytest.raises(ValueError):
        gcoo.coo_to_gcoo(2, 2, np.ones(2, np.float32), np.array([0, 0]), np.array([1, 1]), 2)
    with pytest.raises(ValueError):
        gcoo.coo_to_gcoo(2, 2, np.ones(1, np.float32), np.array([0]), np.array([5]), 2)
    with pytest.raises(ValueError):
        gcoo.coo_to_gcoo(2, 2, np.ones(2, np.float32), np.array([1, 0]), np.array([0, 0]), 2)
    with pytest.raises(ValueError):
        gcoo.coo_to_gcoo(2, 2, np.ones(1, np.float32), np.array([0]), np.array([0]), 3)
    with pytest.raises(ValueError, match="not monotone"):  # CSR non-monotone row_ptr (test_matrix.cpp:99-101)
        gcoo.csr_to_gcoo(2, 2, np.ones(1, np.float32), np.array([0]), np.array([0, 2, 1]), 2)
    # the reference's CsrMatrix::validate messages and order (matrix.hpp:154-162)
    with pytest.raises(ValueError, match="column out of range"):
        gcoo.csr_to_gcoo(2, 3, np.ones(3, np.float32), np.array([0, 2, 7]), np.array([0, 1, 3]), 2)
    with pytest.raises(ValueError, match="not strictly increasing in row 1"):
        gcoo.csr_to_gcoo(3, 3, np.ones(4, np.float32), np.array([0, 2, 2, 1]), np.array([0, 1, 3, 4]), 2)
    with pytest.raises(ValueError, match="not strictly increasing in row 0"):  # first bad element wins
        gcoo.csr_to_gcoo(1, 3, np.ones(3, np.float32), np.array([2, 1, 9]), np.array([0, 3]), 2)


def test_powerlaw_construction_and_multiply(gcoo, cuda, oracle):
    v, r, c = gcoo.generate_powerlaw_coo(2048, 0.99, 1.0, 5)
    go = oracle.coo_to_gcoo(2048, 2048, v, r, c, 4)
    g = gcoo.coo_to_gcoo(2048, 2048, v, r, c, 4)
    for f in FIELDS:
        assert np.array_equal(getattr(g, f), getattr(go, f))
    bm = oracle.uniform_sparse(2048, 0.0, 12)[:, :320].copy()
    assert np.array_equal(gcoo.spdm_gcoo(g, bm), oracle.spdm(go, bm, 64, True)[0])


def test_powerlaw_host_pipeline_bit_exact(gcoo, cuda, oracle):
    """Skewed rows through the pipelined host path: the plan spreads the
    heaviest-first placement over extra, partly filled row blocks (narrow
    strips still fill the GPU); C equals the oracle's FMA chain bit for bit."""
    n = 4096
    v, r, c = gcoo.generate_powerlaw_coo(n, 0.99, 1.0, 7)
    g = gcoo.coo_to_gcoo(n, n, v, r, c, 4)
    go = oracle.coo_to_gcoo(n, n, v, r, c, 4)
    bm = oracle.uniform_sparse(n, 0.0, 13)[:, :2304].copy()
    assert np.array_equal(gcoo.spdm_gcoo(g, bm), oracle.spdm(go, bm, 64, True)[0])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_device_construction_paths(gcoo, cuda, oracle, dtype):
    """dense / COO / CSR -> GCOO on device arrays, fp32 and fp64: bit-exact
    against the oracle; the CSR device path keeps the reference's errors."""
    import torch
    rng = np.random.default_rng(21)
    a = rand_dense(rng, 333, 517, 0.04, dtype)
    go = oracle.dense_to_gcoo(a, 8)
    d1 = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 8)
    r, c = np.nonzero(a)
    d2 = gcoo.coo_to_gcoo_dev(333, 517, torch.from_numpy(a[r, c]).cuda(),
                              torch.from_numpy(r.astype(np.int32)).cuda(),
                              torch.from_numpy(c.astype(np.int32)).cuda(), 8)
    rp = np.concatenate([[0], np.cumsum(np.count_nonzero(a, axis=1))]).astype(np.int64)
    d3 = gcoo.csr_to_gcoo_dev(333, 517, torch.from_numpy(a[r, c]).cuda(), torch.from_numpy(c.astype(np.int32)).cuda(),
                              torch.from_numpy(rp).cuda(), 8)
    for d in (d1, d2, d3):
        assert d.values.dtype == (torch.float64 if dtype == np.float64 else torch.float32)
        g = d.to_host()
        for f in FIELDS:
            assert np.array_equal(getattr(g, f), getattr(go, f)), f
    # and they multiply: the device GCOO of either precision through the TMEM path
    bm = rand_dense(rng, 517, 260, 1.0, dtype)
    ct = torch.empty((333, 260), dtype=d3.values.dtype, device="cuda")
    gcoo.spdm_gcoo_dev(d3, torch.from_numpy(bm).cuda(), ct)
    torch.cuda.synchronize()
    assert np.array_equal(ct.cpu().numpy(), oracle.spdm(go, bm, 64, fma=True)[0])
    with pytest.raises(ValueError, match="not strictly increasing in row 1"):
        gcoo.csr_to_gcoo_dev(3, 3, torch.ones(4, dtype=torch.float32, device="cuda"),
                             torch.tensor([0, 2, 2, 1], dtype=torch.int32, device="cuda"),
                             torch.tensor([0, 1, 3, 4], dtype=torch.int64, device="cuda"), 2)
    with pytest.raises(ValueError, match="endpoints"):
        gcoo.csr_to_gcoo_dev(2, 3, torch.ones(2, dtype=torch.float32, device="cuda"),
                             torch.tensor([0, 2], dtype=torch.int32, device="cuda"),
                             torch.tensor([0, 1, 3], dtype=torch.int64, device="cuda"), 2)


# ------------------------------------------------ full-size (BASELINE) -----
@pytest.mark.slow
@pytest.mark.parametrize("s", [0.99, 0.995, 0.9])
def test_full_size_n8000_matches_reference_hashes(gcoo, cuda, oracle, golden_hashes, s):
    """configs[1]: n=8000, the paper's headline sparsities, checked against the
    reference's own outputs (hashes of C from the reference built -mfma, and
    the GCOO arrays + KernelStats of the shipped build)."""
    import torch
    ent = golden_hashes[f"n8000_s{s}"]
    a = gcoo.generate_uniform_sparse(8000, s, 1)
    bm = gcoo.generate_uniform_sparse(8000, 0.0, gcoo.derive_seed(1, 8000, 0xB))
    assert oracle.fnv(a) == ent["A_fnv"] and oracle.fnv(bm) == ent["B_fnv"]
    d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
    g = d.to_host()
    for f in FIELDS:
        assert oracle.fnv(getattr(g, f)) == ent["p4"][f], f
    bt = torch.from_numpy(bm).cuda()
    ct = torch.empty((8000, 8000), dtype=torch.float32, device="cuda")
    st = gcoo.KernelStats()
    gcoo.spdm_gcoo_dev(d, bt, ct, stats=st)
    torch.cuda.synchronize()
    c = ct.cpu().numpy()
    assert oracle.fnv(c) == ent["C_fma"]["fnv"]
    assert [st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills] == ent["stats_p4_b64"]
    gcoo.spdm_gcoo_dev(d, bt, ct, flavor=gcoo.FLAVOR_MUL_ADD)
    torch.cuda.synchronize()
    assert oracle.fnv(ct.cpu().numpy()) == ent["C_mad"]["fnv"]
    # the public host API pipelines this size over column strips: same bits
    c_host = gcoo.spdm_gcoo(g, bm, gcoo.ExecConfig(), stats=(st2 := gcoo.KernelStats()))
    assert oracle.fnv(c_host) == ent["C_fma"]["fnv"]
    assert [st2.flops, st2.b_loads_total, st2.b_loads_reused, st2.staging_fills] == ent["stats_p4_b64"]


@pytest.mark.slow
def test_full_size_configs0_n4000_matches_reference_hashes(gcoo, cuda, oracle, golden_hashes):
    """configs[0] (n=4000, s=0.95: BASELINE's correctness-oracle case): the
    inputs, GCOO arrays, KernelStats and C (both flavours) against the hashes
    of the reference's own outputs — through the device API and through the
    host API the drop-in headers call."""
    import torch
    ent = golden_hashes["n4000_s0.95"]
    n = 4000
    a = gcoo.generate_uniform_sparse(n, 0.95, 1)
    bm = gcoo.generate_uniform_sparse(n, 0.0, gcoo.derive_seed(1, n, 0xB))
    assert oracle.fnv(a) == ent["A_fnv"] and oracle.fnv(bm) == ent["B_fnv"]
    g_host = gcoo.dense_to_gcoo(a, 4)
    for f in FIELDS:
        assert oracle.fnv(getattr(g_host, f)) == ent["p4"][f], f
    d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
    for f in FIELDS:
        assert oracle.fnv(getattr(d.to_host(), f)) == ent["p4"][f], f
    bt = torch.from_numpy(bm).cuda()
    ct = torch.empty((n, n), dtype=torch.float32, device="cuda")
    st = gcoo.KernelStats()
    gcoo.spdm_gcoo_dev(d, bt, ct, stats=st)
    torch.cuda.synchronize()
    assert oracle.fnv(ct.cpu().numpy()) == ent["C_fma"]["fnv"]
    assert [st.flops, st.b_loads_total, st.b_loads_reused, st.staging_fills] == ent["stats_p4_b64"]
    gcoo.spdm_gcoo_dev(d, bt, ct, flavor=gcoo.FLAVOR_MUL_ADD)
    torch.cuda.synchronize()
    assert oracle.fnv(ct.cpu().numpy()) == ent["C_mad"]["fnv"]
    c_host = gcoo.spdm_gcoo(g_host, bm, gcoo.ExecConfig())
    assert oracle.fnv(c_host) == ent["C_fma"]["fnv"]


@pytest.mark.parametrize("s", [0.999, 0.9975, 0.993, 0.985, 0.96, 0.85, 0.7])
def test_auto_choice_each_density_band_n8000_bit_exact(gcoo, cuda, oracle, s):
    """The kernel `choose_kind` picks at every density band (16 warps KC 216 /
    KC 192; 28 warps KC 200 / 192 / 160 / 128 / 96 / 64) on the full-size
    reference inputs, against the oracle's FMA chain bit for bit (sampled rows
    for the dense bands to keep the CPU check short)."""
    import torch
    n = 8000
    a = gcoo.generate_uniform_sparse(n, s, 1)
    bm = gcoo.generate_uniform_sparse(n, 0.0, gcoo.derive_seed(1, n, 0xB))
    d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
    ct = torch.empty((n, n), dtype=torch.float32, device="cuda")
    gcoo.spdm_gcoo_dev(d, torch.from_numpy(bm).cuda(), ct)
    torch.cuda.synchronize()
    c = ct.cpu().numpy()
    g = oracle.dense_to_gcoo(a, 4)
    if s >= 0.99:
        want, _ = oracle.spdm(g, bm, fma=True)
        assert c.tobytes() == want.tobytes()
    else:
        rng = np.random.default_rng(int(s * 1000))
        for r0 in sorted(rng.choice(n // 8, 6, replace=False) * 8):
            want = oracle.spdm_rows(g, bm, int(r0), int(r0) + 8, fma=True)[r0:r0 + 8]
            assert c[r0:r0 + 8].tobytes() == want.tobytes(), r0


@pytest.mark.parametrize("n", [2048, 2304, 2050, 3001])
def test_host_pipeline_strips_bitwise_equal(gcoo, cuda, oracle, n):
    """The host-pointer path splits B/C into column strips on three streams
    (n >= 2048); every strip width, including a ragged last strip (n % 4 != 0),
    must give the one-shot device result bit for bit, and the stats."""
    import torch
    rng = np.random.default_rng(n)
    m = k = 8192
    a = rand_dense(rng, m, k, 0.01)
    bm = (1.0 - rng.random((k, n))).astype(np.float32)
    g = gcoo.dense_to_gcoo(a, 4)
    st = gcoo.KernelStats()
    c_host = gcoo.spdm_gcoo(g, bm, gcoo.ExecConfig(), stats=st)
    d = gcoo.DeviceGcoo.from_host(g)
    ct = torch.empty((m, n), dtype=torch.float32, device="cuda")
    gcoo.force_kernel("rowtile")
    try:
        gcoo.spdm_gcoo_dev(d, torch.from_numpy(bm).cuda(), ct)
        torch.cuda.synchronize()
    finally:
        gcoo.force_kernel("auto")
    assert np.array_equal(c_host, ct.cpu().numpy())
    assert st.flops == 2 * g.nnz() * n


def test_host_staging_ring_pageable_and_pinned(gcoo, cuda, oracle):
    """The host-pointer path with pageable buffers packs B strips into and
    unpacks C strips out of a pinned staging ring on host threads; pinned
    buffers skip it; the driver-staged path remains as a switch.  All three
    give the same bits, for a ragged last strip too."""
    import torch
    rng = np.random.default_rng(77)
    m, k, n = 6000, 7000, 3001
    a = rand_dense(rng, m, k, 0.005)
    bm = (1.0 - rng.random((k, n))).astype(np.float32)
    g = gcoo.dense_to_gcoo(a, 4)
    c_ring = gcoo.spdm_gcoo(g, bm)
    gcoo.host_staging(False)
    try:
        c_driver = gcoo.spdm_gcoo(g, bm)
    finally:
        gcoo.host_staging(True)
    b_pin = torch.empty((k, n), dtype=torch.float32, pin_memory=True)
    b_pin.numpy()[:] = bm
    c_pin = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
    gcoo.spdm_gcoo(g, b_pin.numpy(), out=c_pin.numpy())
    assert np.array_equal(c_ring, c_driver) and np.array_equal(c_ring, c_pin.numpy())
    rows = np.random.default_rng(3).choice(m, 24, replace=False)
    go = oracle.dense_to_gcoo(a, 4)
    for r0 in rows:
        want = oracle.spdm_rows(go, bm, int(r0), int(r0) + 1, fma=True)[r0]
        assert c_ring[r0].tobytes() == want.tobytes()


@pytest.mark.slow
@pytest.mark.parametrize("case", ["powerlaw_n16384", "uniform_n32768"])
def test_large_configs_sampled_rows_bit_exact(gcoo, cuda, oracle, case):
    """BASELINE configs[3] and [4] at full size: C from the device path on a
    sample of rows x columns equals the oracle's FMA chain on the same
    entries, bit for bit (the per-element chain depends only on the row's
    entries and the column of B, so a sample is an exact check)."""
    import torch
    if case == "powerlaw_n16384":
        n = 16384
        v, r, c = gcoo.generate_powerlaw_coo(n, 0.99, 1.0, 1)
    else:
        n = 32768
        v, r, c = gcoo.generate_uniform_sparse_coo(n, 0.99, 1)
    dg = gcoo.coo_to_gcoo_dev(n, n, torch.from_numpy(v).cuda(), torch.from_numpy(r).cuda(),
                              torch.from_numpy(c).cuda(), 4)
    gen = torch.Generator(device="cuda").manual_seed(3)
    dB = 1.0 - torch.rand((n, n), device="cuda", dtype=torch.float32, generator=gen)
    dC = torch.empty((n, n), device="cuda", dtype=torch.float32)
    gcoo.spdm_gcoo_dev(dg, dB, dC)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    counts = np.bincount(r, minlength=n)
    rows = np.unique(np.concatenate([rng.choice(n, 48, replace=False), [int(np.argmax(counts))]]))
    cols = np.sort(rng.choice(n, 256, replace=False))
    sel = np.isin(r, rows)
    remap = {int(x): i for i, x in enumerate(rows)}
    a_sub = np.zeros((len(rows), n), np.float32)
    a_sub[[remap[int(x)] for x in r[sel]], c[sel]] = v[sel]
    b_sub = np.ascontiguousarray(dB[:, torch.from_numpy(cols).cuda()].cpu().numpy())
    c_ref, _ = oracle.spdm(oracle.dense_to_gcoo(a_sub, 4), b_sub, 64, fma=True)
    c_gpu = dC[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
    assert np.array_equal(c_gpu, c_ref)


@pytest.mark.slow
def test_output_beyond_2g_elements_bit_exact(gcoo, cuda, oracle):
    """C with more than 2^31 elements (70000 x 40000 fp32 = 11.2 GB): 64-bit
    offsets in the planner, TMA coordinates and the epilogue; sampled rows
    (first, last, random) x columns (incl. the last) equal the oracle bit for
    bit, for the default kernel and a dense-regime configuration."""
    import torch
    m, k, n = 70000, 512, 40000
    rng = np.random.default_rng(77)
    nnz = 700000
    flat = np.unique(rng.integers(0, m * k, size=nnz * 2, dtype=np.int64))[:nnz]
    rng.shuffle(flat)
    flat = np.sort(flat)
    r = (flat // k).astype(np.int32)
    c = (flat % k).astype(np.int32)
    v = (1.0 - rng.random(r.size)).astype(np.float32)
    dg = gcoo.coo_to_gcoo_dev(m, k, torch.from_numpy(v).cuda(), torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda(), 4)
    gen = torch.Generator(device="cuda").manual_seed(9)
    dB = 1.0 - torch.rand((k, n), device="cuda", dtype=torch.float32, generator=gen)
    dC = torch.empty((m, n), device="cuda", dtype=torch.float32)
    rows = np.unique(np.concatenate([[0, m - 1], rng.choice(m, 30, replace=False)]))
    cols = np.unique(np.concatenate([[0, n - 1], rng.choice(n, 100, replace=False)]))
    sel = np.isin(r, rows)
    remap = {int(x): i for i, x in enumerate(rows)}
    a_sub = np.zeros((len(rows), k), np.float32)
    a_sub[[remap[int(x)] for x in r[sel]], c[sel]] = v[sel]
    b_sub = np.ascontiguousarray(dB[:, torch.from_numpy(cols).cuda()].cpu().numpy())
    c_ref, _ = oracle.spdm(oracle.dense_to_gcoo(a_sub, 4), b_sub, 64, fma=True)
    for kern in ("auto", "tacc28_k64"):
        gcoo.force_kernel(kern)
        try:
            dC.fill_(float("nan"))
            gcoo.spdm_gcoo_dev(dg, dB, dC)
            torch.cuda.synchronize()
        finally:
            gcoo.force_kernel("auto")
        c_gpu = dC[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy()
        assert np.array_equal(c_gpu, c_ref), kern
    del dC


@pytest.mark.parametrize("kernel", ["tacc28_k192", "tacc28_k64", "tacc28_k200", "tacc_v4_k216", "tacc28_k176"])
def test_heavy_rows_balanced_placement(gcoo, cuda, oracle, kernel):
    """The TMEM kernels place rows heaviest-first across warps (a permutation
    of rows into accumulator slots): with very uneven rows C must still be
    bit-exact for every group size."""
    rng = np.random.default_rng(11)
    m, k, n = 1500, 3000, 384
    a = rand_dense(rng, m, k, 0.004)
    for r in (0, 17, 700, 1499):  # dense rows
        a[r] = (1.0 - rng.random(k)).astype(np.float32)
    a[900, ::2] = 0.5
    bm = (1.0 - rng.random((k, n))).astype(np.float32)
    gcoo.force_kernel(kernel)
    try:
        # 16 <= p <= 256: the fill ranks by (group, chunk) range; others: the per-entry scan
        for p in (1, 4, 16, 32, 256, 512):
            go = oracle.dense_to_gcoo(a, p)
            c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
            c = gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p))
            assert np.array_equal(c, c_ref), (kernel, p)
    finally:
        gcoo.force_kernel("auto")


# ----------------------------------------------------------- traffic model --
def _traffic_golden():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "traffic.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("n,s", [(512, 0.95), (8000, 0.99)])
def test_traffic_model_device_equals_reference_golden(gcoo, cuda, oracle, n, s):
    """gcoo_model_traffic_dev reproduces the reference's model_gcoo_traffic /
    model_csr_traffic counters exactly on the benchmark patterns (fixtures
    made by tests/golden/make_traffic_golden.py from oracle/_ref)."""
    import torch
    a = gcoo.generate_uniform_sparse(n, s, 1)
    d = gcoo.dense_to_gcoo_dev(torch.from_numpy(a).cuda(), 4)
    gold = _traffic_golden()[f"n{n}_s{s}"]
    for kind in ("gcoo", "csr"):
        for mode in ("cold", "infinite_l2"):
            got = gcoo.model_traffic_dev(d, n, gcoo.ExecConfig(p=4, b=64), mode == "infinite_l2", kind == "csr")
            assert got == gold[f"{kind}_{mode}"], (kind, mode)


def test_traffic_model_device_random_shapes(gcoo, cuda, oracle):
    """Ragged m, k, n; p and b from 1 to 128; empty groups and columns: the
    device model equals the plain-Python restatement (pinned to the reference
    in tests/test_oracle.py)."""
    from oracle import model_traffic
    rng = np.random.default_rng(23)
    for m, k, n, p, b, dens in [(37, 29, 70, 4, 8, 0.2), (64, 64, 64, 1, 1, 0.1), (50, 80, 33, 8, 64, 0.3),
                                (9, 9, 1, 2, 2, 0.5), (100, 7, 129, 64, 4, 0.05), (5, 300, 31, 2, 128, 0.0),
                                (300, 200, 1000, 16, 32, 0.02)]:
        a = rand_dense(rng, m, k, dens)
        g = gcoo.dense_to_gcoo(a, p)
        dg = gcoo.DeviceGcoo.from_host(g)
        rows, cols = np.nonzero(a)
        for inf in (False, True):
            for csr in (False, True):
                got = gcoo.model_traffic_dev(dg, n, gcoo.ExecConfig(p=p, b=b), inf, csr)
                assert got == model_traffic(rows, cols, m, k, n, p, b, inf, csr), (m, k, n, p, b, inf, csr)
    with pytest.raises(ValueError):
        gcoo.model_traffic_dev(dg, 10, gcoo.ExecConfig(p=16, b=3))



@pytest.mark.parametrize("p", [1, 4, 16])
def test_two_class_split_bit_exact(gcoo, cuda, oracle, p):
    """Skewed A (a few dense rows among sparse ones): the heavy rows and the
    light rows run as two plans with their own configurations, concurrently;
    C equals the oracle bit for bit through the device call, a reused plan and
    the pipelined host call, and the split is taken automatically."""
    import torch
    rng = np.random.default_rng(90 + p)
    m, k, n = 3000, 4000, 4096  # well above the small-product gate: the TMEM kernels run
    a = rand_dense(rng, m, k, 0.004)
    for r in rng.choice(m, 12, replace=False):  # dense and half-dense rows
        a[r] = np.where(rng.random(k) < (1.0 if r % 2 else 0.5), 1.0 - rng.random(k), 0.0)
    bm = rand_dense(rng, k, n, 1.0)
    go = oracle.dense_to_gcoo(a, p)
    c_ref, _ = oracle.spdm(go, bm, 64, fma=True)
    dg = gcoo.DeviceGcoo.from_host(to_prod(gcoo, go))
    bt = torch.from_numpy(bm).cuda()
    ct = torch.empty((m, n), device="cuda")
    for mode in ("auto", "always", "never"):
        gcoo.force_split(mode)
        try:
            ct.fill_(float("nan"))
            gcoo.spdm_gcoo_dev(dg, bt, ct, gcoo.ExecConfig(p=p))
            torch.cuda.synchronize()
            split = gcoo.last_split()
        finally:
            gcoo.force_split("auto")
        assert split == (mode != "never"), mode
        assert np.array_equal(ct.cpu().numpy(), c_ref), mode
    plan = gcoo.SpdmPlan(dg)
    ct.fill_(float("nan"))
    l0 = gcoo.launch_count()
    plan.run(bt, ct)
    torch.cuda.synchronize()
    assert gcoo.last_split() and gcoo.launch_count() - l0 == 2  # heavy + light multiply, nothing else
    assert np.array_equal(ct.cpu().numpy(), c_ref)
    plan.close()
    assert np.array_equal(gcoo.spdm_gcoo(to_prod(gcoo, go), bm, gcoo.ExecConfig(p=p)), c_ref)


def test_two_class_split_powerlaw_full_rows(gcoo, cuda, oracle):
    """The power-law generator's matrix (n=4096) splits automatically; sampled
    rows including the heaviest are bit-exact against the oracle."""
    import torch
    n = 4096
    v, r, c = gcoo.generate_powerlaw_coo(n, 0.99, 1.0, 3)
    dg = gcoo.coo_to_gcoo_dev(n, n, torch.from_numpy(v).cuda(), torch.from_numpy(r).cuda(),
                              torch.from_numpy(c).cuda(), 4)
    bm = oracle.uniform_sparse(n, 0.0, 14)[:, :2048].copy()  # 0.7 GFLOP: above the small-product gate
    ct = torch.empty((n, 2048), device="cuda")
    gcoo.spdm_gcoo_dev(dg, torch.from_numpy(bm).cuda(), ct)
    torch.cuda.synchronize()
    assert gcoo.last_split()
    go = oracle.coo_to_gcoo(n, n, v, r, c, 4)
    counts = np.bincount(r, minlength=n)
    rows = np.unique(np.concatenate([np.argsort(-counts)[:20], np.random.default_rng(2).choice(n, 40, replace=False)]))
    got = ct.cpu().numpy()
    for r0 in rows:
        want = oracle.spdm_rows(go, bm, int(r0), int(r0) + 1, fma=True)[r0]
        assert got[r0].tobytes() == want.tobytes(), r0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_spdm_gcoo_auto_device_resident(gcoo, cuda, oracle, dtype):
    """spdm_gcoo_auto keeps the GCOO on the device between EO and KC: C and
    KernelStats equal the two-call path bit for bit, both phases are timed,
    and the pipelined size works from the resident GCOO too."""
    rng = np.random.default_rng(31)
    for m, k, n in [(300, 257, 129), (5000, 6000, 2304)]:
        a = rand_dense(rng, m, k, 0.01, dtype)
        bm = rand_dense(rng, k, n, 1.0, dtype)
        tb = gcoo.TimingBreakdown()
        st = gcoo.KernelStats()
        c = gcoo.spdm_gcoo_auto(a, bm, gcoo.ExecConfig(), tb, st)
        st2 = gcoo.KernelStats()
        c2 = gcoo.spdm_gcoo(gcoo.dense_to_gcoo(a, 4), bm, gcoo.ExecConfig(), stats=st2)
        assert np.array_equal(c, c2), (m, k, n)
        assert st == st2
        assert tb.eo_seconds > 0 and tb.kc_seconds > 0
    with pytest.raises(ValueError):
        gcoo.spdm_gcoo_auto(a, bm[:-1], gcoo.ExecConfig(), gcoo.TimingBreakdown())
