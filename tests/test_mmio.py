"""MatrixMarket ingestion: paper_2005_14469_b200.mmio.

* the reference's own io cases (proj/tests/test_io.cpp:56-270) restated:
  loading, symmetric expansion, pattern/integer fields, array layouts, the
  line number of every parse failure, write -> read round trips;
* byte-equality of written files and equality of parsed results / failure
  lines against the reference's reader and writer themselves (oracle/_ref,
  `ref_mtx_*` in oracle/ref_shim.cpp), on seeded random and mutated files;
* on the GPU: file -> read_matrix_market_gcoo_dev equals the reference's
  coo_to_gcoo / dense_to_gcoo of the same file, bit for bit.
"""
import os
import random
import zlib

import numpy as np
import pytest

from paper_2005_14469_b200 import mmio

EX4 = {(0, 0): 7, (0, 3): 8, (1, 1): 10, (2, 0): 9, (3, 2): 6, (3, 3): 3}


def _w(tmp_path, text, name="f.mtx"):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def _line(path):
    with pytest.raises(mmio.ParseError) as e:
        mmio.read_matrix_market(path, np.float64)
    assert str(e.value).startswith(f"line {e.value.line}: ")
    return e.value.line


def test_coordinate_general_order_independent(tmp_path):
    # test_io.cpp:60-80
    p = _w(tmp_path, "%%MatrixMarket matrix coordinate real general\n% free-form comment\n4 4 6\n"
                     "4 4 3\n1 1 7\n4 3 6\n2 2 10\n1 4 8\n3 1 9\n")
    coo = mmio.read_matrix_market(p, np.float64)
    keys = sorted(EX4)
    assert coo.values.tolist() == [EX4[k] for k in keys]
    assert coo.row_idx.tolist() == [k[0] for k in keys]
    assert coo.col_idx.tolist() == [k[1] for k in keys]
    assert (coo.rows_dim, coo.cols_dim) == (4, 4)
    assert coo.row_idx.dtype == np.int32 and coo.values.dtype == np.float64


def test_symmetric_expands(tmp_path):
    # test_io.cpp:82-103
    p = _w(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 5\n2 1 2\n3 1 3\n3 3 7\n")
    coo = mmio.read_matrix_market(p, np.float64)
    assert coo.nnz() == 6
    d = np.zeros((3, 3))
    d[coo.row_idx, coo.col_idx] = coo.values
    assert d.tolist() == [[5, 2, 3], [2, 0, 0], [3, 0, 7]]


def test_pattern_and_integer(tmp_path):
    # test_io.cpp:105-127
    coo = mmio.read_matrix_market(_w(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n"),
                                  np.float64)
    assert coo.values.tolist() == [1.0, 1.0]
    assert coo.row_idx.tolist() == [0, 1] and coo.col_idx.tolist() == [1, 0]
    coo = mmio.read_matrix_market(_w(tmp_path, "%%MatrixMarket matrix coordinate integer general\n2 2 1\n2 2 -3\n"),
                                  np.float64)
    assert coo.values.tolist() == [-3.0]


def test_array_layouts(tmp_path):
    # test_io.cpp:129-149
    d = mmio.read_matrix_market(_w(tmp_path, "%%MatrixMarket matrix array real general\n2 3\n1\n4\n2\n5\n3\n6\n"),
                                np.float64)
    assert d.shape == (2, 3) and d.ravel().tolist() == [1, 2, 3, 4, 5, 6]
    d = mmio.read_matrix_market(_w(tmp_path, "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n"),
                                np.float64)
    assert d.ravel().tolist() == [1, 2, 3, 2, 4, 5, 3, 5, 6]


BAD = [  # (text, line) — test_io.cpp:151-237
    ("%%NotMatrixMarket matrix coordinate real general\n1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 0\n", 1),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n", 1),
    ("%%MatrixMarket vector coordinate real general\n1 1 0\n", 1),
    ("%%MatrixMarket matrix array pattern general\n1 1\n", 1),
    ("%%MatrixMarket matrix coordinate real general\n% sizes below\n4 four 6\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n0 4 0\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n4 4 99\n", 2),
    ("%%MatrixMarket matrix coordinate real symmetric\n3 4 0\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n% one comment\n4 4 2\n1 1 1.0\n5 1 2.0\n", 5),
    ("%%MatrixMarket matrix coordinate real general\n4 4 3\n2 2 1.0\n1 1 4.0\n2 2 9.0\n", 5),
    ("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1.0\n1 2 1.0\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n4 4 3\n1 1 1.0\n2 2 2.0\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n4 4 1\n1 1 1.0\n2 2 2.0\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n4 4 1\n1 1 abc\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n4 4 1\n1 1 1.0 junk\n", 3),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n", 5),
    # beyond the reference's list
    ("", 1),
    ("%%MatrixMarket matrix coordinate real general\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1 7\n", 2),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n5\n", 7),
    ("%%MatrixMarket matrix array real general\n2 2\n1\nx\n3\n4\n", 4),
    ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1.5 1 2\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 inf\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1\n", 3),
    ("%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1 1\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n\n% c\n2 2 2\n  \n1 1 5\n", 8),
]


@pytest.mark.parametrize("text,line", BAD)
def test_parse_failures_name_the_line(tmp_path, text, line):
    assert _line(_w(tmp_path, text)) == line


def test_missing_file(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        mmio.read_matrix_market(str(tmp_path / "does_not_exist.mtx"))


def _random_dense(rng, rows, cols, density, dtype):
    a = rng.random((rows, cols)).astype(dtype) * (rng.random((rows, cols)) < density)
    a[a != 0] = (rng.standard_normal(int((a != 0).sum())) * 10.0 ** rng.integers(-30, 30, int((a != 0).sum()))).astype(dtype)
    return a


def _dense_to_coo(a):
    r, c = np.nonzero(a)
    return mmio.CooMatrix(a.shape[0], a.shape[1], a[r, c], r.astype(np.int32), c.astype(np.int32))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_roundtrip_exact(tmp_path, dtype):
    # test_io.cpp:239-270: write then read recovers the matrix exactly
    rng = np.random.default_rng(2024)
    p = str(tmp_path / "rt.mtx")
    for _ in range(20):
        rows, cols = (int(x) for x in rng.integers(1, 41, 2))
        coo = _dense_to_coo(_random_dense(rng, rows, cols, 0.3, dtype))
        mmio.write_matrix_market(coo, p)
        back = mmio.read_matrix_market(p, dtype)
        assert np.array_equal(back.values.view(np.uint8), coo.values.view(np.uint8))
        assert back.row_idx.tolist() == coo.row_idx.tolist() and back.col_idx.tolist() == coo.col_idx.tolist()
    a = _random_dense(rng, 7, 5, 1.0, dtype)
    mmio.write_matrix_market(a, p)
    assert np.array_equal(mmio.read_matrix_market(p, dtype), a)


# ---------------------------------------------------------------------------
# against the reference's own reader and writer (oracle/_ref)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_writer_bytes_equal_reference(tmp_path, reference, dtype):
    ref = reference[0]
    rng = np.random.default_rng(7)
    for it in range(6):
        rows, cols = (int(x) for x in rng.integers(1, 60, 2))
        a = _random_dense(rng, rows, cols, 0.25, dtype)
        coo = _dense_to_coo(a)
        mine, theirs = str(tmp_path / "m.mtx"), str(tmp_path / "r.mtx")
        mmio.write_matrix_market(coo, mine)
        ref.write_mtx(theirs, coo=(rows, cols, coo.values, coo.row_idx, coo.col_idx))
        assert open(mine, "rb").read() == open(theirs, "rb").read()
        mmio.write_matrix_market(a, mine)
        ref.write_mtx(theirs, a=a)
        assert open(mine, "rb").read() == open(theirs, "rb").read()


def _mutate(text: str, rnd: random.Random) -> str:
    lines = text.split("\n")
    i = rnd.randrange(len(lines))
    op = rnd.randrange(9)
    if op == 0:
        lines.insert(i, "% comment")
    elif op == 1:
        lines.insert(i, "   ")
    elif op == 2 and len(lines) > 2:
        del lines[max(1, i)]
    elif op == 3:
        lines[i] = lines[i] + " 1"
    elif op == 4:
        lines[i] = lines[i].replace("1", "x", 1)
    elif op == 5:
        lines.insert(max(1, i), lines[max(1, i) - 1] if i > 1 else "1 1 1")
    elif op == 6:
        lines[i] = lines[i].replace(" ", "\t", 1)
    elif op == 7:
        lines[i] = lines[i].replace("2", "9999", 1)
    else:
        lines[i] = " " + lines[i] + "\r"
    return "\n".join(lines)


KINDS = ["coordinate general", "coordinate symmetric", "pattern general", "array general", "array symmetric",
         "integer symmetric"]


def _gen_case(kind, it, rnd, rng):
    fmt, sym = kind.split()
    n = rnd.randrange(1, 9)
    m = n if sym == "symmetric" else rnd.randrange(1, 9)
    a = _random_dense(rng, n, m, 0.4, np.float64)
    if sym == "symmetric":
        a = np.tril(a) + np.tril(a, -1).T
    if fmt == "integer":
        a = rng.integers(-9, 9, a.shape) * (a != 0)
    field = {"coordinate": "real", "pattern": "pattern", "array": "real", "integer": "integer"}[fmt]
    body = []
    if fmt == "array":
        for c in range(m):
            for r in range(c if sym == "symmetric" else 0, n):
                body.append("%.17g" % a[r, c])
        text = f"%%MatrixMarket matrix array {field} {sym}\n{n} {m}\n" + "\n".join(body) + "\n"
    else:
        rr, cc = np.nonzero(np.tril(a) if sym == "symmetric" else a)
        for j in rng.permutation(rr.size):
            v = "" if field == "pattern" else " %.17g" % a[rr[j], cc[j]] if field == "real" else " %d" % a[rr[j], cc[j]]
            body.append(f"{rr[j] + 1} {cc[j] + 1}{v}")
        text = f"%%MatrixMarket matrix coordinate {field} {sym}\n{n} {m} {rr.size}\n" + "\n".join(body) + "\n"
    if it % 3:
        for _ in range(rnd.randrange(1, 3)):
            text = _mutate(text, rnd)
    return text


def _compare_with_reference(ref, p, text):
    for dtype in (np.float32, np.float64):
        theirs = ref.read_mtx(p, dtype)
        try:
            mine = mmio.read_matrix_market(p, dtype)
        except mmio.ParseError as e:
            assert theirs[0] == "error", (text, str(e), theirs)
            assert e.line == theirs[1], (text, str(e), theirs)
            continue
        assert theirs[0] != "error", (text, theirs)
        if theirs[0] == "dense":
            assert isinstance(mine, np.ndarray) and mine.dtype == dtype
            assert np.array_equal(mine, theirs[1])
        else:
            _, m_, k_, v, r, c = theirs
            assert (mine.rows_dim, mine.cols_dim) == (m_, k_)
            assert mine.values.tobytes() == v.tobytes()
            assert mine.row_idx.tolist() == r.tolist() and mine.col_idx.tolist() == c.tolist()


@pytest.mark.parametrize("kind", KINDS)
def test_reader_matches_reference(tmp_path, reference, kind):
    """Random files of each header kind, clean and mutated (deleted/duplicated/
    garbled lines, comments, CRs, extra tokens): same result or same failure
    line as the reference's read_matrix_market."""
    ref = reference[0]
    seed = zlib.crc32(kind.encode())
    rnd, rng = random.Random(seed), np.random.default_rng(seed)
    p = str(tmp_path / "x.mtx")
    for it in range(150):
        text = _gen_case(kind, it, rnd, rng)
        with open(p, "w", newline="") as f:
            f.write(text)
        _compare_with_reference(ref, p, text)


def test_reader_value_rounding_matches_reference(tmp_path, reference):
    """Decimal -> double -> float conversions agree bit for bit (strtod vs numpy)."""
    ref = reference[0]
    rnd = random.Random(11)
    body = []
    for i in range(2000):
        mant = "".join(rnd.choice("0123456789") for _ in range(rnd.randrange(1, 25)))
        dot = rnd.randrange(len(mant) + 1)
        s = mant[:dot] + "." + mant[dot:] if rnd.random() < 0.8 else mant
        if rnd.random() < 0.7:
            sign = rnd.choice(["", "+", "-"])        # subnormal / underflow on the negative side
            s += rnd.choice("eE") + sign + str(rnd.randrange(0, 345 if sign == "-" else 280))
        body.append(f"{i + 1} 1 {rnd.choice(['', '-', '+'])}{s}")
    p = _w(tmp_path, "%%MatrixMarket matrix coordinate real general\n2000 1 2000\n" + "\n".join(body) + "\n")
    for dtype in (np.float32, np.float64):
        theirs = ref.read_mtx(p, dtype)
        mine = mmio.read_matrix_market(p, dtype)
        assert mine.values.tobytes() == theirs[3].tobytes()


# ---------------------------------------------------------------------------
# file -> GCOO on the B200
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 4, 64])
def test_mtx_to_gcoo_dev_matches_reference(tmp_path, cuda, gcoo, oracle, p):
    rng = np.random.default_rng(p)
    a = _random_dense(rng, 300, 257, 0.05, np.float32)
    f = str(tmp_path / "a.mtx")
    mmio.write_matrix_market(_dense_to_coo(a), f)
    d = mmio.read_matrix_market_gcoo_dev(f, p)
    want = oracle.dense_to_gcoo(a, p)
    got = d.to_host()
    for name in ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group"):
        assert np.array_equal(np.asarray(getattr(got, name)), np.asarray(getattr(want, name))), name
    # array format -> dense_to_gcoo_dev
    mmio.write_matrix_market(a, f)
    got = mmio.read_matrix_market_gcoo_dev(f, p).to_host()
    for name in ("values", "row_idx", "col_idx", "g_idxes", "nnz_per_group"):
        assert np.array_equal(np.asarray(getattr(got, name)), np.asarray(getattr(want, name))), name


def test_native_tokenizer_chunking(gcoo):
    """gcoo_mtx_parse_entries gives the same rows for 1..13 newline-aligned
    chunks (chunk edges inside comments, blank lines, CRLF and a missing final
    newline), and flags an irregular line in any chunk."""
    import ctypes as C
    f = gcoo.lib().gcoo_mtx_parse_entries
    f.restype = C.c_int64
    f.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
    rnd = random.Random(5)
    lines = []
    for i in range(400):
        t = rnd.random()
        if t < 0.1:
            lines.append("% comment " + str(i))
        elif t < 0.15:
            lines.append(rnd.choice(["", "  ", "\t\r"]))
        else:
            lines.append(f" {rnd.randrange(1, 99)}\t{rnd.randrange(1, 99)} {rnd.uniform(-1e3, 1e3)!r}" +
                         ("\r" if rnd.random() < 0.2 else ""))
    body = "\n".join(lines).encode()

    def run(text, threads, cap=500):
        idx, vals, line = np.zeros((cap, 2), np.int64), np.zeros(cap), np.zeros(cap, np.int64)
        n = f(text, len(text), 3, cap, idx.ctypes.data, vals.ctypes.data, line.ctypes.data, threads)
        return n, idx[:max(n, 0)], vals[:max(n, 0)], line[:max(n, 0)]

    n1, i1, v1, l1 = run(body, 1)
    want = [j for j, s in enumerate(lines) if s.strip() and not s.lstrip().startswith("%")]
    assert n1 == len(want) and l1.tolist() == want
    assert v1.tolist() == [float(lines[j].split()[2]) for j in want]
    for t in range(2, 14):
        n, i, v, l = run(body, t)
        assert n == n1 and np.array_equal(i, i1) and v.tobytes() == v1.tobytes() and np.array_equal(l, l1)
    bad = lines.copy()
    bad[want[-1]] += " extra"
    for t in (1, 3, 8):
        assert run("\n".join(bad).encode(), t)[0] == -1
    assert run(b"", 4)[0] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("header", ["pattern symmetric", "real symmetric", "integer general"])
def test_mtx_file_to_spdm_on_gpu_bit_exact(tmp_path, cuda, gcoo, oracle, header):
    """A SuiteSparse-style file (symmetric / pattern / integer, scrambled entry
    order, comments) -> read_matrix_market_gcoo_dev -> spdm_gcoo_dev: C
    bit-identical to the oracle's FMA chain on the reference reader's COO."""
    import torch
    field, sym = header.split()
    rng = np.random.default_rng(len(header))
    n = 700
    a = (rng.random((n, n)) < 0.01) * rng.integers(1, 9, (n, n)).astype(np.float64)
    if sym == "symmetric":
        a = np.tril(a) + np.tril(a, -1).T
        rr, cc = np.nonzero(np.tril(a))
    else:
        rr, cc = np.nonzero(a)
    lines = [f"%%MatrixMarket matrix coordinate {field} {sym}", "% generated", f"{n} {n} {rr.size}"]
    for j in rng.permutation(rr.size):
        v = "" if field == "pattern" else f" {int(a[rr[j], cc[j]])}"
        lines.append(f"{rr[j] + 1} {cc[j] + 1}{v}")
    f = _w(tmp_path, "\n".join(lines) + "\n")
    if field == "pattern":
        a = (a != 0).astype(np.float64)
    d = mmio.read_matrix_market_gcoo_dev(f, 4)
    B = rng.random((n, 384)).astype(np.float32)
    Cd = torch.empty((n, 384), dtype=torch.float32, device="cuda")
    gcoo.spdm_gcoo_dev(d, torch.from_numpy(B).cuda(), Cd)
    want, _ = oracle.spdm(oracle.dense_to_gcoo(a.astype(np.float32), 4), B, fma=True)
    assert Cd.cpu().numpy().tobytes() == want.tobytes()
