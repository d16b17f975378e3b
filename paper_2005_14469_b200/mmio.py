"""MatrixMarket exchange files -> GCOO on the B200.

Python mirror of the reference's `read_matrix_market` / `write_matrix_market`
(`proj/include/gcoo/io.hpp:21-109`, parser and writer in `proj/src/io.cpp:57-205`),
with the same accepted headers, the same 1-based line numbers in `ParseError`,
the same output order and the same bytes written:

* headers `%%MatrixMarket matrix coordinate|array real|integer|pattern
  general|symmetric` (io.cpp:66-84); coordinate files load as a `CooMatrix`
  sorted row-major (symmetric entries mirrored, pattern entries = 1), array
  files as a dense row-major ndarray read column-major (io.cpp:138-158);
* every failure the reference reports as a ParseError is reported at the same
  line (io.cpp:86-136, `tests/test_io.cpp` "parse failures name the offending
  line");
* writing prints `%lld %lld %.{digits}g` with digits = max_digits10 of the
  element type (io.cpp:164-191), so reference and mirror files are byte-equal.

Parsing is host work (text -> numbers); the result goes to the device once and
`read_matrix_market_gcoo_dev` builds the GCOO there with the GPU
`coo_to_gcoo_dev` / `dense_to_gcoo_dev` kernels.  The common path is
vectorised with numpy (one tokenise pass, C-level number conversion); any line
that fails the vectorised checks sends the file through a line-by-line
re-parse that reproduces the reference's exact first error.
"""
from __future__ import annotations

import os
import re
from dataclasses import dataclass

import numpy as np

__all__ = ["ParseError", "CooMatrix", "read_matrix_market", "write_matrix_market", "read_matrix_market_gcoo_dev"]

_WS = b" \t\r\v\f"
_INT32_MAX = 2**31 - 1


class ParseError(RuntimeError):
    """io.hpp:36-42: message "line N: what", `.line` = the 1-based line."""

    def __init__(self, what: str, line: int):
        super().__init__(f"line {line}: {what}")
        self.line = line


@dataclass
class CooMatrix:
    """CooMatrix<T> (matrix.hpp:72-116): row-major sorted coordinates."""
    rows_dim: int
    cols_dim: int
    values: np.ndarray
    row_idx: np.ndarray
    col_idx: np.ndarray

    def nnz(self) -> int:
        return int(self.values.size)

    def validate(self) -> None:
        """CooMatrix::validate (matrix.hpp:95-115): same checks, same messages."""
        if self.rows_dim < 1 or self.cols_dim < 1:
            raise ValueError("CooMatrix: dimensions must be >= 1")
        if not (self.values.size == self.row_idx.size == self.col_idx.size):
            raise ValueError("CooMatrix: array lengths differ")
        r = self.row_idx.astype(np.int64, copy=False)
        c = self.col_idx.astype(np.int64, copy=False)
        bad = np.flatnonzero((r < 0) | (r >= self.rows_dim) | (c < 0) | (c >= self.cols_dim))
        if bad.size:
            raise ValueError(f"CooMatrix: coordinate out of range at entry {int(bad[0])}")
        if r.size > 1:
            ok = (r[:-1] < r[1:]) | ((r[:-1] == r[1:]) & (c[:-1] < c[1:]))
            bad = np.flatnonzero(~ok)
            if bad.size:
                raise ValueError(f"CooMatrix: entries not in row-major order (or duplicate) at entry {int(bad[0]) + 1}")


# --------------------------------------------------------------------------
# reading
# --------------------------------------------------------------------------

def _lines(data: bytes):
    """std::getline over '\\n' (io.cpp:34-43): a trailing newline ends the last line."""
    if not data:
        return []
    ls = data.split(b"\n")
    if data.endswith(b"\n"):
        ls.pop()
    return ls


def _is_data(line: bytes) -> bool:
    t = line.lstrip(_WS)
    return bool(t) and t[:1] != b"%"


class _Stream:
    """istringstream >> emulation for one line: long long, double, string."""
    _LL = re.compile(rb"[ \t\r\v\f\n]*([+-]?[0-9]+)")
    _DBL = re.compile(rb"[ \t\r\v\f\n]*([+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?)")
    _TOK = re.compile(rb"[ \t\r\v\f\n]*([^ \t\r\v\f\n]+)")

    def __init__(self, line: bytes):
        self.s, self.pos = line, 0

    def _take(self, rx):
        m = rx.match(self.s, self.pos)
        if not m:
            return None
        self.pos = m.end()
        return m.group(1)

    def ll(self):
        t = self._take(self._LL)
        if t is None:
            return None
        v = int(t)
        return v if -2**63 <= v < 2**63 else None

    def dbl(self):
        # num_get: an out-of-range decimal (strtod overflow) sets failbit;
        # underflow yields 0 or a subnormal and succeeds
        t = self._take(self._DBL)
        if t is None:
            return None
        v = float(t)
        return None if np.isinf(v) else v

    def junk(self):
        return self._take(self._TOK)


def _consumed(st: _Stream, line: int) -> None:
    j = st.junk()
    if j is not None:
        raise ParseError(f"trailing tokens '{j.decode(errors='replace')}'", line)


def _header(data: bytes):
    """Banner and size line (io.cpp:62-107).  Returns (format, field, symmetry,
    rows, cols, declared, body_offset, lines_before_body)."""
    def line_at(pos):
        e = data.find(b"\n", pos)
        return (data[pos:], len(data)) if e < 0 else (data[pos:e], e + 1)

    banner, pos = line_at(0)
    toks = banner.split() + [b""] * 5
    tag, obj, fmt, field, sym = (t.decode(errors="replace").lower() for t in toks[:5])
    if tag != "%%matrixmarket":
        raise ParseError("missing %%MatrixMarket banner", 1)
    if obj != "matrix":
        raise ParseError(f"unsupported object '{obj}'", 1)
    if fmt not in ("coordinate", "array"):
        raise ParseError(f"unsupported format '{fmt}'", 1)
    if field not in ("real", "integer", "pattern"):
        raise ParseError(f"unsupported field '{field}'", 1)
    if sym not in ("general", "symmetric"):
        raise ParseError(f"unsupported symmetry '{sym}'", 1)
    if fmt == "array" and field == "pattern":
        raise ParseError("array format cannot carry a pattern field", 1)
    ln = 1
    while True:
        if pos >= len(data):
            raise ParseError("missing size line", ln + 1)
        line, pos = line_at(pos)
        ln += 1
        if _is_data(line):
            break
    st = _Stream(line)
    rows, cols = st.ll(), None
    if rows is not None:
        cols = st.ll()
    declared = 0
    if fmt == "coordinate":
        declared = st.ll() if cols is not None else None
        if rows is None or cols is None or declared is None:
            raise ParseError("malformed size line", ln)
    elif rows is None or cols is None:
        raise ParseError("malformed size line", ln)
    _consumed(st, ln)
    if rows < 1 or cols < 1:
        raise ParseError("dimensions must be positive", ln)
    if rows > _INT32_MAX or cols > _INT32_MAX:
        raise ParseError("dimension exceeds index range", ln)
    if sym == "symmetric" and rows != cols:
        raise ParseError("symmetric matrix must be square", ln)
    if fmt == "coordinate" and (declared < 0 or declared > rows * cols):
        raise ParseError("entry count outside [0, rows*cols]", ln)
    return fmt, field, sym, rows, cols, declared, pos, ln


def _parse_entries(body: bytes, ln0: int, ncol: int, cap: int):
    """The entry section through the native multi-threaded tokenizer
    (gcoo_mtx_parse_entries, csrc/host_mtx.cpp).  Returns (line_numbers,
    indices (n, 2) int64, values float64) for up to `cap` data lines plus the
    total data-line count, or None when some data line is irregular — the
    caller then re-reads line by line to report the reference's exact error."""
    import ctypes as C

    from . import lib
    f = lib().gcoo_mtx_parse_entries
    f.restype = C.c_int64
    f.argtypes = [C.c_char_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
    idx = np.empty((cap, 2), np.int64)
    vals = np.empty(cap, np.float64)
    line = np.empty(cap, np.int64)
    n = f(body, len(body), ncol, cap, idx.ctypes.data, vals.ctypes.data, line.ctypes.data, 0)
    if n < 0:
        return None
    k = min(n, cap)
    return line[:k] + ln0 + 1, idx[:k], vals[:k], n


def _coord_slow(lines, ln0, field, sym, rows, cols, declared):
    """Line-by-line coordinate parse (io.cpp:112-132): raises the reference's first error."""
    i = 0
    for e in range(declared):
        while i < len(lines) and not _is_data(lines[i]):
            i += 1
        if i >= len(lines):
            raise ParseError(f"expected {declared} entries, file ends after {e}", ln0 + len(lines))
        ln = ln0 + i + 1
        st = _Stream(lines[i])
        r = st.ll()
        c = st.ll() if r is not None else None
        if r is None or c is None:
            raise ParseError("malformed entry", ln)
        if field != "pattern" and st.dbl() is None:
            raise ParseError("malformed or missing value", ln)
        _consumed(st, ln)
        if r < 1 or r > rows or c < 1 or c > cols:
            raise ParseError("coordinate out of range", ln)
        if sym == "symmetric" and c > r:
            raise ParseError("entry above the diagonal in a symmetric file", ln)
        i += 1
    while i < len(lines):
        if _is_data(lines[i]):
            raise ParseError("more entries than the size line declares", ln0 + i + 1)
        i += 1


def _read_coordinate(body, ln0, field, sym, rows, cols, declared, dtype):
    ncol = 2 if field == "pattern" else 3
    got = _parse_entries(body, ln0, ncol, declared + 1)
    fast = got is not None and got[3] == declared
    if fast:
        line_no, ij, v = got[0], got[1], got[2]
        r, c = ij[:, 0].copy(), ij[:, 1].copy()
        if ncol == 2:
            v = np.ones(declared, np.float64)
        bad = (r < 1) | (r > rows) | (c < 1) | (c > cols)
        if sym == "symmetric":
            bad |= c > r
        fast = not bad.any()
    if not fast:
        _coord_slow(_lines(body), ln0, field, sym, rows, cols, declared)
        raise AssertionError("native MatrixMarket checks rejected a file the line parser accepts")
    r, c = r - 1, c - 1
    if sym == "symmetric":
        off = r != c
        r, c = np.concatenate([r, c[off]]), np.concatenate([c, r[off]])
        v = np.concatenate([v, v[off]])
        line_no = np.concatenate([line_no, line_no[off]])
    # io.cpp:122-132: sort by (row, col, line), a repeated coordinate is an error
    key = r * cols + c
    if key.size > 1 and not (key[1:] > key[:-1]).all():       # files written row-major skip the sort
        order = np.argsort(key, kind="stable")
        key = key[order]
        dup = np.flatnonzero(key[1:] == key[:-1])
        if dup.size:
            order = np.lexsort((line_no, c, r))
            r, c, line_no = r[order], c[order], line_no[order]
            j = int(np.flatnonzero((r[1:] == r[:-1]) & (c[1:] == c[:-1]))[0]) + 1
            raise ParseError(f"duplicate entry at ({int(r[j]) + 1}, {int(c[j]) + 1})", int(line_no[j]))
        r, c, v = r[order], c[order], v[order]
    with np.errstate(over="ignore"):                 # static_cast<float>(1e308) = inf, as in C++
        v = v.astype(dtype)
    out = CooMatrix(int(rows), int(cols), v, r.astype(np.int32), c.astype(np.int32))
    out.validate()
    return out


def _read_array(body, ln0, sym, rows, cols, dtype):
    """io.cpp:138-158: column-major values, lower triangle when symmetric."""
    need = rows * cols if sym == "general" else rows * (rows + 1) // 2
    got = _parse_entries(body, ln0, 1, need + 1)
    if got is None or got[3] < need:
        lines = _lines(body)
        n, i = 0, 0
        while n < need and i < len(lines):
            if _is_data(lines[i]):
                st = _Stream(lines[i])
                if st.dbl() is None:
                    raise ParseError("malformed array value", ln0 + i + 1)
                _consumed(st, ln0 + i + 1)
                n += 1
            i += 1
        if n < need:
            raise ParseError(f"file ends after {n} array values", ln0 + len(lines))
        for j in range(i, len(lines)):
            if _is_data(lines[j]):
                raise ParseError("more array values than the shape holds", ln0 + j + 1)
        raise AssertionError("native MatrixMarket checks rejected a file the line parser accepts")
    line_no, vals = got[0], got[2]
    if got[3] > need:
        raise ParseError("more array values than the shape holds", int(line_no[need]))
    vals = vals[:need]
    out = np.zeros((rows, cols), np.float64)
    if sym == "general":
        out[:] = vals.reshape(cols, rows).T
    else:
        rr, cc = np.tril_indices(rows)            # row-major lower triangle ...
        o = np.lexsort((rr, cc))                  # ... visited column by column
        out[rr[o], cc[o]] = vals
        out[cc[o], rr[o]] = vals
    with np.errstate(over="ignore"):
        return out.astype(dtype)


def read_matrix_market(path, dtype=np.float32):
    """read_matrix_market<T> (io.hpp:66-85): CooMatrix for coordinate files,
    a (rows, cols) ndarray for array files.  Raises ParseError (line-numbered)
    for malformed files and RuntimeError("cannot open ...") when unreadable."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise RuntimeError(f"cannot open {os.fspath(path)}") from None
    if not data:
        raise ParseError("empty file", 1)
    fmt, field, sym, rows, cols, declared, off, ln0 = _header(data)
    body = data[off:]
    if fmt == "coordinate":
        return _read_coordinate(body, ln0, field, sym, rows, cols, declared, dtype)
    return _read_array(body, ln0, sym, rows, cols, dtype)


# --------------------------------------------------------------------------
# writing
# --------------------------------------------------------------------------

def _digits(dtype) -> int:
    return 9 if np.dtype(dtype) == np.float32 else 17          # std::numeric_limits<T>::max_digits10


def write_matrix_market(m, path) -> None:
    """write_matrix_market (io.hpp:87-109, io.cpp:164-191): a CooMatrix as
    `coordinate real general`, an ndarray as `array real general` (column-major)."""
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot open {os.fspath(path)} for writing") from None
    with f:
        if isinstance(m, CooMatrix):
            m.validate()
            fmt = "%d %d %.{}g".format(_digits(m.values.dtype))
            f.write("%%MatrixMarket matrix coordinate real general\n")
            f.write(f"{m.rows_dim} {m.cols_dim} {m.nnz()}\n")
            rows = (m.row_idx.astype(np.int64) + 1).tolist()
            cols = (m.col_idx.astype(np.int64) + 1).tolist()
            vals = m.values.astype(np.float64).tolist()
            f.writelines(fmt % t + "\n" for t in zip(rows, cols, vals))
        else:
            a = np.asarray(m)
            fmt = "%.{}g\n".format(_digits(a.dtype))
            f.write("%%MatrixMarket matrix array real general\n")
            f.write(f"{a.shape[0]} {a.shape[1]}\n")
            f.writelines(fmt % v for v in a.T.astype(np.float64).ravel().tolist())


# --------------------------------------------------------------------------
# file -> device GCOO
# --------------------------------------------------------------------------

def read_matrix_market_gcoo_dev(path, p: int, dtype=np.float32, device="cuda", stream=None):
    """Parse a MatrixMarket file and build its GCOO on the GPU: coordinate
    files through `coo_to_gcoo_dev` (matrix.hpp:366-405 semantics), array
    files through `dense_to_gcoo_dev` (matrix.hpp:306-353).  Returns DeviceGcoo."""
    import torch

    from . import coo_to_gcoo_dev, dense_to_gcoo_dev
    got = read_matrix_market(path, dtype)
    if isinstance(got, CooMatrix):
        return coo_to_gcoo_dev(got.rows_dim, got.cols_dim, torch.from_numpy(got.values).to(device),
                               torch.from_numpy(got.row_idx).to(device), torch.from_numpy(got.col_idx).to(device),
                               p, stream=stream)
    return dense_to_gcoo_dev(torch.from_numpy(np.ascontiguousarray(got)).to(device), p, stream=stream)
