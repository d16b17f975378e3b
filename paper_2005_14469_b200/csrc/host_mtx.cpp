// host_mtx.cpp — MatrixMarket entry-section tokenizer (the I/O in front of the
// path; not the hot path).
//
// The reference reads entries one line at a time through istringstream
// (io.cpp:109-158).  Here the text after the size line is split into
// newline-aligned chunks parsed by all host threads: pass 1 counts data lines
// per chunk, pass 2 parses each chunk into its slice of the output.  Values go
// through strtod, which is what libstdc++'s num_get<double> calls, so every
// value is bit-identical to the reference's.  Anything irregular (wrong token
// count, a non-integer index, a non-decimal or overflowing value) makes the
// call return GCOO_MTX_IRREGULAR; the caller (paper_2005_14469_b200/mmio.py)
// then re-reads the file line by line to report the reference's exact
// ParseError.  Range, symmetry, ordering and duplicate checks stay with the
// caller, which has the numbers in arrays.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gcoo_capi.h"

namespace {

inline bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// One integer token: [+-]?[0-9]+, at most 18 digits (anything longer is out
// of every index range and is left to the line parser).
inline bool parse_index(const char* b, const char* e, int64_t* out) {
  bool neg = false;
  if (b < e && (*b == '+' || *b == '-')) neg = (*b++ == '-');
  if (b == e || e - b > 18) return false;
  int64_t v = 0;
  for (; b < e; ++b) {
    if (*b < '0' || *b > '9') return false;
    v = v * 10 + (*b - '0');
  }
  *out = neg ? -v : v;
  return true;
}

// One value token: characters of a plain decimal only (num_get rejects inf,
// nan and hex floats), fully consumed by strtod, not overflowing (num_get sets
// failbit on ERANGE overflow; underflow to a subnormal or zero is accepted).
inline bool parse_value(const char* b, const char* e, double* out) {
  char buf[96];
  const size_t n = static_cast<size_t>(e - b);
  std::string big;
  const char* s;
  if (n < sizeof buf) {
    std::memcpy(buf, b, n);
    buf[n] = 0;
    s = buf;
  } else {
    big.assign(b, n);
    s = big.c_str();
  }
  for (size_t i = 0; i < n; ++i) {
    const char c = s[i];
    if (!((c >= '0' && c <= '9') || c == '+' || c == '-' || c == '.' || c == 'e' || c == 'E')) return false;
  }
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(s, &end);
  if (end != s + n) return false;
  if (errno == ERANGE && std::isinf(v)) return false;
  *out = v;
  return true;
}

struct Chunk {
  const char* b;
  const char* e;
  int64_t lines = 0;      // physical lines starting in the chunk
  int64_t data = 0;       // of which data lines
  bool irregular = false;
};

// Walks the lines of [b, e); for every data line calls fn(line_index_in_chunk, tokens...).
template <typename Fn>
bool for_lines(const char* b, const char* e, Fn&& fn) {
  int64_t line = 0;
  while (b < e) {
    const char* nl = static_cast<const char*>(std::memchr(b, '\n', static_cast<size_t>(e - b)));
    const char* le = nl ? nl : e;
    const char* p = b;
    while (p < le && is_ws(*p)) ++p;
    if (p < le && *p != '%')
      if (!fn(line, p, le)) return false;
    ++line;
    b = nl ? nl + 1 : e;
  }
  return true;
}

// Splits [p, le) into up to `want` tokens; false unless exactly `want`.
inline bool tokens(const char* p, const char* le, int want, const char** tb, const char** te) {
  int n = 0;
  while (p < le) {
    while (p < le && is_ws(*p)) ++p;
    if (p == le) break;
    if (n == want) return false;
    tb[n] = p;
    while (p < le && !is_ws(*p)) ++p;
    te[n++] = p;
  }
  return n == want;
}

}  // namespace

extern "C" int64_t gcoo_mtx_parse_entries(const char* text, int64_t len, int32_t ncol, int64_t cap,
                                          int64_t* idx, double* vals, int64_t* line_of, int32_t threads) {
  if (len < 0 || ncol < 1 || ncol > 3 || cap < 0) return GCOO_MTX_IRREGULAR;
  const char* end = text + len;
  int nt = threads;                   // > 0: exactly that many chunks (tests); else ~1 MiB per thread
  if (nt <= 0)
    nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()),
                                   static_cast<int>(len / (1 << 20)) + 1));
  std::vector<Chunk> ch(static_cast<size_t>(nt));
  const char* cur = text;
  for (int t = 0; t < nt; ++t) {
    const char* e = (t == nt - 1) ? end : text + len / nt * (t + 1);
    if (e < cur) e = cur;
    if (t < nt - 1 && e < end) {      // extend to the end of the line
      const char* nl = static_cast<const char*>(std::memchr(e, '\n', static_cast<size_t>(end - e)));
      e = nl ? nl + 1 : end;
    }
    ch[t].b = cur;
    ch[t].e = e;
    cur = e;
  }
  const int nidx = ncol == 1 ? 0 : 2;
  const bool has_val = ncol != 2;
  auto run = [&](auto&& per_chunk) {
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(per_chunk, t);
    per_chunk(0);
    for (auto& th : pool) th.join();
  };
  // pass 1: line and data-line counts per chunk
  run([&](int t) {
    Chunk& c = ch[static_cast<size_t>(t)];
    const char* b = c.b;
    while (b < c.e) {
      const char* nl = static_cast<const char*>(std::memchr(b, '\n', static_cast<size_t>(c.e - b)));
      const char* le = nl ? nl : c.e;
      const char* p = b;
      while (p < le && is_ws(*p)) ++p;
      if (p < le && *p != '%') ++c.data;
      ++c.lines;
      b = nl ? nl + 1 : c.e;
    }
  });
  std::vector<int64_t> line0(static_cast<size_t>(nt)), row0(static_cast<size_t>(nt));
  int64_t lines = 0, rows = 0;
  for (int t = 0; t < nt; ++t) {
    line0[t] = lines;
    row0[t] = rows;
    lines += ch[t].lines;
    rows += ch[t].data;
  }
  // pass 2: parse each chunk into its slice
  run([&](int t) {
    Chunk& c = ch[static_cast<size_t>(t)];
    int64_t r = row0[t];
    c.irregular = !for_lines(c.b, c.e, [&](int64_t line, const char* p, const char* le) {
      const char* tb[3];
      const char* te[3];
      if (!tokens(p, le, ncol, tb, te)) return false;
      int64_t ij[2] = {0, 0};
      double v = 1.0;
      for (int q = 0; q < nidx; ++q)
        if (!parse_index(tb[q], te[q], &ij[q])) return false;
      if (has_val && !parse_value(tb[ncol - 1], te[ncol - 1], &v)) return false;
      if (r < cap) {
        if (idx && nidx) idx[2 * r] = ij[0], idx[2 * r + 1] = ij[1];
        if (vals) vals[r] = v;
        if (line_of) line_of[r] = line0[t] + line;
      }
      ++r;
      return true;
    });
  });
  for (const Chunk& c : ch)
    if (c.irregular) return GCOO_MTX_IRREGULAR;
  return rows;
}
