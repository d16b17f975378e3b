// host_gen.cpp — synthetic benchmark inputs (harness, not the hot path).
//
// generate_uniform_sparse (io.hpp:129-145; io.cpp:224-258) and derive_seed
// (bench.cpp:55-65) reproduce the reference's inputs bit-for-bit, so the GPU
// arm and the reference CPU arm multiply the same matrices.  The sample is a
// single sequential std::mt19937_64 stream, which is why this stays on the
// host.  The power-law generator is this repository's own.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "gcoo_capi.h"

namespace {

thread_local std::string t_gen_error;

uint64_t bounded(std::mt19937_64& g, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;  // rejection: no modulo bias
  for (;;) {
    const uint64_t x = g();
    if (x >= threshold) return x % bound;
  }
}

double one_minus_u(std::mt19937_64& g) {
  return 1.0 - static_cast<double>(g() >> 11) * 0x1.0p-53;
}

int64_t target_nnz(int64_t n, double s) {
  return std::llround(static_cast<double>(n * n) * (1.0 - s));
}

// Bit set of the chosen cells: the first `want` distinct draws from [0,total)
// (the reference's unordered_set holds exactly these before it sorts).
std::vector<uint64_t> draw_cells(std::mt19937_64& g, int64_t total, int64_t want) {
  std::vector<uint64_t> bits(static_cast<size_t>((total + 63) / 64), 0);
  int64_t have = 0;
  while (have < want) {
    const uint64_t c = bounded(g, static_cast<uint64_t>(total));
    uint64_t& w = bits[c >> 6];
    const uint64_t mask = 1ull << (c & 63);
    if (!(w & mask)) {
      w |= mask;
      ++have;
    }
  }
  return bits;
}

inline bool bit(const std::vector<uint64_t>& b, int64_t c) { return (b[c >> 6] >> (c & 63)) & 1ull; }

void check_args(int64_t n, double s) {
  if (n < 1) throw std::invalid_argument("generate_uniform_sparse: n must be >= 1");
  if (!(s >= 0.0 && s <= 1.0)) throw std::invalid_argument("generate_uniform_sparse: sparsity outside [0,1]");
}

// Visit the sampled pattern row-major; a dense-side sample is drawn as holes.
template <typename Emit>
void uniform_pattern(std::mt19937_64& g, int64_t total, int64_t nnz, Emit&& emit) {
  const bool holes = !(2 * nnz <= total);
  const auto bits = draw_cells(g, total, holes ? total - nnz : nnz);
  for (int64_t c = 0; c < total; ++c)
    if (bit(bits, c) != holes) emit(c);
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return GCOO_OK;
  } catch (const std::invalid_argument& e) {
    t_gen_error = e.what();
    return GCOO_EINVAL;
  } catch (const std::bad_alloc&) {
    return GCOO_ENOMEM;
  } catch (const std::exception& e) {
    t_gen_error = e.what();
    return GCOO_ECUDA;
  }
}

}  // namespace

extern "C" {

uint64_t gcoo_derive_seed(uint64_t base, uint64_t salt_a, uint64_t salt_b) {
  uint64_t z = base + 0x9E3779B97F4A7C15ULL * (salt_a + 1) + 0xBF58476D1CE4E5B9ULL * (salt_b + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int gcoo_generate_uniform_sparse_f32(int64_t n, double s, uint64_t seed, float* out) {
  return guarded([&] {
    check_args(n, s);
    const int64_t total = n * n;
    std::memset(out, 0, sizeof(float) * static_cast<size_t>(total));
    std::mt19937_64 g(seed);
    std::vector<int64_t> cells;
    cells.reserve(static_cast<size_t>(target_nnz(n, s)));
    uniform_pattern(g, total, target_nnz(n, s), [&](int64_t c) { cells.push_back(c); });
    for (int64_t c : cells) out[c] = static_cast<float>(one_minus_u(g));
  });
}

int gcoo_generate_uniform_sparse_coo_f32(int64_t n, double s, uint64_t seed, int64_t capacity, float* values,
                                         int32_t* row_idx, int32_t* col_idx, int64_t* nnz) {
  return guarded([&] {
    check_args(n, s);
    const int64_t want = target_nnz(n, s);
    *nnz = want;
    if (!values) return;
    if (capacity < want) throw std::invalid_argument("generate_uniform_sparse: capacity < nnz");
    std::mt19937_64 g(seed);
    int64_t e = 0;
    uniform_pattern(g, n * n, want, [&](int64_t c) {
      row_idx[e] = static_cast<int32_t>(c / n);
      col_idx[e] = static_cast<int32_t>(c % n);
      ++e;
    });
    for (int64_t i = 0; i < want; ++i) values[i] = static_cast<float>(one_minus_u(g));
  });
}

// Power-law rows: degree of rank r ~ (r+1)^-alpha scaled to exactly nnz
// (capped at n, remainder +1 to the lowest ranks that are not full), ranks
// mapped to rows by a Fisher-Yates permutation, columns uniform without
// replacement per row, values 1-u in row-major order.
int gcoo_generate_powerlaw_coo_f32(int64_t n, double s, double alpha, uint64_t seed, int64_t capacity,
                                   float* values, int32_t* row_idx, int32_t* col_idx, int64_t* nnz) {
  return guarded([&] {
    check_args(n, s);
    const int64_t want = target_nnz(n, s);
    *nnz = want;
    if (!values) return;
    if (capacity < want) throw std::invalid_argument("powerlaw: capacity < nnz");
    std::vector<double> w(static_cast<size_t>(n));
    for (int64_t r = 0; r < n; ++r) w[r] = std::pow(static_cast<double>(r + 1), -alpha);
    auto degree_sum = [&](double scale) {
      int64_t sum = 0;
      for (int64_t r = 0; r < n; ++r) {
        const double d = std::floor(scale * w[r]);
        sum += d >= static_cast<double>(n) ? n : static_cast<int64_t>(d);
      }
      return sum;
    };
    double lo = 0.0, hi = static_cast<double>(want) / w[n - 1] + 1.0;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (degree_sum(mid) <= want) lo = mid; else hi = mid;
    }
    std::vector<int64_t> deg(static_cast<size_t>(n));
    int64_t sum = 0;
    for (int64_t r = 0; r < n; ++r) {
      const double d = std::floor(lo * w[r]);
      deg[r] = d >= static_cast<double>(n) ? n : static_cast<int64_t>(d);
      sum += deg[r];
    }
    while (sum < want)
      for (int64_t r = 0; r < n && sum < want; ++r)
        if (deg[r] < n) { ++deg[r]; ++sum; }
    std::mt19937_64 g(seed);
    std::vector<int64_t> perm(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t i = n - 1; i > 0; --i) std::swap(perm[i], perm[bounded(g, static_cast<uint64_t>(i + 1))]);
    std::vector<int64_t> row_deg(static_cast<size_t>(n));
    for (int64_t rk = 0; rk < n; ++rk) row_deg[perm[rk]] = deg[rk];
    int64_t e = 0;
    for (int64_t r = 0; r < n; ++r) {
      const int64_t d = row_deg[r];
      if (!d) continue;
      const int64_t start = e;
      uniform_pattern(g, n, d, [&](int64_t c) {
        row_idx[e] = static_cast<int32_t>(r);
        col_idx[e] = static_cast<int32_t>(c);
        ++e;
      });
      for (int64_t i = start; i < e; ++i) values[i] = static_cast<float>(one_minus_u(g));
    }
  });
}

}  // extern "C"
