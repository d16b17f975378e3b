/*
 * gcoo_oracle.c — plain-C restatement of the reference GCOOSpDM path.
 *
 * TEST INFRASTRUCTURE ONLY (see gcoo_oracle.h).  Citations are relative to the
 * reference's proj/ directory.  Built by oracle/Makefile with
 * -ffp-contract=off so that the mul+add flavour is not silently contracted,
 * and with -mfma so that fmaf() is a single rounding instruction.
 */
#include "gcoo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG -- */
/* std::mt19937_64 (the generator io.hpp:137 and tests/common.hpp:19 use). */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = MT_N;
}

static void mt64_twist(orc_mt64* g) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
    g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
  }
  g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->idx >= MT_N) mt64_twist(g);
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* derive_seed: splitmix-style finaliser, src/bench.cpp:55-65. */
uint64_t orc_derive_seed(uint64_t base, uint64_t salt_a, uint64_t salt_b) {
  uint64_t z = base + 0x9E3779B97F4A7C15ULL * (salt_a + 1) + 0xBF58476D1CE4E5B9ULL * (salt_b + 1);
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

/* bounded_draw: rejection on the raw 64-bit stream, src/io.cpp:214-220. */
static uint64_t bounded_draw(orc_mt64* g, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = orc_mt64_next(g);
    if (x >= threshold) return x % bound;
  }
}

/* value draw: 1 - u, u = (rng() >> 11) * 2^-53  (io.hpp:141-142). */
static double unit_value(orc_mt64* g) {
  const double u = (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53;
  return 1.0 - u;
}

int64_t orc_realized_nnz(int64_t n, double s) {
  /* io.hpp:134-136: llround(total * (1 - s)) */
  return llround((double)(n * n) * (1.0 - s));
}

/*
 * generate_uniform_pattern (src/io.cpp:224-258).  The reference collects
 * distinct cell ids in an unordered_set until it holds nnz (or, on the dense
 * side, holes_wanted) ids and then emits them sorted row-major; the set's
 * iteration order never leaks because of that sort.  A bitmap over the cells
 * reproduces "the first K distinct draws" exactly.  Calls emit(cell) in
 * row-major order.
 */
typedef void (*emit_fn)(void* ctx, int64_t cell);

static int uniform_pattern(int64_t total, int64_t nnz, orc_mt64* g, emit_fn emit, void* ctx) {
  const int64_t words = (total + 63) / 64;
  uint64_t* bits = (uint64_t*)calloc((size_t)words, sizeof(uint64_t));
  if (!bits) return -1;
  const int dense_side = !(2 * nnz <= total);
  const int64_t want = dense_side ? total - nnz : nnz;
  int64_t have = 0;
  while (have < want) {
    const int64_t c = (int64_t)bounded_draw(g, (uint64_t)total);
    uint64_t* w = &bits[c >> 6];
    const uint64_t m = 1ULL << (c & 63);
    if (!(*w & m)) { *w |= m; ++have; }
  }
  for (int64_t c = 0; c < total; ++c) {
    const int set = (int)((bits[c >> 6] >> (c & 63)) & 1ULL);
    if (set != dense_side) emit(ctx, c);
  }
  free(bits);
  return 0;
}

typedef struct { orc_mt64* g; float* f; double* d; int64_t count; } dense_ctx;
static void emit_dense_f32(void* vctx, int64_t cell) {
  dense_ctx* c = (dense_ctx*)vctx;
  c->f[cell] = (float)unit_value(c->g);
  c->count++;
}
static void emit_dense_f64(void* vctx, int64_t cell) {
  dense_ctx* c = (dense_ctx*)vctx;
  c->d[cell] = unit_value(c->g);
  c->count++;
}

/* Values are drawn after the whole pattern, in row-major order (io.hpp:139-143):
 * the pattern pass consumes the stream first, then one draw per coordinate.
 * We therefore record the pattern into the output as a marker and draw values
 * in a second sweep. */
typedef struct { uint8_t* mark; } mark_ctx;
static void emit_mark(void* vctx, int64_t cell) { ((mark_ctx*)vctx)->mark[cell] = 1; }

static int64_t uniform_sparse_impl(int64_t n, double s, uint64_t seed, float* f, double* d) {
  const int64_t total = n * n;
  const int64_t nnz = orc_realized_nnz(n, s);
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  uint8_t* mark = (uint8_t*)calloc((size_t)total, 1);
  mark_ctx mc = {mark};
  uniform_pattern(total, nnz, &g, emit_mark, &mc);
  dense_ctx dc = {&g, f, d, 0};
  if (f) memset(f, 0, sizeof(float) * (size_t)total);
  if (d) memset(d, 0, sizeof(double) * (size_t)total);
  for (int64_t c = 0; c < total; ++c)
    if (mark[c]) {
      if (f) emit_dense_f32(&dc, c); else emit_dense_f64(&dc, c);
    }
  free(mark);
  return dc.count;
}

int64_t orc_uniform_sparse_f32(int64_t n, double s, uint64_t seed, float* out) {
  return uniform_sparse_impl(n, s, seed, out, NULL);
}
int64_t orc_uniform_sparse_f64(int64_t n, double s, uint64_t seed, double* out) {
  return uniform_sparse_impl(n, s, seed, NULL, out);
}

typedef struct { int64_t n, count, cap; int32_t* rows; int32_t* cols; } coo_ctx;
static void emit_coo(void* vctx, int64_t cell) {
  coo_ctx* c = (coo_ctx*)vctx;
  if (c->count < c->cap) {
    c->rows[c->count] = (int32_t)(cell / c->n);
    c->cols[c->count] = (int32_t)(cell % c->n);
  }
  c->count++;
}

int64_t orc_uniform_sparse_coo_f32(int64_t n, double s, uint64_t seed, float* vals,
                                   int32_t* rows, int32_t* cols, int64_t cap) {
  const int64_t nnz = orc_realized_nnz(n, s);
  if (nnz > cap) return -1;
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  coo_ctx cc = {n, 0, cap, rows, cols};
  uniform_pattern(n * n, nnz, &g, emit_coo, &cc);
  for (int64_t e = 0; e < nnz; ++e) vals[e] = (float)unit_value(&g);
  return nnz;
}

/* ------------------------------------------------------- power-law input -- */
/* Not in the reference.  Specification in DESIGN.md §5.      */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int64_t orc_powerlaw_coo_f32(int64_t n, double s, double alpha, uint64_t seed, float* vals,
                             int32_t* rows, int32_t* cols, int64_t cap) {
  const int64_t nnz = orc_realized_nnz(n, s);
  if (nnz > cap || nnz > n * n) return -1;
  int64_t* deg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t r = 0; r < n; ++r) w[r] = pow((double)(r + 1), -alpha);
  /* largest scale c with sum_r min(n, floor(c * w_r)) <= nnz (bisection) */
  double lo = 0.0, hi = (double)nnz / w[n - 1] + 1.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    int64_t sum = 0;
    for (int64_t r = 0; r < n; ++r) {
      double d = floor(mid * w[r]);
      sum += d >= (double)n ? n : (int64_t)d;
    }
    if (sum <= nnz) lo = mid; else hi = mid;
  }
  int64_t sum = 0;
  for (int64_t r = 0; r < n; ++r) {
    double d = floor(lo * w[r]);
    deg[r] = d >= (double)n ? n : (int64_t)d;
    sum += deg[r];
  }
  /* remainder: +1 to the lowest-rank rows that are not full, cycling */
  while (sum < nnz) {
    for (int64_t r = 0; r < n && sum < nnz; ++r)
      if (deg[r] < n) { deg[r]++; sum++; }
  }
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  /* random row permutation: Fisher-Yates from the top */
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  for (int64_t i = n - 1; i > 0; --i) {
    const int64_t j = (int64_t)bounded_draw(&g, (uint64_t)(i + 1));
    const int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  int64_t* row_deg = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  for (int64_t rk = 0; rk < n; ++rk) row_deg[perm[rk]] = deg[rk];
  uint64_t* bits = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)((n + 63) / 64));
  int64_t pos = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t d = row_deg[r];
    if (d == 0) continue;
    memset(bits, 0, sizeof(uint64_t) * (size_t)((n + 63) / 64));
    const int dense_side = !(2 * d <= n);
    const int64_t want = dense_side ? n - d : d;
    int64_t have = 0;
    while (have < want) {
      const int64_t c = (int64_t)bounded_draw(&g, (uint64_t)n);
      if (!((bits[c >> 6] >> (c & 63)) & 1ULL)) { bits[c >> 6] |= 1ULL << (c & 63); ++have; }
    }
    const int64_t start = pos;
    for (int64_t c = 0; c < n; ++c) {
      const int set = (int)((bits[c >> 6] >> (c & 63)) & 1ULL);
      if (set != dense_side) { rows[pos] = (int32_t)r; cols[pos] = (int32_t)c; ++pos; }
    }
    qsort(cols + start, (size_t)(pos - start), sizeof(int32_t), cmp_i32); /* already sorted; kept for clarity */
    for (int64_t e = start; e < pos; ++e) vals[e] = (float)unit_value(&g);
  }
  free(bits); free(row_deg); free(perm); free(w); free(deg);
  return pos;
}

/* ---------------------------------------------------------- construction -- */
static int is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

/* dense_to_gcoo, matrix.hpp:306-353: pass 1 counts per p-row band, serial
 * exclusive scan, pass 2 walks each band column-major which yields the
 * (col,row) order directly. */
#define DENSE_TO_GCOO(T)                                                              \
  if (!is_pow2(p)) return -1;                                                         \
  const int64_t g = (m + p - 1) / p;                                                  \
  for (int64_t gi = 0; gi < g; ++gi) {                                                \
    const int64_t lo = gi * p, hi = lo + p < m ? lo + p : m;                          \
    int64_t cnt = 0;                                                                  \
    for (int64_t r = lo; r < hi; ++r)                                                 \
      for (int64_t c = 0; c < k; ++c) cnt += a[r * k + c] != (T)0;                    \
    gnnz[gi] = cnt;                                                                   \
  }                                                                                   \
  int64_t total = 0;                                                                  \
  for (int64_t gi = 0; gi < g; ++gi) { g_idxes[gi] = total; total += gnnz[gi]; }      \
  for (int64_t gi = 0; gi < g; ++gi) {                                                \
    const int64_t lo = gi * p, hi = lo + p < m ? lo + p : m;                          \
    int64_t w = g_idxes[gi];                                                          \
    for (int64_t c = 0; c < k; ++c)                                                   \
      for (int64_t r = lo; r < hi; ++r)                                               \
        if (a[r * k + c] != (T)0) {                                                   \
          vals[w] = a[r * k + c]; rows[w] = (int32_t)r; cols[w] = (int32_t)c; ++w;    \
        }                                                                             \
  }                                                                                   \
  return total;

int64_t orc_dense_to_gcoo_f32(int64_t m, int64_t k, const float* a, int32_t p, float* vals,
                              int32_t* rows, int32_t* cols, int64_t* g_idxes, int64_t* gnnz) {
  DENSE_TO_GCOO(float)
}
int64_t orc_dense_to_gcoo_f64(int64_t m, int64_t k, const double* a, int32_t p, double* vals,
                              int32_t* rows, int32_t* cols, int64_t* g_idxes, int64_t* gnnz) {
  DENSE_TO_GCOO(double)
}

/* coo_to_gcoo, matrix.hpp:366-405.  The reference validates (CooMatrix::validate,
 * :95-115), histograms rows/p, scans, and sorts each group's slice by (col,row).
 * Because (col,row) keys are unique inside a group any correct sort gives the
 * same arrays; we use an insertion of each group's indices sorted by qsort on
 * an explicit key. */
typedef struct { int64_t key; int64_t idx; } kv;
static int cmp_kv(const void* a, const void* b) {
  const int64_t x = ((const kv*)a)->key, y = ((const kv*)b)->key;
  return (x > y) - (x < y);
}

int orc_coo_to_gcoo_f32(int64_t m, int64_t k, int64_t nnz, const float* vals, const int32_t* rows,
                        const int32_t* cols, int32_t p, float* ovals, int32_t* orows,
                        int32_t* ocols, int64_t* g_idxes, int64_t* gnnz, int64_t* bad_index) {
  /* validate first (matrix.hpp:368 -> :95-115), then the p check (:369-370) */
  for (int64_t i = 0; i < nnz; ++i) {
    if (rows[i] < 0 || rows[i] >= m || cols[i] < 0 || cols[i] >= k) { *bad_index = i; return -2; }
    if (i > 0) {
      const int ok = rows[i - 1] < rows[i] || (rows[i - 1] == rows[i] && cols[i - 1] < cols[i]);
      if (!ok) { *bad_index = i; return -2; }
    }
  }
  if (!is_pow2(p)) return -1;
  const int64_t g = (m + p - 1) / p;
  memset(gnnz, 0, sizeof(int64_t) * (size_t)g);
  for (int64_t e = 0; e < nnz; ++e) gnnz[rows[e] / p]++;
  int64_t total = 0;
  for (int64_t gi = 0; gi < g; ++gi) { g_idxes[gi] = total; total += gnnz[gi]; }
  kv* buf = (kv*)malloc(sizeof(kv) * (size_t)(nnz > 0 ? nnz : 1));
  for (int64_t gi = 0; gi < g; ++gi) {
    const int64_t lo = g_idxes[gi], cnt = gnnz[gi];
    for (int64_t i = 0; i < cnt; ++i) {
      buf[i].key = (int64_t)cols[lo + i] * (int64_t)(m + 1) + rows[lo + i];
      buf[i].idx = lo + i;
    }
    qsort(buf, (size_t)cnt, sizeof(kv), cmp_kv);
    for (int64_t i = 0; i < cnt; ++i) {
      ovals[lo + i] = vals[buf[i].idx];
      orows[lo + i] = rows[buf[i].idx];
      ocols[lo + i] = cols[buf[i].idx];
    }
  }
  free(buf);
  return 0;
}

/* GcooMatrix::validate, matrix.hpp:206-244. */
int orc_gcoo_validate(int64_t m, int64_t k, int32_t p, int64_t nnz, const int32_t* rows,
                      const int32_t* cols, int64_t groups, const int64_t* g_idxes,
                      const int64_t* gnnz) {
  if (m < 1 || k < 1) return 1;
  if (!is_pow2(p)) return 2;
  if (groups != (m + p - 1) / p) return 3;
  int64_t off = 0;
  for (int64_t gi = 0; gi < groups; ++gi) {
    if (g_idxes[gi] != off) return 4;
    if (gnnz[gi] < 0) return 5;
    const int64_t lo = gi * p, hi = lo + p < m ? lo + p : m;
    for (int64_t e = off; e < off + gnnz[gi]; ++e) {
      if (e >= nnz) return 8;
      if (rows[e] < lo || rows[e] >= hi) return 6;
      if (cols[e] < 0 || cols[e] >= k) return 7;
      if (e > off) {
        const int ok = cols[e - 1] < cols[e] || (cols[e - 1] == cols[e] && rows[e - 1] < rows[e]);
        if (!ok) return 9;
      }
    }
    off += gnnz[gi];
  }
  return off == nnz ? 0 : 10;
}

/* ------------------------------------------------------------ GCOOSpDM -- */
/*
 * detail::spdm_gcoo_impl, kernels.hpp:240-327.  One work item per (group,
 * column strip of width b); the group's slice is streamed through a staging
 * window of at most b entries (:283-290); inside a window, maximal same-column
 * runs share one B row segment (:292-308); every entry accumulates
 * av * B(col, j0:j0+w) into its row's slot (row & (p-1)) (:301-306); the tile
 * is written once (:314-318).  Per C element this is a sequential chain over
 * the row's nonzeros in ascending column order.
 */
#define SPDM_TILE(T, FMA_EXPR)                                                                \
  const int64_t col_tiles = (n + b - 1) / b;                                                  \
  const int64_t groups = (m + p - 1) / p;                                                     \
  uint64_t fl = 0, tot = 0, reu = 0, fills = 0;                                               \
  T* acc = (T*)malloc(sizeof(T) * (size_t)p * (size_t)b);                                     \
  for (int64_t gi = g_begin; gi < g_end; ++gi) {                                              \
    for (int64_t sj = 0; sj < col_tiles; ++sj) {                                              \
      const int64_t i0 = gi * p, j0 = sj * b;                                                 \
      const int64_t h = p < m - i0 ? p : m - i0, w = b < n - j0 ? b : n - j0;                 \
      const int64_t lo = g_idxes[gi], cnt = gnnz[gi];                                         \
      for (int64_t q = 0; q < (int64_t)p * b; ++q) acc[q] = (T)0;                             \
      for (int64_t chunk = 0; chunk < cnt; chunk += b) {                                      \
        const int64_t cs = b < cnt - chunk ? b : cnt - chunk;                                 \
        fills += (uint64_t)cs;                                                                \
        int64_t e = 0;                                                                        \
        while (e < cs) {                                                                      \
          const int32_t col = cols[lo + chunk + e];                                           \
          int64_t run = 1;                                                                    \
          while (e + run < cs && cols[lo + chunk + e + run] == col) ++run;                    \
          const T* bv = B + (int64_t)col * n + j0;                                            \
          tot += (uint64_t)w;                                                                 \
          reu += (uint64_t)(run - 1) * (uint64_t)w;                                           \
          for (int64_t q = 0; q < run; ++q) {                                                 \
            const T av = vals[lo + chunk + e + q];                                            \
            T* arow = acc + ((int64_t)rows[lo + chunk + e + q] & (p - 1)) * b;                \
            for (int64_t j = 0; j < w; ++j) arow[j] = FMA_EXPR;                               \
          }                                                                                   \
          e += run;                                                                           \
        }                                                                                     \
      }                                                                                       \
      fl += 2ULL * (uint64_t)cnt * (uint64_t)w;                                               \
      for (int64_t i = 0; i < h; ++i) {                                                       \
        if (i0 + i < r_begin || i0 + i >= r_end) continue;                                    \
        memcpy(C + (i0 + i) * n + j0, acc + i * b, sizeof(T) * (size_t)w);                    \
      }                                                                                       \
    }                                                                                         \
  }                                                                                           \
  free(acc);                                                                                  \
  (void)groups;                                                                               \
  if (st) { st->flops = fl; st->b_loads_total = tot; st->b_loads_reused = reu;                \
            st->staging_fills = fills; }

static void spdm_f32_fma(int64_t m, int64_t n, int32_t p, int32_t b, const float* vals,
                         const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                         const int64_t* gnnz, const float* B, float* C, orc_stats* st,
                         int64_t g_begin, int64_t g_end, int64_t r_begin, int64_t r_end) {
  SPDM_TILE(float, fmaf(av, bv[j], arow[j]))
}
static void spdm_f32_mad(int64_t m, int64_t n, int32_t p, int32_t b, const float* vals,
                         const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                         const int64_t* gnnz, const float* B, float* C, orc_stats* st,
                         int64_t g_begin, int64_t g_end, int64_t r_begin, int64_t r_end) {
  SPDM_TILE(float, arow[j] + av * bv[j])
}
static void spdm_f64_fma(int64_t m, int64_t n, int32_t p, int32_t b, const double* vals,
                         const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                         const int64_t* gnnz, const double* B, double* C, orc_stats* st,
                         int64_t g_begin, int64_t g_end, int64_t r_begin, int64_t r_end) {
  SPDM_TILE(double, fma(av, bv[j], arow[j]))
}
static void spdm_f64_mad(int64_t m, int64_t n, int32_t p, int32_t b, const double* vals,
                         const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                         const int64_t* gnnz, const double* B, double* C, orc_stats* st,
                         int64_t g_begin, int64_t g_end, int64_t r_begin, int64_t r_end) {
  SPDM_TILE(double, arow[j] + av * bv[j])
}

void orc_spdm_gcoo_f32(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, const float* vals,
                       const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                       const int64_t* gnnz, const float* B, float* C, orc_stats* st, int fma) {
  (void)k;
  const int64_t g = (m + p - 1) / p;
  if (fma) spdm_f32_fma(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, st, 0, g, 0, m);
  else spdm_f32_mad(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, st, 0, g, 0, m);
}

void orc_spdm_gcoo_f64(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, const double* vals,
                       const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                       const int64_t* gnnz, const double* B, double* C, orc_stats* st, int fma) {
  (void)k;
  const int64_t g = (m + p - 1) / p;
  if (fma) spdm_f64_fma(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, st, 0, g, 0, m);
  else spdm_f64_mad(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, st, 0, g, 0, m);
}

void orc_spdm_gcoo_rows_f32(int64_t m, int64_t n, int32_t p, int32_t b, const float* vals,
                            const int32_t* rows, const int32_t* cols, const int64_t* g_idxes,
                            const int64_t* gnnz, const float* B, float* C, int64_t r0, int64_t r1,
                            int fma) {
  const int64_t g0 = r0 / p, g1 = (r1 + p - 1) / p;
  if (fma) spdm_f32_fma(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, NULL, g0, g1, r0, r1);
  else spdm_f32_mad(m, n, p, b, vals, rows, cols, g_idxes, gnnz, B, C, NULL, g0, g1, r0, r1);
}

/* Counters only: kernels.hpp:290 (staging), :298-300 (runs), :310 (flops). */
void orc_gcoo_stats(int64_t n, int32_t b, int64_t groups, const int32_t* cols,
                    const int64_t* g_idxes, const int64_t* gnnz, orc_stats* st) {
  const int64_t col_tiles = (n + b - 1) / b;
  uint64_t runs = 0, nnz = 0;
  for (int64_t gi = 0; gi < groups; ++gi) {
    const int64_t lo = g_idxes[gi], cnt = gnnz[gi];
    for (int64_t e = 0; e < cnt; ++e)
      if (e % b == 0 || cols[lo + e] != cols[lo + e - 1]) ++runs;
    nnz += (uint64_t)cnt;
  }
  st->flops = 2ULL * nnz * (uint64_t)n;
  st->staging_fills = nnz * (uint64_t)col_tiles;
  st->b_loads_total = runs * (uint64_t)n;
  st->b_loads_reused = (nnz - runs) * (uint64_t)n;
}

/* ------------------------------------------------- comparison kernels --
 * The reference's baselines (kernels.hpp:107-232) restated: every C element is
 * the chain over its terms in the reference's order, one rounding per step
 * (fma) or two (mul+add), starting from +0.
 *   spdm_csr   (:163-184): row r's entries in CSR order;
 *   spdm_coo   (:193-232): row r's entries in COO array order (the reference
 *              walks column strips, then b-entry chunks of the stream, then the
 *              chunk's entries: per element that is array order);
 *   gemm_dense (:107-155): l ascending (its kb depth blocks run in order). */
#define ORC_MAC(T, FMA, acc, a, b) ((FMA) ? ORC_FMA_##T((a), (b), (acc)) : (acc) + (T)((a) * (b)))
#define ORC_FMA_float(a, b, c) fmaf((a), (b), (c))
#define ORC_FMA_double(a, b, c) fma((a), (b), (c))

#define ORC_BASELINES(T, SFX)                                                                                 \
  void orc_spdm_csr_##SFX(int64_t m, int64_t n, const T* vals, const int32_t* cols, const int64_t* rp,      \
                          const T* B, T* C, int fma_flavour) {                                             \
    for (int64_t r = 0; r < m; ++r) {                                                                     \
      T* crow = C + r * n;                                                                                \
      for (int64_t j = 0; j < n; ++j) crow[j] = (T)0;                                                     \
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {                                                       \
        const T a = vals[e];                                                                              \
        const T* brow = B + (int64_t)cols[e] * n;                                                         \
        for (int64_t j = 0; j < n; ++j) crow[j] = ORC_MAC(T, fma_flavour, crow[j], a, brow[j]);           \
      }                                                                                                   \
    }                                                                                                     \
  }                                                                                                       \
  void orc_spdm_coo_##SFX(int64_t m, int64_t n, int64_t nnz, const T* vals, const int32_t* rows,           \
                          const int32_t* cols, const T* B, T* C, int fma_flavour) {                        \
    for (int64_t i = 0; i < m * n; ++i) C[i] = (T)0;                                                      \
    for (int64_t e = 0; e < nnz; ++e) {                                                                   \
      const T a = vals[e];                                                                                \
      const T* brow = B + (int64_t)cols[e] * n;                                                           \
      T* crow = C + (int64_t)rows[e] * n;                                                                 \
      for (int64_t j = 0; j < n; ++j) crow[j] = ORC_MAC(T, fma_flavour, crow[j], a, brow[j]);             \
    }                                                                                                     \
  }                                                                                                       \
  void orc_gemm_dense_##SFX(int64_t m, int64_t k, int64_t n, const T* A, const T* B, T* C, int fma_flavour) { \
    for (int64_t i = 0; i < m; ++i) {                                                                     \
      T* crow = C + i * n;                                                                                \
      for (int64_t j = 0; j < n; ++j) crow[j] = (T)0;                                                     \
      for (int64_t l = 0; l < k; ++l) {                                                                   \
        const T a = A[i * k + l];                                                                         \
        const T* brow = B + l * n;                                                                        \
        for (int64_t j = 0; j < n; ++j) crow[j] = ORC_MAC(T, fma_flavour, crow[j], a, brow[j]);           \
      }                                                                                                   \
    }                                                                                                     \
  }
ORC_BASELINES(float, f32)
ORC_BASELINES(double, f64)

uint32_t orc_fnv1a32(const void* data, int64_t nbytes) {
  const uint8_t* q = (const uint8_t*)data;
  uint32_t h = 2166136261u;
  for (int64_t i = 0; i < nbytes; ++i) { h ^= q[i]; h *= 16777619u; }
  return h;
}
