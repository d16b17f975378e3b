// ref_shim.cpp — C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile directly against the
// reference headers and sources under /root/reference/proj (never copied into
// this repository) into oracle/_ref/libgcoo_ref{,_fma}.so.  It lets the tests
// pin oracle/gcoo_oracle.c against the real reference and lets bench.py time
// the reference's own CPU implementation (`--impl reference`,
// cpu_baseline.kind = "reference").
//
// Two numeric flavours are built from the same file:
//   libgcoo_ref.so      default x86-64 ISA (as shipped): mul+add chain
//   libgcoo_ref_fma.so  -mfma: GCC contracts kernels.hpp:305 into FMA
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "gcoo/bench.hpp"
#include "gcoo/io.hpp"
#include "gcoo/kernels.hpp"
#include "gcoo/matrix.hpp"
#include "gcoo/traffic.hpp"

using namespace gcoo;

namespace {
thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

template <typename T>
GcooMatrix<T> make_gcoo(int64_t m, int64_t k, int32_t p, int64_t nnz, const T* vals,
                        const int32_t* rows, const int32_t* cols, int64_t groups,
                        const int64_t* gidx, const int64_t* gnnz) {
  return GcooMatrix<T>(m, k, p, std::vector<T>(vals, vals + nnz),
                       std::vector<index_t>(rows, rows + nnz),
                       std::vector<index_t>(cols, cols + nnz),
                       std::vector<int64_t>(gidx, gidx + groups),
                       std::vector<int64_t>(gnnz, gnnz + groups));
}

template <typename T>
DenseMatrix<T> make_dense(int64_t r, int64_t c, const T* data) {
  DenseMatrix<T> d(r, c);
  std::memcpy(d.data.data(), data, sizeof(T) * static_cast<size_t>(r * c));
  return d;
}

template <typename T>
void copy_gcoo(const GcooMatrix<T>& g, T* vals, int32_t* rows, int32_t* cols, int64_t* gidx,
               int64_t* gnnz) {
  std::memcpy(vals, g.values.data(), sizeof(T) * g.values.size());
  std::memcpy(rows, g.row_idx.data(), sizeof(int32_t) * g.row_idx.size());
  std::memcpy(cols, g.col_idx.data(), sizeof(int32_t) * g.col_idx.size());
  std::memcpy(gidx, g.g_idxes.data(), sizeof(int64_t) * g.g_idxes.size());
  std::memcpy(gnnz, g.nnz_per_group.data(), sizeof(int64_t) * g.nnz_per_group.size());
}

template <typename T>
int spdm(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz, const T* vals,
         const int32_t* rows, const int32_t* cols, int64_t groups, const int64_t* gidx,
         const int64_t* gnnz, const T* B, T* C, uint64_t* stats, int workers,
         const int64_t* tile_order, int64_t tile_count) {
  return guarded([&] {
    const auto a = make_gcoo<T>(m, k, p, nnz, vals, rows, cols, groups, gidx, gnnz);
    const auto bm = make_dense<T>(k, n, B);
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    cfg.workers = workers;
    KernelStats st;
    DenseMatrix<T> c = tile_order
        ? spdm_gcoo(a, bm, cfg, std::span<const int64_t>(tile_order, tile_count), &st)
        : spdm_gcoo(a, bm, cfg, &st);
    std::memcpy(C, c.data.data(), sizeof(T) * c.data.size());
    if (stats) {
      stats[0] = st.flops;
      stats[1] = st.b_loads_total;
      stats[2] = st.b_loads_reused;
      stats[3] = st.staging_fills;
    }
  });
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t base, uint64_t a, uint64_t b) { return derive_seed(base, a, b); }

// generate_uniform_sparse<T>(n, s, seed) -> dense n*n
int ref_uniform_sparse_f32(int64_t n, double s, uint64_t seed, float* out) {
  return guarded([&] {
    const auto d = generate_uniform_sparse<float>(n, s, seed);
    std::memcpy(out, d.data.data(), sizeof(float) * d.data.size());
  });
}
int ref_uniform_sparse_f64(int64_t n, double s, uint64_t seed, double* out) {
  return guarded([&] {
    const auto d = generate_uniform_sparse<double>(n, s, seed);
    std::memcpy(out, d.data.data(), sizeof(double) * d.data.size());
  });
}

// dense_to_gcoo: two calls — size query (vals == nullptr) then fill.
int64_t ref_dense_to_gcoo_f32(int64_t m, int64_t k, const float* a, int32_t p, float* vals,
                              int32_t* rows, int32_t* cols, int64_t* gidx, int64_t* gnnz) {
  int64_t nnz = -1;
  const int rc = guarded([&] {
    const auto g = dense_to_gcoo(make_dense<float>(m, k, a), p);
    nnz = g.nnz();
    if (vals) copy_gcoo(g, vals, rows, cols, gidx, gnnz);
  });
  return rc ? -1 : nnz;
}
int64_t ref_dense_to_gcoo_f64(int64_t m, int64_t k, const double* a, int32_t p, double* vals,
                              int32_t* rows, int32_t* cols, int64_t* gidx, int64_t* gnnz) {
  int64_t nnz = -1;
  const int rc = guarded([&] {
    const auto g = dense_to_gcoo(make_dense<double>(m, k, a), p);
    nnz = g.nnz();
    if (vals) copy_gcoo(g, vals, rows, cols, gidx, gnnz);
  });
  return rc ? -1 : nnz;
}

int ref_coo_to_gcoo_f32(int64_t m, int64_t k, int64_t nnz, const float* vals, const int32_t* rows,
                        const int32_t* cols, int32_t p, float* ovals, int32_t* orows,
                        int32_t* ocols, int64_t* gidx, int64_t* gnnz) {
  return guarded([&] {
    CooMatrix<float> coo;
    coo.rows_dim = m;
    coo.cols_dim = k;
    coo.values.assign(vals, vals + nnz);
    coo.row_idx.assign(rows, rows + nnz);
    coo.col_idx.assign(cols, cols + nnz);
    const auto g = coo_to_gcoo(coo, p);
    copy_gcoo(g, ovals, orows, ocols, gidx, gnnz);
  });
}

int ref_spdm_gcoo_f32(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                      const float* vals, const int32_t* rows, const int32_t* cols, int64_t groups,
                      const int64_t* gidx, const int64_t* gnnz, const float* B, float* C,
                      uint64_t* stats, int workers, const int64_t* tile_order,
                      int64_t tile_count) {
  return spdm<float>(m, k, n, p, b, nnz, vals, rows, cols, groups, gidx, gnnz, B, C, stats,
                     workers, tile_order, tile_count);
}
int ref_spdm_gcoo_f64(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                      const double* vals, const int32_t* rows, const int32_t* cols,
                      int64_t groups, const int64_t* gidx, const int64_t* gnnz, const double* B,
                      double* C, uint64_t* stats, int workers, const int64_t* tile_order,
                      int64_t tile_count) {
  return spdm<double>(m, k, n, p, b, nnz, vals, rows, cols, groups, gidx, gnnz, B, C, stats,
                      workers, tile_order, tile_count);
}

// The reference's comparison kernels (kernels.hpp:107-232), unvalidated as
// there: spdm_csr over a CSR, spdm_coo over a COO in any entry order,
// gemm_dense_blocked.  cfg = {p, b, workers}.
}  // extern "C"
namespace {
template <typename T>
int ref_csr(int64_t m, int64_t k, int64_t n, int64_t nnz, const T* vals, const int32_t* cols, const int64_t* rp,
            const T* B, T* C, int32_t p, int32_t b, int workers) {
  return guarded([&] {
    CsrMatrix<T> a;
    a.rows_dim = m;
    a.cols_dim = k;
    a.values.assign(vals, vals + nnz);
    a.col_idx.assign(cols, cols + nnz);
    a.row_ptr.assign(rp, rp + m + 1);
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    cfg.workers = workers;
    const auto c = spdm_csr(a, make_dense<T>(k, n, B), cfg);
    std::memcpy(C, c.data.data(), sizeof(T) * c.data.size());
  });
}
template <typename T>
int ref_coo(int64_t m, int64_t k, int64_t n, int64_t nnz, const T* vals, const int32_t* rows, const int32_t* cols,
            const T* B, T* C, int32_t p, int32_t b, int workers) {
  return guarded([&] {
    CooMatrix<T> a;
    a.rows_dim = m;
    a.cols_dim = k;
    a.values.assign(vals, vals + nnz);
    a.row_idx.assign(rows, rows + nnz);
    a.col_idx.assign(cols, cols + nnz);
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    cfg.workers = workers;
    const auto c = spdm_coo(a, make_dense<T>(k, n, B), cfg);
    std::memcpy(C, c.data.data(), sizeof(T) * c.data.size());
  });
}
template <typename T>
int ref_dense(int64_t m, int64_t k, int64_t n, const T* A, const T* B, T* C, int32_t p, int32_t b, int workers) {
  return guarded([&] {
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    cfg.workers = workers;
    const auto c = gemm_dense_blocked(make_dense<T>(m, k, A), make_dense<T>(k, n, B), cfg);
    std::memcpy(C, c.data.data(), sizeof(T) * c.data.size());
  });
}
}  // namespace
extern "C" {
int ref_spdm_csr_f32(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* v, const int32_t* c,
                     const int64_t* rp, const float* B, float* C, int32_t p, int32_t b, int w) {
  return ref_csr<float>(m, k, n, nnz, v, c, rp, B, C, p, b, w);
}
int ref_spdm_csr_f64(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* v, const int32_t* c,
                     const int64_t* rp, const double* B, double* C, int32_t p, int32_t b, int w) {
  return ref_csr<double>(m, k, n, nnz, v, c, rp, B, C, p, b, w);
}
int ref_spdm_coo_f32(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* v, const int32_t* r,
                     const int32_t* c, const float* B, float* C, int32_t p, int32_t b, int w) {
  return ref_coo<float>(m, k, n, nnz, v, r, c, B, C, p, b, w);
}
int ref_spdm_coo_f64(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* v, const int32_t* r,
                     const int32_t* c, const double* B, double* C, int32_t p, int32_t b, int w) {
  return ref_coo<double>(m, k, n, nnz, v, r, c, B, C, p, b, w);
}
int ref_gemm_dense_f32(int64_t m, int64_t k, int64_t n, const float* A, const float* B, float* C, int32_t p,
                       int32_t b, int w) {
  return ref_dense<float>(m, k, n, A, B, C, p, b, w);
}
int ref_gemm_dense_f64(int64_t m, int64_t k, int64_t n, const double* A, const double* B, double* C, int32_t p,
                       int32_t b, int w) {
  return ref_dense<double>(m, k, n, A, B, C, p, b, w);
}

// gemm_oracle (kernels.hpp:80-98): double accumulation, used by the
// reference's own ≤1e-5 / ≤1e-12 gates.
int ref_gemm_oracle_f32(int64_t m, int64_t k, int64_t n, const float* A, const float* B,
                        float* C) {
  return guarded([&] {
    const auto c = gemm_oracle(make_dense<float>(m, k, A), make_dense<float>(k, n, B));
    std::memcpy(C, c.data.data(), sizeof(float) * c.data.size());
  });
}
int ref_gemm_oracle_f64(int64_t m, int64_t k, int64_t n, const double* A, const double* B,
                        double* C) {
  return guarded([&] {
    const auto c = gemm_oracle(make_dense<double>(m, k, A), make_dense<double>(k, n, B));
    std::memcpy(C, c.data.data(), sizeof(double) * c.data.size());
  });
}

// The reference's own benchmark entry (bench.hpp:92-163, gcoo branch):
// EO = dense_to_gcoo once, KC = median of `reps` timed spdm_gcoo calls
// (C allocation included, as in the reference).  out = {eo_s, kc_s, gflops,
// workers, nnz}.
int ref_run_benchmark_gcoo_f32(int64_t n, const float* A, const float* B, int32_t p, int32_t b,
                               int workers, int warmup, int reps, double* out) {
  return guarded([&] {
    const auto a = make_dense<float>(n, n, A);
    const auto bm = make_dense<float>(n, n, B);
    BenchOptions opt;
    opt.exec.p = p;
    opt.exec.b = b;
    opt.exec.workers = workers;
    opt.warmup = warmup;
    opt.repetitions = reps;
    const BenchResult r = run_benchmark(KernelKind::gcoo, a, bm, opt);
    out[0] = r.eo_seconds;
    out[1] = r.kc_seconds;
    out[2] = r.gflops;
    out[3] = r.workers;
    out[4] = static_cast<double>(r.nnz);
  });
}

// Timed spdm_gcoo on caller-provided GCOO (for samples whose dense A would be
// too big to materialise): median of `reps` calls after `warmup`.
int ref_time_spdm_gcoo_f32(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                           const float* vals, const int32_t* rows, const int32_t* cols,
                           int64_t groups, const int64_t* gidx, const int64_t* gnnz,
                           const float* B, int workers, int warmup, int reps, double* out) {
  return guarded([&] {
    const auto a = make_gcoo<float>(m, k, p, nnz, vals, rows, cols, groups, gidx, gnnz);
    const auto bm = make_dense<float>(k, n, B);
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    cfg.workers = workers;
    float sink = 0;
    for (int w = 0; w < warmup; ++w) sink += spdm_gcoo(a, bm, cfg).data.back();
    std::vector<double> ts;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      const auto c = spdm_gcoo(a, bm, cfg);
      ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      sink += c.data.back();
    }
    volatile float keep = sink;
    (void)keep;
    out[0] = median(ts);
    out[1] = resolve_workers(workers);
  });
}

// model_gcoo_traffic / model_csr_traffic (traffic.cpp:43-197) on a coordinate
// pattern; out = {n_dm, n_l2, n_shm, tex_l1_trans, flops, b_element_loads,
// b_element_reused, staged_entries, b_load_transactions, sparse_transactions,
// store_transactions}.
int ref_model_traffic(int csr, int64_t nnz, const int32_t* rows, const int32_t* cols, int64_t m, int64_t k,
                      int64_t n, int32_t p, int32_t b, int infinite_l2, uint64_t* out) {
  return guarded([&] {
    std::vector<Coord> pat(static_cast<size_t>(nnz));
    for (int64_t e = 0; e < nnz; ++e) pat[static_cast<size_t>(e)] = Coord{rows[e], cols[e]};
    ExecConfig cfg;
    cfg.p = p;
    cfg.b = b;
    const CacheMode mode = infinite_l2 ? CacheMode::infinite_l2 : CacheMode::cold;
    TrafficDetail det;
    const TrafficReport r = csr ? model_csr_traffic(pat, m, k, n, cfg, mode, &det)
                                : model_gcoo_traffic(pat, m, k, n, cfg, mode, &det);
    const uint64_t v[11] = {r.n_dm, r.n_l2, r.n_shm, r.tex_l1_trans, r.flops, det.b_element_loads,
                            det.b_element_reused, det.staged_entries, det.b_load_transactions,
                            det.sparse_transactions, det.store_transactions};
    std::memcpy(out, v, sizeof v);
  });
}

}  // extern "C"

// MatrixMarket I/O (io.cpp:57-205 through io.hpp:66-109).  ref_mtx_read_*
// parses into a thread-local cache and reports info = {dense, rows, cols,
// count, error_line}; ref_mtx_fetch_* copies the cached arrays out (COO:
// vals/rows/cols of `count` entries; dense: rows*cols row-major values).
namespace {
template <typename T>
struct MtxCache {
  bool dense = false;
  DenseMatrix<T> d;
  CooMatrix<T> c;
};
template <typename T>
MtxCache<T>& mtx_cache() {
  static thread_local MtxCache<T> m;
  return m;
}
template <typename T>
int mtx_read(const char* path, int64_t* info) {
  info[4] = 0;
  try {
    auto got = read_matrix_market<T>(path);
    auto& m = mtx_cache<T>();
    if (std::holds_alternative<DenseMatrix<T>>(got)) {
      m.dense = true;
      m.d = std::move(std::get<DenseMatrix<T>>(got));
      info[0] = 1, info[1] = m.d.rows, info[2] = m.d.cols, info[3] = m.d.rows * m.d.cols;
    } else {
      m.dense = false;
      m.c = std::move(std::get<CooMatrix<T>>(got));
      info[0] = 0, info[1] = m.c.rows_dim, info[2] = m.c.cols_dim, info[3] = m.c.nnz();
    }
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    info[4] = e.line;
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
template <typename T>
void mtx_fetch(T* vals, int32_t* rows, int32_t* cols) {
  auto& m = mtx_cache<T>();
  if (m.dense) {
    std::memcpy(vals, m.d.data.data(), sizeof(T) * m.d.data.size());
    return;
  }
  std::memcpy(vals, m.c.values.data(), sizeof(T) * m.c.values.size());
  std::memcpy(rows, m.c.row_idx.data(), sizeof(int32_t) * m.c.row_idx.size());
  std::memcpy(cols, m.c.col_idx.data(), sizeof(int32_t) * m.c.col_idx.size());
}
template <typename T>
int mtx_write_coo(const char* path, int64_t m, int64_t k, int64_t nnz, const T* vals, const int32_t* rows,
                  const int32_t* cols) {
  return guarded([&] {
    CooMatrix<T> c;
    c.rows_dim = m;
    c.cols_dim = k;
    c.values.assign(vals, vals + nnz);
    c.row_idx.assign(rows, rows + nnz);
    c.col_idx.assign(cols, cols + nnz);
    write_matrix_market(c, path);
  });
}
template <typename T>
int mtx_write_dense(const char* path, int64_t m, int64_t k, const T* data) {
  return guarded([&] { write_matrix_market(make_dense<T>(m, k, data), path); });
}
}  // namespace

extern "C" {
int ref_mtx_read_f32(const char* path, int64_t* info) { return mtx_read<float>(path, info); }
int ref_mtx_read_f64(const char* path, int64_t* info) { return mtx_read<double>(path, info); }
void ref_mtx_fetch_f32(float* v, int32_t* r, int32_t* c) { mtx_fetch<float>(v, r, c); }
void ref_mtx_fetch_f64(double* v, int32_t* r, int32_t* c) { mtx_fetch<double>(v, r, c); }
int ref_mtx_write_coo_f32(const char* path, int64_t m, int64_t k, int64_t nnz, const float* v, const int32_t* r,
                          const int32_t* c) {
  return mtx_write_coo<float>(path, m, k, nnz, v, r, c);
}
int ref_mtx_write_coo_f64(const char* path, int64_t m, int64_t k, int64_t nnz, const double* v, const int32_t* r,
                          const int32_t* c) {
  return mtx_write_coo<double>(path, m, k, nnz, v, r, c);
}
int ref_mtx_write_dense_f32(const char* path, int64_t m, int64_t k, const float* d) {
  return mtx_write_dense<float>(path, m, k, d);
}
int ref_mtx_write_dense_f64(const char* path, int64_t m, int64_t k, const double* d) {
  return mtx_write_dense<double>(path, m, k, d);
}
}  // extern "C"
