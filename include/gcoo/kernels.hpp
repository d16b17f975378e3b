// gcoo/kernels.hpp — drop-in for the reference's kernel API
// (proj/include/gcoo/kernels.hpp:1-369).
//
// spdm_gcoo (both overloads, :334-348) and spdm_gcoo_auto (:353-367) keep the
// reference's signatures, validation order and exception types, and run on the
// B200 through gcoo_spdm_{f32,f64} (libgcoo_cuda.so).  C is bitwise
// independent of p, b, tile order and worker count (as in the reference) and
// equals the reference's column-ascending accumulation chain with FMA
// contraction.  spdm_csr / spdm_coo (:163-232) and gemm_dense_blocked
// (:107-155) run as their own row-split / ungrouped-COO / tiled-GEMM kernels
// on the B200 with the reference's accumulation orders; gemm_oracle (the test
// oracle, double accumulation) stays a host loop.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "gcoo/capi_bridge.hpp"
#include "gcoo/matrix.hpp"
#include "gcoo/types.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace gcoo {

// p x b output tiles; both powers of two (kernels.hpp:27-37).  `workers` is
// accepted for API compatibility; the GPU result does not depend on it.
struct ExecConfig {
  index_t p = 4;
  index_t b = 64;
  int workers = 0;

  void validate() const {
    if (!is_pow2(p) || !is_pow2(b)) throw std::invalid_argument("ExecConfig: p and b must be powers of two");
    if (workers < 0) throw std::invalid_argument("ExecConfig: workers must be >= 0");
  }
};

// kernels.hpp:39-46: all OpenMP threads (1 without OpenMP).  Reported by
// run_benchmark; the GPU result does not depend on it.
inline int resolve_workers(int workers) {
  if (workers > 0) return workers;
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

// Counters of the reference's tile schedule for the caller's b (:52-65):
// flops = 2 nnz N; staging_fills = nnz ceil(N/b); b_loads_total = N x runs
// (maximal same-column stretches inside b-entry chunks of a group slice);
// b_loads_reused = N x (nnz - runs).  Computed by a device run counter.
struct KernelStats {
  std::uint64_t flops = 0;
  std::uint64_t b_loads_total = 0;
  std::uint64_t b_loads_reused = 0;
  std::uint64_t staging_fills = 0;

  KernelStats& operator+=(const KernelStats& o) {
    flops += o.flops;
    b_loads_total += o.b_loads_total;
    b_loads_reused += o.b_loads_reused;
    staging_fills += o.staging_fills;
    return *this;
  }
};

struct TimingBreakdown {
  double eo_seconds = 0.0;
  double kc_seconds = 0.0;
};

// ------------------------------------------------------- host oracle GEMM --
// Serial triple loop accumulating in double (:80-98) — the test oracle.
template <typename T>
DenseMatrix<T> gemm_oracle(const DenseMatrix<T>& a, const DenseMatrix<T>& b) {
  if (a.cols != b.rows) throw std::invalid_argument("gemm_oracle: inner dimensions differ");
  DenseMatrix<T> c(a.rows, b.cols);
  for (std::int64_t i = 0; i < a.rows; ++i)
    for (std::int64_t j = 0; j < b.cols; ++j) {
      double s = 0.0;
      for (std::int64_t l = 0; l < a.cols; ++l) s += static_cast<double>(a(i, l)) * static_cast<double>(b(l, j));
      c(i, j) = static_cast<T>(s);
    }
  return c;
}

// Dense blocked GEMM baseline (:107-155) on the B200 (gcoo_gemm_dense_*):
// per C element the sum runs over l ascending whatever the tile geometry, as
// in the reference, so the result does not depend on cfg.
template <typename T>
DenseMatrix<T> gemm_dense_blocked(const DenseMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg) {
  cfg.validate();
  if (a.cols != b.rows) throw std::invalid_argument("gemm_dense_blocked: inner dimensions differ");
  DenseMatrix<T> c(a.rows, b.cols);
  capi::check(capi::gemm_dense(a.rows, a.cols, b.cols, a.data.data(), b.data.data(), c.data.data()));
  return c;
}

// --------------------------------------------------------------- GCOOSpDM --
namespace detail {
template <typename T>
DenseMatrix<T> spdm_gcoo_impl(const GcooMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg,
                              const std::int64_t* tile_order, std::int64_t tile_count, KernelStats* stats) {
  cfg.validate();  // then the shape checks, in the C ABI, in the reference's order (:244-254)
  DenseMatrix<T> c(a.rows_dim, b.cols);
  gcoo_stats st{};
  capi::check(capi::spdm(a.rows_dim, a.cols_dim, b.cols, a.p, cfg.p, cfg.b, b.rows, a.nnz(), a.values.data(),
                         a.row_idx.data(), a.col_idx.data(), a.groups(), a.g_idxes.data(), a.nnz_per_group.data(),
                         b.data.data(), c.data.data(), stats ? &st : nullptr, tile_order, tile_count));
  if (stats) {
    KernelStats k;
    k.flops = st.flops;
    k.b_loads_total = st.b_loads_total;
    k.b_loads_reused = st.b_loads_reused;
    k.staging_fills = st.staging_fills;
    *stats = k;  // the reference overwrites (:325)
  }
  return c;
}
}  // namespace detail

/// C = A * B with A in GCOO form, on the B200 (kernels.hpp:334-340).
template <typename T>
DenseMatrix<T> spdm_gcoo(const GcooMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg,
                         KernelStats* stats = nullptr) {
  return detail::spdm_gcoo_impl(a, b, cfg, nullptr, 0, stats);
}

/// Same, with the reference's explicit tile order (kernels.hpp:342-348): must
/// hold groups * ceil(N/b) tile ids; a permutation cannot change C.
template <typename T>
DenseMatrix<T> spdm_gcoo(const GcooMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg,
                         std::span<const std::int64_t> tile_order, KernelStats* stats = nullptr) {
  return detail::spdm_gcoo_impl(a, b, cfg, tile_order.data(), static_cast<std::int64_t>(tile_order.size()), stats);
}

/// EO (dense -> GCOO on the GPU) + KC (spdm_gcoo), wall-clock split (:353-367).
/// The GCOO stays resident on the device between the two phases
/// (gcoo_spdm_auto_*): only A, B and C cross PCIe.
template <typename T>
DenseMatrix<T> spdm_gcoo_auto(const DenseMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg,
                              TimingBreakdown& timing, KernelStats* stats = nullptr) {
  cfg.validate();
  if (a.cols != b.rows) throw std::invalid_argument("spdm_gcoo: inner dimensions differ");
  DenseMatrix<T> c(a.rows, b.cols);
  gcoo_stats st{};
  double eo = 0.0, kc = 0.0;
  capi::check(capi::spdm_auto(a.rows, a.cols, b.cols, cfg.p, cfg.b, a.data.data(), b.data.data(), c.data.data(),
                              stats ? &st : nullptr, &eo, &kc));
  if (stats) {
    KernelStats k;
    k.flops = st.flops;
    k.b_loads_total = st.b_loads_total;
    k.b_loads_reused = st.b_loads_reused;
    k.staging_fills = st.staging_fills;
    *stats = k;
  }
  timing.eo_seconds = eo;
  timing.kc_seconds = kc;
  return c;
}

// ---------------------------------------------- CSR / COO baselines (GPU) --
/// Row-split CSR SpDM (:163-184) on the B200 (gcoo_spdm_csr_*): each row's
/// nonzeros in CSR order, no staging or reuse.  Like the reference it does
/// not validate the CSR (out-of-range indices are rejected, not read).
template <typename T>
DenseMatrix<T> spdm_csr(const CsrMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg) {
  cfg.validate();
  if (a.cols_dim != b.rows) throw std::invalid_argument("spdm_csr: inner dimensions differ");
  DenseMatrix<T> c(a.rows_dim, b.cols);
  if (a.row_ptr.size() != static_cast<std::size_t>(a.rows_dim) + 1 || a.col_idx.size() != a.values.size())
    throw std::invalid_argument("spdm_csr: inconsistent CSR arrays");
  capi::check(capi::spdm_csr(a.rows_dim, a.cols_dim, b.cols, a.nnz(), a.values.data(), a.col_idx.data(),
                             a.row_ptr.data(), b.data.data(), c.data.data()));
  return c;
}

/// Ungrouped COO SpDM ablation (:193-232) on the B200 (gcoo_spdm_coo_*): any
/// entry order, as the reference (each row's chain in array order).
template <typename T>
DenseMatrix<T> spdm_coo(const CooMatrix<T>& a, const DenseMatrix<T>& b, const ExecConfig& cfg) {
  cfg.validate();
  if (a.cols_dim != b.rows) throw std::invalid_argument("spdm_coo: inner dimensions differ");
  DenseMatrix<T> c(a.rows_dim, b.cols);
  if (a.row_idx.size() != a.values.size() || a.col_idx.size() != a.values.size())
    throw std::invalid_argument("spdm_coo: inconsistent COO arrays");
  capi::check(capi::spdm_coo(a.rows_dim, a.cols_dim, b.cols, a.nnz(), a.values.data(), a.row_idx.data(),
                             a.col_idx.data(), b.data.data(), c.data.data()));
  return c;
}

}  // namespace gcoo
