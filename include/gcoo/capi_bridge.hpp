// gcoo/capi_bridge.hpp — C++ side of the C ABI (include/gcoo_capi.h): status
// codes become the reference's exception types, and float/double overloads
// pick the f32/f64 entry points.  Used by the drop-in gcoo/*.hpp headers.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "gcoo_capi.h"

namespace gcoo::capi {

// GCOO_EINVAL -> std::invalid_argument (thrown before any device work, where
// the reference throws), GCOO_ENOMEM -> std::bad_alloc, else runtime_error.
inline void check(int status) {
  if (status == GCOO_OK) return;
  const std::string msg = gcoo_last_error();
  if (status == GCOO_EINVAL) throw std::invalid_argument(msg);
  if (status == GCOO_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error("libgcoo_cuda: " + msg);
}

inline int spdm(std::int64_t m, std::int64_t k, std::int64_t n, std::int32_t a_p, std::int32_t cfg_p,
                std::int32_t cfg_b, std::int64_t b_rows, std::int64_t nnz, const float* v, const std::int32_t* r,
                const std::int32_t* c, std::int64_t groups, const std::int64_t* gi, const std::int64_t* gn,
                const float* B, float* C, gcoo_stats* st, const std::int64_t* order, std::int64_t count) {
  return gcoo_spdm_f32(m, k, n, a_p, cfg_p, cfg_b, b_rows, nnz, v, r, c, groups, gi, gn, B, C, st, order, count);
}
inline int spdm(std::int64_t m, std::int64_t k, std::int64_t n, std::int32_t a_p, std::int32_t cfg_p,
                std::int32_t cfg_b, std::int64_t b_rows, std::int64_t nnz, const double* v, const std::int32_t* r,
                const std::int32_t* c, std::int64_t groups, const std::int64_t* gi, const std::int64_t* gn,
                const double* B, double* C, gcoo_stats* st, const std::int64_t* order, std::int64_t count) {
  return gcoo_spdm_f64(m, k, n, a_p, cfg_p, cfg_b, b_rows, nnz, v, r, c, groups, gi, gn, B, C, st, order, count);
}

inline int coo_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, std::int64_t nnz, const float* v,
                       const std::int32_t* r, const std::int32_t* c, float* ov, std::int32_t* orr,
                       std::int32_t* oc, std::int64_t* gi, std::int64_t* gn) {
  return gcoo_coo_to_gcoo_f32(m, k, p, nnz, v, r, c, ov, orr, oc, gi, gn);
}
inline int coo_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, std::int64_t nnz, const double* v,
                       const std::int32_t* r, const std::int32_t* c, double* ov, std::int32_t* orr,
                       std::int32_t* oc, std::int64_t* gi, std::int64_t* gn) {
  return gcoo_coo_to_gcoo_f64(m, k, p, nnz, v, r, c, ov, orr, oc, gi, gn);
}

inline int csr_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, std::int64_t nnz, const float* v,
                       const std::int32_t* c, const std::int64_t* rp, float* ov, std::int32_t* orr,
                       std::int32_t* oc, std::int64_t* gi, std::int64_t* gn) {
  return gcoo_csr_to_gcoo_f32(m, k, p, nnz, v, c, rp, ov, orr, oc, gi, gn);
}
inline int csr_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, std::int64_t nnz, const double* v,
                       const std::int32_t* c, const std::int64_t* rp, double* ov, std::int32_t* orr,
                       std::int32_t* oc, std::int64_t* gi, std::int64_t* gn) {
  return gcoo_csr_to_gcoo_f64(m, k, p, nnz, v, c, rp, ov, orr, oc, gi, gn);
}

inline int dense_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, const float* A, std::int64_t cap,
                         float* ov, std::int32_t* orr, std::int32_t* oc, std::int64_t* gi, std::int64_t* gn,
                         std::int64_t* nnz) {
  return gcoo_dense_to_gcoo_f32(m, k, p, A, cap, ov, orr, oc, gi, gn, nnz);
}
inline int dense_to_gcoo(std::int64_t m, std::int64_t k, std::int32_t p, const double* A, std::int64_t cap,
                         double* ov, std::int32_t* orr, std::int32_t* oc, std::int64_t* gi, std::int64_t* gn,
                         std::int64_t* nnz) {
  return gcoo_dense_to_gcoo_f64(m, k, p, A, cap, ov, orr, oc, gi, gn, nnz);
}

inline int spdm_csr(std::int64_t m, std::int64_t k, std::int64_t n, std::int64_t nnz, const float* v,
                    const std::int32_t* c, const std::int64_t* rp, const float* B, float* C) {
  return gcoo_spdm_csr_f32(m, k, n, nnz, v, c, rp, B, C);
}
inline int spdm_csr(std::int64_t m, std::int64_t k, std::int64_t n, std::int64_t nnz, const double* v,
                    const std::int32_t* c, const std::int64_t* rp, const double* B, double* C) {
  return gcoo_spdm_csr_f64(m, k, n, nnz, v, c, rp, B, C);
}
inline int spdm_coo(std::int64_t m, std::int64_t k, std::int64_t n, std::int64_t nnz, const float* v,
                    const std::int32_t* r, const std::int32_t* c, const float* B, float* C) {
  return gcoo_spdm_coo_f32(m, k, n, nnz, v, r, c, B, C);
}
inline int spdm_coo(std::int64_t m, std::int64_t k, std::int64_t n, std::int64_t nnz, const double* v,
                    const std::int32_t* r, const std::int32_t* c, const double* B, double* C) {
  return gcoo_spdm_coo_f64(m, k, n, nnz, v, r, c, B, C);
}
inline int gemm_dense(std::int64_t m, std::int64_t k, std::int64_t n, const float* A, const float* B, float* C) {
  return gcoo_gemm_dense_f32(m, k, n, A, B, C);
}
inline int gemm_dense(std::int64_t m, std::int64_t k, std::int64_t n, const double* A, const double* B, double* C) {
  return gcoo_gemm_dense_f64(m, k, n, A, B, C);
}

inline int spdm_auto(std::int64_t m, std::int64_t k, std::int64_t n, std::int32_t p, std::int32_t b, const float* A,
                     const float* B, float* C, gcoo_stats* st, double* eo, double* kc) {
  return gcoo_spdm_auto_f32(m, k, n, p, b, A, B, C, st, eo, kc);
}
inline int spdm_auto(std::int64_t m, std::int64_t k, std::int64_t n, std::int32_t p, std::int32_t b, const double* A,
                     const double* B, double* C, gcoo_stats* st, double* eo, double* kc) {
  return gcoo_spdm_auto_f64(m, k, n, p, b, A, B, C, st, eo, kc);
}

}  // namespace gcoo::capi
