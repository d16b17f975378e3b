/*
 * gcoo_capi.h — the C ABI of libgcoo_cuda.so, the B200 (sm_100a) GCOOSpDM path.
 *
 * Plain pointers and sizes only (no C++ or torch types).  Each entry point
 * replaces one function of the reference's header-only C++ API (paths relative
 * to the reference's proj/ directory); include/gcoo/*.hpp are drop-in C++
 * headers that keep the reference's names, struct layouts and exceptions and
 * forward the hot-path bodies here.  See INTEGRATION.md for the bindings.
 *
 * Conventions
 *  - Every function returns a status: GCOO_OK, or an error whose message is
 *    available from gcoo_last_error() (thread-local).  The status classes map
 *    to the reference's exception types: GCOO_EINVAL -> std::invalid_argument
 *    (raised before any device work, exactly where the reference throws),
 *    GCOO_ECUDA -> std::runtime_error, GCOO_ENOMEM -> std::bad_alloc.
 *  - Host-pointer entry points accept ordinary (pageable) or pinned host
 *    memory, copy to the current device, compute, and copy back; they return
 *    after the results are in host memory.
 *  - `_dev` entry points take device pointers and a cudaStream_t (as void*;
 *    NULL = legacy default stream) and are stream-ordered: they enqueue work
 *    and return without synchronising, except where a host-visible scalar
 *    result (an nnz, stats) is requested.
 *  - All device work is hand-written CUDA for sm_100a.  There is no CPU
 *    fallback: without a usable B200 every compute entry point returns
 *    GCOO_ECUDA.
 *  - Results are deterministic and independent of p, b, the tile order and the
 *    number of GPUs: C(i,j) is the sequential FP32 (FP64) fused multiply-add
 *    chain over row i's nonzeros in ascending column order, i.e. bit-identical
 *    to the reference built with FMA contraction (-mfma) and within 4.6e-7
 *    relative of the reference as shipped (mul+add); the `exact_mul_add`
 *    variants reproduce the as-shipped bits instead.
 */
#ifndef GCOO_CAPI_H
#define GCOO_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCOO_OK 0
#define GCOO_EINVAL 1 /* std::invalid_argument */
#define GCOO_ECUDA 2  /* std::runtime_error (CUDA / NCCL failure, no device) */
#define GCOO_ENOMEM 3 /* std::bad_alloc */

#define GCOO_ABI_VERSION 1

/* KernelStats (kernels.hpp:52-65), same field order. */
typedef struct gcoo_stats {
  uint64_t flops;
  uint64_t b_loads_total;
  uint64_t b_loads_reused;
  uint64_t staging_fills;
} gcoo_stats;

/* Numeric flavour of the multiply (see header comment). */
#define GCOO_FLAVOR_FMA 0     /* default: FFMA chain */
#define GCOO_FLAVOR_MUL_ADD 1 /* fl(acc + fl(a*b)): reference as shipped */

/* ------------------------------------------------------------ runtime ---- */
int gcoo_abi_version(void);

/* The B200 roofline profile the reference's table lacks (kProfiles,
 * src/traffic.cpp:223-227 holds gtx980 / titanx / p100): this pool's measured
 * FP32 FFMA peak (tools/microbench/mb.cu, profiles/r01_microbench.json) and
 * HBM copy bandwidth (MEASURED_PEAKS.json), FLOP/s and bytes/s.  No device
 * needed. */
int gcoo_roofline_b200(double* peak_flops, double* bandwidth);
const char* gcoo_last_error(void);
/* Number of visible CUDA devices (0 on a machine without a GPU). */
int gcoo_device_count(int* count);
/* Select the device used by this thread's subsequent host-pointer calls. */
int gcoo_set_device(int device);
/* Kernel launches this process has issued (all entry points).  bench.py
 * reports the delta over its timed region as gpu_launches. */
uint64_t gcoo_launch_count(void);
/* Block until all work this library enqueued on `stream` completed. */
int gcoo_stream_sync(void* stream);

/* ------------------------------------------------------- GCOOSpDM ------- */
/*
 * spdm_gcoo (kernels.hpp:334-348 -> detail::spdm_gcoo_impl :240-327).
 * A in GCOO form (matrix.hpp:176-245): `groups` = ceil(m/p) groups, group i's
 * slice is values/row_idx/col_idx[g_idxes[i] .. g_idxes[i]+nnz_per_group[i]),
 * ordered by (col,row).  B is k x n row-major, C is m x n row-major and is
 * fully overwritten.  cfg = (p, b): both powers of two, p == A's p.
 * tile_order (nullable) must hold groups*ceil(n/b) entries, as the reference
 * requires (:253-254); tiles own disjoint outputs so a permutation does not
 * change C.  stats (nullable) receives KernelStats for the caller's b.
 * Errors (EINVAL, before any work): p or b not a power of two (:32-36),
 * inner dimensions differ (k != rows of B) (:245-246), A grouped with a
 * different p (:247-248), wrong tile_order length (:253-254).
 */
int gcoo_spdm_f32(int64_t m, int64_t k, int64_t n, int32_t a_p, int32_t cfg_p, int32_t cfg_b,
                  int64_t b_rows, int64_t nnz, const float* values, const int32_t* row_idx,
                  const int32_t* col_idx, int64_t groups, const int64_t* g_idxes,
                  const int64_t* nnz_per_group, const float* B, float* C, gcoo_stats* stats,
                  const int64_t* tile_order, int64_t tile_count);
int gcoo_spdm_f64(int64_t m, int64_t k, int64_t n, int32_t a_p, int32_t cfg_p, int32_t cfg_b,
                  int64_t b_rows, int64_t nnz, const double* values, const int32_t* row_idx,
                  const int32_t* col_idx, int64_t groups, const int64_t* g_idxes,
                  const int64_t* nnz_per_group, const double* B, double* C, gcoo_stats* stats,
                  const int64_t* tile_order, int64_t tile_count);

/* Device-pointer, stream-ordered variant.  B has leading dimension ldb >= n,
 * C has ldc >= n (a column shard of a wider matrix is passed by pointer
 * offset).  `stats` (host, nullable) forces a synchronisation.  `flavor` is
 * GCOO_FLAVOR_FMA or GCOO_FLAVOR_MUL_ADD. */
int gcoo_spdm_f32_dev(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                      const float* values, const int32_t* row_idx, const int32_t* col_idx,
                      int64_t groups, const int64_t* g_idxes, const int64_t* nnz_per_group,
                      const float* B, int64_t ldb, float* C, int64_t ldc, gcoo_stats* stats,
                      int flavor, void* stream);
int gcoo_spdm_f64_dev(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                      const double* values, const int32_t* row_idx, const int32_t* col_idx,
                      int64_t groups, const int64_t* g_idxes, const int64_t* nnz_per_group,
                      const double* B, int64_t ldb, double* C, int64_t ldc, gcoo_stats* stats,
                      int flavor, void* stream);

/*
 * Plan / execute split (an extension; the reference recomputes nothing between
 * calls because its kernel reads the GCOO arrays directly).  The B200 multiply
 * runs from a record stream built from A by a ~35 us planner; a caller that
 * multiplies the same A by many B builds it once here.  A's device arrays must
 * stay alive and unchanged while the plan exists.  The plan's buffers are
 * stream-ordered on `stream`: multiplies on other streams must be ordered
 * after the create.  gcoo_plan_spdm_*_dev is stream-ordered and returns the
 * same bits as gcoo_spdm_*_dev (any B/C layout; an unaligned one is planned
 * per call).  gcoo_plan_destroy synchronises the device, then frees.
 */
typedef struct gcoo_plan gcoo_plan;
int gcoo_plan_create_f32_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const float* values,
                             const int32_t* row_idx, const int32_t* col_idx, int64_t groups,
                             const int64_t* g_idxes, const int64_t* nnz_per_group, int flavor,
                             gcoo_plan** plan, void* stream);
int gcoo_plan_spdm_f32_dev(const gcoo_plan* plan, int64_t n, const float* B, int64_t ldb, float* C,
                           int64_t ldc, void* stream);
/* fp64 twins (a plan serves only the element type it was built for). */
int gcoo_plan_create_f64_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const double* values,
                             const int32_t* row_idx, const int32_t* col_idx, int64_t groups,
                             const int64_t* g_idxes, const int64_t* nnz_per_group, int flavor,
                             gcoo_plan** plan, void* stream);
int gcoo_plan_spdm_f64_dev(const gcoo_plan* plan, int64_t n, const double* B, int64_t ldb, double* C,
                           int64_t ldc, void* stream);
int gcoo_plan_destroy(gcoo_plan* plan);

/* KernelStats only (K4 run counter; kernels.hpp:283-310) for a device GCOO. */
int gcoo_stats_dev(int64_t m, int64_t n, int32_t p, int32_t b, int64_t nnz,
                   const int32_t* row_idx, const int32_t* col_idx, int64_t groups,
                   const int64_t* g_idxes, gcoo_stats* stats, void* stream);

/* ------------------------------------------------- traffic model -------- */
/* TrafficReport / TrafficDetail (traffic.hpp:31-56), same field order. */
typedef struct gcoo_traffic {
  uint64_t n_dm;
  uint64_t n_l2;
  uint64_t n_shm;
  uint64_t tex_l1_trans;
  uint64_t flops;
} gcoo_traffic;
typedef struct gcoo_traffic_detail {
  uint64_t b_element_loads;
  uint64_t b_element_reused;
  uint64_t staged_entries;
  uint64_t b_load_transactions;
  uint64_t sparse_transactions;
  uint64_t store_transactions;
} gcoo_traffic_detail;
#define GCOO_CACHE_COLD 0        /* CacheMode::cold */
#define GCOO_CACHE_INFINITE_L2 1 /* CacheMode::infinite_l2 */
#define GCOO_MODEL_GCOO 0        /* model_gcoo_traffic (traffic.cpp:43-137) */
#define GCOO_MODEL_CSR 1         /* model_csr_traffic  (traffic.cpp:140-197) */
/*
 * The reference's analytical traffic model of an m x k pattern times a dense
 * k x n operand under cfg (p, b), evaluated on the device.  The pattern is
 * given as A's GCOO arrays (device pointers, grouped with this p — run
 * coo_to_gcoo first for an arbitrary coordinate list); counts are exact and
 * equal the reference's.  `det` may be NULL.  Synchronises `stream`.
 */
int gcoo_model_traffic_dev(int kind, int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, int64_t nnz,
                           const int32_t* row_idx, const int32_t* col_idx, int64_t groups, const int64_t* g_idxes,
                           const int64_t* nnz_per_group, int cache_mode, gcoo_traffic* rep,
                           gcoo_traffic_detail* det, void* stream);

/* ------------------------------------------------------ construction ---- */
/*
 * coo_to_gcoo (matrix.hpp:366-405).  Input: row-major COO, validated exactly
 * like CooMatrix::validate (:95-115) -> EINVAL naming the first bad entry.
 * Outputs are caller-allocated: nnz entries and ceil(m/p) groups.
 */
int gcoo_coo_to_gcoo_f32(int64_t m, int64_t k, int32_t p, int64_t nnz, const float* values,
                         const int32_t* row_idx, const int32_t* col_idx, float* out_values,
                         int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                         int64_t* nnz_per_group);
int gcoo_coo_to_gcoo_f64(int64_t m, int64_t k, int32_t p, int64_t nnz, const double* values,
                         const int32_t* row_idx, const int32_t* col_idx, double* out_values,
                         int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                         int64_t* nnz_per_group);
int gcoo_coo_to_gcoo_f32_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const float* values,
                             const int32_t* row_idx, const int32_t* col_idx, float* out_values,
                             int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                             int64_t* nnz_per_group, void* stream);
int gcoo_coo_to_gcoo_f64_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const double* values,
                             const int32_t* row_idx, const int32_t* col_idx, double* out_values,
                             int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                             int64_t* nnz_per_group, void* stream);

/*
 * csr_to_gcoo — new entry point (the north star's "COO/CSR-to-GCOO"); the
 * reference only has coo_to_csr (matrix.hpp:407-419).  CSR validated like
 * CsrMatrix::validate (:122-165); row_ptr has m+1 int64 offsets.
 */
int gcoo_csr_to_gcoo_f32(int64_t m, int64_t k, int32_t p, int64_t nnz, const float* values,
                         const int32_t* col_idx, const int64_t* row_ptr, float* out_values,
                         int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                         int64_t* nnz_per_group);
int gcoo_csr_to_gcoo_f64(int64_t m, int64_t k, int32_t p, int64_t nnz, const double* values,
                         const int32_t* col_idx, const int64_t* row_ptr, double* out_values,
                         int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                         int64_t* nnz_per_group);
/* Device variants (all arrays device pointers; synchronise `stream` for the
 * validation verdict). */
int gcoo_csr_to_gcoo_f32_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const float* values,
                             const int32_t* col_idx, const int64_t* row_ptr, float* out_values,
                             int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                             int64_t* nnz_per_group, void* stream);
int gcoo_csr_to_gcoo_f64_dev(int64_t m, int64_t k, int32_t p, int64_t nnz, const double* values,
                             const int32_t* col_idx, const int64_t* row_ptr, double* out_values,
                             int32_t* out_row_idx, int32_t* out_col_idx, int64_t* g_idxes,
                             int64_t* nnz_per_group, void* stream);

/*
 * dense_to_gcoo (matrix.hpp:306-353).  A is m x k row-major; entries != 0
 * are kept.  Two-call protocol because nnz is unknown up front:
 *   1. out_values == NULL: count, build the GCOO on the device, keep it in a
 *      per-thread slot keyed by (A, m, k, p) and return *nnz.
 *   2. out arrays sized from *nnz: copy the kept result out (or rebuild if
 *      the key differs) and release the slot.
 * `capacity` is the size of the caller's entry arrays in call 2.
 */
int gcoo_dense_to_gcoo_f32(int64_t m, int64_t k, int32_t p, const float* A, int64_t capacity,
                           float* out_values, int32_t* out_row_idx, int32_t* out_col_idx,
                           int64_t* g_idxes, int64_t* nnz_per_group, int64_t* nnz);
int gcoo_dense_to_gcoo_f64(int64_t m, int64_t k, int32_t p, const double* A, int64_t capacity,
                           double* out_values, int32_t* out_row_idx, int32_t* out_col_idx,
                           int64_t* g_idxes, int64_t* nnz_per_group, int64_t* nnz);
/*
 * spdm_gcoo_auto (kernels.hpp:353-367) with the GCOO kept on the device: A
 * (m x k, host) is grouped on the GPU and multiplied by B (k x n, host) into C
 * (m x n, host) without the GCOO arrays crossing PCIe.  eo_seconds /
 * kc_seconds (nullable) receive the wall-clock phases (EO: A up + grouping;
 * KC: B up + multiply + C down), stats (nullable) the KernelStats for b.
 */
int gcoo_spdm_auto_f32(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, const float* A, const float* B,
                       float* C, gcoo_stats* stats, double* eo_seconds, double* kc_seconds);
int gcoo_spdm_auto_f64(int64_t m, int64_t k, int64_t n, int32_t p, int32_t b, const double* A, const double* B,
                       double* C, gcoo_stats* stats, double* eo_seconds, double* kc_seconds);
/* Device variant: counts into g_idxes/nnz_per_group (device, ceil(m/p)),
 * returns *nnz (host; synchronises), and fills the entry arrays when
 * capacity >= *nnz (otherwise leaves them untouched and returns GCOO_OK so
 * the caller can allocate and call again). */
int gcoo_dense_to_gcoo_f32_dev(int64_t m, int64_t k, int32_t p, const float* A, int64_t capacity,
                               float* out_values, int32_t* out_row_idx, int32_t* out_col_idx,
                               int64_t* g_idxes, int64_t* nnz_per_group, int64_t* nnz,
                               void* stream);
int gcoo_dense_to_gcoo_f64_dev(int64_t m, int64_t k, int32_t p, const double* A, int64_t capacity,
                               double* out_values, int32_t* out_row_idx, int32_t* out_col_idx,
                               int64_t* g_idxes, int64_t* nnz_per_group, int64_t* nnz,
                               void* stream);

/* ------------------------------------------- baselines */
/*
 * The reference's comparison kernels on the GPU, each with the reference's
 * per-element accumulation order (bit-identical to it built with FMA
 * contraction; `flavor` as for spdm):
 *  - spdm_csr (kernels.hpp:163-184): row-split over a CSR (int64 row_ptr[m+1],
 *    int32 columns, any order inside a row), C(r,:) = chain in CSR order;
 *  - spdm_coo (kernels.hpp:193-232): any COO entry order (duplicates too),
 *    C(r,:) = chain over row r's entries in array order;
 *  - gemm_dense (kernels.hpp:107-155, gemm_dense_blocked): C = A*B with every
 *    element summed over l ascending.
 * The reference does not validate these inputs (an out-of-range index is
 * undefined behaviour there); here it is GCOO_EINVAL.  C is fully written.
 */
int gcoo_spdm_csr_f32(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* values, const int32_t* col_idx,
                      const int64_t* row_ptr, const float* B, float* C);
int gcoo_spdm_csr_f64(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* values, const int32_t* col_idx,
                      const int64_t* row_ptr, const double* B, double* C);
int gcoo_spdm_csr_f32_dev(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* values, const int32_t* col_idx,
                          const int64_t* row_ptr, const float* B, int64_t ldb, float* C, int64_t ldc, int flavor,
                          void* stream);
int gcoo_spdm_csr_f64_dev(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* values,
                          const int32_t* col_idx, const int64_t* row_ptr, const double* B, int64_t ldb, double* C,
                          int64_t ldc, int flavor, void* stream);
int gcoo_spdm_coo_f32(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* values, const int32_t* row_idx,
                      const int32_t* col_idx, const float* B, float* C);
int gcoo_spdm_coo_f64(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* values, const int32_t* row_idx,
                      const int32_t* col_idx, const double* B, double* C);
int gcoo_spdm_coo_f32_dev(int64_t m, int64_t k, int64_t n, int64_t nnz, const float* values, const int32_t* row_idx,
                          const int32_t* col_idx, const float* B, int64_t ldb, float* C, int64_t ldc, int flavor,
                          void* stream);
int gcoo_spdm_coo_f64_dev(int64_t m, int64_t k, int64_t n, int64_t nnz, const double* values,
                          const int32_t* row_idx, const int32_t* col_idx, const double* B, int64_t ldb, double* C,
                          int64_t ldc, int flavor, void* stream);
int gcoo_gemm_dense_f32(int64_t m, int64_t k, int64_t n, const float* A, const float* B, float* C);
int gcoo_gemm_dense_f64(int64_t m, int64_t k, int64_t n, const double* A, const double* B, double* C);
int gcoo_gemm_dense_f32_dev(int64_t m, int64_t k, int64_t n, const float* A, int64_t lda, const float* B,
                            int64_t ldb, float* C, int64_t ldc, int flavor, void* stream);
int gcoo_gemm_dense_f64_dev(int64_t m, int64_t k, int64_t n, const double* A, int64_t lda, const double* B,
                            int64_t ldb, double* C, int64_t ldc, int flavor, void* stream);

/* ------------------------------------------------ synthetic inputs ------ */
/*
 * generate_uniform_sparse<T>(n, s, seed) (io.hpp:129-145, io.cpp:224-258):
 * the reference's own benchmark inputs (std::mt19937_64 stream, exact nnz =
 * llround(n*n*(1-s)), values 1-u in (0,1]).  Host-side harness code (the
 * stream is sequential); bit-identical to the reference.  derive_seed is
 * bench.cpp:55-65.
 */
int gcoo_generate_uniform_sparse_f32(int64_t n, double s, uint64_t seed, float* out);
int gcoo_generate_uniform_sparse_coo_f32(int64_t n, double s, uint64_t seed, int64_t capacity,
                                         float* values, int32_t* row_idx, int32_t* col_idx,
                                         int64_t* nnz);
uint64_t gcoo_derive_seed(uint64_t base, uint64_t salt_a, uint64_t salt_b);
/* Power-law rows (not in the reference): row-major COO. */
int gcoo_generate_powerlaw_coo_f32(int64_t n, double s, double alpha, uint64_t seed,
                                   int64_t capacity, float* values, int32_t* row_idx,
                                   int32_t* col_idx, int64_t* nnz);

/* ------------------------------------------------ MatrixMarket ---------- */
/*
 * Entry section of a MatrixMarket file — the text after the size line — parsed
 * on the host's threads (threads <= 0: up to one per MiB of text and core;
 * threads > 0: exactly that many newline-aligned chunks).  The tokenising
 * half of read_matrix_market_raw (io.cpp:109-158): blank and '%' lines are
 * skipped; every other line must hold exactly ncol tokens (3 coordinate
 * real/integer, 2 pattern, 1 array), the first two of a coordinate line
 * integers (1-based, written to idx[2*i], idx[2*i+1]), the last of a
 * real/integer/array line a finite decimal (vals[i], via strtod: bit-identical
 * to the reference's num_get<double>).  line_of[i] = 0-based line index of
 * data line i within `text`.  At most `cap` rows are written; any pointer may
 * be NULL.  Returns the number of data lines, or GCOO_MTX_IRREGULAR when some
 * data line breaks the rules above (the caller re-reads that file line by
 * line for the reference's exact ParseError).  No range, symmetry, order or
 * duplicate checks here.
 */
#define GCOO_MTX_IRREGULAR (-1)
int64_t gcoo_mtx_parse_entries(const char* text, int64_t len, int32_t ncol, int64_t cap, int64_t* idx,
                               double* vals, int64_t* line_of, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif /* GCOO_CAPI_H */
