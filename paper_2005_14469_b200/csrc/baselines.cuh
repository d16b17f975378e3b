// baselines.cuh — the reference's comparison kernels on the B200 (SURVEY §8f
// row 3): row-split CSR SpDM (kernels.hpp:163-184), the ungrouped COO ablation
// (kernels.hpp:193-232) and the blocked dense GEMM (kernels.hpp:107-155).
//
// These are yardsticks for the paper's GCOO-vs-CSR/COO/dense comparison, not
// the hot path.  Each keeps the reference's per-element accumulation order,
// so its C is bit-identical to the reference built with FMA contraction (and,
// in the mul+add flavour, to the reference as shipped):
//   * spdm_csr: C(r, :) = chain over row r's entries in CSR order (the
//     reference does not require sorted columns, and neither does this);
//   * spdm_coo: C(r, :) = chain over row r's entries in COO array order (any
//     order, duplicates allowed) — the entries are stably sorted by row on the
//     device, which keeps that order inside each row;
//   * gemm_dense: C(i, j) = chain over l = 0, 1, ..., k-1 of A(i,l)·B(l,j)
//     (the reference's depth blocking never reorders l).
//
// Row-split (both sparse formats): one warp owns a row range x a strip of 32·V
// columns (V = one 16-byte vector per lane), reads the range's entries with
// coalesced 32-wide loads, broadcasts each entry by shuffle and streams its B
// row segment with 16-byte loads (8 in flight), accumulating in registers; no
// staging or reuse, which is what the paper's GCOO grouping adds.  CSR takes
// one row per warp (the reference's row-split); the COO ablation instead cuts
// the row-sorted entry stream into chunks of ~equal nnz aligned to row
// boundaries (the ungrouped stream, load-balanced by entries).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "spdm_rowtile.cuh"

namespace gcoo_b200 {

constexpr int kSplitWarps = 8;

// [row_lo, row_hi) x column tile ct; entries [rp[r], rp[r+1]) of each row.
template <typename T, bool VEC, bool FMA>
__device__ __forceinline__ void rowsplit_warp(int64_t row_lo, int64_t row_hi, int64_t ct, int64_t n,
                                              const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                                              const T* __restrict__ vals, const T* __restrict__ B, int64_t ldb,
                                              T* __restrict__ C, int64_t ldc) {
  constexpr int V = VecOf<T>::V;
  const int lane = threadIdx.x & 31;
  const int64_t j0 = ct * (32 * V) + (int64_t)lane * V;
  for (int64_t r = row_lo; r < row_hi; ++r) {
    T acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = T(0);
    const int64_t lo = rp[r], hi = rp[r + 1];
    for (int64_t base = lo; base < hi; base += 32) {
      const int cnt = (int)min((int64_t)32, hi - base);
      T my_v = T(0);
      int32_t my_c = 0;
      if (lane < cnt) {
        my_v = vals[base + lane];
        my_c = cols[base + lane];
      }
      int q = 0;
      for (; q + 8 <= cnt; q += 8) {
        T bv[8][V], av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          av[u] = __shfl_sync(0xffffffffu, my_v, q + u);
          load_b<T, V, VEC>(B, ldb, __shfl_sync(0xffffffffu, my_c, q + u), j0, n, bv[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) mac_row<T, V, FMA>(acc, av[u], bv[u]);
      }
      for (; q < cnt; ++q) {
        T bv[V];
        const T a = __shfl_sync(0xffffffffu, my_v, q);
        load_b<T, V, VEC>(B, ldb, __shfl_sync(0xffffffffu, my_c, q), j0, n, bv);
        mac_row<T, V, FMA>(acc, a, bv);
      }
    }
    T* dst = C + r * ldc + j0;
    if (VEC) {
      if (j0 < n) {
        typename VecOf<T>::type x;
        T* px = reinterpret_cast<T*>(&x);
#pragma unroll
        for (int v = 0; v < V; ++v) px[v] = acc[v];
        *reinterpret_cast<typename VecOf<T>::type*>(dst) = x;
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (j0 + v < n) dst[v] = acc[v];
    }
  }
}

// ranges == nullptr: warp w owns row w (CSR row-split); else rows
// [ranges[w], ranges[w+1]) (COO chunks).  Row units vary fastest in the grid so
// co-resident warps share a B column strip in L2.
template <typename T, bool VEC, bool FMA>
__global__ void __launch_bounds__(kSplitWarps * 32)
spdm_rowsplit_kernel(int64_t units, int64_t n, const int64_t* __restrict__ ranges, const int64_t* __restrict__ rp,
                     const int32_t* __restrict__ cols, const T* __restrict__ vals, const T* __restrict__ B,
                     int64_t ldb, T* __restrict__ C, int64_t ldc, int64_t unit_blocks) {
  const int warp = threadIdx.x >> 5;
  const int64_t ub = blockIdx.x % unit_blocks;
  const int64_t ct = blockIdx.x / unit_blocks;
  const int64_t u = ub * kSplitWarps + warp;
  if (u >= units) return;
  const int64_t lo = ranges ? ranges[u] : u, hi = ranges ? ranges[u + 1] : u + 1;
  rowsplit_warp<T, VEC, FMA>(lo, hi, ct, n, rp, cols, vals, B, ldb, C, ldc);
}

// COO chunks: unit u starts at the first row whose entries begin at or after
// u*chunk (a row straddling the boundary stays with the unit it starts in);
// rows before the first entry and empty rows belong to a unit too, so every
// row of C is written exactly once.
__global__ void coo_chunk_ranges_kernel(int64_t units, int64_t m, int64_t nnz, int64_t chunk,
                                        const int64_t* __restrict__ rp, int64_t* __restrict__ ranges) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= units;
       u += (int64_t)gridDim.x * blockDim.x) {
    if (u == 0) { ranges[0] = 0; continue; }
    if (u == units) { ranges[u] = m; continue; }
    const int64_t e = min(u * chunk, nnz);
    // first row r with rp[r] >= e (rp is non-decreasing, rp[m] = nnz)
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rp[mid] < e) lo = mid + 1; else hi = mid;
    }
    ranges[u] = lo;
  }
}

// Range checks the reference's unvalidated baselines leave to undefined
// behaviour (they would read out of bounds): first bad index, or ~0.
__global__ void coo_range_kernel(int64_t nnz, int64_t m, int64_t k, const int32_t* __restrict__ rows,
                                 const int32_t* __restrict__ cols, unsigned long long* __restrict__ first_bad,
                                 int* __restrict__ unsorted) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i], c = cols[i];
    if (r < 0 || r >= m || c < 0 || c >= k) atomicMin(first_bad, (unsigned long long)i);
    if (i > 0 && rows[i - 1] > r) *unsorted = 1;
  }
}

__global__ void csr_range_kernel(int64_t m, int64_t k, int64_t nnz, const int64_t* __restrict__ rp,
                                 const int32_t* __restrict__ cols, unsigned long long* __restrict__ first_bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rp[r], b = rp[r + 1];
    if (a > b || a < 0 || b > nnz) {
      atomicMin(first_bad, (unsigned long long)r);
      continue;
    }
    for (int64_t e = a; e < b; ++e)
      if (cols[e] < 0 || cols[e] >= k) {
        atomicMin(first_bad, (unsigned long long)r);
        break;
      }
  }
}

__global__ void iota_kernel(int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

// Entries in their row-sorted (stable) order: out[e] = in[perm[e]].
template <typename T>
__global__ void gather_entries_kernel(int64_t nnz, const int64_t* __restrict__ perm, const T* __restrict__ vals,
                                      const int32_t* __restrict__ cols, T* __restrict__ ovals,
                                      int32_t* __restrict__ ocols) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = perm[e];
    ovals[e] = vals[s];
    ocols[e] = cols[s];
  }
}

// ------------------------------------------------------------ dense GEMM --
// Register-tiled GEMM: a CTA computes BM x BN of C with 256 threads, each a
// TM x TN register tile; A (transposed) and B tiles of depth BK pass through
// shared memory.  Depth runs l = 0, 1, ... in order for every C element.
template <typename T>
struct GemmCfg;
template <>
struct GemmCfg<float> { static constexpr int TM = 8, TN = 8, BK = 8; };
template <>
struct GemmCfg<double> { static constexpr int TM = 4, TN = 8, BK = 8; };

constexpr int kGemmThreads = 256;

template <typename T, bool FMA>
__global__ void __launch_bounds__(kGemmThreads)
gemm_dense_kernel(int64_t m, int64_t k, int64_t n, const T* __restrict__ A, int64_t lda, const T* __restrict__ B,
                  int64_t ldb, T* __restrict__ C, int64_t ldc) {
  constexpr int TM = GemmCfg<T>::TM, TN = GemmCfg<T>::TN, BK = GemmCfg<T>::BK;
  constexpr int TX = 16, TY = kGemmThreads / TX;  // thread grid
  constexpr int BM = TY * TM, BN = TX * TN;
  __shared__ T As[BK][BM];
  __shared__ T Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int64_t bm = (int64_t)blockIdx.y * BM, bn = (int64_t)blockIdx.x * BN;
  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  for (int64_t k0 = 0; k0 < k; k0 += BK) {
    for (int x = tid; x < BM * BK; x += kGemmThreads) {  // A tile, transposed
      const int i = x / BK, kk = x % BK;
      const int64_t gi = bm + i, gk = k0 + kk;
      As[kk][i] = (gi < m && gk < k) ? A[gi * lda + gk] : T(0);
    }
    for (int x = tid; x < BK * BN; x += kGemmThreads) {
      const int kk = x / BN, j = x % BN;
      const int64_t gk = k0 + kk, gj = bn + j;
      Bs[kk][j] = (gk < k && gj < n) ? B[gk * ldb + gj] : T(0);
    }
    __syncthreads();
    const int kmax = (int)min((int64_t)BK, k - k0);  // never add padding products (-0 + 0 keeps signs exact)
    for (int kk = 0; kk < kmax; ++kk) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = mac<T, FMA>(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t gi = bm + ty * TM + i;
    if (gi >= m) break;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t gj = bn + tx * TN + j;
      if (gj < n) C[gi * ldc + gj] = acc[i][j];
    }
  }
}

}  // namespace gcoo_b200
