// construct.cuh — GCOO construction and counter kernels (K2-K5).
//
//  K2 coo_to_gcoo   (matrix.hpp:366-405): validate -> row offsets -> group
//     offsets -> log2(p) rounds of pairwise merges of (col,row)-sorted runs.
//     A row-major COO is a sequence of single-row runs, each sorted by col;
//     round t merges runs of 2^t rows pairwise, every entry computing its
//     destination with one binary search in the partner run.  After log2(p)
//     rounds each p-row band is one (col,row)-sorted slice: the GCOO.  Keys
//     (col,row) are unique inside a band, so the result is the unique sorted
//     order — bit-exact with the reference's std::sort, no tie-breaking.
//  K3 dense_to_gcoo (matrix.hpp:306-353): per (band, 256-column tile) count ->
//     device exclusive scan -> per-tile fill in column-major-within-band order.
//  K4 run counter   (kernels.hpp:283-310): KernelStats for the caller's b.
//  K5 csr_to_gcoo   (new): validate CSR -> expand row_ptr to row indices -> K2.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

namespace gcoo_b200 {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// ---------------------------------------------------------------- scan ----
// Block-wide exclusive scan of per-thread int64 values; returns the block total.
template <int NT>
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t x, int64_t& total) {
  __shared__ int64_t warp_sums[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < NT / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < NT / 32) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int64_t warp_off = warp ? warp_sums[warp - 1] : 0;
  total = warp_sums[NT / 32 - 1];
  __syncthreads();
  return warp_off + incl - x;
}

__global__ void __launch_bounds__(kScanThreads)
scan_tiles_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                  int64_t* __restrict__ tile_sums) {
  griddep_wait();  // PDL: predecessor complete
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  int64_t total;
  int64_t run = block_exclusive_scan<kScanThreads>(s, total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0) {
    tile_sums[blockIdx.x] = total;
    if (gridDim.x == 1) out[n] = total;  // single tile: the total is final (no write_total launch)
  }
}

__global__ void add_tile_offsets_kernel(int64_t* __restrict__ out, int64_t n,
                                        const int64_t* __restrict__ tile_off) {
  griddep_wait();  // PDL: predecessor complete
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / kScanTile];
}

__global__ void write_total_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  griddep_wait();  // PDL: predecessor complete
  out[n] = n > 0 ? out[n - 1] + in[n - 1] : 0;
}

// --------------------------------------------------------------- K2 -------
// First invalid entry, encoded 2*i + kind (kind 0: coordinate out of range,
// 1: not strictly row-major / duplicate), in CooMatrix::validate's order.
__global__ void validate_coo_kernel(int64_t nnz, int64_t m, int64_t k, const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ cols, unsigned long long* first_bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[i], c = cols[i];
    unsigned long long code = ~0ull;
    if (r < 0 || r >= m || c < 0 || c >= k) {
      code = 2ull * (unsigned long long)i;
    } else if (i > 0) {
      const int32_t pr = rows[i - 1], pc = cols[i - 1];
      if (!(pr < r || (pr == r && pc < c))) code = 2ull * (unsigned long long)i + 1ull;
    }
    if (code != ~0ull) atomicMin(first_bad, code);
  }
}

// row_ptr[r] = #entries with row < r, r in [0, m] (binary search; rows sorted)
__global__ void row_ptr_kernel(int64_t m, int64_t nnz, const int32_t* __restrict__ rows,
                               int64_t* __restrict__ rp) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > m) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rows[mid] < r) lo = mid + 1; else hi = mid;
  }
  rp[r] = lo;
}

__global__ void group_offsets_kernel(int64_t groups, int64_t m, int32_t p, const int64_t* __restrict__ rp,
                                     int64_t* __restrict__ gidx, int64_t* __restrict__ gnnz) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  const int64_t lo = g * p;
  const int64_t hi = lo + p < m ? lo + p : m;
  gidx[g] = rp[lo];
  gnnz[g] = rp[hi] - rp[lo];
}

// One merge round: runs of 2^t rows -> runs of 2^(t+1) rows.
template <typename T>
__global__ void merge_round_kernel(int64_t nnz, int64_t m, int t, const int64_t* __restrict__ rp,
                                   const T* __restrict__ vin, const int32_t* __restrict__ rin,
                                   const int32_t* __restrict__ cin, T* __restrict__ vout,
                                   int32_t* __restrict__ rout, int32_t* __restrict__ cout) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rin[i], c = cin[i];
    const int64_t q = (int64_t)r >> t;           // own run
    const int64_t pq = q ^ 1;                    // partner run
    const int64_t own_lo = rp[q << t];
    const int64_t pair_lo = rp[(q >> 1) << (t + 1)];
    int64_t plo_row = pq << t, phi_row = (pq + 1) << t;
    if (plo_row > m) plo_row = m;
    if (phi_row > m) phi_row = m;
    int64_t lo = rp[plo_row], hi = rp[phi_row];
    // count partner entries with (col,row) < (c,r)
    const int64_t start = lo;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const int32_t mc = cin[mid], mr = rin[mid];
      if (mc < c || (mc == c && mr < r)) lo = mid + 1; else hi = mid;
    }
    const int64_t dst = pair_lo + (i - own_lo) + (lo - start);
    vout[dst] = vin[i];
    rout[dst] = r;
    cout[dst] = c;
  }
}

// --------------------------------------------------------------- K5 -------
// CsrMatrix::validate (matrix.hpp:122-165) after the host-side size checks:
// first bad row r and its first error, code 4r + kind (0: row_ptr not
// monotone, 1: column out of range, 2: columns not strictly increasing),
// checked in the reference's order.  A row whose range leaves [0, nnz) is
// reported as non-monotone (row_ptr starts at 0 and ends at nnz, so some
// offset decreases) and its columns are never read.
__global__ void validate_csr_kernel(int64_t m, int64_t k, int64_t nnz, const int64_t* __restrict__ rp,
                                    const int32_t* __restrict__ cols, unsigned long long* first_bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rp[r], b = rp[r + 1];
    unsigned long long code = ~0ull;
    if (a > b || a < 0 || b > nnz) {
      code = 4ull * (unsigned long long)r;
    } else {
      for (int64_t e = a; e < b; ++e) {
        const int32_t c = cols[e];
        if (c < 0 || c >= k) { code = 4ull * (unsigned long long)r + 1ull; break; }
        if (e > a && cols[e - 1] >= c) { code = 4ull * (unsigned long long)r + 2ull; break; }
      }
    }
    if (code != ~0ull) atomicMin(first_bad, code);
  }
}

__global__ void expand_rows_kernel(int64_t nnz, int64_t m, const int64_t* __restrict__ rp,
                                   int32_t* __restrict__ rows) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m + 1;  // first index with rp[idx] > i
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rp[mid] <= i) lo = mid + 1; else hi = mid;
    }
    rows[i] = (int32_t)(lo - 1);
  }
}

// --------------------------------------------------------------- K3 -------
constexpr int kDenseTileCols = 256;

// counts[g * n_ct + ct] = nonzeros of band g in columns [ct*256, ct*256+256)
// A thread owns VEC consecutive columns of a p-row band (one 16-byte load per
// row when the rows allow it, else VEC = 1): a tile is kDenseTileCols * VEC
// columns of one group's band.
template <typename T, int VEC>
struct DenseVec;
template <typename T>
struct DenseVec<T, 1> {
  static __device__ __forceinline__ void load(const T* p, T (&v)[1]) { v[0] = __ldg(p); }
};
template <>
struct DenseVec<float, 4> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[4]) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
};
template <>
struct DenseVec<double, 2> {
  static __device__ __forceinline__ void load(const double* p, double (&v)[2]) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(p));
    v[0] = x.x; v[1] = x.y;
  }
};

// nonzeros of this thread's VEC columns over the band's rows (k % VEC == 0 when VEC > 1)
template <typename T, int VEC>
__device__ __forceinline__ int64_t dense_band_count(const T* __restrict__ A, int64_t k, int64_t lo, int64_t hi,
                                                    int64_t c) {
  int64_t cnt = 0;
  if (c < k) {
#pragma unroll 4
    for (int64_t r = lo; r < hi; ++r) {
      T v[VEC];
      DenseVec<T, VEC>::load(A + r * k + c, v);
#pragma unroll
      for (int q = 0; q < VEC; ++q) cnt += v[q] != T(0);
    }
  }
  return cnt;
}

template <typename T, int VEC>
__global__ void __launch_bounds__(kDenseTileCols)
dense_count_kernel(int64_t m, int64_t k, int32_t p, const T* __restrict__ A, int64_t n_ct,
                   int64_t tiles, int64_t* __restrict__ counts) {
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t g = tile / n_ct, ct = tile % n_ct;
    const int64_t c = (ct * kDenseTileCols + threadIdx.x) * VEC;
    const int64_t lo = g * p;
    const int64_t hi = lo + p < m ? lo + p : m;
    int64_t cnt = dense_band_count<T, VEC>(A, k, lo, hi, c);
    // block reduction
#pragma unroll
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    __shared__ int64_t ws[kDenseTileCols / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t s = 0;
      for (int w = 0; w < kDenseTileCols / 32; ++w) s += ws[w];
      counts[tile] = s;
    }
    __syncthreads();
  }
}

// Entries in (col, row) order inside the band: a thread writes its columns one
// after the other, each down the band's rows, at its exclusive-scan offset.
template <typename T, int VEC>
__global__ void __launch_bounds__(kDenseTileCols)
dense_fill_kernel(int64_t m, int64_t k, int32_t p, const T* __restrict__ A, int64_t n_ct, int64_t tiles,
                  const int64_t* __restrict__ tile_off, T* __restrict__ vals, int32_t* __restrict__ rows,
                  int32_t* __restrict__ cols) {
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t g = tile / n_ct, ct = tile % n_ct;
    const int64_t c = (ct * kDenseTileCols + threadIdx.x) * VEC;
    const int64_t lo = g * p;
    const int64_t hi = lo + p < m ? lo + p : m;
    const int64_t cnt = dense_band_count<T, VEC>(A, k, lo, hi, c);
    int64_t total;
    int64_t w = tile_off[tile] + block_exclusive_scan<kDenseTileCols>(cnt, total);
    if (c < k && cnt > 0)
#pragma unroll
      for (int q = 0; q < VEC; ++q)
        for (int64_t r = lo; r < hi; ++r) {
          const T a = A[r * k + c + q];
          if (a != T(0)) {
            vals[w] = a;
            rows[w] = (int32_t)r;
            cols[w] = (int32_t)(c + q);
            ++w;
          }
        }
  }
}

__global__ void dense_groups_kernel(int64_t groups, int64_t n_ct, const int64_t* __restrict__ tile_off,
                                    int64_t* __restrict__ gidx, int64_t* __restrict__ gnnz) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  gidx[g] = tile_off[g * n_ct];
  gnnz[g] = tile_off[(g + 1) * n_ct] - tile_off[g * n_ct];
}

// --------------------------------------------------------------- K4 -------
// Number of staged runs summed over groups: a position e (0-based inside its
// group's slice) starts a run iff e % b == 0 (a staging refill,
// kernels.hpp:283) or its column differs from the previous entry's (:294-296).
__global__ void run_count_kernel(int64_t nnz, int32_t p, int32_t b, int64_t groups,
                                 const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                 const int64_t* __restrict__ gidx, unsigned long long* runs) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)rows[i] / p;
    if (g < 0 || g >= groups) continue;
    const int64_t e = i - gidx[g];
    if ((e & (b - 1)) == 0 || cols[i] != cols[i - 1]) ++local;
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) local += __shfl_xor_sync(0xffffffffu, local, d);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(runs, local);
}

// Per-group run counts (for an explicit, non-permutation tile order).
__global__ void group_runs_kernel(int64_t nnz, int32_t p, int32_t b, int64_t groups,
                                  const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                  const int64_t* __restrict__ gidx, unsigned long long* runs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)rows[i] / p;
    if (g < 0 || g >= groups) continue;
    const int64_t e = i - gidx[g];
    if ((e & (b - 1)) == 0 || cols[i] != cols[i - 1]) atomicAdd(&runs[g], 1ull);
  }
}

// Stats over an explicit tile list (duplicates count twice, as in the
// reference's loop over tile_order) and coverage counts per tile.
__global__ void tile_list_kernel(int64_t count, const int64_t* __restrict__ order, int64_t col_tiles,
                                 int64_t n, int32_t b, const int64_t* __restrict__ gnnz,
                                 const unsigned long long* __restrict__ gruns, unsigned int* cover,
                                 unsigned long long* st) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = order[t];
    const int64_t g = tile / col_tiles, sj = tile % col_tiles;
    const int64_t j0 = sj * b;
    const unsigned long long w = (unsigned long long)(b < n - j0 ? b : n - j0);
    const unsigned long long cnt = (unsigned long long)gnnz[g], runs = gruns[g];
    atomicAdd(&cover[tile], 1u);
    atomicAdd(&st[0], 2ull * cnt * w);
    atomicAdd(&st[1], runs * w);
    atomicAdd(&st[2], (cnt - runs) * w);
    atomicAdd(&st[3], cnt);
  }
}

// Tiles absent from the list are never written by the reference: C stays 0.
template <typename T>
__global__ void zero_uncovered_kernel(int64_t m, int64_t n, int32_t p, int32_t b, int64_t col_tiles,
                                      const unsigned int* __restrict__ cover, T* __restrict__ C,
                                      int64_t ldc) {
  const int64_t total = m * n;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = x / n, j = x % n;
    if (!cover[(i / p) * col_tiles + j / b]) C[i * ldc + j] = T(0);
  }
}

// ------------------------------------------------- row load balancing --
// Entries per row; lanes holding the same row combine first (one atomic per
// distinct row per warp: a dense power-law row is not 16K same-address atomics).
__global__ void row_nnz_kernel(int64_t nnz, const int32_t* __restrict__ rows, int32_t* __restrict__ row_nnz) {
  griddep_wait();  // PDL: predecessor complete
  const int lane = threadIdx.x & 31;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31); base < nnz;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = base + lane;
    const bool valid = e < nnz;
    const int32_t r = valid ? rows[e] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, r);
    if (valid && lane == __ffs(same) - 1) atomicAdd(&row_nnz[r], __popc(same));
  }
}

// Planner scratch initialisation in one launch (replaces five memsets so the
// planner's kernel chain stays programmatically dependent end to end).
// `ident` (unit_of != nullptr): the placement row_balance_kernel gives an
// A whose rows are known to be even (the host's cached degree statistics):
// row r at position r, block r / rpb, dealt over the block's warps — written
// here directly, per row and per slot, so the plan skips the row count,
// histogram and placement kernels.
struct IdentPlace {
  int32_t* unit_of = nullptr;
  int32_t* skew_flag = nullptr;
  int32_t rb_rows = 0, nw = 0, rw = 0, rpb = 0;
};

__global__ void plan_init_kernel(uint32_t* __restrict__ cnt, int64_t cnt_n, int32_t* __restrict__ row_nnz,
                                 int64_t m, int32_t* __restrict__ hist, int32_t* __restrict__ cursor,
                                 int32_t* __restrict__ row_of, int64_t row_of_n, IdentPlace ident) {
  griddep_wait();  // PDL: predecessor complete
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < cnt_n; i += stride) cnt[i] = 0u;
  if (row_nnz)
    for (int64_t i = t0; i < m; i += stride) row_nnz[i] = 0;
  if (ident.unit_of) {
    if (t0 == 0) *ident.skew_flag = 0;
    for (int64_t r = t0; r < m; r += stride) {
      const int64_t blk = r / ident.rpb, j = r % ident.rpb;
      ident.unit_of[r] = (int32_t)(blk * ident.rb_rows + (j % ident.nw) * ident.rw + j / ident.nw);
    }
    for (int64_t u = t0; u < row_of_n; u += stride) {
      const int64_t blk = u / ident.rb_rows, q = u % ident.rb_rows;
      const int64_t j = (q % ident.rw) * ident.nw + q / ident.rw, r = blk * ident.rpb + j;
      row_of[u] = (j < ident.rpb && r < m) ? (int32_t)r : -1;
    }
  } else if (row_of) {
    for (int64_t i = t0; i < row_of_n; i += stride) row_of[i] = -1;
  }
  if (hist && t0 < 33) {
    hist[t0] = 0;
    cursor[t0] = 0;
  }
}

// Load-balanced placement of rows into (row block, warp, slot) units for the
// TMEM kernels: rows are ordered by log2(nnz) bucket, heaviest first (a
// counting sort; order inside a bucket is arbitrary — C does not depend on
// where a row is computed), then sorted position i goes to row block
// i / rpb, warp (i % rpb) % NW, slot (i % rpb) / NW.  Row block 0 then holds
// the heaviest rows; *skew_flag tells the multiply to launch its CTAs first.
__device__ __forceinline__ int nnz_bucket(int32_t c) { return 31 - (c > 0 ? 31 - __clz(c) : -1) - 1; }

// hist[1..32]: rows per bucket; hist[0]: the largest row.
__global__ void bucket_hist_kernel(int64_t m, const int32_t* __restrict__ row_nnz, int32_t* __restrict__ hist) {
  griddep_wait();  // PDL: predecessor complete
  __shared__ int32_t h[33];
  if (threadIdx.x < 33) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&h[nnz_bucket(row_nnz[r]) + 1], 1);
    atomicMax(&h[0], row_nnz[r]);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&hist[0], h[0]);
  if (threadIdx.x >= 1 && threadIdx.x < 33 && h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}

// Rows stay in place (identity placement) unless the largest row exceeds
// `skew` entries: uniform matrices keep their natural order.  A row block may
// hold fewer rows than the kernel's RB (`rpb` <= rb_rows): narrow column strips
// then still give the GPU enough CTAs; block b takes sorted rows
// [b*rpb, (b+1)*rpb), dealt over its warps, and its remaining slots are padding.
__global__ void row_balance_kernel(int64_t m, const int32_t* __restrict__ row_nnz, const int32_t* __restrict__ hist,
                                   int32_t* __restrict__ cursor, int32_t rb_rows, int32_t nw, int32_t rw,
                                   int32_t skew, int32_t rpb, int32_t* __restrict__ unit_of,
                                   int32_t* __restrict__ row_of, int32_t* __restrict__ skew_flag) {
  griddep_wait();  // PDL: predecessor complete
  __shared__ int32_t off[33];
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    off[0] = 0;
    for (int b = 1; b < 33; ++b) {
      off[b] = acc;
      acc += hist[b];
    }
  }
  __syncthreads();
  const bool skewed = hist[0] > skew;
  if (!skewed && rpb == rb_rows) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *skew_flag = 0;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
      unit_of[r] = (int32_t)r;
      row_of[r] = (int32_t)r;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *skew_flag = skewed ? 1 : 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = r;
    if (skewed) {
      const int b = nnz_bucket(row_nnz[r]) + 1;
      i = off[b] + atomicAdd(&cursor[b], 1);
    }
    const int64_t blk = i / rpb, j = i % rpb;
    const int64_t u = blk * rb_rows + (j % nw) * rw + j / nw;
    unit_of[r] = (int32_t)u;
    row_of[u] = (int32_t)r;
  }
}

// ------------------------------------------- two-class split (skewed A) --
// Degree statistics for the host's split decision (capi.cu skew_hint):
// out[0] the largest row, out[1+b] rows and out[34+b] entries in log2 bucket b
// (b = 0: the heaviest bucket, 31 - floor(log2(nnz)); empty rows in bucket 32).
__global__ void skew_probe_kernel(int64_t m, const int32_t* __restrict__ row_nnz, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long cnt[33], sum[33];
  __shared__ int32_t mx;
  if (threadIdx.x < 33) cnt[threadIdx.x] = sum[threadIdx.x] = 0;
  if (threadIdx.x == 0) mx = 0;
  __syncthreads();
  // a thread's rows mostly share one bucket (uniform A: all of them): count
  // runs locally and flush a run when the bucket changes
  int cur = -1;
  unsigned long long c_cnt = 0, c_sum = 0;
  int32_t my_max = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = row_nnz[r];
    const int b = nnz_bucket(c);
    if (b != cur) {
      if (c_cnt) {
        atomicAdd(&cnt[cur], c_cnt);
        atomicAdd(&sum[cur], c_sum);
      }
      cur = b;
      c_cnt = c_sum = 0;
    }
    ++c_cnt;
    c_sum += (unsigned long long)c;
    my_max = max(my_max, c);
  }
  if (c_cnt) {
    atomicAdd(&cnt[cur], c_cnt);
    atomicAdd(&sum[cur], c_sum);
  }
  my_max = __reduce_max_sync(0xffffffffu, my_max);
  if ((threadIdx.x & 31) == 0) atomicMax(&mx, my_max);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&out[0], (unsigned long long)mx);
  if (threadIdx.x < 33) {
    if (cnt[threadIdx.x]) atomicAdd(&out[1 + threadIdx.x], cnt[threadIdx.x]);
    if (sum[threadIdx.x]) atomicAdd(&out[34 + threadIdx.x], sum[threadIdx.x]);
  }
}

// Heaviest-first position of every row (log2-bucket counting sort, order
// inside a bucket arbitrary: C does not depend on where a row is computed).
__global__ void rank_rows_kernel(int64_t m, const int32_t* __restrict__ row_nnz, const int32_t* __restrict__ hist,
                                 int32_t* __restrict__ cursor, int32_t* __restrict__ pos) {
  griddep_wait();  // PDL: predecessor complete
  __shared__ int32_t off[33];
  if (threadIdx.x == 0) {
    int32_t acc = 0;
    for (int b = 1; b < 33; ++b) {
      off[b] = acc;
      acc += hist[b];
    }
  }
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int b = nnz_bucket(row_nnz[r]) + 1;
    pos[r] = off[b] + atomicAdd(&cursor[b], 1);
  }
}

// One class of a two-class split: rows at heaviest-first positions [lo, hi)
// are placed into this plan's units as row_balance_kernel does (block i/rpb,
// dealt over its warps); every other row gets unit -1 (the other plan's).
// Row block 0 holds the class's heaviest rows; `first` = 1 launches its CTAs
// first (*skew_flag), so they never start late and form a tail.
__global__ void place_class_kernel(int64_t m, const int32_t* __restrict__ pos, int64_t lo, int64_t hi,
                                   int32_t rb_rows, int32_t nw, int32_t rw, int32_t rpb,
                                   int32_t* __restrict__ unit_of, int32_t* __restrict__ row_of,
                                   int32_t* __restrict__ skew_flag, int32_t first, int32_t deal) {
  griddep_wait();  // PDL: predecessor complete
  if (blockIdx.x == 0 && threadIdx.x == 0) *skew_flag = first;
  const int64_t nblk = (hi - lo + rpb - 1) / rpb;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos[r];
    if (p < lo || p >= hi) {
      unit_of[r] = -1;
      continue;
    }
    // deal: ranked rows round-robin over the row blocks (every block as heavy
    // as the next); else consecutive ranks fill a block (the heaviest first)
    const int64_t i = p - lo, blk = deal ? i % nblk : i / rpb, j = deal ? i / nblk : i % rpb;
    const int64_t u = blk * rb_rows + (j % nw) * rw + j / nw;
    unit_of[r] = (int32_t)u;
    row_of[u] = (int32_t)r;
  }
}

}  // namespace gcoo_b200

namespace gcoo_b200 {

// ------------------------------------------------------- traffic model --
// Device evaluation of the reference's analytical traffic model
// (traffic.cpp:43-197).  Every counter of model_gcoo_traffic /
// model_csr_traffic is a closed form of four pattern statistics, gathered
// here in one pass over the GCOO arrays (capi.cu assembles the reports):
//   cnt[0] runs R: entries that start a run inside a chunk of b entries of
//          their group's (col,row)-sorted slice (traffic.cpp:81-91)
//   cnt[1] distinct columns D (first touches of (col, strip) in infinite_l2)
//   cnt[2] sum over non-empty groups of trans(3 * nnz_g)  (:101)
//   cnt[3] sum over non-empty rows of trans(2 * nnz_r)    (:170)
__global__ void traffic_entries_kernel(int64_t nnz, int32_t p, int32_t b, int64_t groups,
                                       const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                       const int64_t* __restrict__ gidx, unsigned char* __restrict__ col_flag,
                                       unsigned long long* __restrict__ cnt) {
  unsigned long long runs = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = (int64_t)rows[i] / p;
    const int32_t c = cols[i];
    col_flag[c] = 1;
    if (g < 0 || g >= groups) continue;
    const int64_t e = i - gidx[g];
    if ((e & (b - 1)) == 0 || c != cols[i - 1]) ++runs;
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) runs += __shfl_xor_sync(0xffffffffu, runs, d);
  if ((threadIdx.x & 31) == 0 && runs) atomicAdd(&cnt[0], runs);
}

// sum over i < count of [v_i > 0] * ceil(mult * v_i / 32) into *out
template <typename V>
__global__ void traffic_trans_sum_kernel(int64_t count, const V* __restrict__ v, int64_t mult,
                                         unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = (int64_t)v[i];
    if (x > 0) acc += (unsigned long long)((mult * x + 31) / 32);
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

__global__ void count_flags_kernel(int64_t count, const unsigned char* __restrict__ flag,
                                   unsigned long long* __restrict__ out) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += flag[i];
#pragma unroll
  for (int d = 16; d; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace gcoo_b200
