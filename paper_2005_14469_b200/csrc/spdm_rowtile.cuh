// spdm_rowtile.cuh — K1-general: the GCOOSpDM multiply for any (p, n, dtype).
//
// Replaces detail::spdm_gcoo_impl (kernels.hpp:240-327).  This is the
// always-applicable path (fp64, n not a multiple of 4, unaligned B/C, any p);
// the tuned fp32 paths are spdm_tacc.cuh and spdm_tile.cuh.
//
// Work decomposition (B200-first, not the reference's OpenMP tile loop):
//   * one warp owns a ROW TILE of PMAX consecutive rows x 32*V columns
//     (V = one 16-byte vector per lane), accumulators acc[PMAX][V] in
//     registers; PMAX-row tiles are unions of GCOO groups when p <= PMAX
//     (their slices are streamed back to back — different rows, so order
//     across groups is irrelevant) and sub-bands of one group when p > PMAX
//     (the warp streams the group slice and keeps only its rows);
//   * the warp stages 32 GCOO entries at a time (coalesced loads of
//     values/col_idx/row_idx), compacts the ones it owns into shared memory,
//     and reads each back as one broadcast LDS.128 (Alg. 2's "A group staged
//     in shared memory, read by broadcast");
//   * each entry loads one 16-byte vector of its B row per lane (coalesced
//     512 B per warp) and updates the accumulator row selected by the entry's
//     slot = row & (PMAX-1) through a warp-uniform switch (no local memory);
//   * the tile is written once with 16-byte stores (kernels.hpp:314-318).
// Per C element the FMAs run over the row's nonzeros in ascending column
// order, as the GCOO slice is (col,row)-sorted: bit-identical to the
// reference's sequential chain.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

namespace gcoo_b200 {

template <typename T> struct VecOf;
template <> struct VecOf<float> { static constexpr int V = 4; using type = float4; };
template <> struct VecOf<double> { static constexpr int V = 2; using type = double2; };

template <typename T, bool FMA> __device__ __forceinline__ T mac(T acc, T a, T b);
template <> __device__ __forceinline__ float mac<float, true>(float acc, float a, float b) { return __fmaf_rn(a, b, acc); }
template <> __device__ __forceinline__ float mac<float, false>(float acc, float a, float b) { return __fadd_rn(acc, __fmul_rn(a, b)); }
template <> __device__ __forceinline__ double mac<double, true>(double acc, double a, double b) { return __fma_rn(a, b, acc); }
template <> __device__ __forceinline__ double mac<double, false>(double acc, double a, double b) { return __dadd_rn(acc, __dmul_rn(a, b)); }

template <typename T>
struct alignas(16) StagedEntry {
  T val;
  int32_t col;
  int32_t slot;
};

template <typename T, int V, bool VEC>
__device__ __forceinline__ void load_b(const T* __restrict__ B, int64_t ldb, int32_t col, int64_t j0,
                                       int64_t n, T (&bv)[V]) {
  const T* src = B + (int64_t)col * ldb + j0;
  if (VEC) {
    if (j0 < n) {
      typename VecOf<T>::type x = __ldg(reinterpret_cast<const typename VecOf<T>::type*>(src));
      const T* px = reinterpret_cast<const T*>(&x);
#pragma unroll
      for (int v = 0; v < V; ++v) bv[v] = px[v];
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) bv[v] = T(0);
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) bv[v] = (j0 + v < n) ? __ldg(src + v) : T(0);
  }
}

// One accumulator row += a * B row, element-wise in column order.  fp32 FMA
// flavour: packed f32x2 FMAs (FFMA2: two independent round-to-nearest FMAs,
// the same bits) to halve the FMA issue slots.
template <typename T, int V, bool FMA>
__device__ __forceinline__ void mac_row(T (&acc)[V], T a, const T (&bv)[V]) {
  if constexpr (std::is_same<T, float>::value && FMA && V % 2 == 0) {
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int v = 0; v < V; v += 2) {
      const float2 r = __ffma2_rn(a2, make_float2(bv[v], bv[v + 1]), make_float2(acc[v], acc[v + 1]));
      acc[v] = r.x;
      acc[v + 1] = r.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = mac<T, FMA>(acc[v], a, bv[v]);
  }
}

template <typename T, int PMAX, int V, bool FMA>
__device__ __forceinline__ void accumulate(T (&acc)[PMAX][V], int slot, T a, const T (&bv)[V]) {
  // Warp-uniform switch: slot is the same in every lane, so this is one
  // indirect branch and the accumulator indices below are compile-time.
#define GCOO_CASE(s)                                                        \
  case s:                                                                   \
    if constexpr ((s) < PMAX) {                                             \
      mac_row<T, V, FMA>(acc[s], a, bv);                                     \
    }                                                                       \
    break;
  switch (slot) {
    GCOO_CASE(0) GCOO_CASE(1) GCOO_CASE(2) GCOO_CASE(3)
    GCOO_CASE(4) GCOO_CASE(5) GCOO_CASE(6) GCOO_CASE(7)
    GCOO_CASE(8) GCOO_CASE(9) GCOO_CASE(10) GCOO_CASE(11)
    GCOO_CASE(12) GCOO_CASE(13) GCOO_CASE(14) GCOO_CASE(15)
    default: break;
  }
#undef GCOO_CASE
}

constexpr int kRowTileWarps = 8;

// One warp computes row tile rt (rows [rt*PMAX, rt*PMAX + PMAX)) x column
// tile ct (32V columns).
template <typename T, int PMAX, bool VEC, bool FMA>
__device__ __forceinline__ void rowtile_warp(StagedEntry<T>* stage, int64_t rt, int64_t ct, int64_t m, int64_t k,
                                             int64_t n, int32_t p, int64_t groups, const T* __restrict__ vals,
                                             const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                             const int64_t* __restrict__ gidx, const int64_t* __restrict__ gnnz,
                                             const T* __restrict__ B, int64_t ldb, T* __restrict__ C, int64_t ldc) {
  constexpr int V = VecOf<T>::V;
  const int lane = threadIdx.x & 31;
  const int64_t r0 = rt * PMAX;
  const int64_t j0 = ct * (32 * V) + (int64_t)lane * V;

  T acc[PMAX][V];
#pragma unroll
  for (int s = 0; s < PMAX; ++s)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[s][v] = T(0);

  const bool filter = p > PMAX;
  const int64_t g_first = r0 / p;
  int64_t g_end = (r0 + PMAX + p - 1) / p;
  if (g_end > groups) g_end = groups;
  const unsigned lt_mask = (1u << lane) - 1u;

  for (int64_t g = g_first; g < g_end; ++g) {
    const int64_t lo = gidx[g], cnt = gnnz[g];
    for (int64_t base = 0; base < cnt; base += 32) {
      const bool valid = base + lane < cnt;
      T v = T(0);
      int32_t c = 0, r = 0;
      if (valid) {
        const int64_t e = lo + base + lane;
        v = vals[e];
        c = cols[e];
        r = rows[e];
      }
      // keep entries of this tile's rows whose column is addressable
      const bool mine = valid && (!filter || (r >= r0 && r < r0 + PMAX)) && (uint32_t)c < (uint64_t)k;
      const unsigned mask = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        StagedEntry<T> se;
        se.val = v;
        se.col = c;
        se.slot = r & (PMAX - 1);
        stage[__popc(mask & lt_mask)] = se;
      }
      __syncwarp();
      const int count = __popc(mask);
      int q = 0;
      // 8 independent B loads in flight per lane before their FMAs (latency-bound
      // when a tile holds a long row: one B row segment per entry from L2)
      for (; q + 8 <= count; q += 8) {
        StagedEntry<T> e[8];
        T bv[8][V];
#pragma unroll
        for (int u = 0; u < 8; ++u) e[u] = stage[q + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) load_b<T, V, VEC>(B, ldb, e[u].col, j0, n, bv[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) accumulate<T, PMAX, V, FMA>(acc, e[u].slot, e[u].val, bv[u]);
      }
      for (; q + 4 <= count; q += 4) {
        StagedEntry<T> e0 = stage[q], e1 = stage[q + 1];
        StagedEntry<T> e2 = stage[q + 2], e3 = stage[q + 3];
        T b0[V], b1[V], b2[V], b3[V];
        load_b<T, V, VEC>(B, ldb, e0.col, j0, n, b0);
        load_b<T, V, VEC>(B, ldb, e1.col, j0, n, b1);
        load_b<T, V, VEC>(B, ldb, e2.col, j0, n, b2);
        load_b<T, V, VEC>(B, ldb, e3.col, j0, n, b3);
        accumulate<T, PMAX, V, FMA>(acc, e0.slot, e0.val, b0);
        accumulate<T, PMAX, V, FMA>(acc, e1.slot, e1.val, b1);
        accumulate<T, PMAX, V, FMA>(acc, e2.slot, e2.val, b2);
        accumulate<T, PMAX, V, FMA>(acc, e3.slot, e3.val, b3);
      }
      for (; q < count; ++q) {
        StagedEntry<T> e0 = stage[q];
        T b0[V];
        load_b<T, V, VEC>(B, ldb, e0.col, j0, n, b0);
        accumulate<T, PMAX, V, FMA>(acc, e0.slot, e0.val, b0);
      }
      __syncwarp();
    }
  }

  // single write of the tile; rows past m-1 of a partial tile are not stored
#pragma unroll
  for (int s = 0; s < PMAX; ++s) {
    const int64_t row = r0 + s;
    if (row >= m) break;
    T* dst = C + row * ldc + j0;
    if (VEC) {
      if (j0 < n) {
        typename VecOf<T>::type x;
        T* px = reinterpret_cast<T*>(&x);
#pragma unroll
        for (int v = 0; v < V; ++v) px[v] = acc[s][v];
        *reinterpret_cast<typename VecOf<T>::type*>(dst) = x;
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (j0 + v < n) dst[v] = acc[s][v];
    }
  }
}

template <typename T, int PMAX, bool VEC, bool FMA>
__global__ void __launch_bounds__(kRowTileWarps * 32)
spdm_rowtile_kernel(int64_t m, int64_t k, int64_t n, int32_t p, int64_t groups,
                    const T* __restrict__ vals, const int32_t* __restrict__ rows,
                    const int32_t* __restrict__ cols, const int64_t* __restrict__ gidx,
                    const int64_t* __restrict__ gnnz, const T* __restrict__ B, int64_t ldb,
                    T* __restrict__ C, int64_t ldc, int64_t row_tiles, int64_t row_blocks) {
  static_assert(PMAX <= 16 && (PMAX & (PMAX - 1)) == 0, "PMAX must be a power of two <= 16");
  __shared__ StagedEntry<T> stage[kRowTileWarps][32];
  const int warp = threadIdx.x >> 5;
  // Row blocks vary fastest so co-resident CTAs share one B column strip
  // (k x 32V, L2-resident) and walk it in the same ascending-column order.
  const int64_t rb = blockIdx.x % row_blocks;
  const int64_t ct = blockIdx.x / row_blocks;
  const int64_t rt = rb * kRowTileWarps + warp;
  if (rt >= row_tiles) return;  // warp-uniform; no block-wide barriers
  rowtile_warp<T, PMAX, VEC, FMA>(stage[warp], rt, ct, m, k, n, p, groups, vals, rows, cols, gidx, gnnz, B, ldb, C,
                                  ldc);
}

}  // namespace gcoo_b200
