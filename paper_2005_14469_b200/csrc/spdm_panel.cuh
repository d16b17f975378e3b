// spdm_panel.cuh — K1-fast: fp32 GCOOSpDM with TMA-fed shared-memory B panels.
//
// Replaces detail::spdm_gcoo_impl (kernels.hpp:240-327) for fp32 inputs whose
// B/C rows are 16-byte aligned and p <= RW.  Design:
//
//   * The path is an FP32 FFMA gather.  Every multiply-add consumes one B
//     element that is (almost) never reused in registers at s >= 0.99, so
//     the ceiling is the rate at which B reaches the FMA units, not HBM.
//     Measured on B200 (profiles/r01_microbench.json): shared memory 128
//     B/clk/SM, L2->SM ~34 B/clk/SM, FFMA 128/clk/SM.
//   * A CTA owns a ROW BLOCK of RB = NW*RW rows x a column strip of W = 32*V
//     columns and walks K in chunks of KC rows of B.  A producer warp
//     streams B[chunk, strip] tiles into a STAGES-deep shared-memory ring
//     with TMA (cp.async.bulk.tensor.2d + mbarrier complete_tx); every staged
//     B element is read by all of the RB rows' nonzeros in its column, so
//     L2->SM traffic per FMA falls by ~RB*(1-s): the paper's "traffic moves
//     from DRAM/L2 to shared memory", done B200-style.
//   * Each consumer warp owns RW rows x W columns, acc[RW][V] in registers.
//     Its rows' nonzeros arrive as one stream laid out by the planner
//     (plan_segments_kernel): per chunk, a header of per-row counts and the
//     chunk's entries sorted by (row, col).  The warp walks row slots
//     0..RW-1 with COMPILE-TIME accumulator indices and count-driven loops
//     (no per-entry dispatch, no data-dependent exits), so independent
//     entries' LDG->LDS->FFMA chains overlap.
//   * Entries are read with warp-uniform LDG (one L1 wavefront, broadcast)
//     while the warp keeps 16 L1 lines of its stream prefetched ahead.
//   * Per C element the FMAs still run over the row's nonzeros in ascending
//     column order, one rounding each: bit-identical to the reference built
//     with FMA contraction.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace gcoo_b200 {


// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred done;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      " @!done bra WAIT_%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
template <int V>
__device__ __forceinline__ void lds_vec(uint32_t addr, float (&b)[V]) {
  if constexpr (V == 4) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(b[0]), "=f"(b[1]), "=f"(b[2]), "=f"(b[3])
                 : "r"(addr));
  } else if constexpr (V == 2) {
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(b[0]), "=f"(b[1]) : "r"(addr));
  } else {
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b[0]) : "r"(addr));
  }
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// -------------------------------------------------------- configurations --
template <int V_, int RW_, int KC_, int STAGES_, int CAP_>
struct PanelCfg {
  static constexpr int V = V_;          // floats per lane (16 B for V=4)
  static constexpr int W = 32 * V_;     // columns per CTA strip
  static constexpr int RW = RW_;        // rows per consumer warp
  static constexpr int NW = 16;         // consumer warps
  static constexpr int RB = NW * RW_;   // rows per CTA
  static constexpr int KC = KC_;        // B rows per chunk
  static constexpr int STAGES = STAGES_;
  static constexpr int THREADS = (NW + 1) * 32;
  static constexpr uint32_t CHUNK_BYTES = KC_ * W * 4;
  static constexpr int HDR = RW_ / 8;   // header entries (one count byte per row slot)
  static constexpr int CAP = CAP_;      // staged entries per warp per chunk (header included)
  static constexpr uint32_t SEG_BYTES = CAP_ * 8;
  static constexpr uint32_t STAGE_BYTES = CHUNK_BYTES + NW * SEG_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES_ * STAGE_BYTES + 2 * STAGES_ * 8 + 128;
  static_assert(CHUNK_BYTES <= 65536, "entry B offsets are 16-bit");
  static_assert(KC_ <= 255, "per-slot counts are bytes");
  static_assert(RW_ % 8 == 0 && RW_ <= 32, "header layout");
  static_assert(CAP_ % 2 == 0, "16-byte segments");
};

// <V, RW, KC, STAGES, CAP>
using PanelWide = PanelCfg<4, 16, 64, 4, 128>;   // W=128, RB=256, 48 KB stages: s ~ 0.9
using PanelK96 = PanelCfg<4, 16, 96, 4, 64>;     // W=128, RB=256, 56 KB stages
using PanelK128 = PanelCfg<4, 16, 128, 3, 64>;   // W=128, RB=256, 72 KB stages
using PanelTall = PanelCfg<2, 32, 192, 3, 128>;  // W=64,  RB=512, 64 KB stages: s >= ~0.98

// -------------------------------------------------------------- planner --
// Lays out the caller's GCOO(p) for one panel configuration.  Tile t = rows
// [t*RW, t*RW+RW) = GCOO groups [t*RW/p, (t+1)*RW/p).  Segment (t, c) holds,
// for chunk c of KC columns, a header of RW count bytes (entries of each row
// slot) followed by the tile's entries in that chunk sorted by (row, col),
// padded to 16 bytes; segments are laid out tile-major, chunk-minor, and
// seg_off[t*nchunks + c] is each one's first entry (an exclusive scan of the
// lengths counted by plan_count_kernel).  Entry = {value bits, byte offset of
// its B row inside a chunk stage}.  An entry's rank inside its chunk follows
// from the (col,row)-sorted group slices alone: #chunk entries of lower-row
// groups + #own-group chunk entries before it in (row,col) order.
constexpr int kPlanThreads = 256;

__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ cols, int64_t lo, int64_t hi,
                                                   int32_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cols[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void tile_groups(int64_t t, int RW, int32_t p, int64_t groups, int64_t& g0,
                                            int64_t& g1) {
  const int gper = RW / p;
  g0 = t * gper;
  g1 = g0 + gper < groups ? g0 + gper : groups;
  if (g0 > groups) g0 = groups;
}

// seg_len[t*nchunks + c] = round_up_even(HDR + entries of tile t in chunk c)
template <class Cfg>
__global__ void plan_count_kernel(int32_t p, int64_t groups, int64_t nnz, const int32_t* __restrict__ cols,
                                  const int64_t* __restrict__ gidx, int64_t tiles, int nchunks,
                                  int64_t* __restrict__ seg_len) {
  const int64_t total = tiles * (int64_t)nchunks;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = x / nchunks;
    const int c = (int)(x % nchunks);
    int64_t g0, g1;
    tile_groups(t, Cfg::RW, p, groups, g0, g1);
    int64_t cnt = 0;
    for (int64_t g = g0; g < g1; ++g) {
      const int64_t a = gidx[g];
      const int64_t b = g + 1 < groups ? gidx[g + 1] : nnz;
      cnt += lower_bound_col(cols, a, b, (c + 1) * Cfg::KC) - lower_bound_col(cols, a, b, c * Cfg::KC);
    }
    seg_len[x] = (Cfg::HDR + cnt + 1) & ~int64_t(1);
  }
}

// one block per tile: entries scattered to their segment slot, then headers
template <class Cfg>
__global__ void __launch_bounds__(kPlanThreads)
plan_fill_kernel(int32_t p, int64_t groups, int64_t nnz, const float* __restrict__ vals,
                 const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                 const int64_t* __restrict__ gidx, const int64_t* __restrict__ seg_off, uint2* __restrict__ out,
                 int64_t tiles, int nchunks) {
  constexpr int RW = Cfg::RW, KC = Cfg::KC, W = Cfg::W, HDR = Cfg::HDR;
  __shared__ int64_t goff[RW + 1];
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t g0, g1;
    tile_groups(t, RW, p, groups, g0, g1);
    const int ng = (int)(g1 - g0);
    __syncthreads();
    if (threadIdx.x <= ng) goff[threadIdx.x] = (g0 + threadIdx.x < groups) ? gidx[g0 + threadIdx.x] : nnz;
    __syncthreads();
    const int64_t start = goff[0], end = goff[ng];
    const int64_t row0 = t * RW;
    const int64_t* so = seg_off + t * (int64_t)nchunks;
    for (int64_t i = start + threadIdx.x; i < end; i += blockDim.x) {
      const int32_t r = rows[i], c = cols[i];
      const int ch = c / KC;
      const int own = (int)(r / p - g0);
      const int32_t lo_col = ch * KC, hi_col = lo_col + KC;
      int64_t rank = 0;
      for (int g = 0; g < own; ++g)
        rank += lower_bound_col(cols, goff[g], goff[g + 1], hi_col) - lower_bound_col(cols, goff[g], goff[g + 1], lo_col);
      for (int64_t j = lower_bound_col(cols, goff[own], goff[own + 1], lo_col); j < goff[own + 1] && cols[j] < hi_col;
           ++j) {
        const int32_t rj = rows[j];
        if (rj < r || (rj == r && cols[j] < c)) ++rank;
      }
      const uint32_t off = (uint32_t)(c - lo_col) * (uint32_t)(W * 4);
      out[so[ch] + HDR + rank] = make_uint2(__float_as_uint(vals[i]), off);
    }
    for (int ch = threadIdx.x; ch < nchunks; ch += blockDim.x) {
      const int32_t lo_col = ch * KC, hi_col = lo_col + KC;
      uint32_t words[RW / 4];
#pragma unroll
      for (int w = 0; w < RW / 4; ++w) words[w] = 0;
      for (int g = 0; g < ng; ++g) {
        for (int64_t j = lower_bound_col(cols, goff[g], goff[g + 1], lo_col); j < goff[g + 1] && cols[j] < hi_col;
             ++j) {
          const uint32_t slot = (uint32_t)(rows[j] - row0);
#pragma unroll
          for (int w = 0; w < RW / 4; ++w)
            if ((slot >> 2) == (uint32_t)w) words[w] += 1u << (8 * (slot & 3));
        }
      }
      uint2* h = out + so[ch];
#pragma unroll
      for (int q = 0; q < HDR; ++q) h[q] = make_uint2(words[2 * q], words[2 * q + 1]);
    }
  }
}

// ---------------------------------------------------------- main kernel --
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
spdm_panel_kernel(const __grid_constant__ CUtensorMap tmap_b, int64_t m, int64_t n, const uint2* __restrict__ ent,
                  const int64_t* __restrict__ seg_off, float* __restrict__ C, int64_t ldc, int64_t row_blocks,
                  int64_t col_tiles, int64_t group_rows, int64_t tiles, int nchunks) {
  constexpr int V = Cfg::V, W = Cfg::W, RW = Cfg::RW, NW = Cfg::NW, KC = Cfg::KC, S = Cfg::STAGES;
  constexpr int HDR = Cfg::HDR, CAP = Cfg::CAP;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * Cfg::STAGE_BYTES);
  uint64_t* empty = full + S;
  const uint32_t smem0 = smem_u32(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // rasterisation: bands of `group_rows` row blocks; inside a band the row
  // block varies fastest, so co-resident CTAs share a few B strips
  const int64_t band = blockIdx.x / (group_rows * col_tiles);
  const int64_t in_band = blockIdx.x % (group_rows * col_tiles);
  const int64_t band_rows = (band + 1) * group_rows <= row_blocks ? group_rows : row_blocks - band * group_rows;
  const int64_t rb = band * group_rows + in_band % band_rows;
  const int64_t ct = in_band / band_rows;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NW) {
    // ---------------- producer: per chunk, TMA B[chunk, strip] and one bulk
    // copy per consumer warp of its (header + entries) segment, all on full[s]
    const int64_t my_tile = rb * NW + lane;
    const bool has_tile = lane < NW && my_tile < tiles;
    const int64_t* so = seg_off + (has_tile ? my_tile : 0) * (int64_t)nchunks;
    int64_t s_cur = has_tile ? so[0] : 0;
    int64_t s_nxt = has_tile ? so[1] : 0;  // seg_off has tiles*nchunks+1 entries
    const int32_t x = (int32_t)(ct * W);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % S;
      const int64_t s_after = (has_tile && c + 2 <= nchunks) ? so[c + 2 < nchunks ? c + 2 : nchunks] : 0;
      int64_t len = has_tile ? s_nxt - s_cur : 0;
      if (len > CAP) len = CAP;
      uint32_t bytes = (uint32_t)len * 8u;
      uint32_t total = bytes;
#pragma unroll
      for (int d = 16; d; d >>= 1) total += __shfl_xor_sync(0xffffffffu, total, d);
      if (c >= S) mbar_wait(&empty[s], (uint32_t)((c / S) - 1) & 1u);
      const uint32_t stage = smem0 + (uint32_t)s * Cfg::STAGE_BYTES;
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], Cfg::CHUNK_BYTES + total);
        tma_load_2d(smem_raw + (size_t)s * Cfg::STAGE_BYTES, &tmap_b, x, c * KC, &full[s]);
      }
      __syncwarp();
      if (bytes) bulk_g2s(stage + Cfg::CHUNK_BYTES + lane * Cfg::SEG_BYTES, ent + s_cur, bytes, &full[s]);
      s_cur = s_nxt;
      s_nxt = s_after;
    }
    return;
  }

  // ------------------------------------------------------------- consumers
  const int64_t tile = rb * NW + warp;
  const bool active = tile < tiles;  // rows past m only take part in the ring protocol

  float acc[RW][V];
#pragma unroll
  for (int s = 0; s < RW; ++s)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[s][v] = 0.f;

  for (int c = 0; c < nchunks; ++c) {
    const int s_idx = c % S;
    mbar_wait(&full[s_idx], (uint32_t)(c / S) & 1u);
    if (active) {
      const uint32_t stage = smem0 + (uint32_t)s_idx * Cfg::STAGE_BYTES;
      const uint32_t bbase = stage + (uint32_t)(lane * V * 4);
      uint32_t eaddr = stage + Cfg::CHUNK_BYTES + (uint32_t)warp * Cfg::SEG_BYTES;
      uint32_t hdr[RW / 4];
#pragma unroll
      for (int q = 0; q < HDR; ++q) {
        const uint2 h = lds64(eaddr + q * 8);
        hdr[2 * q] = h.x;
        hdr[2 * q + 1] = h.y;
      }
      uint32_t tot = 0;
#pragma unroll
      for (int q = 0; q < RW / 4; ++q) tot += __dp4a(hdr[q], 0x01010101u, 0u);
      if (HDR + tot <= (uint32_t)CAP) {
        // fast path: the whole segment is staged
        eaddr += HDR * 8;
#pragma unroll
        for (int s = 0; s < RW; ++s) {
          const uint32_t cnt = (hdr[s >> 2] >> (8 * (s & 3))) & 0xffu;
          const uint32_t e_end = eaddr + cnt * 8;
#pragma unroll 2
          for (; eaddr < e_end; eaddr += 8) {
            const uint2 e = lds64(eaddr);
#ifdef GCOO_DEBUG_PANEL
            if (e.y % (W * 4) != 0 || e.y >= Cfg::CHUNK_BYTES) {
              if (lane == 0)
                printf("BAD blk=%d warp=%d c=%d slot=%d tot=%u hdr0=%08x hdr1=%08x idx=%u e=(%08x,%08x)\n",
                       (int)blockIdx.x, warp, c, s, tot, hdr[0], hdr[1],
                       (eaddr - (stage + Cfg::CHUNK_BYTES + (uint32_t)warp * Cfg::SEG_BYTES)) / 8, e.x, e.y);
              __trap();
            }
#endif
            float bv[V];
            lds_vec<V>(bbase + e.y, bv);
            const float a = __uint_as_float(e.x);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[s][v] = __fmaf_rn(a, bv[v], acc[s][v]);
          }
        }
      } else {
        // overflow (very dense rows): entries past CAP come from global memory
        const uint2* g = ent + seg_off[tile * (int64_t)nchunks + c];
        uint32_t idx = HDR;
#pragma unroll
        for (int s = 0; s < RW; ++s) {
          const uint32_t cnt = (hdr[s >> 2] >> (8 * (s & 3))) & 0xffu;
          for (uint32_t i = 0; i < cnt; ++i, ++idx) {
            const uint2 e = idx < (uint32_t)CAP ? lds64(eaddr + idx * 8) : __ldg(g + idx);
            float bv[V];
            lds_vec<V>(bbase + e.y, bv);
            const float a = __uint_as_float(e.x);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[s][v] = __fmaf_rn(a, bv[v], acc[s][v]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s_idx]);
  }

  // single write of the tile
  if (!active) return;
  const int64_t row0 = tile * RW;
  const int64_t j = ct * W + lane * V;
  if (j < n) {
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      const int64_t row = row0 + s;
      if (row < m) {
        float* dst = C + row * ldc + j;
        if constexpr (V == 4) {
          *reinterpret_cast<float4*>(dst) = make_float4(acc[s][0], acc[s][1], acc[s][2], acc[s][3]);
        } else if constexpr (V == 2) {
          *reinterpret_cast<float2*>(dst) = make_float2(acc[s][0], acc[s][1]);
        } else {
          dst[0] = acc[s][0];
        }
      }
    }
  }
}

}  // namespace gcoo_b200
