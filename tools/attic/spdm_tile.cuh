// spdm_tile.cuh — K1-fast: fp32 GCOOSpDM with warp row sets, a TMA-fed
// shared-memory B ring and a packed, slot-major per-chunk record stream.
//
// Replaces detail::spdm_gcoo_impl (kernels.hpp:240-327) for fp32 inputs whose
// B/C rows are 16-byte aligned.  Why this shape (ceilings
// measured in profiles/r01_microbench*.json):
//
//   * Every multiply-add needs one element of B that (at s >= 0.99) is almost
//     never reused from registers, so the kernel is bound by how fast B
//     reaches the FMA units: shared memory delivers 128 B/clk/SM = 32 FMA/clk
//     against 128 FFMA/clk.  An entry (value, B row) is read by all 32 lanes
//     with one broadcast wavefront; its B row segment is one vector load per
//     lane.
//   * A CTA stages B[chunk of KC rows, strip of W columns] once per chunk and
//     every one of its RB rows' nonzeros in that chunk reads it, so L2->SM
//     bytes per FMA are 4 / (RB * density); with ~29 B/clk/SM of L2 delivery
//     RB must be large.  Registers bound RB * W (64 accumulators per lane), so
//     the strip narrows as the matrix gets sparser: a warp owns RW = 64/V rows
//     x W = 32*V columns (V floats per lane), RB = 15 warps x RW.
//     V=4: W=128, RB=240; V=2: W=64, RB=480; V=1: W=32, RB=960.
//   * Records: per (warp, chunk) the warp's entries are grouped by row slot
//     and packed two to a 16-byte record {v0, v1, off0, off1} (off = byte
//     offset of the B row in the stage; 0xFFFFFFFF = absent, an odd count's
//     padding).  The slot loop is unrolled, so every accumulator index is a
//     compile-time register; no per-entry dispatch, no local memory.
//   * Producer warp: per chunk one 2-D TMA of the B tile and one 1-D bulk copy
//     of the CTA's record segment into a STAGES-deep ring (mbarrier
//     complete_tx); consumers release a stage with one arrive per warp.
//   * The record stream is built on the device from the GCOO arrays by the
//     planner kernels below (no host synchronisation).
//
// Per C element the FMAs run over the row's nonzeros in ascending column
// order (chunks in order, a (row, chunk)'s entries in column order), one
// rounding each: bit-identical to the reference built with FMA contraction.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

#include "ptx.cuh"

namespace gcoo_b200 {

template <int V_, int KC_, int STAGES_, int CAP_>
struct TileCfg {
  static constexpr int V = V_;             // floats per lane
  static constexpr int W = 32 * V_;        // columns per CTA strip
  static constexpr int RW = 64 / V_;       // rows (slots) per warp
  static constexpr int NW = 15;            // consumer warps (+1 producer = 4 warps per SMSP, 128 regs)
  static constexpr int RB = NW * RW;       // rows per CTA
  static constexpr int KC = KC_;           // B rows per chunk
  static constexpr int STAGES = STAGES_;
  static constexpr int THREADS = (NW + 1) * 32;
  static constexpr uint32_t BTILE = (uint32_t)KC_ * W * 4;
  static constexpr uint32_t CAP = CAP_;    // record-segment bytes per stage
  static constexpr uint32_t STAGE_BYTES = BTILE + CAP_;
  static constexpr int HDR = RW;           // per-warp header: record count per slot (bytes)
  static constexpr int REC = 16;           // bytes per record
  static constexpr int TABLE = 64;         // per-segment warp offset table (16 x u32)
  static constexpr size_t SMEM = (size_t)STAGES_ * STAGE_BYTES + 2 * STAGES_ * 8;
  static_assert(KC_ <= 256, "TMA box rows");
  static_assert((KC_ + 1) / 2 <= 255, "per-slot record counts are bytes");
  static_assert(CAP_ % 16 == 0 && BTILE % 16 == 0 && HDR % 16 == 0, "16-byte stages");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

//                      V  KC   S  CAP
using TileV4 = TileCfg<4, 48, 5, 16384>;    // W=128, RB=240 : density >~ 3%

// ---------------------------------------------------------------- planner --
// P1: per (unit u = row / RW, chunk, slot = row % RW) entry counts.
template <class Cfg>
__global__ void tile_count_kernel(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                  int nchunks, uint32_t* __restrict__ cnt) {
  griddep_wait();  // PDL: predecessor complete
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[e];
    const int32_t c = cols[e] / Cfg::KC;
    atomicAdd(&cnt[((int64_t)(r / Cfg::RW) * nchunks + c) * Cfg::RW + (r % Cfg::RW)], 1u);
  }
}

template <class Cfg>
__device__ __forceinline__ uint32_t tile_warp_records(const uint32_t* __restrict__ cnt, int64_t units, int nchunks,
                                                      int64_t u, int c) {
  if (u >= units) return 0u;
  const uint32_t* p = cnt + (u * nchunks + c) * Cfg::RW;
  uint32_t r = 0;
#pragma unroll 8
  for (int s = 0; s < Cfg::RW; ++s) r += (p[s] + 1) >> 1;
  return r;
}

// P2: one warp per (rb, c): segment length (table + warp segments).
template <class Cfg>
__global__ void tile_size_kernel(const uint32_t* __restrict__ cnt, int64_t units, int nchunks, int64_t nseg,
                                 int64_t* __restrict__ seg_len) {
  griddep_wait();  // PDL: predecessor complete
  const int lane = threadIdx.x & 31;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < nseg;
       x += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t rb = x / nchunks;
    const int c = (int)(x % nchunks);
    uint32_t sz = lane < Cfg::NW
                      ? Cfg::HDR + Cfg::REC * tile_warp_records<Cfg>(cnt, units, nchunks, rb * Cfg::NW + lane, c)
                      : 0u;
#pragma unroll
    for (int d = 16; d; d >>= 1) sz += __shfl_xor_sync(0xffffffffu, sz, d);
    if (lane == 0) seg_len[x] = Cfg::TABLE + sz;
  }
}

// P4: one warp per (rb, c): warp offset table, per-warp headers, padding
// records pre-filled as absent, and the stream position of every (warp,
// slot) record run for the scatter.
template <class Cfg>
__global__ void tile_header_kernel(const uint32_t* __restrict__ cnt, int64_t units, int nchunks, int64_t nseg,
                                   const int64_t* __restrict__ seg_off, unsigned char* __restrict__ ent,
                                   int64_t* __restrict__ slot_pos) {
  griddep_wait();  // PDL: predecessor complete
  const int lane = threadIdx.x & 31;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < nseg;
       x += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t rb = x / nchunks;
    const int c = (int)(x % nchunks);
    const int64_t u = rb * Cfg::NW + lane;
    const uint32_t nrec = lane < Cfg::NW ? tile_warp_records<Cfg>(cnt, units, nchunks, u, c) : 0u;
    const uint32_t sz = lane < Cfg::NW ? Cfg::HDR + Cfg::REC * nrec : 0u;
    uint32_t incl = sz;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane < Cfg::NW) {
      const uint32_t woff = Cfg::TABLE + incl - sz;
      unsigned char* seg = ent + seg_off[x];
      reinterpret_cast<uint32_t*>(seg)[lane] = woff;
      int64_t pos = seg_off[x] + woff + Cfg::HDR;
      int64_t* sp = slot_pos + (x * Cfg::NW + lane) * Cfg::RW;
      const uint32_t* p = cnt + (u * nchunks + c) * Cfg::RW;
      for (int s0 = 0; s0 < Cfg::RW; s0 += 4) {
        uint32_t word = 0;
        for (int s = s0; s < s0 + 4; ++s) {
          const uint32_t ns = u < units ? (p[s] + 1) >> 1 : 0u;
          word |= ns << (8 * (s - s0));
          sp[s] = pos;
          uint4* rec = reinterpret_cast<uint4*>(ent + pos);
          for (uint32_t j = 0; j < ns; ++j) rec[j] = make_uint4(0u, 0u, ~0u, ~0u);
          pos += (int64_t)Cfg::REC * ns;
        }
        reinterpret_cast<uint32_t*>(seg + woff)[s0 / 4] = word;
      }
    }
  }
}

// P5: scatter every entry into its record.  Its rank among its row's entries
// in the same chunk comes from the (col,row)-sorted group slice: the entries
// of the chunk are contiguous there, so count same-row ones before it.
template <class Cfg>
__global__ void tile_fill_kernel(int64_t nnz, int32_t p, const float* __restrict__ vals,
                                 const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                 const int64_t* __restrict__ gidx, int nchunks,
                                 const int64_t* __restrict__ slot_pos, unsigned char* __restrict__ ent) {
  griddep_wait();  // PDL: predecessor complete
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[e], col = cols[e];
    const int c = col / Cfg::KC;
    const int32_t lo_col = c * Cfg::KC;
    const int64_t glo = gidx[r / p];
    uint32_t rank = 0;
    for (int64_t j = e - 1; j >= glo; --j) {
      if (cols[j] < lo_col) break;
      rank += rows[j] == r;
    }
    const int64_t u = r / Cfg::RW;
    const int64_t rb = u / Cfg::NW;
    const int w = (int)(u % Cfg::NW);
    const int64_t base = slot_pos[((rb * nchunks + c) * Cfg::NW + w) * Cfg::RW + (r % Cfg::RW)];
    uint32_t* word = reinterpret_cast<uint32_t*>(ent + base + (int64_t)Cfg::REC * (rank >> 1));
    word[rank & 1] = __float_as_uint(vals[e]);
    word[2 + (rank & 1)] = (uint32_t)(col - lo_col) * (uint32_t)(Cfg::W * 4);
  }
}

// ---------------------------------------------------------- main kernel --
template <bool GLOBAL>
struct EntrySrc;
template <>
struct EntrySrc<false> {  // staged in shared memory
  using addr_t = uint32_t;
  static __device__ __forceinline__ uint4 ld(addr_t a) { return lds128u(a); }
  static __device__ __forceinline__ uint32_t ld32(addr_t a) { return lds32u(a); }
};
template <>
struct EntrySrc<true> {  // segment larger than a stage: read from global memory
  using addr_t = const unsigned char*;
  static __device__ __forceinline__ uint4 ld(addr_t a) { return __ldg(reinterpret_cast<const uint4*>(a)); }
  static __device__ __forceinline__ uint32_t ld32(addr_t a) { return __ldg(reinterpret_cast<const uint32_t*>(a)); }
};

// One warp walks its records for one chunk, slot by slot.
template <class Cfg, bool GLOBAL>
__device__ __forceinline__ void tile_consume(float (&acc)[Cfg::RW][Cfg::V], typename EntrySrc<GLOBAL>::addr_t seg,
                                             int warp, uint32_t bbase) {
  using Src = EntrySrc<GLOBAL>;
  constexpr int V = Cfg::V;
  const uint32_t woff = Src::ld32(seg + 4 * warp);
  const auto wseg = seg + woff;
  auto rec = wseg + Cfg::HDR;
#pragma unroll
  for (int s0 = 0; s0 < Cfg::RW; s0 += 16) {
    const uint4 np4 = Src::ld(wseg + s0);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const uint32_t w = s < 4 ? np4.x : s < 8 ? np4.y : s < 12 ? np4.z : np4.w;
      const uint32_t n = (w >> (8 * (s & 3))) & 0xffu;
#pragma unroll 2
      for (uint32_t i = 0; i < n; ++i) {
        const uint4 q = Src::ld(rec);
        rec += Cfg::REC;
        {  // the first entry of a record is always present
          float b[V];
          lds_vec<V>(bbase + q.z, b);
          const float a = __uint_as_float(q.x);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[s0 + s][v] = __fmaf_rn(a, b[v], acc[s0 + s][v]);
        }
        if (q.w != ~0u) {
          float b[V];
          lds_vec<V>(bbase + q.w, b);
          const float a = __uint_as_float(q.y);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[s0 + s][v] = __fmaf_rn(a, b[v], acc[s0 + s][v]);
        }
      }
    }
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
spdm_tile_kernel(const __grid_constant__ CUtensorMap tmap_b, int64_t m, int64_t n, const unsigned char* __restrict__ ent,
                 const int64_t* __restrict__ seg_off, float* __restrict__ C, int64_t ldc, int64_t row_blocks,
                 int nchunks) {
  constexpr int W = Cfg::W, NW = Cfg::NW, S = Cfg::STAGES, V = Cfg::V, RW = Cfg::RW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * Cfg::STAGE_BYTES);
  uint64_t* empty = full + S;
  const uint32_t smem0 = smem_u32(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rb = blockIdx.x % row_blocks;  // row blocks fastest: co-resident CTAs share a B strip
  const int64_t ct = blockIdx.x / row_blocks;
  const int64_t* so = seg_off + rb * nchunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_wait();  // PDL: the planner's record stream is complete

  if (warp == NW) {
    // ------------- producer: B tile (TMA 2-D) + record segment (bulk 1-D)
    if (lane == 0) {
      const int32_t x = (int32_t)(ct * W);
      int64_t lo = so[0], hi = so[1];
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % S;
        const int64_t hi_next = so[c + 2 <= nchunks ? c + 2 : nchunks];  // prefetch
        const uint32_t len = (uint32_t)(hi - lo);
        const uint32_t bytes = len <= Cfg::CAP ? len : 0u;  // oversize: consumers read global memory
        if (c >= S) mbar_wait(&empty[s], (uint32_t)((c / S) - 1) & 1u);
        unsigned char* stage = smem_raw + (size_t)s * Cfg::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], Cfg::BTILE + bytes);
        tma_load_2d(stage, &tmap_b, x, c * Cfg::KC, &full[s]);
        if (bytes) bulk_g2s(smem_u32(stage + Cfg::BTILE), ent + lo, bytes, &full[s]);
        lo = hi;
        hi = hi_next;
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  float acc[RW][V];
#pragma unroll
  for (int s = 0; s < RW; ++s)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[s][v] = 0.f;

  int64_t lo = so[0], hi = so[1];
  for (int c = 0; c < nchunks; ++c) {
    const int s_idx = c % S;
    const int64_t hi_next = so[c + 2 <= nchunks ? c + 2 : nchunks];  // prefetch
    mbar_wait(&full[s_idx], (uint32_t)(c / S) & 1u);
    const uint32_t stage = smem0 + (uint32_t)s_idx * Cfg::STAGE_BYTES;
    const uint32_t bbase = stage + (uint32_t)(lane * V * 4);
    if (hi - lo <= (int64_t)Cfg::CAP) {
      tile_consume<Cfg, false>(acc, stage + Cfg::BTILE, warp, bbase);
    } else {
      tile_consume<Cfg, true>(acc, ent + lo, warp, bbase);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s_idx]);
    lo = hi;
    hi = hi_next;
  }

  // single write of the tile
  const int64_t row0 = (rb * NW + warp) * (int64_t)RW;
  const int64_t j = ct * W + lane * V;
  if (j < n) {
#pragma unroll
    for (int s = 0; s < RW; ++s) {
      const int64_t row = row0 + s;
      if (row < m) {
        float* dst = C + row * ldc + j;
        if constexpr (V == 4) {
          __stcs(reinterpret_cast<float4*>(dst), make_float4(acc[s][0], acc[s][1], acc[s][2], acc[s][3]));
        } else if constexpr (V == 2) {
          __stcs(reinterpret_cast<float2*>(dst), make_float2(acc[s][0], acc[s][1]));
        } else {
          __stcs(dst, acc[s][0]);
        }
      }
    }
  }
}

}  // namespace gcoo_b200
