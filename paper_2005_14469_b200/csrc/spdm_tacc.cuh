// spdm_tacc.cuh — K1-fast: fp32 GCOOSpDM with the accumulators in TENSOR
// MEMORY, a TMA-fed shared-memory B ring and a flat slot-major record stream.
//
// Replaces detail::spdm_gcoo_impl (kernels.hpp:240-327) for fp32 inputs whose
// B/C rows are 16-byte aligned.  Design (ceilings measured in
// profiles/r01_microbench*.json):
//
//   * The path is bound by how fast B reaches the FMA units: each
//     multiply-add needs one B element, almost never reused from registers at
//     s >= 0.99.  Shared memory delivers 128 B/clk/SM (32 FMA/clk); an entry
//     is broadcast to the warp with one wavefront and its B row segment is one
//     vector LDS per lane.
//   * A CTA stages B[chunk of KC rows, strip of W = 32*V columns] once per
//     chunk and all its RB rows' nonzeros in the chunk read it, so the L2->SM
//     bytes per FMA are 4 / (RB * density): RB must be large.  Register-held
//     accumulators cap RB*W at ~30K; here they live in TMEM (128 lanes x 512
//     columns = 64K fp32 per SM), so RB doubles: NW consumer warps (16, 24 or
//     28), warp w owns TMEM lane quadrant w%4 and TCOLS = 512/(NW/4) columns
//     = RW = TCOLS/V rows x V columns per lane.  V=4, 28 warps: W=128, RB=504
//     (the default); 16 warps: RB=512; V=2: W=64, RB=1024.
//   * A warp walks its chunk's entries in one flat loop: a 16-byte record
//     carries two consecutive entries of the warp's slot-major stream
//     {v0, v1, off0 | slot0 << 24, off1 | slot1 << 24} (denser
//     configurations: three entries of one slot).  The
//     slot's V accumulators are pulled into registers from TMEM
//     (tcgen05.ld.32x32b) when the slot changes and pushed back
//     (tcgen05.st) when it is left: one ld/st pair per visited (slot, chunk),
//     no per-slot control flow for empty slots and no register-indexed
//     accumulator arrays.
//   * Producer warp: per chunk one 2-D TMA of the B tile and one 1-D bulk copy
//     of the CTA's record segment into a STAGES-deep ring (mbarrier
//     complete_tx); consumers release a stage with one arrive per warp.  The
//     chunk depth KC is matched to the density so that a chunk's records fit
//     the stage (choose_kind in capi.cu).
//   * Tiles (row block x column strip) are walked in launch order by
//     persistent CTAs (one per SM) for even A: the ring runs across tile
//     boundaries, so the next tile's first stages load while the consumers
//     write the previous tile back from TMEM; skewed A launches one CTA per
//     tile and lets the hardware balance them.
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

__device__ __forceinline__ int64_t ceil_div_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

template <int V_, int KC_, int STAGES_, int CAP_, int NW_ = 16, int EPR_ = 2, class E_ = float>
struct TaccCfg {
  using E = E_;                            // element type (float; double: two 32-bit cells)
  static constexpr int V = V_;             // 32-bit cells per lane (= floats per lane)
  static constexpr int VE = V_ * 4 / (int)sizeof(E_);  // elements per lane
  static constexpr int W = 32 * VE;        // columns (elements) per CTA strip
  static constexpr int NW = NW_;           // consumer warps: NW/4 per TMEM lane quadrant
  static constexpr int TCOLS = (512 / (NW_ / 4)) & ~7;  // TMEM columns per warp (128 / 80 / 72 for 16 / 24 / 28 warps)
  static constexpr int RW = TCOLS / V_;    // rows (slots) per warp
  static constexpr int RB = NW * RW;       // rows per CTA
  static constexpr int KC = KC_;           // B rows per chunk
  static constexpr int STAGES = STAGES_;
  static constexpr int THREADS = (NW + 1) * 32;
  static constexpr uint32_t ROWB = (uint32_t)W * sizeof(E_);  // bytes of one staged B row
  static constexpr uint32_t BTILE = (uint32_t)KC_ * ROWB;
  static constexpr uint32_t CAP = CAP_;    // record-segment bytes per stage
  static constexpr uint32_t STAGE_BYTES = BTILE + CAP_;
  static constexpr int HDR = 16;           // per-warp header: record count
  static constexpr int REC = 16;           // bytes per record
  // entries per record: 2 = {v0, v1, off0 | slot0<<24, off1 | slot1<<24} (B byte offsets; any two
  //   consecutive entries of the warp's stream, header = entry count);
  // 3 = {v0, v1, v2, r0 | r1<<8 | r2<<16 | slot<<24} (B row indices in the chunk, 0xFF = absent);
  // 1 (double) = {lo(v), hi(v), off | slot<<24, 0}
  static constexpr int EPR = EPR_;
  static_assert((sizeof(E_) == 4 && (EPR_ == 2 || (EPR_ == 3 && KC_ < 255))) || (sizeof(E_) == 8 && EPR_ == 1),
                "record format");
  static constexpr int TABLE = (4 * NW_ + 15) & ~15;  // per-segment warp offset table (NW x u32)
  // Segment extents from the entry count n alone (two-entry and fp64
  // records): extent(n) bounds table + headers + records (a warp's dense pair
  // stream wastes at most half a record) and keeps 16-byte alignment, so the
  // offsets are a scan of per-segment counts; a segment holds entries iff its
  // extent exceeds EXT_BASE.  Three-entry records keep exact lengths.
  static constexpr bool LINEAR_EXTENT = EPR_ != 3;
  static constexpr uint32_t EXT_BASE = (uint32_t)TABLE + (uint32_t)NW_ * HDR + (EPR_ == 2 ? 8u * NW_ : 0u);
  static __host__ __device__ constexpr int64_t extent(int64_t n) {
    return (int64_t)EXT_BASE + (EPR_ == 2 ? 16 * ((n + 1) / 2) : 16 * n);
  }
  // stages + full/empty barriers + TMEM address slot + per-stage segment offsets (int64) and lengths
  static constexpr size_t SMEM = (size_t)STAGES_ * STAGE_BYTES + 2 * STAGES_ * 8 + 16 + STAGES_ * 16;
  static_assert(KC_ <= 256, "TMA box rows");
  static_assert(NW_ % 4 == 0 && NW_ <= 28 && TCOLS % 8 == 0 && 8 % V_ == 0, "warps tile the 4 TMEM lane quadrants");
  static_assert(BTILE < (1u << 24) && RW <= 256, "24-bit B offsets, 8-bit slots");
  static_assert(CAP_ % 16 == 0 && BTILE % 16 == 0, "16-byte stages");
  static_assert(SMEM <= 227 * 1024 && SMEM > 116 * 1024, "one CTA per SM (it owns all 512 TMEM columns)");
};

//                      V  KC   S  CAP
// 28 consumer warps (RB=504): the chunk depth KC trades run length (swaps per
// entry) against the record-stage capacity, which must hold a row block's
// records for one chunk (an oversize segment is read from global memory):
// denser matrices take shallower chunks and bigger record stages.
using Tacc28K192 = TaccCfg<4, 192, 2, 16384, 28>;     // density 1.1 % .. 1.7 %
// the denser configurations pack three entries per record (long runs fill
// them; 3-10 % faster), the sparsest two (pairs of records in flight matter
// more there)
using Tacc28K160 = TaccCfg<4, 160, 2, 32768, 28, 3>;  // 3.5 %   .. 6 %
using Tacc28K128 = TaccCfg<4, 128, 2, 49152, 28, 3>;  //         .. 12 %
using Tacc28K96 = TaccCfg<4, 96, 2, 65536, 28, 3>;    //         .. 30 %
using Tacc28K64 = TaccCfg<4, 64, 2, 81920, 28, 3>;    //      >= 30 %
// Deeper chunks (fewer TMEM swaps per entry) where a smaller record stage still
// holds a chunk's records: density 0.35 % .. 1.1 % (28 warps) and < 0.22 % (16 warps)
using Tacc28K200 = TaccCfg<4, 200, 2, 12288, 28>;
using Tacc28K176 = TaccCfg<4, 176, 2, 24576, 28, 3>;  // three-entry records, density 1.7 % .. 3.5 %
using TaccV4K216 = TaccCfg<4, 216, 2, 4096>;
// fp64 (the reference's GCOO_SCALAR_F64 build): 64 doubles per CTA strip,
// 504 rows, one entry per 16-byte record
using Tacc28F64K160 = TaccCfg<4, 160, 2, 32768, 28, 1, double>;  // density < 2.5 %
using Tacc28F64K96 = TaccCfg<4, 96, 2, 65536, 28, 1, double>;    //         < 7 %
using Tacc28F64K64 = TaccCfg<4, 64, 2, 81920, 28, 1, double>;    //         >= 7 %

// ---------------------------------------------------------------- planner --
// P1: per (unit u = row / RW, chunk, slot = row % RW) entry counts.
// Rows are placed into (row block, warp, slot) by `unit_of` (see
// row_balance_kernel): heaviest rows first, dealt round-robin over a row
// block's warps, so warps carry similar loads on skewed (power-law) matrices.
template <class Cfg>
__global__ void tacc_count_kernel(int64_t nnz, const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                  int nchunks, uint32_t* __restrict__ cnt, const int32_t* __restrict__ unit_of) {
  griddep_wait();  // PDL: predecessor complete
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = unit_of[rows[e]];
    if (r < 0) continue;  // row of another class's plan (two-class split)
    const int32_t c = cols[e] / Cfg::KC;
    atomicAdd(&cnt[((int64_t)(r / Cfg::RW) * nchunks + c) * Cfg::RW + (r % Cfg::RW)], 1u);
  }
}

template <class Cfg>
__device__ __forceinline__ uint32_t tacc_warp_records(const uint32_t* __restrict__ cnt, int64_t units, int nchunks,
                                                      int64_t u, int c) {
  if (u >= units) return 0u;
  const uint32_t* p = cnt + (u * nchunks + c) * Cfg::RW;
  uint32_t r = 0;
  if constexpr (Cfg::EPR == 2) {  // dense pairs: any two consecutive entries of the warp's stream
#pragma unroll 8
    for (int s = 0; s < Cfg::RW; ++s) r += p[s];
    return (r + 1) / 2;
  } else {
#pragma unroll 8
    for (int s = 0; s < Cfg::RW; ++s) r += (p[s] + Cfg::EPR - 1) / Cfg::EPR;
    return r;
  }
}

// P2: one warp per (rb, c): segment length (table + warp segments) and each
// warp segment's offset inside the segment.
template <class Cfg>
__global__ void tacc_size_kernel(const uint32_t* __restrict__ cnt, int64_t units, int nchunks, int64_t nseg,
                                 int64_t* __restrict__ seg_len, uint32_t* __restrict__ woff) {
  griddep_wait();  // PDL: predecessor complete
  const int lane = threadIdx.x & 31;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < nseg;
       x += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t rb = x / nchunks;
    const int c = (int)(x % nchunks);
    const uint32_t sz = lane < Cfg::NW
                            ? Cfg::HDR + Cfg::REC * tacc_warp_records<Cfg>(cnt, units, nchunks, rb * Cfg::NW + lane, c)
                            : 0u;
    uint32_t incl = sz;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane < Cfg::NW) woff[x * Cfg::NW + lane] = Cfg::TABLE + incl - sz;
    if constexpr (Cfg::LINEAR_EXTENT) {  // the extent from the segment's entry count
      uint32_t ne = 0;
      if (lane < Cfg::NW && rb * Cfg::NW + lane < units) {
        const uint32_t* pc = cnt + ((rb * Cfg::NW + lane) * nchunks + c) * Cfg::RW;
        for (int q = 0; q < Cfg::RW; ++q) ne += pc[q];
      }
#pragma unroll
      for (int d = 16; d >= 1; d >>= 1) ne += __shfl_xor_sync(0xffffffffu, ne, d);
      if (lane == 31) seg_len[x] = Cfg::extent(ne);
    } else {
      if (lane == 31) seg_len[x] = Cfg::TABLE + incl;
    }
  }
}

// P4: one thread per (segment, warp, slot): the stream position of the slot's
// entries (for the scatter); the slot-0 thread also writes the warp's
// offset-table entry and its header.  EPR 2: the warp's entries form one
// dense stream of pairs (slot-major, column order), `slot_pos` = the entry
// index of the slot's first entry counted in 8-byte halves of the stream
// (stream start / 8 + entries before), no absent marks; header {entries}.
// EPR 1/3: records per slot run, absent entries marked; header {records}.
template <class Cfg>
__global__ void tacc_header_kernel(const uint32_t* __restrict__ cnt, int64_t units, int nchunks, int64_t nseg,
                                   const int64_t* __restrict__ seg_off, const uint32_t* __restrict__ woff,
                                   unsigned char* __restrict__ ent, int64_t* __restrict__ slot_pos) {
  griddep_wait();  // PDL: predecessor complete
  const int64_t total = nseg * Cfg::NW * Cfg::RW;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t % Cfg::RW);
    const int64_t xw = t / Cfg::RW;  // segment * NW + warp
    const int w = (int)(xw % Cfg::NW);
    const int64_t x = xw / Cfg::NW;
    const int64_t rb = x / nchunks;
    const int c = (int)(x % nchunks);
    const int64_t u = rb * Cfg::NW + w;
    const uint32_t* p = cnt + (u * nchunks + c) * Cfg::RW;
    const uint32_t wo = woff[xw];
    const int64_t start = seg_off[x] + wo + Cfg::HDR;  // 16-byte aligned
    if constexpr (Cfg::EPR == 2) {
      uint32_t before = 0;
      if (u < units)
        for (int q = 0; q < s; ++q) before += p[q];
      slot_pos[t] = start / 8 + before;
      if (s == 0) {
        uint32_t nent = 0;
        if (u < units)
          for (int q = 0; q < Cfg::RW; ++q) nent += p[q];
        unsigned char* seg = ent + seg_off[x];
        reinterpret_cast<uint32_t*>(seg)[w] = wo;
        *reinterpret_cast<uint4*>(seg + wo) = make_uint4(nent, 0u, 0u, 0u);
      }
    } else {
      uint32_t before = 0;
      if (u < units)
        for (int q = 0; q < s; ++q) before += (p[q] + Cfg::EPR - 1) / Cfg::EPR;
      const uint32_t ns = u < units ? (p[s] + Cfg::EPR - 1) / Cfg::EPR : 0u;
      const int64_t pos = start + (int64_t)Cfg::REC * before;
      slot_pos[t] = pos;
      uint32_t* rec = reinterpret_cast<uint32_t*>(ent + pos);
      // absent-entry marks, overwritten by the entries that exist
      const uint32_t mark = Cfg::EPR == 3 ? 0x00FFFFFFu | ((uint32_t)s << 24) : 0u;
      for (uint32_t j = 0; j < ns; ++j) rec[4 * j + 3] = mark;
      if (s == 0) {
        uint32_t nrec = 0;
        if (u < units)
          for (int q = 0; q < Cfg::RW; ++q) nrec += (p[q] + Cfg::EPR - 1) / Cfg::EPR;
        unsigned char* seg = ent + seg_off[x];
        reinterpret_cast<uint32_t*>(seg)[w] = wo;
        *reinterpret_cast<uint4*>(seg + wo) = make_uint4(nrec, 0u, 0u, 0u);
      }
    }
  }
}

// P5: scatter every entry into its record.  Its rank among its row's entries
// in the same chunk comes from the (col,row)-sorted group slice: the entries
// of the chunk are contiguous there, so count same-row ones before it.
template <class Cfg>
__global__ void tacc_fill_kernel(int64_t nnz, int32_t p, const typename Cfg::E* __restrict__ vals,
                                 const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                 const int64_t* __restrict__ gidx, int nchunks,
                                 const int64_t* __restrict__ slot_pos, unsigned char* __restrict__ ent,
                                 const int32_t* __restrict__ unit_of) {
  griddep_wait();  // PDL: predecessor complete
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[e], col = cols[e];
    const int32_t ur = unit_of[r];
    if (ur < 0) continue;  // row of another class's plan (two-class split)
    const int c = col / Cfg::KC;
    const int32_t lo_col = c * Cfg::KC;
    const int64_t glo = gidx[r / p];
    // the chunk's range in the group slice starts at the first column >= lo_col
    // (columns ascend along the slice): binary search, then count the row's
    // entries before e, four at a time where rows is 16-byte aligned
    int64_t a = glo, b = e;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (cols[mid] < lo_col) a = mid + 1; else b = mid;
    }
    uint32_t rank = 0;
    int64_t j = a;
    if ((reinterpret_cast<uintptr_t>(rows) & 15) == 0) {
      for (; j < e && (j & 3); ++j) rank += rows[j] == r;
      for (; j + 4 <= e; j += 4) {
        const int4 q = __ldg(reinterpret_cast<const int4*>(rows + j));
        rank += (q.x == r) + (q.y == r) + (q.z == r) + (q.w == r);
      }
    }
    for (; j < e; ++j) rank += rows[j] == r;
    const int64_t u = ur / Cfg::RW;
    const int64_t rb = u / Cfg::NW;
    const int w = (int)(u % Cfg::NW);
    const uint32_t slot = (uint32_t)(ur % Cfg::RW);
    const int64_t base = slot_pos[((rb * nchunks + c) * Cfg::NW + w) * Cfg::RW + slot];
    if constexpr (Cfg::EPR == 1) {
      uint32_t* word = reinterpret_cast<uint32_t*>(ent + base + (int64_t)Cfg::REC * rank);
      const double v = (double)vals[e];
      word[0] = (uint32_t)__double2loint(v);
      word[1] = (uint32_t)__double2hiint(v);
      word[2] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
    } else if constexpr (Cfg::EPR == 3) {
      uint32_t* word = reinterpret_cast<uint32_t*>(ent + base + (int64_t)Cfg::REC * (rank / 3));
      word[rank % 3] = __float_as_uint((float)vals[e]);
      reinterpret_cast<unsigned char*>(word + 3)[rank % 3] = (unsigned char)(col - lo_col);  // slot byte: header
    } else {  // dense pairs: entry index base + rank, in 8-byte halves of the stream
      const int64_t ve = base + rank;
      uint32_t* word = reinterpret_cast<uint32_t*>(ent + (ve >> 1) * 16);
      const uint32_t h = (uint32_t)(ve & 1);
      word[h] = __float_as_uint((float)vals[e]);
      word[2 + h] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
    }
  }
}

// P5 by chunk range (general chain, 16 <= p <= kFillRangeMaxP): one warp per
// (group, chunk) — the chunk's entries of a group slice are one contiguous
// (col,row)-sorted range (chunk_table_kernel) — 32 entries at a time, a row's
// entries ranked by lane order (match_any) after its running count in the
// range, kept in shared memory per warp (a tag per row names the range the
// count belongs to, so nothing is cleared).  Linear in the range, where the
// per-entry scan of tacc_fill_kernel is quadratic in it.
constexpr int kFillRangeMinP = 16;
constexpr int kFillRangeMaxP = 256;
constexpr int kFillRangeWarps = 8;

template <class Cfg>
__global__ void __launch_bounds__(kFillRangeWarps * 32)
tacc_fill_range_kernel(int64_t m, int32_t p, int64_t groups, const typename Cfg::E* __restrict__ vals,
                       const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                       const int64_t* __restrict__ gidx, const int64_t* __restrict__ tab, int nchunks,
                       const int64_t* __restrict__ slot_pos, unsigned char* __restrict__ ent,
                       const int32_t* __restrict__ unit_of) {
  __shared__ int64_t s_tag[kFillRangeWarps][kFillRangeMaxP];
  __shared__ uint32_t s_cnt[kFillRangeWarps][kFillRangeMaxP];
  griddep_wait();  // PDL: predecessor complete
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = lane; q < p; q += 32) s_tag[wl][q] = -1;
  __syncwarp();
  const int64_t pairs = groups * (int64_t)nchunks;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < pairs; x += wstride) {
    const int64_t g = x / nchunks;
    const int c = (int)(x % nchunks);
    const int64_t* tg = tab + g * (nchunks + 1) + c;
    const int64_t gs = gidx[g];
    const int64_t e0 = gs + tg[0], e1 = gs + tg[1];
    if (e0 >= e1) continue;
    const int32_t lo_col = c * Cfg::KC;
    for (int64_t b0 = e0; b0 < e1; b0 += 32) {
      const int64_t e = b0 + lane;
      int32_t r = -1, ur = -1;
      if (e < e1) {
        r = rows[e];
        ur = unit_of[r];
      }
      const bool mine = ur >= 0;  // a row of this plan (two-class split: the other class is skipped)
      const unsigned same = __match_any_sync(0xffffffffu, mine ? r : -1 - lane);
      const int rl = mine ? (int)(r - g * p) : 0;
      const uint32_t before = mine && s_tag[wl][rl] == x ? s_cnt[wl][rl] : 0u;
      const uint32_t rank = before + (uint32_t)__popc(same & ((1u << lane) - 1u));
      __syncwarp();
      if (mine && (same >> lane) == 1u) {  // the row's last entry in this batch
        s_tag[wl][rl] = x;
        s_cnt[wl][rl] = rank + 1;
      }
      __syncwarp();
      if (!mine) continue;
      const int32_t col = cols[e];
      const int64_t u = ur / Cfg::RW;
      const int64_t rb = u / Cfg::NW;
      const int w = (int)(u % Cfg::NW);
      const uint32_t slot = (uint32_t)(ur % Cfg::RW);
      const int64_t base = slot_pos[((rb * nchunks + c) * Cfg::NW + w) * Cfg::RW + slot];
      if constexpr (Cfg::EPR == 1) {
        uint32_t* word = reinterpret_cast<uint32_t*>(ent + base + (int64_t)Cfg::REC * rank);
        const double v = (double)vals[e];
        word[0] = (uint32_t)__double2loint(v);
        word[1] = (uint32_t)__double2hiint(v);
        word[2] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
      } else if constexpr (Cfg::EPR == 3) {
        uint32_t* word = reinterpret_cast<uint32_t*>(ent + base + (int64_t)Cfg::REC * (rank / 3));
        word[rank % 3] = __float_as_uint((float)vals[e]);
        reinterpret_cast<unsigned char*>(word + 3)[rank % 3] = (unsigned char)(col - lo_col);
      } else {
        const int64_t ve = base + rank;
        uint32_t* word = reinterpret_cast<uint32_t*>(ent + (ve >> 1) * 16);
        const uint32_t h = (uint32_t)(ve & 1);
        word[h] = __float_as_uint((float)vals[e]);
        word[2 + h] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
      }
    }
  }
}

// ------------------------------------------ segment planner (even A) ------
// For an A whose rows keep identity placement (row r in row block r / rpb,
// warp (r % rpb) % NW, slot (r % rpb) / NW) one CTA per segment (row block,
// chunk) builds its segment straight from the GCOO: the row block's rows are
// whole group slices (or a row-filtered part of one when p > rpb), and inside
// a group slice — sorted by (col, row) — a chunk's entries are one contiguous
// range, found by binary search.  Pass 1 counts per (warp, slot) in shared
// memory and writes the segment length (c == 0 CTAs also write the row
// placement); pass 2, after the scan of the lengths, writes the offset table,
// the warp headers and every entry.  Replaces the count / size / header / fill
// chain (global atomics, per-slot scratch) for even A.
constexpr int kSegThreads = 512;
constexpr int kSegMaxGroups = 512;  // groups per row block (p = 1: rpb <= RB <= 512)
constexpr int kSegRowCache = 4096;  // a segment's entry rows and columns staged in shared memory (pass 2)

// tab[g * (nchunks + 1) + c] = the first entry of group g's slice with a
// column >= c * KC, relative to the slice start (c = nchunks: the slice
// length): every chunk range of every group without a search.  Each entry
// writes the table cells of the chunks its column opens (from the previous
// entry's chunk + 1 up to its own); the slice's last entry closes the rest.
__global__ void chunk_table_kernel(int64_t nnz, int32_t p, int64_t groups, const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ cols, const int64_t* __restrict__ gidx,
                                   const int64_t* __restrict__ gnnz, int32_t kc, int nchunks,
                                   int64_t* __restrict__ tab, int32_t rpb, unsigned long long* __restrict__ n_seg) {
  griddep_wait();  // PDL: predecessor complete
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t e0 = t0 - (threadIdx.x & 31); e0 < nnz; e0 += stride) {  // warp-uniform trip count
    const int64_t e = e0 + (threadIdx.x & 31);
    const bool in = e < nnz;
    int64_t x = -1;
    if (in) {
      const int32_t r = rows[e];
      const int64_t g = r / p;
      const int64_t gs = gidx[g], ge = gs + gnnz[g];
      const int c = cols[e] / kc;
      const int cp = e == gs ? -1 : cols[e - 1] / kc;
      int64_t* t = tab + g * (nchunks + 1);
      for (int q = cp + 1; q <= c; ++q) t[q] = e - gs;
      if (e == ge - 1)
        for (int q = c + 1; q <= nchunks; ++q) t[q] = ge - gs;
      x = (int64_t)(r / rpb) * nchunks + c;  // segment (row block, chunk), identity placement
    }
    if (n_seg) {  // entries per segment: one atomic per run of equal segments in the warp
      const unsigned same = __match_any_sync(0xffffffffu, (unsigned long long)x);
      if (in && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&n_seg[x], (unsigned long long)__popc(same));
    }
  }
  for (int64_t g = t0; g < groups; g += stride)  // empty slices: every range empty
    if (gnnz[g] == 0)
      for (int q = 0; q <= nchunks; ++q) tab[g * (nchunks + 1) + q] = 0;
}

// n -> Cfg::extent(n) in place (the chunk table's per-segment entry counts).
template <class Cfg>
__global__ void seg_extent_kernel(int64_t nseg, int64_t* __restrict__ len) {
  griddep_wait();  // PDL: predecessor complete
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < nseg; x += (int64_t)gridDim.x * blockDim.x)
    len[x] = Cfg::extent(len[x]);
}

template <class Cfg>
struct SegSmem {
  uint32_t cnt[Cfg::NW * Cfg::RW];   // entries per (warp, slot)
  uint32_t base[Cfg::NW * Cfg::RW];  // pass 2: the slot's first entry (EPR 2: 8-byte halves) / record byte, in-segment
  int64_t lo[kSegMaxGroups];         // the chunk's range in each group slice
  int32_t pre[kSegMaxGroups + 1];    // exclusive prefix of the range lengths
  int32_t row[kSegRowCache];         // pass 2: the flattened ranges' rows (ranks) and columns, when they fit
  int32_t col[kSegRowCache];
};

template <class Cfg, int PASS>
__global__ void __launch_bounds__(kSegThreads)
seg_plan_kernel(int64_t m, int64_t nnz, int32_t p, const typename Cfg::E* __restrict__ vals,
                const int32_t* __restrict__ rows, const int32_t* __restrict__ cols, const int64_t* __restrict__ gidx,
                const int64_t* __restrict__ gnnz, const int64_t* __restrict__ tab, int nchunks, int64_t nseg,
                int32_t rpb,
                int64_t* __restrict__ seg_len, int32_t* __restrict__ unit_of, int32_t* __restrict__ row_of,
                int32_t* __restrict__ skew_flag, int64_t* __restrict__ seg_off, unsigned char* __restrict__ ent,
                const int64_t* __restrict__ nscan) {
  // PASS 1: lengths; PASS 2: build at the scanned offsets; PASS 3 (count
  // extents): placement + build at the scan of the extents of the entry
  // counts (chunk_table_kernel, seg_extent_kernel), copied to seg_off
  static_assert(PASS != 3 || Cfg::LINEAR_EXTENT, "single build pass: linear extents only");
  static_assert(Cfg::RB <= kSegMaxGroups, "groups per row block");
  constexpr int NW = Cfg::NW, RW = Cfg::RW, EPR = Cfg::EPR;
  __shared__ SegSmem<Cfg> sm;
  __shared__ int32_t s_total;
  griddep_wait();  // PDL: predecessor complete
  const int tid = threadIdx.x;
  if (PASS != 2 && blockIdx.x == 0 && tid == 0) *skew_flag = 0;
  if (PASS == 3 && blockIdx.x == 0 && tid == 0) seg_off[nseg] = nscan[nseg];
  for (int64_t x = blockIdx.x; x < nseg; x += gridDim.x) {
    const int64_t rb = x / nchunks;
    const int c = (int)(x % nchunks);
    const int64_t r0 = rb * rpb, r1 = r0 + rpb < m ? r0 + rpb : m;
    const int32_t lo_col = c * Cfg::KC, hi_col = lo_col + Cfg::KC;
    if (PASS != 2 && c == 0) {  // identity placement of the row block's rows
      for (int64_t r = r0 + tid; r < r1; r += kSegThreads) {
        const int64_t j = r - r0;
        unit_of[r] = (int32_t)(rb * Cfg::RB + (j % NW) * RW + j / NW);
      }
      for (int q = tid; q < Cfg::RB; q += kSegThreads) {
        const int64_t j = (int64_t)(q % RW) * NW + q / RW, r = r0 + j;
        row_of[rb * Cfg::RB + q] = (j < rpb && r < r1) ? (int32_t)r : -1;
      }
    }
    const int64_t g0 = r0 / p;
    const int ng = r1 > r0 ? (int)((r1 - 1) / p - g0 + 1) : 0;
    for (int i = tid; i < NW * RW; i += kSegThreads) sm.cnt[i] = 0u;
    // the chunk's range in each group slice (chunk_table_kernel)
    for (int t = tid; t < ng; t += kSegThreads) {
      const int64_t* tg = tab + (g0 + t) * (int64_t)(nchunks + 1) + c;
      const int64_t gs = gidx[g0 + t];
      sm.lo[t] = gs + tg[0];
      sm.pre[t + 1] = (int32_t)(tg[1] - tg[0]);
    }
    __syncthreads();
    if (tid < 32) {  // warp 0: exclusive prefix of the range lengths
      const int per = (ng + 31) / 32, t0 = tid * per, t1 = t0 + per < ng ? t0 + per : ng;
      int32_t sum = 0;
      for (int t = t0; t < t1; ++t) sum += sm.pre[t + 1];
      int32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (tid >= d) incl += y;
      }
      int32_t run = incl - sum;
      for (int t = t0; t < t1; ++t) {
        const int32_t len = sm.pre[t + 1];
        sm.pre[t] = run;
        run += len;
      }
      if (tid == 31) {
        sm.pre[ng] = incl;
        s_total = incl;
      }
    }
    __syncthreads();
    const int32_t total = s_total;
    // entry i of the flattened ranges: its group by binary search over pre
    auto locate = [&](int32_t i, int64_t& e, int& g) {
      int a = 0, b = ng;  // pre[a] <= i < pre[b]
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (sm.pre[mid] <= i) a = mid; else b = mid;
      }
      g = a;
      e = sm.lo[a] + (i - sm.pre[a]);
    };
    const bool cached = PASS != 1 && total <= kSegRowCache;
    for (int32_t i = tid; i < total; i += kSegThreads) {
      int64_t e;
      int g;
      locate(i, e, g);
      const int32_t r = rows[e];
      if (cached) {
        sm.row[i] = r;
        sm.col[i] = cols[e];
      }
      if (r < r0 || r >= r1) continue;  // another row block's row of a shared group (p > rpb)
      const int64_t j = r - r0;
      atomicAdd(&sm.cnt[(j % NW) * RW + j / NW], 1u);
    }
    __syncthreads();
    if constexpr (PASS == 1) {
      if (tid < 32) {
        uint32_t sz = 0, ne = 0;
        for (int w = tid; w < NW; w += 32) {
          uint32_t recs = 0, nw = 0;
          for (int q = 0; q < RW; ++q) {
            nw += sm.cnt[w * RW + q];
            recs += (sm.cnt[w * RW + q] + EPR - 1) / EPR;
          }
          if constexpr (EPR == 2) recs = (nw + 1) / 2;
          sz += Cfg::HDR + Cfg::REC * recs;
          ne += nw;
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
          sz += __shfl_xor_sync(0xffffffffu, sz, d);
          ne += __shfl_xor_sync(0xffffffffu, ne, d);
        }
        if (tid == 0) seg_len[x] = Cfg::LINEAR_EXTENT ? Cfg::extent(ne) : Cfg::TABLE + sz;
      }
    } else {
      const int64_t so = PASS == 3 ? nscan[x] : seg_off[x];
      if (PASS == 3 && tid == 0) seg_off[x] = so;
      unsigned char* seg = ent + so;
      if (tid < 32) {  // warp 0: warp segment offsets (one lane per warp), then per-slot bases
        uint32_t recs = 0, nent = 0;
        if (tid < NW) {
          for (int q = 0; q < RW; ++q) {
            nent += sm.cnt[tid * RW + q];
            recs += (sm.cnt[tid * RW + q] + EPR - 1) / EPR;
          }
          if (EPR == 2) recs = (nent + 1) / 2;
        }
        const uint32_t sz = tid < NW ? Cfg::HDR + Cfg::REC * recs : 0u;
        uint32_t incl = sz;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
          if (tid >= d) incl += y;
        }
        if (tid < NW) {
          const uint32_t wo = Cfg::TABLE + incl - sz;
          reinterpret_cast<uint32_t*>(seg)[tid] = wo;
          *reinterpret_cast<uint4*>(seg + wo) = make_uint4(EPR == 2 ? nent : recs, 0u, 0u, 0u);
          uint32_t before = 0;
          for (int q = 0; q < RW; ++q) {
            const uint32_t cq = sm.cnt[tid * RW + q];
            if constexpr (EPR == 2) {
              sm.base[tid * RW + q] = (wo + Cfg::HDR) / 8 + before;
              before += cq;
            } else {
              const uint32_t pos = wo + Cfg::HDR + Cfg::REC * before, ns = (cq + EPR - 1) / EPR;
              sm.base[tid * RW + q] = pos;
              // absent-entry marks, overwritten by the entries that exist
              const uint32_t mark = EPR == 3 ? 0x00FFFFFFu | ((uint32_t)q << 24) : 0u;
              for (uint32_t jj = 0; jj < ns; ++jj) reinterpret_cast<uint32_t*>(seg + pos)[4 * jj + 3] = mark;
              before += ns;
            }
          }
        }
      }
      // entry e (row r of this block, column col) at its rank among row r's
      // entries of this chunk
      auto emit = [&](int64_t e, int32_t r, uint32_t rank, int32_t col) {
        const int64_t j = r - r0;
        const uint32_t slot = (uint32_t)(j / NW);
        const uint32_t bse = sm.base[(j % NW) * RW + slot];
        if constexpr (EPR == 1) {
          uint32_t* word = reinterpret_cast<uint32_t*>(seg + bse + (int64_t)Cfg::REC * rank);
          const double v = (double)vals[e];
          word[0] = (uint32_t)__double2loint(v);
          word[1] = (uint32_t)__double2hiint(v);
          word[2] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
        } else if constexpr (EPR == 3) {
          uint32_t* word = reinterpret_cast<uint32_t*>(seg + bse + (int64_t)Cfg::REC * (rank / 3));
          word[rank % 3] = __float_as_uint((float)vals[e]);
          reinterpret_cast<unsigned char*>(word + 3)[rank % 3] = (unsigned char)(col - lo_col);
        } else {
          const int64_t ve = so / 8 + bse + rank;
          uint32_t* word = reinterpret_cast<uint32_t*>(ent + (ve >> 1) * 16);
          const uint32_t h = (uint32_t)(ve & 1);
          word[h] = __float_as_uint((float)vals[e]);
          word[2 + h] = ((uint32_t)(col - lo_col) * Cfg::ROWB) | (slot << 24);
        }
      };
      if (total <= 32 * ng) {
        // short group ranges (small p): one thread per entry, its rank by
        // counting same-row entries earlier in its group's range
        __syncthreads();
        for (int32_t i = tid; i < total; i += kSegThreads) {
          int64_t e;
          int g;
          locate(i, e, g);
          const int32_t r = cached ? sm.row[i] : rows[e];
          if (r < r0 || r >= r1) continue;
          uint32_t rank = 0;
          if (cached) {
            for (int32_t jx = sm.pre[g]; jx < i; ++jx) rank += sm.row[jx] == r;
          } else {
            for (int64_t jx = sm.lo[g]; jx < e; ++jx) rank += rows[jx] == r;
          }
          emit(e, r, rank, cached ? sm.col[i] : cols[e]);
        }
      } else {
        // long group ranges (large p): one warp per group range, 32 entries
        // at a time — a row's entries in the batch rank by lane order
        // (match_any) after its running count, which the row's last lane
        // advances; rows belong to one group, so no other warp touches them
        __syncthreads();  // the bases are read; cnt becomes the running counts
        for (int q2 = tid; q2 < NW * RW; q2 += kSegThreads) sm.cnt[q2] = 0u;
        __syncthreads();
        const int wid = tid >> 5, ln = tid & 31;
        for (int g = wid; g < ng; g += kSegThreads / 32) {
          const int32_t i0 = sm.pre[g], i1 = sm.pre[g + 1];
          for (int32_t b0 = i0; b0 < i1; b0 += 32) {
            const int32_t i = b0 + ln;
            const int64_t e = sm.lo[g] + (i - i0);
            int32_t r = -1;
            if (i < i1) r = cached ? sm.row[i] : rows[e];
            const bool mine = r >= r0 && r < r1;
            const unsigned same = __match_any_sync(0xffffffffu, mine ? r : -1 - ln);
            const int64_t j = r - r0;
            const int sidx = mine ? (int)((j % NW) * RW + j / NW) : 0;
            const uint32_t rank = mine ? sm.cnt[sidx] + (uint32_t)__popc(same & ((1u << ln) - 1u)) : 0u;
            __syncwarp();
            if (mine && (same >> ln) == 1u) sm.cnt[sidx] += (uint32_t)__popc(same);
            __syncwarp();
            if (mine) emit(e, r, rank, cached ? sm.col[i] : cols[e]);
          }
        }
      }
    }
    __syncthreads();  // shared state is reused by the next segment
  }
}

// ---------------------------------------------------------- main kernel --
template <bool GLOBAL>
struct RecSrc;
template <>
struct RecSrc<false> {  // staged in shared memory
  using addr_t = uint32_t;
  static __device__ __forceinline__ uint4 ld(addr_t a) { return lds128u(a); }
  static __device__ __forceinline__ uint32_t ld32(addr_t a) { return lds32u(a); }
};
template <>
struct RecSrc<true> {  // segment larger than a stage: read from global memory
  using addr_t = const unsigned char*;
  static __device__ __forceinline__ uint4 ld(addr_t a) { return __ldg(reinterpret_cast<const uint4*>(a)); }
  static __device__ __forceinline__ uint32_t ld32(addr_t a) { return __ldg(reinterpret_cast<const uint32_t*>(a)); }
};

#ifndef GCOO_ABL
#define GCOO_ABL 0  // ablation builds (tools/ablate.sh, wrong results): 1 no TMEM swap, 2 no B loads, 3 both
#endif
#ifndef GCOO_PRODUCER_HINT_NS
#define GCOO_PRODUCER_HINT_NS 0  // suspend-time hint of the producer's stage-release wait (0: spin)
#endif
#ifndef GCOO_PROF
#define GCOO_PROF 0  // measurement builds (tools/prof_probe.py): per-warp cycle accounting into g_prof
#endif
#if GCOO_PROF
// [0] consumer cycles in full-barrier waits, [1] consumer cycles chunk loop total, [2] consumer
// epilogue cycles, [3] producer cycles in empty-barrier waits, [4] producer loop cycles,
// [5] consumer warps, [6] records consumed, [7] TMEM swaps, [8] loop cycles of heavy row-block
// warps (skewed placement, row block 0), [9] their count, [10] max loop cycles of any warp
__device__ unsigned long long g_prof[12];
// per-warp event counters in shared memory (lane 0 bumps them: no global atomics in the loop)
__shared__ unsigned g_prof_swaps[32], g_prof_recs[32];
#define GCOO_PROF_ADD(i, v) atomicAdd(&g_prof[i], (unsigned long long)(v))
#else
#define GCOO_PROF_ADD(i, v) ((void)0)
#endif

// `cur` always names a slot whose TMEM copy the registers may overwrite: it
// starts at slot 0 with zero accumulators (slot 0's TMEM is zero too), so the
// first swap needs no "nothing held yet" test.
template <class Cfg>
__device__ __forceinline__ void tacc_switch(float (&acc)[Cfg::V], uint32_t& cur, uint32_t tacc, uint32_t s) {
  if ((GCOO_ABL & 1) && s != cur) {
    cur = s;
    return;
  }
  if (s != cur) {  // warp-uniform: swap the slot's accumulators through TMEM
#if GCOO_PROF
    if ((threadIdx.x & 31) == 0) ++g_prof_swaps[threadIdx.x >> 5];
#endif
    tmem_st<Cfg::V>(tacc + cur * Cfg::V, acc);
    tmem_ld<Cfg::V>(tacc + s * Cfg::V, acc);
    tmem_wait_ld();
    cur = s;
  }
}

// acc[v] = fma(a, b[v], acc[v]) in column order per element.  PACKED: f32x2 FMAs
// (FFMA2, two independent round-to-nearest FMAs: the same bits) halve the issue
// slots the FMAs take — used by the two-entry-record loops (s=0.99 0.950 ->
// 0.931 ms, 0.995 0.597 -> 0.574); the three-entry loop is faster with scalar
// FFMA (s=0.98 1.68 vs 1.85 ms packed).
template <int V, bool PACKED = false>
__device__ __forceinline__ void tacc_fma(float (&acc)[V], float a, const float (&b)[V]) {
  if constexpr (PACKED && V % 2 == 0) {
    const float2 a2 = make_float2(a, a);
#pragma unroll
    for (int v = 0; v < V; v += 2) {
      const float2 r = __ffma2_rn(a2, make_float2(b[v], b[v + 1]), make_float2(acc[v], acc[v + 1]));
      acc[v] = r.x;
      acc[v + 1] = r.y;
    }
  } else {
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = __fmaf_rn(a, b[v], acc[v]);
  }
}

// One entry {v, off | slot << 24}.
template <class Cfg>
__device__ __forceinline__ void tacc_entry(float (&acc)[Cfg::V], uint32_t& cur, uint32_t tacc, uint32_t v, uint32_t o,
                                           uint32_t bbase) {
  float b[Cfg::V];
  lds_vec<Cfg::V>(bbase + (o & 0xffffffu), b);
  tacc_switch<Cfg>(acc, cur, tacc, o >> 24);
  tacc_fma<Cfg::V, true>(acc, __uint_as_float(v), b);
}

// Three-entry records (dense regime: long runs fill them): B row r of the
// staged tile sits at r * W * 4 bytes; one record per step.
template <class Cfg, bool GLOBAL>
__device__ __forceinline__ void tacc_consume3(float (&acc)[Cfg::V], uint32_t& cur, uint32_t tacc,
                                             typename RecSrc<GLOBAL>::addr_t seg, int warp, uint32_t bbase) {
  using Src = RecSrc<GLOBAL>;
  constexpr int V = Cfg::V;
  constexpr uint32_t ROWB = Cfg::ROWB;
  asm volatile("mov.b32 %0, %0;" : "+r"(bbase));
  const uint32_t woff = Src::ld32(seg + 4 * warp);
  const auto wseg = seg + woff;
  const uint32_t nrec = Src::ld32(wseg);
  auto rec = wseg + Cfg::HDR;
  for (uint32_t r = 0; r < nrec; ++r, rec += Cfg::REC) {
    const uint4 q = Src::ld(rec);
    const uint32_t r0 = q.w & 0xffu, r1 = (q.w >> 8) & 0xffu, r2 = (q.w >> 16) & 0xffu;
    const bool h1 = r1 != 0xffu, h2 = r2 != 0xffu;
    float b0[V], b1[V], b2[V];
    lds_vec<V>(bbase + r0 * ROWB, b0);
    if (h1) lds_vec<V>(bbase + r1 * ROWB, b1);
    if (h2) lds_vec<V>(bbase + r2 * ROWB, b2);
    tacc_switch<Cfg>(acc, cur, tacc, q.w >> 24);
    tacc_fma<V>(acc, __uint_as_float(q.x), b0);
    if (h1) tacc_fma<V>(acc, __uint_as_float(q.y), b1);
    if (h2) tacc_fma<V>(acc, __uint_as_float(q.z), b2);
  }
}

// fp64 (one entry per record; a lane's two doubles are four TMEM/shared
// cells): two records per step, DFMA on the reinterpreted cells.
__device__ __forceinline__ void tacc_dfma(float (&acc)[4], double a, const float (&b)[4]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double bv = __hiloint2double(__float_as_int(b[2 * h + 1]), __float_as_int(b[2 * h]));
    const double av = __hiloint2double(__float_as_int(acc[2 * h + 1]), __float_as_int(acc[2 * h]));
    const double r = __fma_rn(a, bv, av);
    acc[2 * h] = __int_as_float(__double2loint(r));
    acc[2 * h + 1] = __int_as_float(__double2hiint(r));
  }
}

template <class Cfg, bool GLOBAL>
__device__ __forceinline__ void tacc_consume1(float (&acc)[Cfg::V], uint32_t& cur, uint32_t tacc,
                                              typename RecSrc<GLOBAL>::addr_t seg, int warp, uint32_t bbase) {
  using Src = RecSrc<GLOBAL>;
  static_assert(Cfg::V == 4, "two doubles per lane");
  asm volatile("mov.b32 %0, %0;" : "+r"(bbase));
  const uint32_t woff = Src::ld32(seg + 4 * warp);
  const auto wseg = seg + woff;
  const uint32_t nrec = Src::ld32(wseg);
  auto rec = wseg + Cfg::HDR;
  for (uint32_t r = 1; r < nrec; r += 2, rec += 2 * Cfg::REC) {
    const uint4 qa = Src::ld(rec), qb = Src::ld(rec + Cfg::REC);
    float ba[4], bb[4];
    lds_vec<4>(bbase + (qa.z & 0xffffffu), ba);
    lds_vec<4>(bbase + (qb.z & 0xffffffu), bb);
    tacc_switch<Cfg>(acc, cur, tacc, qa.z >> 24);
    tacc_dfma(acc, __hiloint2double((int)qa.y, (int)qa.x), ba);
    tacc_switch<Cfg>(acc, cur, tacc, qb.z >> 24);
    tacc_dfma(acc, __hiloint2double((int)qb.y, (int)qb.x), bb);
  }
  if (nrec & 1u) {
    const uint4 q = Src::ld(rec);
    float b[4];
    lds_vec<4>(bbase + (q.z & 0xffffffu), b);
    tacc_switch<Cfg>(acc, cur, tacc, q.z >> 24);
    tacc_dfma(acc, __hiloint2double((int)q.y, (int)q.x), b);
  }
}

// One warp walks its entries for one chunk: a dense stream of pairs
// {v0, v1, off0 | slot0 << 24, off1 | slot1 << 24} in slot-major, column
// order, two pairs (four entries, their four B rows in flight) per step, then
// the 0-3 left over — no absent entries, so no predicated FMAs.  `cur` (the
// slot whose accumulators are in registers) persists across chunks.
template <class Cfg, bool GLOBAL>
__device__ __forceinline__ void tacc_consume(float (&acc)[Cfg::V], uint32_t& cur, uint32_t tacc,
                                             typename RecSrc<GLOBAL>::addr_t seg, int warp, uint32_t bbase) {
  using Src = RecSrc<GLOBAL>;
  constexpr int V = Cfg::V;
  // keep the stage base in a register (ptxas otherwise rematerialises it from
  // special registers inside the loop when registers are tight)
  asm volatile("mov.b32 %0, %0;" : "+r"(bbase));
  const uint32_t woff = Src::ld32(seg + 4 * warp);
  const auto wseg = seg + woff;
  const uint32_t nent = Src::ld32(wseg);
#if GCOO_PROF
  if ((threadIdx.x & 31) == 0) g_prof_recs[threadIdx.x >> 5] += (nent + 1) / 2;
#endif
  auto rec = wseg + Cfg::HDR;
  uint32_t r = 0;
  for (; r + 4 <= nent; r += 4, rec += 2 * Cfg::REC) {
    const uint4 qa = Src::ld(rec);
    const uint4 qb = Src::ld(rec + Cfg::REC);
    float b0[V], b1[V], b2[V], b3[V];
    if constexpr (GCOO_ABL & 2) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        b0[v] = __uint_as_float(qa.z + v);
        b1[v] = __uint_as_float(qa.w + v);
        b2[v] = __uint_as_float(qb.z + v);
        b3[v] = __uint_as_float(qb.w + v);
      }
    } else {
      lds_vec<V>(bbase + (qa.z & 0xffffffu), b0);
      lds_vec<V>(bbase + (qa.w & 0xffffffu), b1);
      lds_vec<V>(bbase + (qb.z & 0xffffffu), b2);
      lds_vec<V>(bbase + (qb.w & 0xffffffu), b3);
    }
    tacc_switch<Cfg>(acc, cur, tacc, qa.z >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(qa.x), b0);
    tacc_switch<Cfg>(acc, cur, tacc, qa.w >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(qa.y), b1);
    tacc_switch<Cfg>(acc, cur, tacc, qb.z >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(qb.x), b2);
    tacc_switch<Cfg>(acc, cur, tacc, qb.w >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(qb.y), b3);
  }
  const uint32_t left = nent - r;  // 0..3
  if (left >= 2) {
    const uint4 q = Src::ld(rec);
    float b0[V], b1[V];
    lds_vec<V>(bbase + (q.z & 0xffffffu), b0);
    lds_vec<V>(bbase + (q.w & 0xffffffu), b1);
    tacc_switch<Cfg>(acc, cur, tacc, q.z >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(q.x), b0);
    tacc_switch<Cfg>(acc, cur, tacc, q.w >> 24);
    tacc_fma<V, true>(acc, __uint_as_float(q.y), b1);
    rec += Cfg::REC;
  }
  if (left & 1u) {
    const uint4 q = Src::ld(rec);
    tacc_entry<Cfg>(acc, cur, tacc, q.x, q.z, bbase);
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS, 1)
spdm_tacc_kernel(const __grid_constant__ CUtensorMap tmap_b, int64_t m, int64_t n, const unsigned char* __restrict__ ent,
                 const int64_t* __restrict__ seg_off, typename Cfg::E* __restrict__ C, int64_t ldc, int64_t row_blocks,
                 int nchunks, const int32_t* __restrict__ row_of, const int32_t* __restrict__ skewed) {
  constexpr int W = Cfg::W, NW = Cfg::NW, S = Cfg::STAGES, V = Cfg::V, RW = Cfg::RW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)S * Cfg::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + S);
  // the producer publishes each stage's record-segment offset and length here
  // (ordered by the full barrier), so consumers never read seg_off
  int64_t* stage_lo = reinterpret_cast<int64_t*>(tmem_slot + 4);
  uint32_t* stage_len = reinterpret_cast<uint32_t*>(stage_lo + S);
  const uint32_t smem0 = smem_u32(smem_raw);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t col_tiles = ceil_div_dev(n, W);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, 512);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *tmem_slot;
  griddep_wait();  // PDL: the planner's record stream is complete
  // Tiles (row block, column tile) in launch order; CTA i takes tiles i,
  // i + gridDim.x, ... (one each when the grid covers every tile; persistent
  // otherwise: the producer then streams the next tile's first chunks while
  // the consumers write the previous tile back).  Row blocks vary fastest, so
  // the tiles in flight share a few B strips and every B tile crosses HBM
  // once.  A skewed matrix (*skewed, row_balance_kernel) has its heaviest rows
  // in row block 0: those tiles go first so they overlap everything else
  // instead of forming a tail.
  const int64_t tiles = row_blocks * col_tiles;
  const bool skew = *skewed && row_blocks > 1;
  auto tile_of = [&](int64_t t, int64_t& rb, int64_t& ct) {
    if (skew && t < col_tiles) {
      rb = 0;
      ct = t;
    } else if (skew) {
      const int64_t x = t - col_tiles;
      rb = 1 + x % (row_blocks - 1);
      ct = x / (row_blocks - 1);
    } else {
      rb = t % row_blocks;
      ct = t / row_blocks;
    }
  };

  if (warp == NW) {
    // ------------- producer: B tile (TMA 2-D) + record segment (bulk 1-D)
    if (lane == 0) {
      // every column tile re-reads the row block's records: keep them in L2
      // while the B strips stream through (configs[3]: DRAM reads per launch
      // would otherwise carry the record stream once per column tile)
      const uint64_t keep = l2_policy_evict_last();
#if GCOO_PROF
      const long long p0 = clock64();
      long long pw = 0;
#endif
      uint32_t q = 0;  // chunks issued by this CTA so far: stage q % S, ring round q / S
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t rb, ct;
        tile_of(t, rb, ct);
        const int64_t* so = seg_off + rb * nchunks;
        const int32_t x = (int32_t)(ct * W);
        int64_t lo = so[0], hi = so[1];
        for (int c = 0; c < nchunks; ++c, ++q) {
          const int s = (int)(q % S);
          const int64_t hi_next = so[c + 2 <= nchunks ? c + 2 : nchunks];  // prefetch
          const uint32_t len = (uint32_t)(hi - lo);
          const uint32_t bytes = len <= Cfg::CAP ? len : 0u;  // oversize: consumers read global memory
          // a segment of empty warp headers only: no consumer reads this chunk's B tile
          const bool any = len > (Cfg::LINEAR_EXTENT ? Cfg::EXT_BASE : (uint32_t)(Cfg::TABLE + Cfg::NW * Cfg::HDR));
#if GCOO_PROF
          const long long w0 = clock64();
#endif
          if (q >= S) {
#if GCOO_PRODUCER_HINT_NS
            mbar_wait_sleep(&empty[s], (q / S - 1) & 1u, GCOO_PRODUCER_HINT_NS);
#else
            mbar_wait(&empty[s], (q / S - 1) & 1u);
#endif
          }
#if GCOO_PROF
          pw += clock64() - w0;
#endif
          unsigned char* stage = smem_raw + (size_t)s * Cfg::STAGE_BYTES;
          stage_lo[s] = lo;
          stage_len[s] = len;
          mbar_arrive_expect_tx(&full[s], (any ? Cfg::BTILE : 0u) + bytes);
          if (any) tma_load_2d(stage, &tmap_b, x, c * Cfg::KC, &full[s]);
          if (bytes) bulk_g2s_hint(smem_u32(stage + Cfg::BTILE), ent + lo, bytes, &full[s], keep);
          lo = hi;
          hi = hi_next;
        }
      }
#if GCOO_PROF
      GCOO_PROF_ADD(3, pw);
      GCOO_PROF_ADD(4, clock64() - p0);
#endif
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  // my accumulators: TMEM lanes 32*(warp%4).., columns (warp/4)*TCOLS + slot*V + v
  const uint32_t tacc = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * Cfg::TCOLS);
  uint32_t q = 0;  // chunks consumed by this CTA so far (the producer's count)
  // the shared-memory window base and this lane's offset stay in registers
  // (ptxas otherwise rematerialises them from special registers every chunk)
  uint32_t sbase = smem0 + (uint32_t)(lane * V * 4);
  asm volatile("mov.b32 %0, %0;" : "+r"(sbase));
#if GCOO_PROF
  if (lane == 0) g_prof_swaps[warp] = g_prof_recs[warp] = 0;
  __syncwarp();
  long long qw = 0, qloop = 0, qepi = 0;
#endif
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    int64_t rb, ct;
    tile_of(t, rb, ct);
    // this tile's accumulators start at zero (the previous tile's were read back)
#pragma unroll
    for (int c0 = 0; c0 < Cfg::TCOLS; c0 += 8) tmem_st8_zero(tacc + c0);
    tmem_wait_st();
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    uint32_t cur = 0;  // slot 0, zero accumulators (see tacc_switch)
#if GCOO_PROF
    const long long q0 = clock64();
#endif
    for (int c = 0; c < nchunks; ++c, ++q) {
      const int s_idx = (int)(q % S);
#if GCOO_PROF
      const long long w0 = clock64();
      mbar_wait(&full[s_idx], (q / S) & 1u);
      qw += clock64() - w0;
#else
      mbar_wait(&full[s_idx], (q / S) & 1u);
#endif
      tmem_wait_st();  // slots pushed during earlier chunks are complete before they are pulled again
      const uint32_t bbase = sbase + (uint32_t)s_idx * Cfg::STAGE_BYTES;
      const uint32_t stage = bbase - (uint32_t)(lane * V * 4);
      const int64_t lo = stage_lo[s_idx];
      if (stage_len[s_idx] <= Cfg::CAP) {
        if constexpr (Cfg::EPR == 1)
          tacc_consume1<Cfg, false>(acc, cur, tacc, stage + Cfg::BTILE, warp, bbase);
        else if constexpr (Cfg::EPR == 3)
          tacc_consume3<Cfg, false>(acc, cur, tacc, stage + Cfg::BTILE, warp, bbase);
        else
          tacc_consume<Cfg, false>(acc, cur, tacc, stage + Cfg::BTILE, warp, bbase);
      } else {
        if constexpr (Cfg::EPR == 1)
          tacc_consume1<Cfg, true>(acc, cur, tacc, ent + lo, warp, bbase);
        else if constexpr (Cfg::EPR == 3)
          tacc_consume3<Cfg, true>(acc, cur, tacc, ent + lo, warp, bbase);
        else
          tacc_consume<Cfg, true>(acc, cur, tacc, ent + lo, warp, bbase);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s_idx]);
    }
    tmem_st<V>(tacc + cur * V, acc);
    tmem_wait_st();
#if GCOO_PROF
    const long long q1 = clock64();
    qloop += q1 - q0;
    if (lane == 0 && *skewed && rb == 0) {
      GCOO_PROF_ADD(8, q1 - q0);
      GCOO_PROF_ADD(9, 1);
    }
    if (lane == 0) atomicMax(&g_prof[10], (unsigned long long)(q1 - q0));
#endif

    // read back and single write of the tile: slot s, value v at column s*V + v
    const int64_t row0 = (rb * NW + warp) * (int64_t)RW;
    const int64_t j = ct * W + lane * Cfg::VE;  // first element (column) of this lane
#pragma unroll 1
    for (int c0 = 0; c0 < Cfg::TCOLS; c0 += 8) {
      float r[8];
      tmem_ld8(tacc + c0, r);
      tmem_wait_ld();
      if (j < n) {
#pragma unroll
        for (int k = 0; k < 8 / V; ++k) {
          const int64_t row = row_of[row0 + c0 / V + k];  // -1: padding slot
          if (row >= 0) {
            typename Cfg::E* dst = C + row * ldc + j;
            if constexpr (V == 4) {  // 16 bytes: four floats or two doubles
              __stcs(reinterpret_cast<float4*>(dst), make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]));
            } else if constexpr (V == 2) {
              __stcs(reinterpret_cast<float2*>(dst), make_float2(r[2 * k], r[2 * k + 1]));
            } else {
              __stcs(dst, r[k]);
            }
          }
        }
      }
    }
#if GCOO_PROF
    qepi += clock64() - q1;
#endif
  }

#if GCOO_PROF
  if (lane == 0) {
    GCOO_PROF_ADD(0, qw);
    GCOO_PROF_ADD(1, qloop);
    GCOO_PROF_ADD(2, qepi);
    GCOO_PROF_ADD(5, 1);
    GCOO_PROF_ADD(6, g_prof_recs[warp]);
    GCOO_PROF_ADD(7, g_prof_swaps[warp]);
  }
#endif
  // free TMEM once every consumer warp is done with it
  tmem_fence_before();
  named_bar_sync(1, NW * 32);
  tmem_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

}  // namespace gcoo_b200
