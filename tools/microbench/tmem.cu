// TMEM read/write bandwidth on B200, alone and concurrent with shared-memory
// LDS: decides whether a B panel staged in tensor memory can feed FFMA
// faster than shared memory alone ("B delivery").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem tmem.cu
//
// One CTA per SM, 512 TMEM columns, 16 warps (4 per TMEM lane quadrant).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ unsigned long long g_cycles[1024];

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t tmem_alloc_512(uint32_t* slot) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  return *slot;
}
__device__ __forceinline__ void tmem_free_512(uint32_t base) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

__device__ __forceinline__ void ld_x1(uint32_t a, uint32_t& r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(a));
}
__device__ __forceinline__ void ld_x4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ld_x16(uint32_t a, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(a));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_x4(uint32_t a, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]));
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// MODE 0: ld x1 (8 per wait); 1: ld x4 (8 per wait); 2: ld x16 (2 per wait);
// 3: ld x1 feeding one FFMA each (the GCOOSpDM inner-loop shape, V=1);
// 4: half the warps ld x1 + FFMA, the other half LDS.128 + 4 FFMA (concurrency);
// 5: every warp alternates ld x1 (+1 FFMA) and LDS.128 (+4 FFMA);
// 6: st x4 (write bandwidth).
template <int MODE>
__global__ void __launch_bounds__(512, 1) k_tmem(float* out, int iters, int active_warps) {
  __shared__ uint32_t slot;
  extern __shared__ float4 sm4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm4[i] = make_float4(i, i + 1, i + 2, i + 3);
  const uint32_t base = tmem_alloc_512(&slot);
  const uint32_t qa = base + ((uint32_t)(32 * (warp & 3)) << 16);
  // initialise my quadrant (so loads read defined data)
  {
    uint32_t r[4] = {1u, 2u, 3u, 4u};
    if ((warp >> 2) == 0)
      for (int c = 0; c < 512; c += 4) st_x4(qa + c, r);
    wait_st();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.f;
  uint32_t sink = 0;
  const bool on = warp < active_warps;
  long long t0 = clock64();
  if (on) {
    for (int i = 0; i < iters; ++i) {
      const uint32_t c0 = (uint32_t)((i * 37 + warp * 8) & 511) & ~15u;
      if constexpr (MODE == 0) {
        uint32_t r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ld_x1(qa + ((c0 + u * 5) & 511), r[u]);
        wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) sink += r[u];
      } else if constexpr (MODE == 1) {
        uint32_t r[8][4];
#pragma unroll
        for (int u = 0; u < 8; ++u) ld_x4(qa + ((c0 + u * 4) & 511), r[u]);
        wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) sink += r[u][0] ^ r[u][1] ^ r[u][2] ^ r[u][3];
      } else if constexpr (MODE == 2) {
        uint32_t r[2][16];
        ld_x16(qa + c0, r[0]);
        ld_x16(qa + ((c0 + 16) & 511), r[1]);
        wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) sink += r[0][u] ^ r[1][u];
      } else if constexpr (MODE == 3) {
        uint32_t r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ld_x1(qa + ((c0 + u * 5) & 511), r[u]);
        wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fmaf(1.0f + u, __uint_as_float(r[u]), acc[u]);
      } else if constexpr (MODE == 4) {
        if (warp & 1) {
          uint32_t r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) ld_x1(qa + ((c0 + u * 5) & 511), r[u]);
          wait_ld();
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[u] = fmaf(1.0f + u, __uint_as_float(r[u]), acc[u]);
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float4 v = sm4[((i * 8 + u) * 32 + lane) & 4095];
            const float a = 1.0f + u;
            acc[(u & 3) * 4 + 0] = fmaf(a, v.x, acc[(u & 3) * 4 + 0]);
            acc[(u & 3) * 4 + 1] = fmaf(a, v.y, acc[(u & 3) * 4 + 1]);
            acc[(u & 3) * 4 + 2] = fmaf(a, v.z, acc[(u & 3) * 4 + 2]);
            acc[(u & 3) * 4 + 3] = fmaf(a, v.w, acc[(u & 3) * 4 + 3]);
          }
        }
      } else if constexpr (MODE == 5) {
        uint32_t r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) ld_x1(qa + ((c0 + u * 5) & 511), r[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float4 v = sm4[((i * 4 + u) * 32 + lane) & 4095];
          const float a = 1.0f + u;
          acc[8 + (u & 1) * 4 + 0] = fmaf(a, v.x, acc[8 + (u & 1) * 4 + 0]);
          acc[8 + (u & 1) * 4 + 1] = fmaf(a, v.y, acc[8 + (u & 1) * 4 + 1]);
          acc[8 + (u & 1) * 4 + 2] = fmaf(a, v.z, acc[8 + (u & 1) * 4 + 2]);
          acc[8 + (u & 1) * 4 + 3] = fmaf(a, v.w, acc[8 + (u & 1) * 4 + 3]);
        }
        wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) acc[u] = fmaf(1.0f + u, __uint_as_float(r[u]), acc[u]);
      } else if constexpr (MODE == 6) {
        uint32_t r[4] = {(uint32_t)i, 2u, 3u, 4u};
#pragma unroll
        for (int u = 0; u < 8; ++u) st_x4(qa + ((c0 + u * 4) & 511), r);
        wait_st();
      } else if constexpr (MODE == 7 || MODE == 8 || MODE == 9) {
        // entries distributed by SHFL from a coalesced LDS.64 (one per 32 entries);
        // B from LDS.128 (7), TMEM x4 (8) or alternating (9); 4 FFMA per entry
        const uint2 ent = reinterpret_cast<const uint2*>(sm4)[((i & 63) * 32 + lane) & 8191];
#pragma unroll
        for (int k = 0; k < 32; k += 2) {
          const float a0 = __shfl_sync(0xffffffffu, __uint_as_float(ent.x), k);
          const uint32_t o0 = __shfl_sync(0xffffffffu, ent.y & 0x3ff0u, k);
          const float a1 = __shfl_sync(0xffffffffu, __uint_as_float(ent.x), k + 1);
          const uint32_t o1 = __shfl_sync(0xffffffffu, ent.y & 0x3ff0u, k + 1);
          float b0[4], b1[4];
          uint32_t r0[4], r1[4];
          if constexpr (MODE == 8) ld_x4(qa + ((o0 >> 2) & 508), r0);
          if constexpr (MODE != 7) ld_x4(qa + ((o1 >> 2) & 508), r1);
          if constexpr (MODE == 7 || MODE == 9) {
            const float4 v = sm4[(o0 + lane) & 4095];
            b0[0] = v.x; b0[1] = v.y; b0[2] = v.z; b0[3] = v.w;
          }
          if constexpr (MODE == 7) {
            const float4 v = sm4[(o1 + lane) & 4095];
            b1[0] = v.x; b1[1] = v.y; b1[2] = v.z; b1[3] = v.w;
          }
          if constexpr (MODE != 7) {
            wait_ld();
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if constexpr (MODE == 8) b0[v] = __uint_as_float(r0[v]);
              b1[v] = __uint_as_float(r1[v]);
            }
          }
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            acc[(k & 2) * 2 + v] = fmaf(a0, b0[v], acc[(k & 2) * 2 + v]);
            acc[8 + (k & 2) * 2 + v] = fmaf(a1, b1[v], acc[8 + (k & 2) * 2 + v]);
          }
        }
      } else if constexpr (MODE == 10) {
        // broadcast-entry baseline: LDS.64 broadcast per entry + LDS.128 B + 4 FFMA
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint2 e = reinterpret_cast<const uint2*>(sm4)[(i * 8 + k) & 8191];
          const float4 v = sm4[((e.y & 0x3ff0u) + lane) & 4095];
          const float a = __uint_as_float(e.x) + 1.0f;
          acc[(k & 3) * 4 + 0] = fmaf(a, v.x, acc[(k & 3) * 4 + 0]);
          acc[(k & 3) * 4 + 1] = fmaf(a, v.y, acc[(k & 3) * 4 + 1]);
          acc[(k & 3) * 4 + 2] = fmaf(a, v.z, acc[(k & 3) * 4 + 2]);
          acc[(k & 3) * 4 + 3] = fmaf(a, v.w, acc[(k & 3) * 4 + 3]);
        }
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cycles[blockIdx.x] = t1 - t0;
  float s = (float)sink;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  tmem_free_512(base);
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

static double max_cycles(int nblocks) {
  std::vector<unsigned long long> c(1024);
  cudaMemcpyFromSymbol(c.data(), g_cycles, sizeof(unsigned long long) * 1024);
  double mx = 0;
  for (int i = 0; i < nblocks && i < 1024; ++i) if (c[i] > mx) mx = c[i];
  return mx;
}

template <int MODE>
void run(const char* name, int sms, float* out, int warps, double bytes_per_warp_iter, double fma_per_warp_iter) {
  const int iters = 20000, th = 512, smem = 65536;
  CK(cudaFuncSetAttribute(k_tmem<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_tmem<MODE><<<sms, th, smem>>>(out, 10, warps);
  CK(cudaDeviceSynchronize());
  Timer t;
  float best = 1e30f;
  double cyc = 0;
  for (int r = 0; r < 3; ++r) {
    t.start();
    k_tmem<MODE><<<sms, th, smem>>>(out, iters, warps);
    float ms = t.stop();
    CK(cudaGetLastError());
    if (ms < best) { best = ms; cyc = max_cycles(sms); }
  }
  const double per_sm_iters = (double)warps * iters;
  printf("{\"test\": \"%s\", \"warps\": %d, \"ms\": %.3f, \"bytes_per_clk_per_sm\": %.1f, \"fma_per_clk_per_sm\": %.1f, "
         "\"tflops\": %.2f, \"sm_mhz_est\": %.0f}\n",
         name, warps, best, per_sm_iters * bytes_per_warp_iter / cyc, per_sm_iters * fma_per_warp_iter / cyc,
         2.0 * per_sm_iters * fma_per_warp_iter * sms / (best * 1e-3) / 1e12, cyc / (best * 1e3));
  fflush(stdout);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  float* out;
  CK(cudaMalloc(&out, sizeof(float) * sms * 512));
  for (int w : {4, 8, 16}) run<0>("tmem_ld_x1", sms, out, w, 8 * 128.0, 0);
  for (int w : {4, 8, 16}) run<1>("tmem_ld_x4", sms, out, w, 8 * 512.0, 0);
  for (int w : {4, 16}) run<2>("tmem_ld_x16", sms, out, w, 2 * 2048.0, 0);
  for (int w : {8, 16}) run<3>("tmem_ld_x1_ffma", sms, out, w, 8 * 128.0, 8 * 32.0);
  // mode 4: odd warps 8 x1-loads + 8 FMA/lane; even warps 8 LDS.128 + 32 FMA/lane (averaged per warp)
  run<4>("mix_split_tmem_lds", sms, out, 16, (8 * 128.0 + 8 * 512.0) / 2, (8 * 32.0 + 32 * 32.0) / 2);
  run<5>("mix_interleaved", sms, out, 16, 8 * 128.0 + 4 * 512.0, 8 * 32.0 + 16 * 32.0);
  for (int w : {4, 16}) run<6>("tmem_st_x4", sms, out, w, 8 * 512.0, 0);
  // per iteration 32 entries x 4 FMA per lane = 4096 FMA per warp
  for (int w : {8, 16}) run<7>("shfl_entries_lds_b", sms, out, w, 32 * 512.0 + 256, 32 * 128.0);
  for (int w : {8, 16}) run<8>("shfl_entries_tmem_b", sms, out, w, 32 * 512.0, 32 * 128.0);
  for (int w : {8, 16}) run<9>("shfl_entries_mix_b", sms, out, w, 32 * 512.0 + 256, 32 * 128.0);
  for (int w : {8, 16}) run<10>("bcast_entries_lds_b", sms, out, w, 8 * 512.0, 8 * 128.0);
  return 0;
}
