// tcgen05.cp.32x128b.warpx4 as a B-row broadcaster: one 512-byte row of a
// shared-memory B tile (128 fp32 = 32 lanes x 16 B) lands in 4 TMEM columns
// of all four lane quadrants, so every warp can then read B[l][4t..4t+3] with
// one tcgen05.ld.32x32b.x4.  Checks the layout (descriptor: no swizzle, core
// matrices of 8 rows x 16 B, SBO = 128 B) and times smem -> TMEM copies and
// TMEM-sourced FMA streams.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_cp tmem_cp.cu && ./tmem_cp
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t cp_desc(uint32_t saddr) {
  // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start>>4 [0,14), LBO>>4 [16,30),
  // SBO>>4 [32,46), version=1 [46,48), layout SWIZZLE_NONE=0 [61,64)
  const uint64_t start = (saddr >> 4) & 0x3FFF;
  const uint64_t lbo = (128 >> 4) & 0x3FFF;
  const uint64_t sbo = (128 >> 4) & 0x3FFF;
  return start | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

constexpr int KC = 48;

__global__ void k_check(const float* __restrict__ g, int* bad, int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* tile = reinterpret_cast<float*>(sm);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < KC * 128; i += blockDim.x) tile[i] = g[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes visible to tcgen05.cp
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tslot;
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      for (int l = 0; l < KC; ++l)
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tbase + 4 * l),
                     "l"(cp_desc(smem_u32(tile + l * 128))));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            smem_u32(&bar)),
        "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  // check: warp w reads quadrant w
  int nbad = 0;
  for (int l = 0; l < KC; ++l) {
    float r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3])
                 : "r"(tbase + ((uint32_t)(32 * warp) << 16) + 4 * l));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int v = 0; v < 4; ++v)
      if (r[v] != g[l * 128 + 4 * lane + v]) ++nbad;
  }
  atomicAdd(bad, nbad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  float* g;
  int* bad;
  long long* cyc;
  CK(cudaMalloc(&g, KC * 128 * 4));
  CK(cudaMalloc(&bad, 4));
  CK(cudaMalloc(&cyc, 8));
  float h[KC * 128];
  for (int i = 0; i < KC * 128; ++i) h[i] = (float)i + 0.25f;
  CK(cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice));
  CK(cudaMemset(bad, 0, 4));
  CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, KC * 512));
  k_check<<<1, 128, KC * 512>>>(g, bad, 1, cyc);
  CK(cudaDeviceSynchronize());
  int hb;
  long long hc;
  CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
  printf("{\"test\": \"tcgen05.cp.32x128b.warpx4 layout\", \"mismatches\": %d}\n", hb);
  k_check<<<1, 128, KC * 512>>>(g, bad, 1000, cyc);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"test\": \"cp 48 rows (24 KB) + commit + wait\", \"cycles_per_iter\": %.1f, \"bytes_per_clk\": %.1f}\n",
         hc / 1000.0, 48 * 512 / (hc / 1000.0));
  return hb != 0;
}
