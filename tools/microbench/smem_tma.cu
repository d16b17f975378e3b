// Do TMA (bulk copy) writes into shared memory take shared-memory bandwidth
// from LDS reads?  16 warps stream LDS.128 over one 64 KB region while one
// producer warp keeps bulk-copying L2-resident data into a second region;
// reports LDS and TMA bytes/clk/SM with and without the TMA stream
// (the GCOOSpDM kernel does both at once).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_tma smem_tma.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ unsigned long long g_cyc[1024];
__device__ unsigned long long g_tma_bytes[1024];

constexpr int kLdsWarps = 16;
constexpr uint32_t kChunk = 32768;

// with_tma: the producer warp streams bulk copies until the LDS warps finish
__global__ void __launch_bounds__((kLdsWarps + 1) * 32, 1)
k_mix(const char* __restrict__ src, size_t window, int iters, int with_tma, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  float4* lds_region = reinterpret_cast<float4*>(sm);           // 64 KB
  unsigned char* tma_region = sm + 65536;                        // 2 x 32 KB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) lds_region[i] = make_float4(i, i + 1, i + 2, i + 3);
  if (threadIdx.x == 0) {
    done = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kLdsWarps) {
    unsigned long long bytes = 0;
    if (lane == 0 && with_tma) {
      uint32_t phase = 0;
      size_t off = (size_t)blockIdx.x * kChunk;
      while (!done) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(kChunk)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(tma_region + (phase & 1) * kChunk)),
                     "l"(src + off % window), "r"(kChunk), "r"(smem_u32(&bar))
                     : "memory");
        asm volatile("{ .reg .pred d; W%=: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1; @!d bra W%=; }" ::"r"(
                         smem_u32(&bar)), "r"(phase & 1) : "memory");
        ++phase;
        off += kChunk;
        bytes += kChunk;
      }
      g_tma_bytes[blockIdx.x] = bytes;
    }
    return;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4 v = lds_region[(threadIdx.x + u * 128 + i * 32) & 4095];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  const long long t1 = clock64();
  asm volatile("bar.sync 1, %0;" ::"r"(kLdsWarps * 32));
  if (threadIdx.x == 0) {
    g_cyc[blockIdx.x] = t1 - t0;
    done = 1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const size_t window = (size_t)48 << 20;  // L2-resident source
  char* src;
  float* out;
  CK(cudaMalloc(&src, window + kChunk));
  CK(cudaMemset(src, 1, window + kChunk));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  const int smem = 65536 + 2 * kChunk;
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 20000;
  for (int with_tma : {0, 1, 0, 1}) {
    k_mix<<<sms, (kLdsWarps + 1) * 32, smem>>>(src, window, iters, with_tma, out);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> cyc(sms), tb(sms);
    CK(cudaMemcpyFromSymbol(cyc.data(), g_cyc, sizeof(unsigned long long) * sms));
    CK(cudaMemcpyFromSymbol(tb.data(), g_tma_bytes, sizeof(unsigned long long) * sms));
    double c = 0, t = 0;
    for (int i = 0; i < sms; ++i) {
      c += (double)cyc[i];
      t += with_tma ? (double)tb[i] : 0.0;
    }
    c /= sms;
    t /= sms;
    const double lds_bytes = (double)kLdsWarps * 32 * iters * 8 * 16;
    printf("{\"test\": \"lds128_with_tma_stream\", \"tma\": %d, \"lds_bytes_per_clk_per_sm\": %.1f, "
           "\"tma_bytes_per_clk_per_sm\": %.1f, \"sum\": %.1f}\n",
           with_tma, lds_bytes / c, t / c, lds_bytes / c + t / c);
    fflush(stdout);
  }
  return 0;
}
