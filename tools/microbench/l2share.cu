// L2 -> SM delivery when groups of G CTAs (one per SM) stream the SAME bytes
// at about the same time — the access pattern of CTAs that share a column
// strip of B.  G=1: every SM reads distinct data.
// Two read paths: LDG.128 (ld.global.cg) and 1-D bulk TMA (cp.async.bulk into
// shared memory, mbarrier completion), plus TMA multicast within a cluster.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2share l2share.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// every CTA of group g = blockIdx.x / G reads [g*span, g*span + bytes_per_cta) (mod window)
__global__ void k_ldg(const float4* __restrict__ p, size_t window4, size_t per_cta4, int G, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t base = (size_t)(blockIdx.x / G) * per_cta4;
  for (size_t i = threadIdx.x; i < per_cta4; i += blockDim.x) {
    const float4 v = __ldcg(p + (base + i) % window4);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

constexpr int kStages = 4;
constexpr uint32_t kChunk = 32768;  // bytes per bulk copy

// one thread issues 1-D bulk copies of kChunk bytes into a 4-stage ring; the
// whole CTA waits on each stage and touches one word (so the data is consumed)
template <int CLUSTER>
__global__ void k_bulk(const char* __restrict__ p, size_t window, size_t per_cta, int G, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t full[kStages], empty[kStages];
  const size_t base = (size_t)(blockIdx.x / G) * per_cta;
  const int nchunks = (int)(per_cta / kChunk);
  uint32_t crank = 0;
  if (CLUSTER > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"((int)(blockDim.x / 32) * CLUSTER));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (CLUSTER > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  float acc = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % kStages;
    const uint32_t ph = (uint32_t)(c / kStages) & 1u;
    if (threadIdx.x == 0) {
      if (c >= kStages && crank == 0) {
        asm volatile("{ .reg .pred d; W%=: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1; @!d bra W%=; }" ::"r"(
                         smem_u32(&empty[s])), "r"(ph ^ 1u) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(kChunk)
                   : "memory");
      const char* src = p + (base + (size_t)c * kChunk) % window;
      if (CLUSTER == 1) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + s * kChunk)), "l"(src), "r"(kChunk), "r"(smem_u32(&full[s]))
                     : "memory");
      } else if (crank == 0) {
        // rank 0 multicasts each chunk to every CTA of the cluster
        const uint16_t mask = (uint16_t)((1u << CLUSTER) - 1u);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
                smem_u32(sm + s * kChunk)), "l"(src), "r"(kChunk), "r"(smem_u32(&full[s])), "h"(mask)
            : "memory");
      }
    }
    asm volatile("{ .reg .pred d; W%=: mbarrier.try_wait.parity.shared::cta.b64 d, [%0], %1; @!d bra W%=; }" ::"r"(
                     smem_u32(&full[s])), "r"(ph) : "memory");
    acc += reinterpret_cast<const float*>(sm + s * kChunk)[threadIdx.x * 8];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (CLUSTER == 1) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      } else {
        // release the slot in the multicasting CTA (rank 0) of the cluster
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(&empty[s])));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
    }
  }
  if (CLUSTER > 1) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  const size_t buf = (size_t)1 << 30;
  char* p;
  float* out;
  CK(cudaMalloc(&p, buf));
  CK(cudaMemset(p, 1, buf));
  CK(cudaMalloc(&out, sizeof(float) * sms * 1024));
  Timer t;
  const size_t per_cta = (size_t)64 << 20;  // 64 MiB streamed by every CTA
  for (size_t window_mb : {48, 1024}) {
    const size_t window = window_mb << 20;
    for (int G : {1, 2, 4, 8, 37, 148}) {
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        t.start();
        k_ldg<<<sms, 512>>>(reinterpret_cast<const float4*>(p), window / 16, per_cta / 16, G, out);
        float ms = t.stop();
        CK(cudaGetLastError());
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"ldg_cg_shared\", \"window_mb\": %zu, \"G\": %d, \"delivered_tb_s\": %.2f, \"unique_tb_s\": %.2f}\n",
             window_mb, G, (double)sms * per_cta / best / 1e9, (double)sms / G * per_cta / best / 1e9);
      fflush(stdout);
    }
  }
  const int smem = kStages * kChunk;
  CK(cudaFuncSetAttribute(k_bulk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_bulk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (size_t window_mb : {48, 1024}) {
    const size_t window = window_mb << 20;
    for (int G : {1, 4, 8, 37, 148}) {
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        t.start();
        k_bulk<1><<<sms, 256, smem>>>(p, window, per_cta, G, out);
        float ms = t.stop();
        CK(cudaGetLastError());
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"bulk_tma_shared\", \"window_mb\": %zu, \"G\": %d, \"delivered_tb_s\": %.2f, \"unique_tb_s\": %.2f}\n",
             window_mb, G, (double)sms * per_cta / best / 1e9, (double)sms / G * per_cta / best / 1e9);
      fflush(stdout);
    }
  }
  // multicast: clusters of C CTAs, rank 0 multicasts; groups of G=C share data
  for (int C : {2, 4}) {
    const int grid = (sms / C) * C;
    for (size_t window_mb : {48, 1024}) {
      const size_t window = window_mb << 20;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = C;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        t.start();
        cudaError_t e = C == 2 ? cudaLaunchKernelEx(&cfg, k_bulk<2>, (const char*)p, window, per_cta, C, out)
                               : cudaLaunchKernelEx(&cfg, k_bulk<4>, (const char*)p, window, per_cta, C, out);
        float ms = t.stop();
        CK(e);
        CK(cudaGetLastError());
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"bulk_tma_multicast\", \"cluster\": %d, \"window_mb\": %zu, \"delivered_tb_s\": %.2f, \"unique_tb_s\": %.2f}\n",
             C, window_mb, (double)grid * per_cta / best / 1e9, (double)grid / C * per_cta / best / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}
