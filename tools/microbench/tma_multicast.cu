// TMA multicast vs unicast for the B-tile stream of spdm_tacc (sparse end).
//
// Every CTA streams the KC x 128 fp32 tiles of one 4 MB column strip (the
// kernel's B-tile stream: same strip for the CTAs of neighbouring row blocks)
// through a 2-stage shared-memory ring.  csz = 1: each CTA loads whole tiles
// itself (what the kernel does).  csz = 2/4/8: a cluster of csz CTAs shares
// each tile — rank r loads rows [r*KC/csz, (r+1)*KC/csz) with
// .multicast::cluster to all csz CTAs, and a stage is refilled only after
// every CTA of the cluster released it (remote mbarrier arrives).
// Reports delivered bytes per SM per clock and chip TB/s, and checks the
// delivered tile contents.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_multicast tma_multicast.cu -lcuda && ./tma_multicast
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int W = 128, KC = 192, STAGES = 2, K = 8000;
constexpr int TILE = KC * W * 4;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(bar),
               "r"(ph) : "memory");
}

__global__ void __launch_bounds__(64) k_stream(const __grid_constant__ CUtensorMap map, int csz, int nstrips,
                                               int iters, long long* cyc, int* bad) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const uint32_t rank = csz > 1 ? cluster_rank() : 0;
  const int cluster = blockIdx.x / csz;
  const int strip = cluster % nstrips;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(csz));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (csz > 1) cluster_sync(); else __syncthreads();
  const int nch = (K + KC - 1) / KC;
  const int total = nch * iters;
  const int rows = KC / csz;
  long long t0 = clock64();
  if (threadIdx.x == 0) {                       // producer
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      if (i >= STAGES) wait(smem_u32(&empty[s]), ((i / STAGES) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(TILE)
                   : "memory");
      const int y = (i % nch) * KC + rank * rows;
      const uint32_t dst = smem_u32(sm + s * TILE + rank * rows * W * 4);
      if (csz == 1)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&map)),
                     "r"(strip * W), "r"(y), "r"(smem_u32(&full[s])) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
                     " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst), "l"(reinterpret_cast<uint64_t>(&map)),
                     "r"(strip * W), "r"(y), "r"(smem_u32(&full[s])), "h"((uint16_t)((1u << csz) - 1)) : "memory");
    }
  } else if (threadIdx.x == 32) {               // consumer: wait, spot-check, release cluster-wide
    int nb = 0;
    for (int i = 0; i < total; ++i) {
      const int s = i % STAGES;
      wait(smem_u32(&full[s]), (i / STAGES) & 1);
      const float* t = reinterpret_cast<const float*>(sm + s * TILE);
      const int r = (i * 37) % KC, c = (i * 11) % W;
      const int gy = (i % nch) * KC + r;
      const float want = gy < K ? (float)(gy * 1024 + strip * W + c) : 0.f;
      if (t[r * W + c] != want) ++nb;
      for (int q = 0; q < csz; ++q) {
        if (csz == 1) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        } else {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[s])), "r"(q));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
      }
    }
    if (nb) atomicAdd(bad, nb);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (csz > 1) cluster_sync();
}

int main() {
  const int NSTR = 1024 / W;                     // B is K x 1024 fp32: 8 column strips of 4 MB
  float* g;
  CK(cudaMalloc(&g, (size_t)K * 1024 * 4));
  std::vector<float> h((size_t)K * 1024);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  CK(cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap map;
  const cuuint64_t dims[2] = {1024, (cuuint64_t)K};
  const cuuint64_t strides[1] = {1024 * 4};
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  long long* cyc;
  int* bad;
  CK(cudaMalloc(&cyc, 8 * 1024));
  CK(cudaMalloc(&bad, 4));
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * TILE));
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const int iters = 40;
  for (int csz : {1, 2, 4, 8}) {
    const cuuint32_t box[2] = {W, (cuuint32_t)(KC / csz)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int grid = sms / csz * csz;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = STAGES * TILE;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemset(bad, 0, 4));
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0));
      CK(cudaLaunchKernelEx(&cfg, k_stream, map, csz, NSTR, iters, cyc, bad));
      CK(cudaEventRecord(e1));
      CK(cudaDeviceSynchronize());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::vector<long long> hc(grid);
      int hb;
      CK(cudaMemcpy(hc.data(), cyc, 8 * grid, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
      long long mx = 0;
      for (long long c : hc) mx = c > mx ? c : mx;
      const double per_sm = (double)((K + KC - 1) / KC) * iters * TILE;
      if (rep)
        printf("{\"test\": \"tma_b_stream\", \"cluster\": %d, \"ctas\": %d, \"mismatches\": %d, \"bytes_per_clk_per_sm\": %.1f,"
               " \"delivered_tb_s\": %.2f, \"l2_read_tb_s\": %.2f, \"ms\": %.3f}\n",
               csz, grid, hb, per_sm / mx, per_sm * grid / (ms * 1e9), per_sm * grid / csz / (ms * 1e9), ms);
    }
  }
  return 0;
}
