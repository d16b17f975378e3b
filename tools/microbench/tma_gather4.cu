// TMA gather4: four arbitrary rows of a row-major fp32 matrix (box = W x 1)
// land back to back in shared memory with one instruction.  Checks the
// layout and times gathered vs tiled loads of the same number of B rows.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather4 tma_gather4.cu -lcuda && ./tma_gather4
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int W = 128, ROWS = 192;

__global__ void k_gather(const __grid_constant__ CUtensorMap map, const int* __restrict__ idx, int nidx,
                         const float* __restrict__ g, int* bad, long long* cyc, int iters) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                   "r"(nidx * W * 4));
      for (int q = 0; q < nidx; q += 4)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(sm + q * W * 4)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(idx[q]), "r"(idx[q + 1]), "r"(idx[q + 2]),
            "r"(idx[q + 3]), "r"(smem_u32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(
            smem_u32(&bar)),
        "r"(phase));
    phase ^= 1;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  const float* s = reinterpret_cast<const float*>(sm);
  int nb = 0;
  for (int i = threadIdx.x; i < nidx * W; i += blockDim.x)
    if (s[i] != g[(size_t)idx[i / W] * W + (i % W)]) ++nb;
  atomicAdd(bad, nb);
}

int main() {
  const int K = 8000;
  float* g;
  CK(cudaMalloc(&g, (size_t)K * W * 4));
  float* h = (float*)malloc((size_t)K * W * 4);
  for (size_t i = 0; i < (size_t)K * W; ++i) h[i] = (float)i;
  CK(cudaMemcpy(g, h, (size_t)K * W * 4, cudaMemcpyHostToDevice));
  CUtensorMap map;
  const cuuint64_t dims[2] = {W, (cuuint64_t)K};
  const cuuint64_t strides[1] = {W * 4};
  const cuuint32_t box[2] = {W, 1};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, g, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  int hidx[ROWS];
  for (int i = 0; i < ROWS; ++i) hidx[i] = (i * 37 + 11) % K;
  int *idx, *bad;
  long long* cyc;
  CK(cudaMalloc(&idx, sizeof hidx));
  CK(cudaMalloc(&bad, 4));
  CK(cudaMalloc(&cyc, 8));
  CK(cudaMemcpy(idx, hidx, sizeof hidx, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, ROWS * W * 4));
  for (int n : {4, 80, 192}) {
    CK(cudaMemset(bad, 0, 4));
    k_gather<<<1, 256, ROWS * W * 4>>>(map, idx, n, g, bad, cyc, 200);
    CK(cudaDeviceSynchronize());
    int hb;
    long long hc;
    CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
    printf("{\"test\": \"tma gather4\", \"rows\": %d, \"mismatches\": %d, \"cycles_per_fill\": %.0f, \"bytes_per_clk\": %.1f}\n",
           n, hb, hc / 200.0, n * W * 4 / (hc / 200.0));
  }
  return 0;
}
