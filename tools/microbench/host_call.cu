// Host cost of the C ABI calls without Python: gcoo_plan_spdm_f32_dev and the
// planned gcoo_spdm_f32_dev, with the device held busy so calls only enqueue.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../../include -o host_call host_call.cu \
//        -L../../paper_2005_14469_b200/lib -lgcoo_cuda -Xlinker -rpath=$PWD/../../paper_2005_14469_b200/lib
#include <cuda_runtime.h>
#include <algorithm>
#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda.h>

#include "gcoo_capi.h"

__global__ void empty_k(const __grid_constant__ CUtensorMap m, int x) {
  if (x == 12345) printf("%p", &m);
}
__global__ void __launch_bounds__(928, 1) big_k(const __grid_constant__ CUtensorMap m, int x) {
  extern __shared__ unsigned char sm[];
  if (x == 12345) printf("%p %d", &m, sm[threadIdx.x]);
}

__global__ void spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

int main() {
  const int64_t n = 8000, nnz_cap = n * n / 50;
  std::vector<float> a((size_t)n * n);
  gcoo_generate_uniform_sparse_f32(n, 0.99, 1, a.data());
  float *dA, *dB, *dC, *vals;
  int32_t *rows, *cols;
  int64_t *gidx, *gnnz, nnz = 0;
  cudaMalloc(&dA, n * n * 4);
  cudaMalloc(&dB, n * n * 4);
  cudaMalloc(&dC, n * n * 4);
  cudaMalloc(&vals, nnz_cap * 4);
  cudaMalloc(&rows, nnz_cap * 4);
  cudaMalloc(&cols, nnz_cap * 4);
  cudaMalloc(&gidx, n / 4 * 8);
  cudaMalloc(&gnnz, n / 4 * 8);
  cudaMemcpy(dA, a.data(), n * n * 4, cudaMemcpyHostToDevice);
  cudaMemset(dB, 0, n * n * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (gcoo_dense_to_gcoo_f32_dev(n, n, 4, dA, nnz_cap, vals, rows, cols, gidx, gnnz, &nnz, s)) {
    printf("construct failed: %s\n", gcoo_last_error());
    return 1;
  }
  gcoo_plan* plan = nullptr;
  if (gcoo_plan_create_f32_dev(n, n, 4, nnz, vals, rows, cols, n / 4, gidx, gnnz, GCOO_FLAVOR_FMA, &plan, s)) {
    printf("plan failed: %s\n", gcoo_last_error());
    return 1;
  }
  auto spdm = [&] {
    gcoo_spdm_f32_dev(n, n, n, 4, 64, nnz, vals, rows, cols, n / 4, gidx, gnnz, dB, n, dC, n, nullptr,
                      GCOO_FLAVOR_FMA, s);
  };
  auto prun = [&] { gcoo_plan_spdm_f32_dev(plan, n, dB, n, dC, n, s); };
  auto prun_narrow = [&] { gcoo_plan_spdm_f32_dev(plan, 128, dB, n, dC, n, s); };
  for (int64_t w : {1024, 2048, 4096, 8000}) {
    double idle = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      cudaStreamSynchronize(s);
      const auto i0 = std::chrono::steady_clock::now();
      gcoo_plan_spdm_f32_dev(plan, w, dB, n, dC, n, s);
      const auto i1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      const auto i2 = std::chrono::steady_clock::now();
      idle = std::min(idle, std::chrono::duration<double, std::micro>(i1 - i0).count());
      if (rep == 2) printf("{\"plan_call_idle_n\": %lld, \"host_us\": %.1f, \"call_to_sync_us\": %.1f}\n", (long long)w, idle,
                           std::chrono::duration<double, std::micro>(i2 - i0).count());
    }
  }
  for (int i = 0; i < 3; ++i) spdm(), prun();
  cudaStreamSynchronize(s);
  for (auto [name, fn] : {std::pair<const char*, std::function<void()>>{"spdm_f32_dev", spdm}, {"plan_spdm_f32_dev", prun},
                          {"plan_spdm_f32_dev_n128", prun_narrow}}) {
    double best = 1e30, idle = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      const auto i0 = std::chrono::steady_clock::now();
      fn();
      const auto i1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      idle = std::min(idle, std::chrono::duration<double, std::micro>(i1 - i0).count());
      spin<<<1, 1, 0, s>>>(200000000LL);
      const auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < 20; ++i) fn();
      const auto t1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(s);
      best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / 20);
    }
    printf("{\"call\": \"%s\", \"host_us\": %.1f, \"single_call_idle_device_us\": %.1f}\n", name, best, idle);
  }
  // pieces of a launch
  CUtensorMap map;
  {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(p);
    const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)n * 4};
    const cuuint32_t box[2] = {128, 192};
    const cuuint32_t es[2] = {1, 1};
    auto encode = [&] {
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    cudaFuncSetAttribute(big_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 229376);
    auto launch = [&](bool big, bool pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1008);
      cfg.blockDim = dim3(big ? 928 : 64);
      cfg.dynamicSmemBytes = big ? 229376 : 0;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      if (big) cudaLaunchKernelEx(&cfg, big_k, map, 0);
      else cudaLaunchKernelEx(&cfg, empty_k, map, 0);
    };
    std::vector<std::pair<const char*, std::function<void()>>> probes = {
        {"tensor_map_encode", encode},
        {"launch_small", [&] { launch(false, false); }},
        {"launch_small_pdl", [&] { launch(false, true); }},
        {"launch_big_smem", [&] { launch(true, false); }},
        {"launch_big_smem_pdl", [&] { launch(true, true); }},
        {"malloc_free_async_1MB", [&] { void* q; cudaMallocAsync(&q, 1 << 20, s); cudaFreeAsync(q, s); }}};
    for (auto& [name, fn] : probes) {
      double best = 1e30;
      for (int rep = 0; rep < 3; ++rep) {
        spin<<<1, 1, 0, s>>>(200000000LL);
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 20; ++i) fn();
        const auto t1 = std::chrono::steady_clock::now();
        cudaStreamSynchronize(s);
        best = std::min(best, std::chrono::duration<double, std::micro>(t1 - t0).count() / 20);
      }
      printf("{\"call\": \"%s\", \"host_us\": %.2f}\n", name, best);
    }
  }
  gcoo_plan_destroy(plan);
  return 0;
}
