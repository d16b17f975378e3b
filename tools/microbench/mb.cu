// Microbenchmarks that set the ceilings for the GCOOSpDM kernel on B200:
// FP32 FFMA peak (scalar and f32x2), shared-memory LDS.128 bandwidth,
// L1-hit / L2-hit / HBM read bandwidth, warp-shuffle rate, and the SM clock
// under each load.  Standalone (no torch); prints one JSON object per line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb mb.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

static int g_sms = 0;

struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() { cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); return ms; }
};

__device__ unsigned long long g_cycles[1024];

// ---------------------------------------------------------------- FFMA
__global__ void k_ffma(float* out, int iters, float x) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, x, 0.5f); a1 = fmaf(a1, x, 0.5f); a2 = fmaf(a2, x, 0.5f); a3 = fmaf(a3, x, 0.5f);
      a4 = fmaf(a4, x, 0.5f); a5 = fmaf(a5, x, 0.5f); a6 = fmaf(a6, x, 0.5f); a7 = fmaf(a7, x, 0.5f);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

// register-register-register form (x, y both registers)
__global__ void k_ffma_rrr(float* out, int iters, float x, float y) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(x, y, a[j]);
      x += 1e-7f;
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters, float x) {
  // packed f32x2 FMA (sm_100+): d = a*b + c on two lanes of a 64-bit register pair
  unsigned long long acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float lo = threadIdx.x + j, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1,%2};" : "=l"(acc[j]) : "f"(lo), "f"(hi));
  }
  unsigned long long xx, hh;
  asm("mov.b64 %0, {%1,%1};" : "=l"(xx) : "f"(x));
  float h = 0.5f;
  asm("mov.b64 %0, {%1,%1};" : "=l"(hh) : "f"(h));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[j]) : "l"(xx), "l"(hh));
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[j]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---------------------------------------------------------------- LDS
template <int VEC>
__global__ void k_lds(float* out, int iters) {
  extern __shared__ float4 sm4[];
  const int n4 = 4096;  // 64 KB
  for (int i = threadIdx.x; i < n4; i += blockDim.x) sm4[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = sm4[(idx + u * 128 + i * 32) & (n4 - 1)];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// LDS.128 feeding FFMA: the GCOOSpDM inner loop shape (1 float of smem per FMA)
__global__ void k_lds_fma(float* out, int iters) {
  extern __shared__ float4 sm4[];
  const int n4 = 4096;
  for (int i = threadIdx.x; i < n4; i += blockDim.x) sm4[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  int lane = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = sm4[((i * 8 + u) * 32 + lane) & (n4 - 1)];
      float a = 1.0f + u;
      acc[(u & 3) * 4 + 0] = fmaf(a, v.x, acc[(u & 3) * 4 + 0]);
      acc[(u & 3) * 4 + 1] = fmaf(a, v.y, acc[(u & 3) * 4 + 1]);
      acc[(u & 3) * 4 + 2] = fmaf(a, v.z, acc[(u & 3) * 4 + 2]);
      acc[(u & 3) * 4 + 3] = fmaf(a, v.w, acc[(u & 3) * 4 + 3]);
    }
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// ---------------------------------------------------------------- SHFL
__global__ void k_shfl(float* out, int iters) {
  float v = threadIdx.x, acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) { acc += __shfl_sync(0xffffffffu, v, (u + i) & 31); v += 1.0f; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// ---------------------------------------------------------------- global reads
// Each block streams a window of `win` bytes starting at a per-block offset
// (wrapping inside the buffer of `bytes`). With bytes <= a few MB every read
// after the first is an L2 hit; with bytes >> L2 it is HBM.
template <bool CG>
__global__ void k_read(const float4* __restrict__ p, size_t n4, size_t per_block, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  size_t base = (size_t)blockIdx.x * per_block;
  for (size_t i = threadIdx.x; i < per_block; i += blockDim.x) {
    size_t j = (base + i) % n4;
    float4 v;
    if (CG) v = __ldcg(p + j); else v = __ldg(p + j);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// L1-hit: every block re-reads its own 64 KB window many times
__global__ void k_l1(const float4* __restrict__ p, int reps, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const float4* q = p + (size_t)blockIdx.x * 4096;
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) {
      float4 v = __ldg(q + ((i + r * 32) & 4095));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

static double clock_mhz(int nblocks, float ms) {
  std::vector<unsigned long long> c(1024);
  cudaMemcpyFromSymbol(c.data(), g_cycles, sizeof(unsigned long long) * 1024);
  int n = nblocks < 1024 ? nblocks : 1024;
  double mx = 0;
  for (int i = 0; i < n; ++i) if (c[i] > mx) mx = c[i];
  return mx / (ms * 1e3);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_per_block_optin\": %zu, \"regs_per_sm\": %d}\n",
         prop.name, g_sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin, prop.regsPerMultiprocessor);
  float* out;
  CK(cudaMalloc(&out, sizeof(float) * 148 * 64 * 1024));
  Timer t;

  // FFMA peak: 148*8 blocks of 256 threads
  {
    int blocks = g_sms * 8, th = 256, iters = 4000;
    k_ffma<<<blocks, th>>>(out, 10, 1.0001f);
    CK(cudaDeviceSynchronize());
    float best = 1e30f; double mhz = 0;
    for (int r = 0; r < 5; ++r) {
      t.start(); k_ffma<<<blocks, th>>>(out, iters, 1.0001f); float ms = t.stop();
      if (ms < best) { best = ms; mhz = clock_mhz(blocks, ms); }
    }
    double fma = (double)blocks * th * iters * 16 * 8;
    printf("{\"test\": \"ffma_imm\", \"tflops\": %.2f, \"fma_per_clk_per_sm\": %.1f, \"sm_mhz_est\": %.0f}\n",
           2 * fma / best / 1e9, fma / (best * 1e-3) / (mhz * 1e6) / g_sms, mhz);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      t.start(); k_ffma_rrr<<<blocks, th>>>(out, iters, 1.0001f, 0.999f); float ms = t.stop();
      if (ms < best) best = ms;
    }
    printf("{\"test\": \"ffma_rrr\", \"tflops\": %.2f, \"fma_per_clk_per_sm@est\": %.1f}\n",
           2 * fma / best / 1e9, fma / (best * 1e-3) / (mhz * 1e6) / g_sms);
    best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      t.start(); k_ffma2<<<blocks, th>>>(out, iters, 1.0001f); float ms = t.stop();
      if (ms < best) best = ms;
    }
    printf("{\"test\": \"ffma2_f32x2\", \"tflops\": %.2f, \"fma_per_clk_per_sm@est\": %.1f}\n",
           2 * 2 * fma / best / 1e9, 2 * fma / (best * 1e-3) / (mhz * 1e6) / g_sms);
  }
  // LDS.128 bandwidth
  {
    int th = 512, iters = 4000;
    CK(cudaFuncSetAttribute(k_lds<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_lds_fma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    for (int per_sm : {1, 2, 3}) {
      int blocks = g_sms * per_sm;
      k_lds<4><<<blocks, th, 65536>>>(out, 10);
      CK(cudaDeviceSynchronize());
      float best = 1e30f; double mhz = 0;
      for (int r = 0; r < 5; ++r) {
        t.start(); k_lds<4><<<blocks, th, 65536>>>(out, iters); float ms = t.stop();
        if (ms < best) { best = ms; mhz = clock_mhz(blocks, ms); }
      }
      double bytes = (double)blocks * th * iters * 8 * 16;
      printf("{\"test\": \"lds128\", \"ctas_per_sm\": %d, \"tb_s\": %.2f, \"bytes_per_clk_per_sm\": %.1f, \"sm_mhz_est\": %.0f}\n",
             per_sm, bytes / best / 1e9, bytes / (best * 1e-3) / (mhz * 1e6) / g_sms, mhz);
    }
    int blocks = g_sms * 2;
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      t.start(); k_lds_fma<<<blocks, th, 65536>>>(out, iters); float ms = t.stop();
      if (ms < best) best = ms;
    }
    double fma = (double)blocks * th * iters * 8 * 4;
    printf("{\"test\": \"lds128_ffma_1float_per_fma\", \"tflops\": %.2f}\n", 2 * fma / best / 1e9);
  }
  // SHFL
  {
    int blocks = g_sms * 4, th = 512, iters = 4000;
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      t.start(); k_shfl<<<blocks, th>>>(out, iters); float ms = t.stop();
      if (ms < best) best = ms;
    }
    double warp_ops = (double)blocks * (th / 32) * iters * 16;
    printf("{\"test\": \"shfl\", \"warp_shfl_per_ns\": %.1f, \"per_sm_per_ns\": %.3f}\n",
           warp_ops / (best * 1e6), warp_ops / (best * 1e6) / g_sms);
  }
  // global reads: L1-hit, L2-hit windows, HBM
  {
    size_t big = (size_t)4 << 30;  // 4 GiB
    float4* p;
    CK(cudaMalloc(&p, big));
    CK(cudaMemset(p, 0, big));
    int th = 512;
    {
      int blocks = g_sms * 2, reps = 400;
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        t.start(); k_l1<<<blocks, th>>>(p, reps, out); float ms = t.stop();
        if (ms < best) best = ms;
      }
      double bytes = (double)blocks * reps * 4096 * 16;
      printf("{\"test\": \"l1_hit_ldg128\", \"tb_s\": %.2f}\n", bytes / best / 1e9);
    }
    for (size_t win_mb : {8, 32, 96}) {
      size_t n4 = win_mb * (1 << 20) / 16;
      int blocks = g_sms * 4;
      size_t per_block = (size_t)1 << 20;  // 16 MB per block of float4 reads
      for (int cg = 0; cg < 2; ++cg) {
        float best = 1e30f;
        for (int r = 0; r < 4; ++r) {
          t.start();
          if (cg) k_read<true><<<blocks, th>>>(p, n4, per_block, out);
          else k_read<false><<<blocks, th>>>(p, n4, per_block, out);
          float ms = t.stop();
          if (ms < best) best = ms;
        }
        double bytes = (double)blocks * per_block * 16;
        printf("{\"test\": \"l2_window_read\", \"window_mb\": %zu, \"cg\": %d, \"tb_s\": %.2f}\n", win_mb, cg, bytes / best / 1e9);
      }
    }
    {
      size_t n4 = big / 16;
      int blocks = g_sms * 4;
      size_t per_block = n4 / blocks;
      float best = 1e30f;
      for (int r = 0; r < 4; ++r) {
        t.start(); k_read<true><<<blocks, th>>>(p, n4, per_block, out); float ms = t.stop();
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"hbm_read\", \"tb_s\": %.2f}\n", (double)blocks * per_block * 16 / best / 1e9);
    }
    CK(cudaFree(p));
  }
  return 0;
}
