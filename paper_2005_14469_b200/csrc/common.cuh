// common.cuh — error plumbing, launch accounting and the stream-ordered
// device allocator shared by every translation unit of libgcoo_cuda.so.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "gcoo_capi.h"

namespace gcoo_b200 {

// Thrown inside the library, converted to a status code at the C boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky-free errors so the next call starts clean
  if (e == cudaErrorMemoryAllocation) fail(GCOO_ENOMEM, std::string(what) + ": out of device memory");
  fail(GCOO_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define GCOO_CUDA(x) ::gcoo_b200::check_cuda((x), #x)

extern std::atomic<uint64_t> g_launches;

// Every kernel launch goes through this so bench.py can report how many of
// this library's kernels ran inside its timed region.
#define GCOO_LAUNCH(kernel, grid, block, smem, stream, ...)                  \
  do {                                                                       \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);              \
    ::gcoo_b200::check_cuda(cudaGetLastError(), #kernel);                    \
    ::gcoo_b200::g_launches.fetch_add(1, std::memory_order_relaxed);         \
  } while (0)

// Programmatic dependent launch (PDL) for chains of small kernels on one
// stream (the multiply's planner): the next kernel is launched while the
// previous one drains, and waits in griddep_wait() for its predecessor's
// completion and memory.  Every kernel launched this way must call
// griddep_wait() before it touches memory an earlier kernel wrote.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(const char* name, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const bool pdl_off = std::getenv("GCOO_NO_PDL") != nullptr;  // A/B switch for measurements
  cfg.numAttrs = pdl_off ? 0 : 1;
  check_cuda(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...), name);
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

#define GCOO_LAUNCH_PDL(kernel, grid, block, smem, stream, ...) \
  ::gcoo_b200::launch_pdl(#kernel, kernel, (grid), (block), (smem), (stream), __VA_ARGS__)

// Stream-ordered scratch buffer from the device's default memory pool (the
// pool keeps freed blocks, so steady-state calls do not hit cudaMalloc).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) : count(n), stream(s) {
    if (n) GCOO_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) { o.ptr = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    ptr = o.ptr; count = o.count; stream = o.stream; o.ptr = nullptr;
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
  }
  T* get() const { return ptr; }
  size_t bytes() const { return count * sizeof(T); }
};

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int ilog2(int64_t v) { int r = 0; while ((int64_t(1) << r) < v) ++r; return r; }

// Per-thread device context: the stream host-pointer entry points use.
cudaStream_t thread_stream();
int sm_count();
void ensure_pool_retains();

}  // namespace gcoo_b200
