// Cross-GPU stream signalling for the peer windows (csrc/peer.cpp): a 1-thread
// kernel publishes a sequence number into the partner's window header with a
// system-scope release store, another spins on the local header with
// system-scope acquire loads. Stream order carries the rest: everything
// before the signal on the producer's stream (the GEMM that wrote the
// contribution) is visible to everything after the wait on the consumer's.
#include <cuda_runtime.h>

#include <cstdint>

#include "../core.h"
#include "kernels.h"

namespace tess {

namespace {

__global__ void peer_signal_kernel(uint32_t* flag, uint32_t v) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

// Spins until *flag >= v (wrap-safe); traps after `timeout_ns` so a dead
// partner surfaces as a launch error instead of a hung GPU.
__global__ void peer_wait_kernel(const uint32_t* flag, uint32_t v, uint64_t timeout_ns) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
    if (static_cast<int32_t>(x - v) >= 0) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();
    __nanosleep(256);
  }
}

__global__ void peer_fill_kernel(float* dst, size_t n, float base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = base + static_cast<float>(i % 4093);
}

__global__ void peer_check_kernel(const float* src, size_t n, float base,
                                  unsigned long long* bad) {
  unsigned long long b = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b += src[i] != base + static_cast<float>(i % 4093);
  if (b) atomicAdd(bad, b);
}

__global__ void count_mismatch_kernel(const float* a, const float* b, size_t n,
                                      unsigned long long* bad) {
  unsigned long long m = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    m += __float_as_uint(a[i]) != __float_as_uint(b[i]);
  if (m) atomicAdd(bad, m);
}

}  // namespace

void k_count_mismatch(const float* a, const float* b, size_t n, unsigned long long* bad,
                      cudaStream_t s) {
  count_mismatch_kernel<<<148, 256, 0, s>>>(a, b, n, bad);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_peer_signal(uint32_t* flag, uint32_t v, cudaStream_t s) {
  peer_signal_kernel<<<1, 1, 0, s>>>(flag, v);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_peer_wait(const uint32_t* flag, uint32_t v, cudaStream_t s) {
  peer_wait_kernel<<<1, 1, 0, s>>>(flag, v, 60ull * 1000000000ull);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_peer_fill(float* dst, size_t n, float base, cudaStream_t s) {
  peer_fill_kernel<<<148, 256, 0, s>>>(dst, n, base);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_peer_check(const float* src, size_t n, float base, unsigned long long* bad,
                  cudaStream_t s) {
  peer_check_kernel<<<148, 256, 0, s>>>(src, n, base, bad);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

}  // namespace tess
