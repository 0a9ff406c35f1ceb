// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma_rate tools/mma_rate_probe.cu
// clk per tcgen05.mma (cta_group::1, kind::f16, M=128, K=16) vs N, SS and TS
// operand sources, issued back to back by one thread (operands = zeros).
#include <cstdio>
#include <cstdint>
#include "../paper_2105_14500_b200/csrc/kernels/sm100_ptx.cuh"
using namespace tess::sm100;
template <int N, bool TS>
__global__ void k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, N, false, false);
    const uint32_t a = smem_u32(sm), b = a + 32768;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (TS) mma_bf16_ts(tmem + 256, tmem + 0 + kk * 8, make_sdesc(b + (kk & 3) * 32, 16, 1024), idesc, 1);
        else mma_bf16(tmem + 256, make_sdesc(a + (kk & 3) * 32, 16, 1024), make_sdesc(b + (kk & 3) * 32, 16, 1024), idesc, 1);
      }
    }
    long long t1 = clock64();
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)); }
}
template <int N, bool TS> void run(long long* d) {
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  int iters = 256;
  k<N, TS><<<1, 128, 65536>>>(d, iters);
  long long h[2]; cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d %s: issue %.1f clk/mma, complete %.1f clk/mma  (%s)\n", N, TS ? "TS" : "SS", h[0] / (iters * 8.0), h[1] / (iters * 8.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  run<64, false>(d); run<64, true>(d); run<128, false>(d); run<128, true>(d); run<256, false>(d); run<256, true>(d);
  return 0;
}
