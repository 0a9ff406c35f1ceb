// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o mma2 tools/mma_rate_probe_2cta.cu
// clk per tcgen05.mma.cta_group::2 (M=256 across a CTA pair, K=16) vs N,
// issued back to back by the leader CTA (operands = zeros).
#include <cstdio>
#include <cstdint>
#include "../paper_2105_14500_b200/csrc/kernels/sm100_ptx.cuh"
using namespace tess::sm100;
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory"); }
template <int N>
__global__ void __cluster_dims__(2, 1, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before(); csync(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && ctarank() == 0) {
    constexpr uint32_t idesc = idesc_bf16(256, N, false, false);
    const uint32_t a = smem_u32(sm), b = a + 32768;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem + 256), "l"(make_sdesc(a + (kk & 3) * 32, 16, 1024)), "l"(make_sdesc(b + (kk & 3) * 32, 16, 1024)), "r"(idesc), "r"(1));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)1) : "memory");
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  tc_fence_before(); csync();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)); }
}
template <int N> void run(long long* d) {
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  int iters = 256;
  k<N><<<2, 128, 65536>>>(d, iters);
  long long h[2]; cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("cta_group::2 M=256 N=%3d: issue %.1f clk/mma, complete %.1f clk/mma (%s)\n", N, h[0] / (iters * 8.0), h[1] / (iters * 8.0), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  run<64>(d); run<128>(d); run<256>(d);
  return 0;
}
