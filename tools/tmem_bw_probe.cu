// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tmem_bw tools/tmem_bw_probe.cu
// tcgen05.ld throughput without register spills: W warps (warp w reads TMEM
// lanes 32*(w%4)..+31), each issuing L 32x32b.x32 loads (4 KB per
// warp-instruction) per tcgen05.wait::ld, all results folded into one
// register (constant indices, fully unrolled). Reports bytes/clk per SM and
// clk per wait. The r1 probe (tmem_ld_probe.cu) indexed its result arrays
// with a loop variable, which put them in local memory.
#include <cstdint>
#include <cstdio>

#include "../paper_2105_14500_b200/csrc/kernels/sm100_ptx.cuh"
using namespace tess::sm100;

template <int L>
__global__ void probe(long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) & 3) * 32;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[L][32];
#pragma unroll
    for (int l = 0; l < L; ++l) tmem_ld32_nowait(tmem + (uint32_t)(l * 128 % 512), r[l]);
    tmem_wait_ld();
#pragma unroll
    for (int l = 0; l < L; ++l) {
      reg_fence32(r[l]);
#pragma unroll
      for (int e = 0; e < 32; ++e) acc ^= r[l][e];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (acc == 0x12345678u) out[1] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
  }
}

template <int L>
void run(long long* d, int w) {
  const int iters = 2048;
  probe<L><<<1, 32 * w>>>(d, iters);
  long long h = 0;
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)w * iters * L * 4096.0;
  printf("%2d warps, %d loads/wait: %7.1f B/clk per SM, %6.1f clk per wait  %s\n", w, L,
         bytes / h, (double)h / iters, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int w : {1, 4, 8, 16}) {
    run<1>(d, w);
    run<2>(d, w);
    run<4>(d, w);
  }
  return 0;
}
