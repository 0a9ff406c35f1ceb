// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tmem_ld tools/tmem_ld_probe.cu
// tcgen05.ld throughput: W warps (warp w reads TMEM lanes 32*(w%4)..+31) each
// load 32x32b.x32 (4 KB per warp-instruction) repeatedly; bytes/clk per SM.
#include <cstdio>
#include <cstdint>
#include "../paper_2105_14500_b200/csrc/kernels/sm100_ptx.cuh"
using namespace tess::sm100;
__global__ void k(long long* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
    tmem_ld32_nowait(tmem + (it & 15) * 32, r);
    tmem_wait_ld();
    reg_fence32(r);
    acc += r[it & 31];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512)); }
}
__global__ void k4(long long* out, int iters) {  // 4 loads in flight per wait
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it += 4) {
    uint32_t a[32], b[32], c[32], d[32];
    tmem_ld32_nowait(tmem + 0, a); tmem_ld32_nowait(tmem + 32, b);
    tmem_ld32_nowait(tmem + 64, c); tmem_ld32_nowait(tmem + 96, d);
    tmem_wait_ld();
    reg_fence32(a); reg_fence32(b); reg_fence32(c); reg_fence32(d);
    acc += a[it & 31] + b[3] + c[5] + d[7];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = acc; }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512)); }
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  const int iters = 4096;
  for (int w : {1, 2, 4, 8, 16}) {
    for (int v = 0; v < 2; ++v) {
      if (v == 0) k<<<1, 32 * w>>>(d, iters); else k4<<<1, 32 * w>>>(d, iters);
      long long h[2]; cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      const double bytes = (double)w * iters * 32 * 32 * 4;
      printf("%2d warps, %s: %.1f B/clk per SM (%.1f clk per warp-load)  %s\n", w, v ? "4 loads/wait" : "1 load/wait ",
             bytes / h[0], (double)h[0] / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
