// Persistent, warp-specialised bf16 GEMM for sm_100a (tcgen05 + TMEM + TMA).
//
// This is the B200 replacement for the reference's local block products
// matmul / matmul_nt / matmul_tn (proj/src/matrix.cpp:142-216) as called by
// nn_product_rank / nt_product_rank / tn_product_rank
// (proj/src/algorithms.cpp:34-76) and by the per-head attention loops
// (proj/src/layers.cpp:392-405, 430-448).
//
// CTA layout (192 threads, one CTA per SM, grid = min(tiles, #SMs)):
//   warp 0      TMA producer: one elected lane streams A/B k-blocks into a
//               STAGES-deep shared-memory ring (128B-swizzled boxes).
//   warp 1      MMA issuer + TMEM owner: one lane issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN, K=16) into a
//               double-buffered fp32 accumulator in tensor memory and
//               commits each stage back to the producer.
//   warps 2..5  epilogue: tcgen05.ld the accumulator (warp w reads TMEM lanes
//               32*(w%4)..+31), apply alpha / bias-free epilogue (store,
//               accumulate, residual add, exact-erf GeLU) and write C.
// The accumulator is double buffered (2*BN TMEM columns), so the epilogue of
// tile i overlaps the MMAs of tile i+1.
//
// Operand majorness is a template parameter, so the three Tesseract
// variants need no transposes in HBM:
//   NN  A K-major (row-major [M,K]),  B MN-major (row-major [K,N])
//   NT  A K-major,                    B K-major  (row-major [N,K])
//   TN  A MN-major (row-major [K,M]), B MN-major
#include "gemm.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "sm100_ptx.cuh"

namespace tess {
namespace sm100 {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int kThreads = 320;  // 2 non-epilogue + 8 epilogue warps
constexpr int kEpiHalves = 2;   // epilogue warps per TMEM lane quadrant

struct Params {
  CUtensorMap tma_a[kMaxSegments];
  CUtensorMap tma_b[kMaxSegments];
  int seg_kb[kMaxSegments];
  int nseg;
  int total_kb;
  int M, N;
  int nb0;
  int tiles_m, tiles_n, tiles_per_batch, num_tiles;
  int group_m;
  void* c;
  int c_bf16;
  long long ldc, cs0, cs1;
  const void* r;
  long long ldr, rs0, rs1;
  void* z;
  long long ldz, zs0, zs1;
  float alpha;
  int epi;
  const float* vec;
  long long vs0, vs1;
  float* stats;
  long long ss0, ss1;
  int nst, tile_n;
};

__device__ __forceinline__ float gelu_erf(float v) {
  return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
}

// d/dz of the exact-erf GeLU (ref layers.cpp:34-42)
__device__ __forceinline__ float gelu_erf_grad(float v) {
  return 0.5f * (1.0f + erff(v * 0.70710678118654752f)) +
         v * 0.39894228040143268f * __expf(-0.5f * v * v);
}

// Online (max, sum-exp) of the valid values of one 32-column chunk merged
// into the running pair of the row (RowStats epilogue).
// Works in the log2 domain: v*alpha*log2(e) via one FFMA per element feeding
// ex2.approx; the running pair is kept as (max in log2 units, sum).

__device__ __forceinline__ void row_stats_chunk(const uint32_t (&acc)[32], float alpha,
                                                int nvalid, float& rmax, float& rsum) {
  const float a2 = alpha * 1.4426950408889634f;  // alpha * log2(e)
  float cm = -INFINITY;
  if (nvalid == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) cm = fmaxf(cm, __uint_as_float(acc[j]));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) cm = fmaxf(cm, __uint_as_float(acc[j]));
  }
  if (cm == -INFINITY) return;
  cm *= a2;  // alpha > 0: max commutes with the scaling
  const float nm = fmaxf(rmax, cm);
  float s = rsum * ex2_approx(rmax - nm);
  if (nvalid == 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j) s += ex2_approx(fmaf(__uint_as_float(acc[j]), a2, -nm));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) s += ex2_approx(fmaf(__uint_as_float(acc[j]), a2, -nm));
  }
  rmax = nm;
  rsum = s;
}

// Tile index -> (batch0, batch1, m0, n0). Within a batch, tiles are grouped
// group_m tiles tall so that one wave of CTAs shares A and B panels in L2.
__device__ __forceinline__ void decode_tile(const Params& p, int tile, int& b0,
                                            int& b1, int& m0, int& n0) {
  const int b = tile / p.tiles_per_batch;
  const int r = tile - b * p.tiles_per_batch;
  b0 = b % p.nb0;
  b1 = b / p.nb0;
  const int width = p.group_m * p.tiles_n;
  const int g = r / width;
  const int first_m = g * p.group_m;
  const int gm = min(p.tiles_m - first_m, p.group_m);
  const int in = r - g * width;
  const int tm = first_m + in % gm;
  const int tn = in / gm;
  m0 = tm * BM;
  n0 = tn;  // scaled by BN by the caller
}

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

template <typename T>
__device__ __forceinline__ T* batch_ptr(void* base, long long s0, long long s1,
                                        int b0, int b1) {
  return reinterpret_cast<T*>(base) + s0 * b0 + s1 * b1;
}

// ---- epilogue ---------------------------------------------------------------
// Every loop runs over exactly 32 columns with compile-time indices (tail
// columns are predicated), so the per-thread chunk arrays stay in registers.
__device__ __forceinline__ void load32_bf16(const __nv_bfloat16* row, int nvalid, float (&o)[32]) {
  if (nvalid == 32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + q * 8);
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[q * 8 + e] = __bfloat162float(b[e]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = j < nvalid ? __bfloat162float(row[j]) : 0.f;
  }
}

__device__ __forceinline__ void load32_f32(const float* row, int nvalid, float (&o)[32]) {
  if (nvalid == 32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 f = *reinterpret_cast<const float4*>(row + q * 4);
      o[q * 4 + 0] = f.x;
      o[q * 4 + 1] = f.y;
      o[q * 4 + 2] = f.z;
      o[q * 4 + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = j < nvalid ? row[j] : 0.f;
  }
}

__device__ __forceinline__ void store32_bf16(__nv_bfloat16* row, int nvalid, const float (&v)[32]) {
  if (nvalid == 32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 out;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
      for (int e = 0; e < 4; ++e)
        o2[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
      *reinterpret_cast<uint4*>(row + q * 8) = out;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) row[j] = __float2bfloat16_rn(v[j]);
  }
}

__device__ __forceinline__ void store32_f32(float* row, int nvalid, const float (&v)[32]) {
  if (nvalid == 32) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(row + q * 4) =
          make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) row[j] = v[j];
  }
}

// Epilogue input other than the accumulator: R (Resid / DGelu / SoftmaxBwd)
// or the old C (Accum). Loaded BEFORE the tcgen05.ld of the chunk so the
// global-memory latency overlaps the TMEM read.
__device__ __forceinline__ bool epi_needs_aux(int epi) {
  return epi == (int)Epi::Resid || epi == (int)Epi::DGelu || epi == (int)Epi::SoftmaxBwd ||
         epi == (int)Epi::Accum;
}

__device__ __forceinline__ void epilogue_load_aux(const Params& p, int b0, int b1, int m, int n,
                                                  int nvalid, float (&aux)[32]) {
  if (p.epi == (int)Epi::Accum) {
    load32_f32(batch_ptr<float>(p.c, p.cs0, p.cs1, b0, b1) + (long long)m * p.ldc + n, nvalid,
               aux);
  } else if (p.c_bf16) {
    load32_bf16(batch_ptr<__nv_bfloat16>(const_cast<void*>(p.r), p.rs0, p.rs1, b0, b1) +
                    (long long)m * p.ldr + n,
                nvalid, aux);
  } else {
    load32_f32(batch_ptr<float>(const_cast<void*>(p.r), p.rs0, p.rs1, b0, b1) +
                   (long long)m * p.ldr + n,
               nvalid, aux);
  }
}

// Writes 32 consecutive columns [n, n + nvalid) of one output row.
__device__ __forceinline__ void epilogue_row_chunk(const Params& p, int b0, int b1, int m, int n,
                                                   int nvalid, const uint32_t (&acc)[32],
                                                   const float (&aux)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]) * p.alpha;
  const int epi = p.epi;
  if (epi == (int)Epi::Resid || epi == (int)Epi::Accum) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += aux[j];
  } else if (epi == (int)Epi::DGelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= gelu_erf_grad(aux[j]);
  } else if (epi == (int)Epi::SoftmaxBwd) {
    const float d = p.alpha * p.vec[p.vs0 * b0 + p.vs1 * b1 + m];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = aux[j] * (v[j] - d);
  } else if (epi == (int)Epi::SoftmaxFwd) {
    const float lse2 = p.vec[p.vs0 * b0 + p.vs1 * b1 + m];  // log2 units
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = ex2_approx(fmaf(v[j], 1.4426950408889634f, -lse2));
  } else if (epi == (int)Epi::Gelu) {
    if (p.c_bf16)
      store32_bf16(batch_ptr<__nv_bfloat16>(p.z, p.zs0, p.zs1, b0, b1) + (long long)m * p.ldz + n,
                   nvalid, v);
    else
      store32_f32(batch_ptr<float>(p.z, p.zs0, p.zs1, b0, b1) + (long long)m * p.ldz + n, nvalid,
                  v);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
  }
  if (p.c_bf16)
    store32_bf16(batch_ptr<__nv_bfloat16>(p.c, p.cs0, p.cs1, b0, b1) + (long long)m * p.ldc + n,
                 nvalid, v);
  else
    store32_f32(batch_ptr<float>(p.c, p.cs0, p.cs1, b0, b1) + (long long)m * p.ldc + n, nvalid, v);
}

// Epilogue of this thread's accumulator row m over the 32-column chunks
// half, half + kEpiHalves, ... of the tile [n0, n0 + width): two epilogue
// warps share each TMEM lane quadrant and split its chunks. RowStats writes
// one (max, sum-exp) partial per (tile, half).
__device__ __forceinline__ void epilogue_tile(const Params& p, int b0, int b1, int m, int n0,
                                              int width, uint32_t trow, int half) {
  const bool stats = p.epi == (int)Epi::RowStats;
  const bool aux_in = epi_needs_aux(p.epi);
  float rmax = -INFINITY, rsum = 0.f;
  // aux operand of chunk c is fetched one chunk ahead (software pipeline) so
  // its global-load latency hides under the previous chunk's work
  float aux[32], aux_next[32];
  auto nvalid_of = [&](int c) {
    const int n = n0 + c * 32;
    return (m < p.M && n < p.N) ? min(32, p.N - n) : 0;
  };
  if (aux_in && nvalid_of(half) > 0)
    epilogue_load_aux(p, b0, b1, m, n0 + half * 32, nvalid_of(half), aux);
#pragma unroll 1
  for (int c = half; c < width / 32; c += kEpiHalves) {
    const int n = n0 + c * 32;
    const int nvalid = nvalid_of(c);
    const int cn = c + kEpiHalves;
    if (aux_in && cn < width / 32 && nvalid_of(cn) > 0)
      epilogue_load_aux(p, b0, b1, m, n0 + cn * 32, nvalid_of(cn), aux_next);
    uint32_t r[32];
    tmem_ld32(trow + c * 32, r);  // warp-collective: executed by every lane
    if (nvalid > 0) {
      if (stats)
        row_stats_chunk(r, p.alpha, nvalid, rmax, rsum);
      else
        epilogue_row_chunk(p, b0, b1, m, n, nvalid, r, aux);
    }
    if (aux_in) {
#pragma unroll
      for (int j = 0; j < 32; ++j) aux[j] = aux_next[j];
    }
  }
  if (stats && m < p.M && n0 < p.N) {
    float* dst = p.stats +
                 (p.ss0 * b0 + p.ss1 * b1 + (long long)m * p.nst + (n0 / p.tile_n) * kEpiHalves +
                  half) * 2;
    dst[0] = rmax;
    dst[1] = rsum;
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ Params p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4 * kEpiHalves);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < p.nseg; ++s) {
      prefetch_tmap(&p.tma_a[s]);
      prefetch_tmap(&p.tma_b[s]);
    }
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            smem_u32(tmem_slot)),
        "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        int b0, b1, m0, tn;
        decode_tile(p, tile, b0, b1, m0, tn);
        const int n0 = tn * BN;
        for (int s = 0; s < p.nseg; ++s) {
          const CUtensorMap* ma = &p.tma_a[s];
          const CUtensorMap* mb = &p.tma_b[s];
          for (int kb = 0; kb < p.seg_kb[s]; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * C::STAGE_BYTES;
            uint8_t* sb = sa + C::A_BYTES;
            mbar_expect_tx(&full_bar[stage], C::STAGE_BYTES);
            const int k = kb * BK;
            if (!A_MN) {
              tma_load_4d(sa, ma, &full_bar[stage], k, m0, b0, b1);
            } else {
#pragma unroll
              for (int c = 0; c < BM / 64; ++c)
                tma_load_4d(sa + c * 8192, ma, &full_bar[stage], m0 + c * 64, k, b0, b1);
            }
            if (!B_MN) {
              tma_load_4d(sb, mb, &full_bar[stage], k, n0, b0, b1);
            } else {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c)
                tma_load_4d(sb + c * 8192, mb, &full_bar[stage], n0 + c * 64, k, b0, b1);
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      const uint32_t idesc = (1u << 4)     // D = f32
                             | (1u << 7)   // A = bf16
                             | (1u << 10)  // B = bf16
                             | ((A_MN ? 1u : 0u) << 15) | ((B_MN ? 1u : 0u) << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.total_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc(sa + k * 2048, 8192, 1024)
                                     : make_sdesc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc(sb + k * 2048, 8192, 1024)
                                     : make_sdesc(sb + k * 32, 16, 1024);
            mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // -------------------------------------------------- epilogue warps
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
      int b0, b1, m0, tn;
      decode_tile(p, tile, b0, b1, m0, tn);
      const int n0 = tn * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = m0 + quad * 32 + lane;
      const uint32_t trow = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      epilogue_tile(p, b0, b1, m, n0, BN, trow, (warp - 2) / 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(
                     tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ============================================================ 2-CTA kernel
// CTA pair (cluster of 2 on one TPC) computing a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16): each CTA stages its own 128
// rows of A and its 128-column half of B per k-block (32 KB/stage instead of
// 48 KB for the 1-CTA 128x256 tile), so shared-memory and L2 operand traffic
// per flop drop by a third. Only the leader CTA (rank 0) issues MMAs; both
// producers' TMA loads signal the leader's full barrier (peer bit cleared),
// MMA commits multicast to both CTAs' empty / tmem-full barriers, and both
// CTAs' epilogue warps release the accumulator on the leader's tmem-empty
// barrier with remote arrives.
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1),
      "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void mma_bf16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(0));
  // relaxed: the arrive only publishes "TMEM drained" (tcgen05.wait::ld has
  // completed the reads); a release would add a GPU-scope MEMBAR that waits
  // for every outstanding epilogue store of this thread.
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

template <int ST>
struct Cfg2 {
  static constexpr int HALF = 128;  // rows of A / columns of B per CTA
  static constexpr int A_BYTES = HALF * BK * 2;
  static constexpr int B_BYTES = HALF * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = ST;
  static constexpr int TMEM_COLS = 512;  // 2 accumulators x 256 fp32 columns
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

// Pair-tile index -> (batch0, batch1, m0 (multiple of 256), n0 (multiple of 256)).
__device__ __forceinline__ void decode_pair_tile(const Params& p, int tile, int& b0, int& b1,
                                                 int& m0, int& n0) {
  const int b = tile / p.tiles_per_batch;
  const int r = tile - b * p.tiles_per_batch;
  b0 = b % p.nb0;
  b1 = b / p.nb0;
  const int width = p.group_m * p.tiles_n;
  const int g = r / width;
  const int first_m = g * p.group_m;
  const int gm = min(p.tiles_m - first_m, p.group_m);
  const int in = r - g * width;
  m0 = (first_m + in % gm) * 256;
  n0 = (in / gm) * 256;
}

template <bool A_MN, bool B_MN, int ST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_2cta_kernel(const __grid_constant__ Params p) {
  using C = Cfg2<ST>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t cta = cluster_ctarank();
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8 * kEpiHalves);  // epilogue warps of both CTAs (leader's copy used)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < p.nseg; ++s) {
      prefetch_tmap(&p.tma_a[s]);
      prefetch_tmap(&p.tma_b[s]);
    }
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            smem_u32(tmem_slot)),
        "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // -------------------------------------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
        int b0, b1, m0, n0;
        decode_pair_tile(p, tile, b0, b1, m0, n0);
        const int mr = m0 + (int)cta * C::HALF;
        const int nr = n0 + (int)cta * C::HALF;
        for (int s = 0; s < p.nseg; ++s) {
          const CUtensorMap* ma = &p.tma_a[s];
          const CUtensorMap* mb = &p.tma_b[s];
          for (int kb = 0; kb < p.seg_kb[s]; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * C::STAGE_BYTES;
            uint8_t* sb = sa + C::A_BYTES;
            if (cta == 0) mbar_expect_tx(&full_bar[stage], 2 * C::STAGE_BYTES);
            const int k = kb * BK;
            if (!A_MN) {
              tma_load_4d_2sm(sa, ma, &full_bar[stage], k, mr, b0, b1);
            } else {
#pragma unroll
              for (int c = 0; c < C::HALF / 64; ++c)
                tma_load_4d_2sm(sa + c * 8192, ma, &full_bar[stage], mr + c * 64, k, b0, b1);
            }
            if (!B_MN) {
              tma_load_4d_2sm(sb, mb, &full_bar[stage], k, nr, b0, b1);
            } else {
#pragma unroll
              for (int c = 0; c < C::HALF / 64; ++c)
                tma_load_4d_2sm(sb + c * 8192, mb, &full_bar[stage], nr + c * 64, k, b0, b1);
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && cta == 0) {
      // ------------------------------------------ MMA issuer (leader CTA)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) |
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int kb = 0; kb < p.total_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? make_sdesc(sa + k * 2048, 8192, 1024)
                                     : make_sdesc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sdesc(sb + k * 2048, 8192, 1024)
                                     : make_sdesc(sb + k * 32, 16, 1024);
            mma_bf16_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          mma_commit_2sm(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2sm(&tfull_bar[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------- epilogue warps (both CTAs)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cluster; tile < p.num_tiles; tile += nclusters) {
      int b0, b1, m0, n0;
      decode_pair_tile(p, tile, b0, b1, m0, n0);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int m = m0 + (int)cta * C::HALF + quad * 32 + lane;
      const uint32_t trow = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 256;
      epilogue_tile(p, b0, b1, m, n0, 256, trow, (warp - 2) / 4);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty_bar[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  return fn;
}

// Encodes a 4-D bf16 view [inner, outer, nb0, nb1] with a {64, box_outer}
// box and 128B swizzle. Strides are in elements.
bool encode_view(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer,
                 int64_t ld, int64_t nb0, int64_t s0, int64_t nb1, int64_t s1,
                 int box_outer, std::string* err) {
  auto fn = encode_fn();
  if (!fn) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  const int64_t dense = ld * outer;
  if (nb0 <= 1) s0 = dense;
  if (nb1 <= 1) s1 = s0 * (nb0 > 1 ? nb0 : 1);
  cuuint64_t dims[4] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)nb0,
                        (cuuint64_t)nb1};
  cuuint64_t strides[3] = {(cuuint64_t)ld * 2, (cuuint64_t)s0 * 2,
                           (cuuint64_t)s1 * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int i = 0; i < 3; ++i) {
    if (strides[i] % 16 != 0) {
      *err = "bf16 GEMM operand stride not 16-byte aligned (TMA)";
      return false;
    }
  }
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) {
    *err = "bf16 GEMM operand base not 16-byte aligned (TMA)";
    return false;
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr),
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch(const Params& p, cudaStream_t stream) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;  // per instantiation; benign race
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(
        kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int grid = std::min(p.num_tiles, num_sms());
  kern<<<grid, kThreads, C::SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

template <bool A_MN, bool B_MN, int ST>
cudaError_t launch_2cta(const Params& p, cudaStream_t stream) {
  auto kern = gemm_bf16_2cta_kernel<A_MN, B_MN, ST>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg2<ST>::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int pairs = std::max(1, num_sms() / 2);
  const int grid = 2 * std::min(p.num_tiles, pairs);
  kern<<<grid, kThreads, Cfg2<ST>::SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

template <int ST>
cudaError_t launch_pair_st(const Params& p, bool a_mn, bool b_mn, cudaStream_t s) {
  if (!a_mn && b_mn) return launch_2cta<false, true, ST>(p, s);
  if (!a_mn && !b_mn) return launch_2cta<false, false, ST>(p, s);
  if (a_mn && b_mn) return launch_2cta<true, true, ST>(p, s);
  return launch_2cta<true, false, ST>(p, s);
}

cudaError_t launch_pair(const Params& p, bool a_mn, bool b_mn, cudaStream_t s) {
  static int stages = 0;  // TESS_GEMM_STAGES=6|7 (smem ring depth of the pair kernel)
  if (!stages) {
    const char* e = std::getenv("TESS_GEMM_STAGES");
    stages = (e && e[0] == '6') ? 6 : 7;
  }
  return stages == 6 ? launch_pair_st<6>(p, a_mn, b_mn, s) : launch_pair_st<7>(p, a_mn, b_mn, s);
}

bool use_pair_kernel(int64_t M, int64_t N) {
  static int mode = -1;  // TESS_GEMM_2CTA=0 forces the 1-CTA kernel (A/B testing)
  if (mode < 0) {
    const char* e = std::getenv("TESS_GEMM_2CTA");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1 && M > 128 && N > 128;
}

template <int BN>
cudaError_t launch_bn(const Params& p, bool a_mn, bool b_mn, cudaStream_t s) {
  if (!a_mn && b_mn) return launch<BN, false, true>(p, s);
  if (!a_mn && !b_mn) return launch<BN, false, false>(p, s);
  if (a_mn && b_mn) return launch<BN, true, true>(p, s);
  return launch<BN, true, false>(p, s);
}

}  // namespace sm100

namespace {
thread_local std::string g_gemm_err;
}

const char* gemm_last_error() { return g_gemm_err.c_str(); }

std::string gemm_kernel_name(const GemmDesc& d) {
  const int am = d.trans_a ? 1 : 0, bm = d.trans_b ? 0 : 1;
  if (d.in == DType::F32)
    return "gemm_f32_kernel<" + std::to_string((int)d.trans_a) + "," +
           std::to_string((int)d.trans_b) + ">";
  if (sm100::use_pair_kernel(d.M, d.N))
    return "gemm_bf16_2cta_kernel<" + std::to_string(am) + "," + std::to_string(bm) + ">";
  return "gemm_bf16_kernel<" + std::to_string(d.N > 128 ? 256 : 128) + "," + std::to_string(am) +
         "," + std::to_string(bm) + ">";
}

int gemm_bf16_stat_tiles(const GemmDesc& d) {
  const int t = gemm_bf16_tile_n(d);
  return static_cast<int>((d.N + t - 1) / t) * sm100::kEpiHalves;
}

int gemm_bf16_tile_n(const GemmDesc& d) {
  return (sm100::use_pair_kernel(d.M, d.N) || d.N > 128) ? 256 : 128;
}

cudaError_t gemm_bf16_sm100(const GemmDesc& d, cudaStream_t stream) {
  using namespace sm100;
  if (d.in != DType::BF16) {
    g_gemm_err = "gemm_bf16_sm100: inputs must be bf16";
    return cudaErrorInvalidValue;
  }
  if (d.nseg < 1 || d.nseg > kMaxSegments || d.M <= 0 || d.N <= 0) {
    g_gemm_err = "gemm_bf16_sm100: bad shape/segments";
    return cudaErrorInvalidValue;
  }
  Params p;
  std::memset(&p, 0, sizeof(p));
  const bool pair = use_pair_kernel(d.M, d.N);
  const int BN = d.N > 128 ? 256 : 128;
  // TMA box rows for K-major operands: 128 (A, and B in the pair kernel) or BN.
  const int a_box = BM;
  const int b_box = pair ? 128 : BN;
  const bool a_mn = d.trans_a;   // A stored [K, M]: M contiguous
  const bool b_mn = !d.trans_b;  // B stored [K, N]: N contiguous
  int total_kb = 0;
  for (int s = 0; s < d.nseg; ++s) {
    const int64_t K = d.seg[s].k;
    if (K <= 0 || K % 8 != 0) {
      g_gemm_err = "gemm_bf16_sm100: K must be a positive multiple of 8";
      return cudaErrorInvalidValue;
    }
    std::string err;
    bool ok;
    if (!a_mn)
      ok = encode_view(&p.tma_a[s], d.seg[s].a, K, d.M, d.lda, d.nb0, d.as0, d.nb1,
                       d.as1, a_box, &err);
    else
      ok = encode_view(&p.tma_a[s], d.seg[s].a, d.M, K, d.lda, d.nb0, d.as0, d.nb1,
                       d.as1, 64, &err);
    if (ok) {
      if (!b_mn)
        ok = encode_view(&p.tma_b[s], d.seg[s].b, K, d.N, d.ldb, d.nb0, d.bs0, d.nb1,
                         d.bs1, b_box, &err);
      else
        ok = encode_view(&p.tma_b[s], d.seg[s].b, d.N, K, d.ldb, d.nb0, d.bs0, d.nb1,
                         d.bs1, 64, &err);
    }
    if (!ok) {
      g_gemm_err = "gemm_bf16_sm100: " + err;
      return cudaErrorInvalidValue;
    }
    p.seg_kb[s] = static_cast<int>((K + BK - 1) / BK);
    total_kb += p.seg_kb[s];
  }
  const int cvec = d.c_type == DType::BF16 ? 8 : 4;
  if (d.ldc % cvec != 0 || reinterpret_cast<uintptr_t>(d.c) % 16 != 0 ||
      (d.r && (d.ldr % cvec != 0 || reinterpret_cast<uintptr_t>(d.r) % 16 != 0)) ||
      (d.z && (d.ldz % cvec != 0 || reinterpret_cast<uintptr_t>(d.z) % 16 != 0))) {
    g_gemm_err = "gemm_bf16_sm100: output rows must be 16-byte aligned";
    return cudaErrorInvalidValue;
  }
  const bool needs_r = d.epi == Epi::Resid || d.epi == Epi::DGelu || d.epi == Epi::SoftmaxBwd;
  const bool bf16_only = d.epi == Epi::DGelu || d.epi == Epi::SoftmaxFwd ||
                         d.epi == Epi::SoftmaxBwd;
  const bool needs_vec = d.epi == Epi::SoftmaxFwd || d.epi == Epi::SoftmaxBwd;
  if ((needs_r && !d.r) || (d.epi == Epi::Gelu && !d.z) ||
      (d.epi == Epi::Accum && d.c_type != DType::F32) ||
      (bf16_only && d.c_type != DType::BF16) || (needs_vec && !d.vec) ||
      (d.epi == Epi::RowStats && !d.stats)) {
    g_gemm_err = "gemm_bf16_sm100: epilogue operands missing or wrong type";
    return cudaErrorInvalidValue;
  }
  p.nseg = d.nseg;
  p.total_kb = total_kb;
  p.M = static_cast<int>(d.M);
  p.N = static_cast<int>(d.N);
  p.nb0 = static_cast<int>(d.nb0);
  const int tile_m = pair ? 256 : BM, tile_n = pair ? 256 : BN;
  p.tiles_m = static_cast<int>((d.M + tile_m - 1) / tile_m);
  p.tiles_n = static_cast<int>((d.N + tile_n - 1) / tile_n);
  p.tiles_per_batch = p.tiles_m * p.tiles_n;
  const long long nt = (long long)p.tiles_per_batch * d.nb0 * d.nb1;
  if (nt > (1ll << 31) - 1) {
    g_gemm_err = "gemm_bf16_sm100: too many tiles";
    return cudaErrorInvalidValue;
  }
  p.num_tiles = static_cast<int>(nt);
  p.group_m = pair ? 8 : 16;
  p.c = d.c;
  p.c_bf16 = d.c_type == DType::BF16;
  p.ldc = d.ldc;
  p.cs0 = d.cs0;
  p.cs1 = d.cs1;
  p.r = d.r;
  p.ldr = d.ldr;
  p.rs0 = d.rs0;
  p.rs1 = d.rs1;
  p.z = d.z;
  p.ldz = d.ldz;
  p.zs0 = d.zs0;
  p.zs1 = d.zs1;
  p.alpha = d.alpha;
  p.epi = static_cast<int>(d.epi);
  p.vec = d.vec;
  p.vs0 = d.vs0;
  p.vs1 = d.vs1;
  p.stats = d.stats;
  p.ss0 = d.ss0;
  p.ss1 = d.ss1;
  p.tile_n = tile_n;
  p.nst = static_cast<int>((d.N + tile_n - 1) / tile_n) * kEpiHalves;
  cudaError_t e = pair        ? launch_pair(p, a_mn, b_mn, stream)
                  : BN == 256 ? launch_bn<256>(p, a_mn, b_mn, stream)
                              : launch_bn<128>(p, a_mn, b_mn, stream);
  if (e != cudaSuccess) g_gemm_err = std::string("gemm_bf16_sm100 launch: ") +
                                     cudaGetErrorString(e);
  return e;
}

}  // namespace tess
