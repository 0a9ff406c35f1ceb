// Persistent, warp-specialised bf16 GEMM for sm_100a (tcgen05 + TMEM + TMA).
//
// This is the B200 replacement for the reference's local block products
// matmul / matmul_nt / matmul_tn (proj/src/matrix.cpp:142-216) as called by
// nn_product_rank / nt_product_rank / tn_product_rank
// (proj/src/algorithms.cpp:34-76) and by the per-head attention loops
// (proj/src/layers.cpp:392-405, 430-448).
//
// Two kernels, both persistent and warp-specialised (320 threads, one CTA per
// SM):
//   warp 0      TMA producer: one elected lane streams A/B k-blocks into a
//               STAGES-deep shared-memory ring (128B-swizzled boxes).
//   warp 1      MMA issuer + TMEM owner: one lane issues tcgen05.mma into
//               fp32 accumulators in tensor memory and commits each stage
//               back to the producer.
//   warps 2..9  epilogue: two warps per TMEM lane quadrant (warp w reads
//               lanes 32*(w%4)..+31) split the 32-column chunks; alpha and the
//               fused epilogue (store, accumulate, residual add, exact-erf
//               GeLU / GeLU', softmax forward / backward, row statistics).
// * gemm_bf16_kernel<BN>: one CTA, M=128 x N=BN MMAs (cta_group::1), the
//   accumulator double buffered (2*BN TMEM columns) so the epilogue of tile i
//   overlaps the MMAs of tile i+1; used for N <= 128.
// * gemm_bf16_2cta_kernel<.., NH, BNP>: a CTA pair on one TPC
//   (cta_group::2, M=256 x N=BNP MMAs, each CTA stages half of A and half of
//   B); pair tiles 256 x 256 (two TMEM accumulators) or 256 x 512 (NH = 2:
//   both 256-column halves in TMEM, a quarter less L2->SM traffic per flop,
//   TMA-store / TMA-reduce-add epilogue); tiles handed out in order from an
//   atomic counter so concurrently running tiles share their A/B panels in
//   L2, odd waves walking K backwards (serpentine) and, for 256 x 512 tiles,
//   the next tile's half-0 MMAs leading while the epilogue drains half 1.
//   (DESIGN.md section 3 has the measurements behind each choice.)
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

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
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
  // TMA-store epilogue (pair kernel): C and Z views [N, M, nb0, nb1], box
  // {32 bf16 | 16 f32 columns, 32 rows}, SWIZZLE_64B (64-byte box rows)
  CUtensorMap tma_c, tma_z;
  int tma_epi;
  int seg_kb[kMaxSegments];
  int nseg;
  int total_kb;
  int M, N;
  int nb0;
  int tiles_m, tiles_n, tiles_per_batch, num_tiles;
  // pair kernel, NH = 2: tile ids >= num_full are HALF tiles (256 x 256):
  // the tiles of a partial last wave, split in two so they fill the pairs a
  // 256 x 512 remainder would leave idle (id num_full + 2t + h = half h of
  // full tile num_full + t); num_tiles counts both kinds
  int num_full;
  int group_m;
  int mma_lead;                 // NH == 2: half-0 MMAs lead while half 1 drains
  int* tile_counter;            // pair kernel: dynamic tile order (zeroed per launch)
  // Pair kernel: the first wave takes tiles = pair index, later ones
  // wave + atomicAdd(tile_counter); odd waves walk K backwards (serpentine).
  int wave;
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
  // fused bias / dropout (GemmDesc)
  const float* bias;
  int drop;
  uint32_t drop_thresh;
  float drop_scale;
  unsigned long long drop_seed;
  long long drop_row0, drop_col0;
  // segment readiness (GemmReady)
  int rdy;
  const uint32_t* rdy_a[kMaxSegments];
  const uint32_t* rdy_b[kMaxSegments];
  uint32_t rdy_ea[kMaxSegments], rdy_eb[kMaxSegments];
  int rdy_chunks, rdy_chunk_rows;
};

// Producer-side wait for a panel chunk delivered while the GEMM runs
// (GemmReady). `seen` caches satisfied (segment, chunk) pairs of this
// producer: one system-scope acquire load per pair, then nothing. The proxy
// fence orders the acquire before the async-proxy (TMA) reads of the panel.
// A panel that never lands traps after 120 s instead of hanging the GPU.
__device__ __noinline__ void wait_flag(const uint32_t* f, uint32_t epoch) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 120ull * 1000000000ull) __trap();
    __nanosleep(128);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void wait_seg_a(const Params& p, int s, int row, uint64_t& seen) {
  const uint32_t* f = p.rdy_a[s];
  if (!f) return;
  int c = p.rdy_chunk_rows ? row / p.rdy_chunk_rows : 0;
  if (c >= p.rdy_chunks) c = p.rdy_chunks - 1;
  const int bit = s * p.rdy_chunks + c;  // < 32 (host checks chunks * nseg)
  if ((seen >> bit) & 1ull) return;
  wait_flag(f + c, p.rdy_ea[s]);
  seen |= 1ull << bit;
}

__device__ __forceinline__ void wait_seg_b(const Params& p, int s, uint64_t& seen) {
  const uint32_t* f = p.rdy_b[s];
  if (!f) return;
  const int bit = 32 + s;  // B panels cached in the high word
  if ((seen >> bit) & 1ull) return;
  wait_flag(f, p.rdy_eb[s]);
  seen |= 1ull << bit;
}

// Exact-erf GeLU for the tcgen05 epilogues (ref layers.cpp:25-42), whose
// outputs are stored in bf16: Phi(x) = 0.5 (1 + erf(x / sqrt 2)) by
// Abramowitz & Stegun 7.1.26 (|erf error| <= 1.5e-7, far below bf16's 2^-9),
// sharing one exp2 with phi(x) = exp(-x^2/2) / sqrt(2 pi):
//   E = exp(-x^2/2), t = 1 / (1 + p |x| / sqrt 2),
//   Q = 0.5 t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) E  = Phi(-|x|)
//   Phi(x) = x >= 0 ? 1 - Q : Q;  gelu = x Phi;  gelu' = Phi + x phi.
// Two MUFU ops (ex2, rcp) and ~12 FMA-pipe ops instead of erff + expf.
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void gelu_phi(float x, float& Phi, float& E) {
  E = ex2_approx(-0.72134752044448170f * x * x);  // exp(-x^2/2) = 2^(-x^2 log2(e)/2)
  const float t = rcp_approx(fmaf(0.23164190f, fabsf(x), 1.0f));  // p / sqrt 2
  float q = fmaf(t, 1.061405429f, -1.453152027f);
  q = fmaf(t, q, 1.421413741f);
  q = fmaf(t, q, -0.284496736f);
  q = fmaf(t, q, 0.254829592f);
  const float Q = 0.5f * t * q * E;
  Phi = x >= 0.f ? 1.0f - Q : Q;
}

__device__ __forceinline__ float gelu_erf(float v) {
  float Phi, E;
  gelu_phi(v, Phi, E);
  return v * Phi;
}

// d/dz of the exact-erf GeLU (ref layers.cpp:34-42)
__device__ __forceinline__ float gelu_erf_grad(float v) {
  float Phi, E;
  gelu_phi(v, Phi, E);
  return fmaf(v * 0.39894228040143268f, E, Phi);
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

// Bias of columns [n, n + 32) (clamped to N: columns past it are clipped).
__device__ __forceinline__ void add_bias32(const Params& p, int n, float (&v)[32]) {
  if (!p.bias) return;
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] += __ldg(p.bias + min(n + j, p.N - 1));
}

__device__ __forceinline__ void dropout32(const Params& p, int m, int n, float (&v)[32]) {
  if (!p.drop) return;
  const unsigned long long row = (unsigned long long)(p.drop_row0 + m);
#pragma unroll
  for (int j = 0; j < 32; ++j)
    v[j] = dropout_keep(p.drop_seed, row, (unsigned long long)(p.drop_col0 + n + j),
                        p.drop_thresh)
               ? v[j] * p.drop_scale
               : 0.f;
}

// Writes 32 consecutive columns [n, n + nvalid) of one output row.
__device__ __forceinline__ void epilogue_row_chunk(const Params& p, int b0, int b1, int m, int n,
                                                   int nvalid, const uint32_t (&acc)[32],
                                                   const float (&aux)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]) * p.alpha;
  add_bias32(p, n, v);
  const int epi = p.epi;
  if (epi == (int)Epi::Resid || epi == (int)Epi::Accum) {
    dropout32(p, m, n, v);
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
    dropout32(p, m, n, v);
  } else if (epi == (int)Epi::Store) {
    dropout32(p, m, n, v);
  }
  if (p.c_bf16)
    store32_bf16(batch_ptr<__nv_bfloat16>(p.c, p.cs0, p.cs1, b0, b1) + (long long)m * p.ldc + n,
                 nvalid, v);
  else
    store32_f32(batch_ptr<float>(p.c, p.cs0, p.cs1, b0, b1) + (long long)m * p.ldc + n, nvalid, v);
}

// v = epilogue(alpha * acc) for one 32-column chunk of row m, without
// storing (TMA-store path); for Gelu v is the pre-activation (the GeLU is
// applied after Z is staged). Rows past M (partial tiles) compute garbage
// that the TMA store clips.
__device__ __forceinline__ void epilogue_values(const Params& p, int b0, int b1, int m, int n,
                                                const uint32_t (&acc)[32], const float (&aux)[32],
                                                float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]) * p.alpha;
  add_bias32(p, n, v);
  const int epi = p.epi;
  const bool in_m = m < p.M;
  if (epi == (int)Epi::Store || epi == (int)Epi::Accum) {
    dropout32(p, m, n, v);
  } else if (epi == (int)Epi::Resid) {
    dropout32(p, m, n, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += aux[j];
  } else if (epi == (int)Epi::DGelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= gelu_erf_grad(aux[j]);
  } else if (epi == (int)Epi::SoftmaxBwd) {
    const float d = in_m ? p.alpha * p.vec[p.vs0 * b0 + p.vs1 * b1 + m] : 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = aux[j] * (v[j] - d);
  } else if (epi == (int)Epi::SoftmaxFwd) {
    const float lse2 = in_m ? p.vec[p.vs0 * b0 + p.vs1 * b1 + m] : 0.f;  // log2 units
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = ex2_approx(fmaf(v[j], 1.4426950408889634f, -lse2));
  }
}

// Per-warp double-buffered staging of 32 rows x 64 bytes for the TMA store
// epilogue (SWIZZLE_64B: 16-byte unit u of row r at u ^ ((r >> 1) & 3), which
// keeps the 8-lane phases of st.shared.v4 conflict-free).
struct EpiStage {
  uint32_t buf;  // two 2 KB buffers
  int bi;
};

__device__ __forceinline__ void stage_store(const CUtensorMap* map, EpiStage& st, int lane,
                                            const float* v, bool bf16, bool reduce, int n,
                                            int mrow0, int b0, int b1) {
  const uint32_t dst = st.buf + (uint32_t)st.bi * 2048u;
  if (lane == 0) bulk_wait_read<1>();  // the store issued from this buffer 2 units ago
  __syncwarp();
  const uint32_t row = dst + (uint32_t)lane * 64u;
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint32_t a, b, c, d;
    if (bf16) {
      a = pack_bf16x2(v[u * 8 + 0], v[u * 8 + 1]);
      b = pack_bf16x2(v[u * 8 + 2], v[u * 8 + 3]);
      c = pack_bf16x2(v[u * 8 + 4], v[u * 8 + 5]);
      d = pack_bf16x2(v[u * 8 + 6], v[u * 8 + 7]);
    } else {
      a = __float_as_uint(v[u * 4 + 0]);
      b = __float_as_uint(v[u * 4 + 1]);
      c = __float_as_uint(v[u * 4 + 2]);
      d = __float_as_uint(v[u * 4 + 3]);
    }
    st_shared_v4(row + (uint32_t)((u ^ sw) << 4), a, b, c, d);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (reduce)
      tma_reduce_add_4d(map, dst, n, mrow0, b0, b1);
    else
      tma_store_4d(map, dst, n, mrow0, b0, b1);
    bulk_commit();
  }
  st.bi ^= 1;
}

// One 32-column chunk through the TMA path: bf16 = one 32-column box, f32 =
// two 16-column boxes; Gelu stores Z first; Accum is a TMA reduce-add into C.
__device__ __forceinline__ void epilogue_chunk_tma(const Params& p, EpiStage& st, int lane,
                                                   int b0, int b1, int n, int mrow0, int m,
                                                   float (&v)[32]) {
  const bool bf16 = p.c_bf16;
  const bool reduce = p.epi == (int)Epi::Accum;
  if (p.epi == (int)Epi::Gelu) {
    if (bf16) {
      stage_store(&p.tma_z, st, lane, v, true, false, n, mrow0, b0, b1);
    } else {
      stage_store(&p.tma_z, st, lane, v, false, false, n, mrow0, b0, b1);
      stage_store(&p.tma_z, st, lane, v + 16, false, false, n + 16, mrow0, b0, b1);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
    dropout32(p, m, n, v);
  }
  if (bf16) {
    stage_store(&p.tma_c, st, lane, v, true, reduce, n, mrow0, b0, b1);
  } else {
    stage_store(&p.tma_c, st, lane, v, false, reduce, n, mrow0, b0, b1);
    stage_store(&p.tma_c, st, lane, v + 16, false, reduce, n + 16, mrow0, b0, b1);
  }
}

// Epilogue of this thread's accumulator row m over the 32-column chunks
// half, half + kEpiHalves, ... of the tile [n0, n0 + width): two epilogue
// warps share each TMEM lane quadrant and split its chunks. RowStats writes
// one (max, sum-exp) partial per (tile, half).
__device__ __forceinline__ void epilogue_tile(const Params& p, int b0, int b1, int m, int n0,
                                              int width, uint32_t trow, int half,
                                              EpiStage* st = nullptr, int lane = 0,
                                              int mrow0 = 0) {
  const bool stats = p.epi == (int)Epi::RowStats;
  // Accum through TMA is a reduce-add: the old C is not read by the SM
  const bool aux_in = epi_needs_aux(p.epi) && !(st && p.epi == (int)Epi::Accum);
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
    if (st) {
      // warp-uniform: every lane stages its row, the store clips rows >= M
      if (n < p.N) {
        float v[32];
        epilogue_values(p, b0, b1, m, n, r, aux, v);
        epilogue_chunk_tma(p, *st, lane, b0, b1, n, mrow0, m, v);
      }
    } else if (nvalid > 0) {
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
      uint64_t seen = 0;
      for (int tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        int b0, b1, m0, tn;
        decode_tile(p, tile, b0, b1, m0, tn);
        const int n0 = tn * BN;
        for (int s = 0; s < p.nseg; ++s) {
          const CUtensorMap* ma = &p.tma_a[s];
          const CUtensorMap* mb = &p.tma_b[s];
          if (p.rdy) {
            wait_seg_b(p, s, seen);
            if (!A_MN) wait_seg_a(p, s, m0, seen);
          }
          for (int kb = 0; kb < p.seg_kb[s]; ++kb) {
            if (A_MN && p.rdy) wait_seg_a(p, s, kb * BK, seen);
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

constexpr unsigned long long kEvictNormal = 0x1000000000000000ull;  // L2 policy of operand loads

__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int c0, int c1, int c2, int c3,
                                                unsigned long long policy = kEvictNormal) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerBitMask), "r"(c0), "r"(c1),
      "r"(c2), "r"(c3), "l"(policy)
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

__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar, uint16_t mask = 0x3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar, uint32_t leader = 0) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(leader));
  // relaxed: the arrive only publishes "TMEM drained" (tcgen05.wait::ld has
  // completed the reads); a release would add a GPU-scope MEMBAR that waits
  // for every outstanding epilogue store of this thread.
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}

// NH = 256-column accumulator halves per pair tile: NH = 1 is a 256 x 256
// tile with two TMEM accumulators (the epilogue of tile i overlaps the MMAs
// of tile i+1); NH = 2 is a 256 x 512 tile (A staged once for 512 output
// columns: a quarter less L2->SM traffic and fewer DRAM re-reads per flop,
// the cuBLAS sm_100 tile shape) whose two halves fill all 512 TMEM columns;
// each half has its own empty barrier, so the next tile's half-0 MMAs start
// while the epilogue still drains half 1.
// ---- dynamic tile order for the persistent pair kernel ----------------------
// A statically strided persistent schedule lets clusters drift apart over
// their ~40 tiles until tiles that share A/B panels no longer run together,
// and the L2 reuse between them collapses (2-3x the DRAM reads, measured).
// Instead the pair leader's producer takes tiles from a global atomic
// counter (first wave static), so running tiles stay contiguous in tile
// order like a hardware-scheduled grid, and broadcasts each tile id through
// a small shared-memory queue to every role of both CTAs.
constexpr int kTQ = 4;

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_cluster_u32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC;\n\t"
      "bra LAB_WAITC;\n"
      "DONEC:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct TileQ {
  int* ids;
  uint64_t* full;
  uint64_t* empty;  // the leader CTA's copy counts every consumer
  int slot;
  uint32_t ph;
  __device__ __forceinline__ void advance() {
    if (++slot == kTQ) {
      slot = 0;
      ph ^= 1;
    }
  }
  // Consumer: next tile id (-1 = done). A single thread (whole_warp false)
  // or all 32 lanes of a warp (whole_warp true: every lane reads, then lane 0
  // releases the slot) to the leader CTA's empty barrier.
  __device__ __forceinline__ int pop(uint32_t rank, bool whole_warp) {
    mbar_wait_cluster(&full[slot], ph);
    const int t = *reinterpret_cast<volatile int*>(&ids[slot]);
    bool arrive = true;
    if (whole_warp) {
      __syncwarp();
      arrive = (threadIdx.x % 32) == 0;
    }
    if (arrive) {
      if (rank == 0)
        mbar_arrive(&empty[slot]);
      else
        mbar_arrive_cluster(mapa_u32(smem_u32(&empty[slot]), 0));
    }
    advance();
    return t;
  }
  // Cluster leader's producer: publish t to all `ncta` CTAs of the cluster.
  __device__ __forceinline__ void push(int t, int ncta) {
    mbar_wait(&empty[slot], ph ^ 1);
    ids[slot] = t;
    for (int r = 1; r < ncta; ++r) st_cluster_u32(mapa_u32(smem_u32(&ids[slot]), r), t);
    mbar_arrive(&full[slot]);
    for (int r = 1; r < ncta; ++r) mbar_arrive_cluster(mapa_u32(smem_u32(&full[slot]), r));
    advance();
  }
};
// consumers per tile: the MMA thread, 8 epilogue warps per CTA, the
// non-leader CTA's producer
constexpr int kTQConsumers = 1 + 16 + 1;

template <int ST, int NH, int BNP = 256>
struct Cfg2 {
  static constexpr int HALF = 128;       // rows of A per CTA
  static constexpr int BH = BNP / 2;     // columns of B per CTA and half (MMA N = BNP)
  static constexpr int A_BYTES = HALF * BK * 2;
  static constexpr int B_BYTES = NH * BH * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = ST;
  static constexpr int TMEM_COLS = 512;  // 2 accumulator slots of up to 256 fp32 columns
  // NH = 2: per-epilogue-warp TMA-store staging (2 x 2 KB per warp)
  static constexpr int EPI_BYTES = NH == 2 ? 8 * 4096 : 0;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
};

// Pair-tile index -> (batch0, batch1, m0 (multiple of 256), n0 (multiple of
// p.tile_n)).
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
  n0 = (in / gm) * p.tile_n;
}

// Tile id -> tile coordinates; `half` for the split tiles of the last wave
// (n0 then names the 256-column half).
template <int BNP>
__device__ __forceinline__ void decode_pair_id(const Params& p, int id, int& b0, int& b1, int& m0,
                                               int& n0, bool& half) {
  half = id >= p.num_full;
  if (!half) {
    decode_pair_tile(p, id, b0, b1, m0, n0);
    return;
  }
  const int t = p.num_full + ((id - p.num_full) >> 1);
  decode_pair_tile(p, t, b0, b1, m0, n0);
  n0 += ((id - p.num_full) & 1) * BNP;
}

template <bool A_MN, bool B_MN, int ST, int NH, int BNP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_2cta_kernel(const __grid_constant__ Params p) {
  using C = Cfg2<ST, NH, BNP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(epi_smem + C::EPI_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;  // per 256-column accumulator slot
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* tq_full = tempty_bar + 2;
  uint64_t* tq_empty = tq_full + kTQ;
  int* tq_ids = reinterpret_cast<int*>(tq_empty + kTQ);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_ids + kTQ);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const uint32_t cta = rank;              // role in the CTA pair (0 = MMA leader)
  const int cluster = blockIdx.x / 2;
  TileQ tq{tq_ids, tq_full, tq_empty, 0, 0};

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8 * kEpiHalves);  // epilogue warps of both CTAs (leader's copy used)
    }
    for (int q = 0; q < kTQ; ++q) {
      mbar_init(&tq_full[q], 1);
      mbar_init(&tq_empty[q], kTQConsumers);
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
      uint64_t seen = 0;
      int next = cluster;  // first wave static
      for (;;) {
        int tile;
        if (rank == 0) {
          tile = next < p.num_tiles ? next : -1;
          // fetch the following tile now: the atomic's latency hides under this one's loads
          if (tile >= 0) next = p.wave + atomicAdd(p.tile_counter, 1);
          tq.push(tile, 2);
          if (tile < 0) break;
        } else {
          tile = tq.pop(rank, false);
          if (tile < 0) break;
        }
        int b0, b1, m0, n0;
        bool half;
        decode_pair_id<BNP>(p, tile, b0, b1, m0, n0, half);
        const int nh = half ? 1 : NH;
        const int mr = m0 + (int)cta * C::HALF;
        // Serpentine K: odd waves walk K backwards, so a wave starts on the
        // k-blocks the previous wave touched last -- still in L2 for the
        // operand panels the two waves share.
        const bool rev = (tile / p.wave) & 1;
        for (int si = 0; si < p.nseg; ++si) {
          const int s = rev ? p.nseg - 1 - si : si;
          const CUtensorMap* ma = &p.tma_a[s];
          const CUtensorMap* mb = &p.tma_b[s];
          if (p.rdy) {
            // this CTA loads B columns of the pair tile and its own A rows
            wait_seg_b(p, s, seen);
            if (!A_MN) wait_seg_a(p, s, mr, seen);
          }
          for (int ki = 0; ki < p.seg_kb[s]; ++ki) {
            const int kb = rev ? p.seg_kb[s] - 1 - ki : ki;
            if (A_MN && p.rdy) wait_seg_a(p, s, kb * BK, seen);
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * C::STAGE_BYTES;
            uint8_t* sb = sa + C::A_BYTES;
            if (cta == 0)
              mbar_expect_tx(&full_bar[stage], 2 * (C::A_BYTES + nh * C::BH * BK * 2));
            const int k = kb * BK;
            if (!A_MN) {
              tma_load_4d_2sm(sa, ma, &full_bar[stage], k, mr, b0, b1);
            } else {
#pragma unroll
              for (int c = 0; c < C::HALF / 64; ++c)
                tma_load_4d_2sm(sa + c * 8192, ma, &full_bar[stage], mr + c * 64, k, b0, b1);
            }
#pragma unroll
            for (int h = 0; h < NH; ++h) {
              if (h >= nh) break;
              // the pair's columns [n0 + 256h, +256): this CTA stages its 128
              const int nr = n0 + h * BNP + (int)cta * C::BH;
              uint8_t* sbh = sb + h * (C::BH * BK * 2);
              if (!B_MN) {
                tma_load_4d_2sm(sbh, mb, &full_bar[stage], k, nr, b0, b1);
              } else {
#pragma unroll
                for (int c = 0; c < C::BH / 64; ++c)
                  tma_load_4d_2sm(sbh + c * 8192, mb, &full_bar[stage], nr + c * 64, k, b0, b1);
              }
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
                             ((B_MN ? 1u : 0u) << 16) | ((uint32_t)(BNP >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;  // NH == 1: alternating slot; NH == 2: both slots every tile
      uint32_t slot_phase = 0;  // bit s = phase of slot s
      for (;;) {
        const int id = tq.pop(rank, false);
        if (id < 0) break;
        const bool half = id >= p.num_full;  // one 256-column half only
        const int nh = half ? 1 : NH;
        int kb0 = 0;
        if (NH == 2 && p.mma_lead && !half) {
          // Lead phase: the epilogue drains half 0 first, so start this
          // tile's half-0 MMAs on up to STAGES k-blocks while it is still
          // draining half 1, then catch half 1 up on the same (still held)
          // stages and release them. Hides the half-1 drain under MMAs.
          const int lead = p.total_kb < C::STAGES ? p.total_kb : C::STAGES;
          const int st0 = stage;
          const uint32_t ph0 = phase;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&tempty_bar[h], ((slot_phase >> h) & 1) ^ 1);
            tc_fence_after();
            int sg = st0;
            uint32_t ph = ph0;
#pragma unroll 1
            for (int kb = 0; kb < lead; ++kb) {
              if (h == 0) {
                mbar_wait(&full_bar[sg], ph);
                tc_fence_after();
              }
              const uint32_t sa = smem_u32(smem + sg * C::STAGE_BYTES);
              const uint32_t sbh = sa + C::A_BYTES + h * (C::BH * BK * 2);
              const uint32_t d_tmem = tmem_base + h * BNP;
#pragma unroll
              for (int k = 0; k < BK / 16; ++k) {
                const uint64_t ad = A_MN ? make_sdesc(sa + k * 2048, 8192, 1024)
                                         : make_sdesc(sa + k * 32, 16, 1024);
                const uint64_t bd = B_MN ? make_sdesc(sbh + k * 2048, 8192, 1024)
                                         : make_sdesc(sbh + k * 32, 16, 1024);
                mma_bf16_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
              }
              if (h == 1) mma_commit_2sm(&empty_bar[sg]);
              if (++sg == C::STAGES) {
                sg = 0;
                ph ^= 1;
              }
            }
            if (h == 1) {
              stage = sg;
              phase = ph;
            }
          }
          kb0 = lead;
        }
        for (int kb = kb0; kb < p.total_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if (h >= nh) break;
            const int slot = NH == 1 ? acc : h;
            if (kb == 0 && kb0 == 0) {
              // the accumulator slot must have been drained by the epilogue
              mbar_wait(&tempty_bar[slot], ((slot_phase >> slot) & 1) ^ 1);
              tc_fence_after();
            }
            const uint32_t d_tmem = tmem_base + slot * BNP;
            const uint32_t sbh = sb + h * (C::BH * BK * 2);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = A_MN ? make_sdesc(sa + k * 2048, 8192, 1024)
                                       : make_sdesc(sa + k * 32, 16, 1024);
              const uint64_t bd = B_MN ? make_sdesc(sbh + k * 2048, 8192, 1024)
                                       : make_sdesc(sbh + k * 32, 16, 1024);
              mma_bf16_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          mma_commit_2sm(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          if (h >= nh) break;
          const int slot = NH == 1 ? acc : h;
          mma_commit_2sm(&tfull_bar[slot]);
          slot_phase ^= 1u << slot;
        }
        if (NH == 1) acc ^= 1;
      }
    }
  } else {
    // ------------------------------------------- epilogue warps (both CTAs)
    const int quad = warp & 3;
    int acc = 0;
    uint32_t slot_phase = 0;
    EpiStage st{smem_u32(epi_smem) + (uint32_t)(warp - 2) * 4096u, 0};
    const bool tma_epi = NH == 2 && p.tma_epi;
    for (;;) {
      const int tile = tq.pop(rank, true);
      if (tile < 0) break;
      int b0, b1, m0, n0;
      bool half;
      decode_pair_id<BNP>(p, tile, b0, b1, m0, n0, half);
      const int nh = half ? 1 : NH;
      const int mrow0 = m0 + (int)cta * C::HALF + quad * 32;
      const int m = mrow0 + lane;
#pragma unroll 1
      for (int h = 0; h < nh; ++h) {
        const int slot = NH == 1 ? acc : h;
        mbar_wait(&tfull_bar[slot], (slot_phase >> slot) & 1);
        tc_fence_after();
        const uint32_t trow = tmem_base + ((uint32_t)(quad * 32) << 16) + slot * BNP;
        epilogue_tile(p, b0, b1, m, n0 + h * BNP, BNP, trow, (warp - 2) / 4,
                      tma_epi ? &st : nullptr, lane, mrow0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(&tempty_bar[slot]);
        slot_phase ^= 1u << slot;
      }
      if (NH == 1) acc ^= 1;
    }
    if (tma_epi && lane == 0) bulk_wait_all();
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


// Output view for the TMA-store epilogue: [N, M, nb0, nb1] of bf16 / f32
// with a {32 | 16, 32, 1, 1} box (64-byte rows) and SWIZZLE_64B.
bool encode_out(CUtensorMap* map, const void* ptr, bool bf16, int64_t N, int64_t M, int64_t ld,
                int64_t nb0, int64_t s0, int64_t nb1, int64_t s1) {
  auto fn = encode_fn();
  if (!fn || !ptr) return false;
  const int64_t esz = bf16 ? 2 : 4;
  if (nb0 <= 1) s0 = ld * M;
  if (nb1 <= 1) s1 = s0 * (nb0 > 1 ? nb0 : 1);
  cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)nb0, (cuuint64_t)nb1};
  cuuint64_t strides[3] = {(cuuint64_t)(ld * esz), (cuuint64_t)(s0 * esz), (cuuint64_t)(s1 * esz)};
  for (int i = 0; i < 3; ++i)
    if (strides[i] % 16 != 0) return false;
  if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0) return false;
  cuuint32_t box[4] = {(cuuint32_t)(bf16 ? 32 : 16), 32, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
            const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

std::atomic<int> g_sm_reserve{0};

constexpr int kMaxDevices = 64;

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < kMaxDevices) ? dev : 0;
}

// SMs the persistent GEMMs may occupy: all of them, minus the ones left for
// NCCL kernels when this process has peers (gemm_set_sm_reserve), so that
// collectives on the comm stream run concurrently with the GEMMs.
int num_sms() {
  static int count[kMaxDevices] = {};
  static std::once_flag once[kMaxDevices];
  const int dev = current_device();
  std::call_once(once[dev], [dev] {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    count[dev] = n > 0 ? n : 148;
  });
  const int n = count[dev];
  const int r = g_sm_reserve.load(std::memory_order_relaxed);
  return (r > 0 && r < n - 2) ? ((n - r) & ~1) : n;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device
// (thread-safe: the in-process backend launches from one thread per rank).
template <auto Kern>
cudaError_t ensure_smem(int bytes) {
  static cudaError_t status[kMaxDevices];
  static std::once_flag once[kMaxDevices];
  const int dev = current_device();
  std::call_once(once[dev], [&] {
    status[dev] = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  });
  return status[dev];
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch(const Params& p, cudaStream_t stream) {
  using C = Cfg<BN>;
  auto kern = gemm_bf16_kernel<BN, A_MN, B_MN>;
  const cudaError_t e = ensure_smem<gemm_bf16_kernel<BN, A_MN, B_MN>>(C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int grid = std::min(p.num_tiles, num_sms());
  kern<<<grid, kThreads, C::SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

// Per-device ring of tile counters for the pair kernel's dynamic schedule;
// each launch takes the next slot and zeroes it on its stream.
int* tile_counter_slot(cudaStream_t stream) {
  constexpr int kSlots = 65536;  // a slot is reused only 65536 launches later
  static std::mutex mu;
  static int* bufs[kMaxDevices] = {};
  static unsigned next[kMaxDevices] = {};
  const int dev = current_device();
  int* slot;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!bufs[dev] && cudaMalloc(&bufs[dev], kSlots * sizeof(int)) != cudaSuccess) {
      bufs[dev] = nullptr;
      return nullptr;
    }
    slot = bufs[dev] + (next[dev]++ % kSlots);
  }
  if (cudaMemsetAsync(slot, 0, sizeof(int), stream) != cudaSuccess) return nullptr;
  return slot;
}

template <bool A_MN, bool B_MN, int ST, int NH, int BNP>
cudaError_t launch_2cta(const Params& p_in, cudaStream_t stream) {
  using C = Cfg2<ST, NH, BNP>;
  auto kern = gemm_bf16_2cta_kernel<A_MN, B_MN, ST, NH, BNP>;
  const cudaError_t e = ensure_smem<gemm_bf16_2cta_kernel<A_MN, B_MN, ST, NH, BNP>>(C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  Params p = p_in;
  p.tile_counter = tile_counter_slot(stream);
  if (!p.tile_counter) return cudaErrorMemoryAllocation;
  const int n = std::min(p.num_tiles, std::max(1, num_sms() / 2));  // persistent: one pair per TPC
  p.wave = n;
  p.num_full = p.num_tiles;
  if (NH == 2) {
    // a partial last wave of at most half the pairs runs as twice as many
    // 256 x 256 halves: all of it in half a tile's time instead of one
    const int rem = p.num_tiles % n;
    if (p.num_tiles > n && rem > 0 && 2 * rem <= n) {
      p.num_full = p.num_tiles - rem;
      p.num_tiles = p.num_full + 2 * rem;
    }
  }
  kern<<<2 * n, kThreads, C::SMEM_BYTES, stream>>>(p);
  return cudaGetLastError();
}

template <int ST, int NH, int BNP>
cudaError_t launch_pair_st(const Params& p, bool a_mn, bool b_mn, cudaStream_t s) {
  if (!a_mn && b_mn) return launch_2cta<false, true, ST, NH, BNP>(p, s);
  if (!a_mn && !b_mn) return launch_2cta<false, false, ST, NH, BNP>(p, s);
  if (a_mn && b_mn) return launch_2cta<true, true, ST, NH, BNP>(p, s);
  return launch_2cta<true, false, ST, NH, BNP>(p, s);
}

// tile_n = 256: 256 x 256 pair tiles, two TMEM accumulators; 512: 256 x 512
// (NH = 2, see Cfg2). Shared-memory ring: 7 x 32 KB (256), 4 x 48 KB (512).
cudaError_t launch_pair(const Params& p, int tile_n, bool a_mn, bool b_mn, cudaStream_t s) {
  if (tile_n == 512) return launch_pair_st<4, 2, 256>(p, a_mn, b_mn, s);
  return launch_pair_st<7, 1, 256>(p, a_mn, b_mn, s);
}

// 256-column halves per pair tile (see Cfg2): 2 when the wider tile costs at
// most 10 % of extra wave time over the 148 SMs (74 pairs) -- measured +3.5 %
// step throughput under the power cap even at a partial extra wave -- and the
// epilogue has no per-256-column-tile layout (RowStats partials, attention
// epilogues). TESS_GEMM_NH=1|2 forces the choice (tests pin both tiles).
int pair_halves(const GemmDesc& d) {
  static const int env = [] {
    const char* e = std::getenv("TESS_GEMM_NH");
    return e ? std::atoi(e) : 0;
  }();
  if (env == 1) return 1;
  if (d.epi == Epi::RowStats || d.epi == Epi::SoftmaxFwd || d.epi == Epi::SoftmaxBwd) return 1;
  if (d.N <= 256) return 1;
  if (env == 2) return 2;
  const long long pairs = std::max(1, num_sms() / 2);
  const long long tm = (d.M + 255) / 256, b = d.nb0 * d.nb1;
  const long long t1 = tm * ((d.N + 255) / 256) * b, t2 = tm * ((d.N + 511) / 512) * b;
  const long long w1 = (t1 + pairs - 1) / pairs, w2 = (t2 + pairs - 1) / pairs;
  return (2 * w2 * 100 <= 110 * w1) ? 2 : 1;
}

int pair_tile_n(const GemmDesc& d) { return 256 * pair_halves(d); }

// The pair kernel for M > 128 and N > 128. N <= 128 (the dQ = dS K product,
// N = head_dim) stays on the 1-CTA 128 x 128 kernel: that product is
// HBM-bound on reading dS^T, where 256 x 128 pair tiles measured no better.
bool use_pair_kernel(int64_t M, int64_t N) { return M > 128 && N > 128; }

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

void gemm_set_sm_reserve(int sms) {
  int cur = sm100::g_sm_reserve.load();
  while (sms > cur && !sm100::g_sm_reserve.compare_exchange_weak(cur, sms)) {
  }
}

std::string gemm_kernel_name(const GemmDesc& d) {
  const int am = d.trans_a ? 1 : 0, bm = d.trans_b ? 0 : 1;
  if (d.in == DType::F32)
    return "gemm_f32_kernel<" + std::to_string((int)d.trans_a) + "," +
           std::to_string((int)d.trans_b) + ">";
  if (sm100::use_pair_kernel(d.M, d.N))
    return "gemm_bf16_2cta_kernel<" + std::to_string(am) + "," + std::to_string(bm) + "," +
           std::to_string(sm100::pair_tile_n(d)) + ">";
  return "gemm_bf16_kernel<" + std::to_string(d.N > 128 ? 256 : 128) + "," + std::to_string(am) +
         "," + std::to_string(bm) + ">";
}

int gemm_bf16_stat_tiles(const GemmDesc& d) {
  const int t = gemm_bf16_tile_n(d);
  return static_cast<int>((d.N + t - 1) / t) * sm100::kEpiHalves;
}

int gemm_bf16_tile_n(const GemmDesc& d) {
  if (sm100::use_pair_kernel(d.M, d.N)) return sm100::pair_tile_n(d);
  return d.N > 128 ? 256 : 128;
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
  p.mma_lead = 1;
  const bool pair = use_pair_kernel(d.M, d.N);
  const int pair_tn = pair ? pair_tile_n(d) : 0;
  const int nh = pair_tn == 512 ? 2 : 1;
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
  const int tile_m = pair ? 256 : BM, tile_n = pair ? pair_tn : BN;
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
  if (pair && nh == 2 && d.epi != Epi::RowStats) {
    const bool bf = d.c_type == DType::BF16;
    p.tma_epi = encode_out(&p.tma_c, d.c, bf, d.N, d.M, d.ldc, d.nb0, d.cs0, d.nb1, d.cs1) &&
                (d.epi != Epi::Gelu ||
                 encode_out(&p.tma_z, d.z, bf, d.N, d.M, d.ldz, d.nb0, d.zs0, d.nb1, d.zs1));
  }
  p.nst = static_cast<int>((d.N + tile_n - 1) / tile_n) * kEpiHalves;
  if (d.bias || d.drop_p > 0.f) {
    const bool ok_epi = d.epi == Epi::Store || d.epi == Epi::Accum || d.epi == Epi::Resid ||
                        d.epi == Epi::Gelu;
    if (!ok_epi || d.nb0 != 1 || d.nb1 != 1 || !(d.drop_p >= 0.f && d.drop_p < 1.f)) {
      g_gemm_err = "gemm_bf16_sm100: bias / dropout need an unbatched Store, Accum, Resid or "
                   "Gelu epilogue and 0 <= p < 1";
      return cudaErrorInvalidValue;
    }
    p.bias = d.bias;
    if (d.drop_p > 0.f) {
      p.drop = 1;
      p.drop_thresh = (uint32_t)std::min(16777216.0, std::ceil((double)d.drop_p * 16777216.0));
      p.drop_scale = 1.0f / (1.0f - d.drop_p);
      p.drop_seed = d.drop_seed;
      p.drop_row0 = d.drop_row0;
      p.drop_col0 = d.drop_col0;
    }
  }
  if (d.ready.any()) {
    const GemmReady& r = d.ready;
    if (r.chunks < 1 || r.chunks * d.nseg > 32 || r.chunk_rows < 0 || r.chunk_rows > (1 << 30) ||
        (r.chunks > 1 && r.chunk_rows == 0)) {
      g_gemm_err = "gemm_bf16_sm100: bad segment readiness layout";
      return cudaErrorInvalidValue;
    }
    p.rdy = 1;
    for (int s = 0; s < kMaxSegments; ++s) {
      p.rdy_a[s] = s < d.nseg ? r.a_flags[s] : nullptr;
      p.rdy_b[s] = s < d.nseg ? r.b_flags[s] : nullptr;
      p.rdy_ea[s] = r.a_epoch[s];
      p.rdy_eb[s] = r.b_epoch[s];
    }
    p.rdy_chunks = r.chunks;
    p.rdy_chunk_rows = static_cast<int>(r.chunk_rows);
  }
  cudaError_t e = pair        ? launch_pair(p, pair_tn, a_mn, b_mn, stream)
                  : BN == 256 ? launch_bn<256>(p, a_mn, b_mn, stream)
                              : launch_bn<128>(p, a_mn, b_mn, stream);
  if (e != cudaSuccess) g_gemm_err = std::string("gemm_bf16_sm100 launch: ") +
                                     cudaGetErrorString(e);
  return e;
}

}  // namespace tess
