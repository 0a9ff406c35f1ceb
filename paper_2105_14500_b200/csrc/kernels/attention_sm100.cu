// Fused attention forward / backward for sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces, for bf16, the per-(sample, head) loop of the reference's
// attn_forward_rank / attn_backward_rank (proj/src/layers.cpp:383-456):
//   S = Q K^T / sqrt(hd), P = softmax_rows(S) (layers.cpp:44-58, no mask),
//   O = P V; backward dV = P^T dO, dP = dO V^T, dS = P * (dP - rowsum(dP*P))
//   / sqrt(hd) (layers.cpp:60-74), dQ = dS K, dK = dS^T Q. The row term
//   rowsum(dP*P) is computed as rowsum(dO*O) (k_attn_delta).
// Neither S nor P reaches HBM: the forward keeps one log2-sum-exp per query
// row, the backward recomputes P from it.
//
// ---------------------------------------------------------------- forward
// One CTA = one (sample, head) and two 128-query tiles A and B that share
// every K/V tile (halving K/V traffic). 320 threads:
//   warp 0      TMA producer: Q_A, Q_B once, then K_j, V_j into a ring of
//               KV_STAGES 128-key tiles (128B-swizzled boxes {64, 128}).
//   warp 1      MMA issuer + TMEM owner. Per key tile j:
//                 S_A(j+1) = Q_A K_{j+1}^T, S_B(j+1) = Q_B K_{j+1}^T
//                 O_A += P_A(j) V_j,         O_B += P_B(j) V_j
//               interleaved so the tensor core works on one tile's MMAs
//               while the other tile's softmax runs.
//   warps 2-5   softmax of tile A (warp w owns TMEM lanes 32*(w%4)..+31:
//               thread = query row), warps 6-9 tile B. Row max / exp2 /
//               row sum in registers; P (bf16) written back over the consumed
//               S columns of tensor memory, the P V MMA reading its A operand
//               from TMEM (only V streams from shared memory); lazy rescaling of O
//               (only when the running max grows by more than 2^8, exact
//               because the final normalisation uses the same max).
// TMEM: S_A [0,128), S_B [128,256), O_A [256,256+hd), O_B [384,384+hd).
#include "attention.h"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "sm100_ptx.cuh"

namespace tess {

namespace {
thread_local std::string g_attn_err;
}
long long* g_attn_trace = nullptr;  // debug: device buffer of the last traced backward

const char* attn_last_error() { return g_attn_err.c_str(); }
long long* attn_debug_trace() { return g_attn_trace; }

namespace sm100 {
namespace attn {

// 2^x on the FMA/ALU pipes (round-to-nearest split, degree-3 polynomial on
// [-0.5, 0.5], max rel. error 2.2e-4 -- far below the bf16 rounding of P):
// the backward's exp2/dS math is MUFU-bound (16 K ex2 per tile at 16/clk),
// so a share of the exponentials moves here. x is clamped at -125 so the
// exponent add cannot underflow (2^-125 instead of 0 for masked columns,
// whose dO / Q rows are zero).
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -125.0f);
  const float t = x + 12582912.0f;  // 1.5 * 2^23: rint(x) in the low mantissa bits
  const float j = t - 12582912.0f;
  const float f = x - j;
  const float p =
      fmaf(fmaf(fmaf(0.05286731571f, f, 0.2421521395f), f, 0.6935868263f), f, 0.9999627471f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

constexpr int kThreads = 320;
// which of every 8 exponentials of the forward use exp2_fma (bit e & 7)
#ifndef TESS_ATTN_FWD_POLY
#define TESS_ATTN_FWD_POLY 0
#endif
constexpr int kFwdPolyMask = TESS_ATTN_FWD_POLY;
constexpr int kBwdThreads = 576;  // backward: TMA + MMA warps + 16 softmax-gradient warps
constexpr int BQ = 128;   // query rows per tile (UMMA M)
constexpr int BKV = 128;  // keys per tile (UMMA N of S, K of P V)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units


struct FwdParams {
  CUtensorMap tm_qkv;  // 3-D view [cols, S, samples] of qkv, box {64, 128, 1}
  int S, H, n_pairs, n_kv;
  int hd;
  float c;  // scale * log2(e)
  __nv_bfloat16* o;
  long long ld_o;
  float* lse;
};

template <int HD>
struct FwdCfg {
  static constexpr int Q_BYTES = BQ * HD * 2;    // one 128-row tile of Q (or K, V)
  static constexpr int KV_BYTES = BKV * HD * 2;
  static constexpr int KV_STAGES = HD == 128 ? 5 : 10;
  static constexpr int OFF_QA = 0;
  static constexpr int OFF_QB = Q_BYTES;
  static constexpr int OFF_KV = 2 * Q_BYTES;
  static constexpr int OFF_BAR = OFF_KV + KV_STAGES * KV_BYTES;
  static constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;  // + barriers + alignment slack
  static constexpr int TMEM_COLS = 512;
  static constexpr int TM_S0 = 0, TM_O0 = 256;
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ FwdParams p) {
  using C = FwdCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;                        // 1
  uint64_t* kv_full = bars + 1;                   // KV_STAGES
  uint64_t* kv_empty = kv_full + C::KV_STAGES;    // KV_STAGES
  uint64_t* s_full = kv_empty + C::KV_STAGES;     // 2 (tile A, B)
  uint64_t* p_full = s_full + 2;                  // 2
  uint64_t* o_full = p_full + 2;                  // 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int pair = blockIdx.x % p.n_pairs;
  const int head = (blockIdx.x / p.n_pairs) % p.H;
  const int smp = blockIdx.x / (p.n_pairs * p.H);
  const int q0 = pair * 2 * BQ;
  const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
    }
    mbar_init(o_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&p.tm_qkv);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------ TMA producer
      mbar_expect_tx(q_full, 2 * C::Q_BYTES);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_3d(smem + C::OFF_QA + c * 16384, &p.tm_qkv, q_full, col_q + c * 64, q0, smp);
        tma_load_3d(smem + C::OFF_QB + c * 16384, &p.tm_qkv, q_full, col_q + c * 64, q0 + BQ,
                    smp);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0; j < p.n_kv; ++j) {
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // K_j then V_j
          mbar_wait(&kv_empty[stage], phase ^ 1);
          uint8_t* dst = smem + C::OFF_KV + stage * C::KV_BYTES;
          mbar_expect_tx(&kv_full[stage], C::KV_BYTES);
          const int col = which == 0 ? col_k : col_v;
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(dst + c * 16384, &p.tm_qkv, &kv_full[stage], col + c * 64, j * BKV, smp);
          if (++stage == C::KV_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16(BQ, HD, false, true);
      const uint32_t sq0 = smem_u32(smem + C::OFF_QA);  // Q_B, P_B follow at fixed offsets
      int stage = 0;
      uint32_t phase = 0;
      auto next_kv = [&]() {
        const int s = stage;
        mbar_wait(&kv_full[s], phase);
        tc_fence_after();
        if (++stage == C::KV_STAGES) {
          stage = 0;
          phase ^= 1;
        }
        return s;
      };
      auto issue_s = [&](int t, uint32_t skv) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (uint32_t)(kk >> 2) * 16384u + (uint32_t)(kk & 3) * 32u;
          mma_bf16(tmem + C::TM_S0 + t * BKV, make_sdesc(sq0 + t * C::Q_BYTES + off, 16, 1024),
                   make_sdesc(skv + off, 16, 1024), idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[t]);
      };
      // O += P V with P (bf16 pairs) in tensor memory: the consumed S columns
      // [0, 64) of the tile's S buffer, 8 columns per 16 keys
      auto issue_pv = [&](int t, uint32_t skv, bool acc) {
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_bf16_ts(tmem + C::TM_O0 + t * 128, tmem + C::TM_S0 + t * BKV + kk * 8,
                      make_sdesc(skv + (uint32_t)kk * 2048u, 16384, 1024), idesc_pv,
                      (acc || kk > 0) ? 1u : 0u);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      int ks = next_kv();
      const uint32_t sk0 = smem_u32(smem + C::OFF_KV + ks * C::KV_BYTES);
      issue_s(0, sk0);
      issue_s(1, sk0);
      mma_commit(&kv_empty[ks]);
      for (int j = 0; j < p.n_kv; ++j) {
        const int vs = next_kv();
        const uint32_t sv = smem_u32(smem + C::OFF_KV + vs * C::KV_BYTES);
        const bool more = j + 1 < p.n_kv;
        uint32_t skn = 0;
        mbar_wait(&p_full[0], j & 1);
        tc_fence_after();
        issue_pv(0, sv, j > 0);
        if (more) {
          ks = next_kv();
          skn = smem_u32(smem + C::OFF_KV + ks * C::KV_BYTES);
          issue_s(0, skn);
        }
        mbar_wait(&p_full[1], j & 1);
        tc_fence_after();
        issue_pv(1, sv, j > 0);
        mma_commit(&kv_empty[vs]);
        if (more) {
          issue_s(1, skn);
          mma_commit(&kv_empty[ks]);
        }
      }
      mma_commit(o_full);
    }
  } else {
    // --------------------------------------------------- softmax warps
    const int t = (warp - 2) >> 2;   // tile A (0) or B (1)
    const int quad = warp & 3;       // TMEM lane quadrant
    const int r = quad * 32 + lane;  // query row within the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t t_s = tmem + lane_off + C::TM_S0 + t * BKV;
    const uint32_t t_o = tmem + lane_off + C::TM_O0 + t * 128;
    const float cl2 = p.c;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < p.n_kv; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      float s[BKV];
      {
        uint32_t a0[32], a1[32], a2[32], a3[32];
        tmem_ld32_nowait(t_s + 0, a0);
        tmem_ld32_nowait(t_s + 32, a1);
        tmem_ld32_nowait(t_s + 64, a2);
        tmem_ld32_nowait(t_s + 96, a3);
        tmem_wait_ld();
        reg_fence32(a0);
        reg_fence32(a1);
        reg_fence32(a2);
        reg_fence32(a3);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          s[e] = __uint_as_float(a0[e]);
          s[32 + e] = __uint_as_float(a1[e]);
          s[64 + e] = __uint_as_float(a2[e]);
          s[96 + e] = __uint_as_float(a3[e]);
        }
      }
      const int nvalid = p.S - j * BKV;  // keys of this tile inside the sequence
      if (nvalid < BKV) {
#pragma unroll
        for (int e = 0; e < BKV; ++e)
          if (e >= nvalid) s[e] = -INFINITY;
      }
      // row max / row sum as 8 independent chains (a single 128-long
      // dependent fmax / fadd chain is ~4 clk x 128 of latency per tile)
      float mp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mp[k] = s[k];
#pragma unroll
      for (int e = 8; e < BKV; ++e) mp[e & 7] = fmaxf(mp[e & 7], s[e]);
      const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                             fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
      const float m_new = fmaxf(m_used, mx * cl2);
      const bool need = m_new > m_used + kRescaleThreshold;
      if (__any_sync(0xffffffffu, need)) {
        // lazy rescale: whole warp moves to the new max (factor <= 1)
        const float f = ex2_approx(m_used - m_new);  // 0 on the first tile
        if (j > 0) {
          l *= f;
#pragma unroll 1
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t ov[16];
            tmem_ld16_nowait(t_o + c * 16, ov);
            tmem_wait_ld();
            reg_fence16(ov);
#pragma unroll
            for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * f);
            tmem_st16(t_o + c * 16, ov);
          }
          tmem_wait_st();
        }
        m_used = m_new;
      }
      // all exponentials on MUFU: moving a share to the FMA pipe (a degree-5
      // polynomial exp2) measured slower (25 %: +6 %, 50 %: +22 %) -- the
      // softmax is issue-bound, not MUFU-bound
      float rp[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int e = 0; e < BKV; ++e) {
        const float xv = fmaf(s[e], cl2, -m_used);
        s[e] = (kFwdPolyMask >> (e & 7)) & 1 ? exp2_fma(xv) : ex2_approx(xv);
        rp[e & 7] += s[e];
      }
      l += ((rp[0] + rp[1]) + (rp[2] + rp[3])) + ((rp[4] + rp[5]) + (rp[6] + rp[7]));
      // P (bf16 pairs, lower key in the low half) over the consumed S columns
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) pk[e] = pack_bf16x2(s[h * 64 + 2 * e], s[h * 64 + 2 * e + 1]);
        tmem_st32(t_s + h * 32, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int qrow = q0 + t * BQ + r;
    const float inv = 1.0f / l;
    __nv_bfloat16* orow = p.o + ((long long)smp * p.S + qrow) * p.ld_o + (long long)head * HD;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t ov[32];
      tmem_ld32_nowait(t_o + c * 32, ov);
      tmem_wait_ld();
      reg_fence32(ov);
      if (qrow < p.S) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(ov[u * 8 + 0]) * inv, __uint_as_float(ov[u * 8 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(ov[u * 8 + 2]) * inv, __uint_as_float(ov[u * 8 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(ov[u * 8 + 4]) * inv, __uint_as_float(ov[u * 8 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(ov[u * 8 + 6]) * inv, __uint_as_float(ov[u * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + u * 8) = w;
        }
      }
    }
    if (qrow < p.S) p.lse[((long long)smp * p.H + head) * p.S + qrow] = m_used + __log2f(l);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}


// --------------------------------------------------------------- backward
// One CTA = one (sample, head, 128-key tile); it walks the 128-query tiles
// i of the sequence. 320 threads:
//   warp 0      TMA producer: K, V of the key tile once; then Q_i, dO_i
//               (128 x hd, boxes {64, 128}) through a RING-slot FIFO.
//   warp 1      MMA issuer + TMEM owner. Per query tile, all MMAs at
//               M=128, N=128 (full tcgen05 rate; N=64 tiles run at ~70 %):
//                 S^T(i) = K Q_i^T, dP^T(i) = V dO_i^T   (A = K / V, smem)
//                 dV += P^T(i) dO_i   (A = P^T in TMEM, written by the softmax
//                                      over the consumed S^T columns)
//                 dK += dS^T(i) Q_i   (A = dS^T in shared memory)
//               S^T / dP^T are single-buffered (TMEM holds S^T, dP^T, dV, dK);
//               dP^T(i+1) is issued as soon as tile i's scores sit in
//               registers; dV(i) as soon as P^T(i) is in TMEM (its own
//               barrier, before the dS^T stores), S^T(i+1) right behind it,
//               then dK(i) once dS^T(i) is in shared memory -- the next
//               tile's softmax overlaps dK(i) (-4 %, r2_attn_bwd_order_ab).
//   warps 2-17  four groups of 4 warps split each tile's 128 queries (group
//               g: columns [32g, 32g+32)); thread = key row (TMEM lane):
//               P^T = 2^(c*S^T - lse[q]) -> TMEM (bf16 pairs), dS^T = P^T
//               (dP^T - delta[q]) -> shared memory (UMMA K-major SW128, chunk
//               g/2) and, by TMA store, to HBM for dQ = dS K (one batched
//               GEMM; the 1/sqrt(hd) goes to dK's epilogue and dQ's alpha).
// Q_i and dO_i tiles are used twice with different majorness: K-major B of
// the score MMAs ([N=q][K=hd]) and MN-major B of dV/dK ([K=q][N=hd]) -- the
// same bytes under two descriptors.
// TMEM: S^T / P^T [0,128), dP^T [128,256), dV [256, 256+hd), dK [384, 384+hd).
constexpr int BQB = 128;  // queries per backward tile
// which of every 4 exponentials of the backward use exp2_fma (bit u)
#ifndef TESS_ATTN_BWD_POLY
#define TESS_ATTN_BWD_POLY 8
#endif
constexpr int kBwdPolyMask = TESS_ATTN_BWD_POLY;

struct BwdParams {
  CUtensorMap tm_kv;   // qkv view, box {64, 128}: K, V of the key tile
  CUtensorMap tm_q;    // qkv view, box {64, 128}: Q_i
  CUtensorMap tm_do;   // dO view [hq cols, S, samples], box {64, 128}
  CUtensorMap tm_dst;  // dS^T view [S q, S k, samples*H], box {64, 128} (store)
  int S, H, n_kt, n_qt;
  float c;      // scale * log2(e)
  float scale;  // 1/sqrt(hd)
  const float* lse;
  const float* delta;
  __nv_bfloat16* dqkv;
  long long ld_qkv;
  long long* trace;  // debug (TESS_ATTN_TRACE): per-phase clock64 of CTA 0, [event][tile]
};

// trace events (CTA 0 only)
enum {
  TR_MMA_S = 0, TR_MMA_P = 1, TR_SM_IN = 2, TR_SM_MATH = 3, TR_SM_OUT = 4,
  TR_SM_LOADED = 5, TR_MMA_FREE = 6, TR_MMA_GDONE = 7, TR_N = 8
};
__device__ __forceinline__ void trace_ev(const BwdParams& p, int ev, int tile) {
  if (p.trace && blockIdx.x == 0 && tile < 64) p.trace[ev * 64 + tile] = clock64();
}

template <int HD>
struct BwdCfg {
  static constexpr int KV_BYTES = 128 * HD * 2;    // K or V tile
  static constexpr int SLOT_BYTES = BQB * HD * 2;  // Q_i or dO_i
  static constexpr int RING = HD == 128 ? 4 : 8;
  static constexpr int DS_BYTES = 128 * BQB * 2;   // dS^T tile (2 chunks of 64 queries)
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = KV_BYTES;
  static constexpr int OFF_RING = 2 * KV_BYTES;
  static constexpr int OFF_DS = OFF_RING + RING * SLOT_BYTES;
  static constexpr int OFF_LD = OFF_DS + DS_BYTES;  // 4 groups x 2 bufs: lse 32 | delta 32
  static constexpr int OFF_BAR = OFF_LD + 4 * 2 * 64 * 4;
  static constexpr int USED = OFF_BAR + 512;
  // the dynamic window is 1024-aligned in practice; the kernel checks and
  // traps if the slack we could afford does not cover its misalignment
  static constexpr int SMEM_BYTES = USED + 1024 <= 232448 ? USED + 1024 : 232448;
  static constexpr int TMEM_COLS = 512;
  static constexpr int TM_ST = 0, TM_DPT = 128, TM_DV = 256, TM_DK = 384;
};


// 32 bf16 values of row r (columns [u0*8, u0*8+32) of a 64-column K-major
// SW128 tile) -> shared memory.
__device__ __forceinline__ void store_row32(uint32_t base, int r, int u0, const float (&v)[32]) {
  const uint32_t row_base = base + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int k0 = u * 8;
    st_shared_v4(row_base + (uint32_t)(((u0 + u) ^ (r & 7)) << 4), pack_bf16x2(v[k0], v[k0 + 1]),
                 pack_bf16x2(v[k0 + 2], v[k0 + 3]), pack_bf16x2(v[k0 + 4], v[k0 + 5]),
                 pack_bf16x2(v[k0 + 6], v[k0 + 7]));
  }
}

template <int HD>
__global__ void __launch_bounds__(kBwdThreads, 1) attn_bwd_kernel(const __grid_constant__ BwdParams p) {
  using C = BwdCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((smem - smem_raw) + C::USED > C::SMEM_BYTES) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars;                   // 1
  uint64_t* r_full = bars + 1;                // RING
  uint64_t* r_empty = r_full + C::RING;       // RING
  uint64_t* sdp_full = r_empty + C::RING;     // 1: S^T(i) and dP^T(i) in TMEM
  uint64_t* loaded = sdp_full + 1;            // 1: all 8 warps hold tile i's scores (count 8)
  uint64_t* pds_full = loaded + 1;            // 1: dS^T (smem) written (count 16)
  uint64_t* ds_free = pds_full + 1;           // 1: dK(i) done reading dS^T smem
  uint64_t* st_free = ds_free + 1;            // 2: TMA store of dS^T chunk g done reading
  uint64_t* fin = st_free + 2;                // 1
  uint64_t* p_full = fin + 1;                 // 1: P^T (TMEM) written (count 16)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_full + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kt = blockIdx.x % p.n_kt;
  const int head = (blockIdx.x / p.n_kt) % p.H;
  const int smp = blockIdx.x / (p.n_kt * p.H);
  const int k0 = kt * 128;
  const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < C::RING; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    mbar_init(sdp_full, 1);
    mbar_init(loaded, 16);
    mbar_init(pds_full, 16);
    mbar_init(ds_free, 1);
    mbar_init(&st_free[0], 1);
    mbar_init(&st_free[1], 1);  // chunk c's storer: group 2c
    mbar_init(fin, 1);
    mbar_init(p_full, 16);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&p.tm_kv);
    prefetch_tmap(&p.tm_q);
    prefetch_tmap(&p.tm_do);
    prefetch_tmap(&p.tm_dst);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------ TMA producer
      mbar_expect_tx(kv_full, 2 * C::KV_BYTES);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_3d(smem + C::OFF_K + c * 16384, &p.tm_kv, kv_full, col_k + c * 64, k0, smp);
        tma_load_3d(smem + C::OFF_V + c * 16384, &p.tm_kv, kv_full, col_v + c * 64, k0, smp);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int i = 0; i < p.n_qt; ++i) {
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // Q_i then dO_i
          mbar_wait(&r_empty[stage], phase ^ 1);
          uint8_t* dst = smem + C::OFF_RING + stage * C::SLOT_BYTES;
          mbar_expect_tx(&r_full[stage], C::SLOT_BYTES);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c) {
            if (which == 0)
              tma_load_3d(dst + c * 16384, &p.tm_q, &r_full[stage], col_q + c * 64, i * BQB, smp);
            else
              tma_load_3d(dst + c * 16384, &p.tm_do, &r_full[stage], head * HD + c * 64, i * BQB,
                          smp);
          }
          if (++stage == C::RING) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc_s = idesc_bf16(128, BQB, false, false);
      constexpr uint32_t idesc_g = idesc_bf16(128, HD, false, true);
      const uint32_t sk = smem_u32(smem + C::OFF_K), sv = smem_u32(smem + C::OFF_V);
      const uint32_t ring = smem_u32(smem + C::OFF_RING);
      const uint32_t sds = smem_u32(smem + C::OFF_DS);
      int stage = 0;
      uint32_t phase = 0;
      auto next_slot = [&]() {
        const int s = stage;
        mbar_wait(&r_full[s], phase);
        tc_fence_after();
        if (++stage == C::RING) {
          stage = 0;
          phase ^= 1;
        }
        return s;
      };
      // A [128 x HD] K-major (chunk stride 16 KB) times B [128 x HD] K-major
      // (chunk stride 16 KB) -> TMEM columns [d, d + 128)
      auto issue_scores = [&](uint32_t d, uint32_t a, uint32_t b) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (uint32_t)(kk >> 2) * 16384u + (uint32_t)(kk & 3) * 32u;
          mma_bf16(d, make_sdesc(a + off, 16, 1024), make_sdesc(b + off, 16, 1024), idesc_s,
                   kk > 0 ? 1u : 0u);
        }
      };
      mbar_wait(kv_full, 0);
      tc_fence_after();
      int qs = next_slot();
      int ds = next_slot();
      trace_ev(p, TR_MMA_S, 0);
      issue_scores(tmem + C::TM_ST, sk, ring + qs * C::SLOT_BYTES);
      issue_scores(tmem + C::TM_DPT, sv, ring + ds * C::SLOT_BYTES);
      mma_commit(sdp_full);
      for (int i = 0; i < p.n_qt; ++i) {
        const bool more = i + 1 < p.n_qt;
        int qn = 0, dn = 0;
        // tile i's scores are in registers: dP^T(i+1) into the dP^T columns
        mbar_wait(loaded, i & 1);
        tc_fence_after();
        trace_ev(p, TR_MMA_FREE, i);
        if (more) {
          qn = next_slot();
          dn = next_slot();
          issue_scores(tmem + C::TM_DPT, sv, ring + dn * C::SLOT_BYTES);
        }
        // dV(i) as soon as P^T(i) sits in TMEM
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        trace_ev(p, TR_MMA_P, i);
#pragma unroll
        for (int kk = 0; kk < BQB / 16; ++kk)  // dV += P^T dO_i, P^T from TMEM
          mma_bf16_ts(tmem + C::TM_DV, tmem + C::TM_ST + kk * 8,
                      make_sdesc(ring + ds * C::SLOT_BYTES + (uint32_t)kk * 2048u, 16384, 1024),
                      idesc_g, (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&r_empty[ds]);
        if (more) {
          // S^T(i+1) over the P^T columns right behind dV(i) (in-order
          // execution: dV has read them): tile i+1's softmax starts while
          // dK(i) runs
          trace_ev(p, TR_MMA_S, i + 1);
          issue_scores(tmem + C::TM_ST, sk, ring + qn * C::SLOT_BYTES);
          mma_commit(sdp_full);
        }
        // dK(i) once dS^T(i) is in shared memory
        mbar_wait(pds_full, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BQB / 16; ++kk)  // dK += dS^T Q_i
          mma_bf16(tmem + C::TM_DK,
                   make_sdesc(sds + (uint32_t)(kk >> 2) * 16384u + (uint32_t)(kk & 3) * 32u, 16,
                              1024),
                   make_sdesc(ring + qs * C::SLOT_BYTES + (uint32_t)kk * 2048u, 16384, 1024),
                   idesc_g, (i > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&r_empty[qs]);
        mma_commit(ds_free);
        trace_ev(p, TR_MMA_GDONE, i);
        qs = qn;
        ds = dn;
      }
      mma_commit(fin);
    }
  } else {
    // ------------------------------------------ softmax-gradient warps
    const int quad = warp & 3;
    const int g = (warp - 2) >> 2;   // query columns [32g, 32g+32) of each tile
    const int r = quad * 32 + lane;  // key row within the tile
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float cl2 = p.c, scale = p.scale;
    // TMA store of dS^T chunk c (64 queries = groups 2c, 2c+1) by group 2c's thread
    const bool storer = quad == 0 && lane == 0 && (g & 1) == 0;
    const int chunk = g >> 1;
    const float* lse_h = p.lse + ((long long)smp * p.H + head) * p.S;
    const float* dlt_h = p.delta + ((long long)smp * p.H + head) * p.S;
    // (lse, delta) of the group's 32 query columns staged through shared
    // memory, double buffered per group: the quad-0 warp loads tile i+1's
    // values while tile i is processed, a 128-thread named barrier at the
    // start of each tile orders them against the readers.
    const uint32_t ldg_base = smem_u32(smem + C::OFF_LD) + (uint32_t)g * 512u;  // [buf][lse|delta]
    const bool ld_writer = quad == 0;
    auto gload = [&](int i, float (&v)[2]) {
      const int q = i * BQB + g * 32 + lane;
      const bool ok = i < p.n_qt && q < p.S;
      v[0] = ok ? __ldg(lse_h + q) : INFINITY;  // 2^(x - inf) = 0: no contribution
      v[1] = ok ? __ldg(dlt_h + q) : 0.f;
    };
    auto sstore = [&](int i, const float (&v)[2]) {
      const uint32_t a = ldg_base + (uint32_t)(i & 1) * 256u + lane * 4;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v[0]) : "memory");
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(a + 128), "f"(v[1]) : "memory");
    };
    if (ld_writer) {
      float v[2];
      gload(0, v);
      sstore(0, v);
    }
    const uint32_t ds_chunk = smem_u32(smem + C::OFF_DS) + (uint32_t)chunk * 16384u;
    for (int i = 0; i < p.n_qt; ++i) {
      const uint32_t ph = (uint32_t)i & 1u;
      const uint32_t ldw = ldg_base + ph * 256u;  // this tile's (lse, delta)
      named_bar_sync(1 + g, 128);  // tile i's staging written; tile i-1's readers done
      float nv[2];
      if (ld_writer) gload(i + 1, nv);
      if (storer) {
        // dS^T chunk was last stored at tile i-1 by this thread: wait for the
        // TMA store to finish reading shared memory
        bulk_wait_read<0>();
        mbar_arrive(&st_free[chunk]);
      }
      mbar_wait(sdp_full, ph);
      tc_fence_after();
      if (quad == 0 && lane == 0 && g == 0) trace_ev(p, TR_SM_IN, i);
      // the group's 32 columns of S^T and dP^T into registers
      uint32_t sr[32], dr[32];
      tmem_ld32_nowait(tmem + lane_off + C::TM_ST + g * 32, sr);
      tmem_ld32_nowait(tmem + lane_off + C::TM_DPT + g * 32, dr);
      tmem_wait_ld();
      reg_fence32(sr);
      reg_fence32(dr);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(loaded);
      if (quad == 0 && lane == 0 && g == 0) trace_ev(p, TR_SM_LOADED, i);
      // P^T into sr, unscaled dS^T = P^T (dP^T - delta) into dr (in place);
      // the 1/sqrt(hd) is applied once to dK (epilogue) and dQ (GEMM alpha)
#pragma unroll
      for (int e4 = 0; e4 < 8; ++e4) {
        float4 l4, d4;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(l4.x), "=f"(l4.y), "=f"(l4.z), "=f"(l4.w)
                     : "r"(ldw + (uint32_t)(4 * e4) * 4u));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(d4.x), "=f"(d4.y), "=f"(d4.z), "=f"(d4.w)
                     : "r"(ldw + 128u + (uint32_t)(4 * e4) * 4u));
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = 4 * e4 + u;
          const float xv = fmaf(__uint_as_float(sr[e]), cl2, -lv[u]);
          const float pv = (kBwdPolyMask >> u) & 1 ? exp2_fma(xv) : ex2_approx(xv);
          dr[e] = __float_as_uint(pv * (__uint_as_float(dr[e]) - dv[u]));
          sr[e] = __float_as_uint(pv);
        }
      }
      if (quad == 0 && lane == 0 && g == 0) trace_ev(p, TR_SM_MATH, i);
      // P^T over the S^T columns [16g, 16g+16) once all 16 warps read theirs
      mbar_wait(loaded, ph);
      {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = pack_bf16x2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1]));
        tmem_st16(tmem + lane_off + C::TM_ST + g * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);  // dV(i) may start
      // dS^T chunk: free once dK(i-1) read it and its TMA store read it
      mbar_wait(ds_free, ph ^ 1u);
      mbar_wait(&st_free[chunk], ph);
      store_row32(ds_chunk, r, (g & 1) * 4, *reinterpret_cast<const float(*)[32]>(dr));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pds_full);
      if (quad == 0 && lane == 0 && g == 0) trace_ev(p, TR_SM_OUT, i);
      if (storer) {
        mbar_wait(pds_full, ph);  // all rows of the chunk written
        tma_store_3d(&p.tm_dst, smem + C::OFF_DS + chunk * 16384, i * BQB + chunk * 64, k0,
                     smp * p.H + head);
        bulk_commit();
      }
      // tile i+1's (lse, delta) into the other staging buffer (last read at tile i-1)
      if (ld_writer) sstore(i + 1, nv);
    }
    // ------------------------------------------------- dK, dV epilogue
    mbar_wait(fin, 0);
    tc_fence_after();
    const int krow = k0 + r;
    __nv_bfloat16* drow = p.dqkv + ((long long)smp * p.S + krow) * p.ld_qkv + col_k;
#pragma unroll
    for (int which = 0; which < 2; ++which) {  // dK then dV
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {  // group g: columns [g*HD/4, (g+1)*HD/4)
        const int col = g * (HD / 4) + c * 16;
        uint32_t v[16];
        tmem_ld16_nowait(tmem + lane_off + (which == 0 ? C::TM_DK : C::TM_DV) + col, v);
        tmem_wait_ld();
        reg_fence16(v);
        if (krow < p.S) {
          __nv_bfloat16* dst = drow + which * HD + col;
          const float f = which == 0 ? scale : 1.0f;  // dK carries the dS scale
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[u * 8 + 0]) * f, __uint_as_float(v[u * 8 + 1]) * f);
            w.y = pack_bf16x2(__uint_as_float(v[u * 8 + 2]) * f, __uint_as_float(v[u * 8 + 3]) * f);
            w.z = pack_bf16x2(__uint_as_float(v[u * 8 + 4]) * f, __uint_as_float(v[u * 8 + 5]) * f);
            w.w = pack_bf16x2(__uint_as_float(v[u * 8 + 6]) * f, __uint_as_float(v[u * 8 + 7]) * f);
            *reinterpret_cast<uint4*>(dst + u * 8) = w;
          }
        }
      }
    }
    if (storer) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 3-D bf16 view [cols, seq, samples] (row stride ld, sample stride seq*ld),
// box {64, box_rows, 1}, 128B swizzle; rows past seq read as zero.
bool encode_3d(CUtensorMap* map, const void* base, int64_t cols, int64_t seq, int64_t samples,
               int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    g_attn_err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)seq, (cuuint64_t)samples};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)(seq * ld) * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_attn_err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

template <int HD>
cudaError_t launch_fwd(const FwdParams& p, int grid, cudaStream_t s) {
  using C = FwdCfg<HD>;
  // once per instantiation and process (host threads of in-process ranks race here)
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_fwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_fwd_kernel<HD><<<grid, kThreads, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

template <int HD>
cudaError_t launch_bwd(const BwdParams& p, int grid, cudaStream_t s) {
  using C = BwdCfg<HD>;
  // once per instantiation and process (host threads of in-process ranks race here)
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_bwd_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_bwd_kernel<HD><<<grid, kBwdThreads, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

}  // namespace attn
}  // namespace sm100

bool attn_fused_supported(const AttnDesc& d) {
  if (!(d.head_dim == 64 || d.head_dim == 128)) return false;
  if (d.seq <= 0 || d.seq % 8 != 0 || d.heads <= 0 || d.samples <= 0) return false;
  if (d.ld_qkv % 8 != 0 || d.ld_o % 8 != 0) return false;
  if (reinterpret_cast<uintptr_t>(d.qkv) % 16 || reinterpret_cast<uintptr_t>(d.o) % 16)
    return false;
  if (d.seq > (1 << 30) / 2 || d.samples > 65535) return false;
  return true;
}

cudaError_t attn_fwd_sm100(const AttnDesc& d, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d)) {
    g_attn_err = "attn_fwd_sm100: unsupported shape (head_dim must be 64 or 128, rows 16-byte aligned)";
    return cudaErrorInvalidValue;
  }
  FwdParams p;
  std::memset(&p, 0, sizeof(p));
  if (!encode_3d(&p.tm_qkv, d.qkv, 3 * d.heads * d.head_dim, d.seq, d.samples, d.ld_qkv, 128))
    return cudaErrorInvalidValue;
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.hd = (int)d.head_dim;
  p.n_pairs = (int)((d.seq + 2 * BQ - 1) / (2 * BQ));
  p.n_kv = (int)((d.seq + BKV - 1) / BKV);
  p.c = d.scale * kLog2e;
  p.o = static_cast<__nv_bfloat16*>(d.o);
  p.ld_o = d.ld_o;
  p.lse = d.lse;
  const long long grid = (long long)p.n_pairs * d.heads * d.samples;
  if (grid > 0x7fffffffLL) {
    g_attn_err = "attn_fwd_sm100: grid too large";
    return cudaErrorInvalidValue;
  }
  cudaError_t e = d.head_dim == 128 ? launch_fwd<128>(p, (int)grid, s) : launch_fwd<64>(p, (int)grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_fwd_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

cudaError_t attn_bwd_sm100(const AttnDesc& d, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d) || !d.dout || !d.delta || !d.dqkv || !d.dst || !d.lse ||
      d.ld_o % 8 != 0 || reinterpret_cast<uintptr_t>(d.dout) % 16 ||
      reinterpret_cast<uintptr_t>(d.dqkv) % 16 || reinterpret_cast<uintptr_t>(d.dst) % 16) {
    g_attn_err = "attn_bwd_sm100: unsupported shape or missing operand";
    return cudaErrorInvalidValue;
  }
  BwdParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t cols = 3 * d.heads * d.head_dim;
  if (!encode_3d(&p.tm_kv, d.qkv, cols, d.seq, d.samples, d.ld_qkv, 128) ||
      !encode_3d(&p.tm_q, d.qkv, cols, d.seq, d.samples, d.ld_qkv, BQB) ||
      !encode_3d(&p.tm_do, d.dout, d.heads * d.head_dim, d.seq, d.samples, d.ld_o, BQB) ||
      !encode_3d(&p.tm_dst, d.dst, d.seq, d.seq, d.samples * d.heads, d.seq, 128))
    return cudaErrorInvalidValue;
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.n_kt = (int)((d.seq + 127) / 128);
  p.n_qt = (int)((d.seq + BQB - 1) / BQB);
  p.c = d.scale * kLog2e;
  p.scale = d.scale;
  p.lse = d.lse;
  p.delta = d.delta;
  p.dqkv = static_cast<__nv_bfloat16*>(d.dqkv);
  p.ld_qkv = d.ld_qkv;
  p.trace = nullptr;
  if (std::getenv("TESS_ATTN_TRACE")) {
    static long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 8 * 64 * sizeof(long long));
    cudaMemsetAsync(tr, 0, 8 * 64 * sizeof(long long), s);
    p.trace = tr;
    g_attn_trace = tr;
  }
  const long long grid = (long long)p.n_kt * d.heads * d.samples;
  if (grid > 0x7fffffffLL) {
    g_attn_err = "attn_bwd_sm100: grid too large";
    return cudaErrorInvalidValue;
  }
  cudaError_t e = d.head_dim == 128 ? launch_bwd<128>(p, (int)grid, s) : launch_bwd<64>(p, (int)grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_bwd_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace tess
// shared-memory budgets (227 KB opt-in per CTA)
static_assert(tess::sm100::attn::FwdCfg<128>::SMEM_BYTES <= 232448, "attn fwd smem");
static_assert(tess::sm100::attn::BwdCfg<128>::USED <= 232448, "attn bwd smem");
static_assert(tess::sm100::attn::BwdCfg<64>::USED <= 232448, "attn bwd smem");
