// Fused attention forward / backward for sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces, for bf16, the per-(sample, head) loop of the reference's
// attn_forward_rank / attn_backward_rank (proj/src/layers.cpp:383-456):
//   S = Q K^T / sqrt(hd), P = softmax_rows(S) (layers.cpp:44-58, no mask),
//   O = P V; backward dV = P^T dO, dP = dO V^T, dS = P * (dP - rowsum(dP*P))
//   / sqrt(hd) (layers.cpp:60-74), dQ = dS K, dK = dS^T Q. The row term
//   rowsum(dP*P) is computed as rowsum(dO*O) inside the dQ pass.
// Neither S nor P reaches HBM: the forward keeps one log2-sum-exp per query
// row, the backward recomputes P from it.
//
// ---------------------------------------------------------------- forward
// Unit = one (sample, head) and two 128-query tiles A and B that share
// every K/V tile (halving K/V traffic). Persistent: one CTA per SM takes
// units in a strided order; the next unit's Q tiles load once the current
// unit's last score MMAs have read its own, its first scores run while the
// current unit's O is written out. 320 threads:
//   warp 0      TMA producer: Q_A, Q_B per unit, K_j, V_j into a ring of
//               KV_STAGES 128-key tiles (128B-swizzled boxes {64, 128}),
//               continuing across units.
//   warp 1      MMA issuer + TMEM owner (warp-wide, one elected lane; each
//               K=128 block of MMAs one PTX statement). Per key tile j:
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

// exp2_fma on a pair with packed fp32 ops (FFMA2 / FADD2): 2 lanes' worth of
// the polynomial per issue slot, for the pair-aligned share of the forward's
// exponentials moved off the MUFU pipe.
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 K = make_float2(12582912.0f, 12582912.0f);  // 1.5 * 2^23
  const float2 t = add2(x, K);
  const float2 j = add2(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = fma2(j, make_float2(-1.0f, -1.0f), x);
  float2 q = fma2(make_float2(0.05286731571f, 0.05286731571f), f,
                  make_float2(0.2421521395f, 0.2421521395f));
  q = fma2(q, f, make_float2(0.6935868263f, 0.6935868263f));
  q = fma2(q, f, make_float2(0.9999627471f, 0.9999627471f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

constexpr int kThreads = 320;
// which of every 8 exponentials of the forward use exp2_fma (bit e & 7)
#ifndef TESS_ATTN_FWD_POLY
#define TESS_ATTN_FWD_POLY 0
#endif
constexpr int kFwdPolyMask = TESS_ATTN_FWD_POLY;
constexpr int BQ = 128;   // query rows per tile (UMMA M)
constexpr int BKV = 128;  // keys per tile (UMMA N of S, K of P V)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units


struct FwdParams {
  CUtensorMap tm_qkv;  // 3-D view [cols, S, samples] of qkv, box {64, 128, 1}
  int S, H, n_pairs, n_kv;
  int hd;
  int units;  // samples * H * n_pairs
  float c;    // scale * log2(e)
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
  uint64_t* q_full = bars;                        // 1: Q_A, Q_B of the unit
  uint64_t* q_free = bars + 1;                    // 1: ... read by its last S MMA
  uint64_t* kv_full = bars + 2;                   // KV_STAGES
  uint64_t* kv_empty = kv_full + C::KV_STAGES;    // KV_STAGES
  uint64_t* s_full = kv_empty + C::KV_STAGES;     // 2 (tile A, B)
  uint64_t* p_full = s_full + 2;                  // 2
  uint64_t* o_full = p_full + 2;                  // 1
  uint64_t* acc_free = o_full + 1;                // 2: O_t read out (4 warps each)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n = p.n_kv;
  // unit = (sample * H + head) * n_pairs + pair
  auto unit_coords = [&](int unit, int& q0, int& head, int& smp) {
    q0 = (unit % p.n_pairs) * 2 * BQ;
    head = (unit / p.n_pairs) % p.H;
    smp = unit / (p.n_pairs * p.H);
  };

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_free, 1);
    for (int s = 0; s < C::KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
      mbar_init(&acc_free[t], 4);
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
      int stage = 0, round = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < p.units; unit += gridDim.x, ++round) {
      int q0, head, smp;
      unit_coords(unit, q0, head, smp);
      const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;
      // Q_A, Q_B: free once the previous unit's last score MMA has read them
      if (round > 0) mbar_wait(q_free, (round - 1) & 1);
      mbar_expect_tx(q_full, 2 * C::Q_BYTES);
#pragma unroll
      for (int c = 0; c < HD / 64; ++c) {
        tma_load_3d(smem + C::OFF_QA + c * 16384, &p.tm_qkv, q_full, col_q + c * 64, q0, smp);
        tma_load_3d(smem + C::OFF_QB + c * 16384, &p.tm_qkv, q_full, col_q + c * 64, q0 + BQ,
                    smp);
      }
      for (int j = 0; j < n; ++j) {
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
    }
  } else if (warp == 1) {
    // --------------------------------------------------------- MMA issuer
    // warp-wide: one elected lane issues each K=128 block of MMAs as one PTX
    // statement (descriptors advanced in registers)
    constexpr uint32_t idesc_s = idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16(BQ, HD, false, true);
    const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t kmaj_q = make_sdesc(sbase + C::OFF_QA, 16, 1024);  // Q_B at Q_BYTES
    const uint64_t kmaj_kv = make_sdesc(sbase + C::OFF_KV, 16, 1024);
    const uint64_t mn_kv = make_sdesc(sbase + C::OFF_KV, 16384, 1024);
    constexpr uint64_t kQ = (uint64_t)(C::Q_BYTES >> 4), kKV = (uint64_t)(C::KV_BYTES >> 4);
    auto kmaj_off = [](int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); };
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
    auto issue_s = [&](int t, int ks) {
      const uint32_t d = tm + C::TM_S0 + t * BKV;
      const uint64_t qa = kmaj_q + (uint64_t)t * kQ, kb = kmaj_kv + (uint64_t)ks * kKV;
      if constexpr (HD == 128) {
        mma_k128_ss_kk(d, qa, kb, idesc_s, 0u);
      } else {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_warp(d, qa + kmaj_off(kk), kb + kmaj_off(kk), idesc_s, kk > 0 ? 1u : 0u);
      }
      mma_commit_warp(&s_full[t]);
    };
    // O += P V with P (bf16 pairs) in tensor memory: the consumed S columns
    // [0, 64) of the tile's S buffer, 8 columns per 16 keys
    auto issue_pv = [&](int t, int vs, bool acc) {
      mma_k128_ts_n(tm + C::TM_O0 + t * 128, tm + C::TM_S0 + t * BKV, mn_kv + (uint64_t)vs * kKV,
                    idesc_pv, acc ? 1u : 0u);
    };
    // persistent over units; g counts key steps over all units (barrier
    // parities), round the units of this CTA
    int g = 0, round = 0;
    for (int unit = blockIdx.x; unit < p.units; unit += gridDim.x, ++round) {
      mbar_wait(q_full, round & 1);
      tc_fence_after();
      int ks = next_kv();
      issue_s(0, ks);  // over the previous unit's P_A: in order behind its P V
      issue_s(1, ks);
      mma_commit_warp(&kv_empty[ks]);
      if (n == 1) mma_commit_warp(q_free);
      for (int j = 0; j < n; ++j, ++g) {
        const int vs = next_kv();
        const bool more = j + 1 < n;
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&p_full[t], g & 1);
          if (j == 0 && round > 0) mbar_wait(&acc_free[t], (round - 1) & 1);  // O_t read out
          tc_fence_after();
          issue_pv(t, vs, j > 0);
          if (t == 0 && more) {
            ks = next_kv();
            issue_s(0, ks);
          }
        }
        mma_commit_warp(&kv_empty[vs]);
        if (more) {
          issue_s(1, ks);
          mma_commit_warp(&kv_empty[ks]);
          if (j + 2 == n) mma_commit_warp(q_free);  // the unit's last reads of Q_A, Q_B
        }
      }
      mma_commit_warp(o_full);
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
    int g = 0, round = 0;
    for (int unit = blockIdx.x; unit < p.units; unit += gridDim.x, ++round) {
    int q0, head, smp;
    unit_coords(unit, q0, head, smp);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j, ++g) {
      mbar_wait(&s_full[t], g & 1);
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
      // dependent fmax / fadd chain is ~4 clk x 128 of latency per tile);
      // 3-input max and packed fp32 pairs halve their issue slots
      float mp[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mp[k] = s[k];
#pragma unroll
      for (int e = 8; e < BKV; e += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k) mp[k] = max3f(mp[k], s[e + k], s[e + 8 + k < BKV ? e + 8 + k : e + k]);
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
      float2 rp[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      const float2 c2 = make_float2(cl2, cl2), nm2 = make_float2(-m_used, -m_used);
#pragma unroll
      for (int e = 0; e < BKV; e += 2) {
        const float2 xv = fma2(make_float2(s[e], s[e + 1]), c2, nm2);
        if ((kFwdPolyMask >> (e & 7)) & 1) {  // pair on the FMA pipe
          const float2 pv = exp2_fma2(xv);
          s[e] = pv.x;
          s[e + 1] = pv.y;
        } else {
          s[e] = ex2_approx(xv.x);
          s[e + 1] = ex2_approx(xv.y);
        }
        rp[(e >> 1) & 3] = add2(rp[(e >> 1) & 3], make_float2(s[e], s[e + 1]));
      }
      l += ((rp[0].x + rp[0].y) + (rp[1].x + rp[1].y)) + ((rp[2].x + rp[2].y) + (rp[3].x + rp[3].y));
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
    mbar_wait(o_full, round & 1);
    tc_fence_after();
    const int qrow = q0 + t * BQ + r;
    const float inv = 1.0f / l;
    __nv_bfloat16* orow = p.o + ((long long)smp * p.S + qrow) * p.ld_o + (long long)head * HD;
    // the row of O_t: all loads in flight, one wait, then O_t is released to
    // the next unit's first P V before the stores
    uint32_t ov[HD];
#pragma unroll
    for (int c = 0; c < HD / 32; ++c)
      tmem_ld32_nowait(t_o + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&ov[c * 32]));
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) reg_fence32(*reinterpret_cast<uint32_t(*)[32]>(&ov[c * 32]));
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_free[t]);
    if (qrow < p.S) {
#pragma unroll
      for (int u = 0; u < HD / 8; ++u) {
        const uint32_t* x = &ov[u * 8];
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(x[0]) * inv, __uint_as_float(x[1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(x[2]) * inv, __uint_as_float(x[3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(x[4]) * inv, __uint_as_float(x[5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(x[6]) * inv, __uint_as_float(x[7]) * inv);
        *reinterpret_cast<uint4*>(orow + u * 8) = w;
      }
    }
    if (qrow < p.S) p.lse[((long long)smp * p.H + head) * p.S + qrow] = m_used + __log2f(l);
    }
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
// which of every 4 exponentials of the backward use exp2_fma (bit u)
#ifndef TESS_ATTN_BWD_POLY
#define TESS_ATTN_BWD_POLY 8
#endif
constexpr int kBwdPolyMask = TESS_ATTN_BWD_POLY;



// ---------------------------------------------------- backward: dK, dV pass
// dV = P^T dO and dK = scale * dS^T Q per 128-key tile, walking the query
// tiles; dQ is the separate dQ pass (no dS leaves the SM in either).
// Persistent: one CTA per SM takes (sample, head, key tile) units in a
// strided order; the next unit's K / V load as soon as the current unit's
// last score MMAs have read theirs, and its first scores run while the
// current unit's dK / dV are written out. 320 threads:
//   warp 0      TMA: K, V per unit; Q_i (+ its lse and delta rows) and dO_i
//               into two-slot rings (continuing across units).
//   warp 1      MMA issuer (warp-wide, one elected lane; each K=128 block
//               of MMAs one PTX statement), all M=128 N=128:
//                 dV += P^T(i) dO_i          (A = P^T in TMEM)
//                 S^T(i+1) = K Q_{i+1}^T     (over the consumed P^T, in order)
//                 dK += dS^T(i) Q_i          (A = dS^T in TMEM)
//                 dP^T(i+1) = V dO_{i+1}^T   (over dS^T(i), in order behind dK)
//   warps 2-9   thread = key row, group g = queries [64g, 64g+64):
//               P^T = 2^(c S^T - lse) -> bf16 pairs over the thread's own
//               consumed S^T columns, then dS^T = P^T (dP^T - delta) -> bf16
//               over its own consumed dP^T columns (unscaled; the 1/sqrt(hd)
//               goes to dK's epilogue); at the end dK, dV out.
// No dS^T in shared memory: the kernel is bound by the shared-memory port
// (SS score MMAs alone need all 128 B/clk), and a dS^T store + its dK read
// were 64 KB of the ~320 KB it moved per query tile.
// TMEM: S^T / P^T [0,128), dP^T / dS^T [128,256), dV [256,256+hd),
// dK [384,384+hd).
constexpr int kKvThreads = 320;

struct KvParams {
  CUtensorMap tm_kv;   // qkv view [3*H*hd, S, samples], box {64, 128}: K, V, Q tiles
  CUtensorMap tm_do;   // dO view [H*hd, S, samples], box {64, 128}
  CUtensorMap tm_lse;  // lse [S, samples*H] fp32, box {128, 1} (rows past S read 0)
  CUtensorMap tm_dlt;  // delta, same view
  int S, H, n;         // n = key tiles = query tiles
  int units;           // samples * H * n
  float c, scale;
  __nv_bfloat16* dqkv;
  long long ld_qkv;
};

template <int HD>
struct KvCfg {
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;         // 2 slots
  static constexpr int OFF_DO = 4 * TILE;        // 2 slots
  static constexpr int OFF_LD = 6 * TILE;        // per Q slot: lse[128] | delta[128]
  static constexpr int OFF_BAR = OFF_LD + 2 * 1024;
  static constexpr int USED = OFF_BAR + 256;
  static constexpr int SMEM_BYTES = USED + 1024 <= 232448 ? USED + 1024 : 232448;
  static constexpr int TMEM_COLS = 512;
  static constexpr int TM_S = 0, TM_DP = 128, TM_DV = 256, TM_DK = 384;
};

template <int HD>
__global__ void __launch_bounds__(kKvThreads, 1) attn_bwd_kv_kernel(const __grid_constant__ KvParams p) {
  using C = KvCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((smem - smem_raw) + C::USED > C::SMEM_BYTES) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;     // 2
  uint64_t* q_empty = bars + 3;    // 2
  uint64_t* do_full = bars + 5;    // 2
  uint64_t* do_empty = bars + 7;   // 2
  uint64_t* s_full = bars + 9;     // S^T(i) in TMEM
  uint64_t* p_full = bars + 10;    // P^T(i) in TMEM (8 warps)
  uint64_t* dp_full = bars + 11;   // dP^T(i) in TMEM
  uint64_t* ds_full = bars + 12;   // dS^T(i) in TMEM (8 warps)
  uint64_t* fin = bars + 13;       // dK, dV of the unit complete
  uint64_t* kv_empty = bars + 14;  // the unit's last MMA reading K / V done
  uint64_t* acc_free = bars + 15;  // dK, dV read out of TMEM (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n = p.n;
  const int units = p.units;  // (sample * H + head) * n + key tile

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&do_full[s], 1);
      mbar_init(&do_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(fin, 1);
    mbar_init(kv_empty, 1);
    mbar_init(acc_free, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&p.tm_kv);
    prefetch_tmap(&p.tm_do);
    prefetch_tmap(&p.tm_lse);
    prefetch_tmap(&p.tm_dlt);
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
      int gs = 0, round = 0;
      for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
        const int job = unit / n, k0 = (unit % n) * 128;  // job = sample * H + head
        const int head = job % p.H, smp = job / p.H;
        const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;
        if (round > 0) mbar_wait(kv_empty, (round - 1) & 1);
        mbar_expect_tx(kv_full, 2 * C::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_3d(smem + C::OFF_K + c * 16384, &p.tm_kv, kv_full, col_k + c * 64, k0, smp);
          tma_load_3d(smem + C::OFF_V + c * 16384, &p.tm_kv, kv_full, col_v + c * 64, k0, smp);
        }
        for (int i = 0; i < n; ++i, ++gs) {
          const int s = gs & 1, u = gs >> 1;
          if (u > 0) mbar_wait(&q_empty[s], (u - 1) & 1);
          mbar_expect_tx(&q_full[s], C::TILE + 1024);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_Q + s * C::TILE + c * 16384, &p.tm_kv, &q_full[s],
                        col_q + c * 64, i * 128, smp);
          tma_load_2d(smem + C::OFF_LD + s * 1024, &p.tm_lse, &q_full[s], i * 128, job);
          tma_load_2d(smem + C::OFF_LD + s * 1024 + 512, &p.tm_dlt, &q_full[s], i * 128, job);
          if (u > 0) mbar_wait(&do_empty[s], (u - 1) & 1);
          mbar_expect_tx(&do_full[s], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_DO + s * C::TILE + c * 16384, &p.tm_do, &do_full[s],
                        head * HD + c * 64, i * 128, smp);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);  // S^T, dP^T
    constexpr uint32_t idesc_g = idesc_bf16(128, HD, false, true);    // dV, dK
    const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t kmaj_k = make_sdesc(sbase + C::OFF_K, 16, 1024);
    const uint64_t kmaj_v = make_sdesc(sbase + C::OFF_V, 16, 1024);
    const uint64_t kmaj_q = make_sdesc(sbase + C::OFF_Q, 16, 1024);
    const uint64_t kmaj_do = make_sdesc(sbase + C::OFF_DO, 16, 1024);
    const uint64_t mn_q = make_sdesc(sbase + C::OFF_Q, 16384, 1024);
    const uint64_t mn_do = make_sdesc(sbase + C::OFF_DO, 16384, 1024);
    constexpr uint64_t kTile = (uint64_t)(C::TILE >> 4);
    auto kmaj_off = [](int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); };
    auto issue_scores = [&](uint32_t d, uint64_t a, uint64_t b) {
      if constexpr (HD == 128) {
        mma_k128_ss_kk(d, a, b, idesc_s, 0u);
      } else {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_warp(d, a + kmaj_off(kk), b + kmaj_off(kk), idesc_s, kk > 0 ? 1u : 0u);
      }
    };
    int gs = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
      mbar_wait(kv_full, round & 1);
      mbar_wait(&q_full[gs & 1], (gs >> 1) & 1);
      tc_fence_after();
      issue_scores(tm + C::TM_S, kmaj_k, kmaj_q + (gs & 1) * kTile);
      mma_commit_warp(s_full);
      mbar_wait(&do_full[gs & 1], (gs >> 1) & 1);
      tc_fence_after();
      issue_scores(tm + C::TM_DP, kmaj_v, kmaj_do + (gs & 1) * kTile);
      mma_commit_warp(dp_full);
      if (n == 1) mma_commit_warp(kv_empty);
      for (int i = 0; i < n; ++i, ++gs) {
        const int s = gs & 1;
        // dV += P^T(i) dO_i; P^T of queries [16kk, 16kk+16) at column 32(kk/2) + 8(kk%2)
        mbar_wait(p_full, gs & 1);
        if (i == 0 && round > 0) mbar_wait(acc_free, (round - 1) & 1);  // previous dK, dV out
        tc_fence_after();
        mma_k128_ts_n_pairs(tm + C::TM_DV, tm + C::TM_S, mn_do + s * kTile, idesc_g, i > 0 ? 1u : 0u);
        mma_commit_warp(&do_empty[s]);
        const int sn = s ^ 1, un = (gs + 1) >> 1;
        if (i + 1 < n) {
          mbar_wait(&q_full[sn], un & 1);
          tc_fence_after();
          issue_scores(tm + C::TM_S, kmaj_k, kmaj_q + sn * kTile);
          mma_commit_warp(s_full);
        }
        // dK += dS^T(i) Q_i; dS^T of queries [16kk, 16kk+16) at column
        // 64(kk/4) + 8(kk%4) of the dP^T columns
        mbar_wait(ds_full, gs & 1);
        tc_fence_after();
        mma_k128_ts_n_quads(tm + C::TM_DK, tm + C::TM_DP, mn_q + s * kTile, idesc_g, i > 0 ? 1u : 0u);
        mma_commit_warp(&q_empty[s]);
        if (i + 1 < n) {
          // dP^T(i+1) over dS^T(i): in order behind dK(i), its reader
          mbar_wait(&do_full[sn], un & 1);
          tc_fence_after();
          issue_scores(tm + C::TM_DP, kmaj_v, kmaj_do + sn * kTile);
          mma_commit_warp(dp_full);
          if (i + 2 == n) mma_commit_warp(kv_empty);  // the unit's last K / V readers issued
        }
      }
      mma_commit_warp(fin);
    }
  } else {
    // ------------------------------------------ softmax-gradient warps
    const int quad = warp & 3;
    const int g = (warp - 2) >> 2;   // queries [64g, 64g+64) of each tile
    const int r = quad * 32 + lane;  // key row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float cl2 = p.c, scale = p.scale;
    int gs = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
    const int job = unit / n, k0 = (unit % n) * 128;
    const int head = job % p.H, smp = job / p.H;
    const int col_q = head * 3 * HD;
    for (int i = 0; i < n; ++i, ++gs) {
      const int s = gs & 1;
      const uint32_t ldw = smem_u32(smem + C::OFF_LD + s * 1024) + (uint32_t)g * 256u;
      mbar_wait(&q_full[s], (gs >> 1) & 1);  // lse, delta rows of the slot
      mbar_wait(s_full, gs & 1);
      tc_fence_after();
      // ---- P^T = 2^(c S^T - lse) over the group's 64 query columns
      float pr[64];
      {
        uint32_t a0[32], a1[32];
        tmem_ld32_nowait(tmem + lane_off + C::TM_S + g * 64, a0);
        tmem_ld32_nowait(tmem + lane_off + C::TM_S + g * 64 + 32, a1);
        tmem_wait_ld();
        reg_fence32(a0);
        reg_fence32(a1);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          pr[e] = __uint_as_float(a0[e]);
          pr[32 + e] = __uint_as_float(a1[e]);
        }
      }
#pragma unroll
      for (int e4 = 0; e4 < 16; ++e4) {
        float4 l4;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(l4.x), "=f"(l4.y), "=f"(l4.z), "=f"(l4.w)
                     : "r"(ldw + (uint32_t)(16 * e4)));
        const float lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
        for (int u = 0; u < 4; u += 2) {
          const int e = 4 * e4 + u;
          const float2 xv = fma2(make_float2(pr[e], pr[e + 1]), make_float2(cl2, cl2),
                                 make_float2(-lv[u], -lv[u + 1]));
          pr[e] = (kBwdPolyMask >> u) & 1 ? exp2_fma(xv.x) : ex2_approx(xv.x);
          pr[e + 1] = (kBwdPolyMask >> (u + 1)) & 1 ? exp2_fma(xv.y) : ex2_approx(xv.y);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // queries [64g+32h, +32) -> cols [64g+32h, +16)
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(pr[32 * h + 2 * e], pr[32 * h + 2 * e + 1]);
        tmem_st16(tmem + lane_off + C::TM_S + g * 64 + h * 32, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // ---- dS^T = P^T (dP^T - delta) (unscaled) over the thread's own
      // consumed dP^T columns: 64 queries -> 32 bf16-pair columns
      mbar_wait(dp_full, gs & 1);
      tc_fence_after();
      const uint32_t dpc = tmem + lane_off + C::TM_DP + g * 64;
      uint32_t d[64];
      {
        uint32_t (&d0)[32] = *reinterpret_cast<uint32_t(*)[32]>(d);
        uint32_t (&d1)[32] = *reinterpret_cast<uint32_t(*)[32]>(d + 32);
        tmem_ld32_nowait(dpc, d0);
        tmem_ld32_nowait(dpc + 32, d1);
        tmem_wait_ld();
        reg_fence32(d0);
        reg_fence32(d1);
      }
      uint32_t pk[32];
#pragma unroll
      for (int e4 = 0; e4 < 16; ++e4) {
        float4 d4;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(d4.x), "=f"(d4.y), "=f"(d4.z), "=f"(d4.w)
                     : "r"(ldw + 512u + (uint32_t)(16 * e4)));
        const int e = 4 * e4;
        const float2 a = mul2(make_float2(pr[e], pr[e + 1]),
                              add2(make_float2(__uint_as_float(d[e]), __uint_as_float(d[e + 1])),
                                   make_float2(-d4.x, -d4.y)));
        const float2 b = mul2(make_float2(pr[e + 2], pr[e + 3]),
                              add2(make_float2(__uint_as_float(d[e + 2]), __uint_as_float(d[e + 3])),
                                   make_float2(-d4.z, -d4.w)));
        pk[2 * e4] = pack_bf16x2(a.x, a.y);
        pk[2 * e4 + 1] = pack_bf16x2(b.x, b.y);
      }
      tmem_st32(dpc, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    // ---- dK, dV out (dK carries the dS scale)
    mbar_wait(fin, round & 1);
    tc_fence_after();
    const int krow = k0 + r;
    __nv_bfloat16* drow = p.dqkv + ((long long)smp * p.S + krow) * p.ld_qkv + col_q;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {  // group g: columns [g*HD/2, (g+1)*HD/2)
        const int col = g * (HD / 2) + c * 16;
        uint32_t v[16];
        tmem_ld16_nowait(tmem + lane_off + (which == 0 ? C::TM_DK : C::TM_DV) + col, v);
        tmem_wait_ld();
        reg_fence16(v);
        if (krow < p.S) {
          __nv_bfloat16* dst = drow + (which + 1) * HD + col;
          const float f = which == 0 ? scale : 1.0f;
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
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_free);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------- backward: dQ pass
// dQ = scale * dS K computed per 128-query tile with S, P, dP and dS
// recomputed on chip (the flash-attention "dQ pass"): no dS ever reaches
// HBM, dQ accumulates in TMEM over the key tiles in order (deterministic, no
// atomics). Persistent: one CTA per SM takes (sample, head, query tile)
// units in a strided order; the next unit's Q / dO load as soon as the
// current unit's last score MMA has read its own. 320 threads:
//   warp 0      TMA: Q_i, dO_i per unit; K_j into a 3-slot ring, V_j into a
//               2-slot ring.
//   warp 1      MMA issuer (warp-wide, one elected lane; each K=128 block
//               one PTX statement), all M=128 N=128:
//                 S(j+1) = Q K^T      (A = Q in smem)   once S(j) is loaded
//                 dP(j+1) = dO V^T    (A = dO in smem)  into the other dP
//                                      buffer, right behind S(j+1)
//                 dQ += dS(j) K_j     (A = dS in TMEM over the consumed
//                                      columns of dP(j)'s buffer, B = K_j
//                                      read MN-major)
//               dP is double-buffered, so dP(j+1) does not wait for dQ(j):
//               the softmax warps find S and dP of the next key tile ready.
//   warps 2-9   thread = query row, group g = keys [64g, 64g+64): first
//               delta = rowsum(dO * O) of its row (each group one half of
//               hd, dO from shared memory, summed through shared memory;
//               written out for the dK/dV pass, which runs after this one),
//               then per key tile P = 2^(c S - lse) (lse, delta are the
//               row's own: registers) while dP loads, dS = P (dP - delta) ->
//               bf16 pairs over its own consumed dP columns; at the end dQ
//               out of TMEM (scaled) into the Q slot of dqkv.
// TMEM: S [0,128), dP / dS buffers [128,256) and [256,384), dQ [384,384+hd).
// (Q and dO in TMEM as TS operands instead -- round 2's earlier form --
// leaves no room for the second dP buffer: 3-4 % slower,
// profiles/r2_attn_dq_dp_double_buffer_ab.log.)
constexpr int kDqThreads = 320;

struct DqParams {
  CUtensorMap tm_kv;  // qkv view, box {64, 128}: Q_i, K_j, V_j
  CUtensorMap tm_do;  // dO view, box {64, 128}
  int S, H, n_qt, n_kt;
  int units;          // samples * H * n_qt
  float c, scale;
  const float* lse;
  float* delta;                // out: rowsum(dO * O) [samples, H, S]
  const __nv_bfloat16* o;      // forward output O (ld_o)
  long long ld_o;
  __nv_bfloat16* dqkv;
  long long ld_qkv;
};

template <int HD>
struct DqCfg {
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int K_STAGES = 3, V_STAGES = 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_DO = TILE;
  static constexpr int OFF_K = 2 * TILE;
  static constexpr int OFF_V = OFF_K + K_STAGES * TILE;
  static constexpr int OFF_BAR = OFF_V + V_STAGES * TILE;
  static constexpr int OFF_RED = OFF_BAR + 256;  // delta halves: 2 x 128 fp32
  static constexpr int USED = OFF_RED + 1024;
  static constexpr int SMEM_BYTES = USED + 1024 <= 232448 ? USED + 1024 : 232448;
  static constexpr int TMEM_COLS = 512;
  // dP / dS double-buffered: dP(j+1) is computed while dS(j) waits for dQ(j)
  static constexpr int TM_S = 0, TM_DP = 128, TM_DQ = 384;
};

template <int HD>
__global__ void __launch_bounds__(kDqThreads, 1) attn_dq_kernel(const __grid_constant__ DqParams p) {
  using C = DqCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((smem - smem_raw) + C::USED > C::SMEM_BYTES) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* qd_full = bars + 0;                 // Q_i, dO_i of the unit in shared memory
  uint64_t* qd_free = bars + 1;                 // ... read by the unit's last score MMA
  uint64_t* k_full = bars + 2;                  // K_STAGES
  uint64_t* k_empty = k_full + C::K_STAGES;     // K_STAGES
  uint64_t* v_full = k_empty + C::K_STAGES;     // V_STAGES
  uint64_t* v_empty = v_full + C::V_STAGES;     // V_STAGES
  uint64_t* s_full = v_empty + C::V_STAGES;     // S(j) in TMEM
  uint64_t* s_loaded = s_full + 1;              // S(j) in registers (8 warps)
  // per dP buffer: the softmax warps run up to one step ahead of the issuer
  uint64_t* dp_full = s_loaded + 1;             // 2: dP(j) in TMEM buffer j & 1
  uint64_t* ds_full = dp_full + 2;              // 2: dS(j) in TMEM buffer j & 1 (8 warps)
  uint64_t* fin = ds_full + 2;                  // dQ of the unit complete
  uint64_t* acc_free = fin + 1;                 // dQ read out of TMEM (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n = p.n_kt;
  const int units = p.units;  // (sample * H + head) * n_qt + query tile

  if (warp == 0 && lane == 0) {
    mbar_init(qd_full, 1);
    mbar_init(qd_free, 1);
    for (int s = 0; s < C::K_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::V_STAGES; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_loaded, 8);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dp_full[b], 1);
      mbar_init(&ds_full[b], 8);
    }
    mbar_init(fin, 1);
    mbar_init(acc_free, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&p.tm_kv);
    prefetch_tmap(&p.tm_do);
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
      int gk = 0, round = 0;  // key steps over all units, units of this CTA
      for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
        const int job = unit / p.n_qt, q0 = (unit % p.n_qt) * 128;
        const int head = job % p.H, smp = job / p.H;
        const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;
        // Q / dO tiles: free once the previous unit's last score MMA read them
        if (round > 0) mbar_wait(qd_free, (round - 1) & 1);
        mbar_expect_tx(qd_full, 2 * C::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_3d(smem + C::OFF_Q + c * 16384, &p.tm_kv, qd_full, col_q + c * 64, q0, smp);
          tma_load_3d(smem + C::OFF_DO + c * 16384, &p.tm_do, qd_full, head * HD + c * 64, q0,
                      smp);
        }
        for (int j = 0; j < n; ++j, ++gk) {
          const int ks = gk % C::K_STAGES, ku = gk / C::K_STAGES;
          if (ku > 0) mbar_wait(&k_empty[ks], (ku - 1) & 1);
          mbar_expect_tx(&k_full[ks], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_K + ks * C::TILE + c * 16384, &p.tm_kv, &k_full[ks],
                        col_k + c * 64, j * 128, smp);
          const int vs = gk % C::V_STAGES, vu = gk / C::V_STAGES;
          if (vu > 0) mbar_wait(&v_empty[vs], (vu - 1) & 1);
          mbar_expect_tx(&v_full[vs], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_V + vs * C::TILE + c * 16384, &p.tm_kv, &v_full[vs],
                        col_v + c * 64, j * 128, smp);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);  // S, dP: B K-major
    constexpr uint32_t idesc_q = idesc_bf16(128, HD, false, true);    // dQ: B = K MN-major
    const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t kmaj_k = make_sdesc(sbase + C::OFF_K, 16, 1024);
    const uint64_t kmaj_v = make_sdesc(sbase + C::OFF_V, 16, 1024);
    const uint64_t kmaj_q = make_sdesc(sbase + C::OFF_Q, 16, 1024);
    const uint64_t kmaj_do = make_sdesc(sbase + C::OFF_DO, 16, 1024);
    const uint64_t mn_k = make_sdesc(sbase + C::OFF_K, 16384, 1024);
    constexpr uint64_t kTile = (uint64_t)(C::TILE >> 4);
    auto kmaj_off = [](int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); };
    auto issue_scores = [&](uint32_t d, uint64_t a, uint64_t b) {  // A, B K-major in smem
      if constexpr (HD == 128) {
        mma_k128_ss_kk(d, a, b, idesc_s, 0u);
      } else {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_warp(d, a + kmaj_off(kk), b + kmaj_off(kk), idesc_s, kk > 0 ? 1u : 0u);
      }
    };
    auto wait_k = [&](int g2) {
      mbar_wait(&k_full[g2 % C::K_STAGES], (g2 / C::K_STAGES) & 1);
      tc_fence_after();
    };
    auto wait_v = [&](int g2) {
      mbar_wait(&v_full[g2 % C::V_STAGES], (g2 / C::V_STAGES) & 1);
      tc_fence_after();
    };
    auto issue_s = [&](int g2) {
      wait_k(g2);
      issue_scores(tm + C::TM_S, kmaj_q, kmaj_k + (g2 % C::K_STAGES) * kTile);
      mma_commit_warp(s_full);
    };
    auto issue_dp = [&](int g2) {  // into buffer g2 & 1, whose dS(g2 - 2) dQ has read
      wait_v(g2);
      issue_scores(tm + C::TM_DP + (uint32_t)(g2 & 1) * 128u, kmaj_do, kmaj_v + (g2 % C::V_STAGES) * kTile);
      mma_commit_warp(&dp_full[g2 & 1]);
      mma_commit_warp(&v_empty[g2 % C::V_STAGES]);
    };
    int gk = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
      mbar_wait(qd_full, round & 1);
      tc_fence_after();
      issue_s(gk);
      issue_dp(gk);
      for (int j = 0; j < n; ++j, ++gk) {
        if (j + 1 < n) {
          // S(j+1) over S(j) once every warp holds S(j) in registers, and
          // dP(j+1) into the other buffer right behind it
          mbar_wait(s_loaded, gk & 1);
          issue_s(gk + 1);
          issue_dp(gk + 1);
          if (j + 2 == n) mma_commit_warp(qd_free);  // the unit's last reads of Q / dO
        }
        // dQ += dS(j) K_j; dS of keys [16kk, 16kk+16) at column 64(kk/4) +
        // 8(kk%4) of its dP buffer
        mbar_wait(&ds_full[gk & 1], (gk >> 1) & 1);
        if (j == 0 && round > 0) mbar_wait(acc_free, (round - 1) & 1);  // previous dQ out
        tc_fence_after();
        mma_k128_ts_n_quads(tm + C::TM_DQ, tm + C::TM_DP + (uint32_t)(gk & 1) * 128u,
                            mn_k + (gk % C::K_STAGES) * kTile, idesc_q, j > 0 ? 1u : 0u);
        mma_commit_warp(&k_empty[gk % C::K_STAGES]);
        if (n == 1) mma_commit_warp(qd_free);
      }
      mma_commit_warp(fin);
    }
  } else {
    // ------------------------------------------ softmax-gradient warps
    const int quad = warp & 3;
    const int g = (warp - 2) >> 2;   // keys [64g, 64g+64) of each key tile
    const int r = quad * 32 + lane;  // query row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float cl2 = p.c, scale = p.scale;
    constexpr int HW = HD / 2;  // hd columns per group
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);
    int gk = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
      const int job = unit / p.n_qt, q0 = (unit % p.n_qt) * 128;
      const int head = job % p.H, smp = job / p.H;
      const int qrow = q0 + r;
      const bool valid = qrow < p.S;
      const long long lrow = (long long)job * p.S + qrow;
      // padded query rows: Q, dO are zero there, dS = 0 whatever lse is
      const float lse = valid ? __ldg(p.lse + lrow) : 0.f;
      // the row's O half, loaded while Q / dO arrive
      uint4 ov[HW / 8];
      {
        const uint4* orow = reinterpret_cast<const uint4*>(
            p.o + ((long long)smp * p.S + qrow) * p.ld_o + (long long)head * HD + g * HW);
#pragma unroll
        for (int u = 0; u < HW / 8; ++u) ov[u] = valid ? __ldg(orow + u) : make_uint4(0, 0, 0, 0);
      }
      float dpart = 0.f;
      {
        // this half of rowsum(dO * O), dO from the unit's shared-memory tile
        // (16-byte pieces of the SW128 tile), in column order
        mbar_wait(qd_full, round & 1);
        const uint32_t base = smem_u32(smem + C::OFF_DO);
#pragma unroll
        for (int u = 0; u < HW / 8; ++u) {
          const int col = g * HW + 8 * u;  // first hd column of the piece
          const uint32_t a = base + (uint32_t)(col >> 6) * 16384u + (uint32_t)(r >> 3) * 1024u +
                             (uint32_t)(r & 7) * 128u + (uint32_t)((((col & 63) >> 3) ^ (r & 7)) << 4);
          uint32_t v[4];
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                       : "r"(a));
          const uint32_t ow[4] = {ov[u].x, ov[u].y, ov[u].z, ov[u].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 a2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[e]));
            const float2 b2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[e]));
            dpart = fmaf(a2.x, b2.x, dpart);
            dpart = fmaf(a2.y, b2.y, dpart);
          }
        }
      }
      // delta = (low half) + (high half), the same order in both groups
      red[g * 128 + r] = dpart;
      named_bar_sync(1, 256);
      const float dlt = red[r] + red[128 + r];
      named_bar_sync(1, 256);  // red is rewritten by the next unit
      if (g == 0 && valid) p.delta[lrow] = dlt;
      for (int j = 0; j < n; ++j, ++gk) {
        mbar_wait(s_full, gk & 1);
        tc_fence_after();
        float pr[64];
        {
          uint32_t a0[32], a1[32];
          tmem_ld32_nowait(tmem + lane_off + C::TM_S + g * 64, a0);
          tmem_ld32_nowait(tmem + lane_off + C::TM_S + g * 64 + 32, a1);
          tmem_wait_ld();
          reg_fence32(a0);
          reg_fence32(a1);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            pr[e] = __uint_as_float(a0[e]);
            pr[32 + e] = __uint_as_float(a1[e]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_loaded);
        // dP(j) (computed alongside S(j)) loads while the exponentials run
        mbar_wait(&dp_full[gk & 1], (gk >> 1) & 1);
        tc_fence_after();
        const uint32_t dpc = tmem + lane_off + C::TM_DP + (gk & 1) * 128 + g * 64;
        uint32_t d[64];
        uint32_t (&d0)[32] = *reinterpret_cast<uint32_t(*)[32]>(d);
        uint32_t (&d1)[32] = *reinterpret_cast<uint32_t(*)[32]>(d + 32);
        tmem_ld32_nowait(dpc, d0);
        tmem_ld32_nowait(dpc + 32, d1);
        // one exponential in four on the FMA pipe (same split as the dK/dV pass)
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float2 xv =
              fma2(make_float2(pr[e], pr[e + 1]), make_float2(cl2, cl2), make_float2(-lse, -lse));
          pr[e] = (kBwdPolyMask >> (e & 3)) & 1 ? exp2_fma(xv.x) : ex2_approx(xv.x);
          pr[e + 1] = (kBwdPolyMask >> ((e + 1) & 3)) & 1 ? exp2_fma(xv.y) : ex2_approx(xv.y);
        }
        tmem_wait_ld();
        reg_fence32(d0);
        reg_fence32(d1);
        // dS = P (dP - delta), unscaled (the 1/sqrt(hd) goes to the epilogue),
        // 64 keys -> columns [64g, 64g+32) of the consumed dP
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float2 v = mul2(make_float2(pr[2 * e], pr[2 * e + 1]),
                                add2(make_float2(__uint_as_float(d[2 * e]), __uint_as_float(d[2 * e + 1])),
                                     make_float2(-dlt, -dlt)));
          pk[e] = pack_bf16x2(v.x, v.y);
        }
        tmem_st32(dpc, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[gk & 1]);
      }
      // ---------------------------------------------- dQ of the unit out
      mbar_wait(fin, round & 1);
      tc_fence_after();
      __nv_bfloat16* drow =
          p.dqkv + ((long long)smp * p.S + qrow) * p.ld_qkv + (long long)head * 3 * HD;
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {  // group g: columns [g*HD/2, (g+1)*HD/2)
        const int col = g * (HD / 2) + c * 16;
        uint32_t v[16];
        tmem_ld16_nowait(tmem + lane_off + C::TM_DQ + col, v);
        tmem_wait_ld();
        reg_fence16(v);
        if (valid) {
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[u * 8 + 0]) * scale, __uint_as_float(v[u * 8 + 1]) * scale);
            w.y = pack_bf16x2(__uint_as_float(v[u * 8 + 2]) * scale, __uint_as_float(v[u * 8 + 3]) * scale);
            w.z = pack_bf16x2(__uint_as_float(v[u * 8 + 4]) * scale, __uint_as_float(v[u * 8 + 5]) * scale);
            w.w = pack_bf16x2(__uint_as_float(v[u * 8 + 6]) * scale, __uint_as_float(v[u * 8 + 7]) * scale);
            *reinterpret_cast<uint4*>(drow + col + u * 8) = w;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_free);
    }
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

// 2-D fp32 view [cols, rows] (row stride cols), box {128, 1}; columns past
// `cols` read as zero.
bool encode_rows_f32(CUtensorMap* map, const float* base, int64_t cols, int64_t rows) {
  auto fn = encode_fn();
  if (!fn) {
    g_attn_err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {128, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_attn_err = "cuTensorMapEncodeTiled (rows) failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

int device_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::mutex mu;
  static int cache[64] = {0};
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
  return cache[dev];
}

template <int HD>
cudaError_t launch_kv(const KvParams& p, int grid, cudaStream_t s) {
  using C = KvCfg<HD>;
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_bwd_kv_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_bwd_kv_kernel<HD><<<grid, kKvThreads, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

template <int HD>
cudaError_t launch_dq(const DqParams& p, int grid, cudaStream_t s) {
  using C = DqCfg<HD>;
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_dq_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_dq_kernel<HD><<<grid, kDqThreads, C::SMEM_BYTES, s>>>(p);
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
  const long long units = (long long)p.n_pairs * d.heads * d.samples;
  if (units > 0x7fffffffLL) {
    g_attn_err = "attn_fwd_sm100: too many units";
    return cudaErrorInvalidValue;
  }
  p.units = (int)units;
  const int grid = (int)std::min<long long>(units, device_sms());  // persistent
  cudaError_t e = d.head_dim == 128 ? launch_fwd<128>(p, grid, s) : launch_fwd<64>(p, grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_fwd_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

cudaError_t attn_bwd_kv_sm100(const AttnDesc& d, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d) || !d.dout || !d.delta || !d.dqkv || !d.lse || d.ld_o % 8 != 0 ||
      d.seq % 4 != 0 || reinterpret_cast<uintptr_t>(d.dout) % 16 ||
      reinterpret_cast<uintptr_t>(d.dqkv) % 16 || reinterpret_cast<uintptr_t>(d.lse) % 16 ||
      reinterpret_cast<uintptr_t>(d.delta) % 16) {
    g_attn_err = "attn_bwd_kv_sm100: unsupported shape or missing operand";
    return cudaErrorInvalidValue;
  }
  KvParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t cols = 3 * d.heads * d.head_dim;
  if (!encode_3d(&p.tm_kv, d.qkv, cols, d.seq, d.samples, d.ld_qkv, 128) ||
      !encode_3d(&p.tm_do, d.dout, d.heads * d.head_dim, d.seq, d.samples, d.ld_o, 128) ||
      !encode_rows_f32(&p.tm_lse, d.lse, d.seq, d.samples * d.heads) ||
      !encode_rows_f32(&p.tm_dlt, d.delta, d.seq, d.samples * d.heads))
    return cudaErrorInvalidValue;
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.n = (int)((d.seq + 127) / 128);
  p.c = d.scale * kLog2e;
  p.scale = d.scale;
  p.dqkv = static_cast<__nv_bfloat16*>(d.dqkv);
  p.ld_qkv = d.ld_qkv;
  const long long units = (long long)p.n * d.heads * d.samples;
  if (units > 0x7fffffffLL) {
    g_attn_err = "attn_bwd_kv_sm100: too many units";
    return cudaErrorInvalidValue;
  }
  p.units = (int)units;
  const int grid = (int)std::min<long long>(units, std::max(1, device_sms()));
  cudaError_t e = d.head_dim == 128 ? launch_kv<128>(p, grid, s) : launch_kv<64>(p, grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_bwd_kv_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

cudaError_t attn_dq_sm100(const AttnDesc& d, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d) || !d.dout || !d.delta || !d.dqkv || !d.lse || !d.o ||
      d.ld_o % 8 != 0 || reinterpret_cast<uintptr_t>(d.dout) % 16 ||
      reinterpret_cast<uintptr_t>(d.dqkv) % 16) {
    g_attn_err = "attn_dq_sm100: unsupported shape or missing operand";
    return cudaErrorInvalidValue;
  }
  DqParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t cols = 3 * d.heads * d.head_dim;
  if (!encode_3d(&p.tm_kv, d.qkv, cols, d.seq, d.samples, d.ld_qkv, 128) ||
      !encode_3d(&p.tm_do, d.dout, d.heads * d.head_dim, d.seq, d.samples, d.ld_o, 128))
    return cudaErrorInvalidValue;
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.n_qt = p.n_kt = (int)((d.seq + 127) / 128);
  p.c = d.scale * kLog2e;
  p.scale = d.scale;
  p.lse = d.lse;
  p.delta = d.delta;
  p.o = static_cast<const __nv_bfloat16*>(d.o);
  p.ld_o = d.ld_o;
  p.dqkv = static_cast<__nv_bfloat16*>(d.dqkv);
  p.ld_qkv = d.ld_qkv;
  const long long units = (long long)p.n_qt * d.heads * d.samples;
  if (units > 0x7fffffffLL) {
    g_attn_err = "attn_dq_sm100: too many units";
    return cudaErrorInvalidValue;
  }
  p.units = (int)units;
  const int grid = (int)std::min<long long>(units, std::max(1, device_sms()));
  cudaError_t e = d.head_dim == 128 ? launch_dq<128>(p, grid, s) : launch_dq<64>(p, grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_dq_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace tess
// shared-memory budgets (227 KB opt-in per CTA)
static_assert(tess::sm100::attn::FwdCfg<128>::SMEM_BYTES <= 232448, "attn fwd smem");
static_assert(tess::sm100::attn::DqCfg<128>::USED <= 232448, "attn dQ smem");
static_assert(tess::sm100::attn::DqCfg<128>::OFF_RED % 16 == 0, "attn dQ smem");
static_assert(tess::sm100::attn::KvCfg<128>::USED <= 232448, "attn dK/dV smem");
