// Tool-only experiment (not built into libtess): a single-query-tile
// forward, for attn_check. Measured against the product's two-tile
// attn_fwd_kernel at the cfg4 head shape (b 4, s 2048, 96 heads, hd 128;
// profiles/r2_attn_fwd_one_tile_ab.log): 0.77-0.80 ms vs 0.765 ms with one
// exponential in four on the FMA pipe, 0.80 ms with all on MUFU, and slower
// (0.83-0.85 ms) with the score stream running across units. ncu: tensor
// pipe 49.6 % (two-tile 48.8 %), XU 38.8 % (50.6 %). The softmax step takes
// about twice its MUFU time: the two warps of a sub-partition cover the same
// rows (TMEM lane quadrant) and swap row maxima every step, so they run in
// lock step and neither hides the other's TMEM-load / max / store latency.
// Included after kernels/attention_sm100.cu (same namespaces, helpers).
#pragma once

namespace tess {
namespace sm100 {
namespace attn {

// ------------------------------------------- forward, one query tile per CTA
// O = softmax(c Q K^T) V for one 128-query tile per unit, persistent over
// (sample, head, query tile) units. The score buffer is double-buffered in
// tensor memory, so S(j+1) runs on the tensor pipe while the softmax warps
// work on S(j), and Q sits in tensor memory (TS score MMAs: shared memory
// carries only K_j and V_j). 320 threads:
//   warp 0      TMA: Q per unit, K_j / V_j into 3- / 2-slot rings.
//   warp 1      MMA issuer (warp-wide): S(0), S(1); per key step j
//                 O (+)= P(j) V_j    (A = P over the consumed S(j) columns)
//                 S(j+2) = Q K_{j+2}^T into S(j)'s buffer, in order behind it
//   warps 2-9   thread = query row, group g = keys [64g, 64g+64) of each key
//               tile: the two groups of a row swap their partial row maxima
//               through shared memory (one 64-thread barrier per step), then
//               P = 2^(c S - m) -> bf16 pairs over their own consumed S
//               columns; lazy O rescale of their half of hd once PV(j-1) is
//               done; at the end O / l and lse out.
// TMEM: S buffers [0,128), [128,256), O [256,256+hd), Q [384,384+hd/2).
constexpr int kFwd1Threads = 320;
// which key pairs of every 8 keys take exp2_fma2 (bits 0, 2, 4, 6)
#ifndef TESS_ATTN_FWD1_POLY
#define TESS_ATTN_FWD1_POLY 0
#endif
constexpr int kFwd1PolyMask = TESS_ATTN_FWD1_POLY;

struct Fwd1Params {
  CUtensorMap tm_qkv;  // qkv view [3*H*hd, S, samples], box {64, 128}
  int S, H, n_qt, n_kt;
  int units;  // samples * H * n_qt
  float c;    // scale * log2(e)
  __nv_bfloat16* o;
  long long ld_o;
  float* lse;
};

template <int HD>
struct Fwd1Cfg {
  static constexpr int TILE = 128 * HD * 2;
  static constexpr int K_STAGES = 3, V_STAGES = 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = TILE;
  static constexpr int OFF_V = OFF_K + K_STAGES * TILE;
  static constexpr int OFF_BAR = OFF_V + V_STAGES * TILE;
  static constexpr int OFF_RED = OFF_BAR + 256;  // row maxima (2 steps) and row sums, 2 groups x 128 fp32 each
  static constexpr int USED = OFF_RED + 3072;
  static constexpr int SMEM_BYTES = USED + 1024 <= 232448 ? USED + 1024 : 232448;
  static constexpr int TMEM_COLS = 512;
  static constexpr int TM_S = 0, TM_O = 256, TM_Q = 384;
};

template <int HD>
__global__ void __launch_bounds__(kFwd1Threads, 1) attn_fwd1_kernel(const __grid_constant__ Fwd1Params p) {
  using C = Fwd1Cfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((smem - smem_raw) + C::USED > C::SMEM_BYTES) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;                  // Q of the unit in shared memory
  uint64_t* q_tmem = bars + 1;                  // ... copied into TMEM (8 warps)
  uint64_t* k_full = bars + 2;                  // K_STAGES
  uint64_t* k_empty = k_full + C::K_STAGES;     // K_STAGES
  uint64_t* v_full = k_empty + C::K_STAGES;     // V_STAGES
  uint64_t* v_empty = v_full + C::V_STAGES;     // V_STAGES
  uint64_t* s_full = v_empty + C::V_STAGES;     // 2: S in buffer b
  uint64_t* p_full = s_full + 2;                // P(j) in TMEM (8 warps)
  uint64_t* pv_done = p_full + 1;               // O += P(j) V_j complete
  uint64_t* fin = pv_done + 1;                  // O of the unit complete
  uint64_t* acc_free = fin + 1;                 // O read out of TMEM (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n = p.n_kt;
  const int units = p.units;  // (sample * H + head) * n_qt + query tile

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_tmem, 8);
    for (int s = 0; s < C::K_STAGES; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::V_STAGES; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(p_full, 8);
    mbar_init(pv_done, 1);
    mbar_init(fin, 1);
    mbar_init(acc_free, 8);
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
      int gk = 0, round = 0;  // key steps over all units, units of this CTA
      for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
        const int job = unit / p.n_qt, q0 = (unit % p.n_qt) * 128;
        const int head = job % p.H, smp = job / p.H;
        const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;
        if (round > 0) mbar_wait(q_tmem, (round - 1) & 1);  // Q slot free
        mbar_expect_tx(q_full, C::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c)
          tma_load_3d(smem + C::OFF_Q + c * 16384, &p.tm_qkv, q_full, col_q + c * 64, q0, smp);
        for (int j = 0; j < n; ++j, ++gk) {
          const int ks = gk % C::K_STAGES, ku = gk / C::K_STAGES;
          if (ku > 0) mbar_wait(&k_empty[ks], (ku - 1) & 1);
          mbar_expect_tx(&k_full[ks], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_K + ks * C::TILE + c * 16384, &p.tm_qkv, &k_full[ks],
                        col_k + c * 64, j * 128, smp);
          const int vs = gk % C::V_STAGES, vu = gk / C::V_STAGES;
          if (vu > 0) mbar_wait(&v_empty[vs], (vu - 1) & 1);
          mbar_expect_tx(&v_full[vs], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_V + vs * C::TILE + c * 16384, &p.tm_qkv, &v_full[vs],
                        col_v + c * 64, j * 128, smp);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);  // S: B = K K-major
    constexpr uint32_t idesc_pv = idesc_bf16(128, HD, false, true);   // O: B = V MN-major
    const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint64_t kmaj_k = make_sdesc(sbase + C::OFF_K, 16, 1024);
    const uint64_t mn_v = make_sdesc(sbase + C::OFF_V, 16384, 1024);
    constexpr uint64_t kTile = (uint64_t)(C::TILE >> 4);
    auto kmaj_off = [](int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); };
    auto issue_s = [&](int g2) {  // S(g2) = Q K^T into buffer g2 & 1
      mbar_wait(&k_full[g2 % C::K_STAGES], (g2 / C::K_STAGES) & 1);
      tc_fence_after();
      const uint32_t d = tm + C::TM_S + (uint32_t)(g2 & 1) * 128u;
      const uint64_t b = kmaj_k + (g2 % C::K_STAGES) * kTile;
      if constexpr (HD == 128) {
        mma_k128_ts_k(d, tm + C::TM_Q, b, idesc_s, 0u);
      } else {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_ts_warp(d, tm + C::TM_Q + 8 * kk, b + kmaj_off(kk), idesc_s, kk > 0 ? 1u : 0u);
      }
      mma_commit_warp(&s_full[g2 & 1]);
      mma_commit_warp(&k_empty[g2 % C::K_STAGES]);
    };
    // n >= 2: the score stream runs across units -- the next unit's S(0),
    // S(1) follow PV(n-2), PV(n-1) of this one, so they overlap its last
    // softmax step and the O read-out
    const bool xu = n >= 2;
    int gk = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
      const bool has_next = unit + (int)gridDim.x < units;
      if (!xu || round == 0) {
        mbar_wait(q_tmem, round & 1);
        tc_fence_after();
        issue_s(gk);
        if (n > 1) issue_s(gk + 1);
      }
      for (int j = 0; j < n; ++j, ++gk) {
        // O (+)= P(j) V_j; P of keys [16kk, 16kk+16) at column 64(kk/4) +
        // 8(kk%4) of the S buffer
        mbar_wait(p_full, gk & 1);
        if (j == 0 && round > 0) mbar_wait(acc_free, (round - 1) & 1);  // previous O out
        mbar_wait(&v_full[gk % C::V_STAGES], (gk / C::V_STAGES) & 1);
        tc_fence_after();
        mma_k128_ts_n_quads(tm + C::TM_O, tm + C::TM_S + (uint32_t)(gk & 1) * 128u,
                            mn_v + (gk % C::V_STAGES) * kTile, idesc_pv, j > 0 ? 1u : 0u);
        mma_commit_warp(pv_done);
        mma_commit_warp(&v_empty[gk % C::V_STAGES]);
        if (j == n - 1) mma_commit_warp(fin);  // ahead of the next unit's S(1)
        // S two steps ahead over P(j), in order behind its reader
        if (j + 2 < n) {
          issue_s(gk + 2);
        } else if (xu && has_next) {
          if (j + 2 == n) {  // the next unit's Q in TMEM (copied once S(n-1) was read)
            mbar_wait(q_tmem, (round + 1) & 1);
            tc_fence_after();
          }
          issue_s(gk + 2);
        }
      }
    }
  } else {
    // --------------------------------------------------- softmax warps
    const int quad = warp & 3;
    const int g = (warp - 2) >> 2;   // keys [64g, 64g+64) of each key tile
    const int r = quad * 32 + lane;  // query row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float cl2 = p.c;
    constexpr int HW = HD / 2;  // hd columns per group
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED);
    const bool xu = n >= 2;  // Q of the next unit copied during this one's last step
    int gk = 0, round = 0;
    for (int unit = blockIdx.x; unit < units; unit += gridDim.x, ++round) {
      const int job = unit / p.n_qt, q0 = (unit % p.n_qt) * 128;
      const int head = job % p.H, smp = job / p.H;
      const int qrow = q0 + r;
      const bool has_next = unit + (int)gridDim.x < units;
      // the Q row of unit round `rr` into TMEM (A operand of S): group g
      // copies its half of hd (16-byte pieces of the SW128 tile). Called once
      // every score MMA of the previous unit is complete.
      auto copy_q = [&](int rr) {
        mbar_wait(q_full, rr & 1);
        const uint32_t base = smem_u32(smem + C::OFF_Q);
        uint32_t v[HW / 2];
#pragma unroll
        for (int u = 0; u < HW / 8; ++u) {
          const int col = g * HW + 8 * u;
          const uint32_t a = base + (uint32_t)(col >> 6) * 16384u + (uint32_t)(r >> 3) * 1024u +
                             (uint32_t)(r & 7) * 128u + (uint32_t)((((col & 63) >> 3) ^ (r & 7)) << 4);
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v[4 * u]), "=r"(v[4 * u + 1]), "=r"(v[4 * u + 2]), "=r"(v[4 * u + 3])
                       : "r"(a));
        }
        const uint32_t t = tmem + lane_off + C::TM_Q + g * (HW / 2);
        if constexpr (HW / 2 == 32) {
          tmem_st32(t, *reinterpret_cast<const uint32_t(*)[32]>(v));
        } else {
          tmem_st16(t, *reinterpret_cast<const uint32_t(*)[16]>(v));
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(q_tmem);
      };
      if (!xu || round == 0) copy_q(round);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j, ++gk) {
        const int b = gk & 1;
        mbar_wait(&s_full[b], (gk >> 1) & 1);
        tc_fence_after();
        const uint32_t t_s = tmem + lane_off + C::TM_S + b * 128 + g * 64;
        float s[64];
        {
          uint32_t a0[32], a1[32];
          tmem_ld32_nowait(t_s, a0);
          tmem_ld32_nowait(t_s + 32, a1);
          tmem_wait_ld();
          reg_fence32(a0);
          reg_fence32(a1);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            s[e] = __uint_as_float(a0[e]);
            s[32 + e] = __uint_as_float(a1[e]);
          }
        }
        // the unit's last scores are in: its Q columns are free for the next
        if (xu && j == n - 1 && has_next) copy_q(round + 1);
        const int nvalid = p.S - j * 128 - g * 64;  // keys of this group inside the sequence
        if (nvalid < 64) {
#pragma unroll
          for (int e = 0; e < 64; ++e)
            if (e >= nvalid) s[e] = -INFINITY;
        }
        float mp[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mp[k] = max3f(s[k], s[8 + k], s[16 + k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) mp[k] = max3f(mp[k], s[24 + k], s[32 + k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) mp[k] = max3f(mp[k], s[40 + k], s[48 + k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) mp[k] = fmaxf(mp[k], s[56 + k]);
        const float mg = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                               fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
        // the row's maximum over both groups (same value, same order in both)
        float* rb = red + (gk & 1) * 256;
        rb[g * 128 + r] = mg;
        named_bar_sync(1 + quad, 64);
        const float mx = fmaxf(rb[r], rb[128 + r]);
        const float m_new = fmaxf(m_used, mx * cl2);
        const bool need = m_new > m_used + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          // lazy rescale (same decision in both groups: same rows, same maxima)
          const float f = ex2_approx(m_used - m_new);  // 0 on the first tile
          if (j > 0) {
            l *= f;
            mbar_wait(pv_done, (gk - 1) & 1);  // O += P(j-1) V_{j-1} complete
            tc_fence_after();
            const uint32_t t_o = tmem + lane_off + C::TM_O + g * HW;
#pragma unroll 1
            for (int c = 0; c < HW / 16; ++c) {
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
        float2 rp[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        const float2 c2 = make_float2(cl2, cl2), nm2 = make_float2(-m_used, -m_used);
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 64; e += 2) {
          const float2 xv = fma2(make_float2(s[e], s[e + 1]), c2, nm2);
          const float2 pv = (kFwd1PolyMask >> (e & 7)) & 1 ? exp2_fma2(xv)
                                                           : make_float2(ex2_approx(xv.x), ex2_approx(xv.y));
          rp[(e >> 1) & 3] = add2(rp[(e >> 1) & 3], pv);
          pk[e >> 1] = pack_bf16x2(pv.x, pv.y);
        }
        l += ((rp[0].x + rp[0].y) + (rp[1].x + rp[1].y)) + ((rp[2].x + rp[2].y) + (rp[3].x + rp[3].y));
        // P (bf16 pairs, lower key in the low half) over the consumed S columns
        tmem_st32(t_s, pk);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
      }
      // ---------------------------------------------- O of the unit out
      float* rl = red + 512;  // after the two max buffers
      rl[g * 128 + r] = l;
      named_bar_sync(1 + quad, 64);
      const float lt = rl[r] + rl[128 + r];
      mbar_wait(fin, round & 1);
      tc_fence_after();
      const float inv = 1.0f / lt;
      __nv_bfloat16* orow = p.o + ((long long)smp * p.S + qrow) * p.ld_o + (long long)head * HD + g * HW;
      uint32_t ov[HW];  // the row's O half: all loads in flight, one wait
#pragma unroll
      for (int c = 0; c < HW / 32; ++c)
        tmem_ld32_nowait(tmem + lane_off + C::TM_O + g * HW + c * 32,
                         *reinterpret_cast<uint32_t(*)[32]>(ov + c * 32));
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < HW / 32; ++c) reg_fence32(*reinterpret_cast<uint32_t(*)[32]>(ov + c * 32));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_free);  // the next unit's first PV may start
      if (qrow < p.S) {
#pragma unroll
        for (int u = 0; u < HW / 8; ++u) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(ov[u * 8 + 0]) * inv, __uint_as_float(ov[u * 8 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(ov[u * 8 + 2]) * inv, __uint_as_float(ov[u * 8 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(ov[u * 8 + 4]) * inv, __uint_as_float(ov[u * 8 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(ov[u * 8 + 6]) * inv, __uint_as_float(ov[u * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + u * 8) = w;
        }
      }
      if (g == 0 && qrow < p.S) p.lse[(long long)job * p.S + qrow] = m_used + __log2f(lt);
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


template <int HD>
cudaError_t launch_fwd1(const Fwd1Params& p, int grid, cudaStream_t s) {
  using C = Fwd1Cfg<HD>;
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_fwd1_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_fwd1_kernel<HD><<<grid, kFwd1Threads, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

}  // namespace attn
}  // namespace sm100

cudaError_t attn_fwd1_sm100(const AttnDesc& d, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d)) {
    g_attn_err = "attn_fwd_sm100: unsupported shape (head_dim must be 64 or 128, rows 16-byte aligned)";
    return cudaErrorInvalidValue;
  }
  Fwd1Params p;
  std::memset(&p, 0, sizeof(p));
  if (!encode_3d(&p.tm_qkv, d.qkv, 3 * d.heads * d.head_dim, d.seq, d.samples, d.ld_qkv, 128))
    return cudaErrorInvalidValue;
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.n_qt = p.n_kt = (int)((d.seq + 127) / 128);
  const long long units = (long long)p.n_qt * d.heads * d.samples;
  if (units > 0x7fffffffLL) {
    g_attn_err = "attn_fwd_sm100: too many units";
    return cudaErrorInvalidValue;
  }
  p.units = (int)units;
  p.c = d.scale * kLog2e;
  p.o = static_cast<__nv_bfloat16*>(d.o);
  p.ld_o = d.ld_o;
  p.lse = d.lse;
  const int grid = (int)std::min<long long>(units, device_sms());
  cudaError_t e = d.head_dim == 128 ? launch_fwd1<128>(p, grid, s) : launch_fwd1<64>(p, grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_fwd_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace tess

static_assert(tess::sm100::attn::Fwd1Cfg<128>::USED <= 232448, "attn fwd1 smem");
