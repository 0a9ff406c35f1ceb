// EXPERIMENT (not part of libtess): the attention backward with dQ fused
// into the key-tile kernel, kept to reproduce the round-2 measurements in
// profiles/r2_attn_bwd_dq_fused_*.log / r2_attn_bwd_modes_ab.log (DESIGN.md
// section 3). Compiled only into tools/attn_check, in one translation unit
// with the product kernels (it reuses their helpers).
//
// Result: slower than the round-1 split path (attn_bwd_kernel + one batched
// dQ GEMM over dS^T, 2.49 ms at the cfg4 head shape on an unconstrained
// B200; the kernel is kept below as the harness's baseline): fused dQ 3.2-3.3 ms, of which ~1 ms is the ordered fp32 exchange of
// dQ partials through L2 (64 KB per key tile and query tile, 6.4 GB per
// call, twice the dS^T bytes) and ~0.65 ms the fifth MMA serialised behind
// the TMEM drain (TMEM holds S^T, dP^T, dV, dK: dQ must reuse dP^T's
// columns). Without any dS output the restructured kernel (8 softmax warps,
// P^T first into its own consumed columns, warp-wide MMA issue with
// precomputed descriptors) runs dK/dV in 1.50 ms (mode 2); writing dS^T
// back costs 0.35-1.0 ms in every form tried (TMA store per group or per
// warp, st.global from registers), which puts mode 3 + the dQ GEMM back at
// the split path's time.
#pragma once

#include "../kernels/attention_sm100.cu"

namespace tess {

// Geometry of the fused-dQ backward: n = key tiles = query tiles per
// (sample, head); `gangs` groups of n co-resident CTAs (gangs * n <= #SMs).
struct AttnBwdPlan {
  bool ok = false;
  int n = 0, gangs = 0;
  size_t acc_bytes = 0, sem_bytes = 0;
};

// Extra operands of the experiment (AttnDesc has none of them).
struct AttnBwdDqArgs {
  float* dq_acc = nullptr;     // fp32 accumulator, plan.acc_bytes
  uint32_t* dq_sem = nullptr;  // ordering counters, plan.sem_bytes (zeroed by the launch)
  void* dst = nullptr;         // mode 3: dS^T [samples*H][S keys][S queries] bf16
};
// The round-1 split backward: dK, dV into dqkv, unscaled dS^T into dst.
cudaError_t attn_bwd_split_sm100(const AttnDesc& d, void* dst, cudaStream_t s);

namespace sm100 {
namespace attn {

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

// ------------------------------------------- the round-1 split backward
// (shipped until round 2; the harness's baseline) dK, dV and dS^T to HBM,
// dQ by a batched GEMM over dS^T.
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
constexpr int kBwdThreads = 576;  // TMA + MMA warps + 16 softmax-gradient warps
constexpr int BQB = 128;  // queries per backward tile
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

// ------------------------------------------ backward with dQ fused (gangs)
// The same per-(key tile) work as attn_bwd_kernel plus dQ(i) = dS(i) K as a
// fifth MMA per query tile, so dS never leaves the SM. The dQ partials of the
// n key tiles of a (sample, head) are summed in a FIXED order (bitwise
// deterministic, no atomics): the n CTAs of one "gang" run the same
// (sample, head) jobs side by side, CTA j walking the query tiles in the
// rotated order i = (j + t) mod n. Query tile i therefore receives its
// contributions at steps t = 0, 1, ..., n-1 (CTAs i, i-1, ..., i+1), each one
// step after the previous, and a per-(gang, tile) counter orders them:
//   t = 0      TMA bulk store of the fp32 partial into the gang's
//              accumulator (tile-sized, L2 resident, reused across jobs),
//   0<t<n-1    TMA bulk fp32 reduce-add into it (the add runs in L2),
//   t = n-1    the last contributor loads the sum of the others, adds its
//              own partial, scales by 1/sqrt(hd) and stores dQ in bf16.
// Each step waits for the counter to reach (job round * n + t) and releases
// +1; a CTA waits only on its successor's previous step, which all
// co-resident gang members reach in lockstep. Grid = gangs * n <= #SMs (one
// CTA per SM), so every gang's members are resident together.
//
// 16 warps (512 threads):
//   warp 0      TMA: K, V per job; Q_i (+ its lse and delta rows) into a
//               2-slot ring, dO_i into one slot.
//   warp 1      MMA issuer + TMEM owner; per step, all M=128 (full rate):
//                 dV += P^T(i) dO_i          (A = P^T in TMEM)
//                 dP^T(i) = V dO_i^T         (after dQ(i-1) left TMEM)
//                 S^T(i+1) = K Q_{i+1}^T     (over the consumed P^T)
//                 dK += dS^T(i) Q_i          (A = dS^T in shared memory)
//                 dQ(i) = dS(i) K            (A = the same dS^T bytes read
//                                             MN-major; into the dP^T columns)
//   warps 4-7   dQ drain: TMEM -> registers (frees the columns at once),
//               then the ordered accumulation above through a 2 x 16 KB
//               staging buffer.
//   warps 8-15  softmax gradient, thread = key row, group g = queries
//               [64g, 64g+64): P^T = 2^(c S^T - lse) written as bf16 pairs
//               over its own consumed S^T columns (no cross-warp barrier),
//               then dS^T = P^T (dP^T - delta) -> shared memory; after the
//               last step of a job, dK and dV out of TMEM to HBM.
// TMEM: S^T / P^T [0,128), dP^T / dQ [128,256), dV [256,256+hd), dK [384,384+hd).
constexpr int kBwd2Threads = 512;
// per-thread registers by role (setmaxnreg): 128 x ctl + 128 x drain + 256 x
// softmax <= 64 K
#ifndef TESS_BWD2_REG_CTL
#define TESS_BWD2_REG_CTL 80
#define TESS_BWD2_REG_DRAIN 168
#define TESS_BWD2_REG_SOFTMAX 128
#endif
constexpr int kBwd2RegCtl = TESS_BWD2_REG_CTL, kBwd2RegDrain = TESS_BWD2_REG_DRAIN,
              kBwd2RegSoftmax = TESS_BWD2_REG_SOFTMAX;
static_assert(128 * kBwd2RegCtl + 128 * kBwd2RegDrain + 256 * kBwd2RegSoftmax <= 65536, "register pool");

struct Bwd2Params {
  CUtensorMap tm_kv;   // qkv view [3*H*hd, S, samples], box {64, 128}: K, V, Q tiles
  CUtensorMap tm_do;   // dO view [H*hd, S, samples], box {64, 128}
  CUtensorMap tm_lse;  // lse [S, samples*H] fp32, box {128, 1} (rows past S read 0)
  CUtensorMap tm_dlt;  // delta, same view
  int S, H, n, jobs, n_gangs;
  float c;      // scale * log2(e)
  float scale;  // 1/sqrt(hd)
  __nv_bfloat16* dqkv;
  long long ld_qkv;
  float* dq_acc;     // [gangs * n tiles][hd/32 chunks][128 rows x 32] fp32, rows swizzled
  uint32_t* dq_sem;  // [gangs * n], zero at launch
  __nv_bfloat16* dst;  // mode 3: dS^T [samples*H][S keys][S queries]
  long long* trace;  // debug (TESS_ATTN_TRACE): [event][warp][step] clock64, CTA 0, job 0
};

enum {
  T2_DV = 0, T2_DP = 1, T2_S = 2, T2_DK = 3, T2_DQ = 4,          // MMA issue times
  T2_SM_S = 5, T2_SM_P = 6, T2_SM_DP = 7, T2_SM_DS = 8,          // softmax warps
  T2_DR_IN = 9, T2_DR_FREE = 10, T2_DR_SEM = 11, T2_DR_DONE = 12,  // drain warps
  T2_N = 13
};
__device__ __forceinline__ void trace2(const Bwd2Params& p, int ev, int warp, int step) {
  if (p.trace && blockIdx.x == 0 && step < 16) p.trace[(ev * 16 + warp) * 16 + step] = clock64();
}

template <int HD>
struct Bwd2Cfg {
  static constexpr int TILE = 128 * HD * 2;      // K, V, Q_i or dO_i (bf16, 64-col SW128 chunks)
  static constexpr int NCH = HD / 32;            // dQ fp32 chunks of 32 columns
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;         // 2 slots
  static constexpr int OFF_DO = 4 * TILE;        // 1 slot
  static constexpr int OFF_DS = 5 * TILE;        // dS^T: 128 keys x 128 queries, 2 x 16 KB chunks
  static constexpr int OFF_STG = OFF_DS + 32768; // dQ staging, 2 x 16 KB
  static constexpr int OFF_LD = OFF_STG + 32768; // per Q slot: lse[128] | delta[128]
  static constexpr int OFF_BAR = OFF_LD + 2 * 1024;
  static constexpr int USED = OFF_BAR + 256;
  static constexpr int SMEM_BYTES = USED + 1024 <= 232448 ? USED + 1024 : 232448;
  static constexpr int TMEM_COLS = 512;
  static constexpr int TM_S = 0, TM_DP = 128, TM_DV = 256, TM_DK = 384;
};

__device__ __forceinline__ void sem_wait(const uint32_t* s, uint32_t target) {
  while ((int)(ld_relaxed_u32(s) - target) < 0) __nanosleep(20);
  (void)ld_acquire_u32(s);
}

// MODE: 0 = dQ fused (the product); 1 = dQ MMA but no global accumulation
// (timing only); 2 = no dQ, dS^T not stored (timing only); 3 = no dQ, dS^T
// TMA-stored for the batched dQ GEMM (the split path). Modes 2/3 issue
// dP^T(i+1) as soon as dP^T(i) sits in registers (no dQ in its columns) and
// keep dO in two slots (the dQ staging space).
template <int HD, int MODE>
__global__ void __launch_bounds__(kBwd2Threads, 1) attn_bwd_dq_kernel(const __grid_constant__ Bwd2Params p) {
  using C = Bwd2Cfg<HD>;
  constexpr bool kDq = MODE < 2;
  // without the drain's 128 dQ registers the softmax keeps dP^T(i) whole
  constexpr int kRegDrain = kDq ? kBwd2RegDrain : 56;
  constexpr int kRegSoftmax = kDq ? kBwd2RegSoftmax : 168;
  static_assert(128 * kBwd2RegCtl + 128 * kRegDrain + 256 * kRegSoftmax <= 65536, "register pool");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if ((smem - smem_raw) + C::USED > C::SMEM_BYTES) __trap();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* q_full = bars + 2;    // 2
  uint64_t* q_empty = bars + 4;   // 2
  uint64_t* do_full = bars + 6;   // kDoSlots
  uint64_t* do_empty = bars + 8;  // kDoSlots
  uint64_t* s_full = bars + 10;   // S^T(i) in TMEM
  uint64_t* p_full = bars + 11;   // P^T(i) in TMEM (8 softmax warps)
  uint64_t* dp_full = bars + 12;  // dP^T(i) in TMEM
  uint64_t* ds_full = bars + 13;  // dS^T(i) in smem, dP^T(i) read (8 warps)
  uint64_t* ds_free = bars + 14;  // dK(i) (and dQ(i)) done reading dS^T
  uint64_t* dq_full = bars + 15;  // dQ(i) in TMEM
  uint64_t* dq_free = bars + 16;  // dQ(i) read out of TMEM (4 drain warps)
  uint64_t* fin = bars + 17;      // dK, dV of the job complete
  uint64_t* acc_free = bars + 18; // dK, dV read out of TMEM (8 softmax warps)
  uint64_t* dp_loaded = bars + 19;  // modes 2/3: dP^T(i) in registers (8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n = p.n;
  const int gang = blockIdx.x / n;
  const int j = blockIdx.x % n;  // key tile
  const int k0 = j * 128;
  auto do_off = [](int s) { return s == 0 ? C::OFF_DO : C::OFF_STG; };

  if (warp == 0 && lane == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
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
    mbar_init(ds_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(fin, 1);
    mbar_init(acc_free, 8);
    mbar_init(dp_loaded, 8);
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

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kBwd2RegCtl));
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------ TMA producer
      int gs = 0, round = 0;
      for (int job = gang; job < p.jobs; job += p.n_gangs, ++round) {
        const int smp = job / p.H, head = job % p.H;
        const int col_q = head * 3 * HD, col_k = col_q + HD, col_v = col_q + 2 * HD;
        if (round > 0) mbar_wait(kv_empty, (round - 1) & 1);
        mbar_expect_tx(kv_full, 2 * C::TILE);
#pragma unroll
        for (int c = 0; c < HD / 64; ++c) {
          tma_load_3d(smem + C::OFF_K + c * 16384, &p.tm_kv, kv_full, col_k + c * 64, k0, smp);
          tma_load_3d(smem + C::OFF_V + c * 16384, &p.tm_kv, kv_full, col_v + c * 64, k0, smp);
        }
        for (int t = 0; t < n; ++t, ++gs) {
          const int tile = (j + t) % n;
          const int qs = gs & 1, u = gs >> 1;
          if (u > 0) mbar_wait(&q_empty[qs], (u - 1) & 1);
          mbar_expect_tx(&q_full[qs], C::TILE + 1024);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + C::OFF_Q + qs * C::TILE + c * 16384, &p.tm_kv, &q_full[qs],
                        col_q + c * 64, tile * 128, smp);
          tma_load_2d(smem + C::OFF_LD + qs * 1024, &p.tm_lse, &q_full[qs], tile * 128, job);
          tma_load_2d(smem + C::OFF_LD + qs * 1024 + 512, &p.tm_dlt, &q_full[qs], tile * 128, job);
          const int ds_ = kDq ? 0 : (gs & 1), du = kDq ? gs : (gs >> 1);
          if (du > 0) mbar_wait(&do_empty[ds_], (du - 1) & 1);
          mbar_expect_tx(&do_full[ds_], C::TILE);
#pragma unroll
          for (int c = 0; c < HD / 64; ++c)
            tma_load_3d(smem + do_off(ds_) + c * 16384, &p.tm_do, &do_full[ds_],
                        head * HD + c * 64, tile * 128, smp);
        }
      }
    } else if (warp == 1) {
      // ------------------------------------------------------- MMA issuer
      // Warp-wide (one elected lane issues) with descriptors built once from
      // warp-uniform bases: each MMA is a constant add on the uniform
      // datapath, so the issuer keeps up although it shares its SM
      // sub-partition with two busy softmax warps.
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idesc_g = idesc_bf16(128, HD, false, true);    // dV, dK
      constexpr uint32_t idesc_q = idesc_bf16(128, HD, true, true);     // dQ
      const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      // K-major SW128 (S^T, dP^T operands; dS^T as dK's A): +kk -> chunk kk/4, 32 B
      const uint64_t kmaj_k = make_sdesc(sbase + C::OFF_K, 16, 1024);
      const uint64_t kmaj_v = make_sdesc(sbase + C::OFF_V, 16, 1024);
      const uint64_t kmaj_q0 = make_sdesc(sbase + C::OFF_Q, 16, 1024);
      const uint64_t kmaj_ds = make_sdesc(sbase + C::OFF_DS, 16, 1024);
      // MN-major SW128 (dO / Q as B of dV / dK; dS^T, K as dQ's A, B): +kk -> 2 KB
      const uint64_t mn_q0 = make_sdesc(sbase + C::OFF_Q, 16384, 1024);
      const uint64_t mn_do0 = make_sdesc(sbase + C::OFF_DO, 16384, 1024);
      const uint64_t mn_do1 = make_sdesc(sbase + C::OFF_STG, 16384, 1024);
      const uint64_t mn_ds = make_sdesc(sbase + C::OFF_DS, 16384, 1024);
      const uint64_t mn_k = make_sdesc(sbase + C::OFF_K, 16384, 1024);
      constexpr uint64_t kTileStep = (uint64_t)(C::TILE >> 4);
      auto kmaj_off = [](int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); };
      auto issue_scores = [&](uint32_t d, uint64_t a, uint64_t b) {
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_bf16_warp(d, a + kmaj_off(kk), b + kmaj_off(kk), idesc_s, kk > 0 ? 1u : 0u);
      };
      auto wait_do = [&](int g2) {  // dO of global step g2 -> its MN-major descriptor
        const int s = kDq ? 0 : (g2 & 1), u = kDq ? g2 : (g2 >> 1);
        mbar_wait(&do_full[s], u & 1);
        return s == 0 ? mn_do0 : mn_do1;
      };
      auto kmaj_do = [&](uint64_t mn) {  // same tile, K-major view
        return mn == mn_do0 ? make_sdesc(sbase + C::OFF_DO, 16, 1024)
                            : make_sdesc(sbase + C::OFF_STG, 16, 1024);
      };
      const uint64_t kmaj_do0 = make_sdesc(sbase + C::OFF_DO, 16, 1024);
      const uint64_t kmaj_do1 = make_sdesc(sbase + C::OFF_STG, 16, 1024);
      (void)kmaj_do;
      int gs = 0, round = 0;
      for (int job = gang; job < p.jobs; job += p.n_gangs, ++round) {
        mbar_wait(kv_full, round & 1);
        tc_fence_after();
        mbar_wait(&q_full[gs & 1], (gs >> 1) & 1);
        tc_fence_after();
        if (lane == 0) trace2(p, T2_S, 1, 0);
        issue_scores(tm + C::TM_S, kmaj_k, kmaj_q0 + (gs & 1) * kTileStep);
        mma_commit_warp(s_full);
        if (!kDq) {
          // dP^T(0); later dP^T(i+1) goes out while tile i is being finished
          if (gs > 0) mbar_wait(dp_loaded, (gs - 1) & 1);
          const uint64_t mdo = wait_do(gs);
          tc_fence_after();
          if (lane == 0) trace2(p, T2_DP, 1, 0);
          issue_scores(tm + C::TM_DP, kmaj_v, mdo == mn_do0 ? kmaj_do0 : kmaj_do1);
          mma_commit_warp(dp_full);
        }
        for (int t = 0; t < n; ++t, ++gs) {
          const bool last = t + 1 == n;
          const int qs = gs & 1;
          // dV += P^T(i) dO_i
          mbar_wait(p_full, gs & 1);
          const uint64_t mdo = wait_do(gs);
          if (t == 0 && round > 0) mbar_wait(acc_free, (round - 1) & 1);
          tc_fence_after();
          if (lane == 0) trace2(p, T2_DV, 1, t);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // P^T of queries [16kk, 16kk+16): cols 32(kk/2) + 8(kk%2)
            mma_bf16_ts_warp(tm + C::TM_DV, tm + C::TM_S + 32 * (kk >> 1) + 8 * (kk & 1),
                             mdo + (uint64_t)kk * 128u, idesc_g, (t > 0 || kk > 0) ? 1u : 0u);
          if (kDq) {
            // dP^T(i) into the dP^T / dQ columns once dQ(i-1) is out of TMEM
            if (gs > 0) {
              mbar_wait(dq_free, (gs - 1) & 1);
              tc_fence_after();
            }
            if (lane == 0) trace2(p, T2_DP, 1, t);
            issue_scores(tm + C::TM_DP, kmaj_v, kmaj_do0);
            mma_commit_warp(dp_full);
            mma_commit_warp(&do_empty[0]);
          } else {
            mma_commit_warp(&do_empty[gs & 1]);
          }
          // S^T(i+1) over P^T(i) (in order behind dV)
          if (!last) {
            mbar_wait(&q_full[qs ^ 1], ((gs + 1) >> 1) & 1);
            tc_fence_after();
            if (lane == 0) trace2(p, T2_S, 1, t + 1);
            issue_scores(tm + C::TM_S, kmaj_k, kmaj_q0 + (qs ^ 1) * kTileStep);
            mma_commit_warp(s_full);
            if (!kDq) {
              // dP^T(i+1) once tile i's dP^T is in registers
              mbar_wait(dp_loaded, gs & 1);
              const uint64_t mdn = wait_do(gs + 1);
              tc_fence_after();
              if (lane == 0) trace2(p, T2_DP, 1, t + 1);
              issue_scores(tm + C::TM_DP, kmaj_v, mdn == mn_do0 ? kmaj_do0 : kmaj_do1);
              mma_commit_warp(dp_full);
            }
          }
          // dK += dS^T(i) Q_i (, dQ(i) = dS(i) K)
          mbar_wait(ds_full, gs & 1);
          tc_fence_after();
          if (lane == 0) trace2(p, T2_DK, 1, t);
          const uint64_t mq = mn_q0 + qs * kTileStep;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16_warp(tm + C::TM_DK, kmaj_ds + kmaj_off(kk), mq + (uint64_t)kk * 128u, idesc_g,
                          (t > 0 || kk > 0) ? 1u : 0u);
          mma_commit_warp(&q_empty[qs]);
          if (kDq) {
            if (lane == 0) trace2(p, T2_DQ, 1, t);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // K = keys: 16 key rows of dS^T / K per step
              mma_bf16_warp(tm + C::TM_DP, mn_ds + (uint64_t)kk * 128u, mn_k + (uint64_t)kk * 128u,
                            idesc_q, kk > 0 ? 1u : 0u);
            mma_commit_warp(dq_full);
          }
          mma_commit_warp(ds_free);
          if (last) {
            mma_commit_warp(kv_empty);
            mma_commit_warp(fin);
          }
        }
      }
    }
  } else if (warp < 8) {
    if constexpr (kDq)
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegDrain));
    else
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegDrain));
    if (kDq) {
    // ----------------------------------------------------------- dQ drain
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // query row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const bool issuer = warp == 4 && lane == 0;
    const uint32_t stg = smem_u32(smem + C::OFF_STG);
    const float scale = p.scale;
    int gs = 0, round = 0;
    for (int job = gang; job < p.jobs; job += p.n_gangs, ++round) {
      const int smp = job / p.H, head = job % p.H;
      for (int t = 0; t < n; ++t, ++gs) {
        const int tile = (j + t) % n;
        mbar_wait(dq_full, gs & 1);
        tc_fence_after();
        if (lane == 0) trace2(p, T2_DR_IN, warp, t);
        uint32_t v[C::NCH][32];
#pragma unroll
        for (int c = 0; c < C::NCH; ++c) tmem_ld32_nowait(tmem + lane_off + C::TM_DP + c * 32, v[c]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < C::NCH; ++c) reg_fence32(v[c]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(dq_free);
          trace2(p, T2_DR_FREE, warp, t);
        }
        if (MODE == 1) continue;
        uint32_t* sem = p.dq_sem + (size_t)gang * n + tile;
        float* acc = p.dq_acc + ((size_t)gang * n + tile) * (C::NCH * 4096);
        const uint32_t target = (uint32_t)(round * n + t);
        if (t + 1 == n) {
          // last contributor: dQ = scale * (sum of the others + own partial)
          sem_wait(sem, target);
          if (issuer) trace2(p, T2_DR_SEM, warp, t);
          const int qrow = tile * 128 + r;
          __nv_bfloat16* drow =
              p.dqkv + ((long long)smp * p.S + qrow) * p.ld_qkv + (long long)head * 3 * HD;
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            float f[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(v[c][e]);
            if (n > 1) {
              const float* arow = acc + c * 4096 + r * 32;
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const float4 a = *reinterpret_cast<const float4*>(arow + ((u ^ (r & 7)) << 2));
                f[4 * u + 0] = a.x + f[4 * u + 0];
                f[4 * u + 1] = a.y + f[4 * u + 1];
                f[4 * u + 2] = a.z + f[4 * u + 2];
                f[4 * u + 3] = a.w + f[4 * u + 3];
              }
            }
            if (qrow < p.S) {
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                uint4 w;
                w.x = pack_bf16x2(f[8 * u + 0] * scale, f[8 * u + 1] * scale);
                w.y = pack_bf16x2(f[8 * u + 2] * scale, f[8 * u + 3] * scale);
                w.z = pack_bf16x2(f[8 * u + 4] * scale, f[8 * u + 5] * scale);
                w.w = pack_bf16x2(f[8 * u + 6] * scale, f[8 * u + 7] * scale);
                *reinterpret_cast<uint4*>(drow + c * 32 + u * 8) = w;
              }
            }
          }
          named_bar_sync(1, 128);  // all rows of the accumulator read
          if (issuer) {
            st_release_u32(sem, target + 1);
            trace2(p, T2_DR_DONE, warp, t);
          }
        } else {
#pragma unroll
          for (int c = 0; c < C::NCH; ++c) {
            const uint32_t buf = stg + (uint32_t)(c & 1) * 16384u;
            if (issuer && c >= 2) bulk_wait_read<1>();  // chunk c-2 has left buffer c&1
            named_bar_sync(1, 128);
            const uint32_t row = buf + (uint32_t)r * 128u;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              st_shared_v4(row + (uint32_t)((u ^ (r & 7)) << 4), v[c][4 * u], v[c][4 * u + 1],
                           v[c][4 * u + 2], v[c][4 * u + 3]);
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (issuer) {
              if (c == 0) {
                sem_wait(sem, target);
                fence_proxy_async_global();
                trace2(p, T2_DR_SEM, warp, t);
              }
              if (t == 0)
                bulk_store(acc + c * 4096, buf, 16384);
              else
                bulk_reduce_add_f32(acc + c * 4096, buf, 16384);
              bulk_commit();
            }
          }
          if (issuer) {
            bulk_wait_all();
            fence_proxy_async_global();
            st_release_u32(sem, target + 1);
            trace2(p, T2_DR_DONE, warp, t);
          }
        }
      }
    }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    // ------------------------------------------ softmax-gradient warps
    const int quad = warp & 3;
    const int g = (warp - 8) >> 2;   // queries [64g, 64g+64) of each tile
    const int r = quad * 32 + lane;  // key row within the tile (TMEM lane)
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float cl2 = p.c, scale = p.scale;
    const uint32_t ds_chunk = smem_u32(smem + C::OFF_DS) + (uint32_t)g * 16384u;
    int gs = 0, round = 0;
    for (int job = gang; job < p.jobs; job += p.n_gangs, ++round) {
      const int smp = job / p.H, head = job % p.H;
      for (int t = 0; t < n; ++t, ++gs) {
        const int qs = gs & 1;
        const int tile = (j + t) % n;
        const uint32_t ldw = smem_u32(smem + C::OFF_LD + qs * 1024) + (uint32_t)g * 256u;
        mbar_wait(&q_full[qs], (gs >> 1) & 1);  // lse, delta rows of the slot
        mbar_wait(s_full, gs & 1);
        tc_fence_after();
        if (lane == 0) trace2(p, T2_SM_S, warp, t);
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
          for (int u = 0; u < 4; ++u) {
            const int e = 4 * e4 + u;
            const float xv = fmaf(pr[e], cl2, -lv[u]);
            pr[e] = (kBwdPolyMask >> u) & 1 ? exp2_fma(xv) : ex2_approx(xv);
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
        if (lane == 0) {
          mbar_arrive(p_full);
          trace2(p, T2_SM_P, warp, t);
        }
        // ---- dS^T = P^T (dP^T - delta) -> shared memory (unscaled)
        mbar_wait(dp_full, gs & 1);
        tc_fence_after();
        if (lane == 0) trace2(p, T2_SM_DP, warp, t);
        uint32_t d[64];
        auto load_dp = [&](int h) {
          uint32_t (&dh)[32] = *reinterpret_cast<uint32_t(*)[32]>(d + 32 * h);
          tmem_ld32_nowait(tmem + lane_off + C::TM_DP + g * 64 + 32 * h, dh);
        };
        if (!kDq) {
          // modes 2/3: both halves now, so dP^T(i+1) can take the columns
          load_dp(0);
          load_dp(1);
          tmem_wait_ld();
          reg_fence32(*reinterpret_cast<uint32_t(*)[32]>(d));
          reg_fence32(*reinterpret_cast<uint32_t(*)[32]>(d + 32));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_loaded);
        }
        if (gs > 0) mbar_wait(ds_free, (gs - 1) & 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (kDq) {
            load_dp(h);
            tmem_wait_ld();
            reg_fence32(*reinterpret_cast<uint32_t(*)[32]>(d + 32 * h));
          }
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            float4 d4;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(d4.x), "=f"(d4.y), "=f"(d4.z), "=f"(d4.w)
                         : "r"(ldw + 512u + (uint32_t)(128 * h + 16 * e4)));
            const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int e = 32 * h + 4 * e4 + u;
              d[e] = __float_as_uint(pr[e] * (__uint_as_float(d[e]) - dv[u]));
            }
          }
          if (MODE == 3) {
            // dS^T row segment straight from registers to HBM as well (the
            // TMA unit stays free for the Q / dO loads)
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              pk[e] = pack_bf16x2(__uint_as_float(d[32 * h + 2 * e]), __uint_as_float(d[32 * h + 2 * e + 1]));
            const uint32_t row_base = ds_chunk + (uint32_t)(r >> 3) * 1024u + (uint32_t)(r & 7) * 128u;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              st_shared_v4(row_base + (uint32_t)(((4 * h + u) ^ (r & 7)) << 4), pk[4 * u], pk[4 * u + 1],
                           pk[4 * u + 2], pk[4 * u + 3]);
            const int krow = k0 + r, q0 = tile * 128 + g * 64 + h * 32;
            if (krow < p.S) {
              __nv_bfloat16* gdst = p.dst + ((long long)job * p.S + krow) * p.S + q0;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (q0 + 8 * u < p.S)
                  *reinterpret_cast<uint4*>(gdst + 8 * u) =
                      make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            }
          } else {
            store_row32(ds_chunk, r, 4 * h, *reinterpret_cast<const float(*)[32]>(d + 32 * h));
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(ds_full);
          trace2(p, T2_SM_DS, warp, t);
        }
      }
      // ---- dK, dV of the job (dK carries the dS scale)
      mbar_wait(fin, round & 1);
      tc_fence_after();
      const int krow = k0 + r;
      __nv_bfloat16* drow = p.dqkv + ((long long)smp * p.S + krow) * p.ld_qkv + (long long)head * 3 * HD;
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

template <int HD, int MODE>
cudaError_t launch_bwd_dq(const Bwd2Params& p, int grid, cudaStream_t s) {
  using C = Bwd2Cfg<HD>;
  static cudaError_t attr = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(attn_bwd_dq_kernel<HD, MODE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  });
  if (attr != cudaSuccess) return attr;
  attn_bwd_dq_kernel<HD, MODE><<<grid, kBwd2Threads, C::SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

template <int HD>
cudaError_t launch_bwd_dq_mode(const Bwd2Params& p, int grid, int mode, cudaStream_t s) {
  switch (mode) {
    case 1: return launch_bwd_dq<HD, 1>(p, grid, s);
    case 2: return launch_bwd_dq<HD, 2>(p, grid, s);
    case 3: return launch_bwd_dq<HD, 3>(p, grid, s);
    default: return launch_bwd_dq<HD, 0>(p, grid, s);
  }
}




}  // namespace attn
}  // namespace sm100

cudaError_t attn_bwd_split_sm100(const AttnDesc& d, void* dst, cudaStream_t s) {
  using namespace sm100::attn;
  if (!attn_fused_supported(d) || !d.dout || !d.delta || !d.dqkv || !dst || !d.lse ||
      d.ld_o % 8 != 0 || reinterpret_cast<uintptr_t>(d.dout) % 16 ||
      reinterpret_cast<uintptr_t>(d.dqkv) % 16 || reinterpret_cast<uintptr_t>(dst) % 16) {
    g_attn_err = "attn_bwd_split_sm100: unsupported shape or missing operand";
    return cudaErrorInvalidValue;
  }
  BwdParams p;
  std::memset(&p, 0, sizeof(p));
  const int64_t cols = 3 * d.heads * d.head_dim;
  if (!encode_3d(&p.tm_kv, d.qkv, cols, d.seq, d.samples, d.ld_qkv, 128) ||
      !encode_3d(&p.tm_q, d.qkv, cols, d.seq, d.samples, d.ld_qkv, BQB) ||
      !encode_3d(&p.tm_do, d.dout, d.heads * d.head_dim, d.seq, d.samples, d.ld_o, BQB) ||
      !encode_3d(&p.tm_dst, dst, d.seq, d.seq, d.samples * d.heads, d.seq, 128))
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
    g_attn_err = "attn_bwd_split_sm100: grid too large";
    return cudaErrorInvalidValue;
  }
  cudaError_t e = d.head_dim == 128 ? launch_bwd<128>(p, (int)grid, s) : launch_bwd<64>(p, (int)grid, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_bwd_split_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

AttnBwdPlan attn_bwd_dq_plan(const AttnDesc& d) {
  AttnBwdPlan pl;
  const int64_t n = (d.seq + 127) / 128, jobs = d.samples * d.heads;
  const int sms = sm100::attn::device_sms();
  if (n <= 0 || jobs <= 0 || sms <= 0 || n > sms) return pl;
  pl.n = (int)n;
  pl.gangs = (int)std::min<int64_t>(sms / n, jobs);
  pl.acc_bytes = (size_t)pl.gangs * n * 128 * d.head_dim * 4;
  pl.sem_bytes = (size_t)pl.gangs * n * 4;
  pl.ok = true;
  return pl;
}

cudaError_t attn_bwd_dq_sm100(const AttnDesc& d, const AttnBwdDqArgs& x, cudaStream_t s, int mode) {
  using namespace sm100::attn;
  const AttnBwdPlan pl = attn_bwd_dq_plan(d);
  if (!attn_fused_supported(d) || !pl.ok || !d.dout || !d.delta || !d.dqkv || !d.lse ||
      !x.dq_acc || !x.dq_sem || d.ld_o % 8 != 0 || reinterpret_cast<uintptr_t>(d.dout) % 16 ||
      reinterpret_cast<uintptr_t>(d.dqkv) % 16 || reinterpret_cast<uintptr_t>(x.dq_acc) % 16 ||
      reinterpret_cast<uintptr_t>(d.lse) % 16 || reinterpret_cast<uintptr_t>(d.delta) % 16) {
    g_attn_err = "attn_bwd_dq_sm100: unsupported shape or missing operand";
    return cudaErrorInvalidValue;
  }
  Bwd2Params p;
  std::memset(&p, 0, sizeof(p));
  const int64_t cols = 3 * d.heads * d.head_dim;
  if (!encode_3d(&p.tm_kv, d.qkv, cols, d.seq, d.samples, d.ld_qkv, 128) ||
      !encode_3d(&p.tm_do, d.dout, d.heads * d.head_dim, d.seq, d.samples, d.ld_o, 128) ||
      !encode_rows_f32(&p.tm_lse, d.lse, d.seq, d.samples * d.heads) ||
      !encode_rows_f32(&p.tm_dlt, d.delta, d.seq, d.samples * d.heads))
    return cudaErrorInvalidValue;
  if (mode == 3 && !x.dst) return cudaErrorInvalidValue;
  p.dst = static_cast<__nv_bfloat16*>(x.dst);
  p.S = (int)d.seq;
  p.H = (int)d.heads;
  p.n = pl.n;
  p.jobs = (int)(d.samples * d.heads);
  p.n_gangs = pl.gangs;
  p.c = d.scale * kLog2e;
  p.scale = d.scale;
  p.dqkv = static_cast<__nv_bfloat16*>(d.dqkv);
  p.ld_qkv = d.ld_qkv;
  p.dq_acc = x.dq_acc;
  p.dq_sem = x.dq_sem;
  p.trace = nullptr;
  if (std::getenv("TESS_ATTN_TRACE")) {
    static long long* tr = nullptr;
    const size_t nb = (size_t)T2_N * 16 * 16 * sizeof(long long);
    if (!tr) cudaMalloc(&tr, nb);
    cudaMemsetAsync(tr, 0, nb, s);
    p.trace = tr;
    g_attn_trace = tr;
  }
  cudaError_t e = cudaMemsetAsync(x.dq_sem, 0, pl.sem_bytes, s);
  if (e == cudaSuccess)
    e = d.head_dim == 128 ? launch_bwd_dq_mode<128>(p, pl.gangs * pl.n, mode, s)
                          : launch_bwd_dq_mode<64>(p, pl.gangs * pl.n, mode, s);
  if (e != cudaSuccess) g_attn_err = std::string("attn_bwd_dq_sm100 launch: ") + cudaGetErrorString(e);
  return e;
}

}  // namespace tess
