// Inline-PTX building blocks shared by the sm_100a tensor-core kernels
// (gemm_sm100.cu, attention_sm100.cu): mbarriers, TMA, UMMA shared-memory
// descriptors, tcgen05.mma / commit / ld / st.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace tess {
namespace sm100 {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map,
                                            uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::"
      "bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0),
      "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor for a 128B-swizzled canonical layout.
//   K-major : rows of 128 B (64 bf16 of K), 8-row atoms SBO=1024 B apart.
//   MN-major: rows of 128 B (64 bf16 of M/N) per K index, 8-K-row atoms
//             SBO=1024 B apart, 64-wide M/N chunks LBO bytes apart.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo,
                                               uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc,
                                         uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 "
      "[%0];" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]),
        "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- additions for the fused attention kernels ------------------------------
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// tcgen05.ld of 32 consecutive fp32 columns of this warp's 32 TMEM lanes
// (thread = lane = row) WITHOUT the wait; pair with tmem_wait_ld + reg_fence.
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Ties registers filled by tcgen05.ld to a point after tmem_wait_ld, so the
// compiler cannot consume them before the wait.
__device__ __forceinline__ void reg_fence32(uint32_t (&r)[32]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
  asm volatile(""
               : "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                 "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Generic-proxy shared-memory writes -> visible to the async proxy (UMMA/TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// UMMA instruction descriptor: bf16 x bf16 -> fp32, M x N, operand majorness.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void reg_fence16(uint32_t (&r)[16]) {
  asm volatile(""
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// global (f32) += shared tile, performed by the TMA unit (no read-back by the SM)
__device__ __forceinline__ void tma_reduce_add_4d(const CUtensorMap* map, uint32_t src, int c0,
                                                  int c1, int c2, int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], "
      "[%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Non-tensor bulk copies shared -> global performed by the TMA unit: a plain
// store, or an fp32 add into global (the reduction happens in L2).
__device__ __forceinline__ void bulk_store(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(ssrc), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_reduce_add_f32(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                   gdst),
               "r"(ssrc), "r"(bytes)
               : "memory");
}
// Orders this thread's global accesses between the generic and async proxies.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp-wide forms: every lane of a converged warp executes them with the same
// (warp-uniform) operands, one elected lane issues. Keeps the descriptor math
// on the uniform datapath instead of per-MMA ELECT / R2UR loops.
__device__ __forceinline__ void mma_bf16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_bf16_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}



// Blackwell packed fp32 pairs (FFMA2 / FADD2 / FMUL2, one issue slot per two
// lanes' worth of work) and the 3-input max (FMNMX3): the softmax loops of the
// attention kernels are issue-bound.
__device__ __forceinline__ unsigned long long f2_bits(float2 v) {
  return (unsigned long long)__float_as_uint(v.x) | ((unsigned long long)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 bits_f2(unsigned long long b) {
  return make_float2(__uint_as_float((uint32_t)b), __uint_as_float((uint32_t)(b >> 32)));
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return bits_f2(d);
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// One K=128 block (8 MMAs of K=16) as ONE warp-wide statement: a single
// elect, descriptors advanced in PTX registers (K-major SW128 operands +32 B
// per step and the next 16 KB chunk after four; MN-major ones +2 KB; TMEM A
// +8 columns). The attention kernels' MMA warp shares its SM sub-partition
// with two busy softmax warps; per-MMA elect / R2UR sequences there kept the
// tensor pipe waiting for instructions.
// A, B K-major (smem)
__device__ __forceinline__ void mma_k128_ss_kk(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 a, b;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 a, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, p;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 1018;\n\t"
      "add.u64 b, b, 1018;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0));
}
// A K-major, B MN-major (smem)
__device__ __forceinline__ void mma_k128_ss_kn(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 a, b;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 a, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, p;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 1018;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "add.u64 a, a, 2;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0));
}
// A in TMEM, B K-major (smem)
__device__ __forceinline__ void mma_k128_ts_k(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 b;\n\t"
      ".reg .b32 ta;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 ta, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, p;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 1018;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc0));
}
// A in TMEM, B MN-major (smem)
__device__ __forceinline__ void mma_k128_ts_n(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 b;\n\t"
      ".reg .b32 ta;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 ta, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, p;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc0));
}
// A in TMEM in 8-column pairs 32 columns apart (columns 0, 8, 32, 40, ...),
// B MN-major (smem)
__device__ __forceinline__ void mma_k128_ts_n_pairs(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 b;\n\t"
      ".reg .b32 ta;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 ta, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, p;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 24;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 24;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 24;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc0));
}
// A in TMEM in 32-column quads 64 columns apart (columns 0, 8, 16, 24, 64,
// 72, 80, 88), B MN-major (smem)
__device__ __forceinline__ void mma_k128_ts_n_quads(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                   uint32_t acc0) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q, e;\n\t"
      ".reg .b64 b;\n\t"
      ".reg .b32 ta;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b32 ta, %1;\n\t"
      "mov.b64 b, %2;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, p;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 40;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "add.u32 ta, ta, 8;\n\t"
      "add.u64 b, b, 128;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], b, %3, q;\n\t"
      "}" ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc0));
}

// D[tmem] (+)= A[tmem] * B[smem]: the A operand (M x 16, bf16 packed two per
// 32-bit column, K-major) is read from tensor memory at column tmem_a.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}


}  // namespace sm100
}  // namespace tess
