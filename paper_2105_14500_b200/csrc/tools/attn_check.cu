// Standalone check + timing of the attention backward on the GPU box (cfg4
// head shape by default: b=4, s=2048, 96 heads, hd=128):
//   * the round-1 split path: attn_bwd_split_sm100 + the batched dQ GEMM over the
//     stored dS^T, against
//   * the round-2 experiment attn_bwd_dq_sm100 (attn_bwd_experiments.cuh:
//     dQ fused with an ordered on-chip accumulation, and its modes);
//   * the single-query-tile forward experiment (attn_fwd_experiments.cuh)
//     against the product forward: max |dO|, |dlse| and timing
//     (TESS_FWD_ONLY=1 stops after it).
// dQ of the split path is also recomputed by a CUDA-core loop over dS^T, so
// both dQs have an independent check; dK / dV are compared between the two
// kernels. The product parity tests go through the C-ABI and the fp64 oracle.
//   attn_check [b s heads hd] [reps] [profile mode: -1 split, 10 dQ pass, 11 dK/dV pass, 12 fwd1]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../kernels/gemm.h"
#include "attn_bwd_experiments.cuh"
#include "attn_fwd_experiments.cuh"

using namespace tess;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::printf("CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e_), __FILE__, __LINE__, \
                  attn_last_error());                                                           \
      std::exit(2);                                                                             \
    }                                                                                           \
  } while (0)

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16((((x & 0xFFFFFF) / 16777216.0f) * 2.f - 1.f) * scale);
  }
}

// delta[smp, h, q] = sum_d dO * O
__global__ void delta_k(const __nv_bfloat16* dout, const __nv_bfloat16* o, float* delta, int S,
                        int H, int hd, long long ld) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // (smp, h, q)
  const int q = idx % S, h = (idx / S) % H, smp = idx / ((long long)S * H);
  const __nv_bfloat16* a = dout + ((long long)smp * S + q) * ld + h * hd;
  const __nv_bfloat16* b = o + ((long long)smp * S + q) * ld + h * hd;
  float s = 0.f;
  for (int d = 0; d < hd; ++d) s += __bfloat162float(a[d]) * __bfloat162float(b[d]);
  delta[idx] = s;
}

// dQ[q, d] = scale * sum_k dS^T[k, q] K[k, d]  (fp32 CUDA cores), written as fp32
__global__ void dq_ref(const __nv_bfloat16* dst, const __nv_bfloat16* qkv, float* out, int S, int H,
                       int hd, long long ld) {
  const int d = threadIdx.x;
  const int q = blockIdx.x;
  const int job = blockIdx.y;  // smp * H + h
  const int smp = job / H, h = job % H;
  const __nv_bfloat16* ds = dst + (long long)job * S * S;
  const __nv_bfloat16* kk = qkv + (long long)smp * S * ld + h * 3 * hd + hd;
  float acc = 0.f;
  for (int k = 0; k < S; ++k)
    acc += __bfloat162float(ds[(long long)k * S + q]) * __bfloat162float(kk[(long long)k * ld + d]);
  out[((long long)smp * S + q) * (H * hd) + h * hd + d] = acc / sqrtf((float)hd);
}

static std::vector<float> to_f32(const __nv_bfloat16* d, size_t n) {
  std::vector<__nv_bfloat16> h(n);
  CK(cudaMemcpy(h.data(), d, n * 2, cudaMemcpyDeviceToHost));
  std::vector<float> f(n);
  for (size_t i = 0; i < n; ++i) f[i] = __bfloat162float(h[i]);
  return f;
}

int main(int argc, char** argv) {
  int B = 4, S = 2048, H = 96, hd = 128, reps = 10;
  if (argc >= 5) {
    B = atoi(argv[1]);
    S = atoi(argv[2]);
    H = atoi(argv[3]);
    hd = atoi(argv[4]);
  }
  if (argc >= 6) reps = atoi(argv[5]);
  const long long ldq = 3LL * H * hd, ldo = (long long)H * hd, rows = (long long)B * S;
  const float scale = 1.0f / std::sqrt((float)hd);
  __nv_bfloat16 *qkv, *dout, *o, *dqkv1, *dqkv2, *dqkv3, *dst;
  float *lse, *delta, *dqr, *acc;
  uint32_t* sem;
  CK(cudaMalloc(&qkv, rows * ldq * 2));
  CK(cudaMalloc(&dout, rows * ldo * 2));
  CK(cudaMalloc(&o, rows * ldo * 2));
  CK(cudaMalloc(&dqkv1, rows * ldq * 2));
  CK(cudaMalloc(&dqkv2, rows * ldq * 2));
  CK(cudaMalloc(&dqkv3, rows * ldq * 2));
  CK(cudaMalloc(&dst, (size_t)B * H * S * S * 2));
  CK(cudaMalloc(&lse, (size_t)B * H * S * 4));
  CK(cudaMalloc(&delta, (size_t)B * H * S * 4));
  CK(cudaMalloc(&dqr, rows * ldo * 4));
  fill_bf16<<<1184, 256>>>(qkv, rows * ldq, 11u, 1.0f);
  fill_bf16<<<1184, 256>>>(dout, rows * ldo, 29u, 1.0f);
  CK(cudaMemset(dqkv1, 0, rows * ldq * 2));
  CK(cudaMemset(dqkv2, 0, rows * ldq * 2));
  CK(cudaMemset(dqkv3, 0, rows * ldq * 2));

  AttnDesc a;
  a.qkv = qkv;
  a.ld_qkv = ldq;
  a.o = o;
  a.ld_o = ldo;
  a.lse = lse;
  a.samples = B;
  a.heads = H;
  a.seq = S;
  a.head_dim = hd;
  a.scale = scale;
  CK(attn_fwd_sm100(a, 0));
  {  // single-tile forward vs the two-tile forward
    __nv_bfloat16* o1;
    float* lse1;
    CK(cudaMalloc(&o1, rows * ldo * 2));
    CK(cudaMalloc(&lse1, (size_t)B * H * S * 4));
    AttnDesc a1 = a;
    a1.o = o1;
    a1.lse = lse1;
    CK(attn_fwd1_sm100(a1, 0));
    CK(cudaDeviceSynchronize());
    std::vector<__nv_bfloat16> h0(rows * ldo), h1(rows * ldo);
    std::vector<float> l0((size_t)B * H * S), l1((size_t)B * H * S);
    CK(cudaMemcpy(h0.data(), o, rows * ldo * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h1.data(), o1, rows * ldo * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(l0.data(), lse, l0.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(l1.data(), lse1, l1.size() * 4, cudaMemcpyDeviceToHost));
    double dmax = 0, ref = 0, lmax = 0;
    for (size_t i = 0; i < h0.size(); ++i) {
      const double x = __bfloat162float(h0[i]), y = __bfloat162float(h1[i]);
      dmax = std::max(dmax, std::fabs(x - y));
      ref = std::max(ref, std::fabs(x));
    }
    for (size_t i = 0; i < l0.size(); ++i) lmax = std::max(lmax, (double)std::fabs(l0[i] - l1[i]));
    std::printf("fwd1 vs fwd: max|dO| %.3e (max|O| %.3e), max|dlse| %.3e\n", dmax, ref, lmax);
    if (argc >= 7 && atoi(argv[6]) == 12) {
      std::printf("profiled fwd1\n");
      return 0;
    }
    auto t1 = [&](const char* name, auto fn) {
      cudaEvent_t x0, x1;
      cudaEventCreate(&x0);
      cudaEventCreate(&x1);
      for (int w = 0; w < 2; ++w) fn();
      CK(cudaEventRecord(x0));
      for (int i = 0; i < reps; ++i) fn();
      CK(cudaEventRecord(x1));
      CK(cudaEventSynchronize(x1));
      float ms = 0;
      cudaEventElapsedTime(&ms, x0, x1);
      std::printf("%-26s %8.3f ms/iter\n", name, ms / reps);
    };
    t1("attn_fwd (two-tile)", [&]() { CK(attn_fwd_sm100(a, 0)); });
    t1("attn_fwd1 (one-tile)", [&]() { CK(attn_fwd1_sm100(a1, 0)); });
    t1("attn_fwd (two-tile) again", [&]() { CK(attn_fwd_sm100(a, 0)); });
    t1("attn_fwd1 (one-tile) again", [&]() { CK(attn_fwd1_sm100(a1, 0)); });
    if (std::getenv("TESS_FWD_ONLY")) return 0;
  }
  delta_k<<<(unsigned)((B * H * (long long)S + 127) / 128), 128>>>(dout, o, delta, S, H, hd, ldo);
  a.dout = dout;
  a.delta = delta;
  AttnBwdPlan pl = attn_bwd_dq_plan(a);
  std::printf("shape b=%d s=%d heads=%d hd=%d | fused plan ok=%d n=%d gangs=%d (%d CTAs) acc %.1f MB\n",
              B, S, H, hd, pl.ok, pl.n, pl.gangs, pl.gangs * pl.n, pl.acc_bytes / 1e6);
  CK(cudaMalloc(&acc, pl.acc_bytes ? pl.acc_bytes : 16));
  CK(cudaMalloc(&sem, pl.sem_bytes ? pl.sem_bytes : 16));
  AttnBwdDqArgs dqx;
  dqx.dq_acc = acc;
  dqx.dq_sem = sem;
  dqx.dst = dst;

  // split path: attention backward (dK, dV, dS^T) + batched dQ GEMM
  GemmDesc gq;
  gq.M = S;
  gq.N = hd;
  gq.nb0 = H;
  gq.nb1 = B;
  gq.in = DType::BF16;
  gq.trans_a = true;
  gq.seg[0] = {dst, qkv + hd, S};
  gq.lda = S;
  gq.as0 = (int64_t)S * S;
  gq.as1 = (int64_t)H * S * S;
  gq.ldb = ldq;
  gq.bs0 = 3 * hd;
  gq.bs1 = (int64_t)S * ldq;
  gq.c = dqkv1;
  gq.c_type = DType::BF16;
  gq.ldc = ldq;
  gq.cs0 = 3 * hd;
  gq.cs1 = (int64_t)S * ldq;
  gq.alpha = scale;
  auto split = [&]() {
    a.dqkv = dqkv1;
    CK(attn_bwd_split_sm100(a, dst, 0));
    CK(gemm_bf16_sm100(gq, 0));
  };
  auto fused = [&]() {
    a.dqkv = dqkv2;
    CK(attn_bwd_dq_sm100(a, dqx, 0, 0));
  };
  auto mode_only = [&](int mode) {
    a.dqkv = dqkv3;
    CK(attn_bwd_dq_sm100(a, dqx, 0, mode));
  };
  GemmDesc gq3 = gq;
  gq3.c = dqkv3;
  auto split3 = [&]() {
    mode_only(3);
    CK(gemm_bf16_sm100(gq3, 0));
  };
  if (argc >= 7) {  // profiling: one launch of the given mode (-1: the split kernel), nothing else
    const int m = atoi(argv[6]);
    if (m < 0) {
      a.dqkv = dqkv1;
      CK(attn_bwd_split_sm100(a, dst, 0));
    } else if (m == 10) {
      a.dqkv = dqkv3;
      CK(attn_dq_sm100(a, 0));
    } else if (m == 11) {
      a.dqkv = dqkv3;
      CK(attn_bwd_kv_sm100(a, 0));
    } else {
      mode_only(m);
    }
    CK(cudaDeviceSynchronize());
    std::printf("profiled mode %d\n", m);
    return 0;
  }
  split();
  if (pl.ok) fused();
  CK(cudaDeviceSynchronize());
  dq_ref<<<dim3(S, B * H), hd>>>(dst, qkv, dqr, S, H, hd, ldq);
  CK(cudaDeviceSynchronize());

  // --- compare
  {
    auto d1 = to_f32(dqkv1, rows * ldq);
    auto d2 = to_f32(dqkv2, rows * ldq);
    std::vector<float> r(rows * ldo);
    CK(cudaMemcpy(r.data(), dqr, rows * ldo * 4, cudaMemcpyDeviceToHost));
    // parts: 0 dQ, 1 dK, 2 dV
    double num1[3] = {0, 0, 0}, num2[3] = {0, 0, 0}, den[3] = {0, 0, 0}, mx2[3] = {0, 0, 0};
    long long nan2 = 0;
    for (long long row = 0; row < rows; ++row)
      for (int h = 0; h < H; ++h)
        for (int part = 0; part < 3; ++part)
          for (int d = 0; d < hd; ++d) {
            const long long i = row * ldq + (long long)h * 3 * hd + part * hd + d;
            const double want = part == 0 ? r[row * ldo + h * hd + d] : d1[i];
            const double e1 = part == 0 ? d1[i] - want : 0.0;
            const double e2 = d2[i] - want;
            if (!std::isfinite(d2[i])) ++nan2;
            num1[part] += e1 * e1;
            num2[part] += e2 * e2;
            den[part] += want * want;
            mx2[part] = std::fmax(mx2[part], std::fabs(e2));
          }
    const char* nm[3] = {"dQ", "dK", "dV"};
    for (int part = 0; part < 3; ++part)
      std::printf("%s: split-vs-ref %.3e | fused-vs-%s %.3e (max abs %.3e)\n", nm[part],
                  std::sqrt(num1[part] / den[part]), part == 0 ? "ref" : "split",
                  std::sqrt(num2[part] / den[part]), mx2[part]);
    std::printf("fused non-finite: %lld\n", nan2);
    bool ok = nan2 == 0;
    for (int part = 0; part < 3; ++part) ok = ok && std::sqrt(num2[part] / den[part]) < 1e-2;
    std::printf("CHECK %s\n", ok ? "PASS" : "FAIL");
    if (pl.ok) {
      split3();
      CK(cudaDeviceSynchronize());
      auto d4 = to_f32(dqkv3, rows * ldq);
      double nn[3] = {0, 0, 0}, dd[3] = {0, 0, 0};
      long long same[3] = {0, 0, 0}, tot[3] = {0, 0, 0};
      for (long long row = 0; row < rows; ++row)
        for (int h = 0; h < H; ++h)
          for (int part = 0; part < 3; ++part)
            for (int dd_ = 0; dd_ < hd; ++dd_) {
              const long long i = row * ldq + (long long)h * 3 * hd + part * hd + dd_;
              const double e = d4[i] - d1[i];
              nn[part] += e * e;
              dd[part] += (double)d1[i] * d1[i];
              same[part] += d4[i] == d1[i];
              ++tot[part];
            }
      for (int part = 0; part < 3; ++part)
        std::printf("mode3+GEMM vs split %s: %.3e (bitwise equal %.4f)\n", nm[part],
                    std::sqrt(nn[part] / dd[part]), (double)same[part] / tot[part]);
    }
    {
      // the two-pass path: dK/dV pass + dQ pass
      CK(cudaMemset(dqkv3, 0, rows * ldq * 2));
      a.dqkv = dqkv3;
      CK(attn_bwd_kv_sm100(a, 0));
      CK(attn_dq_sm100(a, 0));
      CK(cudaDeviceSynchronize());
      auto d5 = to_f32(dqkv3, rows * ldq);
      double nn[3] = {0, 0, 0}, dd[3] = {0, 0, 0};
      long long bad = 0;
      for (long long row = 0; row < rows; ++row)
        for (int h = 0; h < H; ++h)
          for (int part = 0; part < 3; ++part)
            for (int dd_ = 0; dd_ < hd; ++dd_) {
              const long long i = row * ldq + (long long)h * 3 * hd + part * hd + dd_;
              const double want = part == 0 ? r[row * ldo + h * hd + dd_] : d1[i];
              const double e = d5[i] - want;
              if (!std::isfinite(d5[i])) ++bad;
              nn[part] += e * e;
              dd[part] += want * want;
            }
      for (int part = 0; part < 3; ++part)
        std::printf("kv+dQpass %s vs %s: %.3e\n", nm[part], part == 0 ? "ref" : "split",
                    std::sqrt(nn[part] / dd[part]));
      std::printf("kv+dQpass non-finite %lld -> %s\n", bad,
                  bad == 0 && std::sqrt(nn[0] / dd[0]) < 1e-2 && std::sqrt(nn[1] / dd[1]) < 1e-2 &&
                          std::sqrt(nn[2] / dd[2]) < 1e-2
                      ? "PASS"
                      : "FAIL");
    }
    // determinism: a second fused run must match bitwise
    if (pl.ok) {
      fused();
      CK(cudaDeviceSynchronize());
      auto d3 = to_f32(dqkv2, rows * ldq);
      std::printf("fused rerun bitwise equal: %s\n",
                  std::memcmp(d2.data(), d3.data(), d2.size() * 4) == 0 ? "yes" : "NO");
    }
  }

  // --- timing
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](const char* name, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) fn();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("%-26s %8.3f ms/iter\n", name, ms / reps);
  };
  time_it("attn_fwd", [&]() { CK(attn_fwd_sm100(a, 0)); });
  time_it("attn_bwd (split, no dQ)", [&]() {
    a.dqkv = dqkv1;
    CK(attn_bwd_split_sm100(a, dst, 0));
  });
  time_it("dQ GEMM", [&]() { CK(gemm_bf16_sm100(gq, 0)); });
  time_it("split total", split);
  if (pl.ok) {
    time_it("fused (dQ inside)", fused);
    time_it("mode1 (dQ MMA, no accum)", [&]() { mode_only(1); });
    time_it("mode2 (no dQ, no store)", [&]() { mode_only(2); });
    time_it("mode3 (no dQ, dS^T store)", [&]() { mode_only(3); });
    time_it("mode3 + dQ GEMM", split3);
    time_it("dQ pass (recompute)", [&]() {
      a.dqkv = dqkv3;
      CK(attn_dq_sm100(a, 0));
    });
    time_it("dK/dV pass", [&]() {
      a.dqkv = dqkv3;
      CK(attn_bwd_kv_sm100(a, 0));
    });
    time_it("dK/dV pass + dQ pass", [&]() {
      a.dqkv = dqkv3;
      CK(attn_bwd_kv_sm100(a, 0));
      CK(attn_dq_sm100(a, 0));
    });
    time_it("split total (again)", split);
  }

  for (int tm = 0; tm < 4 && std::getenv("TESS_ATTN_TRACE") && pl.ok; ++tm) {
    mode_only(tm);
    std::printf("trace mode %d\n", tm);
    CK(cudaDeviceSynchronize());
    std::vector<long long> tr(13 * 16 * 16);
    CK(cudaMemcpy(tr.data(), attn_debug_trace(), tr.size() * 8, cudaMemcpyDeviceToHost));
    long long t0 = 0;
    for (long long v : tr)
      if (v && (!t0 || v < t0)) t0 = v;
    auto at = [&](int ev, int w, int st) {
      long long v = tr[(ev * 16 + w) * 16 + st];
      return v ? v - t0 : -1;
    };
    std::printf("step |  MMA: dV     dP     S(i+1)  dK     dQ  | SM(w8): S_in  P_out  dP_in  dS_out"
                " | SM(w15) P_out dS_out | DR(w4): in  free  sem  done\n");
    for (int st = 0; st < 16; ++st)
      std::printf("%4d | %6lld %6lld %6lld %6lld %6lld | %6lld %6lld %6lld %6lld | %6lld %6lld | %6lld "
                  "%6lld %6lld %6lld\n",
                  st, at(0, 1, st), at(1, 1, st), at(2, 1, st + 1 < 16 ? st + 1 : st), at(3, 1, st),
                  at(4, 1, st), at(5, 8, st), at(6, 8, st), at(7, 8, st), at(8, 8, st), at(6, 15, st),
                  at(8, 15, st), at(9, 4, st), at(10, 4, st), at(11, 4, st), at(12, 4, st));
    std::printf("softmax warps 8..15 per step: S_in / P_out / dP_in / dS_out\n");
    for (int st = 4; st < 8; ++st) {
      for (int ev = 5; ev <= 8; ++ev) {
        std::printf("%4d ev%d:", st, ev);
        for (int w = 8; w < 16; ++w) std::printf(" %6lld", at(ev, w, st));
        std::printf("\n");
      }
    }
  }
  return 0;
}
