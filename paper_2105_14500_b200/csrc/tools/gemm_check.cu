// Standalone device-side check + timing of the tcgen05 GEMM against a naive
// fp32 CUDA-core reference on identical bf16 inputs. Used during kernel
// bring-up on the GPU box (`gemm_check [--bench]`); the product parity tests
// go through the C-ABI and the fp64 oracle instead.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../kernels/gemm.h"

using namespace tess;

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      std::printf("CUDA error %s at %s:%d (%s)\n", cudaGetErrorString(e_), \
                  __FILE__, __LINE__, gemm_last_error());                  \
      std::exit(2);                                                        \
    }                                                                      \
  } while (0)

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed, float scale) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    float v = ((x & 0xFFFFFF) / 16777216.0f) * 2.f - 1.f;
    p[i] = __float2bfloat16(v * scale);
  }
}

__global__ void ref_gemm(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C,
                         int M, int N, int K, long long lda, long long ldb, bool ta,
                         bool tb, int nb0, int nb1, long long as0, long long as1,
                         long long bs0, long long bs1) {
  long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = (long long)M * N * nb0 * nb1;
  if (idx >= total) return;
  int n = idx % N;
  int m = (idx / N) % M;
  int b = idx / ((long long)M * N);
  int b0 = b % nb0, b1 = b / nb0;
  const __nv_bfloat16* a = A + b0 * as0 + b1 * as1;
  const __nv_bfloat16* bb = B + b0 * bs0 + b1 * bs1;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) {
    float av = __bfloat162float(ta ? a[(long long)k * lda + m] : a[(long long)m * lda + k]);
    float bv = __bfloat162float(tb ? bb[(long long)n * ldb + k] : bb[(long long)k * ldb + n]);
    acc += av * bv;
  }
  C[idx] = acc;
}

struct Case {
  int M, N, K, nb0, nb1;
  bool ta, tb;
  int nseg;
  Epi epi;
  bool c_bf16;
};

static bool run_case(const Case& cs) {
  const int M = cs.M, N = cs.N, K = cs.K;
  const int nb = cs.nb0 * cs.nb1;
  // Pad leading dims to exercise strided views.
  auto up8 = [](long long v) { return (v + 7) / 8 * 8; };
  const long long lda = up8(cs.ta ? M : K) + 8;
  const long long ldb = up8(cs.tb ? K : N) + 8;
  const long long arows = cs.ta ? K : M, brows = cs.tb ? N : K;
  const long long as0 = arows * lda, as1 = as0 * cs.nb0;
  const long long bs0 = brows * ldb, bs1 = bs0 * cs.nb0;
  __nv_bfloat16 *A, *B;
  CK(cudaMalloc(&A, sizeof(__nv_bfloat16) * as0 * nb));
  CK(cudaMalloc(&B, sizeof(__nv_bfloat16) * bs0 * nb));
  fill_bf16<<<512, 256>>>(A, as0 * nb, 1234u, 1.f);
  fill_bf16<<<512, 256>>>(B, bs0 * nb, 777u, 1.f);
  float* ref;
  CK(cudaMalloc(&ref, sizeof(float) * (size_t)M * N * nb));
  long long total = (long long)M * N * nb;
  ref_gemm<<<(total + 255) / 256, 256>>>(A, B, ref, M, N, K, lda, ldb, cs.ta, cs.tb,
                                         cs.nb0, cs.nb1, as0, as1, bs0, bs1);
  CK(cudaGetLastError());

  const long long ldc = (N + 7) / 8 * 8 + 16;
  const long long cs0 = (long long)M * ldc, cs1 = cs0 * cs.nb0;
  const size_t csz = cs0 * nb;
  void* C;
  CK(cudaMalloc(&C, csz * 4));
  CK(cudaMemset(C, 0, csz * 4));
  void* R = nullptr;
  void* Z = nullptr;
  const int esz = cs.c_bf16 ? 2 : 4;
  if (cs.epi == Epi::Resid) {
    CK(cudaMalloc(&R, csz * esz));
    if (cs.c_bf16) fill_bf16<<<512, 256>>>((__nv_bfloat16*)R, csz, 99u, 1.f);
    else CK(cudaMemset(R, 0, csz * 4));
  }
  if (cs.epi == Epi::Gelu) CK(cudaMalloc(&Z, csz * esz));
  if (cs.epi == Epi::Accum) {
    std::vector<float> ones(csz, 0.5f);
    CK(cudaMemcpy(C, ones.data(), csz * 4, cudaMemcpyHostToDevice));
  }

  GemmDesc d;
  d.M = M;
  d.N = N;
  d.nb0 = cs.nb0;
  d.nb1 = cs.nb1;
  d.trans_a = cs.ta;
  d.trans_b = cs.tb;
  d.lda = lda;
  d.as0 = as0;
  d.as1 = as1;
  d.ldb = ldb;
  d.bs0 = bs0;
  d.bs1 = bs1;
  d.nseg = cs.nseg;
  const int kseg = K / cs.nseg;
  for (int s = 0; s < cs.nseg; ++s) {
    const long long k0 = (long long)s * kseg;
    const long long kk = s == cs.nseg - 1 ? K - k0 : kseg;
    d.seg[s].a = A + (cs.ta ? k0 * lda : k0);
    d.seg[s].b = B + (cs.tb ? k0 : k0 * ldb);
    d.seg[s].k = kk;
  }
  d.in = DType::BF16;
  d.c = C;
  d.c_type = cs.c_bf16 ? DType::BF16 : DType::F32;
  d.ldc = ldc;
  d.cs0 = cs0;
  d.cs1 = cs1;
  d.r = R;
  d.ldr = ldc;
  d.rs0 = cs0;
  d.rs1 = cs1;
  d.z = Z;
  d.ldz = ldc;
  d.zs0 = cs0;
  d.zs1 = cs1;
  d.alpha = 1.0f;
  d.epi = cs.epi;
  CK(gemm(d, 0));
  CK(cudaDeviceSynchronize());

  std::vector<float> hr((size_t)M * N * nb);
  CK(cudaMemcpy(hr.data(), ref, hr.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> hc(csz * esz), hrr, hz;
  CK(cudaMemcpy(hc.data(), C, hc.size(), cudaMemcpyDeviceToHost));
  if (R) {
    hrr.resize(csz * esz);
    CK(cudaMemcpy(hrr.data(), R, hrr.size(), cudaMemcpyDeviceToHost));
  }
  if (Z) {
    hz.resize(csz * esz);
    CK(cudaMemcpy(hz.data(), Z, hz.size(), cudaMemcpyDeviceToHost));
  }
  auto load = [&](const std::vector<uint8_t>& buf, size_t i) -> float {
    if (cs.c_bf16) {
      uint16_t h;
      std::memcpy(&h, buf.data() + i * 2, 2);
      uint32_t u = (uint32_t)h << 16;
      float f;
      std::memcpy(&f, &u, 4);
      return f;
    }
    float f;
    std::memcpy(&f, buf.data() + i * 4, 4);
    return f;
  };
  double maxd = 0, maxr = 0;
  for (int b = 0; b < nb; ++b) {
    const int b0 = b % cs.nb0, b1 = b / cs.nb0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        size_t ci = b0 * cs0 + b1 * cs1 + (size_t)m * ldc + n;
        double want = hr[((size_t)b * M + m) * N + n];
        if (cs.epi == Epi::Accum) want += 0.5;
        if (cs.epi == Epi::Resid) want += cs.c_bf16 ? load(hrr, ci) : 0.0;
        if (cs.epi == Epi::Gelu) {
          double zg = load(hz, ci);
          maxd = std::max(maxd, std::fabs(zg - want));
          want = 0.5 * want * (1.0 + std::erf(want / std::sqrt(2.0)));
        }
        double got = load(hc, ci);
        maxd = std::max(maxd, std::fabs(got - want));
        maxr = std::max(maxr, std::fabs(want));
      }
  }
  double rel = maxd / std::max(maxr, 1e-30);
  double tol = cs.c_bf16 ? 1e-2 : 1e-5;
  bool ok = rel <= tol;
  std::printf("%s M=%d N=%d K=%d nb=%dx%d %s%s seg=%d epi=%d c=%s rel=%.3e\n",
              ok ? "PASS" : "FAIL", M, N, K, cs.nb0, cs.nb1, cs.ta ? "T" : "N",
              cs.tb ? "T" : "N", cs.nseg, (int)cs.epi, cs.c_bf16 ? "bf16" : "f32",
              rel);
  cudaFree(A);
  cudaFree(B);
  cudaFree(ref);
  cudaFree(C);
  if (R) cudaFree(R);
  if (Z) cudaFree(Z);
  return ok;
}

static void bench(int M, int N, int K, bool ta, bool tb, int iters) {
  __nv_bfloat16 *A, *B;
  float* C;
  CK(cudaMalloc(&A, sizeof(__nv_bfloat16) * (size_t)M * K));
  CK(cudaMalloc(&B, sizeof(__nv_bfloat16) * (size_t)K * N));
  CK(cudaMalloc(&C, sizeof(__nv_bfloat16) * (size_t)M * N));
  fill_bf16<<<1024, 256>>>(A, (size_t)M * K, 1u, 1.f);
  fill_bf16<<<1024, 256>>>(B, (size_t)K * N, 2u, 1.f);
  GemmDesc d;
  d.M = M;
  d.N = N;
  d.trans_a = ta;
  d.trans_b = tb;
  d.lda = ta ? M : K;
  d.ldb = tb ? K : N;
  d.seg[0] = {A, B, K};
  d.nseg = 1;
  d.in = DType::BF16;
  d.c = C;
  d.c_type = DType::BF16;
  d.ldc = N;
  for (int i = 0; i < 3; ++i) CK(gemm(d, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) CK(gemm(d, 0));
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= iters;
  double tf = 2.0 * M * N * (double)K / (ms * 1e-3) / 1e12;
  std::printf("BENCH %s%s M=%d N=%d K=%d  %.3f ms  %.1f TFLOP/s\n", ta ? "T" : "N",
              tb ? "T" : "N", M, N, K, ms, tf);
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
}

int main(int argc, char** argv) {
  bool do_bench = argc > 1 && std::strcmp(argv[1], "--bench") == 0;
  bool all = true;
  std::vector<Case> cases = {
      {128, 256, 64, 1, 1, false, false, 1, Epi::Store, false},
      {128, 256, 64, 1, 1, false, true, 1, Epi::Store, false},
      {128, 256, 64, 1, 1, true, false, 1, Epi::Store, false},
      {128, 128, 128, 1, 1, true, true, 1, Epi::Store, false},
      {256, 512, 320, 1, 1, false, false, 1, Epi::Store, false},
      {256, 512, 320, 1, 1, false, true, 1, Epi::Store, false},
      {256, 512, 320, 1, 1, true, false, 1, Epi::Store, false},
      {300, 260, 200, 1, 1, false, false, 1, Epi::Store, false},
      {300, 260, 200, 1, 1, false, true, 1, Epi::Store, false},
      {300, 260, 200, 1, 1, true, false, 1, Epi::Store, false},
      {512, 768, 1024, 1, 1, false, false, 2, Epi::Store, true},
      {512, 768, 1024, 1, 1, false, true, 2, Epi::Accum, false},
      {512, 768, 1024, 1, 1, true, false, 2, Epi::Accum, false},
      {256, 384, 512, 1, 1, false, false, 1, Epi::Resid, true},
      {256, 384, 512, 1, 1, false, false, 1, Epi::Gelu, true},
      {256, 256, 128, 3, 2, false, true, 1, Epi::Store, false},
      {256, 128, 256, 3, 2, false, false, 1, Epi::Store, true},
      {256, 128, 256, 3, 2, true, false, 1, Epi::Store, false},
      {1024, 1024, 1024, 1, 1, false, false, 4, Epi::Store, false},
  };
  for (const auto& c : cases) all &= run_case(c);
  if (do_bench) {
    bench(8192, 8192, 8192, false, false, 10);
    bench(8192, 8192, 8192, false, true, 10);
    bench(8192, 8192, 8192, true, false, 10);
    bench(8192, 49152, 12288, false, false, 3);
  }
  std::printf(all ? "ALL PASS\n" : "SOME FAILED\n");
  return all ? 0 : 1;
}
