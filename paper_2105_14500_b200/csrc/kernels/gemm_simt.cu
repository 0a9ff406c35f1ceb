// fp32 CUDA-core GEMM: the fp32 parity path.
//
// BASELINE.json config 1 asks for the Tesseract product in fp32 within 1e-5
// of the fp64 reference (reference proj/src/matrix.cpp:142-216 computes in
// fp64). Tensor cores have no fp32 input mode at that accuracy (TF32 keeps
// 10 mantissa bits), so fp32 runs here on FMA units. It honours the same
// GemmDesc contract as the tcgen05 kernel (segments, two batch levels,
// transposed storage, epilogues), so every schedule and layer runs unchanged
// in fp32 mode and can be checked against the oracle at 1e-5.
#include "gemm.h"

#include <cuda_bf16.h>

#include <string>

namespace tess {
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16;

struct Params {
  GemmSeg seg[kMaxSegments];
  int nseg;
  long long M, N;
  int nb0;
  long long lda, as0, as1, ldb, bs0, bs1;
  void* c;
  long long ldc, cs0, cs1;
  const float* r;
  long long ldr, rs0, rs1;
  float* z;
  long long ldz, zs0, zs1;
  float alpha;
  int epi;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const Params p) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int batch = blockIdx.z;
  const int b0 = batch % p.nb0;
  const int b1 = batch / p.nb0;
  const long long m0 = (long long)blockIdx.y * TM;
  const long long n0 = (long long)blockIdx.x * TN;
  const int tx = threadIdx.x % 16;
  const int ty = threadIdx.x / 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int s = 0; s < p.nseg; ++s) {
    const float* A = reinterpret_cast<const float*>(p.seg[s].a) + p.as0 * b0 + p.as1 * b1;
    const float* B = reinterpret_cast<const float*>(p.seg[s].b) + p.bs0 * b0 + p.bs1 * b1;
    const long long K = p.seg[s].k;
    for (long long k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int idx = threadIdx.x + i * 256;
        if (!TA) {
          const int r = idx / TK, c = idx % TK;
          const long long m = m0 + r, k = k0 + c;
          As[c][r] = (m < p.M && k < K) ? A[m * p.lda + k] : 0.f;
        } else {
          const int r = idx / TM, c = idx % TM;
          const long long k = k0 + r, m = m0 + c;
          As[r][c] = (m < p.M && k < K) ? A[k * p.lda + m] : 0.f;
        }
        if (!TB) {
          const int r = idx / TN, c = idx % TN;
          const long long k = k0 + r, n = n0 + c;
          Bs[r][c] = (n < p.N && k < K) ? B[k * p.ldb + n] : 0.f;
        } else {
          const int r = idx / TK, c = idx % TK;
          const long long n = n0 + r, k = k0 + c;
          Bs[c][r] = (n < p.N && k < K) ? B[n * p.ldb + k] : 0.f;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

  float* C = reinterpret_cast<float*>(p.c) + p.cs0 * b0 + p.cs1 * b1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long m = m0 + ty * 4 + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const long long n = n0 + tx * 4 + j;
      if (n >= p.N) continue;
      float v = acc[i][j] * p.alpha;
      float* cp = C + m * p.ldc + n;
      switch (p.epi) {
        case (int)Epi::Accum: v += *cp; break;
        case (int)Epi::Resid:
          v += p.r[p.rs0 * b0 + p.rs1 * b1 + m * p.ldr + n];
          break;
        case (int)Epi::Gelu:
          p.z[p.zs0 * b0 + p.zs1 * b1 + m * p.ldz + n] = v;
          v = 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
          break;
        default: break;
      }
      *cp = v;
    }
  }
}

}  // namespace simt

namespace {
thread_local std::string g_simt_err;
}

cudaError_t gemm_f32_simt(const GemmDesc& d, cudaStream_t stream) {
  using namespace simt;
  if (d.in != DType::F32 || d.c_type != DType::F32) return cudaErrorInvalidValue;
  if (d.bias || d.drop_p > 0.f) return cudaErrorInvalidValue;  // tcgen05 epilogue only
  if (d.nseg < 1 || d.nseg > kMaxSegments) return cudaErrorInvalidValue;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  Params p;
  for (int s = 0; s < d.nseg; ++s) p.seg[s] = d.seg[s];
  p.nseg = d.nseg;
  p.M = d.M;
  p.N = d.N;
  p.nb0 = static_cast<int>(d.nb0);
  p.lda = d.lda;
  p.as0 = d.as0;
  p.as1 = d.as1;
  p.ldb = d.ldb;
  p.bs0 = d.bs0;
  p.bs1 = d.bs1;
  p.c = d.c;
  p.ldc = d.ldc;
  p.cs0 = d.cs0;
  p.cs1 = d.cs1;
  p.r = reinterpret_cast<const float*>(d.r);
  p.ldr = d.ldr;
  p.rs0 = d.rs0;
  p.rs1 = d.rs1;
  p.z = reinterpret_cast<float*>(d.z);
  p.ldz = d.ldz;
  p.zs0 = d.zs0;
  p.zs1 = d.zs1;
  p.alpha = d.alpha;
  p.epi = static_cast<int>(d.epi);
  dim3 grid((unsigned)((d.N + TN - 1) / TN), (unsigned)((d.M + TM - 1) / TM),
            (unsigned)(d.nb0 * d.nb1));
  if (!d.trans_a && !d.trans_b)
    gemm_f32_kernel<false, false><<<grid, 256, 0, stream>>>(p);
  else if (!d.trans_a && d.trans_b)
    gemm_f32_kernel<false, true><<<grid, 256, 0, stream>>>(p);
  else if (d.trans_a && !d.trans_b)
    gemm_f32_kernel<true, false><<<grid, 256, 0, stream>>>(p);
  else
    gemm_f32_kernel<true, true><<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t gemm(const GemmDesc& d, cudaStream_t stream) {
  if (d.in == DType::F32) return gemm_f32_simt(d, stream);
  if (d.in == DType::BF16) return gemm_bf16_sm100(d, stream);
  return cudaErrorInvalidValue;
}

}  // namespace tess
