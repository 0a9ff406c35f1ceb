// Memory-bound kernels: conversions, residual/bias adds, GeLU backward,
// LayerNorm (row-distributed statistics), softmax and its backward,
// deterministic column sums, and the slot-ordered sum used by the in-process
// communicator. Each replaces a CPU loop of the reference (file:line at the
// declaration in kernels.h).
#include <cuda_bf16.h>

#include "../core.h"
#include <algorithm>
#include <map>
#include <mutex>

#include "kernels.h"

namespace tess {

namespace {

constexpr int kBlock = 256;

int grid_for(size_t n, int per_thread = 1) {
  size_t blocks = (n + (size_t)kBlock * per_thread - 1) / ((size_t)kBlock * per_thread);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return static_cast<int>(blocks);
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p, size_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, size_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p, size_t i) {
  return __bfloat162float(p[i]);
}
template <>
__device__ __forceinline__ float ldf<double>(const double* p, size_t i) {
  return static_cast<float>(p[i]);
}

template <typename T>
__device__ __forceinline__ void stf(T* p, size_t i, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, size_t i, float v) {
  p[i] = v;
}
template <>
__device__ __forceinline__ void stf<__nv_bfloat16>(__nv_bfloat16* p, size_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ void stf<double>(double* p, size_t i, float v) {
  p[i] = v;
}

// Dispatch a functor templated on element type.
#define TESS_DISPATCH(dt, T, ...)                     \
  switch (dt) {                                       \
    case DType::F32: {                                \
      using T = float;                                \
      __VA_ARGS__;                                    \
      break;                                          \
    }                                                 \
    case DType::BF16: {                               \
      using T = __nv_bfloat16;                        \
      __VA_ARGS__;                                    \
      break;                                          \
    }                                                 \
    default:                                          \
      fail(TESS_ERR_INVALID, "unsupported dtype");    \
  }

__device__ __forceinline__ float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) t += red[w];  // fixed order: deterministic
  return t;
}

// ------------------------------------------------------------- convert
template <typename S, typename D>
__device__ __forceinline__ D cvt(S v);
template <> __device__ __forceinline__ float cvt<double, float>(double v) { return (float)v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<double, __nv_bfloat16>(double v) {
  return __double2bfloat16(v);
}
template <> __device__ __forceinline__ double cvt<float, double>(float v) { return v; }
template <> __device__ __forceinline__ double cvt<__nv_bfloat16, double>(__nv_bfloat16 v) {
  return (double)__bfloat162float(v);
}
template <> __device__ __forceinline__ __nv_bfloat16 cvt<float, __nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <> __device__ __forceinline__ float cvt<__nv_bfloat16, float>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> __device__ __forceinline__ float cvt<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double cvt<double, double>(double v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 v) {
  return v;
}

template <typename S, typename D>
__global__ void convert_kernel(const S* __restrict__ src, D* __restrict__ dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = cvt<S, D>(src[i]);
}

template <typename S>
void convert_from(const S* src, void* dst, DType dt, size_t n, cudaStream_t s) {
  const int g = grid_for(n);
  switch (dt) {
    case DType::F32:
      convert_kernel<S, float><<<g, kBlock, 0, s>>>(src, (float*)dst, n);
      break;
    case DType::BF16:
      convert_kernel<S, __nv_bfloat16><<<g, kBlock, 0, s>>>(src, (__nv_bfloat16*)dst, n);
      break;
    case DType::F64:
      convert_kernel<S, double><<<g, kBlock, 0, s>>>(src, (double*)dst, n);
      break;
  }
}

// ----------------------------------------------------------------- add
template <typename TA, typename TB, typename TO>
__global__ void add_kernel(const TA* a, const TB* b, TO* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    stf<TO>(out, i, ldf<TA>(a, i) + ldf<TB>(b, i));
}

template <typename T>
__global__ void bias_add_kernel(const T* x, const float* bias, T* out, int64_t rows,
                                int64_t cols) {
  const size_t n = (size_t)rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    stf<T>(out, i, ldf<T>(x, i) + bias[i % cols]);
}

template <typename T>
__global__ void gelu_bwd_kernel(const float* __restrict__ dh, const T* __restrict__ z,
                                T* __restrict__ dz, size_t n) {
  const float kInvSqrt2 = 0.70710678118654752f, kInvSqrt2Pi = 0.39894228040143268f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = ldf<T>(z, i);
    const float g = 0.5f * (1.0f + erff(v * kInvSqrt2)) + v * kInvSqrt2Pi * __expf(-0.5f * v * v);
    stf<T>(dz, i, dh[i] * g);
  }
}

// Column partial sums over row chunks: scratch[chunk][c] (+ optional second
// quantity for LayerNorm parameter gradients).
constexpr int kRowChunk = 64;

template <typename T>
__global__ void colsum_partial_kernel(const T* x, int64_t rows, int64_t cols, float* part) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * kRowChunk;
  if (c >= cols) return;
  float acc = 0.f;
  const int64_t r1 = min(rows, r0 + kRowChunk);
  for (int64_t r = r0; r < r1; ++r) acc += ldf<T>(x, r * cols + c);
  part[(int64_t)blockIdx.y * cols + c] = acc;
}

__global__ void colsum_finalize_kernel(const float* part, int64_t nchunk, int64_t cols,
                                       int64_t nq, float* out) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= cols * nq) return;
  const int64_t qi = c / cols, cc = c % cols;
  // four interleaved partial sums (fixed order: deterministic) keep several
  // independent loads in flight per thread
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  const float* pc = part + qi * cols + cc;
  const int64_t stride = nq * cols;
  int64_t k = 0;
  for (; k + 4 <= nchunk; k += 4) {
    a0 += pc[(k + 0) * stride];
    a1 += pc[(k + 1) * stride];
    a2 += pc[(k + 2) * stride];
    a3 += pc[(k + 3) * stride];
  }
  for (; k < nchunk; ++k) a0 += pc[k * stride];
  out[c] = (a0 + a1) + (a2 + a3);
}

// ------------------------------------------------------------ LayerNorm
template <typename T>
__global__ void ln_stats_kernel(const T* __restrict__ x, int64_t w, float* __restrict__ stats) {
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const T* row = x + r * w;
  float s = 0.f;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) s += ldf<T>(row, c);
  s = block_sum(s, red);
  const float mu = s / (float)w;
  float m2 = 0.f;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    const float dv = ldf<T>(row, c) - mu;
    m2 += dv * dv;
  }
  m2 = block_sum(m2, red);
  if (threadIdx.x == 0) {
    stats[3 * r + 0] = s;
    stats[3 * r + 1] = m2;
    stats[3 * r + 2] = (float)w * mu * mu;
  }
}

template <typename T>
__global__ void ln_apply_kernel(const T* __restrict__ x, const float* __restrict__ stats,
                                int64_t w, float n, const float* __restrict__ gain,
                                const float* __restrict__ bias, float eps, T* __restrict__ y,
                                float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  const int64_t r = blockIdx.x;
  const float s0 = stats[3 * r], s1 = stats[3 * r + 1], s2 = stats[3 * r + 2];
  const float mean = s0 / n;
  float var = (s1 + (s2 - n * mean * mean)) / n;
  if (var < 0.f) var = 0.f;
  const float rstd = 1.0f / sqrtf(var + eps);
  const T* row = x + r * w;
  T* yrow = y + r * w;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x)
    stf<T>(yrow, c, gain[c] * ((ldf<T>(row, c) - mean) * rstd) + bias[c]);
  if (threadIdx.x == 0) {
    mean_out[r] = mean;
    rstd_out[r] = rstd;
  }
}

template <typename TD, typename TX>
__global__ void ln_bwd_stats_kernel(const TD* __restrict__ dy, const TX* __restrict__ x,
                                    const float* __restrict__ mean, const float* __restrict__ rstd,
                                    const float* __restrict__ gain, int64_t w,
                                    float* __restrict__ stats) {
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const float mu = mean[r], rs = rstd[r];
  float a = 0.f, b = 0.f;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    const float dxh = ldf<TD>(dy, r * w + c) * gain[c];
    const float xh = (ldf<TX>(x, r * w + c) - mu) * rs;
    a += dxh;
    b += xh * dxh;
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    stats[2 * r] = a;
    stats[2 * r + 1] = b;
  }
}

template <typename TD, typename TX, typename TR, typename TO>
__global__ void ln_bwd_apply_kernel(const TD* __restrict__ dy, const TX* __restrict__ x,
                                    const float* __restrict__ mean, const float* __restrict__ rstd,
                                    const float* __restrict__ gain, const float* __restrict__ stats,
                                    int64_t w, float n, const TR* __restrict__ resid,
                                    TO* __restrict__ dx) {
  const int64_t r = blockIdx.x;
  const float mu = mean[r], rs = rstd[r];
  const float md = stats[2 * r] / n, mxd = stats[2 * r + 1] / n;
  for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
    const size_t i = r * w + c;
    const float dxh = ldf<TD>(dy, i) * gain[c];
    const float xh = (ldf<TX>(x, i) - mu) * rs;
    float v = rs * (dxh - md - xh * mxd);
    if (resid) v += ldf<TR>(resid, i);
    stf<TO>(dx, i, v);
  }
}

template <typename TD, typename TX>
__global__ void ln_params_partial_kernel(const TD* dy, const TX* x, const float* mean,
                                         const float* rstd, int64_t rows, int64_t w,
                                         float* part) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * kRowChunk;
  if (c >= w) return;
  float dg = 0.f, db = 0.f;
  const int64_t r1 = min(rows, r0 + kRowChunk);
  for (int64_t r = r0; r < r1; ++r) {
    const float d = ldf<TD>(dy, r * w + c);
    dg += d * (ldf<TX>(x, r * w + c) - mean[r]) * rstd[r];
    db += d;
  }
  part[((int64_t)blockIdx.y * 2 + 0) * w + c] = dg;
  part[((int64_t)blockIdx.y * 2 + 1) * w + c] = db;
}

// ---- vectorised LayerNorm (ref layers.cpp:242-345) --------------------------
// A block owns whole rows, register-resident: thread t holds columns
// [t*8 + v*span, +8) for v < NV (span = 8 * blockDim.x, w = NV * span),
// loaded with 16-byte vectors. Two forms:
//  * fused (q == 1: the row all-reduce moves nothing): statistics + apply
//    (forward), statistics + dx + dgain/dbias partials (backward) in ONE pass
//    over HBM;
//  * split (q > 1): a partial pass writes per-row partials (forward
//    [sum x, M2, n*mean^2] of the local columns; backward [sum dxhat,
//    sum xhat*dxhat] plus the dgain/dbias column partials), the row group
//    all-reduces them, and an apply pass finishes the rows: 2 reads of x and
//    1 write forward, 2 reads of dy / x and 1 write backward.
// Supported widths: w = NV * 8 * threads, NV <= 4, threads a multiple of 32
// in [128, 1024] (ln_vec_config): 2048 ... 32768 in steps the hidden sizes
// of the configs hit (4096 * k, 6144, 3072, 2048, ...).
constexpr int kLnMaxThreads = 1024;



__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&v)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void st8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// 8 values held as raw 16-byte vectors (bf16: one uint4, fp32: two) -> floats.
__device__ __forceinline__ void unpack8(const uint4 (&u)[1], float (&v)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[0]);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(h[e]);
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}
__device__ __forceinline__ void unpack8(const uint4 (&u)[2], float (&v)[8]) {
  v[0] = __uint_as_float(u[0].x); v[1] = __uint_as_float(u[0].y);
  v[2] = __uint_as_float(u[0].z); v[3] = __uint_as_float(u[0].w);
  v[4] = __uint_as_float(u[1].x); v[5] = __uint_as_float(u[1].y);
  v[6] = __uint_as_float(u[1].z); v[7] = __uint_as_float(u[1].w);
}

// Deterministic block sums of two values: warp butterflies, then the warps'
// partials summed by one more butterfly over lanes [0, nw). Every thread
// gets the same (bitwise) result: a butterfly combines v_l + v_(l^o), which
// commutes. TH: compile-time block size (0 = blockDim.x).
template <int TH>
__device__ __forceinline__ float2 block_sum2(float a, float b, float2* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (TH ? TH : (int)blockDim.x) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();  // red is reused row after row
  if (lane == 0) red[warp] = make_float2(a, b);
  __syncthreads();
  float2 t = lane < nw ? red[lane] : make_float2(0.f, 0.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t.x += __shfl_xor_sync(0xffffffffu, t.x, o);
    t.y += __shfl_xor_sync(0xffffffffu, t.y, o);
  }
  return t;
}

// Deterministic block (mean, M2) of equal-count (n) per-thread partials:
// Chan's pairwise combination in a warp butterfly (symmetric, so every lane
// holds the same pair), then across the nw warps the exact two-level form
// mean = avg(m_w), M2 = sum M2_w + n_w sum (m_w - mean)^2, each sum a lane
// butterfly -- no E[x^2] - E[x]^2 anywhere, so a row whose mean is large
// against its spread (or an outlier element) does not cancel, and no
// division sits in the per-row dependency chain.
template <int TH>
__device__ __forceinline__ float2 block_meanvar(float m, float M2, float n, float2* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (TH ? TH : (int)blockDim.x) >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, o);
    const float Mo = __shfl_xor_sync(0xffffffffu, M2, o);
    const float dlt = mo - m;
    M2 = M2 + Mo + dlt * dlt * (0.5f * n);
    m = 0.5f * (m + mo);
    n *= 2.f;
  }
  __syncthreads();  // red is reused row after row
  if (lane == 0) red[warp] = make_float2(m, M2);
  __syncthreads();
  const float2 w = lane < nw ? red[lane] : make_float2(0.f, 0.f);
  float sm = w.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  const float mean = sm * (TH ? 1.0f / (float)(TH >> 5) : __frcp_rn((float)nw));
  const float dl = lane < nw ? w.x - mean : 0.f;
  float m2 = lane < nw ? fmaf(n * dl, dl, w.y) : 0.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m2 += __shfl_xor_sync(0xffffffffu, m2, o);
  return make_float2(mean, m2);
}

// Row mean / M2 of the register-resident slice (every thread gets the pair).
template <int NV, int TH>
__device__ __forceinline__ float2 row_meanvar(const float (&v)[NV][8], float2* red) {
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) s += v[k][e];
  constexpr float kN = (float)(NV * 8);
  const float lm = s / kN;
  float m2 = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = v[k][e] - lm;
      m2 = fmaf(d, d, m2);
    }
  return block_meanvar<TH>(lm, m2, kN, red);
}

// SPLIT = false: y = LN(x) with the row's own statistics (q == 1).
// SPLIT = true: stats[3r..] = (sum x, M2, n mean^2) of the local columns, the
// row group's all-reduce sums them (ln_vec_apply_kernel combines).
// TH: compile-time block size (0 = blockDim.x; the launchers use 512 for
// widths that are multiples of 4096, cfg4's 12288 among them).
template <typename T, int NV, bool SPLIT, int TH>
__global__ void __launch_bounds__(NV == 1 ? kLnMaxThreads : 512) ln_vec_fwd_kernel(
    const T* __restrict__ x, int64_t rows, const float* __restrict__ gain,
    const float* __restrict__ bias, float eps, T* __restrict__ y, float* __restrict__ mean_out,
    float* __restrict__ rstd_out, float* __restrict__ stats) {
  __shared__ float2 red[32];
  const int span = (TH ? TH : (int)blockDim.x) * 8;
  const int w = NV * span;
  const int c0 = threadIdx.x * 8;
  // the thread's gain / bias columns are the same for every row: registers
  // (one 512-thread block per SM then, but with the next row in flight:
  // 0.282 -> 0.237 ms per step for the two launches, r2_ln_fwd_prefetch_ab.log)
  float g[NV][8], b[NV][8];
  if (!SPLIT) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      ld8(gain + c0 + k * span, g[k]);
      ld8(bias + c0 + k * span, b[k]);
    }
  }
  // raw 16-byte vectors of the next row are loaded before this row's
  // reduction, so the HBM latency of row r+grid overlaps row r's work
  constexpr int RV = sizeof(T) / 2;  // uint4 per 8 elements
  uint4 nxt[NV][RV];
  auto load_raw = [&](int64_t rr) {
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int u = 0; u < RV; ++u)
        nxt[k][u] = __ldg(reinterpret_cast<const uint4*>(x + rr * w + c0 + k * span) + u);
  };
  if (blockIdx.x < rows) load_raw(blockIdx.x);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float v[NV][8];
#pragma unroll
    for (int k = 0; k < NV; ++k) unpack8(nxt[k], v[k]);
    if (r + gridDim.x < rows) load_raw(r + gridDim.x);
    const float2 t = row_meanvar<NV, TH>(v, red);
    if (SPLIT) {
      if (threadIdx.x == 0) {
        stats[3 * r + 0] = t.x * (float)w;
        stats[3 * r + 1] = t.y;
        stats[3 * r + 2] = (float)w * t.x * t.x;
      }
      continue;
    }
    const float mu = t.x;
    const float var = fmaxf(t.y / (float)w, 0.f);
    const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = g[k][e] * ((v[k][e] - mu) * rstd) + b[k][e];
      st8(y + r * w + c0 + k * span, o);
    }
    if (threadIdx.x == 0) {
      mean_out[r] = mu;
      rstd_out[r] = rstd;
    }
  }
}

// Apply with the row group's summed partials (n = hidden_total):
// mean = sum/n, var = (sum M2 + (sum n_g mean_g^2 - n mean^2)) / n.
template <typename T, int NV>
__global__ void __launch_bounds__(NV == 1 ? kLnMaxThreads : 512) ln_vec_apply_kernel(
    const T* __restrict__ x, const float* __restrict__ stats, int64_t rows, float n,
    const float* __restrict__ gain, const float* __restrict__ bias, float eps, T* __restrict__ y,
    float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  const int span = blockDim.x * 8;
  const int w = NV * span;
  const int c0 = threadIdx.x * 8;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    float v[NV][8];
#pragma unroll
    for (int k = 0; k < NV; ++k) ld8(x + r * w + c0 + k * span, v[k]);
    const float s0 = stats[3 * r], s1 = stats[3 * r + 1], s2 = stats[3 * r + 2];
    const float mu = s0 / n;
    const float var = fmaxf((s1 + (s2 - n * mu * mu)) / n, 0.f);
    const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float g[8], b[8], o[8];
      ld8(gain + c0 + k * span, g);
      ld8(bias + c0 + k * span, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = g[e] * ((v[k][e] - mu) * rstd) + b[e];
      st8(y + r * w + c0 + k * span, o);
    }
    if (threadIdx.x == 0) {
      mean_out[r] = mu;
      rstd_out[r] = rstd;
    }
  }
}

// Backward. SPLIT = false (q == 1): dx = rstd * (dxhat - mean(dxhat) - xhat *
// mean(xhat*dxhat)) (+ resid) with the row's own sums. SPLIT = true: only
// the row partials stats[2r..] = (sum dxhat, sum xhat*dxhat) over the local
// columns (ln_vec_bwd_apply_kernel finishes after the row all-reduce). Both
// add this block's dgain = sum dy*xhat, dbias = sum dy column partials to
// part[block][2][w] (summed over blocks in fixed order afterwards).
template <typename TD, typename TX, typename TR, typename TO, int NV, bool SPLIT, int TH>
__global__ void __launch_bounds__(NV == 1 ? kLnMaxThreads : 512) ln_vec_bwd_kernel(
    const TD* __restrict__ dy, const TX* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gain, int64_t rows,
    const TR* __restrict__ resid, TO* __restrict__ dx, float* __restrict__ part,
    float* __restrict__ stats) {
  __shared__ float2 red[32];
  const int span = (TH ? TH : (int)blockDim.x) * 8;
  const int w = NV * span;
  const int c0 = threadIdx.x * 8;
  float dg[NV][8], db[NV][8];  // gain is re-read per row (L1-resident) to save registers
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) dg[k][e] = db[k][e] = 0.f;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float mu = mean[r], rs = rstd[r];
    float d[NV][8], xh[NV][8];
    float a = 0.f, b = 0.f;
    // the residual is loaded with dy / x (raw 16-byte vectors), not after
    // the block reduction: one HBM round trip per row instead of two
    uint4 rr[NV][sizeof(TR) / 2];
    if (!SPLIT && resid) {
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int u = 0; u < (int)(sizeof(TR) / 2); ++u)
          rr[k][u] = __ldg(reinterpret_cast<const uint4*>(resid + r * w + c0 + k * span) + u);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float g[8];
      ld8(dy + r * w + c0 + k * span, d[k]);
      ld8(x + r * w + c0 + k * span, xh[k]);
      ld8(gain + c0 + k * span, g);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[k][e] = (xh[k][e] - mu) * rs;
        const float dxh = d[k][e] * g[e];
        a += dxh;
        b += xh[k][e] * dxh;
        dg[k][e] += d[k][e] * xh[k][e];
        db[k][e] += d[k][e];
        d[k][e] = dxh;  // only dy * gain is needed from here on
      }
    }
    const float2 t = block_sum2<TH>(a, b, red);
    if (SPLIT) {
      if (threadIdx.x == 0) {
        stats[2 * r] = t.x;
        stats[2 * r + 1] = t.y;
      }
      continue;
    }
    const float md = t.x / (float)w, mxd = t.y / (float)w;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float o[8];
      if (resid) unpack8(rr[k], o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v = rs * (d[k][e] - md - xh[k][e] * mxd);
        o[e] = resid ? o[e] + v : v;
      }
      st8(dx + r * w + c0 + k * span, o);
    }
  }
  if (part) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      st8(part + ((int64_t)blockIdx.x * 2 + 0) * w + c0 + k * span, dg[k]);
      st8(part + ((int64_t)blockIdx.x * 2 + 1) * w + c0 + k * span, db[k]);
    }
  }
}

// dx from the row group's summed (sum dxhat, sum xhat*dxhat), n = hidden_total.
template <typename TD, typename TX, typename TR, typename TO, int NV>
__global__ void __launch_bounds__(NV == 1 ? kLnMaxThreads : 512) ln_vec_bwd_apply_kernel(
    const TD* __restrict__ dy, const TX* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const float* __restrict__ gain,
    const float* __restrict__ stats, int64_t rows, float n, const TR* __restrict__ resid,
    TO* __restrict__ dx) {
  const int span = blockDim.x * 8;
  const int w = NV * span;
  const int c0 = threadIdx.x * 8;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float mu = mean[r], rs = rstd[r];
    const float md = stats[2 * r] / n, mxd = stats[2 * r + 1] / n;
    uint4 rr[NV][sizeof(TR) / 2];
    if (resid) {
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int u = 0; u < (int)(sizeof(TR) / 2); ++u)
          rr[k][u] = __ldg(reinterpret_cast<const uint4*>(resid + r * w + c0 + k * span) + u);
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float d[8], xv[8], g[8], o[8];
      ld8(dy + r * w + c0 + k * span, d);
      ld8(x + r * w + c0 + k * span, xv);
      ld8(gain + c0 + k * span, g);
      if (resid) unpack8(rr[k], o);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (xv[e] - mu) * rs;
        const float v = rs * (d[e] * g[e] - md - xh * mxd);
        o[e] = resid ? o[e] + v : v;
      }
      st8(dx + r * w + c0 + k * span, o);
    }
  }
}

// ------------------------------------------------------------- softmax
// One warp per row; rows cached in registers when L % 4 == 0 and L <= 128*NV.
template <typename T, int NV>
__global__ void softmax_fwd_reg_kernel(const float* __restrict__ S, T* __restrict__ P,
                                       int64_t rows, int64_t L) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float4* srow = reinterpret_cast<const float4*>(S + r * L);
  const int nv = static_cast<int>(L / 4);
  float4 v[NV];
  float mx = -INFINITY;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int idx = lane + k * 32;
    if (idx < nv) {
      v[k] = srow[idx];
      mx = fmaxf(mx, fmaxf(fmaxf(v[k].x, v[k].y), fmaxf(v[k].z, v[k].w)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int idx = lane + k * 32;
    if (idx < nv) {
      v[k].x = __expf(v[k].x - mx);
      v[k].y = __expf(v[k].y - mx);
      v[k].z = __expf(v[k].z - mx);
      v[k].w = __expf(v[k].w - mx);
      sum += (v[k].x + v[k].y) + (v[k].z + v[k].w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.0f / sum;
  T* prow = P + r * L;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int idx = lane + k * 32;
    if (idx < nv) {
      stf<T>(prow, 4 * idx + 0, v[k].x * inv);
      stf<T>(prow, 4 * idx + 1, v[k].y * inv);
      stf<T>(prow, 4 * idx + 2, v[k].z * inv);
      stf<T>(prow, 4 * idx + 3, v[k].w * inv);
    }
  }
}

template <typename T>
__global__ void softmax_fwd_generic_kernel(const float* __restrict__ S, T* __restrict__ P,
                                           int64_t rows, int64_t L) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* srow = S + r * L;
  float mx = -INFINITY;
  for (int64_t c = lane; c < L; c += 32) mx = fmaxf(mx, srow[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (int64_t c = lane; c < L; c += 32) sum += __expf(srow[c] - mx);
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float inv = 1.0f / sum;
  for (int64_t c = lane; c < L; c += 32) stf<T>(P + r * L, c, __expf(srow[c] - mx) * inv);
}

template <typename T>
__global__ void softmax_bwd_kernel(const T* __restrict__ P, const float* __restrict__ dP,
                                   T* __restrict__ dS, int64_t rows, int64_t L, float scale) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* prow = P + r * L;
  const float* drow = dP + r * L;
  float dot = 0.f;
  for (int64_t c = lane; c < L; c += 32) dot += ldf<T>(prow, c) * drow[c];
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  for (int64_t c = lane; c < L; c += 32) {
    const float p = ldf<T>(prow, c);
    stf<T>(dS + r * L, c, scale * p * (drow[c] - dot));
  }
}

__global__ void lse_combine_kernel(const float2* __restrict__ stats, int64_t rows, int nst,
                                   float* __restrict__ lse) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  // partials are (max, sum) in log2 units (RowStats epilogue); so is lse
  const float2* s = stats + r * nst;
  float m = -INFINITY;
  for (int i = 0; i < nst; ++i) m = fmaxf(m, s[i].x);
  float sum = 0.f;
  for (int i = 0; i < nst; ++i)
    if (s[i].x != -INFINITY) sum += s[i].y * exp2f(s[i].x - m);
  lse[r] = m + log2f(sum);
}

// one warp per (row, head)
template <typename T>
__global__ void attn_delta_kernel(const T* __restrict__ dO, const T* __restrict__ O, int64_t ld,
                                  int64_t S, int64_t H, int64_t hd, float* __restrict__ delta) {
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (w >= S * H) return;
  const int64_t r = w / H, h = w % H;
  const T* a = dO + r * ld + h * hd;
  const T* b = O + r * ld + h * hd;
  float acc = 0.f;
  for (int64_t d = lane; d < hd; d += 32) acc += ldf<T>(a, d) * ldf<T>(b, d);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) delta[h * S + r] = acc;
}

// Vectorised delta for bf16 with hd % 8 == 0 and 32 % (hd / 8) == 0: a group
// of hd/8 lanes per (row, head), one 16-byte load of dO and of O per lane,
// all samples in one launch (rows = samples * S; delta[(smp*H + h)*S + r]).
template <int LPG>
__global__ void attn_delta_vec_kernel(const __nv_bfloat16* __restrict__ dO,
                                      const __nv_bfloat16* __restrict__ O, int64_t ld, int64_t S,
                                      int64_t H, int64_t rows, float* __restrict__ delta) {
  constexpr int kGroups = 32 / LPG;
  const int lane = threadIdx.x & 31;
  const int64_t item = (blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32) * kGroups +
                       lane / LPG;  // (row, head) pair
  const int sub = lane % LPG;
  float acc = 0.f;
  const bool ok = item < rows * H;
  int64_t ri = 0, h = 0;
  if (ok) {
    ri = item / H;
    h = item % H;
    const int64_t off = ri * ld + h * (LPG * 8) + sub * 8;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(dO + off));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(O + off));
    const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __bfloat1622float2(a2[e]), y = __bfloat1622float2(b2[e]);
      acc = fmaf(x.x, y.x, acc);
      acc = fmaf(x.y, y.y, acc);
    }
  }
#pragma unroll
  for (int o = LPG / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (ok && sub == 0) {
    const int64_t smp = ri / S, r = ri % S;
    delta[(smp * H + h) * S + r] = acc;
  }
}

// --------------------------------------------------------- toy training
constexpr int kMseBlocks = 1024;

template <typename T>
__global__ void mse_grad_kernel(const T* __restrict__ y, const T* __restrict__ t, size_t n,
                                float scale, T* __restrict__ dy, double* __restrict__ part) {
  __shared__ double red[kBlock];
  double acc = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float d = ldf<T>(y, i) - ldf<T>(t, i);
    acc += (double)d * d;
    stf<T>(dy, i, scale * d);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void sum_doubles_kernel(const double* part, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];  // fixed order: deterministic
    *out = s;
  }
}

template <typename T>
__global__ void sgd_kernel(T* w, float* master, const float* g, float lr, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    if (master) {
      master[i] -= lr * g[i];
      stf<T>(w, i, master[i]);
    } else {
      stf<T>(w, i, ldf<T>(w, i) - lr * g[i]);
    }
  }
}

// ------------------------------------------------------- comm helper
struct SumArgs {
  const float* in[8];
};

__global__ void sum_kernel(SumArgs a, int n_in, float* out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    float acc = a.in[0][i];
    for (int k = 1; k < n_in; ++k) acc += a.in[k][i];  // slot-ascending
    out[i] = acc;
  }
}

}  // namespace

std::atomic<uint64_t> g_launches{0};

void launch_sum_f32(const float* const* in, int n_in, float* out, size_t n, cudaStream_t s) {
  SumArgs a;
  for (int k = 0; k < n_in && k < 8; ++k) a.in[k] = in[k];
  sum_kernel<<<grid_for(n), kBlock, 0, s>>>(a, n_in, out, n);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_convert(const void* src, DType st, void* dst, DType dt, size_t n, cudaStream_t s) {
  if (!n) return;
  switch (st) {
    case DType::F32: convert_from((const float*)src, dst, dt, n, s); break;
    case DType::BF16: convert_from((const __nv_bfloat16*)src, dst, dt, n, s); break;
    case DType::F64: convert_from((const double*)src, dst, dt, n, s); break;
  }
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_add(const void* a, DType ta, const void* b, DType tb, void* out, DType to, size_t n,
           cudaStream_t s) {
  if (!n) return;
  const int g = grid_for(n);
  TESS_DISPATCH(ta, TA, TESS_DISPATCH(tb, TB, TESS_DISPATCH(to, TO,
      add_kernel<TA, TB, TO><<<g, kBlock, 0, s>>>((const TA*)a, (const TB*)b, (TO*)out, n))));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_bias_add(const void* x, const float* bias, void* out, DType t, int64_t rows,
                int64_t cols, cudaStream_t s) {
  const size_t n = (size_t)rows * cols;
  if (!n) return;
  TESS_DISPATCH(t, T, bias_add_kernel<T><<<grid_for(n), kBlock, 0, s>>>((const T*)x, bias,
                                                                          (T*)out, rows, cols));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_gelu_bwd(const float* dh, const void* z, void* dz, DType t, size_t n, cudaStream_t s) {
  if (!n) return;
  TESS_DISPATCH(t, T, gelu_bwd_kernel<T><<<grid_for(n), kBlock, 0, s>>>(dh, (const T*)z,
                                                                          (T*)dz, n));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

size_t k_colsum_scratch_floats(int64_t rows, int64_t cols) {
  return (size_t)((rows + kRowChunk - 1) / kRowChunk) * cols;
}

void k_colsum(const void* x, DType t, int64_t rows, int64_t cols, float* out, float* scratch,
              cudaStream_t s) {
  if (cols <= 0) return;
  const int64_t nchunk = (rows + kRowChunk - 1) / kRowChunk;
  if (nchunk == 0) {
    TESS_CUDA(cudaMemsetAsync(out, 0, cols * 4, s));
    return;
  }
  dim3 g((unsigned)((cols + kBlock - 1) / kBlock), (unsigned)nchunk);
  TESS_DISPATCH(t, T, colsum_partial_kernel<T><<<g, kBlock, 0, s>>>((const T*)x, rows, cols,
                                                                      scratch));
  colsum_finalize_kernel<<<(unsigned)((cols + kBlock - 1) / kBlock), kBlock, 0, s>>>(
      scratch, nchunk, cols, 1, out);
  count_launch(2);
  TESS_CUDA(cudaGetLastError());
}

void k_ln_stats(const void* x, DType t, int64_t rows, int64_t w, float* stats, cudaStream_t s) {
  if (!rows) return;
  TESS_DISPATCH(t, T, ln_stats_kernel<T><<<(unsigned)rows, kBlock, 0, s>>>((const T*)x, w, stats));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_apply(const void* x, DType t, const float* stats, int64_t rows, int64_t w,
                double hidden_total, const float* gain, const float* bias, double eps, void* y,
                float* mean, float* rstd, cudaStream_t s) {
  if (!rows) return;
  TESS_DISPATCH(t, T, ln_apply_kernel<T><<<(unsigned)rows, kBlock, 0, s>>>(
                          (const T*)x, stats, w, (float)hidden_total, gain, bias, (float)eps,
                          (T*)y, mean, rstd));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_bwd_stats(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, int64_t rows, int64_t w, float* stats,
                    cudaStream_t s) {
  if (!rows) return;
  TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX,
      ln_bwd_stats_kernel<TD, TX><<<(unsigned)rows, kBlock, 0, s>>>(
          (const TD*)dy, (const TX*)x, mean, rstd, gain, w, stats)));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_bwd_apply(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, const float* stats, int64_t rows,
                    int64_t w, double hidden_total, const void* resid, DType tr, void* dx,
                    DType to, cudaStream_t s) {
  if (!rows) return;
  TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX, TESS_DISPATCH(tr, TR, TESS_DISPATCH(to, TO,
      ln_bwd_apply_kernel<TD, TX, TR, TO><<<(unsigned)rows, kBlock, 0, s>>>(
          (const TD*)dy, (const TX*)x, mean, rstd, gain, stats, w, (float)hidden_total,
          (const TR*)resid, (TO*)dx)))));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

size_t k_ln_params_scratch_floats(int64_t rows, int64_t w) {
  return (size_t)((rows + kRowChunk - 1) / kRowChunk) * 2 * w;
}

void k_ln_bwd_params(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                     const float* rstd, int64_t rows, int64_t w, float* out2w, float* scratch,
                     cudaStream_t s) {
  const int64_t nchunk = (rows + kRowChunk - 1) / kRowChunk;
  if (nchunk == 0) {
    TESS_CUDA(cudaMemsetAsync(out2w, 0, 2 * w * 4, s));
    return;
  }
  dim3 g((unsigned)((w + kBlock - 1) / kBlock), (unsigned)nchunk);
  TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX,
      ln_params_partial_kernel<TD, TX><<<g, kBlock, 0, s>>>((const TD*)dy, (const TX*)x, mean,
                                                            rstd, rows, w, scratch)));
  colsum_finalize_kernel<<<(unsigned)((2 * w + kBlock - 1) / kBlock), kBlock, 0, s>>>(
      scratch, nchunk, w, 2, out2w);
  count_launch(2);
  TESS_CUDA(cudaGetLastError());
}

void k_softmax_fwd(const float* S, void* P, DType t, int64_t rows, int64_t L, cudaStream_t s) {
  if (!rows) return;
  const int warps = 8;
  const unsigned g = (unsigned)((rows + warps - 1) / warps);
  if (L % 4 == 0 && L <= 128 * 16) {
    TESS_DISPATCH(t, T, softmax_fwd_reg_kernel<T, 16><<<g, 32 * warps, 0, s>>>(S, (T*)P, rows, L));
  } else if (L % 4 == 0 && L <= 128 * 32) {
    TESS_DISPATCH(t, T, softmax_fwd_reg_kernel<T, 32><<<g, 32 * warps, 0, s>>>(S, (T*)P, rows, L));
  } else {
    TESS_DISPATCH(t, T, softmax_fwd_generic_kernel<T><<<g, 32 * warps, 0, s>>>(S, (T*)P, rows, L));
  }
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

size_t k_mse_scratch_doubles(size_t) { return kMseBlocks; }

void k_mse_grad(const void* y, const void* target, DType t, size_t n, double denom, void* dy,
                double* sum, double* scratch, cudaStream_t s) {
  const float scale = (float)(2.0 / denom);
  TESS_DISPATCH(t, T, mse_grad_kernel<T><<<kMseBlocks, kBlock, 0, s>>>(
                          (const T*)y, (const T*)target, n, scale, (T*)dy, scratch));
  sum_doubles_kernel<<<1, 32, 0, s>>>(scratch, kMseBlocks, sum);
  count_launch(2);
  TESS_CUDA(cudaGetLastError());
}

void k_sgd(void* w, DType t, float* master, const float* g, double lr, size_t n, cudaStream_t s) {
  if (!n) return;
  TESS_DISPATCH(t, T, sgd_kernel<T><<<grid_for(n), kBlock, 0, s>>>((T*)w, master, g, (float)lr, n));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_lse_combine(const float* stats, int64_t rows, int nst, float* lse, cudaStream_t s) {
  if (!rows) return;
  lse_combine_kernel<<<(unsigned)((rows + kBlock - 1) / kBlock), kBlock, 0, s>>>(
      reinterpret_cast<const float2*>(stats), rows, nst, lse);
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_attn_delta(const void* dO, const void* O, DType t, int64_t ld, int64_t S, int64_t H,
                  int64_t hd, float* delta, cudaStream_t s, int64_t samples) {
  if (!S || !H || !samples) return;
  const int warps = 8;
  const bool vec = t == DType::BF16 && (hd == 128 || hd == 64 || hd == 32) && ld % 8 == 0 &&
                   reinterpret_cast<uintptr_t>(dO) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(O) % 16 == 0;
  if (vec) {
    const int64_t items = samples * S * H;
    const int lpg = (int)(hd / 8), per_block = warps * (32 / lpg);
    const unsigned g = (unsigned)((items + per_block - 1) / per_block);
    const auto* a = static_cast<const __nv_bfloat16*>(dO);
    const auto* b = static_cast<const __nv_bfloat16*>(O);
    if (lpg == 16)
      attn_delta_vec_kernel<16><<<g, 32 * warps, 0, s>>>(a, b, ld, S, H, samples * S, delta);
    else if (lpg == 8)
      attn_delta_vec_kernel<8><<<g, 32 * warps, 0, s>>>(a, b, ld, S, H, samples * S, delta);
    else
      attn_delta_vec_kernel<4><<<g, 32 * warps, 0, s>>>(a, b, ld, S, H, samples * S, delta);
    count_launch();
    TESS_CUDA(cudaGetLastError());
    return;
  }
  const unsigned g = (unsigned)((S * H + warps - 1) / warps);
  const size_t esz = dtype_size(t);
  for (int64_t smp = 0; smp < samples; ++smp) {
    const char* a = static_cast<const char*>(dO) + (size_t)smp * S * ld * esz;
    const char* b = static_cast<const char*>(O) + (size_t)smp * S * ld * esz;
    TESS_DISPATCH(t, T, attn_delta_kernel<T><<<g, 32 * warps, 0, s>>>(
                            (const T*)a, (const T*)b, ld, S, H, hd, delta + (size_t)smp * H * S));
    count_launch();
  }
  TESS_CUDA(cudaGetLastError());
}

void k_softmax_bwd(const void* P, const float* dP, void* dS, DType t, int64_t rows, int64_t L,
                   float scale, cudaStream_t s) {
  if (!rows) return;
  const int warps = 8;
  const unsigned g = (unsigned)((rows + warps - 1) / warps);
  TESS_DISPATCH(t, T, softmax_bwd_kernel<T><<<g, 32 * warps, 0, s>>>((const T*)P, dP, (T*)dS,
                                                                       rows, L, scale));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}


// ---- vectorised LayerNorm launchers ------------------------------------------
struct LnCfg {
  int nv = 0, threads = 0;
};

// w = nv * 8 * threads. Widths that are multiples of 4096 keep 512-thread
// blocks (the measured configuration at cfg4's 12288); others take the
// fewest passes whose block is a whole number of warps in [128, 1024].
LnCfg ln_vec_config(int64_t w) {
  LnCfg c;
  if (w <= 0 || w % 8 != 0) return c;
  if (w % 4096 == 0 && w / 4096 <= 4) return {(int)(w / 4096), 512};
  for (int nv = 1; nv <= 4; ++nv) {
    if (w % (8 * nv) != 0) continue;
    const int64_t t = w / (8 * nv);
    // registers: one pass fits 1024 threads, several passes at most 512
    if (t % 32 == 0 && t >= 128 && t <= (nv == 1 ? kLnMaxThreads : 512)) return {nv, (int)t};
  }
  return c;
}

bool ln_vec_ok(int64_t w, std::initializer_list<const void*> ptrs) {
  if (ln_vec_config(w).nv == 0) return false;
  for (const void* p : ptrs)
    if (p && reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
  return true;
}

// Blocks: up to 2048 resident threads per SM; the backward (whose blocks
// each write a [2, w] dgain/dbias partial) at most 2 blocks per SM. Upper
// bound for the partial scratch; the launch grid is the resident count.
int ln_vec_blocks(int64_t rows, int threads, int per_sm_cap) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int per_sm = std::max(1, std::min(per_sm_cap, 2048 / threads));
  const int64_t b = std::min<int64_t>(rows, (int64_t)sms * per_sm);
  return (int)std::max<int64_t>(b, 1);
}

// Grid of a row-looping LayerNorm kernel: the blocks that are resident at
// once (registers bound the 512-thread blocks to 1-2 per SM), capped by
// per_sm_cap and rows -- a second partial wave of blocks would run its rows
// after the first wave instead of beside it.
int ln_grid(const void* fn, int threads, int64_t rows, int per_sm_cap) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> occ;
  int per = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ.find({fn, threads});
    if (it == occ.end()) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, 0) != cudaSuccess) {
        cudaGetLastError();
        per = 1;
      }
      occ[{fn, threads}] = per;
    } else {
      per = it->second;
    }
  }
  return ln_vec_blocks(rows, threads, std::max(1, std::min(per, per_sm_cap)));
}

#define TESS_LN_TH(threads, ...)                                                   \
  if ((threads) == 512) {                                                          \
    constexpr int TH = 512;                                                        \
    __VA_ARGS__;                                                                   \
  } else {                                                                         \
    constexpr int TH = 0;                                                          \
    __VA_ARGS__;                                                                   \
  }

bool k_ln_fused_supported(int64_t w) { return ln_vec_config(w).nv > 0; }

size_t k_ln_fused_scratch_floats(int64_t rows, int64_t w) {
  const LnCfg c = ln_vec_config(w);
  return (size_t)ln_vec_blocks(rows, c.threads ? c.threads : 512, 2) * 2 * w;
}

#define TESS_LN_NV(nv, ...)                                                        \
  switch (nv) {                                                                    \
    case 1: { constexpr int NV = 1; __VA_ARGS__; } break;                          \
    case 2: { constexpr int NV = 2; __VA_ARGS__; } break;                          \
    case 3: { constexpr int NV = 3; __VA_ARGS__; } break;                          \
    case 4: { constexpr int NV = 4; __VA_ARGS__; } break;                          \
    default: fail(TESS_ERR_UNSUPPORTED, "vectorised LayerNorm: unsupported width"); \
  }

void k_ln_fused_fwd(const void* x, DType t, int64_t rows, int64_t w, const float* gain,
                    const float* bias, double eps, void* y, float* mean, float* rstd,
                    cudaStream_t s) {
  if (!rows) return;
  const LnCfg c = ln_vec_config(w);
  TESS_LN_NV(c.nv, TESS_DISPATCH(t, T, TESS_LN_TH(c.threads, {
    auto* k = ln_vec_fwd_kernel<T, NV, false, TH>;
    const int g = ln_grid((const void*)k, c.threads, rows, 4);
    k<<<g, c.threads, 0, s>>>((const T*)x, rows, gain, bias, (float)eps, (T*)y, mean, rstd,
                              nullptr);
  })));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_fused_bwd(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, int64_t rows, int64_t w,
                    const void* resid, DType tr, void* dx, DType tdx, float* out2w,
                    float* scratch, cudaStream_t s) {
  if (!rows) {
    if (out2w) TESS_CUDA(cudaMemsetAsync(out2w, 0, 2 * w * 4, s));
    return;
  }
  const LnCfg c = ln_vec_config(w);
  int g = 1;
  float* part = out2w ? scratch : nullptr;
  TESS_LN_NV(c.nv, TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX, TESS_DISPATCH(tr, TR,
      TESS_DISPATCH(tdx, TO, TESS_LN_TH(c.threads, {
        auto* k = ln_vec_bwd_kernel<TD, TX, TR, TO, NV, false, TH>;
        g = ln_grid((const void*)k, c.threads, rows, 2);
        k<<<g, c.threads, 0, s>>>((const TD*)dy, (const TX*)x, mean, rstd, gain, rows,
                                  (const TR*)resid, (TO*)dx, part, nullptr);
      }))))));
  count_launch();
  TESS_CUDA(cudaGetLastError());
  if (out2w) {
    colsum_finalize_kernel<<<(unsigned)((2 * w + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        scratch, g, w, 2, out2w);
    count_launch();
    TESS_CUDA(cudaGetLastError());
  }
}

bool k_ln_split_supported(int64_t w, const void* gain, const void* bias) {
  return ln_vec_ok(w, {gain, bias});
}

void k_ln_split_stats(const void* x, DType t, int64_t rows, int64_t w, float* stats,
                      cudaStream_t s) {
  if (!rows) return;
  const LnCfg c = ln_vec_config(w);
  TESS_LN_NV(c.nv, TESS_DISPATCH(t, T, {
    auto* k = ln_vec_fwd_kernel<T, NV, true, 0>;
    const int g = ln_grid((const void*)k, c.threads, rows, 4);
    k<<<g, c.threads, 0, s>>>((const T*)x, rows, nullptr, nullptr, 0.f, nullptr, nullptr,
                              nullptr, stats);
  }));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_split_apply(const void* x, DType t, const float* stats, int64_t rows, int64_t w,
                      double hidden_total, const float* gain, const float* bias, double eps,
                      void* y, float* mean, float* rstd, cudaStream_t s) {
  if (!rows) return;
  const LnCfg c = ln_vec_config(w);
  TESS_LN_NV(c.nv, TESS_DISPATCH(t, T, {
    auto* k = ln_vec_apply_kernel<T, NV>;
    const int g = ln_grid((const void*)k, c.threads, rows, 4);
    k<<<g, c.threads, 0, s>>>((const T*)x, stats, rows, (float)hidden_total, gain, bias,
                              (float)eps, (T*)y, mean, rstd);
  }));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

void k_ln_split_bwd_stats(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                          const float* rstd, const float* gain, int64_t rows, int64_t w,
                          float* stats, float* out2w, float* scratch, cudaStream_t s) {
  if (!rows) {
    if (out2w) TESS_CUDA(cudaMemsetAsync(out2w, 0, 2 * w * 4, s));
    return;
  }
  const LnCfg c = ln_vec_config(w);
  int g = 1;
  float* part = out2w ? scratch : nullptr;
  TESS_LN_NV(c.nv, TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX, {
    auto* k = ln_vec_bwd_kernel<TD, TX, float, float, NV, true, 0>;
    g = ln_grid((const void*)k, c.threads, rows, 2);
    k<<<g, c.threads, 0, s>>>((const TD*)dy, (const TX*)x, mean, rstd, gain, rows, nullptr,
                              nullptr, part, stats);
  })));
  count_launch();
  TESS_CUDA(cudaGetLastError());
  if (out2w) {
    colsum_finalize_kernel<<<(unsigned)((2 * w + kBlock - 1) / kBlock), kBlock, 0, s>>>(
        scratch, g, w, 2, out2w);
    count_launch();
    TESS_CUDA(cudaGetLastError());
  }
}

void k_ln_split_bwd_apply(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                          const float* rstd, const float* gain, const float* stats, int64_t rows,
                          int64_t w, double hidden_total, const void* resid, DType tr, void* dx,
                          DType tdx, cudaStream_t s) {
  if (!rows) return;
  const LnCfg c = ln_vec_config(w);
  TESS_LN_NV(c.nv, TESS_DISPATCH(tdy, TD, TESS_DISPATCH(tx, TX, TESS_DISPATCH(tr, TR,
      TESS_DISPATCH(tdx, TO, {
        auto* k = ln_vec_bwd_apply_kernel<TD, TX, TR, TO, NV>;
        const int g = ln_grid((const void*)k, c.threads, rows, 4);
        k<<<g, c.threads, 0, s>>>((const TD*)dy, (const TX*)x, mean, rstd, gain, stats, rows,
                                  (float)hidden_total, (const TR*)resid, (TO*)dx);
      })))));
  count_launch();
  TESS_CUDA(cudaGetLastError());
}

}  // namespace tess
