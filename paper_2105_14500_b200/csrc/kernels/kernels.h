// Memory-bound kernels of the Tesseract layers (HBM-bound; see DESIGN.md for
// the algorithmic bytes each one moves). All launchers are stream-ordered.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "gemm.h"

namespace tess {

// ---- conversion / arithmetic --------------------------------------------
// dst = (dst_type) src, elementwise (f64 <-> f32 <-> bf16).
void k_convert(const void* src, DType st, void* dst, DType dt, size_t n, cudaStream_t s);
// out[i] = a[i] + b[i]; a/out of type t, b of type tb.
void k_add(const void* a, DType ta, const void* b, DType tb, void* out, DType to, size_t n,
           cudaStream_t s);
// out[r, c] = x[r, c] + bias[c] (bias fp32 [cols]); ref layers.cpp:491-503.
void k_bias_add(const void* x, const float* bias, void* out, DType t, int64_t rows,
                int64_t cols, cudaStream_t s);
// dz = dh * gelu'(z) (exact erf derivative, ref layers.cpp:34-42, 365).
void k_gelu_bwd(const float* dh, const void* z, void* dz, DType t, size_t n, cudaStream_t s);
// Column sums of x [rows, cols] (type t) into out fp32 [cols]; deterministic
// fixed-order two-stage reduction (ref layers.cpp:507-510 colsum).
void k_colsum(const void* x, DType t, int64_t rows, int64_t cols, float* out, float* scratch,
              cudaStream_t s);
size_t k_colsum_scratch_floats(int64_t rows, int64_t cols);

// ---- toy training (ref layers.cpp:947-1036) --------------------------------
// dy = (2/denom) * (y - target); partial[b] = per-block sums of (y - target)^2
// (fixed-order two-stage sum into *sum, fp64). y/target of type t.
void k_mse_grad(const void* y, const void* target, DType t, size_t n, double denom, void* dy,
                double* sum, double* scratch, cudaStream_t s);
size_t k_mse_scratch_doubles(size_t n);
// w -= lr * g (w of type t, g fp32; when master != nullptr the fp32 master copy
// is updated and w is rewritten from it).
void k_sgd(void* w, DType t, float* master, const float* g, double lr, size_t n, cudaStream_t s);

// ---- LayerNorm (ref layers.cpp:242-345) -----------------------------------
// Local partial statistics per row for the row-group all-reduce:
// stats[r] = {sum x, sum (x - mu_r)^2, w * mu_r^2} with mu_r the local mean.
void k_ln_stats(const void* x, DType t, int64_t rows, int64_t w, float* stats, cudaStream_t s);
// Normalise with the (all-reduced) statistics over hidden_total columns:
// y = gain * (x - mean) * rstd + bias; writes mean/rstd per row (cache).
void k_ln_apply(const void* x, DType t, const float* stats, int64_t rows, int64_t w,
                double hidden_total, const float* gain, const float* bias, double eps,
                void* y, float* mean, float* rstd, cudaStream_t s);
// Backward partial row sums: stats[r] = {sum dxhat, sum xhat*dxhat},
// dxhat = dy * gain, xhat = (x - mean) * rstd.
void k_ln_bwd_stats(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, int64_t rows, int64_t w,
                    float* stats, cudaStream_t s);
// dx = rstd * (dxhat - s0/n - xhat * s1/n) (+ resid); out of type to.
void k_ln_bwd_apply(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, const float* stats, int64_t rows,
                    int64_t w, double hidden_total, const void* resid, DType tr, void* dx,
                    DType to, cudaStream_t s);
// Column partials for dgain/dbias: out[0][c] = sum_r dy*xhat, out[1][c] = sum_r dy.
void k_ln_bwd_params(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                     const float* rstd, int64_t rows, int64_t w, float* out2w, float* scratch,
                     cudaStream_t s);
size_t k_ln_params_scratch_floats(int64_t rows, int64_t w);

// Vectorised LayerNorm (16-byte accesses, rows register-resident in a
// block): w = nv * 8 * threads with nv <= 4 and a whole number of warps in
// [128, 1024] per block (every 4096 * k up to 16384, 6144, 3072, 2048, ...),
// gain / bias 16-byte aligned. Bitwise-deterministic.
bool k_ln_split_supported(int64_t w, const void* gain, const void* bias);
// Fused single pass for a one-member row group (q == 1: the row all-reduce
// between statistics and apply moves nothing).
bool k_ln_fused_supported(int64_t w);
// y = gain * (x - mean) * rstd + bias over the local w columns (= hidden).
void k_ln_fused_fwd(const void* x, DType t, int64_t rows, int64_t w, const float* gain,
                    const float* bias, double eps, void* y, float* mean, float* rstd,
                    cudaStream_t s);
// dx (+ resid) and, if out2w, [dgain | dbias] column sums (fixed-order
// two-stage reduction through scratch).
void k_ln_fused_bwd(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                    const float* rstd, const float* gain, int64_t rows, int64_t w,
                    const void* resid, DType tr, void* dx, DType tdx, float* out2w,
                    float* scratch, cudaStream_t s);
// q > 1 (statistics all-reduced over the row group between two passes):
// forward partials stats[r] = {sum x, M2 of the local columns, w * mean_r^2}
// (one pass), then apply with the summed partials (hidden_total columns);
void k_ln_split_stats(const void* x, DType t, int64_t rows, int64_t w, float* stats,
                      cudaStream_t s);
void k_ln_split_apply(const void* x, DType t, const float* stats, int64_t rows, int64_t w,
                      double hidden_total, const float* gain, const float* bias, double eps,
                      void* y, float* mean, float* rstd, cudaStream_t s);
// backward partials stats[r] = {sum dxhat, sum xhat*dxhat} plus, if out2w,
// the [dgain | dbias] column sums in the same pass; then dx (+ resid).
void k_ln_split_bwd_stats(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                          const float* rstd, const float* gain, int64_t rows, int64_t w,
                          float* stats, float* out2w, float* scratch, cudaStream_t s);
void k_ln_split_bwd_apply(const void* dy, DType tdy, const void* x, DType tx, const float* mean,
                          const float* rstd, const float* gain, const float* stats, int64_t rows,
                          int64_t w, double hidden_total, const void* resid, DType tr, void* dx,
                          DType tdx, cudaStream_t s);
size_t k_ln_fused_scratch_floats(int64_t rows, int64_t w);

// ---- softmax (ref layers.cpp:44-74) ---------------------------------------
// P = softmax_rows(S) with max subtraction; S fp32 [rows, L] (already scaled).
void k_softmax_fwd(const float* S, void* P, DType t, int64_t rows, int64_t L, cudaStream_t s);
// lse[r] = log-sum-exp (log2 units) over the nst RowStats partials
// (max, sum-exp2) of row r.
void k_lse_combine(const float* stats, int64_t rows, int nst, float* lse, cudaStream_t s);
// delta[(smp*H + h)*S + r] = sum_d dO[smp*S + r, h*hd + d] * O[smp*S + r, h*hd + d]
// (= rowsum(P * dP), the softmax-backward row term) for `samples` samples of
// S rows, heads H, row stride ld (one launch on the bf16 path).
void k_attn_delta(const void* dO, const void* O, DType t, int64_t ld, int64_t S, int64_t H,
                  int64_t hd, float* delta, cudaStream_t s, int64_t samples = 1);
// dS = scale * P * (dP - sum_c P*dP); dP fp32.
void k_softmax_bwd(const void* P, const float* dP, void* dS, DType t, int64_t rows, int64_t L,
                   float scale, cudaStream_t s);

// ---- peer windows (kernels/peer.cu) ----------------------------------------
// System-scope release store of v into *flag (a partner's window header).
void k_peer_signal(uint32_t* flag, uint32_t v, cudaStream_t s);
// Spins with acquire loads until *flag >= v; traps after 60 s.
void k_peer_wait(const uint32_t* flag, uint32_t v, cudaStream_t s);
// Self-test pattern: dst[i] = base + (i % 4093); check counts mismatches.
void k_peer_fill(float* dst, size_t n, float base, cudaStream_t s);
// *bad += number of elements whose bits differ (a vs b)
void k_count_mismatch(const float* a, const float* b, size_t n, unsigned long long* bad,
                      cudaStream_t s);
void k_peer_check(const float* src, size_t n, float base, unsigned long long* bad,
                  cudaStream_t s);

}  // namespace tess
