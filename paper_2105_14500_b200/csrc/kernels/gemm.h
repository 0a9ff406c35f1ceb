// Local block GEMM interface used by the SUMMA schedules and the layers.
//
// Replaces the reference's CPU kernels matmul / matmul_nt / matmul_tn
// (reference proj/src/matrix.cpp:142-216) and the `add` that accumulates
// SUMMA steps (proj/src/algorithms.cpp:42). One call computes
//
//     C[b] (op)= alpha * sum_seg  opA(A_seg[b]) * opB(B_seg[b])
//
// for a (possibly two-level batched) set of row-major views, where
// opA(A) = A ([M,K]) or A^T (A stored [K,M]), opB(B) = B ([K,N]) or B^T
// (B stored [N,K]). The K dimension may be split over up to kMaxSegments
// separately-stored panels: this is how the q SUMMA steps of one
// Tesseract product accumulate in a single tensor-memory accumulator
// instead of q launches plus q-1 HBM round trips of C.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <string>

namespace tess {

enum class DType : int { F32 = 0, BF16 = 1, F64 = 2 };

inline int dtype_size(DType t) {
  return t == DType::F32 ? 4 : t == DType::BF16 ? 2 : 8;
}

// Epilogue applied to v = alpha * acc (fp32) for every output element.
enum class Epi : int {
  Store = 0,       // C = v
  Accum = 1,       // C += v            (C fp32; weight-gradient accumulation)
  Resid = 2,       // C = v + R         (residual add fused into the producer)
  Gelu = 3,        // Z = v; C = gelu(v) with the exact erf GeLU
  // The following are tcgen05-kernel only (bf16 inputs).
  DGelu = 4,       // C = v * gelu'(R)  (R = FF1 pre-activation z; ref layers.cpp:365)
  SoftmaxFwd = 5,  // C = 2^(v*log2e - vec[row])  (vec = row log-sum-exp in log2 units)
  SoftmaxBwd = 6,  // C = R * (v - alpha*vec[row]) (R = P, vec = rowsum(dO*O))
  RowStats = 7,    // no C: stats[row][part] = (max v*log2e, sum 2^(v*log2e - max))
};

constexpr int kMaxSegments = 8;

struct GemmSeg {
  const void* a = nullptr;  // A panel for this K range
  const void* b = nullptr;  // B panel for this K range
  int64_t k = 0;            // K extent of the panel
};

// Segment readiness: SUMMA panels that are still landing when the GEMM is
// launched (summa.cpp, Comm::panel_async). A producer waits, before its
// first TMA load of segment s touching chunk c, until
//   a_flags[s][c] >= a_epoch[s]  (a_flags[s] != nullptr; chunked, see below)
//   b_flags[s][0] >= b_epoch[s]  (b_flags[s] != nullptr; whole panel)
// (wrap-safe). c = row of the stored A panel / chunk_rows: the tile's M rows
// when A is stored [M, K], its k-block when A is stored [K, M] (TN). The
// panel transport writes the flags in stream order after the bytes landed
// (cuStreamWriteValue32: no SM is involved, so a waiting persistent GEMM
// cannot starve the transfer).
struct GemmReady {
  const uint32_t* a_flags[kMaxSegments] = {};
  const uint32_t* b_flags[kMaxSegments] = {};
  uint32_t a_epoch[kMaxSegments] = {};
  uint32_t b_epoch[kMaxSegments] = {};
  int chunks = 1;
  int64_t chunk_rows = 0;  // 0: one chunk per panel
  bool any() const {
    for (int s = 0; s < kMaxSegments; ++s)
      if (a_flags[s] || b_flags[s]) return true;
    return false;
  }
};

struct GemmDesc {
  int64_t M = 0, N = 0;
  int64_t nb0 = 1, nb1 = 1;  // batch extents (attention: heads, samples)
  int nseg = 1;
  GemmSeg seg[kMaxSegments];
  bool trans_a = false;  // A stored [K, M] (TN products)
  bool trans_b = false;  // B stored [N, K] (NT products)
  int64_t lda = 0, as0 = 0, as1 = 0;  // element strides: row, batch0, batch1
  int64_t ldb = 0, bs0 = 0, bs1 = 0;
  DType in = DType::BF16;             // A and B element type
  void* c = nullptr;
  DType c_type = DType::F32;
  int64_t ldc = 0, cs0 = 0, cs1 = 0;
  const void* r = nullptr;            // residual, same type/strides as C
  int64_t ldr = 0, rs0 = 0, rs1 = 0;
  void* z = nullptr;                  // Gelu pre-activation output (bf16 or C type)
  int64_t ldz = 0, zs0 = 0, zs1 = 0;
  float alpha = 1.0f;
  Epi epi = Epi::Store;
  // Per-row vector (SoftmaxFwd / SoftmaxBwd): vec[b0*vs0 + b1*vs1 + m].
  const float* vec = nullptr;
  int64_t vs0 = 0, vs1 = 0;
  // RowStats output: float2 at stats[(b0*ss0 + b1*ss1 + m*nst + tile)*2],
  // nst = gemm_bf16_stat_tiles(d) tiles per row.
  float* stats = nullptr;
  int64_t ss0 = 0, ss1 = 0;
  GemmReady ready;
  // Fused bias / dropout (tcgen05 kernels, Store / Accum / Resid / Gelu;
  // unbatched): v = alpha*acc + bias[n]; Gelu: Z = v, v = gelu(v); dropout:
  // v = keep(drop_seed, drop_row0 + m, drop_col0 + n) ? v / (1 - drop_p) : 0
  // (dropout_keep(), a counter hash of the GLOBAL element coordinate, so a
  // sharded product drops exactly the elements the unsharded one drops);
  // Resid: v += R after the dropout. Not part of the reference (its blocks
  // have neither linear biases nor dropout, layers.hpp:42-49).
  const float* bias = nullptr;
  float drop_p = 0.f;
  uint64_t drop_seed = 0;
  int64_t drop_row0 = 0, drop_col0 = 0;
};

// Dropout mask of element (row, col) under `seed` (host and device): keep
// iff the top 24 bits of a splitmix64-style hash are >= p * 2^24.
#ifdef __CUDACC__
__host__ __device__
#endif
inline bool dropout_keep(uint64_t seed, uint64_t row, uint64_t col, uint32_t thresh24) {
  uint64_t x = seed ^ (row * 0x9E3779B97F4A7C15ull) ^ (col * 0xC2B2AE3D27D4EB4Full);
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 32;
  return (uint32_t)(x >> 40) >= thresh24;
}

// Name of the kernel instantiation gemm() launches for d (profiling).
std::string gemm_kernel_name(const GemmDesc& d);

// Column-tile width the tcgen05 dispatcher uses for d (RowStats layout).
int gemm_bf16_tile_n(const GemmDesc& d);
// RowStats partials per row (column tiles x epilogue warps per lane quadrant).
int gemm_bf16_stat_tiles(const GemmDesc& d);

// bf16 inputs on 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
cudaError_t gemm_bf16_sm100(const GemmDesc& d, cudaStream_t stream);

// fp32 inputs, fp32 FMA on CUDA cores: the fp32 parity path (config 1 of
// BASELINE.json: fp32 within 1e-5 of the fp64 reference).
cudaError_t gemm_f32_simt(const GemmDesc& d, cudaStream_t stream);

// Dispatch on d.in. Returns cudaErrorInvalidValue on unsupported layouts
// (e.g. bf16 rows that are not 16-byte aligned, which TMA cannot address).
cudaError_t gemm(const GemmDesc& d, cudaStream_t stream);

// Leave `sms` SMs free of the persistent GEMM grids (process-wide maximum of
// all requests): set by the NCCL backend so its kernels overlap the GEMMs.
void gemm_set_sm_reserve(int sms);

// Last dispatch-level error text (thread local), for the C-ABI's
// tess_last_error.
const char* gemm_last_error();

}  // namespace tess
