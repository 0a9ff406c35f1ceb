// Rank-level Tesseract operators (SUMMA-in-depth products and the layers
// built on them). Reference counterparts:
//   nn/nt/tn_product    proj/src/algorithms.cpp:34-76
//   ln/ff/attn/block    proj/src/layers.cpp:242-487
//   bias_add            proj/src/layers.cpp:491-517
#pragma once

#include "ctx.h"
#include "kernels/gemm.h"

namespace tess {

// Where and how a product's result is written.
struct Out {
  void* c = nullptr;
  DType t = DType::F32;
  int64_t ldc = 0;
  Epi epi = Epi::Store;
  const void* r = nullptr;  // residual (Resid), same type/ld as c
  int64_t ldr = 0;
  void* z = nullptr;  // pre-activation (Gelu)
  int64_t ldz = 0;
  float alpha = 1.0f;
  // fused bias / dropout (GemmDesc; tess_matmul_ex)
  const float* bias = nullptr;
  float drop_p = 0.f;
  uint64_t drop_seed = 0;
  int64_t drop_row0 = 0, drop_col0 = 0;
};

// Launches one local GEMM (tcgen05 for bf16, CUDA cores for fp32); failures
// become tess::Error. When profiling is on, the launch is bracketed by CUDA
// events on its stream (tess_profile_*).
void run_gemm(const GemmDesc& g, cudaStream_t s);

// The q panels of one operand after a family broadcast (slot t -> ptr[t]).
// With the SM-free transport (Comm::panel_async) a remote panel may still be
// landing: its GEMM waits on flags[t] >= epoch[t] (GemmReady), and the
// receiver releases the link once its last reader is enqueued
// (release_panels).
struct Panels {
  bool valid = false;
  void* ptr[kMaxSegments] = {};
  const uint32_t* flags[kMaxSegments] = {};
  uint32_t epoch[kMaxSegments] = {};
  Family fam = COL;
  std::string tag;
};
void release_panels(Ctx& c, const Panels& p, cudaStream_t s);

// Broadcasts every slot's panel of a weight-style operand over family f on
// the comm stream ahead of its use (the weight panels of a whole layer do
// not depend on activations), into workspace buffers named tag<t>.
Panels prefetch_panels(Ctx& c, Family f, const void* local, int64_t rows, int64_t cols,
                       size_t esz, const std::string& tag, cudaStream_t s);

// Makes the compute stream wait for all collectives issued so far.
void join_comm(Ctx& c, cudaStream_t s);

// C[ar, bn] (op)= sum_t A(h,t) B(t,j); A panels row-broadcast, B panels
// column-broadcast (or prefetched: bp), all q panels accumulated in one
// tensor-memory accumulator (one GEMM with q K-segments).
void nn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t ak, const void* b,
                int64_t bn, const Out& out, cudaStream_t s, const Panels* bp = nullptr);

// C(h, j') = sum_j A(h,j) B(j',j)^T reduced over the row to slot j' (fp32).
// out must be fp32 (Store or Accum) or bf16 Store.
void nt_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t br, const Out& out, cudaStream_t s, const Panels* bp = nullptr);

// C(i', j) = sum A(h,i')^T B(h,j) reduced down the column to slot i' and, if
// sum_over_depth, all-reduced over depth. out fp32 Store or Accum. With
// defer, the result is completed on the comm stream only (join_comm later).
void tn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t bn, bool sum_over_depth, const Out& out, cudaStream_t s,
                bool defer = false);

// ------------------------------------------------------------------ layers
struct RankDims {
  int64_t rows = 0;       // local activation rows = samples_local * seq
  int64_t hq = 0;         // hidden / q (1-D scheme: hidden / p, the local head width)
  int64_t hin = 0;        // activation width on this rank: hq (1-D scheme: hidden)
  int64_t seq = 0;
  int64_t head_dim = 0;
  int64_t heads_local = 0;
  int64_t samples_local = 0;
  int64_t hidden_total = 0;
};
RankDims rank_dims(const Ctx& c, const tess_layer_dims& d);

void layer_forward(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                   const tess_block_shard& p, const float* bias_row0, const void* x, void* y,
                   cudaStream_t s);
void layer_step(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                const tess_block_shard& p, const float* bias_row0, const void* x, const void* dy,
                void* y, void* dx, tess_block_grads* g, bool accumulate, float* dbias,
                cudaStream_t s);
void layer_backward(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                    const tess_block_shard& p, const void* dy, void* dx,
                    tess_block_grads* g, bool accumulate, float* dbias, cudaStream_t s);
// `layers` blocks forward then backward (cache slots base..base+layers-1).
void stack_step(Ctx& c, DType t, const RankDims& rd, int layers, const tess_block_shard* p,
                const void* x, const void* dy, void* y, void* dx, tess_block_grads* g,
                bool accumulate, cudaStream_t s);

}  // namespace tess
