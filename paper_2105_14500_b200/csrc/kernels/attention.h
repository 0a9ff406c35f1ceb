// Fused attention (scores -> softmax -> P V and its backward) on sm_100a
// tensor cores, for the per-head loops of the reference's attention layer
// (proj/src/layers.cpp:383-456). Replaces, for bf16, the batched score GEMM,
// the materialised probabilities P ([heads, s, s] per sample, the
// reference's AttnCacheRank::probs, layers.hpp:111-113) and the row softmax
// kernels: S and P live only in tensor memory / shared memory, one row
// log-sum-exp per query is kept for the backward instead of P.
//
// Layout (the rank's activations):
//   qkv  bf16 [samples * S, ld_qkv], head h at columns h*3*hd + {0, hd, 2hd}
//        for Q, K, V (per-head interleaved triples, layers.hpp:38-41)
//   o    bf16 [samples * S, ld_o], head h at columns h*hd
//   lse  fp32 [samples, H, S]: log2-sum-exp2 of (scale*log2(e)) * q.k
// No mask (reference semantics, layers.cpp:399-400).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace tess {

struct AttnDesc {
  const void* qkv = nullptr;
  int64_t ld_qkv = 0;
  void* o = nullptr;  // forward output / backward input O
  int64_t ld_o = 0;
  float* lse = nullptr;
  int64_t samples = 0, heads = 0, seq = 0, head_dim = 0;
  float scale = 1.0f;  // 1/sqrt(head_dim)
  // backward only
  const void* dout = nullptr;  // dO bf16, same layout as o (ld_o)
  float* delta = nullptr;       // [samples, H, S] rowsum(dO * O): written by the dQ pass,
                               // read by the dK/dV pass after it
  void* dqkv = nullptr;        // bf16, same layout as qkv (ld_qkv): dQ, dK, dV written
};

// True when the fused kernels support this shape (head_dim 64 or 128, seq a
// multiple of 8, 16-byte aligned rows); otherwise the layer uses the unfused
// GEMM + softmax path.
bool attn_fused_supported(const AttnDesc& d);

cudaError_t attn_fwd_sm100(const AttnDesc& d, cudaStream_t s);
// The backward is two passes, neither of which writes S, P or dS to HBM
// (both recompute them from lse and delta = rowsum(dO * O); deterministic),
// run in this order:
// dQ pass: delta (written to d.delta) and dQ = scale * dS K, one 128-query
// tile per CTA.
cudaError_t attn_dq_sm100(const AttnDesc& d, cudaStream_t s);
// dK, dV pass: dK = scale * dS^T Q, dV = P^T dO, one 128-key tile per CTA
// (reads d.delta).
cudaError_t attn_bwd_kv_sm100(const AttnDesc& d, cudaStream_t s);

const char* attn_last_error();

// Debug: device buffer of the last traced attention kernel (set only by the
// tool-only experiments under csrc/tools with TESS_ATTN_TRACE), or null.
long long* attn_debug_trace();

}  // namespace tess
