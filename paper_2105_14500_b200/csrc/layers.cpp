// Rank-level Transformer layers on the Tesseract grid (reference
// proj/src/layers.cpp:242-517), B200 version:
//  * LayerNorm: with a one-member row group (q == 1) one fused single-pass
//    kernel each way (stats + apply; stats + dx + dgain/dbias partials);
//    otherwise per-row partial statistics (sum, centred M2, w*mu^2 -- a
//    Chan-style combination that avoids E[x^2]-E[x]^2 cancellation in fp32)
//    all-reduced over the row group, then normalise. The meter charges the
//    reference's [rows, 2] payload either way (layers.cpp:258).
//  * FF: FF1 GEMM with the exact-erf GeLU fused into its epilogue (stores the
//    pre-activation z and h = gelu(z)); FF2 GEMM with the residual add fused;
//    GeLU' fused into the FF2-dgrad epilogue when q == 1.
//  * Attention (bf16): the fused tcgen05 kernels of kernels/attention_sm100.cu
//    (S, P never in HBM; the row log-sum-exp is cached instead of the
//    reference's probs) plus one batched dQ GEMM; the fp32 parity mode keeps
//    batched GEMMs + row softmax with P cached like the reference
//    (layers.cpp:403). Per-head interleaved Q|K|V columns are addressed by
//    TMA coordinates, no copies. No causal mask (reference semantics).
//  * Residual adds are fused into GEMM epilogues (forward) or into the
//    LayerNorm-backward kernels (backward).
// Forward caches live in the context workspace under per-op names until the
// matching backward.
#include <cmath>
#include <cstdlib>
#include <string>

#include "kernels/attention.h"
#include "kernels/kernels.h"
#include "ops.h"

namespace tess {

RankDims rank_dims(const Ctx& c, const tess_layer_dims& d) {
  // ref: layers.cpp:115-136 (divisibility), 230-238 (rank_dims)
  const int q = c.grid.q, dd = c.grid.d;
  auto req = [](bool ok, const std::string& what) {
    if (!ok) fail(TESS_ERR_DIVISIBILITY, what);
  };
  if (c.megatron) {
    // 1-D scheme: every rank holds all rows and heads [k n/p, (k+1) n/p)
    const int p = c.grid.size();
    req(q == 1, "1-D scheme needs a [1,1,p] line grid");
    req(d.heads > 0 && d.heads % p == 0, "heads (" + std::to_string(d.heads) +
                                             ") not divisible by p (" + std::to_string(p) + ")");
    req(d.hidden % d.heads == 0, "hidden (" + std::to_string(d.hidden) +
                                     ") not divisible by heads (" + std::to_string(d.heads) + ")");
    RankDims r;
    r.seq = d.seq;
    r.head_dim = d.hidden / d.heads;
    r.heads_local = d.heads / p;
    r.samples_local = d.batch;
    r.hidden_total = d.hidden;
    r.hq = d.hidden / p;
    r.hin = d.hidden;
    r.rows = (int64_t)d.batch * d.seq;
    return r;
  }
  req(d.batch % (dd * q) == 0, "batch (" + std::to_string(d.batch) + ") not divisible by d*q (" +
                                   std::to_string(dd * q) + ")");
  req(d.hidden % q == 0, "hidden (" + std::to_string(d.hidden) + ") not divisible by q (" +
                             std::to_string(q) + ")");
  req(d.heads > 0 && d.heads % q == 0, "heads (" + std::to_string(d.heads) +
                                           ") not divisible by q (" + std::to_string(q) + ")");
  req(d.hidden % d.heads == 0, "hidden (" + std::to_string(d.hidden) +
                                   ") not divisible by heads (" + std::to_string(d.heads) + ")");
  RankDims r;
  r.seq = d.seq;
  r.head_dim = d.hidden / d.heads;
  r.heads_local = d.heads / q;
  r.samples_local = d.batch / (dd * q);
  r.hidden_total = d.hidden;
  r.hq = d.hidden / q;
  r.hin = r.hq;
  r.rows = r.samples_local * d.seq;
  return r;
}

namespace {

void* wsget(Ctx& c, const std::string& name, size_t bytes) { return c.ws->get(name, bytes); }

Out out_to(void* p, DType t, int64_t ld = 0) {
  Out o;
  o.c = p;
  o.t = t;
  o.ldc = ld;
  return o;
}

// ----------------------------------------------------------- LayerNorm
// The vectorised kernels need w = nv * 8 * threads and 16-byte aligned rows.
bool ln_vec(int64_t w, const float* gain, const float* bias,
            std::initializer_list<const void*> rows) {
  if (!k_ln_split_supported(w, gain, bias)) return false;
  for (const void* p : rows)
    if (p && reinterpret_cast<uintptr_t>(p) % 16 != 0) return false;
  return true;
}

void ln_fwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag, const void* x,
            const float* gain, const float* bias, double eps, void* y, cudaStream_t s) {
  const int64_t rows = rd.rows, w = rd.hin;
  float* stats = static_cast<float*>(wsget(c, "ln.stats", rows * 3 * 4));
  float* mean = static_cast<float*>(wsget(c, tag + ".mean", rows * 4));
  float* rstd = static_cast<float*>(wsget(c, tag + ".rstd", rows * 4));
  const bool vec = ln_vec(w, gain, bias, {x, y});
  if (c.grid.q == 1 && vec) {
    // one-member row group: the [rows, 2] all-reduce moves nothing (still
    // metered and traced like the reference), so stats + apply is one pass
    c.meter.reduce(1, 0, 0, (uint64_t)rows * 2, true);
    if (c.trace_on) c.trace.push_back({c.rank, c.step, 2, ROW, 0, (uint64_t)rows * 2 * 8});
    c.step++;
    ProfMem pm("ln_fused_fwd_kernel", (double)rows * (w * 2.0 * dtype_size(t) + 8), s);
    k_ln_fused_fwd(x, t, rows, w, gain, bias, eps, y, mean, rstd, s);
    return;
  }
  if (vec) {
    // q > 1: one vectorised pass for the [rows, 3] partials
    ProfMem pm("ln_vec_stats_kernel", (double)rows * (w * dtype_size(t) + 12), s);
    k_ln_split_stats(x, t, rows, w, stats, s);
  } else {
    ProfMem pm("ln_stats_kernel", (double)rows * (w * dtype_size(t) + 12), s);
    k_ln_stats(x, t, rows, w, stats, s);
  }
  // ref layers.cpp:258: row all-reduce of the [rows, 2] sums (metered as such)
  c.meter.reduce(c.grid.group_size(ROW), c.grid.slot_in_group(c.coord, ROW), 0,
                 (uint64_t)rows * 2, true);
  if (c.trace_on) c.trace.push_back({c.rank, c.step, 2, ROW, 0, (uint64_t)rows * 2 * 8});
  c.step++;
  cudaStream_t cs = comm_stream(c, s);
  stream_dep(c, s, cs);
  if (!c.comm_noop) c.comm->allreduce(ROW, stats, rows * 3, cs);
  stream_dep(c, cs, s);
  ProfMem pm(vec ? "ln_vec_apply_kernel" : "ln_apply_kernel",
             (double)rows * (w * 2.0 * dtype_size(t) + 20), s);
  if (vec)
    k_ln_split_apply(x, t, stats, rows, w, (double)rd.hidden_total, gain, bias, eps, y, mean,
                     rstd, s);
  else
    k_ln_apply(x, t, stats, rows, w, (double)rd.hidden_total, gain, bias, eps, y, mean, rstd, s);
}

// dx = LN'(dy) (+ resid); optional gain/bias grads (column + depth all-reduce,
// ref layers.cpp:318-343, only when requested).
void ln_bwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag, const void* dy,
            DType tdy, const void* x, const float* gain, const void* resid, DType tr, void* dx,
            DType tdx, float* dgain, float* dbias, bool accumulate, cudaStream_t s) {
  const int64_t rows = rd.rows, w = rd.hin;
  const float* mean = static_cast<const float*>(wsget(c, tag + ".mean", rows * 4));
  const float* rstd = static_cast<const float*>(wsget(c, tag + ".rstd", rows * 4));
  float* stats = static_cast<float*>(wsget(c, "ln.bstats", rows * 2 * 4));
  cudaStream_t cs = comm_stream(c, s);
  const bool want_params = dgain || dbias;
  // per-LN buffers: the all-reduces and the gradient update stay on the
  // comm stream (joined at the end of the layer backward)
  float* packed =
      want_params ? static_cast<float*>(wsget(c, tag + ".packed", 2 * w * 4)) : nullptr;
  const bool vec = ln_vec(w, gain, gain, {dy, x, resid, dx});
  if (c.grid.q == 1 && vec) {
    // one-member row group: the [rows, 2] all-reduce moves nothing, so row
    // statistics, dx and the dgain/dbias partials are one pass over dy, x
    coll_allreduce(c, ROW, stats, rows * 2, cs);  // ref layers.cpp:305 (metered)
    float* scratch = static_cast<float*>(
        wsget(c, "ln.fscratch", k_ln_fused_scratch_floats(rows, w) * 4));
    ProfMem pm("ln_fused_bwd_kernel",
               (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t) + dtype_size(tdx) +
                                            (resid ? dtype_size(tr) : 0)) + 8), s);
    k_ln_fused_bwd(dy, tdy, x, t, mean, rstd, gain, rows, w, resid, tr, dx, tdx, packed,
                   scratch, s);
  } else if (vec) {
    // q > 1: one pass for the row partials and the dgain/dbias column sums,
    // the row all-reduce, one pass for dx
    {
      float* scratch = static_cast<float*>(
          wsget(c, "ln.fscratch", k_ln_fused_scratch_floats(rows, w) * 4));
      ProfMem pm("ln_vec_bwd_stats_kernel",
                 (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t)) + 16), s);
      k_ln_split_bwd_stats(dy, tdy, x, t, mean, rstd, gain, rows, w, stats, packed, scratch, s);
    }
    stream_dep(c, s, cs);
    coll_allreduce(c, ROW, stats, rows * 2, cs);  // ref layers.cpp:305
    stream_dep(c, cs, s);
    ProfMem pm("ln_vec_bwd_apply_kernel",
               (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t) + dtype_size(tdx) +
                                            (resid ? dtype_size(tr) : 0)) + 16), s);
    k_ln_split_bwd_apply(dy, tdy, x, t, mean, rstd, gain, stats, rows, w,
                         (double)rd.hidden_total, resid, tr, dx, tdx, s);
  } else {
    {
      ProfMem pm("ln_bwd_stats_kernel",
                 (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t)) + 16), s);
      k_ln_bwd_stats(dy, tdy, x, t, mean, rstd, gain, rows, w, stats, s);
    }
    stream_dep(c, s, cs);
    coll_allreduce(c, ROW, stats, rows * 2, cs);  // ref layers.cpp:305
    stream_dep(c, cs, s);
    {
      ProfMem pm("ln_bwd_apply_kernel",
                 (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t) + dtype_size(tdx) +
                                              (resid ? dtype_size(tr) : 0)) + 16), s);
      k_ln_bwd_apply(dy, tdy, x, t, mean, rstd, gain, stats, rows, w, (double)rd.hidden_total,
                     resid, tr, dx, tdx, s);
    }
    if (want_params) {
      float* scratch =
          static_cast<float*>(wsget(c, "ln.pscratch", k_ln_params_scratch_floats(rows, w) * 4));
      ProfMem pm("ln_bwd_params_kernel",
                 (double)rows * (w * (double)(dtype_size(tdy) + dtype_size(t)) + 8), s);
      k_ln_bwd_params(dy, tdy, x, t, mean, rstd, rows, w, packed, scratch, s);
    }
  }
  if (want_params) {
    stream_dep(c, s, cs);
    coll_allreduce(c, COL, packed, 2 * w, cs);    // ref layers.cpp:331
    // (1-D scheme: every rank already holds the full, identical LN gradient)
    if (!c.megatron) coll_allreduce(c, DEPTH, packed, 2 * w, cs);  // ref layers.cpp:332
    for (int k = 0; k < 2; ++k) {
      float* dst = k == 0 ? dgain : dbias;
      if (!dst) continue;
      if (accumulate)
        k_add(dst, DType::F32, packed + k * w, DType::F32, dst, DType::F32, w, cs);
      else
        TESS_CUDA(cudaMemcpyAsync(dst, packed + k * w, w * 4, cudaMemcpyDeviceToDevice, cs));
    }
  }
}

Out grad_out(float* g, bool accumulate) {
  Out o = out_to(g, DType::F32);
  o.epi = accumulate ? Epi::Accum : Epi::Store;
  return o;
}

// TN weight-gradient product; with no grads requested the collectives still
// run into scratch (ref layers.cpp:372-377).
void weight_grad(Ctx& c, DType t, const void* a, int64_t ar, int64_t an, const void* b,
                 int64_t bn, float* g, bool accumulate, cudaStream_t s) {
  float* dst = g ? g : static_cast<float*>(wsget(c, "wgrad.discard", (size_t)an * bn * 4));
  // deferred: reduce + depth all-reduce + gradient write hide under the rest
  // of the backward (layer_backward joins the comm stream before returning)
  // (1-D scheme: each rank owns a weight shard, nothing to sum over depth)
  tn_product(c, t, a, ar, an, b, bn, !c.megatron, grad_out(dst, g && accumulate), s,
             /*defer=*/true);
}

// Weight panels of a layer broadcast over the column group up front (they do
// not depend on activations), for the NN (forward) / NT (backward) products.
struct WeightPanels {
  Panels qkv, proj, ff1, ff2;
};

// Panel buffers alternate with the cache slot's parity, so a stack's next
// layer can receive its weights while this layer's GEMMs still read theirs.
WeightPanels prefetch_weights(Ctx& c, DType t, const RankDims& rd, const tess_block_shard& p,
                              bool attn, bool ff, cudaStream_t s) {
  WeightPanels w;
  if (c.grid.q == 1) return w;
  const int64_t hq = rd.hq;
  const size_t e = dtype_size(t);
  const std::string pf = "pf" + std::to_string(c.cache_slot & 1) + ".";
  if (attn) {
    w.qkv = prefetch_panels(c, COL, p.w_qkv, hq, 3 * hq, e, pf + "qkv", s);
    w.proj = prefetch_panels(c, COL, p.w_proj, hq, hq, e, pf + "proj", s);
  }
  if (ff) {
    w.ff1 = prefetch_panels(c, COL, p.w_ff1, hq, 4 * hq, e, pf + "ff1", s);
    w.ff2 = prefetch_panels(c, COL, p.w_ff2, 4 * hq, hq, e, pf + "ff2", s);
  }
  return w;
}

// The receiver's last reads of the layer's weight panels are enqueued.
void release_weights(Ctx& c, const WeightPanels& w, cudaStream_t s) {
  release_panels(c, w.qkv, s);
  release_panels(c, w.proj, s);
  release_panels(c, w.ff1, s);
  release_panels(c, w.ff2, s);
}

// ----------------------------------------------------------------- FF
// ref layers.cpp:349-360. Cache: x (caller-owned), z, h.
void ff_fwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag,
            const tess_block_shard& p, const void* x, const Out& yout, cudaStream_t s,
            const WeightPanels& wp) {
  const int64_t rows = rd.rows, hq = rd.hq;
  const size_t esz = dtype_size(t);
  void* z = wsget(c, tag + ".z", rows * 4 * hq * esz);
  void* h = wsget(c, tag + ".h", rows * 4 * hq * esz);
  Out o1 = out_to(h, t);
  o1.epi = Epi::Gelu;
  o1.z = z;
  nn_product(c, t, x, rows, rd.hin, p.w_ff1, 4 * hq, o1, s, &wp.ff1);
  nn_product(c, t, h, rows, 4 * hq, p.w_ff2, rd.hin, yout, s, &wp.ff2);
}

// ref layers.cpp:362-379: NT, gelu', NT, TN, TN. dx written fp32.
void ff_bwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag,
            const tess_block_shard& p, const void* x, const void* dy, float* dx_f32,
            tess_block_grads* g, bool accumulate, cudaStream_t s, const WeightPanels& wp) {
  const int64_t rows = rd.rows, hq = rd.hq;
  const size_t esz = dtype_size(t);
  const void* z = wsget(c, tag + ".z", rows * 4 * hq * esz);
  const void* h = wsget(c, tag + ".h", rows * 4 * hq * esz);
  void* dz = wsget(c, "ff.dz", rows * 4 * hq * esz);
  if (t == DType::BF16 && c.grid.q == 1) {
    // no row reduce: fuse dz = dh * gelu'(z) into the NT epilogue
    Out od = out_to(dz, t);
    od.epi = Epi::DGelu;
    od.r = z;
    nt_product(c, t, dy, rows, rd.hin, p.w_ff2, 4 * hq, od, s, &wp.ff2);
  } else {
    float* dh = static_cast<float*>(wsget(c, "ff.dh", rows * 4 * hq * 4));
    nt_product(c, t, dy, rows, rd.hin, p.w_ff2, 4 * hq, out_to(dh, DType::F32), s, &wp.ff2);
    ProfMem pm("gelu_bwd_kernel", (double)rows * 4 * hq * (4.0 + 2 * dtype_size(t)), s);
    k_gelu_bwd(dh, z, dz, t, (size_t)rows * 4 * hq, s);  // ref layers.cpp:365
  }
  nt_product(c, t, dz, rows, 4 * hq, p.w_ff1, rd.hin, out_to(dx_f32, DType::F32), s, &wp.ff1);
  weight_grad(c, t, h, rows, 4 * hq, dy, rd.hin, g ? g->w_ff2 : nullptr, accumulate, s);
  weight_grad(c, t, x, rows, rd.hin, dz, 4 * hq, g ? g->w_ff1 : nullptr, accumulate, s);
}

// ----------------------------------------------------------- attention
// The fused tcgen05 attention kernels (kernels/attention_sm100.cu) serve the
// bf16 mode when the head shape allows (head_dim 64 / 128, seq % 8 == 0);
// TESS_ATTN_FUSED=0 selects the unfused GEMM + softmax path (A/B checks).
// Forward and backward make the same choice, so the forward caches what the
// backward reads: the row log-sum-exp (fused) or P (unfused).
AttnDesc attn_desc(const RankDims& rd, const void* qkv, void* o, float* lse) {
  AttnDesc a;
  a.qkv = qkv;
  a.ld_qkv = 3 * rd.hq;
  a.o = o;
  a.ld_o = rd.hq;
  a.lse = lse;
  a.samples = rd.samples_local;
  a.heads = rd.heads_local;
  a.seq = rd.seq;
  a.head_dim = rd.head_dim;
  a.scale = (float)(1.0 / std::sqrt((double)rd.head_dim));
  return a;
}

bool use_fused_attn(DType t, const RankDims& rd) {
  static const bool enabled = [] {
    const char* e = std::getenv("TESS_ATTN_FUSED");
    return !(e && e[0] == '0');
  }();
  if (!enabled || t != DType::BF16) return false;
  AttnDesc a = attn_desc(rd, reinterpret_cast<void*>(256), reinterpret_cast<void*>(256), nullptr);
  return attn_fused_supported(a);
}

enum class AttnPass { Fwd, BwdKV, BwdQ };

void run_attn(AttnPass k, const AttnDesc& a, cudaStream_t s) {
  ProfToken tok;
  // algorithmic flops, in contractions of 2*S*S*hd per (sample, head): 2
  // (fwd: S, PV), 3 (dK/dV pass: dV, dP, dK), 1 (dQ pass: dQ; its S and dP
  // are recomputation)
  const double unit = 2.0 * (double)a.seq * a.seq * a.head_dim * a.heads * a.samples;
  const std::string hd = a.head_dim == 128 ? "<128>" : "<64>";
  static const char* names[] = {"attn_fwd_kernel", "attn_bwd_kv_kernel", "attn_dq_kernel"};
  static const double units[] = {2.0, 3.0, 1.0};
  tok = prof_begin(names[(int)k] + hd, units[(int)k] * unit, s);
  cudaError_t e = k == AttnPass::Fwd     ? attn_fwd_sm100(a, s)
                  : k == AttnPass::BwdKV ? attn_bwd_kv_sm100(a, s)
                                         : attn_dq_sm100(a, s);
  count_launch();
  if (e == cudaErrorInvalidValue) fail(TESS_ERR_UNSUPPORTED, attn_last_error());
  if (e != cudaSuccess)
    fail(TESS_ERR_CUDA, std::string("attention: ") + cudaGetErrorString(e) + " " + attn_last_error());
  prof_end(tok, s);
}

// ref layers.cpp:383-414.
void attn_fwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag,
              const tess_block_shard& p, const void* x, const Out& yout, cudaStream_t s,
              const WeightPanels& wp) {
  const int64_t rows = rd.rows, hq = rd.hq, S = rd.seq, hd = rd.head_dim;
  const int64_t H = rd.heads_local, ld = 3 * hq;
  const size_t esz = dtype_size(t);
  void* qkv = wsget(c, tag + ".qkv", rows * ld * esz);
  if (use_fused_attn(t, rd)) {
    void* o = wsget(c, tag + ".o", rows * hq * esz);
    float* lse = static_cast<float*>(wsget(c, tag + ".lse", (size_t)rd.samples_local * H * S * 4));
    nn_product(c, t, x, rows, rd.hin, p.w_qkv, 3 * hq, out_to(qkv, t), s, &wp.qkv);
    run_attn(AttnPass::Fwd, attn_desc(rd, qkv, o, lse), s);
    nn_product(c, t, o, rows, hq, p.w_proj, rd.hin, yout, s, &wp.proj);
    return;
  }
  void* P = wsget(c, tag + ".P", (size_t)rd.samples_local * H * S * S * esz);
  void* o = wsget(c, tag + ".o", rows * hq * esz);
  const bool fused = t == DType::BF16;
  float* Sbuf = fused ? nullptr : static_cast<float*>(wsget(c, "attn.S", (size_t)H * S * S * 4));
  nn_product(c, t, x, rows, rd.hin, p.w_qkv, 3 * hq, out_to(qkv, t), s, &wp.qkv);
  const float scale = (float)(1.0 / std::sqrt((double)hd));
  const char* base = static_cast<const char*>(qkv);
  for (int64_t smp = 0; smp < rd.samples_local; ++smp) {
    const char* q0 = base + (size_t)smp * S * ld * esz;
    char* Ps = static_cast<char*>(P) + (size_t)smp * H * S * S * esz;
    if (fused) {
      // Two passes of the score GEMM, no fp32 S in HBM: (1) per-row
      // (max, sum-exp) partials per column tile -> log-sum-exp; (2) the
      // epilogue writes P = exp(scale*QK^T - lse) in bf16.
      GemmDesc g;
      g.M = S;
      g.N = S;
      g.nb0 = H;
      g.in = t;
      g.trans_b = true;
      g.seg[0] = {q0, q0 + hd * esz, hd};
      g.lda = ld;
      g.as0 = 3 * hd;
      g.ldb = ld;
      g.bs0 = 3 * hd;
      g.c_type = DType::BF16;
      g.alpha = scale;
      const int nst = gemm_bf16_stat_tiles(g);
      float* st = static_cast<float*>(wsget(c, "attn.stats", (size_t)H * S * nst * 8));
      float* lse = static_cast<float*>(wsget(c, "attn.lse", (size_t)H * S * 4));
      g.epi = Epi::RowStats;
      g.stats = st;
      g.ss0 = S * nst;
      run_gemm(g, s);
      k_lse_combine(st, H * S, nst, lse, s);
      g.epi = Epi::SoftmaxFwd;
      g.stats = nullptr;
      g.vec = lse;
      g.vs0 = S;
      g.c = Ps;
      g.ldc = S;
      g.cs0 = S * S;
      run_gemm(g, s);
    }
    // scores = Q K^T / sqrt(hd) for every local head (batched over heads)
    GemmDesc g;
    g.M = S;
    g.N = S;
    g.nb0 = H;
    g.in = t;
    g.trans_b = true;
    g.seg[0] = {q0, q0 + hd * esz, hd};
    g.lda = ld;
    g.as0 = 3 * hd;
    g.ldb = ld;
    g.bs0 = 3 * hd;
    g.c = Sbuf;
    g.c_type = DType::F32;
    g.ldc = S;
    g.cs0 = S * S;
    g.alpha = scale;
    if (!fused) {
      run_gemm(g, s);
      k_softmax_fwd(Sbuf, Ps, t, H * S, S, s);
    }
    // O = P V
    GemmDesc g2;
    g2.M = S;
    g2.N = hd;
    g2.nb0 = H;
    g2.in = t;
    g2.seg[0] = {Ps, q0 + 2 * hd * esz, S};
    g2.lda = S;
    g2.as0 = S * S;
    g2.ldb = ld;
    g2.bs0 = 3 * hd;
    g2.c = static_cast<char*>(o) + (size_t)smp * S * hq * esz;
    g2.c_type = t;
    g2.ldc = hq;
    g2.cs0 = hd;
    run_gemm(g2, s);
  }
  nn_product(c, t, o, rows, hq, p.w_proj, rd.hin, yout, s, &wp.proj);
}

// ref layers.cpp:416-456: NT, TN, per-head local backward, NT, TN.
void attn_bwd(Ctx& c, DType t, const RankDims& rd, const std::string& tag,
              const tess_block_shard& p, const void* x, const void* dy, float* dx_f32,
              tess_block_grads* g, bool accumulate, cudaStream_t s, const WeightPanels& wp) {
  const int64_t rows = rd.rows, hq = rd.hq, S = rd.seq, hd = rd.head_dim;
  const int64_t H = rd.heads_local, ld = 3 * hq;
  const size_t esz = dtype_size(t);
  const void* qkv = wsget(c, tag + ".qkv", rows * ld * esz);
  if (use_fused_attn(t, rd)) {
    void* o = wsget(c, tag + ".o", rows * hq * esz);
    float* lse = static_cast<float*>(wsget(c, tag + ".lse", (size_t)rd.samples_local * H * S * 4));
    float* dout32 =
        c.grid.q == 1 ? nullptr : static_cast<float*>(wsget(c, "attn.dout32", rows * hq * 4));
    void* dout = wsget(c, "attn.dout", rows * hq * esz);
    void* dqkv = wsget(c, "attn.dqkv", rows * ld * esz);
    float* delta = static_cast<float*>(wsget(c, "attn.delta", (size_t)rd.samples_local * H * S * 4));
    if (c.grid.q == 1) {
      // no row reduce: the GEMM epilogue rounds straight to bf16 (bitwise the
      // same as fp32 + convert)
      nt_product(c, t, dy, rows, rd.hin, p.w_proj, hq, out_to(dout, t), s, &wp.proj);
    } else {
      nt_product(c, t, dy, rows, rd.hin, p.w_proj, hq, out_to(dout32, DType::F32), s, &wp.proj);
      k_convert(dout32, DType::F32, dout, t, (size_t)rows * hq, s);
    }
    weight_grad(c, t, o, rows, hq, dy, rd.hin, g ? g->w_proj : nullptr, accumulate, s);
    AttnDesc a = attn_desc(rd, qkv, o, lse);
    a.dout = dout;
    a.delta = delta;
    a.dqkv = dqkv;
    run_attn(AttnPass::BwdQ, a, s);   // delta = rowsum(dO * O) -> delta, dQ -> dqkv
    run_attn(AttnPass::BwdKV, a, s);  // dK, dV -> dqkv
    nt_product(c, t, dqkv, rows, 3 * hq, p.w_qkv, rd.hin, out_to(dx_f32, DType::F32), s, &wp.qkv);
    weight_grad(c, t, x, rows, rd.hin, dqkv, 3 * hq, g ? g->w_qkv : nullptr, accumulate, s);
    return;
  }
  const void* P = wsget(c, tag + ".P", (size_t)rd.samples_local * H * S * S * esz);
  const void* o = wsget(c, tag + ".o", rows * hq * esz);
  float* dout32 = static_cast<float*>(wsget(c, "attn.dout32", rows * hq * 4));
  void* dout = t == DType::F32 ? dout32 : wsget(c, "attn.dout", rows * hq * esz);
  void* dqkv = wsget(c, "attn.dqkv", rows * ld * esz);
  const bool fused = t == DType::BF16;
  float* dP = fused ? nullptr : static_cast<float*>(wsget(c, "attn.S", (size_t)H * S * S * 4));
  float* delta = fused ? static_cast<float*>(wsget(c, "attn.delta", (size_t)H * S * 4)) : nullptr;
  void* dS = wsget(c, "attn.dS", (size_t)H * S * S * esz);
  nt_product(c, t, dy, rows, rd.hin, p.w_proj, hq, out_to(dout32, DType::F32), s, &wp.proj);
  if (t != DType::F32) k_convert(dout32, DType::F32, dout, t, (size_t)rows * hq, s);
  weight_grad(c, t, o, rows, hq, dy, rd.hin, g ? g->w_proj : nullptr, accumulate, s);
  const float scale = (float)(1.0 / std::sqrt((double)hd));
  for (int64_t smp = 0; smp < rd.samples_local; ++smp) {
    const char* q0 = static_cast<const char*>(qkv) + (size_t)smp * S * ld * esz;
    const char* do0 = static_cast<const char*>(dout) + (size_t)smp * S * hq * esz;
    char* dq0 = static_cast<char*>(dqkv) + (size_t)smp * S * ld * esz;
    const char* Ps = static_cast<const char*>(P) + (size_t)smp * H * S * S * esz;
    // dP = dO V^T (fused path: straight to dS = scale * P * (dP - delta) with
    // delta = rowsum(dO * O) = rowsum(P * dP), no fp32 dP in HBM)
    GemmDesc g1;
    g1.M = S; g1.N = S; g1.nb0 = H; g1.in = t; g1.trans_b = true;
    g1.seg[0] = {do0, q0 + 2 * hd * esz, hd};
    g1.lda = hq; g1.as0 = hd; g1.ldb = ld; g1.bs0 = 3 * hd;
    if (fused) {
      const char* o0 = static_cast<const char*>(o) + (size_t)smp * S * hq * esz;
      k_attn_delta(do0, o0, t, hq, S, H, hd, delta, s);
      g1.c = dS; g1.c_type = t; g1.ldc = S; g1.cs0 = S * S;
      g1.epi = Epi::SoftmaxBwd; g1.r = Ps; g1.ldr = S; g1.rs0 = S * S;
      g1.vec = delta; g1.vs0 = S; g1.alpha = scale;
    } else {
      g1.c = dP; g1.c_type = DType::F32; g1.ldc = S; g1.cs0 = S * S;
    }
    run_gemm(g1, s);
    // dV = P^T dO
    GemmDesc g2;
    g2.M = S; g2.N = hd; g2.nb0 = H; g2.in = t; g2.trans_a = true;
    g2.seg[0] = {Ps, do0, S};
    g2.lda = S; g2.as0 = S * S; g2.ldb = hq; g2.bs0 = hd;
    g2.c = dq0 + 2 * hd * esz; g2.c_type = t; g2.ldc = ld; g2.cs0 = 3 * hd;
    run_gemm(g2, s);
    // dS = P * (dP - rowsum(P*dP)) / sqrt(hd)
    if (!fused) k_softmax_bwd(Ps, dP, dS, t, H * S, S, scale, s);
    // dQ = dS K
    GemmDesc g3;
    g3.M = S; g3.N = hd; g3.nb0 = H; g3.in = t;
    g3.seg[0] = {dS, q0 + hd * esz, S};
    g3.lda = S; g3.as0 = S * S; g3.ldb = ld; g3.bs0 = 3 * hd;
    g3.c = dq0; g3.c_type = t; g3.ldc = ld; g3.cs0 = 3 * hd;
    run_gemm(g3, s);
    // dK = dS^T Q
    GemmDesc g4;
    g4.M = S; g4.N = hd; g4.nb0 = H; g4.in = t; g4.trans_a = true;
    g4.seg[0] = {dS, q0, S};
    g4.lda = S; g4.as0 = S * S; g4.ldb = ld; g4.bs0 = 3 * hd;
    g4.c = dq0 + hd * esz; g4.c_type = t; g4.ldc = ld; g4.cs0 = 3 * hd;
    run_gemm(g4, s);
  }
  nt_product(c, t, dqkv, rows, 3 * hq, p.w_qkv, rd.hin, out_to(dx_f32, DType::F32), s, &wp.qkv);
  weight_grad(c, t, x, rows, rd.hin, dqkv, 3 * hq, g ? g->w_qkv : nullptr, accumulate, s);
}

cudaStream_t copy_stream(Ctx& c) {
  if (!c.copy_s) TESS_CUDA(cudaStreamCreateWithFlags(&c.copy_s, cudaStreamNonBlocking));
  return c.copy_s;
}

// s waits for the pending host copy out of staging buffer `name` (if any).
void join_copy(Ctx& c, const std::string& name, cudaStream_t s) {
  auto it = c.copy_ev.find(name);
  if (it == c.copy_ev.end()) return;
  TESS_CUDA(cudaStreamWaitEvent(s, it->second, 0));
  cudaEventDestroy(it->second);
  c.copy_ev.erase(it);
  c.copy_host.erase(name);
}

// s waits for every pending host copy whose destination overlaps the host
// range [p, p + bytes) about to be read (a host output fed back as an input).
void join_host_overlap(Ctx& c, const void* p, size_t bytes, cudaStream_t s) {
  const char* lo = static_cast<const char*>(p);
  for (auto it = c.copy_host.begin(); it != c.copy_host.end();) {
    const char* a = it->second.first;
    const size_t n = it->second.second;
    const std::string name = it->first;
    ++it;
    if (a < lo + bytes && lo < a + n) join_copy(c, name, s);
  }
}

// Device staging buffer -> host on the context's copy stream, after the work
// enqueued on s so far: the copy overlaps whatever the caller enqueues next
// (the backward, or the next step's input upload: PCIe is full duplex).
void async_d2h(Ctx& c, const std::string& name, void* host, const void* dev, size_t bytes,
               cudaStream_t s) {
  join_copy(c, name, s);
  cudaStream_t cp = copy_stream(c);
  stream_dep(c, s, cp);
  TESS_CUDA(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, cp));
  cudaEvent_t ev;
  TESS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  TESS_CUDA(cudaEventRecord(ev, cp));
  c.copy_ev[name] = ev;
  c.copy_host[name] = {static_cast<const char*>(host), bytes};
}

// 1-D scheme: sum of the ranks' fp32 activation partials (proj / FF2 out,
// QKV / FF1 dgrads) over the line's depth group; a no-op for Tesseract.
void mg_allreduce(Ctx& c, float* buf, size_t n, cudaStream_t s) {
  if (!c.megatron) return;
  cudaStream_t cs = comm_stream(c, s);
  stream_dep(c, s, cs);
  coll_allreduce(c, DEPTH, buf, n, cs);
  stream_dep(c, cs, s);
}

std::string cache_tag(const Ctx& c, tess_layer_op op) {
  return "s" + std::to_string(c.cache_slot) + ".op" + std::to_string((int)op);
}

// ------------------------------------------------------------- host staging
bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

void layer_forward(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                   const tess_block_shard& p, const float* bias_row0, const void* x_in,
                   void* y_out, cudaStream_t s) {
  const int64_t rows = rd.rows, hq = rd.hin;  // activation width
  const size_t act = (size_t)rows * hq * dtype_size(t);
  const std::string tag = cache_tag(c, op);
  // Host buffers are staged through the context (x kept until backward).
  const void* x = x_in;
  if (!is_device_ptr(x_in)) {
    join_host_overlap(c, x_in, act, s);  // x may be a pending host output of ours
    void* xs = wsget(c, tag + ".xstage", act);
    TESS_CUDA(cudaMemcpyAsync(xs, x_in, act, cudaMemcpyHostToDevice, s));
    x = xs;
  }
  void* y = is_device_ptr(y_out) ? y_out : wsget(c, "stage.y", act);
  if (y != y_out) join_copy(c, "stage.y", s);  // its previous host copy must be done
  // weight panels of the whole layer go out on the comm stream first
  const WeightPanels wp =
      prefetch_weights(c, t, rd, p, op == TESS_OP_ATTENTION || op == TESS_OP_BLOCK,
                       op == TESS_OP_FEEDFORWARD || op == TESS_OP_BLOCK, s);
  switch (op) {
    case TESS_OP_LAYERNORM:
      ln_fwd(c, t, rd, tag + ".ln", x, p.ln1_gain, p.ln1_bias, p.eps, y, s);
      break;
    case TESS_OP_FEEDFORWARD:
    case TESS_OP_ATTENTION: {
      Out yo = out_to(y, t);
      float* part = nullptr;
      if (c.megatron) {  // rank partial, summed over the line
        part = static_cast<float*>(wsget(c, "mg.part", (size_t)rows * hq * 4));
        yo = out_to(part, DType::F32);
      }
      if (op == TESS_OP_FEEDFORWARD)
        ff_fwd(c, t, rd, tag + ".ff", p, x, yo, s, wp);
      else
        attn_fwd(c, t, rd, tag + ".attn", p, x, yo, s, wp);
      if (part) {
        mg_allreduce(c, part, (size_t)rows * hq, s);
        k_convert(part, DType::F32, y, t, (size_t)rows * hq, s);
      }
      break;
    }
    case TESS_OP_BIAS_ADD: {
      // ref layers.cpp:491-503: bias lives at i == 0, column broadcast.
      float* b = static_cast<float*>(wsget(c, "bias.row", hq * 4));
      if (c.coord.i == 0) {
        if (!bias_row0) fail(TESS_ERR_INVALID, "bias_add: bias_row0 required on i == 0 ranks");
        TESS_CUDA(cudaMemcpyAsync(b, bias_row0, hq * 4, cudaMemcpyDefault, s));
      }
      cudaStream_t cs = comm_stream(c, s);
      stream_dep(c, s, cs);
      coll_bcast(c, COL, 0, b, hq * 4, (uint64_t)hq, cs);
      stream_dep(c, cs, s);
      k_bias_add(x, b, y, t, rows, hq, s);
      break;
    }
    case TESS_OP_BLOCK: {
      // ref layers.cpp:460-472 (pre-norm; residuals fused into epilogues)
      void* ln1 = wsget(c, tag + ".ln1out", act);
      void* r1 = wsget(c, tag + ".r1", act);
      void* ln2 = wsget(c, tag + ".ln2out", act);
      ln_fwd(c, t, rd, tag + ".ln1", x, p.ln1_gain, p.ln1_bias, p.eps, ln1, s);
      if (c.megatron) {
        // 1-D scheme: the proj / FF2 outputs are rank partials; the residual
        // adds follow their line all-reduces
        float* part = static_cast<float*>(wsget(c, "mg.part", (size_t)rows * hq * 4));
        attn_fwd(c, t, rd, tag + ".attn", p, ln1, out_to(part, DType::F32), s, wp);
        mg_allreduce(c, part, (size_t)rows * hq, s);
        k_add(x, t, part, DType::F32, r1, t, (size_t)rows * hq, s);
        ln_fwd(c, t, rd, tag + ".ln2", r1, p.ln2_gain, p.ln2_bias, p.eps, ln2, s);
        ff_fwd(c, t, rd, tag + ".ff", p, ln2, out_to(part, DType::F32), s, wp);
        mg_allreduce(c, part, (size_t)rows * hq, s);
        k_add(r1, t, part, DType::F32, y, t, (size_t)rows * hq, s);
        break;
      }
      Out ao = out_to(r1, t);
      ao.epi = Epi::Resid;
      ao.r = x;
      attn_fwd(c, t, rd, tag + ".attn", p, ln1, ao, s, wp);
      ln_fwd(c, t, rd, tag + ".ln2", r1, p.ln2_gain, p.ln2_bias, p.eps, ln2, s);
      Out fo = out_to(y, t);
      fo.epi = Epi::Resid;
      fo.r = r1;
      ff_fwd(c, t, rd, tag + ".ff", p, ln2, fo, s, wp);
      break;
    }
    default:
      fail(TESS_ERR_INVALID, "unknown layer op");
  }
  release_weights(c, wp, s);
  join_comm(c, s);
  if (y != y_out) async_d2h(c, "stage.y", y_out, y, act, s);
  c.fwd_x[c.cache_slot * 8 + (int)op] = x;  // the backward needs the forward input
}

void layer_backward(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                    const tess_block_shard& p, const void* dy_in, void* dx_out,
                    tess_block_grads* g, bool accumulate, float* dbias, cudaStream_t s) {
  const int64_t rows = rd.rows, hq = rd.hin;  // activation width
  const size_t act = (size_t)rows * hq * dtype_size(t);
  const std::string tag = cache_tag(c, op);
  const auto it = c.fwd_x.find(c.cache_slot * 8 + (int)op);
  if (it == c.fwd_x.end() || !it->second)
    fail(TESS_ERR_SHAPE, "layer backward: missing forward cache");
  const void* x = it->second;
  const void* dy = dy_in;
  if (!is_device_ptr(dy_in)) {
    join_host_overlap(c, dy_in, act, s);
    void* ds = wsget(c, "stage.dy", act);
    TESS_CUDA(cudaMemcpyAsync(ds, dy_in, act, cudaMemcpyHostToDevice, s));
    dy = ds;
  }
  void* dx = is_device_ptr(dx_out) ? dx_out : wsget(c, "stage.dx", act);
  if (dx != dx_out) join_copy(c, "stage.dx", s);  // its previous host copy must be done
  const WeightPanels wp =
      prefetch_weights(c, t, rd, p, op == TESS_OP_ATTENTION || op == TESS_OP_BLOCK,
                       op == TESS_OP_FEEDFORWARD || op == TESS_OP_BLOCK, s);
  switch (op) {
    case TESS_OP_LAYERNORM:
      ln_bwd(c, t, rd, tag + ".ln", dy, t, x, p.ln1_gain, nullptr, t, dx, t,
             g ? g->ln1_gain : nullptr, g ? g->ln1_bias : nullptr, accumulate, s);
      break;
    case TESS_OP_FEEDFORWARD: {
      float* dxf = static_cast<float*>(wsget(c, "blk.dx32", (size_t)rows * hq * 4));
      ff_bwd(c, t, rd, tag + ".ff", p, x, dy, dxf, g, accumulate, s, wp);
      mg_allreduce(c, dxf, (size_t)rows * hq, s);
      k_convert(dxf, DType::F32, dx, t, (size_t)rows * hq, s);
      break;
    }
    case TESS_OP_ATTENTION: {
      float* dxf = static_cast<float*>(wsget(c, "blk.dx32", (size_t)rows * hq * 4));
      attn_bwd(c, t, rd, tag + ".attn", p, x, dy, dxf, g, accumulate, s, wp);
      mg_allreduce(c, dxf, (size_t)rows * hq, s);
      k_convert(dxf, DType::F32, dx, t, (size_t)rows * hq, s);
      break;
    }
    case TESS_OP_BIAS_ADD: {
      // ref layers.cpp:505-517
      float* csum = static_cast<float*>(wsget(c, "bias.colsum", hq * 4));
      float* scratch =
          static_cast<float*>(wsget(c, "bias.scratch", k_colsum_scratch_floats(rows, hq) * 4));
      ProfMem pm("colsum_kernel", (double)rows * hq * dtype_size(t) + hq * 4.0, s);
      k_colsum(dy, t, rows, hq, csum, scratch, s);
      float* red = static_cast<float*>(wsget(c, "bias.red", hq * 4));
      cudaStream_t cs = comm_stream(c, s);
      stream_dep(c, s, cs);
      coll_reduce(c, COL, 0, csum, red, hq, cs);
      if (c.coord.i == 0) {
        coll_allreduce(c, DEPTH, red, hq, cs);
        if (dbias) TESS_CUDA(cudaMemcpyAsync(dbias, red, hq * 4, cudaMemcpyDefault, cs));
      }
      if (dx != dy) TESS_CUDA(cudaMemcpyAsync(dx, dy, act, cudaMemcpyDeviceToDevice, s));
      break;
    }
    case TESS_OP_BLOCK: {
      // ref layers.cpp:474-487
      const void* r1 = wsget(c, tag + ".r1", act);
      const void* ln1 = wsget(c, tag + ".ln1out", act);
      const void* ln2 = wsget(c, tag + ".ln2out", act);
      float* dff = static_cast<float*>(wsget(c, "blk.dx32", (size_t)rows * hq * 4));
      ff_bwd(c, t, rd, tag + ".ff", p, ln2, dy, dff, g, accumulate, s, wp);
      mg_allreduce(c, dff, (size_t)rows * hq, s);  // 1-D scheme: FF1 dgrad partials
      void* dr1 = wsget(c, "blk.dr1", act);
      ln_bwd(c, t, rd, tag + ".ln2", dff, DType::F32, r1, p.ln2_gain, dy, t, dr1, t,
             g ? g->ln2_gain : nullptr, g ? g->ln2_bias : nullptr, accumulate, s);
      float* dat = static_cast<float*>(wsget(c, "blk.dattn32", (size_t)rows * hq * 4));
      attn_bwd(c, t, rd, tag + ".attn", p, ln1, dr1, dat, g, accumulate, s, wp);
      mg_allreduce(c, dat, (size_t)rows * hq, s);  // 1-D scheme: QKV dgrad partials
      ln_bwd(c, t, rd, tag + ".ln1", dat, DType::F32, x, p.ln1_gain, dr1, t, dx, t,
             g ? g->ln1_gain : nullptr, g ? g->ln1_bias : nullptr, accumulate, s);
      break;
    }
    default:
      fail(TESS_ERR_INVALID, "unknown layer op");
  }
  release_weights(c, wp, s);
  // deferred weight/LN-gradient communication completes before we return
  join_comm(c, s);
  if (dx != dx_out) async_d2h(c, "stage.dx", dx_out, dx, act, s);
}

void ctx_join(Ctx& c, cudaStream_t s) {
  join_comm(c, s);
  for (auto& kv : c.copy_ev) {
    TESS_CUDA(cudaStreamWaitEvent(s, kv.second, 0));
    cudaEventDestroy(kv.second);
  }
  c.copy_ev.clear();
  c.copy_host.clear();
}

namespace {

// Host input -> the next of two device staging buffers `name`0/1 on the
// upload stream, once that buffer's previous reader (two calls ago) is done:
// with the host enqueueing ahead of the GPU the copy overlaps the previous
// step's compute instead of queueing behind it. `used` names the buffer for
// stage_release.
const void* stage_upload(Ctx& c, const std::string& name, const void* host, size_t bytes,
                         std::string* used) {
  if (!c.up_s) TESS_CUDA(cudaStreamCreateWithFlags(&c.up_s, cudaStreamNonBlocking));
  int& par = c.stage_par[name];
  *used = name + std::to_string(par);
  par ^= 1;
  void* d = wsget(c, *used, bytes);
  const auto it = c.stage_free.find(*used);
  if (it != c.stage_free.end()) TESS_CUDA(cudaStreamWaitEvent(c.up_s, it->second, 0));
  join_host_overlap(c, host, bytes, c.up_s);  // the host range may be a pending output of ours
  TESS_CUDA(cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, c.up_s));
  return d;
}

// The staging buffer's last reader has been enqueued on s.
void stage_release(Ctx& c, const std::string& used, cudaStream_t s) {
  if (used.empty()) return;
  cudaEvent_t& e = c.stage_free[used];
  if (!e) TESS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TESS_CUDA(cudaEventRecord(e, s));
}

}  // namespace

// Forward + backward in one call with both inputs known up front (the
// reference's layer_run(op, x, dy, ...), layers.cpp:604-692, at rank level):
// host x and dy are uploaded on the context's upload stream into per-call
// double-buffered staging, x gating the forward and dy only the backward.
void layer_step(Ctx& c, tess_layer_op op, DType t, const RankDims& rd,
                const tess_block_shard& p, const float* bias_row0, const void* x, const void* dy,
                void* y, void* dx, tess_block_grads* g, bool accumulate, float* dbias,
                cudaStream_t s) {
  const size_t act = (size_t)rd.rows * rd.hin * dtype_size(t);
  std::string xb, db;
  const void* xd = x;
  if (!is_device_ptr(x)) {
    xd = stage_upload(c, cache_tag(c, op) + ".xin", x, act, &xb);
    stream_dep(c, c.up_s, s);  // the forward waits for x only
  }
  const void* dyd = dy;
  if (!is_device_ptr(dy)) dyd = stage_upload(c, "stage.dyin", dy, act, &db);
  layer_forward(c, op, t, rd, p, bias_row0, xd, y, s);
  if (dyd != dy) stream_dep(c, c.up_s, s);
  layer_backward(c, op, t, rd, p, dyd, dx, g, accumulate, dbias, s);
  stage_release(c, xb, s);
  stage_release(c, db, s);
}

// A stack of `layers` Transformer blocks, forward through every block then
// backward in reverse (the inner loops of the reference's train_toy,
// layers.cpp:1006-1026, without loss and update; BASELINE config 5's
// 24-layer stack). Block l uses forward-cache slot base + l, so all L
// forwards stay outstanding until their backward; activations between
// blocks live in context buffers. Under the 1-D scheme (c.megatron) the
// same loop drives the Megatron layer. Host x / dy are staged like
// layer_step (x gates the first forward, dy only the last backward).
void stack_step(Ctx& c, DType t, const RankDims& rd, int layers, const tess_block_shard* p,
                const void* x, const void* dy, void* y, void* dx, tess_block_grads* g,
                bool accumulate, cudaStream_t s) {
  if (layers < 1 || !p) fail(TESS_ERR_INVALID, "stack: layers must be >= 1");
  const size_t act = (size_t)rd.rows * rd.hin * dtype_size(t);
  const int base = c.cache_slot;
  std::string xb, db;
  const void* xd = x;
  if (!is_device_ptr(x)) {
    xd = stage_upload(c, "stk.xin", x, act, &xb);
    stream_dep(c, c.up_s, s);
  }
  const void* dyd = dy;
  if (!is_device_ptr(dy)) dyd = stage_upload(c, "stk.dyin", dy, act, &db);
  struct Restore {
    Ctx& c;
    int slot;
    ~Restore() { c.cache_slot = slot; }
  } restore{c, base};
  const void* cur = xd;
  for (int l = 0; l < layers; ++l) {
    c.cache_slot = base + l;
    void* out = l == layers - 1 ? y : wsget(c, "stk.a" + std::to_string(l), act);
    layer_forward(c, TESS_OP_BLOCK, t, rd, p[l], nullptr, cur, out, s);
    cur = out;
  }
  if (dyd != dy) stream_dep(c, c.up_s, s);
  const void* gin = dyd;
  for (int l = layers - 1; l >= 0; --l) {
    c.cache_slot = base + l;
    void* out = l == 0 ? dx : wsget(c, "stk.d" + std::to_string(l & 1), act);
    layer_backward(c, TESS_OP_BLOCK, t, rd, p[l], gin, out, g ? &g[l] : nullptr, accumulate,
                   nullptr, s);
    gin = out;
  }
  stage_release(c, xb, s);
  stage_release(c, db, s);
}

}  // namespace tess
