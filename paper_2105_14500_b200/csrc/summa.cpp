// SUMMA-in-depth products on the [q,q,d] grid (reference
// proj/src/algorithms.cpp:34-76), re-expressed for B200:
//  * every collective runs on the rank's high-priority comm stream, ordered
//    against the compute stream with events, so communication overlaps the
//    GEMMs around it;
//  * NN: the q row/column panel broadcasts land in per-step panel buffers
//    (a rank's own panel is used in place; weight panels may be prefetched
//    for a whole layer, see prefetch_panels), then ONE GEMM with q
//    K-segments accumulates every step in the same tensor-memory accumulator
//    instead of q GEMMs plus q-1 fp32 read-modify-writes of C (reference
//    `add`, algorithms.cpp:42);
//  * NT/TN: the fp32 partial of step t is reduced to its owner slot t on the
//    comm stream while the GEMM of step t+1 fills the other partial buffer
//    (double buffering); with q == 1 the GEMM writes straight into the
//    caller's output with the caller's epilogue;
//  * TN with `defer`: the column reduce, depth all-reduce and the final
//    write into the gradient stay on the comm stream; the caller joins the
//    streams later (join_comm), so weight-gradient communication hides under
//    the remaining backward compute.
// The collective sequence (kind, family, root, payload elements) is the
// reference's, so the host meter reproduces its CommStats.
#include <cstdlib>
#include <string>

#include "kernels/kernels.h"
#include "ops.h"

namespace tess {

namespace {

GemmDesc base_desc(DType in, int64_t M, int64_t N, const Out& out) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.in = in;
  g.c = out.c;
  g.c_type = out.t;
  g.ldc = out.ldc ? out.ldc : N;
  g.r = out.r;
  g.ldr = out.ldr ? out.ldr : g.ldc;
  g.z = out.z;
  g.ldz = out.ldz ? out.ldz : g.ldc;
  g.alpha = out.alpha;
  g.epi = out.epi;
  return g;
}

void check_q(const Ctx& c) {
  if (c.grid.q > kMaxSegments)
    fail(TESS_ERR_UNSUPPORTED, "q > " + std::to_string(kMaxSegments) + " not supported");
}

// Final write of an fp32 owned result into `out` (on stream s).
void finish(const float* res, int64_t rows, int64_t cols, const Out& out, cudaStream_t s) {
  const int64_t ldc = out.ldc ? out.ldc : cols;
  if (ldc != cols) fail(TESS_ERR_UNSUPPORTED, "strided product outputs need q == 1");
  const size_t n = (size_t)rows * cols;
  if (out.epi == Epi::Store) {
    if (out.c != res) k_convert(res, DType::F32, out.c, out.t, n, s);
  } else if (out.epi == Epi::Accum && out.t == DType::F32) {
    k_add(out.c, DType::F32, res, DType::F32, out.c, DType::F32, n, s);
  } else {
    fail(TESS_ERR_UNSUPPORTED, "epilogue not supported after a reduction");
  }
}

// Pair reduce fused into the owner's GEMM (q == 2 groups whose backend maps
// the partner's memory; TESS_PAIR_REDUCE=0 turns it off). Every rank first
// computes the partial it contributes to its partner's result, publishes it,
// then computes its own partial with a Resid epilogue that reads the
// partner's contribution tile by tile from peer memory and adds it: the
// reduce's data movement runs inside the GEMM instead of a collective after
// it. With two members the sum is order-free, so the result is bitwise the
// slot-ascending reduce of the reference (runtime.cpp:310-312).
bool use_pair_reduce(Ctx& c, Family f) {
  static const bool env_off =
      std::getenv("TESS_PAIR_REDUCE") && std::getenv("TESS_PAIR_REDUCE")[0] == '0';
  return !env_off && c.grid.group_size(f) == 2 && c.comm->pair_capable(f);
}

// One partial GEMM of a pair reduce, or its value for an empty contraction:
// `peer` null -> C = A.B (zeros when k == 0); else C = A.B + peer.
void pair_gemm(GemmDesc g, int64_t k, float* dst, const float* peer, size_t n, cudaStream_t s) {
  if (n == 0) return;
  if (k == 0) {
    if (peer)
      TESS_CUDA(cudaMemcpyAsync(dst, peer, n * 4, cudaMemcpyDefault, s));
    else
      TESS_CUDA(cudaMemsetAsync(dst, 0, n * 4, s));
    return;
  }
  g.c = dst;
  g.c_type = DType::F32;
  g.ldc = g.N;
  g.epi = peer ? Epi::Resid : Epi::Store;
  g.r = peer;
  g.ldr = g.N;
  g.alpha = 1.0f;
  run_gemm(g, s);
}

// Where this rank's contribution goes: the backend's exported window (NCCL:
// CUDA IPC) or, for the in-process backend, any workspace buffer.
float* pair_part(Ctx& c, Family f, const std::string& tag, size_t n, cudaStream_t s) {
  float* w = c.comm_noop ? nullptr : c.comm->pair_buffer(f, n, s);
  return w ? w : static_cast<float*>(c.ws->get(tag, n * 4));
}

// Exchange + owner GEMM of a pair reduce over family f.
void pair_reduce_owner(Ctx& c, Family f, const GemmDesc& g, int64_t k, float* part,
                       float* result, size_t n, cudaStream_t s) {
  // comm_noop (exposed-comm timing): same GEMMs, the partner's buffer
  // replaced by this rank's own contribution (no exchange).
  const float* peer = c.comm_noop ? part : c.comm->pair_open(f, part, n, s);
  if (!peer) fail(TESS_ERR_SPMD, "pair reduce: partner buffer unavailable");
  pair_gemm(g, k, result, peer, n, s);
  if (!c.comm_noop) c.comm->pair_close(f, s);
}

}  // namespace

void join_comm(Ctx& c, cudaStream_t s) { stream_dep(c, comm_stream(c, s), s); }

Panels prefetch_panels(Ctx& c, Family f, const void* local, int64_t rows, int64_t cols,
                       size_t esz, const std::string& tag, cudaStream_t s) {
  Panels p;
  const int q = c.grid.q;
  check_q(c);
  cudaStream_t cs = comm_stream(c, s);
  stream_dep(c, s, cs);
  const int mine = c.grid.slot_in_group(c.coord, f);
  for (int t = 0; t < q; ++t) {
    void* buf = t == mine ? const_cast<void*>(local)
                          : c.ws->get(tag + std::to_string(t), rows * cols * esz);
    coll_bcast(c, f, t, buf, rows * cols * esz, (uint64_t)(rows * cols), cs);
    p.ptr[t] = buf;
  }
  p.valid = true;
  return p;
}

void nn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t ak, const void* b,
                int64_t bn, const Out& out, cudaStream_t s, const Panels* bp) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  cudaStream_t cs = comm_stream(c, s);
  GemmDesc g = base_desc(in, ar, bn, out);
  g.nseg = q;
  g.lda = ak;
  g.ldb = bn;
  stream_dep(c, s, cs);  // A (and B) produced on the compute stream
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:39: row broadcast of A(h, t) from slot t
    void* at = c.coord.j == t ? const_cast<void*>(a)
                              : c.ws->get("nn.a" + std::to_string(t), ar * ak * esz);
    coll_bcast(c, ROW, t, at, ar * ak * esz, (uint64_t)(ar * ak), cs);
    // ref algorithms.cpp:40: column broadcast of B(t, j) from slot t
    void* bt;
    if (bp && bp->valid) {
      bt = bp->ptr[t];
    } else {
      bt = c.coord.i == t ? const_cast<void*>(b)
                          : c.ws->get("nn.b" + std::to_string(t), ak * bn * esz);
      coll_bcast(c, COL, t, bt, ak * bn * esz, (uint64_t)(ak * bn), cs);
    }
    g.seg[t] = {at, bt, ak};
  }
  stream_dep(c, cs, s);  // panels landed
  if (ar > 0 && bn > 0) run_gemm(g, s);
  stream_dep(c, s, cs);  // panel buffers free for the next broadcasts
}

void nt_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t br, const Out& out, cudaStream_t s, const Panels* bp) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  const size_t n = (size_t)ar * br;
  cudaStream_t cs = comm_stream(c, s);
  const bool direct = q == 1;
  const bool into_out = out.t == DType::F32 && out.epi == Epi::Store &&
                        (out.ldc == 0 || out.ldc == br);
  float* result = direct ? nullptr
                         : (into_out ? static_cast<float*>(out.c)
                                     : static_cast<float*>(c.ws->get("nt.r", n * 4)));
  stream_dep(c, s, cs);
  if (!direct && use_pair_reduce(c, ROW)) {
    // collectives in the reference's order (algorithms.cpp:53-56): panels
    // move now, the row reduces are fused into the owner GEMM below
    void* bts[2];
    for (int t = 0; t < 2; ++t) {
      if (bp && bp->valid) {
        bts[t] = bp->ptr[t];
      } else {
        bts[t] = c.coord.i == t ? const_cast<void*>(b)
                                : c.ws->get("nt.b" + std::to_string(t), br * an * esz);
        coll_bcast(c, COL, t, bts[t], br * an * esz, (uint64_t)(br * an), cs);
      }
      coll_reduce_note(c, ROW, t, n);
    }
    stream_dep(c, cs, s);
    const int me = c.coord.j;
    GemmDesc g = base_desc(in, ar, br, Out());
    g.trans_b = true;
    g.lda = an;
    g.ldb = an;
    float* part = pair_part(c, ROW, "nt.p0", n, s);
    g.seg[0] = {a, bts[1 - me], an};
    pair_gemm(g, an, part, nullptr, n, s);  // contribution to the partner (slot 1-me)
    g.seg[0] = {a, bts[me], an};
    pair_reduce_owner(c, ROW, g, an, part, result, n, s);
    if (!into_out) finish(result, ar, br, out, s);
    stream_dep(c, s, cs);  // panel buffers free for the next broadcasts
    return;
  }
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:53: column broadcast of B(t, j)
    void* bt;
    if (bp && bp->valid) {
      bt = bp->ptr[t];
    } else {
      bt = c.coord.i == t ? const_cast<void*>(b)
                          : c.ws->get("nt.b" + std::to_string(t & 1), br * an * esz);
      coll_bcast(c, COL, t, bt, br * an * esz, (uint64_t)(br * an), cs);
    }
    stream_dep(c, cs, s);  // B(t) landed; partial buffer t&1 released by reduce t-2
    GemmDesc g;
    if (direct) {
      g = base_desc(in, ar, br, out);
    } else {
      Out po;
      po.c = c.ws->get("nt.p" + std::to_string(t & 1), n * 4);
      po.t = DType::F32;
      g = base_desc(in, ar, br, po);
    }
    g.trans_b = true;
    g.lda = an;
    g.ldb = an;
    g.seg[0] = {a, bt, an};
    if (ar > 0 && br > 0) run_gemm(g, s);
    if (direct) {
      coll_note_single(c, 1, ROW, t, n);  // the reference's 1-member row reduce
      continue;
    }
    stream_dep(c, s, cs);
    // ref algorithms.cpp:55-56: row reduce of the partial to slot t (on the
    // comm stream, overlapping the next step's GEMM)
    coll_reduce(c, ROW, t, static_cast<float*>(g.c), result, n, cs);
  }
  if (direct) return;
  if (!into_out) finish(result, ar, br, out, cs);
  stream_dep(c, cs, s);  // owned result ready for the consumer
}

void tn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t bn, bool sum_over_depth, const Out& out, cudaStream_t s, bool defer) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  const size_t n = (size_t)an * bn;
  cudaStream_t cs = comm_stream(c, s);
  const bool depth = sum_over_depth;
  const bool direct = q == 1 && (!depth || c.grid.d == 1);
  const bool into_out = out.t == DType::F32 && out.epi == Epi::Store &&
                        (out.ldc == 0 || out.ldc == bn);
  // A deferred result outlives this call on the comm stream: give it a buffer
  // of its own (keyed by the destination) so the next product cannot race it.
  const std::string rname = defer ? "tn.r." + std::to_string(reinterpret_cast<uintptr_t>(out.c))
                                  : std::string("tn.r");
  float* result = direct ? nullptr
                         : (into_out ? static_cast<float*>(out.c)
                                     : static_cast<float*>(c.ws->get(rname, n * 4)));
  stream_dep(c, s, cs);
  if (!direct && use_pair_reduce(c, COL)) {
    void* ats[2];
    for (int t = 0; t < 2; ++t) {
      // ref algorithms.cpp:67-70: row broadcast of A(h, t), column reduce to
      // slot t (fused into the owner GEMM below)
      ats[t] = c.coord.j == t ? const_cast<void*>(a)
                              : c.ws->get("tn.a" + std::to_string(t), ar * an * esz);
      coll_bcast(c, ROW, t, ats[t], ar * an * esz, (uint64_t)(ar * an), cs);
      coll_reduce_note(c, COL, t, n);
    }
    stream_dep(c, cs, s);
    const int me = c.coord.i;
    GemmDesc g = base_desc(in, an, bn, Out());
    g.trans_a = true;
    g.lda = an;
    g.ldb = bn;
    float* part = pair_part(c, COL, "tn.p0", n, s);
    g.seg[0] = {ats[1 - me], b, ar};
    pair_gemm(g, ar, part, nullptr, n, s);
    g.seg[0] = {ats[me], b, ar};
    pair_reduce_owner(c, COL, g, ar, part, result, n, s);
    stream_dep(c, s, cs);
    // ref algorithms.cpp:72-74: depth all-reduce of the layer partial
    if (depth) coll_allreduce(c, DEPTH, result, n, cs);
    if (!into_out) finish(result, an, bn, out, cs);
    if (!defer) stream_dep(c, cs, s);
    return;
  }
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:67: row broadcast of A(h, t)
    void* at = c.coord.j == t ? const_cast<void*>(a)
                              : c.ws->get("tn.a" + std::to_string(t & 1), ar * an * esz);
    coll_bcast(c, ROW, t, at, ar * an * esz, (uint64_t)(ar * an), cs);
    stream_dep(c, cs, s);
    Out po = out;
    if (!direct) {
      po = Out();
      po.c = q == 1 ? result : c.ws->get("tn.p" + std::to_string(t & 1), n * 4);
      po.t = DType::F32;
    }
    GemmDesc g = base_desc(in, an, bn, po);
    g.trans_a = true;
    g.lda = an;
    g.ldb = bn;
    g.seg[0] = {at, b, ar};
    if (an > 0 && bn > 0) {
      if (ar > 0) {
        run_gemm(g, s);
      } else if (po.epi == Epi::Store) {
        TESS_CUDA(cudaMemsetAsync(po.c, 0, n * dtype_size(po.t), s));
      }
    }
    if (q == 1) {
      coll_note_single(c, 1, COL, t, n);  // the reference's 1-member column reduce
      continue;
    }
    stream_dep(c, s, cs);
    // ref algorithms.cpp:69-70: column reduce of the partial to slot t
    coll_reduce(c, COL, t, static_cast<float*>(po.c), result, n, cs);
  }
  if (direct) {
    // [1,1,1]: the reference's 1-member depth all-reduce (traced, moves nothing)
    if (depth) coll_note_single(c, 2, DEPTH, 0, n);
    return;
  }
  stream_dep(c, s, cs);  // (q == 1) the GEMM wrote `result` on the compute stream
  // ref algorithms.cpp:72-74: depth all-reduce of the layer partial
  if (depth) coll_allreduce(c, DEPTH, result, n, cs);
  if (!into_out) finish(result, an, bn, out, cs);
  if (!defer) stream_dep(c, cs, s);
}

}  // namespace tess
