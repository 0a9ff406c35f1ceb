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
#include <algorithm>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

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
  g.bias = out.bias;
  g.drop_p = out.drop_p;
  g.drop_seed = out.drop_seed;
  g.drop_row0 = out.drop_row0;
  g.drop_col0 = out.drop_col0;
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

// SM-free panel transport usable for family f with `in` operands: the GEMM
// may then start before remote panels land (tcgen05 GEMMs wait on device
// flags; the fp32 CUDA-core path does not, so it keeps the event order).
bool panels_async(Ctx& c, Family f, DType in) {
  return c.grid.group_size(f) > 1 && !c.comm_noop && in == DType::BF16 &&
         c.comm->panel_async(f);
}

// Rows per transfer chunk of a panel with `rows` stored rows: about
// 32 / q chunks (<= 16) of whole `align` rows (the GEMM's tile rows, or its
// k-block when the panel's rows are the contraction), so the GEMM's first
// tiles start once their chunk landed instead of the whole panel.
int64_t chunk_rows_for(int64_t rows, int64_t align, int q) {
  const int64_t target = std::min<int64_t>(16, 32 / std::max(q, 1));
  int64_t cr = (rows + target - 1) / target;
  cr = ((cr + align - 1) / align) * align;
  return std::max<int64_t>(cr, align);
}

// One panel of a SUMMA step over family f from slot t: the receiver's copy
// may be in flight (flags); `local` is this rank's own panel (used in place
// at the root). Returns the panel pointer; records the flags in *flags /
// *epoch and the link in `links` when the panel is remote.
const void* panel_step(Ctx& c, Family f, int t, const std::string& tag, const void* local,
                       int64_t rows, int64_t cols, size_t esz, int64_t chunk_rows,
                       cudaStream_t cs, const uint32_t** flags, uint32_t* epoch,
                       std::vector<std::pair<Family, std::string>>& links) {
  const bool root = c.grid.slot_in_group(c.coord, f) == t;
  const size_t bytes = (size_t)(rows * cols) * esz;
  void* dst = root || c.comm->panel_owns_buffers() ? nullptr : c.ws->get(tag, bytes);
  const Comm::PanelRecv r =
      coll_bcast_panel(c, f, t, tag, root ? local : nullptr, dst, bytes, (uint64_t)(rows * cols),
                       (size_t)(chunk_rows > 0 ? chunk_rows : rows) * cols * esz, cs);
  if (r.flags) {
    *flags = r.flags;
    *epoch = r.epoch;
    links.push_back({f, tag});
  }
  return r.buf;
}

void release_links(Ctx& c, const std::vector<std::pair<Family, std::string>>& links,
                   cudaStream_t s) {
  for (const auto& l : links) c.comm->panel_done(l.first, l.second, s);
}

}  // namespace

void release_panels(Ctx& c, const Panels& p, cudaStream_t s) {
  if (!p.valid || p.tag.empty()) return;
  for (int t = 0; t < c.grid.q; ++t)
    if (p.flags[t]) c.comm->panel_done(p.fam, p.tag + std::to_string(t), s);
}

void join_comm(Ctx& c, cudaStream_t s) { stream_dep(c, comm_stream(c, s), s); }

Panels prefetch_panels(Ctx& c, Family f, const void* local, int64_t rows, int64_t cols,
                       size_t esz, const std::string& tag, cudaStream_t s) {
  Panels p;
  const int q = c.grid.q;
  check_q(c);
  cudaStream_t cs = comm_stream(c, s);
  stream_dep(c, s, cs);
  const int mine = c.grid.slot_in_group(c.coord, f);
  // bf16 weight panels (the only prefetched operands) may use the SM-free
  // transport: their GEMMs then wait on the panels' flags, not on cs
  const bool async = panels_async(c, f, esz == 2 ? DType::BF16 : DType::F32);
  std::vector<std::pair<Family, std::string>> links;
  for (int t = 0; t < q; ++t) {
    if (async) {
      p.ptr[t] = const_cast<void*>(panel_step(c, f, t, tag + std::to_string(t), local, rows, cols,
                                              esz, 0, cs, &p.flags[t], &p.epoch[t], links));
      continue;
    }
    void* buf = t == mine ? const_cast<void*>(local)
                          : c.ws->get(tag + std::to_string(t), rows * cols * esz);
    coll_bcast(c, f, t, buf, rows * cols * esz, (uint64_t)(rows * cols), cs);
    p.ptr[t] = buf;
  }
  p.valid = true;
  p.fam = f;
  p.tag = async ? tag : std::string();
  return p;
}

// Are all of a prefetched operand's remote panels flag-tracked?
bool panels_flagged(const Ctx& c, const Panels* bp, Family f) {
  if (!bp || !bp->valid || bp->tag.empty()) return false;
  const int mine = c.grid.slot_in_group(c.coord, f);
  for (int t = 0; t < c.grid.q; ++t)
    if (t != mine && !bp->flags[t]) return false;
  return true;
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
  // Both families are probed on every rank (the probes are collective).
  const bool pa = panels_async(c, ROW, in);
  const bool pb = panels_async(c, COL, in);
  const bool prefetched = bp && bp->valid;
  bool join = false;  // some panel moved by an event-ordered collective
  std::vector<std::pair<Family, std::string>> links;
  const int64_t crows = pa ? chunk_rows_for(ar, 256, q) : 0;
  stream_dep(c, s, cs);  // A (and B) produced on the compute stream
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:39: row broadcast of A(h, t) from slot t
    const void* at;
    if (pa) {
      at = panel_step(c, ROW, t, "nn.a" + std::to_string(t), a, ar, ak, esz, crows, cs,
                      &g.ready.a_flags[t], &g.ready.a_epoch[t], links);
    } else {
      void* buf = c.coord.j == t ? const_cast<void*>(a)
                                 : c.ws->get("nn.a" + std::to_string(t), ar * ak * esz);
      coll_bcast(c, ROW, t, buf, ar * ak * esz, (uint64_t)(ar * ak), cs);
      at = buf;
      join = join || q > 1;
    }
    // ref algorithms.cpp:40: column broadcast of B(t, j) from slot t
    const void* bt;
    if (prefetched) {
      bt = bp->ptr[t];
      g.ready.b_flags[t] = bp->flags[t];
      g.ready.b_epoch[t] = bp->epoch[t];
    } else if (pb) {
      bt = panel_step(c, COL, t, "nn.b" + std::to_string(t), b, ak, bn, esz, 0, cs,
                      &g.ready.b_flags[t], &g.ready.b_epoch[t], links);
    } else {
      void* buf = c.coord.i == t ? const_cast<void*>(b)
                                 : c.ws->get("nn.b" + std::to_string(t), ak * bn * esz);
      coll_bcast(c, COL, t, buf, ak * bn * esz, (uint64_t)(ak * bn), cs);
      bt = buf;
      join = join || q > 1;
    }
    g.seg[t] = {at, bt, ak};
  }
  if (prefetched && !panels_flagged(c, bp, COL)) join = join || q > 1;
  if (join) stream_dep(c, cs, s);  // event order: every panel landed
  if (pa) {
    g.ready.chunk_rows = crows;
    g.ready.chunks = (int)((ar + crows - 1) / crows);
  }
  if (ar > 0 && bn > 0) run_gemm(g, s);
  release_links(c, links, s);
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
  const bool pb = !direct && panels_async(c, COL, in);
  const bool prefetched = bp && bp->valid;
  if (!direct && use_pair_reduce(c, ROW)) {
    // collectives in the reference's order (algorithms.cpp:53-56): panels
    // move now, the row reduces are fused into the owner GEMM below
    const void* bts[2];
    const uint32_t* bfl[2] = {nullptr, nullptr};
    uint32_t bep[2] = {0, 0};
    bool join = false;
    std::vector<std::pair<Family, std::string>> links;
    for (int t = 0; t < 2; ++t) {
      if (prefetched) {
        bts[t] = bp->ptr[t];
        bfl[t] = bp->flags[t];
        bep[t] = bp->epoch[t];
      } else if (pb) {
        bts[t] = panel_step(c, COL, t, "nt.b" + std::to_string(t), b, br, an, esz, 0, cs, &bfl[t],
                            &bep[t], links);
      } else {
        void* buf = c.coord.i == t ? const_cast<void*>(b)
                                   : c.ws->get("nt.b" + std::to_string(t), br * an * esz);
        coll_bcast(c, COL, t, buf, br * an * esz, (uint64_t)(br * an), cs);
        bts[t] = buf;
        join = true;
      }
      coll_reduce_note(c, ROW, t, n);
    }
    if (join || (prefetched && !panels_flagged(c, bp, COL))) stream_dep(c, cs, s);
    const int me = c.coord.j;
    GemmDesc g = base_desc(in, ar, br, Out());
    g.trans_b = true;
    g.lda = an;
    g.ldb = an;
    float* part = pair_part(c, ROW, "nt.p0", n, s);
    g.seg[0] = {a, bts[1 - me], an};
    g.ready.b_flags[0] = bfl[1 - me];
    g.ready.b_epoch[0] = bep[1 - me];
    pair_gemm(g, an, part, nullptr, n, s);  // contribution to the partner (slot 1-me)
    g.seg[0] = {a, bts[me], an};
    g.ready.b_flags[0] = bfl[me];
    g.ready.b_epoch[0] = bep[me];
    pair_reduce_owner(c, ROW, g, an, part, result, n, s);
    release_links(c, links, s);
    if (!into_out) finish(result, ar, br, out, s);
    stream_dep(c, s, cs);  // panel buffers free for the next broadcasts
    return;
  }
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:53: column broadcast of B(t, j)
    const void* bt;
    if (bp && bp->valid) {
      bt = bp->ptr[t];
    } else {
      void* buf = c.coord.i == t ? const_cast<void*>(b)
                                 : c.ws->get("nt.b" + std::to_string(t & 1), br * an * esz);
      coll_bcast(c, COL, t, buf, br * an * esz, (uint64_t)(br * an), cs);
      bt = buf;
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
    // The activation panels A(h, t) may use the SM-free transport in chunks
    // of the contraction (their rows): the GEMMs start on the first chunk.
    const bool pa = panels_async(c, ROW, in);
    const int64_t crows = pa ? chunk_rows_for(ar, 64, 2) : 0;
    const void* ats[2];
    const uint32_t* afl[2] = {nullptr, nullptr};
    uint32_t aep[2] = {0, 0};
    std::vector<std::pair<Family, std::string>> links;
    for (int t = 0; t < 2; ++t) {
      // ref algorithms.cpp:67-70: row broadcast of A(h, t), column reduce to
      // slot t (fused into the owner GEMM below)
      if (pa) {
        ats[t] = panel_step(c, ROW, t, "tn.a" + std::to_string(t), a, ar, an, esz, crows, cs,
                            &afl[t], &aep[t], links);
      } else {
        void* buf = c.coord.j == t ? const_cast<void*>(a)
                                   : c.ws->get("tn.a" + std::to_string(t), ar * an * esz);
        coll_bcast(c, ROW, t, buf, ar * an * esz, (uint64_t)(ar * an), cs);
        ats[t] = buf;
      }
      coll_reduce_note(c, COL, t, n);
    }
    if (!pa) stream_dep(c, cs, s);
    const int me = c.coord.i;
    GemmDesc g = base_desc(in, an, bn, Out());
    g.trans_a = true;
    g.lda = an;
    g.ldb = bn;
    if (pa) {
      g.ready.chunk_rows = crows;
      g.ready.chunks = (int)((ar + crows - 1) / crows);
    }
    float* part = pair_part(c, COL, "tn.p0", n, s);
    g.seg[0] = {ats[1 - me], b, ar};
    g.ready.a_flags[0] = afl[1 - me];
    g.ready.a_epoch[0] = aep[1 - me];
    pair_gemm(g, ar, part, nullptr, n, s);
    g.seg[0] = {ats[me], b, ar};
    g.ready.a_flags[0] = afl[me];
    g.ready.a_epoch[0] = aep[me];
    pair_reduce_owner(c, COL, g, ar, part, result, n, s);
    release_links(c, links, s);
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
