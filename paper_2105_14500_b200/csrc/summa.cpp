// SUMMA-in-depth products on the [q,q,d] grid (reference
// proj/src/algorithms.cpp:34-76), re-expressed for B200:
//  * NN: the q row/column panel broadcasts land in per-step panel buffers
//    (a rank's own panel is used in place), then ONE GEMM with q K-segments
//    accumulates every step in the same tensor-memory accumulator, instead of
//    q GEMMs plus q-1 fp32 read-modify-writes of C (reference `add`,
//    algorithms.cpp:42).
//  * NT/TN: the fp32 partial of step t is reduced to its owner slot t; with
//    q == 1 the GEMM writes straight into the caller's output with the
//    caller's epilogue.
// The collective sequence (kind, family, root, payload elements) is exactly
// the reference's, so the host meter reproduces its CommStats.
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

// Final write of an fp32 owned result into `out`.
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

}  // namespace

void nn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t ak, const void* b,
                int64_t bn, const Out& out, cudaStream_t s) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  GemmDesc g = base_desc(in, ar, bn, out);
  g.nseg = q;
  g.lda = ak;
  g.ldb = bn;
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:39: row broadcast of A(h, t) from slot t
    void* at = c.coord.j == t ? const_cast<void*>(a)
                              : c.ws->get("nn.a" + std::to_string(t), ar * ak * esz);
    coll_bcast(c, ROW, t, at, ar * ak * esz, (uint64_t)(ar * ak), s);
    // ref algorithms.cpp:40: column broadcast of B(t, j) from slot t
    void* bt = c.coord.i == t ? const_cast<void*>(b)
                              : c.ws->get("nn.b" + std::to_string(t), ak * bn * esz);
    coll_bcast(c, COL, t, bt, ak * bn * esz, (uint64_t)(ak * bn), s);
    g.seg[t] = {at, bt, ak};
  }
  if (ar > 0 && bn > 0) run_gemm(g, s);
}

void nt_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t br, const Out& out, cudaStream_t s) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  const size_t n = (size_t)ar * br;
  const bool direct = q == 1;
  const bool into_out = out.t == DType::F32 && out.epi == Epi::Store &&
                        (out.ldc == 0 || out.ldc == br);
  float* result = direct ? nullptr
                         : (into_out ? static_cast<float*>(out.c)
                                     : static_cast<float*>(c.ws->get("nt.r", n * 4)));
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:53: column broadcast of B(t, j)
    void* bt = c.coord.i == t ? const_cast<void*>(b)
                              : c.ws->get("nt.b", br * an * esz);
    coll_bcast(c, COL, t, bt, br * an * esz, (uint64_t)(br * an), s);
    if (direct) {
      GemmDesc g = base_desc(in, ar, br, out);
      g.trans_b = true;
      g.lda = an;
      g.ldb = an;
      g.seg[0] = {a, bt, an};
      if (ar > 0 && br > 0) run_gemm(g, s);
      continue;
    }
    // ref algorithms.cpp:54-56: partial, then row reduce to slot t
    float* partial = static_cast<float*>(c.ws->get("nt.p", n * 4));
    Out po;
    po.c = partial;
    po.t = DType::F32;
    GemmDesc g = base_desc(in, ar, br, po);
    g.trans_b = true;
    g.lda = an;
    g.ldb = an;
    g.seg[0] = {a, bt, an};
    if (ar > 0 && br > 0) run_gemm(g, s);
    coll_reduce(c, ROW, t, partial, result, n, s);
  }
  if (!direct && !into_out) finish(result, ar, br, out, s);
}

void tn_product(Ctx& c, DType in, const void* a, int64_t ar, int64_t an, const void* b,
                int64_t bn, bool sum_over_depth, const Out& out, cudaStream_t s) {
  check_q(c);
  const int q = c.grid.q;
  const size_t esz = dtype_size(in);
  const size_t n = (size_t)an * bn;
  const bool depth = sum_over_depth;
  const bool direct = q == 1 && (!depth || c.grid.d == 1);
  const bool into_out = out.t == DType::F32 && out.epi == Epi::Store &&
                        (out.ldc == 0 || out.ldc == bn);
  float* result = direct ? nullptr
                         : (into_out ? static_cast<float*>(out.c)
                                     : static_cast<float*>(c.ws->get("tn.r", n * 4)));
  for (int t = 0; t < q; ++t) {
    // ref algorithms.cpp:67: row broadcast of A(h, t)
    void* at = c.coord.j == t ? const_cast<void*>(a)
                              : c.ws->get("tn.a", ar * an * esz);
    coll_bcast(c, ROW, t, at, ar * an * esz, (uint64_t)(ar * an), s);
    Out po = out;
    if (!direct) {
      po = Out();
      po.c = q == 1 ? result : c.ws->get("tn.p", n * 4);
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
    // ref algorithms.cpp:69-70: column reduce of the partial to slot t
    if (!direct && q > 1) coll_reduce(c, COL, t, static_cast<float*>(po.c), result, n, s);
  }
  if (direct) return;
  // ref algorithms.cpp:72-74: depth all-reduce of the layer partial
  if (depth) coll_allreduce(c, DEPTH, result, n, s);
  if (!into_out) finish(result, an, bn, out, s);
}

}  // namespace tess
