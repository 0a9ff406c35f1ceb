// tsim::b200 -- see tsim_b200.hpp. Compiled against the reference's headers
// (proj/include) and linked with libtess.so; integration/Makefile builds it
// together with the reference's own translation units.
#include "tsim_b200.hpp"

#include <sstream>
#include <string>
#include <vector>

namespace tsim::b200 {
namespace {

// tess_status -> the reference's exception taxonomy (error.hpp:11-48).
[[noreturn]] void rethrow(tess_status s) {
  const std::string m = tess_last_error();
  switch (s) {
    case TESS_ERR_SHAPE: throw ShapeError(m);
    case TESS_ERR_DIVISIBILITY: throw DivisibilityError(m);
    case TESS_ERR_GRID: throw GridError(m);
    case TESS_ERR_CONFIG: throw ConfigError(m);
    case TESS_ERR_IO: throw IoError(m);
    case TESS_ERR_SPMD: throw SpmdError(m);
    default: throw Error("b200 backend: " + m);  // CUDA / unsupported layout / invalid
  }
}

void ok(tess_status s) {
  if (s != TESS_OK) rethrow(s);
}

// A grid the reference accepted with d > q was built with allow_d_gt_q.
int allow_of(const GridSpec& g) { return g.d() > g.q() ? 1 : 0; }

// The reference's CommStats of the last global call, rebuilt from the
// library's per-rank, per-kind send counters and per-rank receive counters.
CommStats last_stats() {
  int p = 0;
  ok(tess_global_last_stats(&p, nullptr, nullptr, 0));
  std::vector<uint64_t> sent((size_t)p * 10), recv((size_t)p * 2);
  ok(tess_global_last_stats(&p, sent.data(), recv.data(), (size_t)p));
  CommStats st(p);
  for (int r = 0; r < p; ++r) {
    for (int k = 0; k < kCollectiveKindCount; ++k) {
      const uint64_t m = sent[10 * r + 2 * k], e = sent[10 * r + 2 * k + 1];
      if (m || e) st.add_send(r, static_cast<CollectiveKind>(k), m, e);
    }
    // receives carry no kind in the reference's meter (runtime.cpp:59-64)
    if (recv[2 * r] || recv[2 * r + 1])
      st.add_recv(r, CollectiveKind::Broadcast, recv[2 * r], recv[2 * r + 1]);
  }
  return st;
}

CollectiveKind kind_of(const std::string& s) {
  if (s == "broadcast") return CollectiveKind::Broadcast;
  if (s == "reduce") return CollectiveKind::Reduce;
  if (s == "all_reduce") return CollectiveKind::AllReduce;
  if (s == "shift") return CollectiveKind::Shift;
  return CollectiveKind::PointToPoint;
}

GroupKind group_of(const std::string& s) {
  if (s == "row") return GroupKind::Row;
  if (s == "col") return GroupKind::Column;
  return GroupKind::Depth;
}

// The last global call's trace as the reference's TraceEvents.
std::vector<TraceEvent> last_trace() {
  size_t need = 0;
  ok(tess_global_last_trace(nullptr, 0, &need));
  std::string text(need, '\0');
  ok(tess_global_last_trace(text.data(), need, nullptr));
  std::vector<TraceEvent> out;
  std::istringstream is(text.c_str());
  std::string rs, kind, group;
  TraceEvent e;
  while (is >> rs >> kind >> group >> e.root >> e.bytes) {
    const auto colon = rs.find(':');
    e.rank = std::stoi(rs.substr(0, colon));
    e.step = std::stoull(rs.substr(colon + 1));
    e.kind = kind_of(kind);
    e.group = group_of(group);
    out.push_back(e);
  }
  return out;
}

// TesseractOptions::meter_initial_replication (algorithms.cpp:120-127): one
// depth broadcast of each rank's weight block from layer 0, charged before
// the product -- meter (flat counting, runtime.hpp:24-29) and, when traced,
// a step-0 event per rank with every later step shifted by one.
void charge_replication(const GridSpec& g, size_t block_elems, CommStats& st,
                        std::vector<TraceEvent>* trace) {
  const int d = g.d();
  for (int r = 0; r < g.size(); ++r) {
    const bool root = g.coord_of(r).k == 0;
    if (d > 1) {
      if (root)
        st.add_send(r, CollectiveKind::Broadcast, d - 1, (uint64_t)(d - 1) * block_elems);
      else
        st.add_recv(r, CollectiveKind::Broadcast, 1, block_elems);
    }
  }
  if (!trace) return;
  std::vector<TraceEvent> out;
  int last = -1;
  for (const TraceEvent& e : *trace) {
    if (e.rank != last) {
      out.push_back({e.rank, 0, CollectiveKind::Broadcast, GroupKind::Depth, 0,
                     block_elems * sizeof(double)});
      last = e.rank;
    }
    TraceEvent s = e;
    s.step += 1;
    out.push_back(s);
  }
  *trace = std::move(out);
}

}  // namespace

AlgoResult tesseract_matmul(const Matrix& a, const Matrix& b, const GridSpec& grid,
                            MatmulVariant variant, const TesseractOptions& options,
                            tess_dtype compute) {
  const size_t rows = variant == MatmulVariant::TN ? a.cols() : a.rows();
  const size_t cols = variant == MatmulVariant::NT ? b.rows() : b.cols();
  AlgoResult res;
  res.value = Matrix(rows, cols);
  ok(tess_set_global_trace(options.record_trace ? 1 : 0));
  ok(tess_tesseract_matmul(grid.q(), grid.d(), allow_of(grid), static_cast<tess_variant>(variant),
                           compute, a.values().data(), (int64_t)a.rows(), (int64_t)a.cols(),
                           b.values().data(), (int64_t)b.rows(), (int64_t)b.cols(),
                           res.value.values().data(), nullptr, nullptr, nullptr));
  ok(tess_set_global_trace(0));
  res.stats = last_stats();
  if (options.record_trace) res.trace = last_trace();
  if (options.meter_initial_replication && variant != MatmulVariant::TN) {
    // the weight-style operand is B: TesseractB blocks [b.rows/q, b.cols/q]
    const size_t blk = (b.rows() / grid.q()) * (b.cols() / grid.q());
    charge_replication(grid, blk, res.stats, options.record_trace ? &res.trace : nullptr);
  }
  return res;
}

DenseBackwardResult tesseract_backward_dense(const Matrix& c_grad, const Matrix& a,
                                             const Matrix& b, const GridSpec& grid,
                                             tess_dtype compute) {
  DenseBackwardResult res;
  res.a_grad = Matrix(a.rows(), a.cols());
  res.b_grad = Matrix(b.rows(), b.cols());
  ok(tess_tesseract_backward(grid.q(), grid.d(), allow_of(grid), compute,
                             c_grad.values().data(), a.values().data(), b.values().data(),
                             (int64_t)a.rows(), (int64_t)a.cols(), (int64_t)b.cols(),
                             res.a_grad.values().data(), res.b_grad.values().data(), nullptr,
                             nullptr, nullptr));
  res.stats = last_stats();
  return res;
}

AlgoResult summa_matmul(const Matrix& a, const Matrix& b, int q, tess_dtype compute) {
  // SUMMA on [q, q] is Tesseract with d = 1, TesseractA/B
  // blocks coinciding with Summa2D blocks at d = 1 (shard.cpp:68-98)
  return tesseract_matmul(a, b, GridSpec(q, 1), MatmulVariant::NN, {}, compute);
}

AlgoResult megatron_1d_linear(const Matrix& x, const Matrix& w1, const Matrix& w2, int p,
                              tess_dtype compute) {
  AlgoResult res;
  res.value = Matrix(x.rows(), w2.cols());
  ok(tess_megatron_1d_linear(p, compute, x.values().data(), (int64_t)x.rows(),
                             (int64_t)x.cols(), w1.values().data(), (int64_t)w1.rows(),
                             (int64_t)w1.cols(), w2.values().data(), (int64_t)w2.rows(),
                             (int64_t)w2.cols(), res.value.values().data(), nullptr, nullptr,
                             nullptr));
  res.stats = last_stats();
  return res;
}

LayerRunResult layer_run(LayerOp op, const Matrix& x, const Matrix& dy, const BlockParams& p,
                         const LayerDims& d, const GridSpec& grid, tess_dtype compute) {
  LayerRunResult r;
  r.y = Matrix(x.rows(), x.cols());
  r.dx = Matrix(x.rows(), x.cols());
  r.grads = zero_grads(d.hidden);
  r.dbias = Matrix(1, (size_t)d.hidden);
  const double* prm[8] = {p.w_qkv.values().data(),    p.w_proj.values().data(),
                          p.w_ff1.values().data(),    p.w_ff2.values().data(),
                          p.ln1_gain.values().data(), p.ln1_bias.values().data(),
                          p.ln2_gain.values().data(), p.ln2_bias.values().data()};
  double* grd[8] = {r.grads.w_qkv.values().data(),    r.grads.w_proj.values().data(),
                    r.grads.w_ff1.values().data(),    r.grads.w_ff2.values().data(),
                    r.grads.ln1_gain.values().data(), r.grads.ln1_bias.values().data(),
                    r.grads.ln2_gain.values().data(), r.grads.ln2_bias.values().data()};
  const tess_layer_dims dims{d.batch, d.seq, d.hidden, d.heads};
  ok(tess_layer_run(static_cast<tess_layer_op>(op), &dims, grid.q(), grid.d(), allow_of(grid),
                    compute, x.values().data(), dy.values().data(), prm, p.eps,
                    r.y.values().data(), r.dx.values().data(), grd, r.dbias.values().data(),
                    nullptr, nullptr, nullptr));
  r.stats = last_stats();
  return r;
}

}  // namespace tsim::b200
