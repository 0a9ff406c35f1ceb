// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library (tesseract-
// sim, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libtsim_ref.so). Used to pin the C restatement
// (oracle/tess_oracle.c) to the reference on identical inputs and as the CPU
// baseline arm of bench.py (`--impl reference`). Never linked by the product.
//
// Each function calls the reference's public API exactly as its own
// drivers do (verify.cpp, layers.cpp:604 layer_run), converting plain
// row-major double arrays to tsim::Matrix and back. Exceptions become a
// non-zero return code with the message available from ref_last_error().
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "tsim/algorithms.hpp"
#include "tsim/error.hpp"
#include "tsim/grid.hpp"
#include "tsim/layers.hpp"
#include "tsim/matrix.hpp"
#include "tsim/rng.hpp"
#include "tsim/shard.hpp"
#include "tsim/verify.hpp"

using namespace tsim;

namespace {

thread_local std::string g_err;

Matrix to_matrix(const double* v, int64_t rows, int64_t cols) {
  Matrix m(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
  if (rows * cols > 0) std::memcpy(m.values().data(), v, sizeof(double) * rows * cols);
  return m;
}

void from_matrix(const Matrix& m, double* out) {
  if (out && m.size()) std::memcpy(out, m.values().data(), sizeof(double) * m.size());
}

void export_stats(const CommStats& s, int p, uint64_t* per_rank, uint64_t* kinds) {
  if (per_rank) {
    for (int r = 0; r < p; ++r) {
      per_rank[4 * r + 0] = s.rank_count() ? s.sent_messages(r) : 0;
      per_rank[4 * r + 1] = s.rank_count() ? s.sent_elements(r) : 0;
      per_rank[4 * r + 2] = s.rank_count() ? s.received_messages(r) : 0;
      per_rank[4 * r + 3] = s.rank_count() ? s.received_elements(r) : 0;
    }
  }
  if (kinds) {
    for (int k = 0; k < kCollectiveKindCount; ++k) {
      auto ks = s.by_kind(static_cast<CollectiveKind>(k));
      kinds[2 * k] = ks.messages;
      kinds[2 * k + 1] = ks.elements;
    }
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const DivisibilityError& e) {
    g_err = e.what();
    return 2;
  } catch (const GridError& e) {
    g_err = e.what();
    return 3;
  } catch (const SpmdError& e) {
    g_err = e.what();
    return 4;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() {
  return g_err.c_str();
}

__attribute__((visibility("default"))) void ref_random_matrix(uint64_t seed,
                                                              uint64_t stream,
                                                              int64_t rows,
                                                              int64_t cols,
                                                              double* out) {
  Rng rng = Rng::stream(seed, stream);
  from_matrix(random_matrix(rows, cols, rng), out);
}

__attribute__((visibility("default"))) int ref_checksum(int64_t rows, int64_t cols,
                                                        const double* v, char* out,
                                                        int cap) {
  std::string s = checksum(to_matrix(v, rows, cols));
  std::strncpy(out, s.c_str(), cap - 1);
  out[cap - 1] = 0;
  return 0;
}

__attribute__((visibility("default"))) int ref_grid(int q, int d, int allow, int rank,
                                                    int* coord_out, int* groups_out) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    RankCoord c = g.coord_of(rank);
    coord_out[0] = c.i;
    coord_out[1] = c.j;
    coord_out[2] = c.k;
    coord_out[3] = g.block_row(c);
    const GroupKind kinds[3] = {GroupKind::Row, GroupKind::Column, GroupKind::Depth};
    for (int f = 0; f < 3; ++f) {
      groups_out[2 * f] = g.group_index(c, kinds[f]);
      groups_out[2 * f + 1] = g.slot_in_group(c, kinds[f]);
    }
  });
}

__attribute__((visibility("default"))) int ref_grid_parse(const char* text, int allow,
                                                          int* q, int* d) {
  return guarded([&] {
    GridSpec g = GridSpec::parse(text, allow != 0);
    *q = g.q();
    *d = g.d();
  });
}

__attribute__((visibility("default"))) int ref_partition(const double* m, int64_t rows,
                                                         int64_t cols, int q, int d,
                                                         int allow, int scheme, int rank,
                                                         double* block) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    ShardedMatrix s = partition(to_matrix(m, rows, cols),
                                scheme == 0 ? Scheme::TesseractA : Scheme::TesseractB, g);
    from_matrix(s.block(rank), block);
  });
}

__attribute__((visibility("default"))) int ref_tesseract_matmul(
    int variant, int q, int d, int allow, const double* a, int64_t ar, int64_t ac,
    const double* b, int64_t br, int64_t bc, double* c, uint64_t* stats_rank,
    uint64_t* stats_kind) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    MatmulVariant v = variant == 0 ? MatmulVariant::NN
                      : variant == 1 ? MatmulVariant::NT
                                     : MatmulVariant::TN;
    AlgoResult r = tesseract_matmul(to_matrix(a, ar, ac), to_matrix(b, br, bc), g, v);
    from_matrix(r.value, c);
    export_stats(r.stats, g.size(), stats_rank, stats_kind);
  });
}

// tesseract_matmul with TesseractOptions::record_trace, trace rendered by
// write_trace (runtime.cpp:90-96) into buf.
__attribute__((visibility("default"))) int ref_tesseract_matmul_trace(
    int variant, int q, int d, int allow, const double* a, int64_t ar, int64_t ac,
    const double* b, int64_t br, int64_t bc, char* buf, int64_t cap) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    MatmulVariant v = variant == 0 ? MatmulVariant::NN
                      : variant == 1 ? MatmulVariant::NT
                                     : MatmulVariant::TN;
    TesseractOptions opt;
    opt.record_trace = true;
    AlgoResult r = tesseract_matmul(to_matrix(a, ar, ac), to_matrix(b, br, bc), g, v, opt);
    std::ostringstream os;
    write_trace(r.trace, os);
    const std::string s = os.str();
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

__attribute__((visibility("default"))) int ref_megatron_1d_linear(
    int p, const double* x, int64_t xr, int64_t xc, const double* w1, int64_t w1c,
    const double* w2, int64_t w2c, double* out, uint64_t* stats_rank, uint64_t* stats_kind) {
  return guarded([&] {
    AlgoResult r = megatron_1d_linear(to_matrix(x, xr, xc), to_matrix(w1, xc, w1c),
                                      to_matrix(w2, w1c, w2c), p);
    from_matrix(r.value, out);
    export_stats(r.stats, p, stats_rank, stats_kind);
  });
}

// load_matrix + checksum of a file written by the B200 library
__attribute__((visibility("default"))) int ref_file_checksum(const char* path, char* out,
                                                             int cap) {
  return guarded([&] {
    std::string s = checksum(load_matrix(path));
    std::strncpy(out, s.c_str(), cap - 1);
    out[cap - 1] = 0;
  });
}

// train_toy (layers.cpp:947-1036): paired serial / sharded SGD training.
__attribute__((visibility("default"))) int ref_train_toy(
    int64_t batch, int64_t seq, int64_t hidden, int64_t heads, int layers, int steps,
    double lr, uint64_t seed, int q, int d, int allow, double* serial_losses,
    double* dist_losses, double* max_div) {
  return guarded([&] {
    ToyConfig c;
    c.dims = LayerDims{static_cast<int>(batch), static_cast<int>(seq), static_cast<int>(hidden),
                       static_cast<int>(heads)};
    c.layers = layers;
    c.steps = steps;
    c.lr = lr;
    c.seed = seed;
    c.q = q;
    c.d = d;
    c.allow_d_gt_q = allow != 0;
    ToyTrainResult r = train_toy(c);
    for (int i = 0; i < steps; ++i) {
      serial_losses[i] = r.serial_loss[i];
      dist_losses[i] = r.dist_loss[i];
    }
    *max_div = r.max_divergence;
  });
}

__attribute__((visibility("default"))) int ref_tesseract_backward(
    int q, int d, int allow, const double* dc, const double* a, const double* b,
    int64_t m, int64_t k, int64_t n, double* da, double* db, uint64_t* stats_rank,
    uint64_t* stats_kind) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    DenseBackwardResult r = tesseract_backward_dense(
        to_matrix(dc, m, n), to_matrix(a, m, k), to_matrix(b, k, n), g);
    from_matrix(r.a_grad, da);
    from_matrix(r.b_grad, db);
    export_stats(r.stats, g.size(), stats_rank, stats_kind);
  });
}

__attribute__((visibility("default"))) void ref_random_block_params(
    int64_t hidden, uint64_t seed, uint64_t stream, double* const* out) {
  Rng rng = Rng::stream(seed, stream);
  BlockParams p = random_block_params(static_cast<int>(hidden), rng);
  const Matrix* ms[8] = {&p.w_qkv,    &p.w_proj,   &p.w_ff1,    &p.w_ff2,
                         &p.ln1_gain, &p.ln1_bias, &p.ln2_gain, &p.ln2_bias};
  for (int i = 0; i < 8; ++i) from_matrix(*ms[i], out[i]);
}

// layer_run (layers.cpp:604-692). params/grads in BlockParams order.
__attribute__((visibility("default"))) int ref_layer_run(
    int op, int64_t batch, int64_t seq, int64_t hidden, int64_t heads, int q, int d,
    int allow, const double* x, const double* dy, const double* const* prm,
    double eps, double* y, double* dx, double* const* grd, double* dbias,
    uint64_t* stats_rank, uint64_t* stats_kind) {
  return guarded([&] {
    GridSpec g(q, d, allow != 0);
    LayerDims dims{static_cast<int>(batch), static_cast<int>(seq),
                   static_cast<int>(hidden), static_cast<int>(heads)};
    const int64_t h = hidden, T = batch * seq;
    BlockParams p;
    p.w_qkv = to_matrix(prm[0], h, 3 * h);
    p.w_proj = to_matrix(prm[1], h, h);
    p.w_ff1 = to_matrix(prm[2], h, 4 * h);
    p.w_ff2 = to_matrix(prm[3], 4 * h, h);
    p.ln1_gain = to_matrix(prm[4], 1, h);
    p.ln1_bias = to_matrix(prm[5], 1, h);
    p.ln2_gain = to_matrix(prm[6], 1, h);
    p.ln2_bias = to_matrix(prm[7], 1, h);
    p.eps = eps;
    static const LayerOp ops[5] = {LayerOp::Feedforward, LayerOp::Attention,
                                   LayerOp::Layernorm, LayerOp::BiasAdd, LayerOp::Block};
    LayerRunResult r = layer_run(ops[op], to_matrix(x, T, h), to_matrix(dy, T, h), p,
                                 dims, g);
    from_matrix(r.y, y);
    from_matrix(r.dx, dx);
    const Matrix* gs[8] = {&r.grads.w_qkv,    &r.grads.w_proj,   &r.grads.w_ff1,
                           &r.grads.w_ff2,    &r.grads.ln1_gain, &r.grads.ln1_bias,
                           &r.grads.ln2_gain, &r.grads.ln2_bias};
    if (grd)
      for (int i = 0; i < 8; ++i)
        if (grd[i]) from_matrix(*gs[i], grd[i]);
    if (dbias && op == 3) from_matrix(r.dbias, dbias);
    export_stats(r.stats, g.size(), stats_rank, stats_kind);
  });
}

// run_verify_suite (verify.cpp:45-161) with `trials` matmul and layer trials.
__attribute__((visibility("default"))) int ref_verify_suite(int trials, int* n_cases,
                                                            int* n_pass,
                                                            double* worst) {
  return guarded([&] {
    VerifyOptions o;
    o.trials = trials;
    o.layer_trials = trials;
    auto cases = run_verify_suite(o);
    *n_cases = static_cast<int>(cases.size());
    int pass = 0;
    double w = 0;
    for (auto& c : cases) {
      pass += c.pass ? 1 : 0;
      w = std::max(w, c.max_rel_err);
    }
    *n_pass = pass;
    *worst = w;
  });
}

}  // extern "C"
