// TEST INFRASTRUCTURE: extern "C" probes that run a reference operator and
// its tsim::b200 drop-in on the same tsim::Matrix inputs (Rng::stream(seed,
// id), rng.hpp) and compare values, CommStats (operator==, runtime.hpp:64)
// and traces (write_trace text). Called by tests/test_integration.py.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "tsim_b200.hpp"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const tsim::ShapeError& e) {
    g_err = std::string("ShapeError: ") + e.what();
    return 1;
  } catch (const tsim::DivisibilityError& e) {
    g_err = std::string("DivisibilityError: ") + e.what();
    return 2;
  } catch (const tsim::GridError& e) {
    g_err = std::string("GridError: ") + e.what();
    return 3;
  } catch (const tsim::SpmdError& e) {
    g_err = std::string("SpmdError: ") + e.what();
    return 4;
  } catch (const tsim::ConfigError& e) {
    g_err = std::string("ConfigError: ") + e.what();
    return 6;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

tsim::Matrix rnd(size_t r, size_t c, uint64_t seed, uint64_t id) {
  tsim::Rng g = tsim::Rng::stream(seed, id);
  return tsim::random_matrix(r, c, g);
}

// fp32 mode: the reference's rel_diff (matrix.cpp:138-140); bf16: relative
// Frobenius.
double err(const tsim::Matrix& v, const tsim::Matrix& r, tess_dtype t) {
  if (t == TESS_F32) return tsim::rel_diff(v, r);
  double num = 0, den = 0;
  for (size_t i = 0; i < r.size(); ++i) {
    const double d = v.values()[i] - r.values()[i];
    num += d * d;
    den += r.values()[i] * r.values()[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

std::string trace_text(const std::vector<tsim::TraceEvent>& t) {
  std::ostringstream os;
  tsim::write_trace(t, os);
  return os.str();
}

}  // namespace

extern "C" {

const char* tsb_last_error() { return g_err.c_str(); }

// out: [value err, stats equal, trace equal, trace lines]
int tsb_check_matmul(int q, int d, int allow, int variant, int dtype, int m, int n, int r,
                     int record_trace, int replicate, double* out) {
  return guarded([&] {
    const auto v = static_cast<tsim::MatmulVariant>(variant);
    tsim::GridSpec g(q, d, allow != 0);
    tsim::Matrix a = rnd(m, n, 42, 0);
    tsim::Matrix b = v == tsim::MatmulVariant::NN   ? rnd(n, r, 42, 1)
                     : v == tsim::MatmulVariant::NT ? rnd(r, n, 42, 1)
                                                    : rnd(m, r, 42, 1);
    tsim::TesseractOptions o;
    o.record_trace = record_trace != 0;
    o.meter_initial_replication = replicate != 0;
    const auto want = tsim::tesseract_matmul(a, b, g, v, o);
    const auto got = tsim::b200::tesseract_matmul(a, b, g, v, o, static_cast<tess_dtype>(dtype));
    out[0] = err(got.value, want.value, static_cast<tess_dtype>(dtype));
    out[1] = got.stats == want.stats ? 1 : 0;
    out[2] = trace_text(got.trace) == trace_text(want.trace) ? 1 : 0;
    out[3] = (double)want.trace.size();
  });
}

// Both traces of tsb_check_matmul's call (diagnostics).
int tsb_matmul_traces(int q, int d, int allow, int variant, int m, int n, int r, char* want,
                      char* got, int cap) {
  return guarded([&] {
    const auto v = static_cast<tsim::MatmulVariant>(variant);
    tsim::GridSpec g(q, d, allow != 0);
    tsim::Matrix a = rnd(m, n, 42, 0);
    tsim::Matrix b = v == tsim::MatmulVariant::NN   ? rnd(n, r, 42, 1)
                     : v == tsim::MatmulVariant::NT ? rnd(r, n, 42, 1)
                                                    : rnd(m, r, 42, 1);
    tsim::TesseractOptions o;
    o.record_trace = true;
    const std::string w = trace_text(tsim::tesseract_matmul(a, b, g, v, o).trace);
    const std::string t = trace_text(tsim::b200::tesseract_matmul(a, b, g, v, o).trace);
    std::snprintf(want, cap, "%s", w.c_str());
    std::snprintf(got, cap, "%s", t.c_str());
  });
}

// The drop-in alone (no reference call first): its status -> exception
// mapping. Returns the guarded() code of the exception class raised.
int tsb_adapter_matmul(int q, int d, int allow, int variant, int m, int n, int r) {
  return guarded([&] {
    const auto v = static_cast<tsim::MatmulVariant>(variant);
    const tsim::Matrix a = rnd(m, n, 1, 0), b = rnd(n, r, 1, 1);
    tsim::b200::tesseract_matmul(a, b, tsim::GridSpec(q, d, allow != 0), v);
  });
}

// out: [dA err, dB err, stats equal]
int tsb_check_backward(int q, int d, int allow, int dtype, int m, int k, int n, double* out) {
  return guarded([&] {
    tsim::GridSpec g(q, d, allow != 0);
    const tsim::Matrix a = rnd(m, k, 7, 0), b = rnd(k, n, 7, 1), dc = rnd(m, n, 7, 2);
    const auto want = tsim::tesseract_backward_dense(dc, a, b, g);
    const auto got = tsim::b200::tesseract_backward_dense(dc, a, b, g,
                                                         static_cast<tess_dtype>(dtype));
    out[0] = err(got.a_grad, want.a_grad, static_cast<tess_dtype>(dtype));
    out[1] = err(got.b_grad, want.b_grad, static_cast<tess_dtype>(dtype));
    out[2] = got.stats == want.stats ? 1 : 0;
  });
}

// out: [worst err over y, dx and every nonzero gradient, stats equal]
int tsb_check_layer(int op, int batch, int seq, int hidden, int heads, int q, int d, int allow,
                    int dtype, double* out) {
  return guarded([&] {
    tsim::GridSpec g(q, d, allow != 0);
    const tsim::LayerDims dims{batch, seq, hidden, heads};
    const tsim::Matrix x = rnd((size_t)batch * seq, hidden, 9, 0);
    const tsim::Matrix dy = rnd((size_t)batch * seq, hidden, 9, 2);
    tsim::Rng pr = tsim::Rng::stream(9, 100);
    const tsim::BlockParams p = tsim::random_block_params(hidden, pr);
    const auto o = static_cast<tsim::LayerOp>(op);
    const auto want = tsim::layer_run(o, x, dy, p, dims, g);
    const auto got = tsim::b200::layer_run(o, x, dy, p, dims, g, static_cast<tess_dtype>(dtype));
    const auto t = static_cast<tess_dtype>(dtype);
    double worst = std::max(err(got.y, want.y, t), err(got.dx, want.dx, t));
    const tsim::Matrix* gw[8] = {&want.grads.w_qkv,    &want.grads.w_proj,  &want.grads.w_ff1,
                                 &want.grads.w_ff2,    &want.grads.ln1_gain, &want.grads.ln1_bias,
                                 &want.grads.ln2_gain, &want.grads.ln2_bias};
    const tsim::Matrix* gg[8] = {&got.grads.w_qkv,    &got.grads.w_proj,  &got.grads.w_ff1,
                                 &got.grads.w_ff2,    &got.grads.ln1_gain, &got.grads.ln1_bias,
                                 &got.grads.ln2_gain, &got.grads.ln2_bias};
    for (int i = 0; i < 8; ++i)
      if (tsim::max_abs(*gw[i]) > 0) worst = std::max(worst, err(*gg[i], *gw[i], t));
    if (o == tsim::LayerOp::BiasAdd) worst = std::max(worst, err(got.dbias, want.dbias, t));
    out[0] = worst;
    out[1] = got.stats == want.stats ? 1 : 0;
  });
}

// SPEC.md:637 degeneracy through the drop-in: Tesseract on [q,q,1] (b200)
// against the reference's SUMMA on [q,q]. out: [value err, stats equal
// (b200 tesseract vs ref summa), stats equal (b200 summa vs ref summa)]
int tsb_check_degeneracy(int q, int m, int k, int n, int dtype, double* out) {
  return guarded([&] {
    const tsim::Matrix a = rnd(m, k, 4, 0), b = rnd(k, n, 4, 1);
    const auto want = tsim::summa_matmul(a, b, q);
    const auto t = static_cast<tess_dtype>(dtype);
    const auto got = tsim::b200::tesseract_matmul(a, b, tsim::GridSpec(q, 1),
                                                  tsim::MatmulVariant::NN, {}, t);
    const auto got2 = tsim::b200::summa_matmul(a, b, q, t);
    out[0] = err(got.value, want.value, t);
    out[1] = got.stats == want.stats ? 1 : 0;
    out[2] = got2.stats == want.stats ? 1 : 0;
  });
}

// out: [value err, stats equal]
int tsb_check_megatron(int p, int dtype, double* out) {
  return guarded([&] {
    const tsim::Matrix x = rnd(64, 128, 15, 0), w1 = rnd(128, 256, 15, 1), w2 = rnd(256, 96, 15, 2);
    const auto want = tsim::megatron_1d_linear(x, w1, w2, p);
    const auto got = tsim::b200::megatron_1d_linear(x, w1, w2, p, static_cast<tess_dtype>(dtype));
    out[0] = err(got.value, want.value, static_cast<tess_dtype>(dtype));
    out[1] = got.stats == want.stats ? 1 : 0;
  });
}

// The reference's own verify-sweep grids (verify.cpp:16-19) through the
// drop-in: every variant at small shapes, fp32. out: [worst err, all stats
// equal, cases]
int tsb_sweep(double* out) {
  return guarded([&] {
    const int grids[][3] = {{1, 1, 0}, {2, 1, 0}, {2, 2, 0}, {3, 3, 1}, {1, 2, 1}};
    double worst = 0;
    bool same = true;
    int cases = 0;
    for (const auto& gq : grids) {
      const int q = gq[0], d = gq[1];
      tsim::GridSpec g(q, d, gq[2] != 0);
      for (int v = 0; v < 3; ++v) {
        const int m = 8 * q * d, n = 4 * q, r = 6 * q;
        const auto var = static_cast<tsim::MatmulVariant>(v);
        tsim::Matrix a = rnd(m, n, 100 + cases, 0);
        tsim::Matrix b = var == tsim::MatmulVariant::NN   ? rnd(n, r, 100 + cases, 1)
                         : var == tsim::MatmulVariant::NT ? rnd(r, n, 100 + cases, 1)
                                                          : rnd(m, r, 100 + cases, 1);
        const auto want = tsim::tesseract_matmul(a, b, g, var);
        const auto got = tsim::b200::tesseract_matmul(a, b, g, var);
        worst = std::max(worst, tsim::rel_diff(got.value, want.value));
        same = same && got.stats == want.stats;
        ++cases;
      }
    }
    out[0] = worst;
    out[1] = same ? 1 : 0;
    out[2] = cases;
  });
}

}  // extern "C"
