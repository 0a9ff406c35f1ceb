// Whole-matrix operators over host fp64 buffers (reference value-semantics
// API): tesseract_matmul (algorithms.cpp:131-186), tesseract_backward_dense
// (algorithms.cpp:188-242) and layer_run (layers.cpp:604-692).
//
// partition -> one host thread per rank driving its own tess_ctx over the
// in-process backend (the SpmdRunner of runtime.cpp:534-554) -> combine with
// the reference's replica checks (shard.cpp:139-183, layers.cpp:184-228).
// Inputs are rounded once to the compute dtype on the device.
#include <array>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

#include "kernels/kernels.h"
#include "ops.h"

using namespace tess;

namespace tess {
extern thread_local std::string g_last_error;
}

namespace {

// What the last global call on this host thread metered and traced: the
// per-rank, per-kind send counters and per-rank receive counters from which
// the reference's CommStats can be rebuilt exactly with add_send / add_recv
// (runtime.hpp:56-59), and the concatenated per-rank trace (the order of
// SpmdRunner::take_trace, runtime.cpp:149-156).
struct LastRun {
  int p = 0;
  std::vector<uint64_t> sent;  // [p][5][2] messages, elements per CollectiveKind
  std::vector<uint64_t> recv;  // [p][2]
  std::string trace;
};
thread_local LastRun g_last_run;
thread_local bool g_global_trace = false;
// tess_set_global_fault: armed for the next global call of this thread
thread_local int g_fault_kind = 0, g_fault_rank = 0;
thread_local int64_t g_fault_at = -1;
thread_local bool g_perturb_next = false;

struct Runner {
  Grid g;
  std::vector<int> devs;
  std::vector<tess_ctx*> ctx;

  Runner(int q, int d, bool allow, const int* devices) : g(q, d, allow) {
    int cur = 0;
    TESS_CUDA(cudaGetDevice(&cur));
    devs.resize(g.size());
    for (int r = 0; r < g.size(); ++r) devs[r] = devices ? devices[r] : cur;
    ctx.resize(g.size(), nullptr);
    if (tess_init_local(q, d, allow, devs.data(), ctx.data()) != TESS_OK)
      fail(TESS_ERR_CUDA, std::string("init_local: ") + g_last_error);
    for (auto* c : ctx) c->trace_on = g_global_trace;
    g_last_run = LastRun{};
    if (g_fault_kind == TESS_FAULT_RANK_FAIL || g_fault_kind == TESS_FAULT_SKIP_COLLECTIVE) {
      if (g_fault_rank >= 0 && g_fault_rank < g.size()) {
        ctx[g_fault_rank]->fault_kind = g_fault_kind;
        ctx[g_fault_rank]->fault_at = g_fault_at;
      }
      g_fault_kind = 0;
    }
  }
  ~Runner() {
    for (auto* c : ctx)
      if (c) tess_destroy(c);
  }

  std::vector<int> unique_devices() const {
    std::vector<int> u;
    for (int dv : devs)
      if (std::find(u.begin(), u.end(), dv) == u.end()) u.push_back(dv);
    return u;
  }

  // Runs fn on every rank in its own thread; the first root-cause failure
  // is rethrown (rank failures become SpmdError with the coordinate, like
  // runtime.cpp:540-553; CUDA / unsupported-layout errors keep their status).
  void run(const std::function<void(Ctx&, cudaStream_t)>& fn) {
    std::mutex mu;
    bool have = false;
    tess_status st = TESS_OK;
    std::string msg;
    int first_rank = -1;
    std::vector<std::thread> th;
    for (int r = 0; r < g.size(); ++r) {
      th.emplace_back([&, r] {
        Ctx& c = *ctx[r];
        cudaStream_t s = nullptr;
        try {
          TESS_CUDA(cudaSetDevice(c.device));
          TESS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
          fn(c, s);
          ctx_join(c, s);  // host copies of layer outputs + deferred collectives
          TESS_CUDA(cudaStreamSynchronize(s));
          local_world_rank_finished(c.world.get(), c.rank);
        } catch (const tess::Error& e) {
          local_world_fail(c.world.get(), e.what());
          std::lock_guard<std::mutex> lk(mu);
          const bool aborted = std::string(e.what()).rfind("aborted:", 0) == 0;
          if (!have || (!aborted && msg.rfind("aborted:", 0) == 0)) {
            have = true;
            st = e.status;
            msg = e.what();
            first_rank = r;
          }
        }
        if (s) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
        }
      });
    }
    for (auto& t : th) t.join();
    if (have) {
      const Coord c = g.coord_of(first_rank);
      const std::string where = "rank (" + std::to_string(c.i) + "," + std::to_string(c.j) +
                                "," + std::to_string(c.k) + ") failed: ";
      if (st == TESS_ERR_CUDA || st == TESS_ERR_UNSUPPORTED) fail(st, where + msg);
      fail(TESS_ERR_SPMD, where + msg);
    }
  }

  void stats(uint64_t* sr, uint64_t* sk) const {
    LastRun& L = g_last_run;
    L.p = g.size();
    L.sent.assign((size_t)L.p * 10, 0);
    L.recv.assign((size_t)L.p * 2, 0);
    std::vector<TraceEvent> all;
    for (int r = 0; r < g.size(); ++r) {
      const Meter& m = ctx[r]->meter;
      for (int k = 0; k < 5; ++k) {
        L.sent[10 * r + 2 * k] = m.kind[k][0];
        L.sent[10 * r + 2 * k + 1] = m.kind[k][1];
      }
      L.recv[2 * r] = m.recv_msgs;
      L.recv[2 * r + 1] = m.recv_elems;
      all.insert(all.end(), ctx[r]->trace.begin(), ctx[r]->trace.end());
    }
    L.trace = trace_text(all);
    if (sr)
      for (int r = 0; r < g.size(); ++r) {
        const Meter& m = ctx[r]->meter;
        sr[4 * r + 0] = m.sent_msgs;
        sr[4 * r + 1] = m.sent_elems;
        sr[4 * r + 2] = m.recv_msgs;
        sr[4 * r + 3] = m.recv_elems;
      }
    if (sk) {
      std::memset(sk, 0, sizeof(uint64_t) * 10);
      for (int r = 0; r < g.size(); ++r)
        for (int k = 0; k < 5; ++k) {
          sk[2 * k] += ctx[r]->meter.kind[k][0];
          sk[2 * k + 1] += ctx[r]->meter.kind[k][1];
        }
    }
  }
};

// Device copy of a host fp64 matrix rounded to `t`, one per device.
struct DevMat {
  std::vector<std::pair<int, void*>> per_dev;
  ~DevMat() {
    for (auto& pd : per_dev) {
      cudaSetDevice(pd.first);
      cudaFree(pd.second);
    }
  }
  void* on(int dev) const {
    for (auto& pd : per_dev)
      if (pd.first == dev) return pd.second;
    fail(TESS_ERR_INVALID, "matrix not resident on device");
  }
};

void upload(DevMat& m, const std::vector<int>& devs, const double* host, size_t n, DType t) {
  for (int dv : devs) {
    TESS_CUDA(cudaSetDevice(dv));
    void* d64 = nullptr;
    void* dt = nullptr;
    TESS_CUDA(cudaMalloc(&d64, std::max<size_t>(n, 1) * 8));
    TESS_CUDA(cudaMalloc(&dt, std::max<size_t>(n, 1) * dtype_size(t)));
    if (n) {
      TESS_CUDA(cudaMemcpy(d64, host, n * 8, cudaMemcpyHostToDevice));
      k_convert(d64, DType::F64, dt, t, n, nullptr);
    }
    TESS_CUDA(cudaDeviceSynchronize());
    TESS_CUDA(cudaFree(d64));
    m.per_dev.push_back({dv, dt});
  }
}

void call(tess_status s) {
  if (s != TESS_OK) fail(s, g_last_error);
}

// Local block of a global device matrix, in workspace `name`.
void* take_block(Ctx& c, tess_scheme sch, DType t, const void* global, int64_t rows,
                 int64_t cols, const std::string& name, cudaStream_t s) {
  const int64_t rb = sch == TESS_SCHEME_A ? rows / (c.grid.q * c.grid.d) : rows / c.grid.q;
  const int64_t cb = cols / c.grid.q;
  void* local = c.ws->get(name, (size_t)rb * cb * dtype_size(t));
  call(tess_partition(&c, sch, t == DType::F32 ? TESS_F32 : TESS_BF16, global, rows, cols, local, s));
  return local;
}

float h2f(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Copies a rank's device block (dtype t) to a host float vector.
std::vector<float> fetch(const void* dev, size_t n, DType t, cudaStream_t s) {
  std::vector<float> out(n);
  if (!n) return out;
  if (t == DType::F32) {
    TESS_CUDA(cudaMemcpyAsync(out.data(), dev, n * 4, cudaMemcpyDeviceToHost, s));
    TESS_CUDA(cudaStreamSynchronize(s));
  } else {
    std::vector<uint16_t> tmp(n);
    TESS_CUDA(cudaMemcpyAsync(tmp.data(), dev, n * 2, cudaMemcpyDeviceToHost, s));
    TESS_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < n; ++i) out[i] = h2f(tmp[i]);
  }
  return out;
}

// Host combine of per-rank blocks (ref shard.cpp:139-183): TesseractA blocks
// placed at (h, j); TesseractB blocks at (i, j) with k > 0 replicas required
// to be bit-identical to k == 0.
void combine(const Grid& g, tess_scheme sch, const std::vector<std::vector<float>>& blocks,
             int64_t rows, int64_t cols, double* out) {
  const int q = g.q, d = g.d;
  const int64_t rb = sch == TESS_SCHEME_A ? rows / ((int64_t)q * d) : rows / q;
  const int64_t cb = cols / q;
  for (int r = 0; r < g.size(); ++r) {
    const Coord c = g.coord_of(r);
    if (sch == TESS_SCHEME_B && c.k > 0) {
      const auto& ref = blocks[g.rank_of({c.i, c.j, 0})];
      if (std::memcmp(ref.data(), blocks[r].data(), ref.size() * 4) != 0)
        fail(TESS_ERR_SHAPE, "combine: replica divergence at rank (" + std::to_string(c.i) + "," +
                                 std::to_string(c.j) + "," + std::to_string(c.k) + ")");
      continue;
    }
    const int64_t r0 = (sch == TESS_SCHEME_A ? g.block_row(c) : c.i) * rb;
    const int64_t c0 = (int64_t)c.j * cb;
    for (int64_t i = 0; i < rb; ++i)
      for (int64_t j = 0; j < cb; ++j) out[(r0 + i) * cols + c0 + j] = blocks[r][i * cb + j];
  }
}

void require_div(int64_t v, int64_t by, const char* scheme, const char* dim) {
  if (by == 0 || v % by != 0)
    fail(TESS_ERR_DIVISIBILITY, std::string(scheme) + ": " + dim + " (" + std::to_string(v) +
                                    ") not divisible by " + std::to_string(by));
}

DType compute_type(tess_dtype t) {
  if (t == TESS_F32) return DType::F32;
  if (t == TESS_BF16) return DType::BF16;
  fail(TESS_ERR_UNSUPPORTED, "compute dtype must be TESS_F32 or TESS_BF16");
}

template <typename F>
tess_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return TESS_OK;
  } catch (const tess::Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TESS_ERR_INVALID;
  }
}

}  // namespace

extern "C" {

tess_status tess_tesseract_matmul(int q, int d, int allow, tess_variant v, tess_dtype compute,
                                  const double* a, int64_t ar, int64_t ac, const double* b,
                                  int64_t br, int64_t bc, double* c, const int* devices,
                                  uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    Grid g(q, d, allow != 0);
    // shape checks (ref algorithms.cpp:23-31, 153-158, 170-174)
    int64_t cr = 0, cc = 0;
    tess_scheme bsch = TESS_SCHEME_B, csch = TESS_SCHEME_A;
    if (v == TESS_NN) {
      if (ac != br) fail(TESS_ERR_SHAPE, "tesseract_matmul(nn): A.cols (" + std::to_string(ac) +
                                             ") != B.rows (" + std::to_string(br) + ")");
      cr = ar, cc = bc;
    } else if (v == TESS_NT) {
      if (ac != bc) fail(TESS_ERR_SHAPE, "tesseract_matmul(nt): A.cols (" + std::to_string(ac) +
                                             ") != B.cols (" + std::to_string(bc) + ")");
      cr = ar, cc = br;
    } else if (v == TESS_TN) {
      if (ar != br) fail(TESS_ERR_SHAPE, "tesseract_matmul(tn): A.rows (" + std::to_string(ar) +
                                             ") != B.rows (" + std::to_string(br) + ")");
      cr = ac, cc = bc;
      bsch = TESS_SCHEME_A;
      csch = TESS_SCHEME_B;
    } else {
      fail(TESS_ERR_INVALID, "bad variant");
    }
    // partition divisibility (ref shard.cpp:74-98)
    require_div(ar, (int64_t)q * d, "tesseract-a", "rows");
    require_div(ac, q, "tesseract-a", "cols");
    require_div(br, bsch == TESS_SCHEME_A ? (int64_t)q * d : q,
                bsch == TESS_SCHEME_A ? "tesseract-a" : "tesseract-b", "rows");
    require_div(bc, q, bsch == TESS_SCHEME_A ? "tesseract-a" : "tesseract-b", "cols");
    Runner R(q, d, allow != 0, devices);
    DevMat dA, dB;
    upload(dA, R.unique_devices(), a, (size_t)ar * ac, t);
    upload(dB, R.unique_devices(), b, (size_t)br * bc, t);
    const int p = g.size();
    std::vector<std::vector<float>> blocks(p);
    R.run([&](Ctx& x, cudaStream_t s) {
      void* la = take_block(x, TESS_SCHEME_A, t, dA.on(x.device), ar, ac, "g.a", s);
      void* lb = take_block(x, bsch, t, dB.on(x.device), br, bc, "g.b", s);
      const int64_t lar = ar / ((int64_t)q * d), lac = ac / q;
      const int64_t lbr = bsch == TESS_SCHEME_A ? br / ((int64_t)q * d) : br / q, lbc = bc / q;
      const int64_t lcr = csch == TESS_SCHEME_A ? cr / ((int64_t)q * d) : cr / q, lcc = cc / q;
      float* lc = static_cast<float*>(x.ws->get("g.c", (size_t)lcr * lcc * 4));
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      call(tess_matmul(&x, v, td, la, lar, lac, lb, lbr, lbc, lc, TESS_F32,
                       v == TESS_TN ? TESS_SUM_OVER_DEPTH : 0u, s));
      blocks[x.rank] = fetch(lc, (size_t)lcr * lcc, DType::F32, s);
    });
    combine(g, csch, blocks, cr, cc, c);
    if (g_perturb_next && cr > 0 && cc > 0) c[0] += 1e-3;  // ref verify.cpp:84-86
    g_perturb_next = false;
    R.stats(sr, sk);
  });
}

tess_status tess_tesseract_backward(int q, int d, int allow, tess_dtype compute, const double* dc,
                                    const double* a, const double* b, int64_t m, int64_t k,
                                    int64_t n, double* da, double* db, const int* devices,
                                    uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    Grid g(q, d, allow != 0);
    require_div(m, (int64_t)q * d, "tesseract-a", "rows");
    require_div(k, q, "tesseract-a", "cols");
    require_div(n, q, "tesseract-a", "cols");
    Runner R(q, d, allow != 0, devices);
    DevMat dDC, dA, dB;
    upload(dDC, R.unique_devices(), dc, (size_t)m * n, t);
    upload(dA, R.unique_devices(), a, (size_t)m * k, t);
    upload(dB, R.unique_devices(), b, (size_t)k * n, t);
    const int p = g.size();
    std::vector<std::vector<float>> ga(p), gb(p);
    const int64_t mr = m / ((int64_t)q * d), kc = k / q, nc = n / q;
    R.run([&](Ctx& x, cudaStream_t s) {
      void* ldc = take_block(x, TESS_SCHEME_A, t, dDC.on(x.device), m, n, "g.dc", s);
      void* la = take_block(x, TESS_SCHEME_A, t, dA.on(x.device), m, k, "g.a", s);
      void* lb = take_block(x, TESS_SCHEME_B, t, dB.on(x.device), k, n, "g.b", s);
      float* lda = static_cast<float*>(x.ws->get("g.da", (size_t)mr * kc * 4));
      float* ldb = static_cast<float*>(x.ws->get("g.db", (size_t)kc * nc * 4));
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      // ref algorithms.cpp:209-216: dA via NT, dB via TN + depth all-reduce
      call(tess_matmul(&x, TESS_NT, td, ldc, mr, nc, lb, kc, nc, lda, TESS_F32, 0u, s));
      call(tess_matmul(&x, TESS_TN, td, la, mr, kc, ldc, mr, nc, ldb, TESS_F32,
                       TESS_SUM_OVER_DEPTH, s));
      ga[x.rank] = fetch(lda, (size_t)mr * kc, DType::F32, s);
      gb[x.rank] = fetch(ldb, (size_t)kc * nc, DType::F32, s);
    });
    combine(g, TESS_SCHEME_A, ga, m, k, da);
    combine(g, TESS_SCHEME_B, gb, k, n, db);
    R.stats(sr, sk);
  });
}

tess_status tess_layer_run(tess_layer_op op, const tess_layer_dims* dims, int q, int d, int allow,
                           tess_dtype compute, const double* x, const double* dy,
                           const double* const* params, double eps, double* y, double* dx,
                           double* const* grads, double* dbias, const int* devices,
                           uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    if (!dims || !x || !dy || !params || !y || !dx) fail(TESS_ERR_INVALID, "null argument");
    Grid g(q, d, allow != 0);
    const tess_layer_dims D = *dims;
    // divisibility as shard_activation (ref layers.cpp:115-136)
    Runner R(q, d, allow != 0, devices);
    tess::RankDims rd0 = rank_dims(*R.ctx[0], D);
    const int64_t h = D.hidden, T = (int64_t)D.batch * D.seq;
    const int64_t wshape[4][2] = {{h, 3 * h}, {h, h}, {h, 4 * h}, {4 * h, h}};
    DevMat dx_, ddy;
    upload(dx_, R.unique_devices(), x, (size_t)T * h, t);
    upload(ddy, R.unique_devices(), dy, (size_t)T * h, t);
    DevMat W[4], LN[4];
    for (int i = 0; i < 4; ++i)
      upload(W[i], R.unique_devices(), params[i], (size_t)(wshape[i][0] * wshape[i][1]), t);
    for (int i = 0; i < 4; ++i) upload(LN[i], R.unique_devices(), params[4 + i], (size_t)h, DType::F32);
    const int p = g.size();
    const int64_t hq = rd0.hq, rows = rd0.rows;
    std::vector<std::vector<float>> ys(p), dxs(p), dbs(p);
    std::vector<std::vector<float>> gw[8];
    for (auto& v : gw) v.resize(p);
    R.run([&](Ctx& c, cudaStream_t s) {
      tess::RankDims rd = rank_dims(c, D);
      void* lx = take_block(c, TESS_SCHEME_A, t, dx_.on(c.device), T, h, "g.x", s);
      void* ldy = take_block(c, TESS_SCHEME_A, t, ddy.on(c.device), T, h, "g.dy", s);
      tess_block_shard sh;
      const void* wl[4];
      for (int i = 0; i < 4; ++i)
        wl[i] = take_block(c, TESS_SCHEME_B, t, W[i].on(c.device), wshape[i][0], wshape[i][1],
                           "g.w" + std::to_string(i), s);
      sh.w_qkv = wl[0];
      sh.w_proj = wl[1];
      sh.w_ff1 = wl[2];
      sh.w_ff2 = wl[3];
      const float* lnv[4];
      for (int i = 0; i < 4; ++i)
        lnv[i] = static_cast<const float*>(LN[i].on(c.device)) + (int64_t)c.coord.j * hq;
      sh.ln1_gain = lnv[0];
      sh.ln1_bias = lnv[1];
      sh.ln2_gain = lnv[2];
      sh.ln2_bias = lnv[3];
      sh.eps = eps;
      const int64_t gsz[8] = {hq * 3 * hq, hq * hq, hq * 4 * hq, 4 * hq * hq, hq, hq, hq, hq};
      float* gp[8];
      for (int i = 0; i < 8; ++i) {
        gp[i] = static_cast<float*>(c.ws->get("g.grad" + std::to_string(i), (size_t)gsz[i] * 4));
        TESS_CUDA(cudaMemsetAsync(gp[i], 0, (size_t)gsz[i] * 4, s));
      }
      tess_block_grads gr{gp[0], gp[1], gp[2], gp[3], gp[4], gp[5], gp[6], gp[7]};
      void* ly = c.ws->get("g.y", (size_t)rows * hq * dtype_size(t));
      void* ldx = c.ws->get("g.dxo", (size_t)rows * hq * dtype_size(t));
      float* ldb = static_cast<float*>(c.ws->get("g.dbias", (size_t)hq * 4));
      TESS_CUDA(cudaMemsetAsync(ldb, 0, hq * 4, s));
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      // ref layers.cpp:631-683; BiasAdd uses ln1_bias owned by the i == 0 row
      const void* brow = c.coord.i == 0 ? lnv[1] : nullptr;
      call(tess_layer_forward(&c, op, td, &D, &sh, brow, lx, ly, s));
      call(tess_layer_backward(&c, op, td, &D, &sh, ldy, ldx, &gr, 1, ldb, s));
      ys[c.rank] = fetch(ly, (size_t)rows * hq, t, s);
      dxs[c.rank] = fetch(ldx, (size_t)rows * hq, t, s);
      dbs[c.rank] = fetch(ldb, (size_t)hq, DType::F32, s);
      for (int i = 0; i < 8; ++i) gw[i][c.rank] = fetch(gp[i], (size_t)gsz[i], DType::F32, s);
    });
    combine(g, TESS_SCHEME_A, ys, T, h, y);
    combine(g, TESS_SCHEME_A, dxs, T, h, dx);
    if (grads) {
      for (int i = 0; i < 4; ++i)
        if (grads[i]) combine(g, TESS_SCHEME_B, gw[i], wshape[i][0], wshape[i][1], grads[i]);
      // LayerNorm vectors: j-slices, replicas over (i, k) must agree
      // (ref layers.cpp:197-213).
      for (int i = 4; i < 8; ++i) {
        if (!grads[i]) continue;
        for (int j = 0; j < q; ++j) {
          const auto& ref = gw[i][g.rank_of({0, j, 0})];
          for (int ii = 0; ii < q; ++ii)
            for (int k = 0; k < d; ++k)
              if (std::memcmp(ref.data(), gw[i][g.rank_of({ii, j, k})].data(), hq * 4) != 0)
                fail(TESS_ERR_SHAPE, "combine_block_grads: layernorm replica divergence");
          for (int64_t cc = 0; cc < hq; ++cc) grads[i][j * hq + cc] = ref[cc];
        }
      }
    }
    if (dbias && op == TESS_OP_BIAS_ADD)
      for (int j = 0; j < q; ++j)
        for (int64_t cc = 0; cc < hq; ++cc) dbias[j * hq + cc] = dbs[g.rank_of({0, j, 0})][cc];
    R.stats(sr, sk);
  });
}

// The 1-D tensor-parallel (Megatron) counterpart of tess_layer_run, BASELINE
// config 5's comparator built from megatron_1d_linear (ref algorithms.cpp:
// 244-265: Column1D / Row1D weight split, depth all-reduce of the partials)
// applied to the whole block: on a [1,1,p] line grid every rank holds x and
// dy, heads [k n/p, (k+1) n/p) -- W_qkv / W_ff1 column shards, W_proj / W_ff2
// row shards -- and the LayerNorm vectors; the proj / FF2 outputs and the
// QKV / FF1 dgrads are all-reduced over the line. Same math as the reference
// block (layers.cpp:460-487), so the oracle's ref::transformer_block checks it.
tess_status tess_megatron_layer_run(tess_layer_op op, const tess_layer_dims* dims, int p,
                                    tess_dtype compute, const double* x, const double* dy,
                                    const double* const* params, double eps, double* y,
                                    double* dx, double* const* grads, const int* devices,
                                    uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    if (!dims || !x || !dy || !params || !y || !dx) fail(TESS_ERR_INVALID, "null argument");
    if (op == TESS_OP_BIAS_ADD) fail(TESS_ERR_UNSUPPORTED, "1-D scheme: no bias_add op");
    if (p < 1) fail(TESS_ERR_GRID, "p must be >= 1");
    const tess_layer_dims D = *dims;
    const int64_t h = D.hidden, T = (int64_t)D.batch * D.seq;
    if (D.heads <= 0 || D.heads % p != 0 || h % D.heads != 0)
      fail(TESS_ERR_DIVISIBILITY, "1-D scheme: heads must divide hidden and be divisible by p");
    const int64_t hp = h / p;
    Runner R(1, p, true, devices);
    DevMat dX, dDY, W[4], LN[4];
    upload(dX, R.unique_devices(), x, (size_t)(T * h), t);
    upload(dDY, R.unique_devices(), dy, (size_t)(T * h), t);
    const int64_t wshape[4][2] = {{h, 3 * h}, {h, h}, {h, 4 * h}, {4 * h, h}};
    const bool colsplit[4] = {true, false, true, false};
    for (int i = 0; i < 4; ++i)
      upload(W[i], R.unique_devices(), params[i], (size_t)(wshape[i][0] * wshape[i][1]), t);
    for (int i = 0; i < 4; ++i)
      upload(LN[i], R.unique_devices(), params[4 + i], (size_t)h, DType::F32);
    std::vector<float> ys, dxs, gl[4];
    std::vector<std::vector<float>> gw[4];
    for (auto& v : gw) v.resize(p);
    const size_t e = dtype_size(t);
    R.run([&](Ctx& c, cudaStream_t s) {
      c.megatron = true;
      const int k = c.coord.k;  // line grid: rank index = depth slot
      const void* wl[4];
      int64_t lsh[4][2];
      for (int i = 0; i < 4; ++i) {
        const int64_t r = wshape[i][0], cols = wshape[i][1];
        const char* src = static_cast<const char*>(W[i].on(c.device));
        if (colsplit[i]) {  // Column1D: columns [k cols/p, (k+1) cols/p)
          const int64_t cw = cols / p;
          void* b = c.ws->get("mg.w" + std::to_string(i), (size_t)(r * cw) * e);
          TESS_CUDA(cudaMemcpy2DAsync(b, cw * e, src + (size_t)(k * cw) * e, cols * e, cw * e, r,
                                      cudaMemcpyDeviceToDevice, s));
          wl[i] = b;
          lsh[i][0] = r;
          lsh[i][1] = cw;
        } else {  // Row1D: rows [k r/p, (k+1) r/p)
          const int64_t rh = r / p;
          wl[i] = src + (size_t)(k * rh * cols) * e;
          lsh[i][0] = rh;
          lsh[i][1] = cols;
        }
      }
      tess_block_shard sh;
      sh.w_qkv = wl[0];
      sh.w_proj = wl[1];
      sh.w_ff1 = wl[2];
      sh.w_ff2 = wl[3];
      sh.ln1_gain = static_cast<const float*>(LN[0].on(c.device));
      sh.ln1_bias = static_cast<const float*>(LN[1].on(c.device));
      sh.ln2_gain = static_cast<const float*>(LN[2].on(c.device));
      sh.ln2_bias = static_cast<const float*>(LN[3].on(c.device));
      sh.eps = eps;
      float* gp[8];
      size_t gsz[8];
      for (int i = 0; i < 8; ++i) {
        gsz[i] = i < 4 ? (size_t)(lsh[i][0] * lsh[i][1]) : (size_t)h;
        gp[i] = static_cast<float*>(c.ws->get("g.grad" + std::to_string(i), gsz[i] * 4));
        TESS_CUDA(cudaMemsetAsync(gp[i], 0, gsz[i] * 4, s));
      }
      tess_block_grads gr{gp[0], gp[1], gp[2], gp[3], gp[4], gp[5], gp[6], gp[7]};
      void* ly = c.ws->get("g.y", (size_t)(T * h) * e);
      void* ldx = c.ws->get("g.dxo", (size_t)(T * h) * e);
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      call(tess_layer_forward(&c, op, td, &D, &sh, nullptr, dX.on(c.device), ly, s));
      call(tess_layer_backward(&c, op, td, &D, &sh, dDY.on(c.device), ldx, &gr, 1, nullptr, s));
      for (int i = 0; i < 4; ++i) gw[i][k] = fetch(gp[i], gsz[i], DType::F32, s);
      if (k == 0) {
        ys = fetch(ly, (size_t)(T * h), t, s);
        dxs = fetch(ldx, (size_t)(T * h), t, s);
        for (int i = 0; i < 4; ++i) gl[i] = fetch(gp[4 + i], (size_t)h, DType::F32, s);
      }
      c.megatron = false;
    });
    for (size_t i = 0; i < ys.size(); ++i) y[i] = ys[i];
    for (size_t i = 0; i < dxs.size(); ++i) dx[i] = dxs[i];
    if (grads) {
      for (int i = 0; i < 4; ++i) {
        if (!grads[i]) continue;
        const int64_t r = wshape[i][0], cols = wshape[i][1];
        for (int k = 0; k < p; ++k) {
          const auto& v = gw[i][k];
          if (colsplit[i]) {
            const int64_t cw = cols / p;
            for (int64_t rr = 0; rr < r; ++rr)
              for (int64_t cc = 0; cc < cw; ++cc) grads[i][rr * cols + k * cw + cc] = v[rr * cw + cc];
          } else {
            const int64_t rh = r / p;
            for (int64_t rr = 0; rr < rh; ++rr)
              for (int64_t cc = 0; cc < cols; ++cc) grads[i][(k * rh + rr) * cols + cc] = v[rr * cols + cc];
          }
        }
      }
      for (int i = 0; i < 4; ++i)
        if (grads[4 + i])
          for (int64_t cc = 0; cc < h; ++cc) grads[4 + i][cc] = gl[i][cc];
    }
    (void)hp;
    R.stats(sr, sk);
  });
}

// BASELINE config 5's layer stack as a global call: `layers` Transformer
// blocks forward then backward (tess_stack_step per rank) under one of the
// three schemes the comparison runs -- Tesseract [q,q,d], SUMMA (= [q,q,1],
// ref algorithms.cpp:105-118) or the 1-D scheme on p = d ranks (the
// megatron_1d_linear split, algorithms.cpp:244-265, applied to every block).
// Same math as chaining the reference's transformer_block forward and
// backward (layers.cpp:460-487) through the stack, so the oracle checks it.
tess_status tess_stack_run(tess_stack_scheme scheme, const tess_layer_dims* dims, int layers,
                           int q, int d, int allow, tess_dtype compute, const double* x,
                           const double* dy, const double* const* params, double eps, double* y,
                           double* dx, double* const* grads, const int* devices, uint64_t* sr,
                           uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    if (!dims || !x || !dy || !params || !y || !dx || layers < 1)
      fail(TESS_ERR_INVALID, "stack_run: bad arguments");
    const bool mg = scheme == TESS_STACK_MEGATRON;
    if (!mg && scheme != TESS_STACK_TESSERACT) fail(TESS_ERR_INVALID, "stack_run: bad scheme");
    if (mg && q != 1) fail(TESS_ERR_GRID, "the 1-D scheme runs on a [1,1,p] line grid (q == 1)");
    const tess_layer_dims D = *dims;
    const int64_t h = D.hidden, T = (int64_t)D.batch * D.seq;
    const int p = mg ? d : q * q * d;
    if (mg && (D.heads <= 0 || D.heads % p != 0 || h % D.heads != 0))
      fail(TESS_ERR_DIVISIBILITY, "1-D scheme: heads must divide hidden and be divisible by p");
    Runner R(q, d, mg || allow != 0, devices);
    const Grid& g = R.g;
    const tess::RankDims rd0 = [&] {
      R.ctx[0]->megatron = mg;
      tess::RankDims r = rank_dims(*R.ctx[0], D);
      R.ctx[0]->megatron = false;
      return r;
    }();
    const int64_t hq = rd0.hq, rows = rd0.rows, hin = rd0.hin;
    const int64_t wshape[4][2] = {{h, 3 * h}, {h, h}, {h, 4 * h}, {4 * h, h}};
    const bool colsplit[4] = {true, false, true, false};  // 1-D: Column1D / Row1D
    const size_t e = dtype_size(t);
    DevMat dX, dDY;
    upload(dX, R.unique_devices(), x, (size_t)(T * h), t);
    upload(dDY, R.unique_devices(), dy, (size_t)(T * h), t);
    std::vector<std::unique_ptr<DevMat>> W, LN;
    for (int l = 0; l < layers; ++l) {
      for (int i = 0; i < 4; ++i) {
        W.push_back(std::make_unique<DevMat>());
        upload(*W.back(), R.unique_devices(), params[l * 8 + i],
               (size_t)(wshape[i][0] * wshape[i][1]), t);
      }
      for (int i = 0; i < 4; ++i) {
        LN.push_back(std::make_unique<DevMat>());
        upload(*LN.back(), R.unique_devices(), params[l * 8 + 4 + i], (size_t)h, DType::F32);
      }
    }
    std::vector<std::vector<float>> ys(p), dxs(p);
    // gw[l*8 + i][rank]
    std::vector<std::vector<std::vector<float>>> gw((size_t)layers * 8,
                                                    std::vector<std::vector<float>>(p));
    int64_t lsh[4][2];  // local weight shard shapes
    for (int i = 0; i < 4; ++i) {
      if (!mg) {
        lsh[i][0] = wshape[i][0] / q;
        lsh[i][1] = wshape[i][1] / q;
      } else if (colsplit[i]) {
        lsh[i][0] = wshape[i][0];
        lsh[i][1] = wshape[i][1] / p;
      } else {
        lsh[i][0] = wshape[i][0] / p;
        lsh[i][1] = wshape[i][1];
      }
    }
    const int64_t lnw = mg ? h : hq;  // LayerNorm vector width on a rank
    R.run([&](Ctx& c, cudaStream_t s) {
      c.megatron = mg;
      const tess::RankDims rd = rank_dims(c, D);
      const void* lx = mg ? dX.on(c.device)
                          : take_block(c, TESS_SCHEME_A, t, dX.on(c.device), T, h, "stk.gx", s);
      const void* ldy = mg ? dDY.on(c.device)
                           : take_block(c, TESS_SCHEME_A, t, dDY.on(c.device), T, h, "stk.gdy", s);
      std::vector<tess_block_shard> sh(layers);
      std::vector<tess_block_grads> gr(layers);
      for (int l = 0; l < layers; ++l) {
        const std::string L = "stk.l" + std::to_string(l);
        const void* wl[4];
        for (int i = 0; i < 4; ++i) {
          const void* src = W[l * 4 + i]->on(c.device);
          const int64_t r = wshape[i][0], cols = wshape[i][1];
          if (!mg) {
            wl[i] = take_block(c, TESS_SCHEME_B, t, src, r, cols, L + ".w" + std::to_string(i), s);
          } else if (colsplit[i]) {
            const int64_t cw = cols / p;
            void* b = c.ws->get(L + ".w" + std::to_string(i), (size_t)(r * cw) * e);
            TESS_CUDA(cudaMemcpy2DAsync(b, cw * e, static_cast<const char*>(src) +
                                                       (size_t)(c.coord.k * cw) * e,
                                        cols * e, cw * e, r, cudaMemcpyDeviceToDevice, s));
            wl[i] = b;
          } else {
            wl[i] = static_cast<const char*>(src) + (size_t)(c.coord.k * (r / p) * cols) * e;
          }
        }
        const float* lnv[4];
        for (int i = 0; i < 4; ++i)
          lnv[i] = static_cast<const float*>(LN[l * 4 + i]->on(c.device)) +
                   (mg ? 0 : (int64_t)c.coord.j * hq);
        sh[l] = {wl[0], wl[1], wl[2], wl[3], lnv[0], lnv[1], lnv[2], lnv[3], eps};
        float* gp[8];
        for (int i = 0; i < 8; ++i) {
          const size_t n = i < 4 ? (size_t)(lsh[i][0] * lsh[i][1]) : (size_t)lnw;
          gp[i] = static_cast<float*>(c.ws->get(L + ".g" + std::to_string(i), n * 4));
        }
        gr[l] = {gp[0], gp[1], gp[2], gp[3], gp[4], gp[5], gp[6], gp[7]};
      }
      void* ly = c.ws->get("stk.gy", (size_t)(rows * hin) * e);
      void* ldx = c.ws->get("stk.gdx", (size_t)(rows * hin) * e);
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      call(tess_stack_step(&c, td, &D, layers, sh.data(), lx, ldy, ly, ldx, gr.data(), 0, s));
      if (!mg || c.coord.k == 0) {
        ys[c.rank] = fetch(ly, (size_t)(rows * hin), t, s);
        dxs[c.rank] = fetch(ldx, (size_t)(rows * hin), t, s);
      }
      if (grads)
        for (int l = 0; l < layers; ++l) {
          const float* gp[8] = {gr[l].w_qkv,    gr[l].w_proj,   gr[l].w_ff1,    gr[l].w_ff2,
                                gr[l].ln1_gain, gr[l].ln1_bias, gr[l].ln2_gain, gr[l].ln2_bias};
          for (int i = 0; i < 8; ++i) {
            if (!grads[l * 8 + i]) continue;
            if (mg && i >= 4 && c.coord.k != 0) continue;
            const size_t n = i < 4 ? (size_t)(lsh[i][0] * lsh[i][1]) : (size_t)lnw;
            gw[(size_t)l * 8 + i][c.rank] = fetch(gp[i], n, DType::F32, s);
          }
        }
      c.megatron = false;
    });
    if (!mg) {
      combine(g, TESS_SCHEME_A, ys, T, h, y);
      combine(g, TESS_SCHEME_A, dxs, T, h, dx);
    } else {
      for (size_t i = 0; i < ys[0].size(); ++i) y[i] = ys[0][i];
      for (size_t i = 0; i < dxs[0].size(); ++i) dx[i] = dxs[0][i];
    }
    if (grads) {
      for (int l = 0; l < layers; ++l) {
        for (int i = 0; i < 4; ++i) {
          double* out = grads[l * 8 + i];
          if (!out) continue;
          const auto& v = gw[(size_t)l * 8 + i];
          const int64_t r = wshape[i][0], cols = wshape[i][1];
          if (!mg) {
            combine(g, TESS_SCHEME_B, v, r, cols, out);
            continue;
          }
          for (int k = 0; k < p; ++k) {
            if (colsplit[i]) {
              const int64_t cw = cols / p;
              for (int64_t rr = 0; rr < r; ++rr)
                for (int64_t cc = 0; cc < cw; ++cc)
                  out[rr * cols + k * cw + cc] = v[k][rr * cw + cc];
            } else {
              const int64_t rh = r / p;
              for (int64_t rr = 0; rr < rh; ++rr)
                for (int64_t cc = 0; cc < cols; ++cc)
                  out[(k * rh + rr) * cols + cc] = v[k][rr * cols + cc];
            }
          }
        }
        for (int i = 4; i < 8; ++i) {
          double* out = grads[l * 8 + i];
          if (!out) continue;
          const auto& v = gw[(size_t)l * 8 + i];
          if (mg) {
            for (int64_t cc = 0; cc < h; ++cc) out[cc] = v[0][cc];
            continue;
          }
          // LayerNorm vectors: j-slices whose (i, k) replicas must agree
          // (ref layers.cpp:197-213)
          for (int j = 0; j < q; ++j) {
            const auto& ref = v[g.rank_of({0, j, 0})];
            for (int ii = 0; ii < q; ++ii)
              for (int k = 0; k < d; ++k)
                if (std::memcmp(ref.data(), v[g.rank_of({ii, j, k})].data(), hq * 4) != 0)
                  fail(TESS_ERR_SHAPE, "combine_block_grads: layernorm replica divergence");
            for (int64_t cc = 0; cc < hq; ++cc) out[j * hq + cc] = ref[cc];
          }
        }
      }
    }
    R.stats(sr, sk);
  });
}

// ref layers.cpp:947-1036 (the sharded half of train_toy): `layers` blocks,
// MSE loss with global_sum_rank (row, column, depth all-reduce of the local
// sum, layers.cpp:519-526), backward through every block, plain SGD on every
// parameter shard. In bf16 mode weights keep an fp32 master copy.
tess_status tess_train_toy(const tess_layer_dims* dims, int layers, int steps, double lr, int q,
                           int d, int allow, tess_dtype compute, const double* x,
                           const double* target, const double* const* params, double eps,
                           double* losses, const int* devices, uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    if (!dims || !x || !target || !params || !losses || layers < 1 || steps < 0)
      fail(TESS_ERR_INVALID, "train_toy: bad arguments");
    Grid g(q, d, allow != 0);
    const tess_layer_dims D = *dims;
    Runner R(q, d, allow != 0, devices);
    tess::RankDims rd0 = rank_dims(*R.ctx[0], D);
    const int64_t h = D.hidden, T = (int64_t)D.batch * D.seq, hq = rd0.hq, rows = rd0.rows;
    const double denom = (double)(T * h);
    const int64_t wshape[4][2] = {{h, 3 * h}, {h, h}, {h, 4 * h}, {4 * h, h}};
    DevMat dX, dT;
    upload(dX, R.unique_devices(), x, (size_t)T * h, t);
    upload(dT, R.unique_devices(), target, (size_t)T * h, t);
    std::vector<std::unique_ptr<DevMat>> W32, LN;  // fp32 uploads of every parameter
    for (int l = 0; l < layers; ++l) {
      for (int i = 0; i < 4; ++i) {
        W32.push_back(std::make_unique<DevMat>());
        upload(*W32.back(), R.unique_devices(), params[l * 8 + i],
               (size_t)(wshape[i][0] * wshape[i][1]), DType::F32);
      }
      for (int i = 0; i < 4; ++i) {
        LN.push_back(std::make_unique<DevMat>());
        upload(*LN.back(), R.unique_devices(), params[l * 8 + 4 + i], (size_t)h, DType::F32);
      }
    }
    std::vector<double> rank0_losses(steps, 0.0);
    R.run([&](Ctx& c, cudaStream_t s) {
      const tess::RankDims rd = rank_dims(c, D);
      const tess_dtype td = t == DType::F32 ? TESS_F32 : TESS_BF16;
      const size_t act = (size_t)rows * hq * dtype_size(t);
      void* lx = take_block(c, TESS_SCHEME_A, t, dX.on(c.device), T, h, "toy.x", s);
      void* lt = take_block(c, TESS_SCHEME_A, t, dT.on(c.device), T, h, "toy.t", s);
      const int64_t gsz[8] = {hq * 3 * hq, hq * hq, hq * 4 * hq, 4 * hq * hq, hq, hq, hq, hq};
      std::vector<tess_block_shard> sh(layers);
      std::vector<tess_block_grads> gr(layers);
      std::vector<std::array<void*, 8>> wptr(layers);
      std::vector<std::array<float*, 8>> master(layers);
      for (int l = 0; l < layers; ++l) {
        const std::string L = "toy.l" + std::to_string(l);
        for (int i = 0; i < 4; ++i) {
          float* m32 = static_cast<float*>(take_block(c, TESS_SCHEME_B, DType::F32,
                                                      W32[l * 4 + i]->on(c.device), wshape[i][0],
                                                      wshape[i][1], L + ".m" + std::to_string(i), s));
          master[l][i] = m32;
          if (t == DType::F32) {
            wptr[l][i] = m32;
            master[l][i] = nullptr;
          } else {
            wptr[l][i] = c.ws->get(L + ".w" + std::to_string(i), (size_t)gsz[i] * 2);
            k_convert(m32, DType::F32, wptr[l][i], t, (size_t)gsz[i], s);
          }
        }
        for (int i = 0; i < 4; ++i) {
          float* v = static_cast<float*>(c.ws->get(L + ".ln" + std::to_string(i), hq * 4));
          TESS_CUDA(cudaMemcpyAsync(v, static_cast<const float*>(LN[l * 4 + i]->on(c.device)) +
                                           (int64_t)c.coord.j * hq,
                                    hq * 4, cudaMemcpyDeviceToDevice, s));
          wptr[l][4 + i] = v;
          master[l][4 + i] = nullptr;
        }
        sh[l] = {wptr[l][0], wptr[l][1], wptr[l][2], wptr[l][3],
                 static_cast<float*>(wptr[l][4]), static_cast<float*>(wptr[l][5]),
                 static_cast<float*>(wptr[l][6]), static_cast<float*>(wptr[l][7]), eps};
        float* gp[8];
        for (int i = 0; i < 8; ++i)
          gp[i] = static_cast<float*>(c.ws->get(L + ".g" + std::to_string(i), (size_t)gsz[i] * 4));
        gr[l] = {gp[0], gp[1], gp[2], gp[3], gp[4], gp[5], gp[6], gp[7]};
      }
      double* dsum = static_cast<double*>(c.ws->get("toy.sum", 8));
      double* scratch =
          static_cast<double*>(c.ws->get("toy.scr", k_mse_scratch_doubles(rows * hq) * 8));
      float* fsum = static_cast<float*>(c.ws->get("toy.fsum", 4));
      void* dyb[2] = {c.ws->get("toy.dy0", act), c.ws->get("toy.dy1", act)};
      for (int st = 0; st < steps; ++st) {
        const void* cur = lx;
        for (int l = 0; l < layers; ++l) {
          c.cache_slot = l;
          void* y = c.ws->get("toy.y" + std::to_string(l), act);
          call(tess_layer_forward(&c, TESS_OP_BLOCK, td, &D, &sh[l], nullptr, cur, y, s));
          cur = y;
        }
        k_mse_grad(cur, lt, t, (size_t)rows * hq, denom, dyb[0], dsum, scratch, s);
        double local = 0;
        TESS_CUDA(cudaMemcpyAsync(&local, dsum, 8, cudaMemcpyDeviceToHost, s));
        TESS_CUDA(cudaStreamSynchronize(s));
        const float lf = (float)local;
        TESS_CUDA(cudaMemcpyAsync(fsum, &lf, 4, cudaMemcpyHostToDevice, s));
        coll_allreduce(c, ROW, fsum, 1, s);  // global_sum_rank, layers.cpp:519-526
        coll_allreduce(c, COL, fsum, 1, s);
        coll_allreduce(c, DEPTH, fsum, 1, s);
        float total = 0;
        TESS_CUDA(cudaMemcpyAsync(&total, fsum, 4, cudaMemcpyDeviceToHost, s));
        TESS_CUDA(cudaStreamSynchronize(s));
        if (c.rank == 0) rank0_losses[st] = (double)total / denom;
        int cur_dy = 0;
        for (int l = layers - 1; l >= 0; --l) {
          c.cache_slot = l;
          call(tess_layer_backward(&c, TESS_OP_BLOCK, td, &D, &sh[l], dyb[cur_dy],
                                   dyb[1 - cur_dy], &gr[l], 0, nullptr, s));
          cur_dy = 1 - cur_dy;
        }
        for (int l = 0; l < layers; ++l) {
          const float* gp[8] = {gr[l].w_qkv, gr[l].w_proj, gr[l].w_ff1, gr[l].w_ff2,
                                gr[l].ln1_gain, gr[l].ln1_bias, gr[l].ln2_gain, gr[l].ln2_bias};
          for (int i = 0; i < 8; ++i)
            k_sgd(wptr[l][i], i < 4 ? t : DType::F32, master[l][i], gp[i], lr, (size_t)gsz[i], s);
        }
      }
      c.cache_slot = 0;
    });
    for (int st = 0; st < steps; ++st) losses[st] = rank0_losses[st];
    R.stats(sr, sk);
  });
}

// ref algorithms.cpp:244-265 (megatron_1d_linear): the 1-D tensor-parallel
// pair of linear layers on a [1,1,p] line grid -- W1 column-split (Column1D),
// W2 row-split (Row1D), every rank computes X W1_k W2_k (two local GEMMs) and
// one all-reduce over the single depth group sums the partial outputs. The
// 1-D comparator of BASELINE config 5.
tess_status tess_megatron_1d_linear(int p, tess_dtype compute, const double* x, int64_t xr,
                                    int64_t xc, const double* w1, int64_t w1r, int64_t w1c,
                                    const double* w2, int64_t w2r, int64_t w2c, double* out,
                                    const int* devices, uint64_t* sr, uint64_t* sk) {
  return guarded([&] {
    const DType t = compute_type(compute);
    if (xc != w1r)
      fail(TESS_ERR_SHAPE, "megatron_1d_linear: A.cols (" + std::to_string(xc) +
                               ") != B.rows (" + std::to_string(w1r) + ")");
    if (w1c != w2r)
      fail(TESS_ERR_SHAPE, "megatron_1d_linear: A.cols (" + std::to_string(w1c) +
                               ") != B.rows (" + std::to_string(w2r) + ")");
    if (p < 1 || w1c % p != 0)
      fail(TESS_ERR_DIVISIBILITY, "megatron_1d_linear: inner width (" + std::to_string(w1c) +
                                      ") not divisible by p (" + std::to_string(p) + ")");
    const int64_t kb = w1c / p;
    Runner R(1, p, true, devices);
    DevMat dX, dW1, dW2;
    upload(dX, R.unique_devices(), x, (size_t)(xr * xc), t);
    upload(dW1, R.unique_devices(), w1, (size_t)(w1r * w1c), t);
    upload(dW2, R.unique_devices(), w2, (size_t)(w2r * w2c), t);
    std::vector<float> res;
    R.run([&](Ctx& c, cudaStream_t s) {
      const size_t e = dtype_size(t);
      const int k = c.coord.k;  // line grid: the rank index is the depth slot
      void* b1 = c.ws->get("mg.w1", (size_t)w1r * kb * e);
      TESS_CUDA(cudaMemcpy2DAsync(b1, kb * e,
                                  static_cast<const char*>(dW1.on(c.device)) + (size_t)k * kb * e,
                                  w1c * e, kb * e, w1r, cudaMemcpyDeviceToDevice, s));
      void* b2 = c.ws->get("mg.w2", (size_t)kb * w2c * e);
      TESS_CUDA(cudaMemcpyAsync(b2,
                                static_cast<const char*>(dW2.on(c.device)) + (size_t)k * kb * w2c * e,
                                (size_t)kb * w2c * e, cudaMemcpyDeviceToDevice, s));
      void* h = c.ws->get("mg.h", (size_t)xr * kb * e);
      float* part = static_cast<float*>(c.ws->get("mg.part", (size_t)xr * w2c * 4));
      GemmDesc g1;
      g1.M = xr; g1.N = kb; g1.in = t; g1.seg[0] = {dX.on(c.device), b1, xc};
      g1.lda = xc; g1.ldb = kb; g1.c = h; g1.c_type = t; g1.ldc = kb;
      run_gemm(g1, s);
      GemmDesc g2;
      g2.M = xr; g2.N = w2c; g2.in = t; g2.seg[0] = {h, b2, kb};
      g2.lda = kb; g2.ldb = w2c; g2.c = part; g2.c_type = DType::F32; g2.ldc = w2c;
      run_gemm(g2, s);
      cudaStream_t cs = comm_stream(c, s);
      stream_dep(c, s, cs);
      coll_allreduce(c, DEPTH, part, (size_t)xr * w2c, cs);  // ref algorithms.cpp:261
      stream_dep(c, cs, s);
      if (c.rank == 0) res = fetch(part, (size_t)xr * w2c, DType::F32, s);
    });
    for (size_t i = 0; i < res.size(); ++i) out[i] = res[i];
    R.stats(sr, sk);
  });
}

}  // extern "C"

extern "C" {

tess_status tess_set_global_fault(tess_fault kind, int rank, int64_t at) {
  return guarded([&] {
    if (kind < TESS_FAULT_NONE || kind > TESS_FAULT_SKIP_COLLECTIVE)
      fail(TESS_ERR_INVALID, "unknown fault kind");
    g_perturb_next = kind == TESS_FAULT_PERTURB;
    g_fault_kind = kind == TESS_FAULT_PERTURB ? 0 : (int)kind;
    g_fault_rank = rank;
    g_fault_at = at;
  });
}

tess_status tess_set_global_trace(int enable) {
  g_global_trace = enable != 0;
  return TESS_OK;
}

tess_status tess_global_last_stats(int* ranks, uint64_t* sent_by_kind, uint64_t* recv,
                                   size_t cap_ranks) {
  return guarded([&] {
    const LastRun& L = g_last_run;
    if (ranks) *ranks = L.p;
    if ((sent_by_kind || recv) && cap_ranks < (size_t)L.p)
      fail(TESS_ERR_INVALID, "tess_global_last_stats: buffers hold fewer ranks than the run");
    if (sent_by_kind) std::copy(L.sent.begin(), L.sent.end(), sent_by_kind);
    if (recv) std::copy(L.recv.begin(), L.recv.end(), recv);
  });
}

tess_status tess_global_last_trace(char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    const std::string& s = g_last_run.trace;
    if (needed) *needed = s.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

}  // extern "C"
