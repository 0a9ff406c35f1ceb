// extern "C" boundary (include/tess.h): argument validation, exception ->
// status conversion, per-rank entry points.
#include <cstring>
#include <string>

#include "kernels/kernels.h"
#include "kernels/attention.h"
#include <algorithm>
#include <cmath>

#include "ops.h"

using namespace tess;

namespace tess {
thread_local std::string g_last_error;
}

namespace {

template <typename F>
tess_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return TESS_OK;
  } catch (const tess::Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return TESS_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TESS_ERR_INVALID;
  }
}

DType to_dtype(tess_dtype t) {
  switch (t) {
    case TESS_F32: return DType::F32;
    case TESS_BF16: return DType::BF16;
    case TESS_F64: return DType::F64;
  }
  fail(TESS_ERR_INVALID, "bad dtype");
}

Family to_family(tess_group g) {
  if (g < TESS_ROW || g > TESS_DEPTH) fail(TESS_ERR_INVALID, "bad group");
  return static_cast<Family>(g);
}

Ctx& need(tess_ctx* c) {
  if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
  TESS_CUDA(cudaSetDevice(c->device));
  return *c;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void init_ctx(Ctx& c, const Grid& g, int rank, int device) {
  c.grid = g;
  c.rank = rank;
  c.coord = g.coord_of(rank);
  c.device = device;
  c.ws = std::make_unique<Workspace>(device);
}

}  // namespace

extern "C" {

const char* tess_last_error(void) { return g_last_error.c_str(); }
const char* tess_version(void) { return "tess-b200 0.1 (sm_100a, tcgen05)"; }
uint64_t tess_kernel_launches(void) { return g_launches.load(); }

tess_status tess_profile_enable(int on) {
  return guarded([&] { profile_enable(on == 2 ? 2 : on != 0 ? 1 : 0); });
}

tess_status tess_debug_attn_trace(long long* out, int n) {
  if (!out || n <= 0) return TESS_ERR_INVALID;
  long long* tr = tess::attn_debug_trace();
  if (!tr) return TESS_ERR_INVALID;
  cudaDeviceSynchronize();
  const int m = n < 512 ? n : 512;
  return cudaMemcpy(out, tr, m * sizeof(long long), cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? TESS_OK
             : TESS_ERR_CUDA;
}

tess_status tess_profile_json(char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    const std::string s = profile_json();
    if (needed) *needed = s.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

tess_status tess_profile_read(double* gemm_ms, double* gemm_flops, uint64_t* gemm_launches) {
  return guarded([&] { profile_read(gemm_ms, gemm_flops, gemm_launches); });
}

tess_status tess_grid_check(int q, int d, int allow) {
  return guarded([&] { Grid g(q, d, allow != 0); });
}

tess_status tess_grid_parse(const char* text, int allow, int* q, int* d) {
  return guarded([&] {
    if (!text) fail(TESS_ERR_INVALID, "null grid text");
    Grid g = parse_grid(text, allow != 0);
    if (q) *q = g.q;
    if (d) *d = g.d;
  });
}

tess_status tess_grid_rank_of(int q, int d, int i, int j, int k, int* rank) {
  return guarded([&] { *rank = Grid(q, d, true).rank_of({i, j, k}); });
}

tess_status tess_grid_coord_of(int q, int d, int rank, int* i, int* j, int* k) {
  return guarded([&] {
    Coord c = Grid(q, d, true).coord_of(rank);
    *i = c.i;
    *j = c.j;
    *k = c.k;
  });
}

tess_status tess_grid_block_row(int q, int d, int i, int j, int k, int* h) {
  return guarded([&] {
    Grid g(q, d, true);
    if (!g.valid({i, j, k})) fail(TESS_ERR_GRID, "coordinate out of range for grid " + g.str());
    *h = g.block_row({i, j, k});
  });
}

tess_status tess_grid_group(int q, int d, int i, int j, int k, tess_group grp, int* gi,
                            int* slot, int* gsize) {
  return guarded([&] {
    Grid g(q, d, true);
    const Coord c{i, j, k};
    if (!g.valid(c)) fail(TESS_ERR_GRID, "coordinate out of range for grid " + g.str());
    const Family f = to_family(grp);
    if (gi) *gi = g.group_index(c, f);
    if (slot) *slot = g.slot_in_group(c, f);
    if (gsize) *gsize = g.group_size(f);
  });
}

tess_status tess_grid_member_at(int q, int d, tess_group grp, int gi, int slot, int* i, int* j,
                                int* k) {
  return guarded([&] {
    Coord c = Grid(q, d, true).member_at(to_family(grp), gi, slot);
    *i = c.i;
    *j = c.j;
    *k = c.k;
  });
}

tess_status tess_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) fail(TESS_ERR_INVALID, "null output");
    nccl_unique_id(out128);
  });
}

tess_status tess_init_nccl(int q, int d, int allow, int rank, int device, const void* uid,
                           tess_ctx** out) {
  return guarded([&] {
    if (!out || !uid) fail(TESS_ERR_INVALID, "null argument");
    Grid g(q, d, allow != 0);
    TESS_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<tess_ctx>();
    init_ctx(*c, g, rank, device);
    c->comm = make_nccl_comm(g, rank, uid);
    *out = c.release();
  });
}

tess_status tess_init_local(int q, int d, int allow, const int* devices, tess_ctx** out) {
  return guarded([&] {
    if (!out) fail(TESS_ERR_INVALID, "null output");
    Grid g(q, d, allow != 0);
    std::vector<int> devs(g.size());
    int cur = 0;
    TESS_CUDA(cudaGetDevice(&cur));
    for (int r = 0; r < g.size(); ++r) devs[r] = devices ? devices[r] : cur;
    auto w = make_local_world(g, devs);
    std::vector<std::unique_ptr<tess_ctx>> made;
    for (int r = 0; r < g.size(); ++r) {
      auto c = std::make_unique<tess_ctx>();
      init_ctx(*c, g, r, devs[r]);
      c->world = w;
      c->comm = make_local_comm(w, r);
      made.push_back(std::move(c));
    }
    for (int r = 0; r < g.size(); ++r) out[r] = made[r].release();
    TESS_CUDA(cudaSetDevice(cur));
  });
}

tess_status tess_destroy(tess_ctx* c) {
  return guarded([&] {
    if (!c) return;
    if (c->world) local_world_rank_finished(c->world.get(), c->rank);
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    delete c;
  });
}

tess_status tess_coord(const tess_ctx* c, int* rank, int* i, int* j, int* k) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    if (rank) *rank = c->rank;
    if (i) *i = c->coord.i;
    if (j) *j = c->coord.j;
    if (k) *k = c->coord.k;
  });
}

tess_status tess_group_comm(tess_ctx* c, tess_group g, void** comm) {
  return guarded([&] { *comm = need(c).comm->nccl_comm(to_family(g)); });
}

tess_status tess_get_comm_stats(const tess_ctx* c, tess_comm_stats* out) {
  return guarded([&] {
    if (!c || !out) fail(TESS_ERR_INVALID, "null argument");
    const Meter& m = c->meter;
    out->sent_messages = m.sent_msgs;
    out->sent_elements = m.sent_elems;
    out->received_messages = m.recv_msgs;
    out->received_elements = m.recv_elems;
    std::memcpy(out->by_kind, m.kind, sizeof(m.kind));
  });
}

tess_status tess_reset_comm_stats(tess_ctx* c) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    c->meter = Meter();
    c->trace.clear();
    c->step = 0;
  });
}

tess_status tess_set_cache_slot(tess_ctx* c, int slot) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    if (slot < 0) fail(TESS_ERR_INVALID, "cache slot must be >= 0");
    c->cache_slot = slot;
  });
}

tess_status tess_stream_join(tess_ctx* c, void* stream) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    TESS_CUDA(cudaSetDevice(c->device));
    ctx_join(*c, static_cast<cudaStream_t>(stream));
  });
}

tess_status tess_inject_fault(tess_ctx* c, tess_fault kind, int64_t at) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    if (kind < TESS_FAULT_NONE || kind > TESS_FAULT_SKIP_COLLECTIVE)
      fail(TESS_ERR_INVALID, "unknown fault kind");
    c->fault_kind = kind == TESS_FAULT_PERTURB ? 0 : (int)kind;
    c->fault_at = at;
  });
}

tess_status tess_set_comm_noop(tess_ctx* c, int enable) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    c->comm_noop = enable != 0;
  });
}

tess_status tess_set_megatron(tess_ctx* c, int enable) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    if (enable && c->grid.q != 1)
      fail(TESS_ERR_GRID, "the 1-D scheme runs on a [1,1,p] line grid (q == 1)");
    c->megatron = enable != 0;
  });
}

tess_status tess_set_trace(tess_ctx* c, int enable) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    c->trace_on = enable != 0;
  });
}

tess_status tess_trace_text(const tess_ctx* c, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    if (!c) fail(TESS_ERR_INVALID, "null tess_ctx");
    const std::string s = trace_text(c->trace);
    if (needed) *needed = s.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

tess_status tess_broadcast(tess_ctx* c, tess_group g, int root, void* buf, size_t bytes,
                           size_t elements, void* stream) {
  return guarded([&] { coll_bcast(need(c), to_family(g), root, buf, bytes, elements, S(stream)); });
}

tess_status tess_reduce(tess_ctx* c, tess_group g, int root, const float* send, float* recv,
                        size_t n, void* stream) {
  return guarded([&] { coll_reduce(need(c), to_family(g), root, send, recv, n, S(stream)); });
}

tess_status tess_all_reduce(tess_ctx* c, tess_group g, float* buf, size_t n, void* stream) {
  return guarded([&] { coll_allreduce(need(c), to_family(g), buf, n, S(stream)); });
}

tess_status tess_barrier(tess_ctx* c) {
  return guarded([&] { need(c).comm->barrier(); });
}

// ref: shard.cpp:68-98 -- the rank's block of a global row-major matrix.
static void block_geometry(const Ctx& c, tess_scheme scheme, int64_t rows, int64_t cols,
                           int64_t* r0, int64_t* rb, int64_t* c0, int64_t* cb) {
  const int q = c.grid.q, d = c.grid.d;
  const char* nm = scheme == TESS_SCHEME_A ? "tesseract-a" : "tesseract-b";
  auto div = [&](int64_t v, int64_t by, const char* dim) {
    if (by == 0 || v % by != 0)
      fail(TESS_ERR_DIVISIBILITY, std::string(nm) + ": " + dim + " (" + std::to_string(v) +
                                      ") not divisible by " + std::to_string(by));
  };
  if (scheme == TESS_SCHEME_A) {
    div(rows, (int64_t)q * d, "rows");
    div(cols, q, "cols");
    *rb = rows / ((int64_t)q * d);
    *r0 = (int64_t)c.grid.block_row(c.coord) * *rb;
  } else if (scheme == TESS_SCHEME_B) {
    div(rows, q, "rows");
    div(cols, q, "cols");
    *rb = rows / q;
    *r0 = (int64_t)c.coord.i * *rb;
  } else {
    fail(TESS_ERR_INVALID, "bad scheme");
  }
  *cb = cols / q;
  *c0 = (int64_t)c.coord.j * *cb;
}

tess_status tess_partition(tess_ctx* c, tess_scheme scheme, tess_dtype dt, const void* global,
                           int64_t rows, int64_t cols, void* local, void* stream) {
  return guarded([&] {
    Ctx& x = need(c);
    int64_t r0, rb, c0, cb;
    block_geometry(x, scheme, rows, cols, &r0, &rb, &c0, &cb);
    const size_t e = dtype_size(to_dtype(dt));
    if (rb * cb == 0) return;
    // bit-exact strided copy on the copy engines
    TESS_CUDA(cudaMemcpy2DAsync(local, cb * e, static_cast<const char*>(global) + (r0 * cols + c0) * e,
                                cols * e, cb * e, rb, cudaMemcpyDefault, S(stream)));
  });
}

tess_status tess_unpartition(tess_ctx* c, tess_scheme scheme, tess_dtype dt, const void* local,
                             int64_t rows, int64_t cols, void* global, void* stream) {
  return guarded([&] {
    Ctx& x = need(c);
    int64_t r0, rb, c0, cb;
    block_geometry(x, scheme, rows, cols, &r0, &rb, &c0, &cb);
    const size_t e = dtype_size(to_dtype(dt));
    if (rb * cb == 0) return;
    TESS_CUDA(cudaMemcpy2DAsync(static_cast<char*>(global) + (r0 * cols + c0) * e, cols * e, local,
                                cb * e, cb * e, rb, cudaMemcpyDefault, S(stream)));
  });
}

tess_status tess_matmul(tess_ctx* c, tess_variant v, tess_dtype in, const void* a, int64_t ar,
                        int64_t ac, const void* b, int64_t br, int64_t bc, void* out,
                        tess_dtype ct, uint32_t flags, void* stream) {
  return tess_matmul_ex(c, v, in, a, ar, ac, b, br, bc, out, ct, flags, nullptr, stream);
}

int tess_dropout_keep(uint64_t seed, int64_t row, int64_t col, float p) {
  if (!(p > 0.f)) return 1;
  const uint32_t th = (uint32_t)std::min(16777216.0, std::ceil((double)p * 16777216.0));
  return dropout_keep(seed, (uint64_t)row, (uint64_t)col, th) ? 1 : 0;
}

tess_status tess_matmul_ex(tess_ctx* c, tess_variant v, tess_dtype in, const void* a, int64_t ar,
                           int64_t ac, const void* b, int64_t br, int64_t bc, void* out,
                           tess_dtype ct, uint32_t flags, const tess_epilogue* ep,
                           void* stream) {
  return guarded([&] {
    Ctx& x = need(c);
    const DType ti = to_dtype(in), tc = to_dtype(ct);
    if (ti == DType::F64) fail(TESS_ERR_UNSUPPORTED, "fp64 inputs: use TESS_F32 or TESS_BF16");
    Out o;
    o.c = out;
    o.t = tc;
    o.epi = (flags & TESS_ACCUMULATE) ? Epi::Accum : Epi::Store;
    if (o.epi == Epi::Accum && tc != DType::F32)
      fail(TESS_ERR_UNSUPPORTED, "TESS_ACCUMULATE needs an fp32 output");
    if (ep && (ep->bias || ep->gelu || ep->dropout_p != 0.f || ep->residual)) {
      if (ti != DType::BF16) fail(TESS_ERR_UNSUPPORTED, "fused epilogues need bf16 inputs");
      if (!(ep->dropout_p >= 0.f && ep->dropout_p < 1.f))
        fail(TESS_ERR_INVALID, "dropout_p must be in [0, 1)");
      const bool reduced = x.grid.q > 1 || (v == TESS_TN && (flags & TESS_SUM_OVER_DEPTH) &&
                                            x.grid.d > 1);
      if (v != TESS_NN && reduced)
        fail(TESS_ERR_UNSUPPORTED, "fused epilogues on NT / TN need q == 1 (no reduction)");
      const int n_epi = (ep->gelu ? 1 : 0) + (ep->residual ? 1 : 0) + (o.epi == Epi::Accum);
      if (n_epi > 1)
        fail(TESS_ERR_UNSUPPORTED, "at most one of gelu, residual, TESS_ACCUMULATE");
      if (ep->gelu) {
        if (!ep->pre_activation) fail(TESS_ERR_INVALID, "gelu needs pre_activation");
        o.epi = Epi::Gelu;
        o.z = ep->pre_activation;
      } else if (ep->residual) {
        o.epi = Epi::Resid;
        o.r = ep->residual;
      }
      o.bias = ep->bias;
      o.drop_p = ep->dropout_p;
      o.drop_seed = ep->dropout_seed;
      o.drop_row0 = ep->row0;
      o.drop_col0 = ep->col0;
    }
    switch (v) {
      case TESS_NN:  // ref algorithms.cpp:34-45; check_inner :23-31
        if (ac != br)
          fail(TESS_ERR_SHAPE, "nn_product: A.cols (" + std::to_string(ac) + ") != B.rows (" +
                                   std::to_string(br) + ")");
        nn_product(x, ti, a, ar, ac, b, bc, o, S(stream));
        break;
      case TESS_NT:
        if (ac != bc)
          fail(TESS_ERR_SHAPE, "nt_product: A.cols (" + std::to_string(ac) + ") != B.cols (" +
                                   std::to_string(bc) + ")");
        nt_product(x, ti, a, ar, ac, b, br, o, S(stream));
        break;
      case TESS_TN:
        if (ar != br)
          fail(TESS_ERR_SHAPE, "tn_product: A.rows (" + std::to_string(ar) + ") != B.rows (" +
                                   std::to_string(br) + ")");
        tn_product(x, ti, a, ar, ac, b, bc, (flags & TESS_SUM_OVER_DEPTH) != 0, o, S(stream));
        break;
      default:
        fail(TESS_ERR_INVALID, "bad variant");
    }
  });
}

tess_status tess_layer_forward(tess_ctx* c, tess_layer_op op, tess_dtype dt,
                               const tess_layer_dims* dims, const tess_block_shard* shard,
                               const void* bias_row0, const void* x, void* y, void* stream) {
  return guarded([&] {
    Ctx& cx = need(c);
    if (!dims || !shard || !x || !y) fail(TESS_ERR_INVALID, "null argument");
    const DType t = to_dtype(dt);
    if (t == DType::F64) fail(TESS_ERR_UNSUPPORTED, "fp64 compute: use TESS_F32 or TESS_BF16");
    layer_forward(cx, op, t, rank_dims(cx, *dims), *shard,
                  static_cast<const float*>(bias_row0), x, y, S(stream));
  });
}

tess_status tess_layer_backward(tess_ctx* c, tess_layer_op op, tess_dtype dt,
                                const tess_layer_dims* dims, const tess_block_shard* shard,
                                const void* dy, void* dx, tess_block_grads* grads, int accumulate,
                                float* dbias, void* stream) {
  return guarded([&] {
    Ctx& cx = need(c);
    if (!dims || !shard || !dy || !dx) fail(TESS_ERR_INVALID, "null argument");
    const DType t = to_dtype(dt);
    if (t == DType::F64) fail(TESS_ERR_UNSUPPORTED, "fp64 compute: use TESS_F32 or TESS_BF16");
    layer_backward(cx, op, t, rank_dims(cx, *dims), *shard, dy, dx, grads, accumulate != 0,
                   dbias, S(stream));
  });
}

tess_status tess_layer_step(tess_ctx* c, tess_layer_op op, tess_dtype dt,
                            const tess_layer_dims* dims, const tess_block_shard* shard,
                            const void* bias_row0, const void* x, const void* dy, void* y,
                            void* dx, tess_block_grads* grads, int accumulate, float* dbias,
                            void* stream) {
  return guarded([&] {
    Ctx& cx = need(c);
    if (!dims || !shard || !x || !dy || !y || !dx) fail(TESS_ERR_INVALID, "null argument");
    const DType t = to_dtype(dt);
    if (t == DType::F64) fail(TESS_ERR_UNSUPPORTED, "fp64 compute: use TESS_F32 or TESS_BF16");
    layer_step(cx, op, t, rank_dims(cx, *dims), *shard, static_cast<const float*>(bias_row0), x,
               dy, y, dx, grads, accumulate != 0, dbias, S(stream));
  });
}

tess_status tess_stack_step(tess_ctx* c, tess_dtype dt, const tess_layer_dims* dims, int layers,
                            const tess_block_shard* shards, const void* x, const void* dy, void* y,
                            void* dx, tess_block_grads* grads, int accumulate, void* stream) {
  return guarded([&] {
    Ctx& cx = need(c);
    if (!dims || !shards || !x || !dy || !y || !dx) fail(TESS_ERR_INVALID, "null argument");
    const DType t = to_dtype(dt);
    if (t == DType::F64) fail(TESS_ERR_UNSUPPORTED, "fp64 compute: use TESS_F32 or TESS_BF16");
    stack_step(cx, t, rank_dims(cx, *dims), layers, shards, x, dy, y, dx, grads, accumulate != 0,
               S(stream));
  });
}

}  // extern "C"
