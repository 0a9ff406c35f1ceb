// Grid geometry (reference proj/src/grid.cpp), workspace, metered collectives.
#include <array>
#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "ctx.h"

namespace tess {

Grid::Grid(int q_, int d_, bool allow) : q(q_), d(d_) {
  // ref: grid.cpp:26-37
  if (q < 1 || d < 1)
    fail(TESS_ERR_GRID, "grid " + str() + ": q and d must be >= 1");
  if (d > q && !allow)
    fail(TESS_ERR_GRID, "grid " + str() +
                            ": depth d exceeds dimension q (pass allow_d_gt_q to permit)");
}

int Grid::rank_of(const Coord& c) const {
  if (!valid(c)) fail(TESS_ERR_GRID, "coordinate out of range for grid " + str());
  return c.k * q * q + c.i * q + c.j;  // ref: grid.cpp:43-49
}

Coord Grid::coord_of(int rank) const {
  if (rank < 0 || rank >= size())
    fail(TESS_ERR_GRID, "rank " + std::to_string(rank) + " out of range for grid " + str());
  Coord c;  // ref: grid.cpp:51-61
  c.k = rank / (q * q);
  c.i = (rank / q) % q;
  c.j = rank % q;
  return c;
}

Coord Grid::member_at(Family f, int gi, int slot) const {
  Coord c;  // ref: grid.cpp:106-131
  if (f == ROW) c = {gi % q, slot, gi / q};
  else if (f == COL) c = {slot, gi % q, gi / q};
  else c = {gi / q, gi % q, slot};
  if (!valid(c)) fail(TESS_ERR_GRID, "group member out of range for grid " + str());
  return c;
}

// ref: grid.cpp:133-169 ("[q,q,d]" with positioned errors)
Grid parse_grid(const std::string& text, bool allow) {
  size_t pos = 0;
  auto bad = [&](size_t at, const std::string& what) {
    fail(TESS_ERR_CONFIG, "grid '" + text + "': " + what + " at position " + std::to_string(at));
  };
  auto expect = [&](char ch) {
    if (pos >= text.size() || text[pos] != ch) bad(pos, std::string("expected '") + ch + "'");
    ++pos;
  };
  auto number = [&]() {
    int v = 0;
    auto res = std::from_chars(text.data() + pos, text.data() + text.size(), v);
    if (res.ec != std::errc() || res.ptr == text.data() + pos) bad(pos, "expected an integer");
    pos = static_cast<size_t>(res.ptr - text.data());
    return v;
  };
  expect('[');
  const int q1 = number();
  expect(',');
  const size_t q2_pos = pos;
  const int q2 = number();
  expect(',');
  const int d = number();
  expect(']');
  if (pos != text.size()) bad(pos, "trailing characters");
  if (q1 != q2)
    bad(q2_pos, "the first two extents must match (got " + std::to_string(q1) + " and " +
                    std::to_string(q2) + ")");
  return Grid(q1, d, allow);
}

// ------------------------------------------------------------ workspace
Workspace::~Workspace() { release_all(); }

void* Workspace::get(const std::string& name, size_t bytes) {
  Buf& b = bufs_[name];
  if (bytes == 0) bytes = 16;
  if (b.bytes < bytes) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    if (b.ptr) TESS_CUDA(cudaFree(b.ptr));
    b.ptr = nullptr;
    b.bytes = 0;
    // round up to 2 MiB to limit regrowth churn
    const size_t rounded = (bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
    TESS_CUDA(cudaMalloc(&b.ptr, rounded));
    b.bytes = rounded;
    cudaSetDevice(prev);
  }
  return b.ptr;
}

void Workspace::release_all() {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device_);
  for (auto& kv : bufs_)
    if (kv.second.ptr) cudaFree(kv.second.ptr);
  bufs_.clear();
  cudaSetDevice(prev);
}

size_t Workspace::bytes_held() const {
  size_t t = 0;
  for (auto& kv : bufs_) t += kv.second.bytes;
  return t;
}

std::string trace_text(const std::vector<TraceEvent>& trace) {
  static const char* kinds[5] = {"broadcast", "reduce", "all_reduce", "shift", "p2p"};
  static const char* groups[3] = {"row", "col", "depth"};
  std::string s;
  for (const auto& e : trace)
    s += std::to_string(e.rank) + ":" + std::to_string(e.step) + " " + kinds[e.kind] + " " +
         groups[e.group] + " " + std::to_string(e.root) + " " + std::to_string(e.bytes) + "\n";
  return s;
}

// ------------------------------------------------------------ local GEMM
namespace {
struct ProfRec {
  cudaEvent_t a, b;
  double flops;  // algorithmic 2*m*n*k (tensor-core launches)
  double bytes;  // compulsory HBM bytes (memory-bound launches)
  int device;
  std::string kernel;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
}  // namespace

ProfToken prof_begin(const std::string& kernel, double flops, cudaStream_t s, double bytes) {
  ProfToken t;
  if (!g_prof_on) return t;
  auto* rec = new ProfRec{nullptr, nullptr, flops, bytes, 0, kernel};
  cudaGetDevice(&rec->device);
  TESS_CUDA(cudaEventCreate(&rec->a));
  TESS_CUDA(cudaEventCreate(&rec->b));
  TESS_CUDA(cudaEventRecord(rec->a, s));
  t.rec = rec;
  return t;
}

void prof_end(ProfToken& t, cudaStream_t s) {
  if (!t.rec) return;
  auto* rec = static_cast<ProfRec*>(t.rec);
  t.rec = nullptr;
  TESS_CUDA(cudaEventRecord(rec->b, s));
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back(*rec);
  delete rec;
}

bool g_prof_detail = false;

bool prof_detail() {
  static const bool detail = [] {
    const char* e = std::getenv("TESS_PROFILE_DETAIL");
    return e && e[0] == '1';
  }();
  return detail || g_prof_detail;
}

void run_gemm(const GemmDesc& g, cudaStream_t s) {
  ProfToken tok;
  if (g_prof_on) {
    std::string name = gemm_kernel_name(g);
    double kk = 0;
    for (int i = 0; i < g.nseg; ++i) kk += (double)g.seg[i].k;
    if (prof_detail())
      name += " M=" + std::to_string(g.M) + " N=" + std::to_string(g.N) +
              " K=" + std::to_string((long long)kk) + " b=" + std::to_string(g.nb0 * g.nb1) +
              " epi=" + std::to_string((int)g.epi);
    tok = prof_begin(name, 2.0 * (double)g.M * (double)g.N * kk * (double)g.nb0 * (double)g.nb1, s);
  }
  cudaError_t e = gemm(g, s);
  count_launch();
  if (e == cudaErrorInvalidValue) fail(TESS_ERR_UNSUPPORTED, gemm_last_error());
  if (e != cudaSuccess)
    fail(TESS_ERR_CUDA, std::string("gemm: ") + cudaGetErrorString(e) + " " + gemm_last_error());
  prof_end(tok, s);
}

void profile_enable(int mode) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const bool on = mode != 0;
  g_prof_detail = mode == 2;
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_prof_on = on;
}

void profile_read(double* ms, double* flops, uint64_t* launches) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double t = 0, f = 0;
  uint64_t n = 0;
  for (auto& r : g_prof) {
    if (r.flops <= 0) continue;  // tensor-core launches only
    ++n;
    cudaSetDevice(r.device);
    TESS_CUDA(cudaEventSynchronize(r.b));
    float m = 0;
    TESS_CUDA(cudaEventElapsedTime(&m, r.a, r.b));
    t += m;
    f += r.flops;
  }
  if (ms) *ms = t;
  if (flops) *flops = f;
  if (launches) *launches = n;
}

// Per kernel instantiation: {"name": [ms, flops, launches, bytes], ...}
std::string profile_json() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::map<std::string, std::array<double, 4>> agg;
  for (auto& r : g_prof) {
    cudaSetDevice(r.device);
    TESS_CUDA(cudaEventSynchronize(r.b));
    float m = 0;
    TESS_CUDA(cudaEventElapsedTime(&m, r.a, r.b));
    auto& a = agg[r.kernel];
    a[0] += m;
    a[1] += r.flops;
    a[2] += 1;
    a[3] += r.bytes;
  }
  std::string s = "{";
  for (auto& kv : agg) {
    if (s.size() > 1) s += ", ";
    char buf[256];
    std::snprintf(buf, sizeof(buf), "\"%s\": [%.6f, %.6e, %.0f, %.6e]", kv.first.c_str(),
                  kv.second[0], kv.second[1], kv.second[2], kv.second[3]);
    s += buf;
  }
  return s + "}";
}

// ------------------------------------------------------- comm stream
cudaStream_t comm_stream(Ctx& c, cudaStream_t s) {
  if (c.grid.size() == 1) return s;
  if (!c.comm_s) {
    int lo = 0, hi = 0;
    TESS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TESS_CUDA(cudaStreamCreateWithPriority(&c.comm_s, cudaStreamNonBlocking, hi));
  }
  return c.comm_s;
}

void stream_dep(Ctx& c, cudaStream_t from, cudaStream_t to) {
  if (from == to) return;
  if (c.ev_ring.empty()) {
    c.ev_ring.resize(64);
    for (auto& e : c.ev_ring) TESS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaEvent_t e = c.ev_ring[c.ev_next++ % c.ev_ring.size()];
  TESS_CUDA(cudaEventRecord(e, from));
  TESS_CUDA(cudaStreamWaitEvent(to, e, 0));
}

// ------------------------------------------------------- collectives
static void trace_event(Ctx& c, int kind, Family f, int root, uint64_t elements) {
  const uint64_t step = c.step++;
  if (c.trace_on)
    c.trace.push_back({c.rank, step, kind, static_cast<int>(f), root, elements * 8});
}

void coll_note_single(Ctx& c, int kind, Family f, int root, uint64_t elements) {
  if (c.grid.group_size(f) != 1) fail(TESS_ERR_SPMD, "coll_note_single on a multi-rank group");
  trace_event(c, kind, f, root, elements);
}

// Fault injection (tess_inject_fault; the reference's verify inject_fault,
// verify.cpp:84-86, carried into the runtime): at this rank's collective
// number fault_at it fails (the SPMD error path) or silently skips the
// collective (its partners then block: deadlock detection names them).
static bool fault_skip(Ctx& c) {
  if (!c.fault_kind || (int64_t)c.step != c.fault_at) return false;
  const int k = c.fault_kind;
  c.fault_kind = 0;
  if (k == TESS_FAULT_RANK_FAIL)
    fail(TESS_ERR_SPMD, "injected failure at collective #" + std::to_string(c.step));
  if (k == TESS_FAULT_SKIP_COLLECTIVE) {
    ++c.step;
    return true;
  }
  return false;
}

void coll_bcast(Ctx& c, Family f, int root, void* buf, size_t bytes, uint64_t elements,
                cudaStream_t s) {
  if (fault_skip(c)) return;
  c.meter.bcast(c.grid.group_size(f), c.grid.slot_in_group(c.coord, f), root, elements);
  trace_event(c, 0, f, root, elements);
  if (!c.comm_noop) c.comm->bcast(f, root, buf, bytes, s);
}

Comm::PanelRecv coll_bcast_panel(Ctx& c, Family f, int root, const std::string& tag,
                                 const void* src, void* dst, size_t bytes, uint64_t elements,
                                 size_t chunk_bytes, cudaStream_t s) {
  if (fault_skip(c)) {
    Comm::PanelRecv r;
    r.buf = c.grid.slot_in_group(c.coord, f) == root ? src : dst;
    return r;
  }
  c.meter.bcast(c.grid.group_size(f), c.grid.slot_in_group(c.coord, f), root, elements);
  trace_event(c, 0, f, root, elements);
  const bool is_root = c.grid.slot_in_group(c.coord, f) == root;
  if (c.comm_noop || c.grid.group_size(f) == 1) {
    Comm::PanelRecv r;
    r.buf = is_root ? src : dst;
    return r;
  }
  return c.comm->panel_bcast(f, root, tag, src, dst, bytes, chunk_bytes, s);
}

void coll_reduce(Ctx& c, Family f, int root, const float* send, float* recv, size_t n,
                 cudaStream_t s) {
  if (fault_skip(c)) return;
  c.meter.reduce(c.grid.group_size(f), c.grid.slot_in_group(c.coord, f), root, n, false);
  trace_event(c, 1, f, root, n);
  if (!c.comm_noop) c.comm->reduce(f, root, send, recv, n, s);
}

void coll_reduce_note(Ctx& c, Family f, int root, size_t n) {
  if (fault_skip(c)) return;
  c.meter.reduce(c.grid.group_size(f), c.grid.slot_in_group(c.coord, f), root, n, false);
  trace_event(c, 1, f, root, n);
}

void coll_allreduce(Ctx& c, Family f, float* buf, size_t n, cudaStream_t s) {
  if (fault_skip(c)) return;
  c.meter.reduce(c.grid.group_size(f), c.grid.slot_in_group(c.coord, f), 0, n, true);
  trace_event(c, 2, f, 0, n);
  if (!c.comm_noop) c.comm->allreduce(f, buf, n, s);
}

}  // namespace tess

tess_ctx::~tess_ctx() {
  cudaSetDevice(device);
  if (comm_s) {
    cudaStreamSynchronize(comm_s);
    cudaStreamDestroy(comm_s);
  }
  if (copy_s) {
    cudaStreamSynchronize(copy_s);
    cudaStreamDestroy(copy_s);
  }
  for (auto& kv : copy_ev) cudaEventDestroy(kv.second);
  for (auto& kv : stage_free) cudaEventDestroy(kv.second);
  if (up_s) {
    cudaStreamSynchronize(up_s);
    cudaStreamDestroy(up_s);
  }
  for (auto e : ev_ring) cudaEventDestroy(e);
}
