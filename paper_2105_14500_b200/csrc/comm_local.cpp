// In-process, thread-per-rank communicator (see comm.h).
//
// Protocol per collective on a group of g ranks (all members call it in the
// same program order, as the reference requires, runtime.hpp:91-94):
//   phase A: every member records a "ready" event on its stream after the
//            data it contributes (or the buffer it will overwrite) is ready,
//            posts {pointer, event, signature} and meets the others at a host
//            barrier; signatures must agree (runtime.cpp:236-248).
//   move   : receivers / reducers make their stream wait on the peers'
//            ready events and move data with device copies or a slot-
//            ascending sum kernel that reads the peers' buffers directly.
//   phase B: members post "done" events and meet again; anyone whose buffer
//            is read by others waits on those events before reusing it.
// Posts are double buffered by call parity, so two barriers per call are
// enough. A failing rank marks the world failed and every waiter aborts
// with TESS_ERR_SPMD instead of deadlocking (runtime.cpp:422-471).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>

#include <cstdlib>
#include <map>

#include "comm.h"
#include "peer.h"

namespace tess {

namespace {

struct Post {
  const void* ptr = nullptr;
  cudaEvent_t ev = nullptr;
  int kind = -1;
  int root = -1;
  size_t bytes = 0;
};

struct Rendezvous {
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<Post> a[2], b[2];
};

}  // namespace

// What a blocked rank is waiting for (deadlock diagnosis).
struct WaitInfo {
  bool active = false;
  const Rendezvous* rv = nullptr;
  std::string what;
};

struct LocalWorld {
  Grid grid;
  std::vector<int> devices;
  std::vector<std::unique_ptr<Rendezvous>> rv[3];
  Rendezvous world;
  std::atomic<bool> failed{false};
  std::mutex fail_mu;
  std::string failure;
  // Deadlock detection (the reference's deadlock_check_locked,
  // runtime.cpp:433-471): every live rank blocked in a rendezvous that can
  // no longer complete means mismatched participation; the failure names
  // each waiting rank and what it waits on.
  std::mutex state_mu;
  std::vector<WaitInfo> waiting;
  std::vector<bool> done;
  int finished = 0;

  void mark_failed(const std::string& why) {
    std::lock_guard<std::mutex> lk(fail_mu);
    if (!failed.exchange(true)) failure = why;
  }

  // Every live rank blocked (caller holds state_mu): the last one to block
  // declares the deadlock. A round that completes clears its waiters first.
  void deadlock_check_locked() {
    int blocked = 0;
    for (const WaitInfo& w : waiting) blocked += w.active;
    if (blocked == 0 || blocked + finished < grid.size()) return;
    std::string msg = "deadlock: mismatched participation; divergent ranks:";
    for (int r = 0; r < grid.size(); ++r) {
      const WaitInfo& w = waiting[r];
      if (!w.active) continue;
      const Coord c = grid.coord_of(r);
      msg += " (" + std::to_string(c.i) + "," + std::to_string(c.j) + "," + std::to_string(c.k) +
             ") waits on " + w.what + ";";
    }
    if (finished > 0) msg += " " + std::to_string(finished) + " rank(s) already finished";
    mark_failed(msg);
  }

  void rank_finished(int rank) {
    std::lock_guard<std::mutex> lk(state_mu);
    if (rank < 0 || rank >= (int)done.size() || done[rank]) return;
    done[rank] = true;
    ++finished;
    if (!failed.load()) deadlock_check_locked();
  }

  void wait(Rendezvous& r, int gsize, int rank = -1, const std::string& what = std::string()) {
    std::unique_lock<std::mutex> lk(r.mu);
    const uint64_t g = r.gen;
    if (++r.arrived == gsize) {
      r.arrived = 0;
      ++r.gen;
      {
        std::lock_guard<std::mutex> sl(state_mu);
        for (WaitInfo& w : waiting)
          if (w.active && w.rv == &r) w.active = false;
      }
      r.cv.notify_all();
      return;
    }
    if (rank >= 0) {
      std::lock_guard<std::mutex> sl(state_mu);
      waiting[rank] = {true, &r, what};
      if (!failed.load()) deadlock_check_locked();
    }
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(600);
    while (r.gen == g) {
      r.cv.wait_for(lk, std::chrono::milliseconds(20));
      if (r.gen != g) break;
      if (failed.load()) {
        if (rank >= 0) {
          std::lock_guard<std::mutex> sl(state_mu);
          waiting[rank].active = false;
        }
        fail(TESS_ERR_SPMD, "aborted: " + failure);
      }
      if (std::chrono::steady_clock::now() > deadline) {
        mark_failed("collective rendezvous timed out after 600 s waiting on " + what);
        fail(TESS_ERR_SPMD, "collective rendezvous timed out after 600 s waiting on " + what);
      }
    }
  }
};

std::shared_ptr<LocalWorld> make_local_world(const Grid& g, const std::vector<int>& devices) {
  auto w = std::make_shared<LocalWorld>();
  w->grid = g;
  w->devices = devices;
  w->waiting.resize(g.size());
  w->done.assign(g.size(), false);
  for (int f = 0; f < 3; ++f) {
    const int n = g.group_count(Family(f));
    const int gs = g.group_size(Family(f));
    for (int i = 0; i < n; ++i) {
      auto r = std::make_unique<Rendezvous>();
      for (int p = 0; p < 2; ++p) {
        r->a[p].resize(gs);
        r->b[p].resize(gs);
      }
      w->rv[f].push_back(std::move(r));
    }
  }
  // Peer access between distinct devices so sum kernels can read peers.
  std::vector<int> uniq;
  for (int dv : devices)
    if (std::find(uniq.begin(), uniq.end(), dv) == uniq.end()) uniq.push_back(dv);
  for (int a : uniq)
    for (int b : uniq) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (can) {
        cudaSetDevice(a);
        cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          fail(TESS_ERR_CUDA, "cudaDeviceEnablePeerAccess failed");
        cudaGetLastError();
      }
    }
  if (!devices.empty()) cudaSetDevice(devices[0]);
  return w;
}

namespace {

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalWorld> w, int rank) : w_(std::move(w)), rank_(rank) {
    c_ = w_->grid.coord_of(rank);
    device_ = w_->devices[rank];
    TESS_CUDA(cudaSetDevice(device_));
    for (int f = 0; f < 3; ++f)
      for (int p = 0; p < 2; ++p) {
        TESS_CUDA(cudaEventCreateWithFlags(&ev_a_[f][p], cudaEventDisableTiming));
        TESS_CUDA(cudaEventCreateWithFlags(&ev_b_[f][p], cudaEventDisableTiming));
      }
  }

  ~LocalComm() override {
    cudaSetDevice(device_);
    for (int f = 0; f < 3; ++f)
      for (int p = 0; p < 2; ++p) {
        cudaEventDestroy(ev_a_[f][p]);
        cudaEventDestroy(ev_b_[f][p]);
      }
    if (scratch_) cudaFree(scratch_);
    for (auto& m : flags_)
      for (auto& kv : m) cudaFree(kv.second);
  }

  void bcast(Family f, int root, void* buf, size_t bytes, cudaStream_t s) override {
    Ctx x = enter(f, 0, root, bytes, buf, s);
    if (!x.rv) return;
    if (x.slot != root && bytes) {
      TESS_CUDA(cudaStreamWaitEvent(s, x.rv->a[x.par][root].ev, 0));
      TESS_CUDA(cudaMemcpyAsync(buf, x.rv->a[x.par][root].ptr, bytes, cudaMemcpyDefault, s));
    }
    TESS_CUDA(cudaEventRecord(ev_b_[f][x.par], s));
    x.rv->b[x.par][x.slot] = {buf, ev_b_[f][x.par], 0, root, bytes};
    w_->wait(*x.rv, x.gsize, rank_, x.what + " (completion)");
    if (x.slot == root)
      for (int o = 0; o < x.gsize; ++o)
        if (o != root) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->b[x.par][o].ev, 0));
  }

  void reduce(Family f, int root, const float* send, float* recv, size_t n,
              cudaStream_t s) override {
    Ctx x = enter(f, 1, root, n * 4, send, s);
    if (!x.rv) {
      if (recv != send && n) TESS_CUDA(cudaMemcpyAsync(recv, send, n * 4, cudaMemcpyDefault, s));
      return;
    }
    if (x.slot == root && n) {
      const float* ptrs[8];
      for (int o = 0; o < x.gsize; ++o) {
        if (o != x.slot) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->a[x.par][o].ev, 0));
        ptrs[o] = static_cast<const float*>(x.rv->a[x.par][o].ptr);
      }
      launch_sum_f32(ptrs, x.gsize, recv, n, s);
    }
    TESS_CUDA(cudaEventRecord(ev_b_[f][x.par], s));
    x.rv->b[x.par][x.slot] = {recv, ev_b_[f][x.par], 1, root, n * 4};
    w_->wait(*x.rv, x.gsize, rank_, x.what + " (completion)");
    if (x.slot != root) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->b[x.par][root].ev, 0));
  }

  void allreduce(Family f, float* buf, size_t n, cudaStream_t s) override {
    Ctx x = enter(f, 2, 0, n * 4, buf, s);
    if (!x.rv) return;
    if (n) {
      ensure_scratch(n);
      const float* ptrs[8];
      for (int o = 0; o < x.gsize; ++o) {
        if (o != x.slot) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->a[x.par][o].ev, 0));
        ptrs[o] = static_cast<const float*>(x.rv->a[x.par][o].ptr);
      }
      launch_sum_f32(ptrs, x.gsize, scratch_, n, s);
    }
    TESS_CUDA(cudaEventRecord(ev_b_[f][x.par], s));
    x.rv->b[x.par][x.slot] = {buf, ev_b_[f][x.par], 2, 0, n * 4};
    w_->wait(*x.rv, x.gsize, rank_, x.what + " (completion)");
    if (n) {
      for (int o = 0; o < x.gsize; ++o)
        if (o != x.slot) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->b[x.par][o].ev, 0));
      TESS_CUDA(cudaMemcpyAsync(buf, scratch_, n * 4, cudaMemcpyDeviceToDevice, s));
    }
  }

  // Phase A of a kind-3 call: exchange {pointer, ready event}; phase B in
  // pair_close. Peer pointers are directly addressable (same device, or a
  // peer device with peer access enabled by make_local_world).
  bool pair_capable(Family f) override {
    const Grid& g = w_->grid;
    if (g.group_size(f) != 2) return false;
    const int other_dev = w_->devices[g.rank_of(
        g.member_at(f, g.group_index(c_, f), 1 - g.slot_in_group(c_, f)))];
    int can = 1;
    if (other_dev != device_) cudaDeviceCanAccessPeer(&can, device_, other_dev);
    return can != 0;
  }

  const float* pair_open(Family f, const float* mine, size_t n, cudaStream_t s) override {
    if (!pair_capable(f)) return nullptr;
    Ctx x = enter(f, 3, 0, n * 4, mine, s);
    pair_ = x;
    pair_f_ = f;
    const Post& o = x.rv->a[x.par][1 - x.slot];
    TESS_CUDA(cudaStreamWaitEvent(s, o.ev, 0));
    return static_cast<const float*>(o.ptr);
  }

  void pair_close(Family f, cudaStream_t s) override {
    Ctx x = pair_;
    if (!x.rv || f != pair_f_) fail(TESS_ERR_SPMD, "pair_close without pair_open");
    pair_ = Ctx();
    TESS_CUDA(cudaEventRecord(ev_b_[f][x.par], s));
    x.rv->b[x.par][x.slot] = {nullptr, ev_b_[f][x.par], 3, 0, 0};
    w_->wait(*x.rv, x.gsize, rank_, x.what + " (completion)");
    TESS_CUDA(cudaStreamWaitEvent(s, x.rv->b[x.par][1 - x.slot].ev, 0));
  }

  // SM-free panel broadcast between two distinct GPUs of this process: the
  // receiver pulls the root's panel with peer copies (copy engines over
  // NVLink) chunk by chunk, each chunk followed by a stream memory write of
  // its ready flag. Ranks sharing one GPU keep the event-ordered bcast: a
  // GEMM spinning on a flag could otherwise hold the SMs the partner's
  // producer kernels need.
  bool panel_async(Family f) override {
    static const bool off = std::getenv("TESS_PANEL_ASYNC") &&
                            std::getenv("TESS_PANEL_ASYNC")[0] == '0';
    const Grid& g = w_->grid;
    if (off || g.group_size(f) != 2 || !memops_available()) return false;
    const int other_dev = w_->devices[g.rank_of(
        g.member_at(f, g.group_index(c_, f), 1 - g.slot_in_group(c_, f)))];
    if (other_dev == device_) return false;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, device_, other_dev);
    return can != 0;
  }

  PanelRecv panel_bcast(Family f, int root, const std::string& tag, const void* src, void* dst,
                        size_t bytes, size_t chunk_bytes, cudaStream_t s) override {
    Ctx x = enter(f, 4, root, bytes, x_slot(f) == root ? src : dst, s);
    PanelRecv r;
    r.buf = x.slot == root ? src : dst;
    if (!x.rv) return r;
    if (x.slot != root && bytes) {
      uint32_t*& fl = flags_[f][tag];
      if (!fl) {
        TESS_CUDA(cudaMalloc(&fl, PanelLink::kMaxChunks * 4));
        TESS_CUDA(cudaMemset(fl, 0, PanelLink::kMaxChunks * 4));
      }
      const uint32_t e = ++epoch_[f][tag];
      if (!chunk_bytes || chunk_bytes > bytes) chunk_bytes = bytes;
      const size_t n = (bytes + chunk_bytes - 1) / chunk_bytes;
      if (n > (size_t)PanelLink::kMaxChunks) fail(TESS_ERR_INVALID, "panel_bcast: too many chunks");
      TESS_CUDA(cudaStreamWaitEvent(s, x.rv->a[x.par][root].ev, 0));
      const char* from = static_cast<const char*>(x.rv->a[x.par][root].ptr);
      for (size_t c = 0; c < n; ++c) {
        const size_t off = c * chunk_bytes, len = std::min(chunk_bytes, bytes - off);
        TESS_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, from + off, len,
                                  cudaMemcpyDefault, s));
        stream_write_u32(s, fl + c, e);
      }
      r.flags = fl;
      r.epoch = e;
    }
    TESS_CUDA(cudaEventRecord(ev_b_[f][x.par], s));
    x.rv->b[x.par][x.slot] = {r.buf, ev_b_[f][x.par], 4, root, bytes};
    w_->wait(*x.rv, x.gsize, rank_, x.what + " (completion)");
    if (x.slot == root)
      for (int o = 0; o < x.gsize; ++o)
        if (o != root) TESS_CUDA(cudaStreamWaitEvent(s, x.rv->b[x.par][o].ev, 0));
    return r;
  }

  void barrier() override { w_->wait(w_->world, w_->grid.size(), rank_, "barrier"); }

 private:
  struct Ctx {
    Rendezvous* rv = nullptr;
    int slot = 0, gsize = 1, par = 0;
    std::string what;
  };

  Ctx enter(Family f, int kind, int root, size_t bytes, const void* ptr, cudaStream_t s) {
    Ctx x;
    const Grid& g = w_->grid;
    x.gsize = g.group_size(f);
    x.slot = g.slot_in_group(c_, f);
    if (root < 0 || root >= x.gsize)
      fail(TESS_ERR_SPMD, "collective root slot " + std::to_string(root) + " out of range");
    if (x.gsize == 1) return x;
    if (x.gsize > 8) fail(TESS_ERR_UNSUPPORTED, "local backend supports groups of <= 8");
    TESS_CUDA(cudaSetDevice(device_));
    x.rv = w_->rv[f][g.group_index(c_, f)].get();
    const uint64_t call = calls_[f]++;
    x.par = static_cast<int>(call & 1);
    TESS_CUDA(cudaEventRecord(ev_a_[f][x.par], s));
    x.rv->a[x.par][x.slot] = {ptr, ev_a_[f][x.par], kind, root, bytes};
    static const char* kinds[] = {"broadcast", "reduce", "all_reduce", "pair exchange",
                                  "panel broadcast"};
    x.what = std::string(kinds[kind]) + " (root slot " + std::to_string(root) + ", " +
             std::to_string(bytes) + " bytes) in " +
             (f == ROW ? "row" : f == COL ? "column" : "depth") + " group " +
             std::to_string(g.group_index(c_, f)) + ", its collective #" + std::to_string(call) +
             " there";
    w_->wait(*x.rv, x.gsize, rank_, x.what);
    const Post& p0 = x.rv->a[x.par][0];
    const Post& me = x.rv->a[x.par][x.slot];
    if (p0.kind != me.kind || p0.root != me.root || p0.bytes != me.bytes) {
      const std::string msg = "mismatched collective in " +
                              std::string(f == ROW ? "row" : f == COL ? "col" : "depth") +
                              " group " + std::to_string(g.group_index(c_, f)) + " at rank " +
                              std::to_string(rank_);
      w_->mark_failed(msg);
      fail(TESS_ERR_SPMD, msg);
    }
    return x;
  }

  void ensure_scratch(size_t n) {
    if (n <= scratch_n_) return;
    if (scratch_) TESS_CUDA(cudaFree(scratch_));
    TESS_CUDA(cudaMalloc(&scratch_, n * 4));
    scratch_n_ = n;
  }

  std::shared_ptr<LocalWorld> w_;
  int rank_;
  Coord c_;
  int device_;
  cudaEvent_t ev_a_[3][2], ev_b_[3][2];
  uint64_t calls_[3] = {0, 0, 0};
  float* scratch_ = nullptr;
  size_t scratch_n_ = 0;
  Ctx pair_;  // open pair exchange (pair_open .. pair_close)
  Family pair_f_ = ROW;
  std::map<std::string, uint32_t*> flags_[3];  // panel_bcast ready flags per link
  std::map<std::string, uint32_t> epoch_[3];

  int x_slot(Family f) const { return w_->grid.slot_in_group(c_, f); }
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank) {
  return std::make_unique<LocalComm>(std::move(w), rank);
}

void local_world_fail(LocalWorld* w, const std::string& why) { w->mark_failed(why); }

void local_world_rank_finished(LocalWorld* w, int rank) { w->rank_finished(rank); }

}  // namespace tess
