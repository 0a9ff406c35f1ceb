// NCCL backend: one process per GPU over NVLink 5 / NVSwitch.
//
// World communicator from a shared ncclUniqueId, then three ncclCommSplits
// whose (color, key) follow the reference's group geometry
// (proj/src/grid.cpp:79-95):
//   row    color = k*q + i, key = j   (slot in row group)
//   column color = k*q + j, key = i
//   depth  color = i*q + j, key = k
// so NCCL rank == reference slot in every group and root slots map 1:1.
// Collective mapping (reference runtime.hpp:105-121):
//   broadcast -> ncclBroadcast(root = slot)
//   reduce    -> ncclReduce(sum, root = slot)
//   all_reduce-> ncclAllReduce(sum)
// For the q = 2, d <= 2 target grids every group is a 2-party exchange, so
// the sums are a single commutative fp32 add and are identical on both ranks.
//
// NCCL is resolved at run time (dlopen) instead of being a link-time
// dependency: the process may already hold a different libnccl.so.2 (e.g. the
// one bundled with PyTorch), and two NCCL builds cannot share one process.
// Order: an already-loaded libnccl.so.2, $TESS_NCCL_LIBRARY, the system one.
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <thread>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>

#include "comm.h"
#include "peer.h"

namespace tess {

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int,
                         ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*CommAbort)(ncclComm_t);
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
      const char* env = std::getenv("TESS_NCCL_LIBRARY");
      if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && err.empty()) err = std::string("libnccl.so.2 lacks ") + n;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
    api.CommCount = reinterpret_cast<decltype(api.CommCount)>(sym("ncclCommCount"));
    api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(sym("ncclCommUserRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.Reduce = reinterpret_cast<decltype(api.Reduce)>(sym("ncclReduce"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.CommGetAsyncError =
        reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
  });
  if (!err.empty()) fail(TESS_ERR_SPMD, err);
  return api;
}

}  // namespace

#define TESS_NCCL(expr)                                                              \
  do {                                                                               \
    ncclResult_t r_ = (expr);                                                        \
    if (r_ != ncclSuccess)                                                           \
      ::tess::fail(TESS_ERR_SPMD, std::string(#expr) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  TESS_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
}

namespace {

class NcclComm : public Comm {
 public:
  NcclComm(const Grid& g, int rank, const void* uid128) : g_(g), rank_(rank) {
    c_ = g.coord_of(rank);
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    TESS_NCCL(nccl().CommInitRank(&world_, g.size(), id, rank));
    // No SMs are set aside for communication by default: the SUMMA panel
    // broadcasts of the q = 2 groups move on copy engines (PanelLink), the
    // NT/TN reduces inside the owner GEMMs (PeerWindow), so no GEMM ever
    // waits on an NCCL kernel; the remaining NCCL calls (LayerNorm row
    // statistics, depth all-reduces of weight gradients) run between GEMMs.
    // TESS_NCCL_SMS=n caps the communicators at n CTAs and makes the
    // persistent GEMMs leave n SMs free (the round-1 scheme).
    const char* env = std::getenv("TESS_NCCL_SMS");
    const int budget = env ? std::atoi(env) : 0;
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (budget > 0) {
      cfg.minCTAs = 1;
      cfg.maxCTAs = budget;
      if (g.size() > 1) gemm_set_sm_reserve(budget);
    }
    for (int f = 0; f < 3; ++f) {
      const Family fam = Family(f);
      if (g.group_size(fam) == 1) {
        comm_[f] = nullptr;
        // Every rank must still take part in the split (collective call).
        TESS_NCCL(nccl().CommSplit(world_, NCCL_SPLIT_NOCOLOR, 0, &comm_[f], nullptr));
        comm_[f] = nullptr;
        continue;
      }
      TESS_NCCL(nccl().CommSplit(world_, g.group_index(c_, fam), g.slot_in_group(c_, fam),
                              &comm_[f], budget > 0 ? &cfg : nullptr));
      int nr = 0, me = 0;
      TESS_NCCL(nccl().CommCount(comm_[f], &nr));
      TESS_NCCL(nccl().CommUserRank(comm_[f], &me));
      if (nr != g.group_size(fam) || me != g.slot_in_group(c_, fam))
        fail(TESS_ERR_SPMD, "ncclCommSplit produced an unexpected group layout");
    }
    const char* to = std::getenv("TESS_NCCL_TIMEOUT_S");
    timeout_s_ = to ? std::atof(to) : 600.0;
    TESS_CUDA(cudaGetDevice(&device_));
    watchdog_ = std::thread([this] { watch(); });
  }

  // Failure semantics (the reference aborts an SPMD run whose rank failed or
  // deadlocked, runtime.cpp:422-471): a watchdog polls every communicator's
  // asynchronous error and the age of the oldest incomplete collective; on
  // an NCCL error or a collective older than TESS_NCCL_TIMEOUT_S (default
  // 600 s: a dead or divergent peer) it aborts all communicators
  // (ncclCommAbort unblocks the kernels waiting on the peer) and every later
  // call of this rank fails with TESS_ERR_SPMD carrying the reason.
  void watch() {
    cudaSetDevice(device_);
    std::unique_lock<std::mutex> lk(wmu_);
    while (!stop_) {
      wcv_.wait_for(lk, std::chrono::milliseconds(50));
      if (stop_ || failed_) continue;
      std::string why;
      for (ncclComm_t cm : {world_, comm_[0], comm_[1], comm_[2]}) {
        if (!cm) continue;
        ncclResult_t st = ncclSuccess;
        if (nccl().CommGetAsyncError(cm, &st) == ncclSuccess && st != ncclSuccess &&
            st != ncclInProgress) {
          why = std::string("NCCL asynchronous error: ") + nccl().GetErrorString(st);
          break;
        }
      }
      while (why.empty() && !pending_.empty()) {
        const cudaError_t q = cudaEventQuery(pending_.front().ev);
        if (q == cudaErrorNotReady) {
          const double age = std::chrono::duration<double>(std::chrono::steady_clock::now() -
                                                           pending_.front().t0)
                                 .count();
          if (age > timeout_s_)
            why = "collective " + pending_.front().what + " did not complete within " +
                  std::to_string((int)timeout_s_) + " s (dead or divergent peer)";
          break;
        }
        cudaGetLastError();
        cudaEventDestroy(pending_.front().ev);
        pending_.pop_front();
      }
      if (!why.empty()) {
        failure_ = "rank (" + std::to_string(c_.i) + "," + std::to_string(c_.j) + "," +
                   std::to_string(c_.k) + "): " + why;
        failed_ = true;
        for (ncclComm_t cm : {comm_[0], comm_[1], comm_[2], world_})
          if (cm) nccl().CommAbort(cm);
        aborted_ = true;
      }
    }
  }

  void check_alive() {
    if (failed_) fail(TESS_ERR_SPMD, "aborted: " + failure_);
  }

  // Tracks the completion of the collective just enqueued on s.
  void track(const char* kind, Family f, cudaStream_t s) {
    cudaEvent_t ev;
    TESS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TESS_CUDA(cudaEventRecord(ev, s));
    std::lock_guard<std::mutex> lk(wmu_);
    pending_.push_back({ev, std::chrono::steady_clock::now(),
                        std::string(kind) + " #" + std::to_string(++ncoll_) + " in the " +
                            (f == ROW ? "row" : f == COL ? "column" : "depth") + " group"});
  }

  ~NcclComm() override {
    {
      std::lock_guard<std::mutex> lk(wmu_);
      stop_ = true;
    }
    wcv_.notify_all();
    if (watchdog_.joinable()) watchdog_.join();
    for (auto& p : pending_) cudaEventDestroy(p.ev);
    pending_.clear();
    if (aborted_) {  // communicators are gone; do not touch them again
      for (int f = 0; f < 3; ++f) comm_[f] = nullptr;
      world_ = nullptr;
    }
    cudaDeviceSynchronize();
    for (auto& m : links_) m.clear();
    for (auto& w : win_) {
      if (!w) continue;
      try {
        w->drain(0);
      } catch (...) {
      }
      w.reset();
    }
    for (int f = 0; f < 3; ++f)
      if (comm_[f]) nccl().CommDestroy(comm_[f]);
    if (world_) nccl().CommDestroy(world_);
  }

  void bcast(Family f, int root, void* buf, size_t bytes, cudaStream_t s) override {
    if (!comm_[f] || !bytes) return;
    check_alive();
    TESS_NCCL(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm_[f], s));
    track("broadcast", f, s);
  }

  void reduce(Family f, int root, const float* send, float* recv, size_t n,
              cudaStream_t s) override {
    if (!comm_[f]) {
      if (recv != send && n) TESS_CUDA(cudaMemcpyAsync(recv, send, n * 4, cudaMemcpyDeviceToDevice, s));
      return;
    }
    if (!n) return;
    check_alive();
    // Non-root recv buffers are ignored by NCCL; pass send to keep it valid.
    const bool is_root = g_.slot_in_group(c_, f) == root;
    TESS_NCCL(nccl().Reduce(send, is_root ? recv : const_cast<float*>(send), n, ncclFloat32,
                         ncclSum, root, comm_[f], s));
    track("reduce", f, s);
  }

  void allreduce(Family f, float* buf, size_t n, cudaStream_t s) override {
    if (!comm_[f] || !n) return;
    check_alive();
    TESS_NCCL(nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, comm_[f], s));
    track("all_reduce", f, s);
  }

  void barrier() override {
    check_alive();
    // A tiny all-reduce on the world communicator, then wait for it.
    float* tmp = nullptr;
    TESS_CUDA(cudaMalloc(&tmp, 4));
    TESS_CUDA(cudaMemset(tmp, 0, 4));
    TESS_NCCL(nccl().AllReduce(tmp, tmp, 1, ncclFloat32, ncclSum, world_, 0));
    TESS_CUDA(cudaStreamSynchronize(0));
    TESS_CUDA(cudaFree(tmp));
  }

  void* nccl_comm(Family f) override { return comm_[f]; }

  // Fused pair reduce over CUDA-IPC peer windows (peer.h): q = 2 groups.
  // Collective on first use per family (both members reach it at the same
  // program point): maps a small window and agrees on the outcome.
  bool pair_capable(Family f) override {
    if (!comm_[f] || g_.group_size(f) != 2) return false;
    if (!probed_[f]) {
      probed_[f] = true;
      make_window(f);
      pair_ok_[f] = win_[f]->probe(0);
      if (!pair_ok_[f]) win_[f].reset();
    }
    return pair_ok_[f];
  }

  float* pair_buffer(Family f, size_t n, cudaStream_t s) override {
    if (!pair_capable(f)) return nullptr;
    return win_[f]->acquire(n, s);
  }

  void make_window(Family f) { win_[f] = std::make_unique<PeerWindow>(exchange(f)); }

  // Blocking swap of `bytes` with the pair partner over f's communicator
  // (each slot broadcasts its own), for IPC handle exchanges.
  std::function<void(const void*, void*, size_t)> exchange(Family f) {
    {
      ncclComm_t cm = comm_[f];
      const int me = g_.slot_in_group(c_, f);
      return [cm, me](const void* mine, void* theirs, size_t bytes) {
        // drain: no earlier operation of this communicator may still be in
        // flight on another stream when the swap runs on the default stream
        TESS_CUDA(cudaDeviceSynchronize());
        void* d = nullptr;
        TESS_CUDA(cudaMalloc(&d, 2 * bytes));
        TESS_CUDA(cudaMemcpy(static_cast<char*>(d) + me * bytes, mine, bytes,
                             cudaMemcpyHostToDevice));
        for (int r = 0; r < 2; ++r) {
          char* slot = static_cast<char*>(d) + r * bytes;
          TESS_NCCL(nccl().Broadcast(slot, slot, bytes, ncclUint8, r, cm, 0));
        }
        TESS_CUDA(cudaStreamSynchronize(0));
        TESS_CUDA(cudaMemcpy(theirs, static_cast<char*>(d) + (1 - me) * bytes, bytes,
                             cudaMemcpyDeviceToHost));
        TESS_CUDA(cudaFree(d));
      };
    }
  }

  // SM-free panel broadcast (PanelLink): copy-engine pushes into the
  // receiver's IPC window + stream memory operations; no NCCL kernel.
  bool panel_async(Family f) override {
    static const bool off = std::getenv("TESS_PANEL_ASYNC") &&
                            std::getenv("TESS_PANEL_ASYNC")[0] == '0';
    return !off && memops_available() && pair_capable(f);
  }

  PanelRecv panel_bcast(Family f, int root, const std::string& tag, const void* src, void*,
                        size_t bytes, size_t chunk_bytes, cudaStream_t s) override {
    check_alive();
    const bool receiver = g_.slot_in_group(c_, f) != root;
    auto& link = links_[f][tag + "/" + std::to_string(root)];
    if (!link) link = std::make_unique<PanelLink>(exchange(f), receiver);
    PanelRecv r;
    r.epoch = link->push(receiver ? nullptr : src, bytes, chunk_bytes, s);
    if (receiver) {
      r.buf = link->data();
      r.flags = link->ready_flags();
      last_link_[f][tag] = link.get();
    } else {
      r.buf = src;
    }
    return r;
  }

  bool panel_owns_buffers() override { return true; }

  void panel_done(Family f, const std::string& tag, cudaStream_t s) override {
    auto it = last_link_[f].find(tag);
    if (it != last_link_[f].end()) it->second->done(s);
  }

  const float* pair_open(Family f, const float* mine, size_t, cudaStream_t s) override {
    if (!win_[f] || mine != win_[f]->local())
      fail(TESS_ERR_SPMD, "pair_open: contribution not in the peer window");
    return win_[f]->open(s);
  }

  void pair_close(Family f, cudaStream_t s) override {
    if (!win_[f]) fail(TESS_ERR_SPMD, "pair_close without pair_open");
    win_[f]->close(s);
  }

 private:
  Grid g_;
  int rank_;
  Coord c_;
  ncclComm_t world_ = nullptr;
  ncclComm_t comm_[3] = {nullptr, nullptr, nullptr};
  std::unique_ptr<PeerWindow> win_[3];
  std::map<std::string, std::unique_ptr<PanelLink>> links_[3];
  std::map<std::string, PanelLink*> last_link_[3];
  // watchdog
  struct Pending {
    cudaEvent_t ev;
    std::chrono::steady_clock::time_point t0;
    std::string what;
  };
  int device_ = 0;
  double timeout_s_ = 600.0;
  std::thread watchdog_;
  std::mutex wmu_;
  std::condition_variable wcv_;
  std::deque<Pending> pending_;
  uint64_t ncoll_ = 0;
  bool stop_ = false;
  std::atomic<bool> failed_{false};
  bool aborted_ = false;
  std::string failure_;
  bool probed_[3] = {false, false, false};
  bool pair_ok_[3] = {false, false, false};
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const Grid& g, int rank, const void* uid128) {
  return std::make_unique<NcclComm>(g, rank, uid128);
}

}  // namespace tess
