// Communicator backends for the three Tesseract group families.
//
// Replaces the reference's in-process rendezvous engine
// (proj/src/runtime.cpp:221-372, CollectiveEngine::collective /
// complete_round_locked). Two backends implement the same stream-ordered
// interface:
//   * NcclComm  -- one process per GPU; ncclCommSplit of a world comm into
//                  row/column/depth communicators (NVLink 5 / NVSwitch).
//   * LocalComm -- one host thread per rank inside one process (devices may
//                  repeat, so a whole [2,2,2] grid runs on one B200 for
//                  parity tests): host rendezvous exchanging device pointers
//                  and CUDA events, data moved by stream-ordered device
//                  copies / peer reads, sums in slot-ascending order exactly
//                  like the reference engine (runtime.cpp:310-312).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "core.h"

namespace tess {

class Comm {
 public:
  virtual ~Comm() = default;
  // Root's `buf` is sent; every other member receives into its own `buf`.
  virtual void bcast(Family f, int root, void* buf, size_t bytes, cudaStream_t s) = 0;
  // Slot-ascending fp32 sum of `send` over the group delivered into `recv`
  // at the root (recv unused elsewhere; may alias send at the root).
  virtual void reduce(Family f, int root, const float* send, float* recv, size_t n,
                      cudaStream_t s) = 0;
  // In-place fp32 sum delivered at every member.
  virtual void allreduce(Family f, float* buf, size_t n, cudaStream_t s) = 0;
  // Pair exchange for reductions fused into a GEMM epilogue (groups of two):
  // publishes `mine` (ready once s reaches this point) and returns the
  // partner's buffer, readable from this rank's device, with s ordered after
  // the partner's ready point; nullptr when the backend cannot map peer
  // memory (the caller then uses reduce). pair_close marks the end of the
  // reads on s and orders s after the partner's reads of `mine`.
  virtual bool pair_capable(Family) { return false; }
  // Buffer for this rank's contribution when the backend needs it in memory
  // it exported to the partner (collective: both members, same n); nullptr
  // = any device buffer will do.
  virtual float* pair_buffer(Family, size_t /*n*/, cudaStream_t) { return nullptr; }
  virtual const float* pair_open(Family, const float* /*mine*/, size_t /*n*/, cudaStream_t) {
    return nullptr;
  }
  virtual void pair_close(Family, cudaStream_t) {}
  // SM-free panel broadcast (summa.cpp): the receiver's GEMM may be launched
  // before the panel lands and waits per chunk on device flags (GemmReady).
  // panel_async(f): the backend can deliver f's panels without any SM
  // (copy engines + stream memory operations) and the group is a pair on
  // distinct GPUs, so a spinning GEMM cannot starve the transfer.
  virtual bool panel_async(Family) { return false; }
  struct PanelRecv {
    const void* buf = nullptr;       // where the panel is (root: src)
    const uint32_t* flags = nullptr; // receiver: ready[c] per chunk
    uint32_t epoch = 0;              // the value ready[c] reaches
  };
  // Collective over f (both members, same program order): root slot
  // `root` sends `src` (bytes, in chunks of chunk_bytes); the receiver's
  // copy lands in `dst` or a backend buffer (returned). Stream order on s
  // after the root's producer; the receiver's flags are written on the
  // transfer's own stream order. `tag` names the link (one per panel role).
  virtual PanelRecv panel_bcast(Family, int /*root*/, const std::string& /*tag*/,
                                const void* /*src*/, void* /*dst*/, size_t /*bytes*/,
                                size_t /*chunk_bytes*/, cudaStream_t) {
    fail(TESS_ERR_UNSUPPORTED, "panel_bcast: backend has no SM-free transport");
  }
  // Receiver: its reads of the link's last panel are done (stream order s).
  virtual void panel_done(Family, const std::string& /*tag*/, cudaStream_t) {}
  // The backend lands received panels in buffers of its own (dst unused).
  virtual bool panel_owns_buffers() { return false; }
  virtual void barrier() = 0;
  virtual void* nccl_comm(Family) { return nullptr; }
};

// ---------------------------------------------------------------- local
struct LocalWorld;

std::shared_ptr<LocalWorld> make_local_world(const Grid& g, const std::vector<int>& devices);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank);
void local_world_fail(LocalWorld* w, const std::string& why);
// The rank will make no further collective calls (its SPMD function
// returned, or its context is destroyed): deadlock detection counts it.
void local_world_rank_finished(LocalWorld* w, int rank);

// ----------------------------------------------------------------- nccl
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const Grid& g, int rank, const void* uid128);

// Sum of `n_in` device arrays (slot order) into out; used by LocalComm.
void launch_sum_f32(const float* const* in, int n_in, float* out, size_t n, cudaStream_t s);

}  // namespace tess
