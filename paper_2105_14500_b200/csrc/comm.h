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
  virtual void barrier() = 0;
  virtual void* nccl_comm(Family) { return nullptr; }
};

// ---------------------------------------------------------------- local
struct LocalWorld;

std::shared_ptr<LocalWorld> make_local_world(const Grid& g, const std::vector<int>& devices);
std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalWorld> w, int rank);
void local_world_fail(LocalWorld* w, const std::string& why);

// ----------------------------------------------------------------- nccl
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> make_nccl_comm(const Grid& g, int rank, const void* uid128);

// Sum of `n_in` device arrays (slot order) into out; used by LocalComm.
void launch_sum_f32(const float* const* in, int n_in, float* out, size_t n, cudaStream_t s);

}  // namespace tess
