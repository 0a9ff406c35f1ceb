// Peer window: a device buffer this rank exports to its partner in a
// two-member group through CUDA IPC (one process per GPU over NVLink /
// NVSwitch), so a GEMM epilogue on one GPU can read the other's partial
// directly — the transport of the fused pair reduce (summa.cpp). Replaces the
// data movement of RankCtx::reduce (reference runtime.cpp:485-513) for q = 2
// groups; ordering is stream-level, with no host synchronisation per use:
//
//   acquire(n, s) -> local buffer; s waits until the partner has finished
//                    reading this buffer's previous contents ("done" >= e)
//   open(s)       -> partner's buffer; signals "ready" = e+1 to the partner
//                    and makes s wait for the partner's "ready" >= e+1
//   close(s)      -> signals "done" = e+1 (this rank stopped reading); e++
//
// The header of each window holds the two sequence words the PARTNER writes
// (system-scope release stores, kernels/peer.cu). Growing the window is
// collective (both members call acquire with the same n): streams are
// drained, the partner's old mapping is closed and new IPC handles are
// exchanged through the caller-supplied blocking `Exchange`.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>

namespace tess {

// Stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32 via
// the driver entry points): executed by the stream's front end, no SM
// involved -- the signalling of the SM-free panel transport. The write is
// preceded by a memory fence (the bytes copied before it on the stream are
// visible first); the wait is wrap-safe ((int32)(*p - v) >= 0).
bool memops_available();
void stream_write_u32(cudaStream_t s, uint32_t* p, uint32_t v);
void stream_wait_u32_geq(cudaStream_t s, const uint32_t* p, uint32_t v);

// One-way panel link of a two-member group for the SM-free broadcast of
// SUMMA panels (summa.cpp; NCCL backend, one process per GPU). The receiver
// owns a window [header | data] exported with CUDA IPC; the root maps it,
// pushes the panel with copy-engine copies in row chunks and after each
// chunk writes ready[c] = epoch into the receiver's header with a stream
// memory operation. The receiver's GEMM waits on ready[c] on the device
// (GemmReady) and, once done reading, writes done = epoch into the root's
// (header-only) window; the root's next push waits for it with a stream
// wait. No kernel and no SM is involved on either side, so a persistent
// GEMM spinning on a chunk cannot starve the transfer.
class PanelLink {
 public:
  using Exchange = std::function<void(const void* mine, void* theirs, size_t bytes)>;
  static constexpr int kMaxChunks = 32;

  PanelLink(Exchange ex, bool receiver) : ex_(std::move(ex)), receiver_(receiver) {}
  ~PanelLink();
  PanelLink(const PanelLink&) = delete;
  PanelLink& operator=(const PanelLink&) = delete;

  // Collective (both members, same program order, same bytes / chunking).
  // Root: pushes `src` on s. Receiver: nothing is enqueued. Returns the
  // epoch of this transfer; the receiver's panel is data(), its flags
  // ready_flags().
  uint32_t push(const void* src, size_t bytes, size_t chunk_bytes, cudaStream_t s);
  // Receiver: its reads of the last panel are done in stream order on s.
  void done(cudaStream_t s);
  const void* data() const;
  const uint32_t* ready_flags() const;

 private:
  static constexpr size_t kHeader = 256;  // ready[0..31] | done (word 32)
  void grow(size_t bytes);

  Exchange ex_;
  bool receiver_;
  void* base_ = nullptr;  // own window (receiver: header + data; root: header)
  void* peer_ = nullptr;  // the partner's window
  size_t cap_ = 0;
  uint32_t epoch_ = 0;
};

class PeerWindow {
 public:
  // exchange(mine, theirs, bytes): blocking swap of `bytes` with the partner.
  using Exchange = std::function<void(const void* mine, void* theirs, size_t bytes)>;

  explicit PeerWindow(Exchange ex) : ex_(std::move(ex)) {}
  ~PeerWindow();
  PeerWindow(const PeerWindow&) = delete;
  PeerWindow& operator=(const PeerWindow&) = delete;

  // Collective first mapping of a small window; false (on both members)
  // when either side cannot map the other's memory (no peer access between
  // the GPUs, devices hidden from the process): the caller then keeps the
  // collective path.
  bool probe(cudaStream_t s);
  float* acquire(size_t n, cudaStream_t s);
  const float* open(cudaStream_t s);
  void close(cudaStream_t s);
  // Blocks until the partner stopped reading our window (before teardown).
  void drain(cudaStream_t s);
  float* local() const { return data(base_); }

 private:
  static constexpr size_t kHeader = 256;  // [0] ready, [1] done (written by the partner)
  static float* data(void* b) {
    return b ? reinterpret_cast<float*>(static_cast<char*>(b) + kHeader) : nullptr;
  }
  static uint32_t* flags(void* b) { return static_cast<uint32_t*>(b); }
  bool grow(size_t n, cudaStream_t s);

  Exchange ex_;
  void* base_ = nullptr;  // own window (cudaMalloc, exported)
  void* peer_ = nullptr;  // partner's window (cudaIpcOpenMemHandle)
  size_t cap_ = 0;        // floats
  uint32_t epoch_ = 0;
  bool opened_ = false;
};

}  // namespace tess
