// Per-rank context: the B200 counterpart of the reference's RankCtx
// (proj/include/tsim/runtime.hpp:95-136) plus the device resources a rank
// owns (communicators, workspace, layer caches).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "comm.h"
#include "core.h"

struct tess_ctx {
  tess::Grid grid;
  tess::Coord coord;
  int rank = 0;
  int device = 0;
  std::unique_ptr<tess::Comm> comm;
  std::shared_ptr<tess::LocalWorld> world;  // in-process backend only
  tess::Meter meter;
  bool trace_on = false;
  // Measurement only (tess_set_comm_noop): collectives are metered and traced
  // but move no data, to time the step without communication (exposed comm).
  bool comm_noop = false;
  // 1-D tensor-parallel (Megatron) layer scheme on a [1,1,p] line grid
  // (tess_set_megatron; BASELINE config 5's comparator): activations
  // replicated, W_qkv / W_ff1 column-split, W_proj / W_ff2 row-split, the
  // partial outputs of proj / FF2 (forward) and QKV / FF1 dgrads (backward)
  // all-reduced over the depth group; weight shards are not depth-reduced.
  bool megatron = false;
  uint64_t step = 0;  // collective sequence number (RankCtx::step_)
  // Fault injection (tess_inject_fault): at collective number fault_at this
  // rank fails (2) or skips the collective (3); one-shot.
  int fault_kind = 0;
  int64_t fault_at = -1;
  std::vector<tess::TraceEvent> trace;
  std::unique_ptr<tess::Workspace> ws;
  // Forward caches are named by (cache slot, layer op); the slot lets several
  // layers keep outstanding forwards (tess_set_cache_slot). The forward input
  // of each (slot, op) is remembered for the backward.
  int cache_slot = 0;
  std::map<int, const void*> fwd_x;
  // High-priority stream carrying this rank's collectives so they overlap
  // the compute stream (created on first use; the compute stream itself when
  // the grid has a single rank). Cross-stream ordering uses a ring of events.
  cudaStream_t comm_s = nullptr;
  // Side stream for host copies of layer outputs (overlaps the next call);
  // pending device->host copies per staging buffer, joined before the buffer
  // is rewritten or by tess_stream_join.
  cudaStream_t copy_s = nullptr;
  std::map<std::string, cudaEvent_t> copy_ev;
  std::map<std::string, std::pair<const char*, size_t>> copy_host;  // host range per copy
  // Upload stream of tess_layer_step: host x and dy go up into staging
  // buffers double-buffered per call (stage_par), each copy waiting only for
  // its buffer's previous reader (stage_free), so it overlaps the previous
  // step's compute.
  cudaStream_t up_s = nullptr;
  std::map<std::string, int> stage_par;
  std::map<std::string, cudaEvent_t> stage_free;
  std::vector<cudaEvent_t> ev_ring;
  size_t ev_next = 0;
  ~tess_ctx();
};

namespace tess {

using Ctx = tess_ctx;

// Metered, traced collectives over the rank's communicator (the
// RankCtx::broadcast / reduce / all_reduce of runtime.cpp:485-513).
// `elements` is the reference's payload element count (for the meter).
void coll_bcast(Ctx& c, Family f, int root, void* buf, size_t bytes, uint64_t elements,
                cudaStream_t s);
// The SM-free form of coll_bcast (Comm::panel_bcast), same meter and trace:
// the receiver's panel may still be landing when this returns on the
// device; its GEMM waits on the returned flags (GemmReady).
Comm::PanelRecv coll_bcast_panel(Ctx& c, Family f, int root, const std::string& tag,
                                 const void* src, void* dst, size_t bytes, uint64_t elements,
                                 size_t chunk_bytes, cudaStream_t s);
void coll_reduce(Ctx& c, Family f, int root, const float* send, float* recv, size_t n,
                 cudaStream_t s);
void coll_allreduce(Ctx& c, Family f, float* buf, size_t n, cudaStream_t s);
// Meters and traces a reduce whose data movement is fused into the owner's
// GEMM epilogue (summa.cpp pair reduce): same CommStats / trace entry.
void coll_reduce_note(Ctx& c, Family f, int root, size_t n);

// Records a collective whose group has a single member (no data moves): the
// reference still counts the call in its trace step sequence.
void coll_note_single(Ctx& c, int kind, Family f, int root, uint64_t elements);

// Makes s wait for everything this context still has in flight on its side
// streams (collectives, host copies of layer outputs): tess_stream_join.
void ctx_join(Ctx& c, cudaStream_t s);

// The rank's comm stream (== s when the grid has one rank).
cudaStream_t comm_stream(Ctx& c, cudaStream_t s);
// Makes `to` wait for everything enqueued on `from` so far (no-op if equal).
void stream_dep(Ctx& c, cudaStream_t from, cudaStream_t to);

}  // namespace tess
