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
  uint64_t step = 0;  // collective sequence number (RankCtx::step_)
  std::vector<tess::TraceEvent> trace;
  std::unique_ptr<tess::Workspace> ws;
  // Forward caches are named by (cache slot, layer op); the slot lets several
  // layers keep outstanding forwards (tess_set_cache_slot). The forward input
  // of each (slot, op) is remembered for the backward.
  int cache_slot = 0;
  std::map<int, const void*> fwd_x;
};

namespace tess {

using Ctx = tess_ctx;

// Metered, traced collectives over the rank's communicator (the
// RankCtx::broadcast / reduce / all_reduce of runtime.cpp:485-513).
// `elements` is the reference's payload element count (for the meter).
void coll_bcast(Ctx& c, Family f, int root, void* buf, size_t bytes, uint64_t elements,
                cudaStream_t s);
void coll_reduce(Ctx& c, Family f, int root, const float* send, float* recv, size_t n,
                 cudaStream_t s);
void coll_allreduce(Ctx& c, Family f, float* buf, size_t n, cudaStream_t s);

}  // namespace tess
