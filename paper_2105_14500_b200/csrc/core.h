// Internal host-side core: errors, grid geometry, meter, workspace.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tess.h"
#include "kernels/gemm.h"

namespace tess {

// Exception carrying a tess_status; the C-ABI converts it at the boundary.
// Mirrors the reference taxonomy (proj/include/tsim/error.hpp:11-48).
class Error : public std::runtime_error {
 public:
  Error(tess_status s, const std::string& m) : std::runtime_error(m), status(s) {}
  tess_status status;
};

[[noreturn]] inline void fail(tess_status s, const std::string& m) { throw Error(s, m); }

#define TESS_CUDA(expr)                                                              \
  do {                                                                               \
    cudaError_t e_ = (expr);                                                         \
    if (e_ != cudaSuccess)                                                           \
      ::tess::fail(TESS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_) + \
                                      " (" + ::tess::gemm_last_error() + ")");       \
  } while (0)

// Counts every kernel this library launches (tess_kernel_launches).
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

enum Family { ROW = 0, COL = 1, DEPTH = 2 };

// Launch profiling (CUDA events around every local GEMM / attention launch
// while enabled; tess_profile_*).
struct ProfToken {
  void* rec = nullptr;
};
ProfToken prof_begin(const std::string& kernel, double flops, cudaStream_t s, double bytes = 0);
void prof_end(ProfToken& t, cudaStream_t s);
// Profiles one memory-bound launch (its compulsory HBM bytes) for the scope.
struct ProfMem {
  ProfToken tok;
  cudaStream_t s;
  ProfMem(const char* kernel, double bytes, cudaStream_t st) : s(st) {
    tok = prof_begin(kernel, 0, st, bytes);
  }
  ~ProfMem() {
    try {
      prof_end(tok, s);
    } catch (...) {
    }
  }
};
bool prof_detail();
void profile_enable(int mode);  // 0 off, 1 per instantiation, 2 + shape/epilogue
void profile_read(double* ms, double* flops, uint64_t* launches);
std::string profile_json();

struct Coord {
  int i = 0, j = 0, k = 0;
};

// GridSpec semantics of proj/src/grid.cpp:26-131.
struct Grid {
  int q = 1, d = 1;
  Grid() = default;
  Grid(int q_, int d_, bool allow);
  int size() const { return d * q * q; }
  bool valid(const Coord& c) const {
    return c.i >= 0 && c.i < q && c.j >= 0 && c.j < q && c.k >= 0 && c.k < d;
  }
  int rank_of(const Coord& c) const;
  Coord coord_of(int rank) const;
  int block_row(const Coord& c) const { return c.i + c.k * q; }
  int group_size(Family f) const { return f == DEPTH ? d : q; }
  int group_count(Family f) const { return f == DEPTH ? q * q : q * d; }
  int group_index(const Coord& c, Family f) const {
    return f == ROW ? c.k * q + c.i : f == COL ? c.k * q + c.j : c.i * q + c.j;
  }
  int slot_in_group(const Coord& c, Family f) const {
    return f == ROW ? c.j : f == COL ? c.i : c.k;
  }
  Coord member_at(Family f, int gi, int slot) const;
  std::string str() const {
    return "[" + std::to_string(q) + "," + std::to_string(q) + "," + std::to_string(d) + "]";
  }
};

Grid parse_grid(const std::string& text, bool allow);

// Flat CommStats meter for one rank (runtime.hpp:24-69 counting rules).
struct Meter {
  uint64_t sent_msgs = 0, sent_elems = 0, recv_msgs = 0, recv_elems = 0;
  uint64_t kind[5][2] = {};
  void bcast(int gsize, int slot, int root, uint64_t n) {
    if (gsize <= 1) return;
    if (slot == root) {
      sent_msgs += gsize - 1;
      sent_elems += uint64_t(gsize - 1) * n;
      kind[0][0] += gsize - 1;
      kind[0][1] += uint64_t(gsize - 1) * n;
    } else {
      recv_msgs += 1;
      recv_elems += n;
    }
  }
  void reduce(int gsize, int slot, int root, uint64_t n, bool all) {
    if (gsize <= 1) return;
    const int k = all ? 2 : 1;
    const int rt = all ? 0 : root;
    if (slot == rt) {
      recv_msgs += gsize - 1;
      recv_elems += uint64_t(gsize - 1) * n;
      if (all) {
        sent_msgs += gsize - 1;
        sent_elems += uint64_t(gsize - 1) * n;
        kind[k][0] += gsize - 1;
        kind[k][1] += uint64_t(gsize - 1) * n;
      }
    } else {
      sent_msgs += 1;
      sent_elems += n;
      kind[k][0] += 1;
      kind[k][1] += n;
      if (all) {
        recv_msgs += 1;
        recv_elems += n;
      }
    }
  }
};

struct TraceEvent {
  int rank;
  uint64_t step;
  int kind;
  int group;
  int root;
  uint64_t bytes;
};

// write_trace() text of a trace ("<rank>:<step> <kind> <group> <root>
// <bytes>" per line, runtime.cpp:90-96).
std::string trace_text(const std::vector<TraceEvent>& trace);

// Device workspace: named, grow-only buffers owned by a context.
class Workspace {
 public:
  explicit Workspace(int device) : device_(device) {}
  ~Workspace();
  void* get(const std::string& name, size_t bytes);
  void release_all();
  size_t bytes_held() const;

 private:
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  int device_;
  std::map<std::string, Buf> bufs_;
};

}  // namespace tess
