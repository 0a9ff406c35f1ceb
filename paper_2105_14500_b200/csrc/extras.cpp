// Plumbing from SURVEY 8(f):
//  * FNV-1a fingerprints and TMX1 / CSV matrix files (reference
//    matrix.cpp:244-370) for exchanging golden vectors with the oracle
//    without rerunning it.
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "kernels/kernels.h"
#include "ops.h"

using namespace tess;

namespace tess {
extern thread_local std::string g_last_error;
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
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TESS_ERR_INVALID;
  }
}

uint64_t fnv1a(int64_t rows, int64_t cols, const double* v) {
  uint64_t h = 0xcbf29ce484222325ULL;
  auto feed = [&h](uint64_t w) {
    for (int i = 0; i < 8; ++i) {
      h ^= (w >> (8 * i)) & 0xff;
      h *= 0x100000001b3ULL;
    }
  };
  feed((uint64_t)rows);
  feed((uint64_t)cols);
  for (int64_t i = 0; i < rows * cols; ++i) {
    uint64_t bits;
    std::memcpy(&bits, &v[i], 8);
    feed(bits);
  }
  return h;
}

}  // namespace

extern "C" {

// ref matrix.cpp:352-370
uint64_t tess_checksum(int64_t rows, int64_t cols, const double* values) {
  return fnv1a(rows, cols, values);
}

// ref matrix.cpp:244-350: "TMX1" magic, uint64 LE rows/cols, LE doubles;
// ".csv" paths use shortest round-trip decimal text.
tess_status tess_save_matrix(const char* path, int64_t rows, int64_t cols, const double* v) {
  return guarded([&] {
    const std::string p = path ? path : "";
    const bool csv = p.size() >= 4 && p.substr(p.size() - 4) == ".csv";
    std::ofstream os(p, csv ? std::ios::out : std::ios::out | std::ios::binary);
    if (!os) fail(TESS_ERR_IO, "save_matrix: cannot open " + p);
    if (csv) {
      char buf[32];
      for (int64_t r = 0; r < rows; ++r) {
        for (int64_t c = 0; c < cols; ++c) {
          auto res = std::to_chars(buf, buf + sizeof(buf), v[r * cols + c]);
          if (c) os << ',';
          os.write(buf, res.ptr - buf);
        }
        os << '\n';
      }
    } else {
      os.write("TMX1", 4);
      const uint64_t dims[2] = {(uint64_t)rows, (uint64_t)cols};
      os.write(reinterpret_cast<const char*>(dims), 16);
      os.write(reinterpret_cast<const char*>(v), (std::streamsize)(rows * cols * 8));
    }
    if (!os) fail(TESS_ERR_IO, "save_matrix: write failed for " + p);
  });
}

// Reads the header (rows, cols) when v is NULL, else the values.
tess_status tess_load_matrix(const char* path, int64_t* rows, int64_t* cols, double* v) {
  return guarded([&] {
    const std::string p = path ? path : "";
    const bool csv = p.size() >= 4 && p.substr(p.size() - 4) == ".csv";
    std::ifstream is(p, csv ? std::ios::in : std::ios::in | std::ios::binary);
    if (!is) fail(TESS_ERR_IO, "load_matrix: cannot open " + p);
    if (csv) {
      std::vector<double> vals;
      std::string line;
      int64_t r = 0, c = -1;
      while (std::getline(is, line)) {
        if (line.empty()) continue;
        int64_t n = 0;
        std::stringstream ss(line);
        std::string cell;
        while (std::getline(ss, cell, ',')) {
          double d = 0;
          auto res = std::from_chars(cell.data(), cell.data() + cell.size(), d);
          if (res.ec != std::errc()) fail(TESS_ERR_IO, "load_matrix: bad number in " + p);
          vals.push_back(d);
          ++n;
        }
        if (c >= 0 && n != c) fail(TESS_ERR_IO, "load_matrix: ragged rows in " + p);
        c = n;
        ++r;
      }
      *rows = r;
      *cols = c < 0 ? 0 : c;
      if (v) std::memcpy(v, vals.data(), vals.size() * 8);
    } else {
      char magic[4];
      uint64_t dims[2];
      is.read(magic, 4);
      is.read(reinterpret_cast<char*>(dims), 16);
      if (!is || std::memcmp(magic, "TMX1", 4) != 0)
        fail(TESS_ERR_IO, "load_matrix: not a TMX1 file: " + p);
      *rows = (int64_t)dims[0];
      *cols = (int64_t)dims[1];
      if (v) {
        is.read(reinterpret_cast<char*>(v), (std::streamsize)(dims[0] * dims[1] * 8));
        if (!is) fail(TESS_ERR_IO, "load_matrix: truncated " + p);
      }
    }
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Self-test of the peer window transport (peer.h) between two PROCESSES that
// swap IPC handles through files in `dir` (no NCCL: it refuses two ranks on
// one GPU, CUDA IPC does not). Each of `iters` rounds: acquire, fill our
// window with a rank/round pattern, open, check the partner's, close; the
// window grows half-way through. *bad = mismatching elements seen.
#include <chrono>
#include <cstdio>
#include <thread>

#include "peer.h"

extern "C" tess_status tess_debug_peer_window(int rank, const char* dir, size_t n, int iters,
                                              unsigned long long* bad) {
  return guarded([&] {
    if ((rank != 0 && rank != 1) || !dir || !bad || n == 0 || iters <= 0)
      fail(TESS_ERR_INVALID, "tess_debug_peer_window: bad arguments");
    int gen = 0;
    const std::string d(dir);
    PeerWindow w([&](const void* mine, void* theirs, size_t bytes) {
      const std::string me = d + "/pw." + std::to_string(rank) + "." + std::to_string(gen);
      const std::string other =
          d + "/pw." + std::to_string(1 - rank) + "." + std::to_string(gen);
      ++gen;
      {
        std::ofstream f(me + ".tmp", std::ios::binary);
        f.write(static_cast<const char*>(mine), (std::streamsize)bytes);
      }
      std::rename((me + ".tmp").c_str(), me.c_str());
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        std::ifstream f(other, std::ios::binary);
        if (f && f.read(static_cast<char*>(theirs), (std::streamsize)bytes)) break;
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
          fail(TESS_ERR_SPMD, "peer window self-test: partner did not publish " + other);
        std::this_thread::sleep_for(std::chrono::milliseconds(5));
      }
    });
    cudaStream_t s;
    TESS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    unsigned long long* dbad = nullptr;
    TESS_CUDA(cudaMalloc(&dbad, sizeof(*dbad)));
    TESS_CUDA(cudaMemset(dbad, 0, sizeof(*dbad)));
    for (int it = 0; it < iters; ++it) {
      const size_t m = it >= iters / 2 ? 2 * n : n;
      float* mine = w.acquire(m, s);
      k_peer_fill(mine, m, (float)(rank * 100000 + it * 7), s);
      const float* theirs = w.open(s);
      k_peer_check(theirs, m, (float)((1 - rank) * 100000 + it * 7), dbad, s);
      w.close(s);
    }
    w.drain(s);
    TESS_CUDA(cudaMemcpy(bad, dbad, sizeof(*bad), cudaMemcpyDeviceToHost));
    cudaFree(dbad);
    cudaStreamDestroy(s);
  });
}
