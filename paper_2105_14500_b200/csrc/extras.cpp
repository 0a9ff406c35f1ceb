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

// ---------------------------------------------------------------------------
// Self-tests of the SM-free panel transport (summa.cpp, peer.h PanelLink).
namespace {

// bf16 [rows, cols] panel filled with a pattern depending on `base`.
void fill_panel(void* dst, float* tmp, int64_t rows, int64_t cols, float base, cudaStream_t s) {
  const size_t n = (size_t)(rows * cols);
  k_peer_fill(tmp, n, base, s);
  // scale into a bf16-friendly range: pattern values (base + i % 4093) * 2^-12
  k_convert(tmp, DType::F32, dst, DType::BF16, n, s);
}

GemmDesc nn_desc(const void* a0, const void* a1, const void* b0, const void* b1, int64_t M,
                 int64_t K, int64_t N, float* c) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.nseg = 2;
  g.seg[0] = {a0, b0, K};
  g.seg[1] = {a1, b1, K};
  g.lda = K;
  g.ldb = N;
  g.in = DType::BF16;
  g.c = c;
  g.c_type = DType::F32;
  g.ldc = N;
  g.alpha = 1.0f / 4096.0f / 4096.0f;
  return g;
}

}  // namespace

// One process: a two-segment tcgen05 GEMM launched while its second A panel
// is not there yet; the panel arrives `delay_ms` later from pinned host
// memory (copy engine) in `chunks` row chunks, each followed by a stream
// memory write of its flag. The result must equal (bitwise) the same GEMM
// run on resident panels. *bad = mismatching outputs; *ms_wait = device time
// of the flagged GEMM's stream from launch to completion.
extern "C" tess_status tess_debug_gemm_ready(int64_t M, int64_t K, int64_t N, int chunks,
                                             int delay_ms, unsigned long long* bad,
                                             float* ms_wait) {
  return guarded([&] {
    if (M <= 0 || K <= 0 || N <= 0 || chunks < 1 || chunks > 16 || !bad)
      fail(TESS_ERR_INVALID, "tess_debug_gemm_ready: bad arguments");
    cudaStream_t s, s2;
    TESS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    TESS_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    const size_t na = (size_t)(M * K), nb = (size_t)(K * N), nc = (size_t)(M * N);
    void *a0, *a1, *a1r, *b0, *b1;
    float *tmp, *c, *cref;
    uint32_t* flags;
    unsigned long long* dbad;
    TESS_CUDA(cudaMalloc(&a0, na * 2));
    TESS_CUDA(cudaMalloc(&a1, na * 2));
    TESS_CUDA(cudaMalloc(&a1r, na * 2));
    TESS_CUDA(cudaMalloc(&b0, nb * 2));
    TESS_CUDA(cudaMalloc(&b1, nb * 2));
    TESS_CUDA(cudaMalloc(&tmp, std::max(na, nb) * 4));
    TESS_CUDA(cudaMalloc(&c, nc * 4));
    TESS_CUDA(cudaMalloc(&cref, nc * 4));
    TESS_CUDA(cudaMalloc(&flags, 64 * 4));
    TESS_CUDA(cudaMalloc(&dbad, 8));
    TESS_CUDA(cudaMemset(flags, 0, 64 * 4));
    TESS_CUDA(cudaMemset(dbad, 0, 8));
    fill_panel(a0, tmp, M, K, 11.f, s);
    fill_panel(a1r, tmp, M, K, 3001.f, s);
    fill_panel(b0, tmp, K, N, 17.f, s);
    fill_panel(b1, tmp, K, N, 29.f, s);
    TESS_CUDA(cudaMemsetAsync(a1, 0xff, na * 2, s));  // NaN garbage until the panel lands
    void* host = nullptr;
    TESS_CUDA(cudaMallocHost(&host, na * 2));
    TESS_CUDA(cudaMemcpyAsync(host, a1r, na * 2, cudaMemcpyDeviceToHost, s));
    // reference: both panels resident
    TESS_CUDA(cudaStreamSynchronize(s));
    if (gemm(nn_desc(a0, a1r, b0, b1, M, K, N, cref), s) != cudaSuccess)
      fail(TESS_ERR_CUDA, gemm_last_error());
    TESS_CUDA(cudaStreamSynchronize(s));
    // flagged GEMM first, panel afterwards
    int64_t cr = (M + chunks - 1) / chunks;
    cr = ((cr + 255) / 256) * 256;
    const int n_ch = (int)((M + cr - 1) / cr);
    GemmDesc g = nn_desc(a0, a1, b0, b1, M, K, N, c);
    g.ready.a_flags[1] = flags;
    g.ready.a_epoch[1] = 1;
    g.ready.chunks = n_ch;
    g.ready.chunk_rows = cr;
    cudaEvent_t e0, e1;
    TESS_CUDA(cudaEventCreate(&e0));
    TESS_CUDA(cudaEventCreate(&e1));
    TESS_CUDA(cudaEventRecord(e0, s));
    if (gemm(g, s) != cudaSuccess) fail(TESS_ERR_CUDA, gemm_last_error());
    TESS_CUDA(cudaEventRecord(e1, s));
    std::this_thread::sleep_for(std::chrono::milliseconds(delay_ms));
    for (int ch = 0; ch < n_ch; ++ch) {
      const int64_t r0 = ch * cr, r1 = std::min<int64_t>(M, r0 + cr);
      TESS_CUDA(cudaMemcpyAsync(static_cast<char*>(a1) + r0 * K * 2,
                                static_cast<char*>(host) + r0 * K * 2, (r1 - r0) * K * 2,
                                cudaMemcpyHostToDevice, s2));
      stream_write_u32(s2, flags + ch, 1);
    }
    TESS_CUDA(cudaStreamSynchronize(s));
    TESS_CUDA(cudaStreamSynchronize(s2));
    if (ms_wait) TESS_CUDA(cudaEventElapsedTime(ms_wait, e0, e1));
    k_count_mismatch(c, cref, nc, dbad, s);
    TESS_CUDA(cudaMemcpyAsync(bad, dbad, 8, cudaMemcpyDeviceToHost, s));
    TESS_CUDA(cudaStreamSynchronize(s));
    for (void* p : {a0, a1, a1r, b0, b1, (void*)tmp, (void*)c, (void*)cref, (void*)flags,
                    (void*)dbad})
      cudaFree(p);
    cudaFreeHost(host);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    cudaStreamDestroy(s2);
  });
}

// Two PROCESSES on one GPU (handles swapped through files in `dir`): rank 0
// (root) pushes a bf16 [M, K] panel through a PanelLink `iters` times, each
// push `delay_ms` after the receiver (rank 1) has already launched the GEMM
// that consumes it (segment 1 of a two-segment NN, waiting on the link's
// ready flags chunk by chunk). The receiver checks every result bitwise
// against the same GEMM over its own copy of the panel and releases the
// link (done); the panel doubles half-way through (window regrowth).
extern "C" tess_status tess_debug_panel_link(int rank, const char* dir, int64_t M, int64_t K,
                                             int64_t N, int iters, int chunks, int delay_ms,
                                             unsigned long long* bad) {
  return guarded([&] {
    if ((rank != 0 && rank != 1) || !dir || !bad || M <= 0 || K <= 0 || N <= 0 || iters <= 0 ||
        chunks < 1 || chunks > 16)
      fail(TESS_ERR_INVALID, "tess_debug_panel_link: bad arguments");
    if (!memops_available()) fail(TESS_ERR_CUDA, "stream memory operations unavailable");
    int gen = 0;
    const std::string d(dir);
    PanelLink link(
        [&](const void* mine, void* theirs, size_t bytes) {
          const std::string me = d + "/pl." + std::to_string(rank) + "." + std::to_string(gen);
          const std::string other =
              d + "/pl." + std::to_string(1 - rank) + "." + std::to_string(gen);
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
              fail(TESS_ERR_SPMD, "panel link self-test: partner did not publish " + other);
            std::this_thread::sleep_for(std::chrono::milliseconds(5));
          }
        },
        rank == 1);
    cudaStream_t s;
    TESS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int64_t Mmax = 2 * M;
    const size_t namax = (size_t)(Mmax * K), nb = (size_t)(K * N), ncmax = (size_t)(Mmax * N);
    void *a0, *a1, *b0, *b1;
    float *tmp, *c, *cref;
    unsigned long long* dbad;
    TESS_CUDA(cudaMalloc(&a0, namax * 2));
    TESS_CUDA(cudaMalloc(&a1, namax * 2));
    TESS_CUDA(cudaMalloc(&b0, nb * 2));
    TESS_CUDA(cudaMalloc(&b1, nb * 2));
    TESS_CUDA(cudaMalloc(&tmp, std::max(namax, nb) * 4));
    TESS_CUDA(cudaMalloc(&c, ncmax * 4));
    TESS_CUDA(cudaMalloc(&cref, ncmax * 4));
    TESS_CUDA(cudaMalloc(&dbad, 8));
    TESS_CUDA(cudaMemset(dbad, 0, 8));
    fill_panel(b0, tmp, K, N, 17.f, s);
    fill_panel(b1, tmp, K, N, 29.f, s);
    for (int it = 0; it < iters; ++it) {
      const int64_t m = it >= iters / 2 ? Mmax : M;
      const size_t bytes = (size_t)(m * K) * 2;
      int64_t cr = (m + chunks - 1) / chunks;
      cr = ((cr + 255) / 256) * 256;
      // both sides know the panel of round `it`: the root sends it, the
      // receiver keeps its own copy for the reference GEMM
      fill_panel(a1, tmp, m, K, 1000.f + 37.f * it, s);
      TESS_CUDA(cudaStreamSynchronize(s));
      if (rank == 0) {
        std::this_thread::sleep_for(std::chrono::milliseconds(delay_ms));
        link.push(a1, bytes, (size_t)(cr * K) * 2, s);
        TESS_CUDA(cudaStreamSynchronize(s));
        continue;
      }
      fill_panel(a0, tmp, m, K, 5.f + it, s);
      const uint32_t e = link.push(nullptr, bytes, (size_t)(cr * K) * 2, s);
      GemmDesc g = nn_desc(a0, link.data(), b0, b1, m, K, N, c);
      g.ready.a_flags[1] = link.ready_flags();
      g.ready.a_epoch[1] = e;
      g.ready.chunks = (int)((m + cr - 1) / cr);
      g.ready.chunk_rows = cr;
      if (gemm(g, s) != cudaSuccess) fail(TESS_ERR_CUDA, gemm_last_error());
      link.done(s);
      if (gemm(nn_desc(a0, a1, b0, b1, m, K, N, cref), s) != cudaSuccess)
        fail(TESS_ERR_CUDA, gemm_last_error());
      k_count_mismatch(c, cref, (size_t)(m * N), dbad, s);
      TESS_CUDA(cudaStreamSynchronize(s));
    }
    TESS_CUDA(cudaMemcpy(bad, dbad, 8, cudaMemcpyDeviceToHost));
    for (void* p : {a0, a1, b0, b1, (void*)tmp, (void*)c, (void*)cref, (void*)dbad}) cudaFree(p);
    cudaStreamDestroy(s);
  });
}
