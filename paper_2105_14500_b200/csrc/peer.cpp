// PeerWindow (see peer.h).
#include "peer.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "core.h"
#include "kernels/kernels.h"

namespace tess {

namespace {

struct MemOps {
  PFN_cuStreamWriteValue32_v8000 write = nullptr;
  PFN_cuStreamWaitValue32_v8000 wait = nullptr;
};

const MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    void* pw = nullptr;
    void* pv = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &pw, cudaEnableDefault, &q1) ==
            cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &pv, cudaEnableDefault, &q2) ==
            cudaSuccess &&
        q2 == cudaDriverEntryPointSuccess) {
      m.write = reinterpret_cast<PFN_cuStreamWriteValue32_v8000>(pw);
      m.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v8000>(pv);
    }
    cudaGetLastError();
  });
  return m;
}

}  // namespace

bool memops_available() { return memops().write && memops().wait; }

void stream_write_u32(cudaStream_t s, uint32_t* p, uint32_t v) {
  if (!memops_available()) fail(TESS_ERR_CUDA, "stream memory operations unavailable");
  const CUresult r = memops().write(reinterpret_cast<CUstream>(s),
                                    reinterpret_cast<CUdeviceptr>(p), v,
                                    CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) fail(TESS_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
}

void stream_wait_u32_geq(cudaStream_t s, const uint32_t* p, uint32_t v) {
  if (!memops_available()) fail(TESS_ERR_CUDA, "stream memory operations unavailable");
  const CUresult r = memops().wait(reinterpret_cast<CUstream>(s),
                                   reinterpret_cast<CUdeviceptr>(const_cast<uint32_t*>(p)), v,
                                   CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) fail(TESS_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
}

// ---------------------------------------------------------------- PanelLink
PanelLink::~PanelLink() {
  if (peer_) cudaIpcCloseMemHandle(peer_);
  if (base_) cudaFree(base_);
}

void PanelLink::grow(size_t bytes) {
  // Both members drained (the exchange synchronises the device) before the
  // old windows go away; the new headers start at zero, so do the epochs.
  TESS_CUDA(cudaDeviceSynchronize());
  if (peer_) {
    TESS_CUDA(cudaIpcCloseMemHandle(peer_));
    peer_ = nullptr;
  }
  void* nb = nullptr;
  const size_t own = kHeader + (receiver_ ? bytes : 0);
  TESS_CUDA(cudaMalloc(&nb, own));
  TESS_CUDA(cudaMemset(nb, 0, kHeader));
  TESS_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t mine, theirs;
  TESS_CUDA(cudaIpcGetMemHandle(&mine, nb));
  ex_(&mine, &theirs, sizeof(mine));
  if (base_) TESS_CUDA(cudaFree(base_));
  base_ = nb;
  cap_ = bytes;
  epoch_ = 0;
  const cudaError_t e = cudaIpcOpenMemHandle(&peer_, theirs, cudaIpcMemLazyEnablePeerAccess);
  const unsigned char ok = e == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    peer_ = nullptr;
  }
  unsigned char ok_theirs = 0;
  ex_(&ok, &ok_theirs, 1);
  if (!ok || !ok_theirs) fail(TESS_ERR_CUDA, "panel link: cannot map the partner's window");
}

uint32_t PanelLink::push(const void* src, size_t bytes, size_t chunk_bytes, cudaStream_t s) {
  if (!base_ || bytes > cap_) grow(bytes);
  const uint32_t e = ++epoch_;
  if (receiver_ || !bytes) return e;
  if (!chunk_bytes || chunk_bytes > bytes) chunk_bytes = bytes;
  const size_t n = (bytes + chunk_bytes - 1) / chunk_bytes;
  if (n > (size_t)kMaxChunks) fail(TESS_ERR_INVALID, "panel link: too many chunks");
  // the receiver finished reading the previous panel of this link
  if (e > 1) stream_wait_u32_geq(s, static_cast<const uint32_t*>(base_) + 32, e - 1);
  uint32_t* ready = static_cast<uint32_t*>(peer_);
  char* dst = static_cast<char*>(peer_) + kHeader;
  for (size_t c = 0; c < n; ++c) {
    const size_t off = c * chunk_bytes, len = std::min(chunk_bytes, bytes - off);
    TESS_CUDA(cudaMemcpyAsync(dst + off, static_cast<const char*>(src) + off, len,
                              cudaMemcpyDeviceToDevice, s));
    stream_write_u32(s, ready + c, e);
  }
  return e;
}

void PanelLink::done(cudaStream_t s) {
  if (!receiver_ || !peer_) return;
  stream_write_u32(s, static_cast<uint32_t*>(peer_) + 32, epoch_);
}

const void* PanelLink::data() const {
  return receiver_ && base_ ? static_cast<const char*>(base_) + kHeader : nullptr;
}

const uint32_t* PanelLink::ready_flags() const {
  return receiver_ ? static_cast<const uint32_t*>(base_) : nullptr;
}

PeerWindow::~PeerWindow() {
  if (peer_) cudaIpcCloseMemHandle(peer_);
  if (base_) cudaFree(base_);
}

bool PeerWindow::grow(size_t n, cudaStream_t s) {
  // Nothing of ours may still touch the old windows: our own reads of the
  // partner's window and the partner's reads of ours (done >= epoch).
  if (base_) k_peer_wait(&flags(base_)[1], epoch_, s);
  TESS_CUDA(cudaStreamSynchronize(s));
  if (peer_) {
    TESS_CUDA(cudaIpcCloseMemHandle(peer_));
    peer_ = nullptr;
  }
  void* nb = nullptr;
  TESS_CUDA(cudaMalloc(&nb, kHeader + n * 4));
  TESS_CUDA(cudaMemset(nb, 0, kHeader));
  TESS_CUDA(cudaDeviceSynchronize());
  cudaIpcMemHandle_t mine, theirs;
  TESS_CUDA(cudaIpcGetMemHandle(&mine, nb));
  // After the swap the partner has closed its mapping of our old window too.
  ex_(&mine, &theirs, sizeof(mine));
  if (base_) TESS_CUDA(cudaFree(base_));
  base_ = nb;
  cap_ = n;
  epoch_ = 0;
  const cudaError_t e = cudaIpcOpenMemHandle(&peer_, theirs, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    peer_ = nullptr;
  }
  // both members must agree before anyone relies on the mapping
  const unsigned char ok = peer_ != nullptr;
  unsigned char ok_theirs = 0;
  ex_(&ok, &ok_theirs, 1);
  if (ok && ok_theirs) return true;
  if (peer_) cudaIpcCloseMemHandle(peer_);
  peer_ = nullptr;
  return false;
}

bool PeerWindow::probe(cudaStream_t s) { return grow(1024, s); }

float* PeerWindow::acquire(size_t n, cudaStream_t s) {
  if (opened_) fail(TESS_ERR_SPMD, "peer window: acquire while open");
  if ((!base_ || n > cap_) && !grow(n, s))
    fail(TESS_ERR_CUDA, "peer window: cannot map the partner's window");
  // the partner finished reading what we published last time
  if (epoch_) k_peer_wait(&flags(base_)[1], epoch_, s);
  return data(base_);
}

const float* PeerWindow::open(cudaStream_t s) {
  if (!base_ || opened_) fail(TESS_ERR_SPMD, "peer window: open without acquire");
  opened_ = true;
  k_peer_signal(&flags(peer_)[0], epoch_ + 1, s);  // our contribution is ready
  k_peer_wait(&flags(base_)[0], epoch_ + 1, s);    // the partner's is
  return data(peer_);
}

void PeerWindow::close(cudaStream_t s) {
  if (!opened_) fail(TESS_ERR_SPMD, "peer window: close without open");
  opened_ = false;
  k_peer_signal(&flags(peer_)[1], epoch_ + 1, s);  // done reading the partner's window
  ++epoch_;
}

void PeerWindow::drain(cudaStream_t s) {
  if (!base_) return;
  if (epoch_) k_peer_wait(&flags(base_)[1], epoch_, s);
  TESS_CUDA(cudaStreamSynchronize(s));
}

}  // namespace tess
