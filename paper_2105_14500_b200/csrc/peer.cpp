// PeerWindow (see peer.h).
#include "peer.h"

#include <cstring>

#include "core.h"
#include "kernels/kernels.h"

namespace tess {

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
