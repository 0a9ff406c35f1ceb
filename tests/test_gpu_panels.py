"""SM-free SUMMA panel transport (summa.cpp panel_step, peer.h PanelLink):
the GEMM of a SUMMA step is launched before its remote panel lands and waits
on the device, per row chunk, for a flag written by a stream memory
operation after the chunk's copy-engine transfer (GemmReady). This is what
overlaps the row/column broadcasts of the reference's nn/tn_product_rank
(algorithms.cpp:34-45, 61-76) with the local GEMM on a multi-GPU grid, and
why no SMs are set aside for NCCL.

On one GPU both hooks run the real kernels and transport:
  * test_gemm_waits_for_late_panel: the panel arrives from pinned host memory
    50 ms after the GEMM was launched; the result must be bitwise the GEMM
    over resident panels, and the GEMM's own stream time must include the
    wait (it started before the panel landed);
  * test_panel_link_two_processes: rank 0 pushes panels into rank 1's CUDA
    IPC window (copy engine) + flag writes, rank 1's GEMM was launched
    before each push; the window grows half-way (IPC handles re-swapped).
"""
import ctypes as C
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


@pytest.mark.parametrize("M,K,N,chunks", [(2048, 1024, 2048, 8), (1000, 512, 768, 3),
                                          (4096, 256, 512, 16)])
def test_gemm_waits_for_late_panel(tess, M, K, N, chunks):
    f = tess.lib.tess_debug_gemm_ready
    f.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                  C.POINTER(C.c_ulonglong), C.POINTER(C.c_float)]
    f.restype = C.c_int
    bad, ms = C.c_ulonglong(0), C.c_float(0)
    st = f(M, K, N, chunks, 50, C.byref(bad), C.byref(ms))
    assert st == 0, tess.lib.tess_last_error().decode()
    assert bad.value == 0
    # launched ~50 ms before its panel existed: the GEMM's stream span covers the wait
    assert ms.value >= 30.0, ms.value


WORKER = r"""
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
import paper_2105_14500_b200 as tess
bad = C.c_ulonglong(0)
f = tess.lib.tess_debug_panel_link
f.argtypes = [C.c_int, C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
              C.POINTER(C.c_ulonglong)]
f.restype = C.c_int
st = f(int(sys.argv[2]), sys.argv[3].encode(), *[int(v) for v in sys.argv[4:10]], C.byref(bad))
print(st, bad.value, tess.lib.tess_last_error().decode() if st else "")
sys.exit(0 if st == 0 and bad.value == 0 else 1)
"""


@pytest.mark.parametrize("M,K,N,iters,chunks", [(1024, 512, 1024, 6, 4), (768, 256, 512, 4, 1)])
def test_panel_link_two_processes(tess, tmp_path, M, K, N, iters, chunks):
    args = [str(v) for v in (M, K, N, iters, chunks, 30)]
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, ROOT, str(r), str(tmp_path), *args],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in (0, 1)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate()[0])
    assert all(p.returncode == 0 for p in procs), outs
