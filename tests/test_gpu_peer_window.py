"""Peer-window transport of the NCCL backend's fused pair reduce (csrc/peer.h).

Two processes on cuda:0 (CUDA IPC works between processes on one GPU; NCCL
does not, so the handle swap goes through files here) run acquire / fill /
open / check / close rounds, growing the window half-way: every element the
partner published must be read back exactly, and the release/acquire
sequence words must order the rounds (a stale or early read would show up as
a pattern mismatch).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import ctypes as C, sys
sys.path.insert(0, sys.argv[1])
import paper_2105_14500_b200 as tess
bad = C.c_ulonglong(0)
f = tess.lib.tess_debug_peer_window
f.argtypes = [C.c_int, C.c_char_p, C.c_size_t, C.c_int, C.POINTER(C.c_ulonglong)]
f.restype = C.c_int
st = f(int(sys.argv[2]), sys.argv[3].encode(), int(sys.argv[4]), int(sys.argv[5]), C.byref(bad))
print(st, bad.value, tess.lib.tess_last_error().decode() if st else "")
sys.exit(0 if st == 0 and bad.value == 0 else 1)
"""


@pytest.mark.parametrize("n,iters", [(1000, 6), (3 << 20, 10)])
def test_peer_window_two_processes(tmp_path, n, iters):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, ROOT, str(r), str(tmp_path), str(n),
                               str(iters)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                              text=True) for r in (0, 1)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            p.kill()
            outs.append(p.communicate()[0])
    assert all(p.returncode == 0 for p in procs), outs
