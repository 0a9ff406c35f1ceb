"""Failure semantics of the runtime (reference runtime.cpp:422-471, 540-553;
verify.cpp:84-86 inject_fault), exercised through fault injection:

  * a perturbed result (element (0,0) += 1e-3, the reference's injected
    fault) is caught by the parity check it would slip past otherwise;
  * a rank that fails aborts every partner, and the call raises SpmdError
    naming the failing coordinate (not a hang, not a partner's error);
  * a rank that silently skips a collective and finishes leaves its partner
    blocked: the in-process backend reports the deadlock at once, naming
    every divergent rank and the collective it waits on (instead of a
    600 s timeout);
  * after any of these the next call on the same thread works.
"""
import time

import numpy as np
import pytest

from test_gpu_parity import f32r, rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


def _ab(orc, n=256):
    return f32r(orc.random_matrix(n, n, 42, 0)), f32r(orc.random_matrix(n, n, 42, 1))


def test_perturb_is_caught(tess, orc):
    a, b = _ab(orc)
    want, _, _ = orc.tesseract_matmul(a, b, 2, 2, "nn")
    grid = tess.GridSpec(2, 2)
    clean = tess.tesseract_matmul(a, b, grid, "nn", dtype="f32").value
    assert rel_diff(clean, want) <= 1e-5
    tess.set_global_fault("perturb")
    bad = tess.tesseract_matmul(a, b, grid, "nn", dtype="f32").value
    assert rel_diff(bad, want) > 1e-5
    assert abs(bad[0, 0] - clean[0, 0] - 1e-3) < 1e-9
    again = tess.tesseract_matmul(a, b, grid, "nn", dtype="f32").value  # one-shot
    assert np.array_equal(again, clean)


@pytest.mark.parametrize("rank,at", [(3, 0), (0, 2), (5, 1)])
def test_rank_failure_aborts_all(tess, orc, rank, at):
    a, b = _ab(orc)
    grid = tess.GridSpec(2, 2)
    c = grid.coord_of(rank)
    tess.set_global_fault("rank_fail", rank, at)
    t0 = time.time()
    with pytest.raises(tess.SpmdError) as ei:
        tess.tesseract_matmul(a, b, grid, "nn", dtype="f32")
    assert time.time() - t0 < 60
    msg = str(ei.value)
    assert f"rank ({c.i},{c.j},{c.k}) failed" in msg and "injected failure" in msg, msg
    ok = tess.tesseract_matmul(a, b, grid, "nn", dtype="f32")
    want, _, _ = orc.tesseract_matmul(a, b, 2, 2, "nn")
    assert rel_diff(ok.value, want) <= 1e-5


def test_skipped_collective_reports_deadlock(tess, orc):
    """NN at [2,2,1]: each rank makes 4 broadcasts (row t=0, col t=0, row
    t=1, col t=1). Rank 1 = (0,1,0) skips its last (the column broadcast
    from slot 1, i.e. from its column partner (1,1,0)) and finishes; the
    root (1,1,0) blocks on it while everyone else finishes -> deadlock
    naming (1,1,0)."""
    a, b = _ab(orc)
    grid = tess.GridSpec(2, 1)
    tess.set_global_fault("skip_collective", 1, 3)
    t0 = time.time()
    with pytest.raises(tess.SpmdError) as ei:
        tess.tesseract_matmul(a, b, grid, "nn", dtype="f32")
    assert time.time() - t0 < 60
    msg = str(ei.value)
    assert "deadlock: mismatched participation" in msg, msg
    assert "(1,1,0) waits on broadcast" in msg and "column group" in msg, msg
    assert "already finished" in msg, msg
    ok = tess.tesseract_matmul(a, b, grid, "nn", dtype="f32")
    want, _, _ = orc.tesseract_matmul(a, b, 2, 1, "nn")
    assert rel_diff(ok.value, want) <= 1e-5


def test_skipped_collective_mismatch(tess, orc):
    """A rank that skips a collective in the middle meets its partner at
    the wrong collective: the signature check fails the run (SpmdError)."""
    a, b = _ab(orc)
    grid = tess.GridSpec(2, 2)
    tess.set_global_fault("skip_collective", 2, 0)
    with pytest.raises(tess.SpmdError):
        tess.tesseract_matmul(a, b, grid, "nn", dtype="f32")
