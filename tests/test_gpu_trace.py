"""The per-rank C-ABI emits the reference's collective trace
(`rank:step kind group root bytes`, runtime.cpp:90-96) line for line, checked
against traces written by the unmodified reference (tests/golden/
reference_traces.json, made by tests/golden/make_golden.py --traces)."""
import json
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


def run_ranks(tess, grid, fn):
    ctxs = tess.init_local(grid)
    errs = []

    def body(r):
        try:
            fn(ctxs[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(grid.size())]
    [t.start() for t in th]
    [t.join() for t in th]
    try:
        assert not errs, errs
        return [cx.trace() for cx in ctxs]
    finally:
        for cx in ctxs:
            cx.close()


@pytest.mark.parametrize("q,d,allow", [(2, 1, False), (2, 2, False), (1, 2, True)])
@pytest.mark.parametrize("variant", ["nn", "nt", "tn"])
def test_trace_matches_reference(tess, orc, q, d, allow, variant):
    import torch
    want = json.load(open(os.path.join(HERE, "golden", "reference_traces.json")))[
        f"{variant}_{q}{q}{d}"]
    m, n, r = 4 * q * d, 4 * q, 6 * q
    a = orc.random_matrix(m, n, 14, 0)
    b = {"nn": orc.random_matrix(n, r, 14, 1), "nt": orc.random_matrix(r, n, 14, 1),
         "tn": orc.random_matrix(m, r, 14, 1)}[variant]
    grid = tess.GridSpec(q, d, allow)
    ab = orc.partition(a, q, d, 0)
    bb = orc.partition(b, q, d, 0 if variant == "tn" else 1)

    def prog(cx):
        cx.set_trace(True)
        la = torch.from_numpy(ab[cx.rank].astype(np.float32)).cuda()
        lb = torch.from_numpy(bb[cx.rank].astype(np.float32)).cuda()
        rows = {"nn": la.shape[0], "nt": la.shape[0], "tn": la.shape[1]}[variant]
        cols = {"nn": lb.shape[1], "nt": lb.shape[0], "tn": lb.shape[1]}[variant]
        lc = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
        cx.matmul(variant, "f32", la.data_ptr(), *la.shape, lb.data_ptr(), *lb.shape,
                  lc.data_ptr(), sum_over_depth=variant == "tn")
        torch.cuda.synchronize()

    got = "".join(run_ranks(tess, grid, prog))
    assert got == want
