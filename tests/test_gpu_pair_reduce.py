"""Pair reduce fused into the owner GEMM (csrc/summa.cpp, use_pair_reduce).

On q == 2 grids the NT row reduce and the TN column reduce (reference
algorithms.cpp:55-56, 69-70) move no data through a collective: each rank
computes its contribution first, then its own partial with a Resid epilogue
that reads the partner's contribution from peer memory. Checked here:
  * bitwise equality with the collective path (TESS_PAIR_REDUCE=0, run in a
    subprocess because the switch is read once per process) for NT / TN
    products, the dense backward and a bf16 transformer block at [2,2,1] and
    [2,2,2] — the two-member sum is order-free, so nothing may differ;
  * identical CommStats (the fused reduces are metered like the reference's);
  * fewer kernel launches (no separate sum kernels), i.e. the fused path ran.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
import paper_2105_14500_b200 as tess
orc = oracle.Oracle()
out = {}
for q, d in ((2, 1), (2, 2)):
    g = tess.GridSpec(q, d)
    m, n, r = 256 * q * d, 192 * q, 128 * q
    a = orc.random_matrix(m, n, 31, 0)
    for dt in ("f32", "bf16"):
        for v, bs in (("nt", (r, n)), ("tn", (m, r))):
            b = orc.random_matrix(*bs, 31, 1)
            l0 = tess.kernel_launches()
            res = tess.tesseract_matmul(a, b, g, v, dtype=dt)
            key = f"{q}{d}_{dt}_{v}"
            out[key] = res.value
            out[key + "_launches"] = np.array(tess.kernel_launches() - l0)
            out[key + "_sr"] = res.stats.per_rank.astype(np.int64)
            out[key + "_sk"] = res.stats.per_kind.astype(np.int64)
        k = 64 * q
        aa = orc.random_matrix(m, k, 32, 0)
        bb = orc.random_matrix(k, r, 32, 1)
        dc = orc.random_matrix(m, r, 32, 2)
        bw = tess.tesseract_backward_dense(dc, aa, bb, g, dtype=dt)
        out[f"{q}{d}_{dt}_bwd_da"] = bw.a_grad
        out[f"{q}{d}_{dt}_bwd_db"] = bw.b_grad
    b_, s_, h_, nh = 2 * d, 128, 256, 4
    x = orc.random_matrix(b_ * s_, h_, 33, 0)
    dy = orc.random_matrix(b_ * s_, h_, 33, 2)
    P = orc.random_block_params(h_, 33, 100)
    lr = tess.layer_run("block", x, dy, P, tess.LayerDims(b_, s_, h_, nh), g, dtype="bf16")
    out[f"{q}{d}_block_y"] = lr.y
    out[f"{q}{d}_block_dx"] = lr.dx
    for kname, v in lr.grads.items():
        out[f"{q}{d}_block_g_{kname}"] = v
    out[f"{q}{d}_block_sk"] = lr.stats.per_kind.astype(np.int64)
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, pair):
    path = str(tmp_path / f"pair{pair}.npz")
    env = dict(os.environ, TESS_PAIR_REDUCE=str(pair))
    subprocess.run([sys.executable, "-c", WORKER, ROOT, path], check=True, env=env, timeout=600)
    return np.load(path)


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    tmp = tmp_path_factory.mktemp("pair")
    return _run(tmp, 1), _run(tmp, 0)


def test_pair_reduce_bitwise_equals_collective_path(runs):
    fused, coll = runs
    assert set(fused.files) == set(coll.files)
    for k in fused.files:
        if k.endswith("_launches"):
            continue
        assert np.array_equal(fused[k], coll[k]), k


def test_pair_reduce_skips_sum_kernels(runs):
    fused, coll = runs
    for k in fused.files:
        if k.endswith("_launches"):
            assert int(fused[k]) < int(coll[k]), (k, int(fused[k]), int(coll[k]))
