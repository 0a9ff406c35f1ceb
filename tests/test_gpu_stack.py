"""BASELINE config 5's layer stack (tess_stack_run / tess_stack_step): L
Transformer blocks forward then backward under the three schemes the
comparison runs -- Tesseract [q,q,d], SUMMA [q,q,1] and the 1-D (Megatron)
scheme on a [1,1,p] line -- against the fp64 oracle's ref::transformer_block
chained through the stack (reference layers.cpp:460-487; the forward /
backward loops of train_toy, layers.cpp:1006-1026). In-process, one GPU.

Tolerances as test_gpu_parity.py: fp32 rel_diff <= 1e-5, bf16 (activations
between blocks stored in bf16) relative Frobenius <= 2e-2. CommStats of a
Tesseract stack are exactly L times the reference block's.
"""
import numpy as np
import pytest

from test_gpu_parity import bf16r, f32r, frob, rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


def stack_inputs(orc, b, s, h, L, seed, rnd):
    x = rnd(orc.random_matrix(b * s, h, seed, 0))
    dy = rnd(orc.random_matrix(b * s, h, seed, 2))
    Ps = []
    for l in range(L):
        P = orc.random_block_params(h, seed, 100 + l)
        Ps.append({k: (rnd(v) if k.startswith("w_") else f32r(v)) for k, v in P.items()})
    return x, dy, Ps


def oracle_stack(orc, x, dy, Ps, b, s, nh):
    """ref::transformer_block forward through the stack, then its backward
    from the top (each call recomputes its block's forward from the cached
    input, like the reference's layer caches)."""
    xs = [x]
    zero = np.zeros_like(x)
    for P in Ps:
        xs.append(orc.layer_run("block", xs[-1], zero, P, b, s, nh)["y"])
    g = dy
    grads = [None] * len(Ps)
    for l in range(len(Ps) - 1, -1, -1):
        r = orc.layer_run("block", xs[l], g, Ps[l], b, s, nh)
        grads[l] = r["grads"]
        g = r["dx"]
    return xs[-1], g, grads


def compare(res, y, dx, grads, tol, metric):
    errs = {"y": metric(res.y, y), "dx": metric(res.dx, dx)}
    for l, gl in enumerate(grads):
        for k, v in gl.items():
            errs[f"l{l}.{k}"] = metric(res.grads[l][k], v)
    worst = max(errs.values())
    assert worst <= tol, errs
    return worst


CASES = [("tesseract", 1, 1, False), ("tesseract", 1, 2, True), ("summa", 2, 1, False),
         ("tesseract", 2, 2, False), ("megatron", 1, 2, True), ("megatron", 1, 4, True)]


@pytest.mark.parametrize("scheme,q,d,allow", CASES)
def test_stack_fp32(tess, orc, scheme, q, d, allow):
    b, s, h, nh, L = 4, 8, 32, 4, 3
    x, dy, Ps = stack_inputs(orc, b, s, h, L, 31, f32r)
    y, dx, grads = oracle_stack(orc, x, dy, Ps, b, s, nh)
    res = tess.stack_run(scheme, x, dy, Ps, tess.LayerDims(b, s, h, nh),
                         tess.GridSpec(q, d, allow), dtype="f32")
    compare(res, y, dx, grads, 1e-5, rel_diff)


@pytest.mark.parametrize("scheme,q,d,allow", [("tesseract", 2, 2, False),
                                              ("summa", 2, 1, False),
                                              ("megatron", 1, 4, True),
                                              ("tesseract", 1, 1, False)])
def test_stack_bf16(tess, orc, scheme, q, d, allow):
    # head_dim 64: the fused tcgen05 attention kernels run in every block
    b, s, h, nh, L = 4, 128, 256, 4, 2
    x, dy, Ps = stack_inputs(orc, b, s, h, L, 32, bf16r)
    y, dx, grads = oracle_stack(orc, x, dy, Ps, b, s, nh)
    res = tess.stack_run(scheme, x, dy, Ps, tess.LayerDims(b, s, h, nh),
                         tess.GridSpec(q, d, allow), dtype="bf16")
    compare(res, y, dx, grads, 2e-2, frob)


@pytest.mark.parametrize("q,d", [(2, 2), (2, 1), (1, 2)])
def test_stack_comm_stats(tess, orc, q, d):
    """A Tesseract stack meters exactly L reference blocks."""
    b, s, h, nh, L = 4, 8, 32, 4, 3
    x, dy, Ps = stack_inputs(orc, b, s, h, L, 33, f32r)
    res = tess.stack_run("tesseract", x, dy, Ps, tess.LayerDims(b, s, h, nh),
                         tess.GridSpec(q, d, d > q), dtype="f32")
    sr, sk = orc.layer_stats("block", q, d, b, s, h)
    assert (np.asarray(res.stats.per_rank) == L * sr.astype(np.int64)).all()
    assert (np.asarray(res.stats.per_kind) == L * sk.astype(np.int64)).all()


def test_stack_equals_layer_calls(tess, orc):
    """One stack_run of L blocks is bitwise the chain of single-block
    layer_run calls fed with each other's outputs (bf16, [2,2,2])."""
    b, s, h, nh, L = 4, 128, 256, 4, 2
    x, dy, Ps = stack_inputs(orc, b, s, h, L, 34, bf16r)
    dims, grid = tess.LayerDims(b, s, h, nh), tess.GridSpec(2, 2)
    res = tess.stack_run("tesseract", x, dy, Ps, dims, grid, dtype="bf16")
    zero = np.zeros_like(x)
    xs = [x]
    for P in Ps:
        xs.append(tess.layer_run("block", xs[-1], zero, P, dims, grid, dtype="bf16").y)
    g = dy
    for l in range(L - 1, -1, -1):
        r = tess.layer_run("block", xs[l], g, Ps[l], dims, grid, dtype="bf16")
        for k, v in r.grads.items():
            assert np.array_equal(res.grads[l][k], v), (l, k)
        g = r.dx
    assert np.array_equal(res.y, xs[-1])
    assert np.array_equal(res.dx, g)
