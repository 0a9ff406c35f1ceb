"""1-D tensor-parallel (Megatron) layer scheme -- BASELINE config 5's
comparator, built from the reference's megatron_1d_linear (algorithms.cpp:
244-265: Column1D / Row1D split, depth all-reduce of the partials) applied
to the whole block. The scheme computes the same function as the reference
block (layers.cpp:460-487), so it is checked against the fp64 oracle's
ref::* layers at the tolerances of test_gpu_parity.py, for p = 1, 2, 4 ranks
(in-process, one GPU), plus the collective count it adds.
"""
import numpy as np
import pytest

from test_gpu_parity import _compare_layer, _layer_inputs, bf16r, f32r, frob, rel_diff

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tess():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2105_14500_b200 as t
    return t


@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("op", ["feedforward", "attention", "layernorm", "block"])
def test_megatron_layers_fp32(tess, orc, p, op):
    b, s, h, nh = 2, 8, 32, 4
    x, dy, P = _layer_inputs(orc, b, s, h, 19, f32r)
    want = orc.layer_run(op, x, dy, P, b, s, nh)
    res = tess.megatron_layer_run(op, x, dy, P, tess.LayerDims(b, s, h, nh), p, dtype="f32")
    _compare_layer(res, want, 1e-5, rel_diff)


@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("op", ["feedforward", "attention", "block"])
def test_megatron_layers_bf16(tess, orc, p, op):
    # head_dim 64: the fused tcgen05 attention kernels serve the local heads
    b, s, h, nh = 2, 128, 256, 4
    x, dy, P = _layer_inputs(orc, b, s, h, 20, bf16r)
    want = orc.layer_run(op, x, dy, P, b, s, nh)
    res = tess.megatron_layer_run(op, x, dy, P, tess.LayerDims(b, s, h, nh), p, dtype="bf16")
    _compare_layer(res, want, 2e-2, frob)


def test_megatron_block_collectives(tess, orc):
    """Two all-reduces of [T, h] per forward (proj, FF2) and two per backward
    (QKV, FF1 dgrads) on each rank of the line; nothing else moves."""
    b, s, h, nh, p = 2, 8, 32, 4, 2
    x, dy, P = _layer_inputs(orc, b, s, h, 21, f32r)
    r2 = tess.megatron_layer_run("block", x, dy, P, tess.LayerDims(b, s, h, nh), p, dtype="f32")
    r1 = tess.megatron_layer_run("block", x, dy, P, tess.LayerDims(b, s, h, nh), 1, dtype="f32")
    k2 = np.asarray(r2.stats.per_kind, dtype=np.int64)
    k1 = np.asarray(r1.stats.per_kind, dtype=np.int64)
    # the extra traffic of p = 2 over p = 1 is all all-reduce (kind 2)
    extra = k2 - k1
    assert extra[0].sum() == 0 and extra[1].sum() == 0, (k1, k2)
    assert extra[2, 1] > 0 and extra[2, 1] % (b * s * h) == 0, (k1, k2)
