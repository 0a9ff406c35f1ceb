"""Host side of the fused dropout epilogue (tess_dropout_keep): the C-ABI
mask equals the vectorised restatement the GPU tests use, and drops a
fraction p of the elements. Runs without a GPU (pure host code in libtess)."""
import numpy as np
import pytest


@pytest.mark.parametrize("p", [0.05, 0.1, 0.5, 0.9])
def test_dropout_keep_host(p):
    import paper_2105_14500_b200 as t
    rng = np.random.default_rng(int(p * 100))
    seed = int(rng.integers(0, 2 ** 63))
    r = rng.integers(0, 1 << 40, 300)
    c = rng.integers(0, 1 << 40, 300)
    ref = np.array([t.lib.tess_dropout_keep(seed, int(a), int(b), p) for a, b in zip(r, c)], bool)
    assert np.array_equal(t.dropout_keep(seed, r, c, p), ref)
    rr, cc = np.meshgrid(np.arange(1024), np.arange(1024), indexing="ij")
    frac = 1 - t.dropout_keep(seed, rr, cc, p).mean()
    assert abs(frac - p) < 0.01, frac
    assert t.lib.tess_dropout_keep(seed, 5, 7, 0.0) == 1
