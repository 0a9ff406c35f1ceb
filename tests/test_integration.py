"""The reference-side drop-in (integration/tsim_b200.{hpp,cpp}): the adapter a
maintainer adds to tesseract-sim, built together with the reference's own
translation units (integration/Makefile) and linked with libtess.so.

Through it, the reference's operators and their B200 replacements run on the
same tsim::Matrix inputs and are compared in the reference's own terms:
values (fp32 mode: the reference's rel_diff <= 1e-5; bf16: relative
Frobenius <= 1e-4 per product on the same fp64 inputs is not reachable, so
bf16 is held to the App. C 5e-3 / 2e-2 layer bounds), CommStats with the
reference's operator== (rebuilt from the library's per-rank, per-kind
counters via add_send / add_recv, runtime.hpp:56-59), traces with
write_trace text equality, and SPEC.md:637's degeneracy criterion.
"""
import ctypes as C
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "integration", "_build", "libtsim_b200_check.so")

ADAPTER_SYMBOLS = ["tesseract_matmul", "tesseract_backward_dense", "summa_matmul",
                   "megatron_1d_linear", "layer_run"]


def _built():
    if not os.path.exists(SO):
        pytest.skip("integration/_build not built (needs the reference sources: make -C "
                    "integration)")


def test_adapter_library_exports():
    _built()
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", SO], capture_output=True,
                         text=True).stdout
    for name in ADAPTER_SYMBOLS:
        assert f"tsim::b200::{name}(" in out, name
    for name in ("tsb_check_matmul", "tsb_check_layer", "tsb_check_degeneracy"):
        assert name in out
    deps = subprocess.run(["readelf", "-d", SO], capture_output=True, text=True).stdout
    assert "libtess.so" in deps  # the adapter calls the C-ABI, nothing else


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _built()
    import paper_2105_14500_b200  # noqa: F401  (libtess.so loaded first, same file)
    L = C.CDLL(SO)
    L.tsb_last_error.restype = C.c_char_p
    return L


def _out(n):
    return (C.c_double * n)()


def _ok(L, rc):
    assert rc == 0, L.tsb_last_error().decode()


GRIDS = [(1, 1, 0), (1, 2, 1), (2, 1, 0), (2, 2, 0)]


@pytest.mark.gpu
@pytest.mark.parametrize("q,d,allow", GRIDS + [(3, 1, 0)])
@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("replicate", [0, 1])
def test_drop_in_matmul_stats_and_trace(lib, q, d, allow, variant, replicate):
    o = _out(4)
    m, n, r = 16 * q * d, 8 * q, 12 * q
    _ok(lib, lib.tsb_check_matmul(q, d, allow, variant, 0, m, n, r, 1, replicate, o))
    assert o[0] <= 1e-5, o[0]
    assert o[1] == 1.0, "CommStats differ from the reference's"
    if o[2] != 1.0:
        w, g = C.create_string_buffer(1 << 16), C.create_string_buffer(1 << 16)
        lib.tsb_matmul_traces(q, d, allow, variant, m, n, r, w, g, 1 << 16)
        assert g.value.decode() == w.value.decode()
    assert o[3] > 0


@pytest.mark.gpu
def test_drop_in_config1_fp32(lib):
    """BASELINE config 1 through the drop-in: 1024^3 NN fp32 at [2,2,2]."""
    o = _out(4)
    _ok(lib, lib.tsb_check_matmul(2, 2, 0, 0, 0, 1024, 1024, 1024, 0, 0, o))
    assert o[0] <= 1e-5 and o[1] == 1.0, list(o)


@pytest.mark.gpu
@pytest.mark.parametrize("q,d,allow", GRIDS)
def test_drop_in_backward(lib, q, d, allow):
    o = _out(3)
    _ok(lib, lib.tsb_check_backward(q, d, allow, 0, 32 * q * d, 16 * q, 24 * q, o))
    assert o[0] <= 1e-5 and o[1] <= 1e-5 and o[2] == 1.0, list(o)


@pytest.mark.gpu
@pytest.mark.parametrize("q,d,allow", GRIDS)
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4])  # Feedforward Attention Layernorm BiasAdd Block
def test_drop_in_layer_run(lib, q, d, allow, op):
    o = _out(2)
    _ok(lib, lib.tsb_check_layer(op, 4, 8, 32, 4, q, d, allow, 0, o))
    assert o[0] <= 1e-5 and o[1] == 1.0, list(o)


@pytest.mark.gpu
@pytest.mark.parametrize("q,d,allow", [(1, 1, 0), (2, 2, 0)])
def test_drop_in_layer_run_bf16(lib, q, d, allow):
    o = _out(2)
    _ok(lib, lib.tsb_check_layer(4, 4, 64, 128, 4, q, d, allow, 1, o))
    assert o[0] <= 2e-2 and o[1] == 1.0, list(o)


@pytest.mark.gpu
@pytest.mark.parametrize("q", [1, 2, 3])
def test_drop_in_degeneracy_spec_637(lib, q):
    """Tesseract on [q,q,1] == SUMMA on [q,q], values and CommStats."""
    o = _out(3)
    _ok(lib, lib.tsb_check_degeneracy(q, 24 * q, 16 * q, 20 * q, 0, o))
    assert o[0] <= 1e-5 and o[1] == 1.0 and o[2] == 1.0, list(o)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_drop_in_megatron(lib, p):
    o = _out(2)
    _ok(lib, lib.tsb_check_megatron(p, 0, o))
    assert o[0] <= 1e-5 and o[1] == 1.0, list(o)


@pytest.mark.gpu
def test_drop_in_verify_sweep(lib):
    o = _out(3)
    _ok(lib, lib.tsb_sweep(o))
    assert o[0] <= 1e-5 and o[1] == 1.0 and o[2] == 15, list(o)


@pytest.mark.gpu
def test_drop_in_error_taxonomy(lib):
    """A shape the reference rejects raises the reference's exception class
    through the adapter (status -> ShapeError / DivisibilityError)."""
    assert lib.tsb_adapter_matmul(2, 2, 0, 0, 6, 8, 8) == 2      # rows % (q*d)
    assert lib.tsb_adapter_matmul(1, 1, 0, 0, 8, 8, 8) == 0
    assert lib.tsb_adapter_matmul(2, 1, 0, 1, 8, 8, 8) == 0
    assert lib.tsb_adapter_matmul(1, 3, 0, 0, 8, 8, 8) == 3      # d > q: GridError
