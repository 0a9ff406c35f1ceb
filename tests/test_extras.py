"""SURVEY 8(f) plumbing on the CPU: FNV-1a fingerprints and TMX1 / CSV matrix
files are interchangeable with the reference's (matrix.cpp:244-370); the
oracle's megatron_1d_linear restatement is pinned to the reference."""
import numpy as np
import pytest

import paper_2105_14500_b200 as tess


def test_checksum_matches_app_b(orc):
    a = orc.random_matrix(1024, 1024, 42, 0)
    assert tess.checksum(a) == "fnv1a:d1778dee67eb0201" == orc.checksum(a)


@pytest.mark.parametrize("ext", [".tmx", ".csv"])
def test_matrix_files_roundtrip_and_reference_reads_them(orc, ref, tmp_path, ext):
    m = orc.random_matrix(7, 5, 3, 0)
    p = str(tmp_path / ("m" + ext))
    tess.save_matrix(m, p)
    assert (tess.load_matrix(p) == m).all()  # exact (shortest round-trip text / raw bits)
    assert ref.file_checksum(p) == tess.checksum(m)


def test_load_errors(tmp_path):
    p = tmp_path / "bad.tmx"
    p.write_bytes(b"NOPE")
    with pytest.raises(tess.IoError):
        tess.load_matrix(str(p))
    with pytest.raises(tess.IoError):
        tess.load_matrix(str(tmp_path / "missing.tmx"))


@pytest.mark.parametrize("p", [1, 2, 4])
def test_megatron_oracle_vs_reference(orc, ref, p):
    x = orc.random_matrix(6, 8, 5, 0)
    w1 = orc.random_matrix(8, 12, 5, 1)
    w2 = orc.random_matrix(12, 4, 5, 2)
    got = orc.megatron_1d_linear(x, w1, w2, p)
    want, sr, sk = ref.megatron_1d_linear(x, w1, w2, p)
    assert np.abs(got - want).max() < 1e-14
