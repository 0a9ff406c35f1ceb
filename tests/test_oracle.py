"""Pins the oracle (oracle/tess_oracle.c, a C restatement of the reference)
to the reference: App. B golden fingerprints + SPEC.md KATs + fixtures made
by the unmodified reference (tests/golden/make_golden.py) + direct
comparison with oracle/_ref when it is built."""
import numpy as np
import pytest

import oracle

GRIDS = [(1, 1, False), (1, 2, True), (2, 1, False), (2, 2, False)]


def test_rng_stream_words(orc):
    # Rng::stream(42,0) first two words, as produced by the reference build
    # (SURVEY App. B lists the same pair in the opposite order).
    assert orc.stream_words(42, 0, 2) == [11572511668999661906, 15353713867457212013]


def test_golden_fingerprints_app_b(orc):
    a = orc.random_matrix(1024, 1024, 42, 0)
    b = orc.random_matrix(1024, 1024, 42, 1)
    assert orc.checksum(a) == "fnv1a:d1778dee67eb0201"
    assert orc.checksum(b) == "fnv1a:ee1db372dccfd0e0"
    assert a[0, 0] == 0.25469422926432839 and a[0, 1] == 0.66465299308179238
    assert a[1023, 1023] == -0.90085099145177971 and b[0, 0] == -0.87645924362003846
    want_a = ["5b24f7f4279b3a7c", "86b898339a31079c", "f7baeb73d9d5d97b", "4750f274f97cfe36",
              "be6ab8ba8f56292f", "5b505fec976e1685", "38d70a17da398b7b", "ff33fd1037052c24"]
    assert [orc.checksum(x) for x in orc.partition(a, 2, 2, 0)] == ["fnv1a:" + w for w in want_a]
    want_b = ["ba632a53a93097de", "5e0ec15860904579", "c538e3d304e3a949", "fa970abde254eb4f"]
    bb = orc.partition(b, 2, 2, 1)
    assert [orc.checksum(x) for x in bb[:4]] == ["fnv1a:" + w for w in want_b]
    assert all((bb[r] == bb[r - 4]).all() for r in range(4, 8))  # replicated over k
    c, sr, sk = orc.tesseract_matmul(a, b, 2, 2, "nn")
    assert orc.checksum(c) == "fnv1a:736692f54d33ee3e"
    assert int(sk[0, 0]) == 16 and int(sk[0, 1]) == 3145728  # App. A probe


def test_spec_kats(orc):
    # matmul_serial [[1,2],[3,4]]x[[5,6],[7,8]]
    assert (orc.matmul([[1, 2], [3, 4]], [[5, 6], [7, 8]]) == [[19, 22], [43, 50]]).all()
    # rank = k*q*q + i*q + j, block row h = i + k*q (grid.cpp:43-69)
    assert orc.rank_of(2, 1, 0, 1) == 6 and orc.coord_of(2, 6) == (1, 0, 1)
    assert orc.block_row(2, 1, 1) == 3
    for r in range(8):
        assert orc.rank_of(2, *orc.coord_of(2, r)) == r
    # group families (grid.cpp:79-95): row (i,k) slot j; col (j,k) slot i; depth (i,j) slot k
    assert orc.group_index(2, (1, 0, 1), 0) == 3 and orc.slot_in_group((1, 0, 1), 0) == 0
    assert orc.group_index(2, (1, 0, 1), 1) == 2 and orc.slot_in_group((1, 0, 1), 1) == 1
    assert orc.group_index(2, (1, 0, 1), 2) == 2 and orc.slot_in_group((1, 0, 1), 2) == 1


def test_partition_combine_roundtrip(orc):
    m = orc.random_matrix(24, 12, 3, 0)
    for q, d, _ in GRIDS + [(3, 1, False)]:
        for scheme in (0, 1):
            blocks = orc.partition(m, q, d, scheme)
            assert (orc.combine(blocks, 24, 12, q, d, scheme) == m).all()
    bad = orc.partition(m, 2, 2, 1)
    bad[5] = bad[5].copy()
    bad[5][0, 0] += 1.0
    with pytest.raises(ValueError):
        orc.combine(bad, 24, 12, 2, 2, 1)


@pytest.mark.parametrize("q,d,allow", GRIDS)
def test_matmul_vs_reference_fixtures(orc, golden, q, d, allow):
    for v in ("nn", "nt", "tn"):
        key = f"mm_{v}_{q}{q}{d}"
        c, sr, sk = orc.tesseract_matmul(golden[key + "_a"], golden[key + "_b"], q, d, v)
        assert (c == golden[key + "_c"]).all()  # bit-exact: same op order
        assert (sr == golden[key + "_sr"]).all() and (sk == golden[key + "_sk"]).all()
    key = f"bwd_{q}{q}{d}"
    da, db, sr, sk = orc.tesseract_backward(golden[key + "_dc"], golden[key + "_a"],
                                            golden[key + "_b"], q, d)
    assert (da == golden[key + "_da"]).all() and (db == golden[key + "_db"]).all()
    assert (sr == golden[key + "_sr"]).all() and (sk == golden[key + "_sk"]).all()


@pytest.mark.parametrize("op", list(oracle.LAYER_OPS))
def test_layers_vs_reference_fixtures(orc, golden, op):
    P = {k: golden["layer_p_" + k] for k in oracle.PARAM_NAMES}
    res = orc.layer_run(op, golden["layer_x"], golden["layer_dy"], P, 4, 3, 4)
    # reference ran sharded on [2,2,2]; serial ref::* agrees to ~1e-15
    assert np.abs(res["y"] - golden[f"layer_{op}_y"]).max() < 1e-13
    assert np.abs(res["dx"] - golden[f"layer_{op}_dx"]).max() < 1e-13
    for k in oracle.PARAM_NAMES:
        assert np.abs(res["grads"][k] - golden[f"layer_{op}_g_{k}"]).max() < 1e-13
    assert np.abs(res["dbias"] - golden[f"layer_{op}_dbias"]).max() < 1e-13
    _, sk = orc.layer_stats(op, 2, 2, 4, 3, 16)
    assert (sk == golden[f"layer_{op}_sk"]).all()


def test_block_message_count_288(orc):
    # SURVEY 2.6 / App. A probe5: 288 metered messages for a Block at [2,2,2]
    _, sk = orc.layer_stats("block", 2, 2, 8, 4, 16)
    assert int(sk[:, 0].sum()) == 288


@pytest.mark.parametrize("q,d,allow", GRIDS + [(3, 1, False)])
def test_restatement_vs_reference_library(orc, ref, q, d, allow):
    m, n, r = 6 * q * d, 4 * q, 3 * q
    a = orc.random_matrix(m, n, 21, 0)
    for v, b in (("nn", orc.random_matrix(n, r, 21, 1)), ("nt", orc.random_matrix(r, n, 21, 1)),
                 ("tn", orc.random_matrix(m, r, 21, 1))):
        c1, s1, k1 = orc.tesseract_matmul(a, b, q, d, v)
        c2, s2, k2 = ref.tesseract_matmul(a, b, q, d, v, allow=allow)
        assert (c1 == c2).all() and (s1 == s2).all() and (k1 == k2).all()
    bb, s, h, nh = 2 * q * d, 3, 8 * q, 2 * q
    x = orc.random_matrix(bb * s, h, 22, 0)
    dy = orc.random_matrix(bb * s, h, 22, 2)
    P = orc.random_block_params(h, 22, 100)
    for op in oracle.LAYER_OPS:
        a1 = orc.layer_run(op, x, dy, P, bb, s, nh)
        a2 = ref.layer_run(op, x, dy, P, bb, s, nh, q=q, d=d, allow=allow)
        for key in ("y", "dx", "dbias"):
            assert np.abs(a1[key] - a2[key]).max() < 1e-13
        for k in oracle.PARAM_NAMES:
            assert np.abs(a1["grads"][k] - a2["grads"][k]).max() < 1e-13
        sr, sk = orc.layer_stats(op, q, d, bb, s, h)
        assert (sr == a2["stats_rank"]).all() and (sk == a2["stats_kind"]).all()


def test_reference_verify_suite_passes(ref):
    n, npass, worst = ref.verify_suite(trials=2)
    assert n == npass == 66 and worst < 1e-10
