"""CPU-only checks of the C-ABI boundary and host logic (no kernels run)."""
import ctypes
import os
import re

import pytest

import paper_2105_14500_b200 as tess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tess.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tess_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(tess.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_version_and_launch_counter():
    assert b"sm_100a" in tess.lib.tess_version()
    assert tess.kernel_launches() >= 0


@pytest.mark.parametrize("q,d,allow", [(1, 1, False), (1, 2, True), (2, 1, False), (2, 2, False),
                                       (3, 1, False), (3, 3, False), (4, 2, False)])
def test_grid_matches_oracle(orc, q, d, allow):
    g = tess.GridSpec(q, d, allow)
    assert g.size() == d * q * q
    for r in range(g.size()):
        c = g.coord_of(r)
        assert (c.i, c.j, c.k) == orc.coord_of(q, r)
        assert g.rank_of(c) == r
        assert g.block_row(c) == orc.block_row(q, c.i, c.k)
        for kind in (0, 1, 2):
            assert g.group_index(c, kind) == orc.group_index(q, (c.i, c.j, c.k), kind)
            assert g.slot_in_group(c, kind) == orc.slot_in_group((c.i, c.j, c.k), kind)
            members = g.group_of(c, kind)
            assert c in members and len(members) == g.group_size(kind)


def test_grid_errors_and_parse():
    with pytest.raises(tess.GridError, match="depth d exceeds dimension q"):
        tess.GridSpec(1, 2)
    with pytest.raises(tess.GridError):
        tess.GridSpec(0, 1)
    g = tess.GridSpec.parse("[2,2,2]")
    assert (g.q(), g.d()) == (2, 2)
    assert tess.GridSpec.parse("[1,1,2]", allow_d_gt_q=True).d() == 2
    with pytest.raises(tess.ConfigError, match="first two extents must match"):
        tess.GridSpec.parse("[2,3,1]")
    with pytest.raises(tess.ConfigError, match="position 0"):
        tess.GridSpec.parse("2,2,2]")
    with pytest.raises(tess.ConfigError, match="trailing"):
        tess.GridSpec.parse("[2,2,2]x")


def test_grid_parse_matches_reference(ref):
    for text in ("[2,2,2]", "[4,4,1]", "[3,3,3]"):
        assert ref.grid_parse(text) == (tess.GridSpec.parse(text).q(), tess.GridSpec.parse(text).d())


def test_comm_stats_struct_layout():
    assert ctypes.sizeof(tess.CommStatsC) == 8 * (4 + 10)
    assert ctypes.sizeof(tess.BlockShardC) == 8 * 9
