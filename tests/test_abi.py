"""CPU tests of the C ABI: the library loads, exports every symbol include/hrp.h declares,
its host-side layout tables equal the oracle's, and argument validation fails loudly."""
import ctypes
import os
import random
import re

import pytest

from oracle import actions as A
from oracle import space as SP
from paper_2405_08754_b200 import build as B
from paper_2405_08754_b200 import hrp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
S10 = tuple(range(10, 100, 10))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hrp.h")).read()
    names = set(re.findall(r"\b(hrp_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 17
    L = ctypes.CDLL(hrp.LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n


@pytest.mark.parametrize("W,cmax,S,mig", [(4, 2, (25, 50, 75), True), (16, 3, S10, True),
                                          (12, 4, S10, True), (64, 4, S10, True),
                                          (12, 4, S10, False), (6, 3, (50,), True)])
def test_layout_table_equals_oracle(W, cmax, S, mig):
    osp = SP.build_space(W, cmax, S, mig)
    t = hrp.hrp_layout_table(hrp.make_space(W, cmax, S, mig))
    assert t["n_layouts"] == osp.L and t["n_types"] == osp.T
    assert t["n_actions"] == A.n_actions(osp)
    for l, lay in enumerate(osp.layouts):
        assert t["nslots"][l] == lay.C
        for k, s in enumerate(lay.slots):
            got = t["slots"][l, k]
            assert (int(got["sm800"]), int(got["b8"]), int(got["dom"])) == (s.sm800, s.b8, s.dom)
            assert t["slot_type"][l, k] == osp.slot_type[l][k]


def test_decode_equals_oracle():
    rng = random.Random(3)
    for (W, cmax, S) in [(4, 2, (25, 50, 75)), (16, 3, S10), (64, 4, S10)]:
        osp = SP.build_space(W, cmax, S)
        sp = hrp.make_space(W, cmax, S)
        off = A.offsets(osp)
        for _ in range(300):
            idx = rng.randrange(A.n_actions(osp))
            assert hrp.hrp_decode_action(sp, idx) == A.decode(osp, idx, off)


def test_validation_errors():
    with pytest.raises(hrp.HrpError) as e:
        hrp.hrp_layout_table(hrp.make_space(65, 2, (50,)))
    assert e.value.status == hrp.HRP_ERANGE
    with pytest.raises(hrp.HrpError) as e:
        hrp.hrp_layout_table(hrp.make_space(4, 5, (50,)))
    assert e.value.status == hrp.HRP_ERANGE
    with pytest.raises(hrp.HrpError) as e:
        hrp.hrp_decode_action(hrp.make_space(4, 2, (25, 50, 75)), 92)
    assert e.value.status == hrp.HRP_ERANGE
    sp = hrp.make_space(4, 2, (25, 50, 75), layouts=[[(800, 8, 0)], [(400, 8, 0), (400, 4, 0)]])
    with pytest.raises(hrp.HrpError) as e:   # slots of one domain must share memory
        hrp.hrp_layout_table(sp)
    assert e.value.status == hrp.HRP_EINVAL
    assert "domain" in hrp.lib().hrp_last_error().decode()


def test_explicit_layout_table_round_trip():
    lay = [[(800, 8, 0)], [(400, 4, 0), (300, 4, 1)], [(200, 8, 0), (600, 8, 0)]]
    t = hrp.hrp_layout_table(hrp.make_space(6, 2, (50,), layouts=lay))
    assert t["n_layouts"] == 3 and list(t["nslots"]) == [1, 2, 2]
    assert t["n_actions"] == 6 + 30 + 30


def test_mig_partitions_and_default_mps_tables_equal_oracle():
    # MIG+MPS Default (R27): libhrp's partitions (the layouts of the space with no MPS
    # splits) and the product-side default-MPS tables equal the oracle's own enumeration
    from paper_2405_08754_b200.schedule import default_mps_table, mig_partitions
    parts = mig_partitions(12, 4)
    ref = SP.mig_partitions(4)
    assert parts == ref and len(parts) == 39
    for p in parts:
        tab = default_mps_table(p, 4)
        oref = SP.default_mps_layouts(p, 4)
        assert tab == [[(s.sm800, s.b8, s.dom) for s in l.slots] for l in oref]
        assert all(1 <= len(l) <= 4 for l in tab)
        t = hrp.hrp_layout_table(hrp.make_space(12, 4, S10, True, layouts=tab))
        assert t["n_layouts"] == len(tab)
