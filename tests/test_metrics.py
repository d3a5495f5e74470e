"""bench.py's metric conventions reproduce the paper's printed Table 1
(tests/golden/table1.txt): GB/s = sites * 592 B / T_prop,
MLUPS = sites / T."""
import os

import pytest

from paper_1703_00186_b200 import perfmodel as pm

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "table1.txt")
SITES = 1920 * 2048


def rows():
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            name, tp, gb, tc, mc, tw, mw = line.split()
            yield name, float(tp), int(gb), float(tc), int(mc), float(tw), int(mw)


@pytest.mark.parametrize("row", list(rows()), ids=lambda r: r[0])
def test_table1_reproduced(row):
    name, tp, gb, tc, mc, tw, mw = row
    assert round(pm.gbs(SITES, tp * 1e-3)) == gb
    assert round(pm.mlups(SITES, tc * 1e-3)) == mc
    assert round(pm.mlups(SITES, tw * 1e-3)) == mw


def test_sites_of_table1():
    assert SITES == 3932160
