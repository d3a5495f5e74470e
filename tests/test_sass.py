"""SASS census of the built library (CPU: cuobjdump, no GPU): the hot kernels
use the Blackwell-native data movement the design claims, and none of them
spills to local memory (tools/sass_census.py; profiles/r02_sass.json)."""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.fixture(scope="module")
def sass():
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    from paper_1703_00186_b200 import _build
    so = _build.build()          # no-op when the library is current
    import sass_census
    return sass_census.census(so)


def test_two_step_kernel_uses_tma_and_mbarriers(sass):
    tb = {k: v for k, v in sass.items() if v["kernel"] == "k_step2_tb"}
    assert len(tb) == 4          # {BGK, regularised} x {monitors off, on}
    for name, v in tb.items():
        assert v["UTMALDG"] >= 1, name   # cp.async.bulk.tensor window loads
        assert v["SYNCS"] >= 4, name     # mbarrier init / expect-tx / try-wait
        assert v["DFMA"] > 200, name     # two collisions of FP64 arithmetic


def test_tma_propagate_issues_one_load_per_population(sass):
    v = [v for v in sass.values() if v["kernel"] == "k_propagate_tma"]
    assert v and v[0]["UTMALDG"] == 37


def test_no_local_memory_in_hot_kernels(sass):
    import sass_census
    hot = {k: v for k, v in sass.items() if v["kernel"] in sass_census.HOT}
    assert len(hot) >= 20
    spills = {k: (v["LDL"], v["STL"]) for k, v in hot.items() if v["LDL"] or v["STL"]}
    assert not spills, spills
