"""Host-side tests of the C-ABI library (no GPU): it loads, exports every symbol
include/lb.h declares, validates parameters, and its host-computed constants
agree with the independently written oracle (K_wall bit for bit, G16)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import paper_1703_00186_b200 as lb
from paper_1703_00186_b200 import lb as lbmod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lb.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lb_[a-z_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    L = lb.lib()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert sorted(lb.EXPORTS) == names
    out = subprocess.run(["nm", "-D", "--defined-only", lb.SO_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lb_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", lb.SO_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_constants_agree_with_oracle():
    c, w, a, t0 = lb.constants()
    assert np.array_equal(c, oracle.velocities())
    assert np.array_equal(w, oracle.weights())
    assert a == oracle.scale_a()
    assert t0 == oracle.t0()


@pytest.mark.parametrize("rel", [1.05, 0.95, 1.0, 0.5, 1.7])
def test_kwall_bit_identical_to_oracle(rel):
    """G16/G25: both sides evaluate the canonical tree on the host -> identical bits."""
    tw = rel * oracle.t0()
    assert np.array_equal(lb.kwall(tw).view(np.uint64), oracle.kwall(tw).view(np.uint64))


def test_layout_arithmetic():
    p = lb.make_params(1920, 2048)
    L = lb.query_layout(p)
    assert (L.lx, L.ly, L.nx) == (1920, 2048, 1926)
    assert L.nyp % 16 == 0 and L.y0 % 16 == 0
    assert L.y0 >= 3 and L.y0 + L.ly + 3 <= L.nyp
    assert L.col_stride == 37 * L.nyp
    assert L.elems == L.nx * L.col_stride and L.bytes == 8 * L.elems
    assert L.sites == 1920 * 2048
    L4 = lb.query_layout(lb.make_params(8192, 8192), rank=3, nranks=4)
    assert (L4.lx, L4.x0_global) == (2048, 3 * 2048)


@pytest.mark.parametrize("kw,ranks,ok", [
    (dict(lx_total=64, ly=32), (0, 1), True),
    (dict(lx_total=3, ly=6), (0, 1), True),          # smallest N=1 walled lattice
    (dict(lx_total=2, ly=6), (0, 1), False),         # pbc needs 3 physical columns
    (dict(lx_total=64, ly=5), (0, 1), False),        # wall bands must be disjoint
    (dict(lx_total=64, ly=3, bc_y="periodic"), (0, 1), True),
    (dict(lx_total=64, ly=32), (1, 2), True),
    (dict(lx_total=65, ly=32), (0, 2), False),       # lx_total % N
    (dict(lx_total=20, ly=32), (0, 4), False),       # per-rank lx 5 < 6
    (dict(lx_total=24, ly=32), (0, 4), True),
    (dict(lx_total=64, ly=32, tau=0.4), (0, 1), False),   # dt/tau > 2
    (dict(lx_total=64, ly=32, tau=0.5), (0, 1), True),    # dt/tau = 2
    (dict(lx_total=64, ly=32, tau=-1.0), (0, 1), False),
    (dict(lx_total=64, ly=32, t_bottom=0.0), (0, 1), False),
    (dict(lx_total=64, ly=32, t_bottom=0.0, bc_y="adiabatic"), (0, 1), True),
    (dict(lx_total=64, ly=32), (2, 2), False),       # rank out of range
])
def test_query_layout_validation(kw, ranks, ok):
    p = lb.make_params(**kw)
    if ok:
        lb.query_layout(p, *ranks)
    else:
        with pytest.raises(lb.LBError) as ei:
            lb.query_layout(p, *ranks)
        assert ei.value.status == 1  # LB_EINVAL
        assert lb.lib().lb_last_error()


def test_strerror_and_no_gpu_construction_fails_loudly():
    assert lb.lib().lb_strerror(5).decode().startswith("non-physical")
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError):
            lb.Lattice(64, 32)


def test_oracle_and_library_share_no_code():
    """The oracle never includes/imports product code and vice versa."""
    bad_in_oracle = re.compile(r"(import\s+paper_1703_00186_b200|from\s+paper_1703_00186_b200|"
                               r"#include\s+\"[^\"]*(lb\.h|lb_device|lb_internal)[^\"]*\")")
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith((".c", ".h", ".py")):
            s = open(os.path.join(ROOT, "oracle", fn)).read()
            assert not bad_in_oracle.search(s), fn
    bad_in_pkg = re.compile(r"(import\s+oracle|from\s+oracle|lbref)")
    pkg = os.path.join(ROOT, "paper_1703_00186_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".cu", ".cuh", ".h", ".py")):
                s = open(os.path.join(dirpath, fn)).read()
                assert not bad_in_pkg.search(s), fn


def test_two_step_strip_height_matches_the_gpu_tests():
    """The strip-layout edge shapes of tests/test_gpu_parity.py are derived
    from TB_HT there; the library reports the height it was built with."""
    import test_gpu_parity
    assert lb.tb_strip_height() == test_gpu_parity.TB_HT
