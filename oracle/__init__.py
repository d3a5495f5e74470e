"""CPU oracle for the D2Q37 time step of arXiv 1703.00186 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It shares
no code with ``paper_1703_00186_b200`` and never imports it.

The arithmetic lives in plain C (``lbref.c``, built ``-O2 -ffp-contract=off``
with optional OpenMP over ix); this module is a ctypes wrapper around it.
Every function cites PAPER.md lines ("P:a-b") or a DESIGN.md reading (G1..G25).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

Q = 37
HALO = 3
WALL_THERMAL, WALL_ADIABATIC, PERIODIC = 0, 1, 2
BGK, REGULARIZED = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblbref.so")
_lib = None


def build(force: bool = False, openmp: bool = True) -> str:
    """Compile lbref.c into liblbref.so (gcc -O2 -ffp-contract=off)."""
    src = os.path.join(_HERE, "lbref.c")
    hdr = os.path.join(_HERE, "lbref.h")
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _SO
    cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
           "-shared", "-Wall", "-Wextra", "-o", _SO + ".tmp", src]
    if openmp:
        cmd.insert(1, "-fopenmp")
    subprocess.check_call(cmd)
    os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        d, i, p, v = ctypes.c_double, ctypes.c_int, ctypes.c_void_p, None
        dp = ctypes.POINTER(ctypes.c_double)
        sig = {
            "lbref_velocities": (v, [p]), "lbref_weights": (v, [p]),
            "lbref_scale_a": (d, []), "lbref_t0": (d, []),
            "lbref_refl": (i, [i]), "lbref_opp": (i, [i]),
            "lbref_macro": (v, [p, p]), "lbref_feq": (v, [d, d, d, d, p]),
            "lbref_kwall": (v, [d, p]), "lbref_collide_site": (v, [p, d]),
            "lbref_project": (v, [p, p]), "lbref_collide_site_reg": (v, [p, d]),
            "lbref_collide_site_force": (v, [p, d, d, d, i]), "lbref_set_gravity": (v, [p, d, d]),
            "lbref_init": (p, [i, i, d, d, d, d, i, i]), "lbref_free": (v, [p]),
            "lbref_nx": (i, [p]), "lbref_ny": (i, [p]), "lbref_buffer": (dp, [p, i]),
            "lbref_set_state": (v, [p, p]), "lbref_get_state": (v, [p, i, p]),
            "lbref_init_macro": (v, [p, p, p, p, p]),
            "lbref_pbc": (v, [p]), "lbref_propagate": (v, [p]), "lbref_bc": (v, [p]),
            "lbref_collide": (v, [p]), "lbref_swap": (v, [p]), "lbref_step": (v, [p, i]),
            "lbref_invariants": (v, [p, i, p]), "lbref_threads": (i, []), "lbref_set_threads": (v, [i]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


# ---- constants and per-site functions -------------------------------------

def velocities() -> np.ndarray:
    """App. A / G1, G2: int array [37, 2] of (cx, cy)."""
    c = np.zeros((Q, 2), dtype=np.int32)
    lib().lbref_velocities(c.ctypes.data_as(ctypes.c_void_p))
    return c.astype(np.int64)


def weights() -> np.ndarray:
    w = np.zeros(Q)
    lib().lbref_weights(_ptr(w))
    return w


def scale_a() -> float:
    return lib().lbref_scale_a()


def t0() -> float:
    return lib().lbref_t0()


def refl(l: int) -> int:
    return lib().lbref_refl(l)


def opp(l: int) -> int:
    return lib().lbref_opp(l)


def macro(f) -> np.ndarray:
    """Eq. 2: returns [rho, ux, uy, T]."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(4)
    lib().lbref_macro(_ptr(f), _ptr(out))
    return out


def feq(rho, ux, uy, T) -> np.ndarray:
    """App. B equilibrium at one site."""
    out = np.zeros(Q)
    lib().lbref_feq(float(rho), float(ux), float(uy), float(T), _ptr(out))
    return out


def kwall(t_wall) -> np.ndarray:
    out = np.zeros(Q)
    lib().lbref_kwall(float(t_wall), _ptr(out))
    return out


def collide_site(f, omega) -> np.ndarray:
    f = np.array(f, dtype=np.float64)
    lib().lbref_collide_site(_ptr(f), float(omega))
    return f


def project(f) -> np.ndarray:
    """Hermite projection onto orders <= 4 (reading G6)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros(Q)
    lib().lbref_project(_ptr(f), _ptr(out))
    return out


def collide_site_force(f, omega, gx, gy, collision=BGK) -> np.ndarray:
    """Collide with body force g: shifted equilibrium (reading G7b)."""
    f = np.array(f, dtype=np.float64)
    lib().lbref_collide_site_force(_ptr(f), float(omega), float(gx), float(gy), int(collision))
    return f


def collide_site_reg(f, omega) -> np.ndarray:
    """Regularised collide: f_eq + (1 - omega)(P f - f_eq)."""
    f = np.array(f, dtype=np.float64)
    lib().lbref_collide_site_reg(_ptr(f), float(omega))
    return f


# ---- lattice stepper --------------------------------------------------------

class Lattice:
    """One slab (N=1) of the canonical layout [37][Lx+6][Ly+6]."""

    def __init__(self, lx, ly, tau=0.8, dt=1.0, t_bottom=None, t_top=None, bc_y=WALL_THERMAL,
                 collision=BGK, gravity=(0.0, 0.0)):
        T0 = t0()
        t_bottom = 1.05 * T0 if t_bottom is None else t_bottom
        t_top = 0.95 * T0 if t_top is None else t_top
        self.lx, self.ly = lx, ly
        self._h = lib().lbref_init(lx, ly, tau, dt, t_bottom, t_top, bc_y, collision)
        if not self._h:
            raise ValueError("lbref_init rejected the parameters")
        lib().lbref_set_gravity(self._h, float(gravity[0]), float(gravity[1]))
        self.nx = lib().lbref_nx(self._h)
        self.ny = lib().lbref_ny(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().lbref_free(h)
            self._h = None

    def buffer(self, which=0) -> np.ndarray:
        """A view of the full canonical buffer A (0) or B (1), [37][NX][NY]."""
        p = lib().lbref_buffer(self._h, which)
        return np.ctypeslib.as_array(p, shape=(Q, self.nx, self.ny))

    def set_state(self, phys):
        phys = np.ascontiguousarray(phys, dtype=np.float64)
        assert phys.shape == (Q, self.lx, self.ly)
        lib().lbref_set_state(self._h, _ptr(phys))

    def get_state(self, which=0) -> np.ndarray:
        out = np.zeros((Q, self.lx, self.ly))
        lib().lbref_get_state(self._h, which, _ptr(out))
        return out

    def init_macro(self, rho, ux, uy, T):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (rho, ux, uy, T)]
        for a in arrs:
            assert a.shape == (self.lx, self.ly)
        lib().lbref_init_macro(self._h, *[_ptr(a) for a in arrs])

    def pbc(self):
        lib().lbref_pbc(self._h)

    def propagate(self):
        lib().lbref_propagate(self._h)

    def bc(self):
        lib().lbref_bc(self._h)

    def collide(self):
        lib().lbref_collide(self._h)

    def swap(self):
        lib().lbref_swap(self._h)

    def step(self, n=1):
        lib().lbref_step(self._h, n)

    def invariants(self, which=0) -> np.ndarray:
        out = np.zeros(4)
        lib().lbref_invariants(self._h, which, _ptr(out))
        return out


def threads() -> int:
    return lib().lbref_threads()


def set_threads(n: int) -> None:
    """Timing harness only: OpenMP threads of the stepper (arithmetic unchanged)."""
    lib().lbref_set_threads(int(n))
