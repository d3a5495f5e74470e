"""Seeded synthetic input generators shared by the tests, the oracle leg and the
CUDA leg of the benchmark.

This module holds NONE of the Lattice Boltzmann arithmetic (no equilibrium, no
moments, no velocity set): it only produces macroscopic fields (rho, u, T) and
plain random numbers.  Each side turns macroscopic fields into populations
with its own equilibrium (oracle: ``lbref_init_macro``; library:
``lb_init_macro``).  The reference temperature ``t_ref`` is passed in by the
caller (T0 = 1/a^2 of DESIGN.md reading G3).

Recipe: an isobaric Rayleigh–Taylor-shaped
state, bottom hot / top cold, interface y_i(x) = (Ly-1)/2 + A cos(2 pi x/Lx_tot)
+ eps_x, A = max(1, Ly/64), eps_x ~ U(-1/4, 1/4) from numpy PCG64, T = t_ref (1
+ 0.05 tanh((y_i(x) - y)/w)), w = 2, rho = t_ref/T (p = rho T uniform), u = 0.
x is the GLOBAL column, so every X-slab of a decomposed lattice gets exactly
the columns the 1-slab lattice has (decomposition invariant).
"""
from __future__ import annotations

import numpy as np

RT_SEED = 1703


def rt_macro(lx_tot: int, ly: int, t_ref: float, seed: int = RT_SEED,
             x0: int = 0, lx: int | None = None, amp: float = 0.05, width: float = 2.0):
    """Rayleigh–Taylor-shaped macroscopic fields for global columns [x0, x0+lx).

    Returns (rho, ux, uy, T), each float64 [lx][ly] (iy fastest)."""
    if lx is None:
        lx = lx_tot - x0
    eps = rt_eps(lx_tot, seed)
    x = np.arange(x0, x0 + lx, dtype=np.float64)
    A = max(1.0, ly / 64.0)
    yi = (ly - 1) / 2.0 + A * np.cos(2.0 * np.pi * x / lx_tot) + eps[x0:x0 + lx]
    yp = np.arange(ly, dtype=np.float64)
    T = t_ref * (1.0 + amp * np.tanh((yi[:, None] - yp[None, :]) / width))
    rho = t_ref / T
    ux = np.zeros_like(T)
    uy = np.zeros_like(T)
    return (np.ascontiguousarray(rho), ux, uy, np.ascontiguousarray(T))


def rt_eps(lx_tot: int, seed: int = RT_SEED):
    """The per-column interface jitter eps_x ~ U(-1/4, 1/4) of rt_macro, for
    all lx_tot global columns (what lb_init_rt takes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-0.25, 0.25, size=lx_tot)


def perturbed_macro(lx: int, ly: int, t_ref: float, seed: int = 7,
                    rho_amp: float = 0.05, u_amp: float = 0.02, t_amp: float = 0.05):
    """Random near-equilibrium macroscopic fields: rho = 1 +- rho_amp,
    |u_x|,|u_y| <= u_amp, T = t_ref (1 +- t_amp), uniform i.i.d. per site."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rho = 1.0 + rng.uniform(-rho_amp, rho_amp, size=(lx, ly))
    ux = rng.uniform(-u_amp, u_amp, size=(lx, ly))
    uy = rng.uniform(-u_amp, u_amp, size=(lx, ly))
    T = t_ref * (1.0 + rng.uniform(-t_amp, t_amp, size=(lx, ly)))
    return rho, ux, uy, T


def uniform_noise(shape, seed: int = 11, lo: float = -1.0, hi: float = 1.0):
    """Plain i.i.d. uniform noise (PCG64), float64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, size=shape)


def random_field(q: int, lx: int, ly: int, seed: int = 5, lo: float = 1e-4, hi: float = 0.3):
    """i.i.d. uniform population values in [lo, hi) — the value range of the
    RT workload (f in [1.94e-4, 0.258]) — for pure data-movement
    tests (propagate, pbc, layout) where no physics is needed."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(lo, hi, size=(q, lx, ly))
