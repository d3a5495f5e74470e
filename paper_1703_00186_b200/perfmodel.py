"""Timing model of the paper's §5, fitted to B200 measurements (NEXT 4).

The paper models one time step on n GPUs as T = max{T_a, T_b} with
T_a = T_bulk + T_borderL + T_borderR, T_b = T_MPI + T_borderL + T_borderR
(P:795-800), and to first approximation

    T(Lx, Ly, n) = max{ alpha (Lx/n) Ly + beta (Lx/n),  gamma Ly } + delta Ly,
    S_r(Lx, Ly, n) = T(Lx, Ly, 1) / T(Lx, Ly, n).

Here alpha is the bulk time per site, beta the per-column cost (the paper's
bc, which scales with Lx), gamma the halo exchange time per row and delta the
border-column processing time per row.  An optional constant latency `eps`
(kernel launch / NCCL latency, absent from the paper's first approximation)
is added to the communication branch when given.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np


@dataclass
class Params:
    alpha: float          # s per bulk site
    beta: float           # s per column
    gamma: float          # s per row of halo exchange
    delta: float          # s per row of border processing (both borders)
    eps: float = 0.0      # s, constant exchange latency (extension; 0 = paper's model)

    def as_dict(self):
        return asdict(self)


def step_time(p: Params, lx: float, ly: float, n: int) -> float:
    """T(Lx, Ly, n) of P:825 (plus eps on the communication branch)."""
    ta = p.alpha * (lx / n) * ly + p.beta * (lx / n)
    tb = p.gamma * ly + (p.eps if n > 1 else 0.0)
    if n == 1:
        tb = 0.0  # no exchange on one device: the wrap is part of the step kernel
    return max(ta, tb) + p.delta * ly


def speedup(p: Params, lx: float, ly: float, n: int) -> float:
    """S_r(Lx, Ly, n) = T(Lx, Ly, 1) / T(Lx, Ly, n), strong scaling."""
    return step_time(p, lx, ly, 1) / step_time(p, lx, ly, n)


def weak_efficiency(p: Params, lx_per_gpu: float, ly: float, n: int) -> float:
    """T(lx, Ly, 1) / T(n lx, Ly, n): fixed work per GPU."""
    return step_time(p, lx_per_gpu, ly, 1) / step_time(p, n * lx_per_gpu, ly, n)


def fit_bulk(samples) -> tuple[float, float]:
    """Least squares T_bulk = alpha * lx * ly + beta * lx over samples (lx, ly, t)."""
    A = np.array([[lx * ly, lx] for lx, ly, _ in samples], dtype=float)
    t = np.array([s[2] for s in samples], dtype=float)
    (alpha, beta), *_ = np.linalg.lstsq(A, t, rcond=None)
    return float(alpha), float(beta)


def fit_rows(samples) -> float:
    """Least squares t = c * ly through the origin over samples (ly, t)."""
    ly = np.array([s[0] for s in samples], dtype=float)
    t = np.array([s[1] for s in samples], dtype=float)
    return float(ly @ t / (ly @ ly))


def exchange_gamma(bytes_per_row: float, link_bytes_per_s: float) -> float:
    """gamma from a link bandwidth: the halo message of one rank per direction is
    3 columns x 37 populations x 8 B per row; both directions and both
    neighbours are in flight at once, so the rank's egress is 2 x that."""
    return bytes_per_row / link_bytes_per_s


# ---- metric conventions (Table 1 / Table 3 of the paper) ----
BYTES_PER_SITE = 592  # 37 fp64 reads + 37 fp64 writes per site and step


def gbs(sites: float, seconds: float, bytes_per_site: float = BYTES_PER_SITE) -> float:
    """Effective bandwidth of a step kernel: sites * 592 B / t."""
    return sites * bytes_per_site / seconds / 1e9


def mlups(sites: float, seconds: float) -> float:
    """Millions of lattice-site updates per second."""
    return sites / seconds / 1e6
