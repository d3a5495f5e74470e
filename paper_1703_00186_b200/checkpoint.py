"""LBFIELD checkpoints (SPEC S:464 raw dump, SURVEY §5 "Checkpoint / resume").

Format: an ASCII header line ``LBFIELD <Q> <NX> <NY>\\n`` followed by Q*NX*NY
little-endian float64 values in canonical order [Q][NX][NY] (iy fastest).  The
library writes physical sites only (NX = Lx_total, NY = Ly), i.e. the array
``Lattice.gather()`` returns, and restarts with ``Lattice.set_state``.
"""
from __future__ import annotations

import numpy as np

MAGIC = "LBFIELD"


def save(path: str, state: np.ndarray) -> None:
    state = np.ascontiguousarray(state, dtype="<f8")
    if state.ndim != 3:
        raise ValueError("state must be [Q][NX][NY]")
    q, nx, ny = state.shape
    with open(path, "wb") as fh:
        fh.write(f"{MAGIC} {q} {nx} {ny}\n".encode())
        state.tofile(fh)


def load(path: str) -> np.ndarray:
    with open(path, "rb") as fh:
        head = fh.readline().decode().split()
        if len(head) != 4 or head[0] != MAGIC:
            raise ValueError(f"{path}: not an LBFIELD file")
        q, nx, ny = (int(v) for v in head[1:])
        data = np.fromfile(fh, dtype="<f8", count=q * nx * ny)
    if data.size != q * nx * ny:
        raise ValueError(f"{path}: truncated LBFIELD file")
    return data.reshape(q, nx, ny).astype(np.float64, copy=False)
