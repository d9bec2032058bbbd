"""ORACLE (test infrastructure only) — backward-Euler time stepping of transient Stokes.

P:L87: the transient problem is discretised in time with mu = 1/dt, so each step solves the
coupled system of eq. (syslin) with the mass term mu M (lumped CR mass |K|/(d+1) per
local face) moved to the right-hand side for the previous step:
    (mu M + nu A) U^{n+1} + D^t P^{n+1} = R + mu M U^n,      D U^{n+1} = g,
and "all the linear systems have the same matrix".  Plain definition: assemble once,
solve each step with the refined direct solve.
"""
from __future__ import annotations

import numpy as np

from .krylov import direct_refined
from .mesh import Mesh
from .scheme import Data, Params, _gidx, assemble_coupled


def lumped_mass(m: Mesh) -> np.ndarray:
    """Diagonal of the lumped CR mass per velocity unknown (d * face_dof + i): the sum over the
    cells K of the face of |K| / (d + 1)."""
    d = m.dim
    gi = _gidx(m)
    vals = np.repeat(m.vol[:, None] / (d + 1), (d + 1) * d, axis=1)
    out = np.zeros(d * m.nf_int)
    keep = gi >= 0
    np.add.at(out, gi[keep], vals[keep])
    return out


def backward_euler(m: Mesh, prm: Params, data: Data, nsteps: int, U0: np.ndarray | None = None):
    """nsteps backward-Euler steps from U0 ([nf_int, d], default 0).  Returns the lists of U
    [nf_int, d] and P [nc] (P_K0 = 0) after each step."""
    M, rhs, nU = assemble_coupled(m, prm, data)
    mass = prm.mu * lumped_mass(m)
    U = np.zeros(nU) if U0 is None else np.asarray(U0, dtype=np.float64).reshape(-1).copy()
    Us, Ps = [], []
    for _ in range(nsteps):
        b = rhs.copy()
        b[:nU] += mass * U
        x = direct_refined(M, b)
        U = x[:nU].copy()
        Us.append(U.reshape(m.nf_int, m.dim).copy())
        Ps.append(np.insert(x[nU:], prm.k0, 0.0))
    return Us, Ps
