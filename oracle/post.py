"""ORACLE (test infrastructure only) — C-8: post-processing.

zero-mean pressure p - (1/|Omega|) int p; discrete L2 errors: velocity
at face centres of gravity with the lumped weights |K|/(d+1) ("errors are
computed at the nodes for the velocities", read as the CR nodes = face centres),
pressure at cell centres of gravity.
"""
from __future__ import annotations

import numpy as np

from .mesh import Mesh


def zero_mean(m: Mesh, P: np.ndarray) -> np.ndarray:
    return P - np.sum(m.vol * P) / np.sum(m.vol)


def errors(m: Mesh, U: np.ndarray, P: np.ndarray, u_exact, p_exact, dirichlet=None):
    """Returns (errl2U, errl2P).  U [nf_int, d]; boundary faces take the Dirichlet
    value (zero when ``dirichlet`` is None)."""
    d = m.dim
    Uf = np.zeros((m.nf, d))
    Uf[m.face_dof >= 0] = U
    if dirichlet is not None:
        bnd = m.face_dof < 0
        K = m.face_cells[bnd, 0]
        f = np.nonzero(bnd)[0]
        l = np.argmax(m.cell_faces[K] == f[:, None], axis=1)
        Uf[bnd] = dirichlet[K, l]
    diff = Uf[m.cell_faces] - u_exact(m.xs)[m.cell_faces]      # [nc, d+1, d]
    eu = np.sqrt(np.sum(m.vol[:, None, None] / (d + 1) * diff ** 2))
    Pz = zero_mean(m, P)
    pe = zero_mean(m, p_exact(m.xK))
    ep = np.sqrt(np.sum(m.vol * (Pz - pe) ** 2))
    return float(eu), float(ep)
