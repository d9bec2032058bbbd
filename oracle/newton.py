"""ORACLE (test infrastructure only) — Newton's method for the steady Navier-Stokes problem.

P:L95-98, L273, L302: each Newton step solves the coupled system (eq. (syslin)) whose A_K is
completed by the derivatives of the convection term at the iterate U^k and whose R_K is completed
by the non-linear terms (increment form, reading 6):
    [A(U^k), D^t; D, 0] [dU; dP] = [-(A_S U^k + r(U^k) + D^t P^k - R_f); -D U^k],
    U^{k+1} = U^k + dU,  P^{k+1} = P^k + dP,
with the wall / lid values on the boundary faces of every iterate (P:L21 Dirichlet data).
Stopping rule (Table 7): ||dU||_2 <= tol ||U^{k+1}||_2.
"""
from __future__ import annotations

import numpy as np

from .krylov import direct_refined
from .mesh import Mesh
from .scheme import Data, Params, assemble_coupled


def cell_face_values(m: Mesh, U: np.ndarray, wall: np.ndarray | None) -> np.ndarray:
    """Per (cell, local face) values of a face field: U on interior faces, the wall value on
    boundary faces ([nc, d+1, d])."""
    d = m.dim
    dof = m.face_dof[m.cell_faces]
    out = np.zeros((m.nc, d + 1, d)) if wall is None else np.array(wall, dtype=np.float64, copy=True)
    inside = dof >= 0
    out[inside] = U[dof[inside]]
    return out


def residual_norm(m: Mesh, prm: Params, fbar: np.ndarray, wall: np.ndarray | None, U: np.ndarray,
                  P: np.ndarray) -> float:
    """||F(U, P)||_2: the right-hand side [R; g] of the increment-form Newton system at (U, P) is
    minus the nonlinear residual of the discrete steady Navier-Stokes equations."""
    _, rhs, _ = assemble_coupled(m, prm, Data(fbar=fbar, u_iter=cell_face_values(m, U, wall), p_iter=P))
    return float(np.linalg.norm(rhs))


def newton_ns(m: Mesh, prm: Params, fbar: np.ndarray, wall: np.ndarray | None, max_newton: int = 30,
              tol: float = 5e-7, damped: bool = False, lam_min: float = 1.0 / 64):
    """Newton iterations from U^0 = 0 (interior), P^0 = 0.  Returns U [nf_int, d], P [nc] and the
    list of ||lam dU|| / ||U^{k+1}||.

    damped=True globalises the iteration (the paper's Re = 1000 cavity, diverges from
    rest with full steps on some meshes): backtracking on the nonlinear residual, the step length
    lam = 1, 1/2, 1/4, ... >= lam_min is the first with ||F(U + lam dU)|| < (1 - 1e-4 lam) ||F(U)||
    (Armijo; lam_min is taken if none is)."""
    U = np.zeros((m.nf_int, m.dim))
    P = np.zeros(m.nc)
    hist = []
    for _ in range(max_newton):
        data = Data(fbar=fbar, u_iter=cell_face_values(m, U, wall), p_iter=P)
        M, rhs, nU = assemble_coupled(m, prm, data)
        x = direct_refined(M, rhs)
        dU = x[:nU].reshape(m.nf_int, m.dim)
        dP = np.insert(x[nU:], prm.k0, 0.0)
        lam = 1.0
        if damped:
            r0 = float(np.linalg.norm(rhs))
            while lam > lam_min:
                if residual_norm(m, prm, fbar, wall, U + lam * dU, P + lam * dP) < (1.0 - 1e-4 * lam) * r0:
                    break
                lam *= 0.5
        U = U + lam * dU
        P = P + lam * dP
        rel = float(np.linalg.norm(lam * dU) / max(np.linalg.norm(U), 1e-300))
        hist.append(rel)
        if rel <= tol:
            break
    return U, P, hist
