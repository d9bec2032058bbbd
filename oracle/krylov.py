"""ORACLE (test infrastructure only) — C-6: global solves.

* ``direct_refined``: sparse LU (SuperLU via scipy, a library primitive) plus
  iterative refinement with the residual b - A x accumulated in binary128, the
  reference "exact" solve of eq. (syslin) / G W = S ("direct method for
  the small cases").
* ``pcg``, ``minres``, ``bicgstab``, ``gmres``: plain textbook Krylov solvers
  with Jacobi-type preconditioning ("a simple preconditioned conjugate
  gradient"; §4.2-4.3 CG / BCGS / GMRES).  They stop on the TRUE relative
  residual ||b - A x||_2 / ||b||_2 <= rtol with x0 = 0 (reading 12).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _p(x):
    return x.ctypes.data_as(ctypes.c_void_p)


def residual_f128(A: sp.csr_matrix, x: np.ndarray, b: np.ndarray) -> np.ndarray:
    """b - A x with all products and sums in binary128, rounded once."""
    from . import lib
    A = A.tocsr()
    rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.indices, dtype=np.int32)
    v = np.ascontiguousarray(A.data, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    r = np.empty(A.shape[0])
    lib().or_residual_f128(ctypes.c_int64(A.shape[0]), _p(rp), _p(ci), _p(v), _p(x), _p(b), _p(r))
    return r


def direct_refined(A, b, max_refine: int = 8, info: dict | None = None):
    lu = spla.splu(sp.csc_matrix(A))
    x = lu.solve(b)
    nb = np.linalg.norm(b)
    hist = []
    for _ in range(max_refine):
        r = residual_f128(A, x, b)
        rn = np.linalg.norm(r) / (nb if nb > 0 else 1.0)
        hist.append(rn)
        if rn == 0.0 or (len(hist) > 1 and rn >= 0.5 * hist[-2]):
            break
        x = x + lu.solve(r)
    if info is not None:
        info["refine_hist"] = hist
    return x


class Report(dict):
    pass


def _true_rel(A, x, b, nb):
    return np.linalg.norm(b - A @ x) / nb


def pcg(A, b, rtol=1e-10, max_iter=10**7, dinv=None, x0=None):
    """Jacobi-preconditioned CG (M^{-1} = diag(A)^{-1}), residual replacement at
    recursive convergence until the true residual meets rtol."""
    n = len(b)
    dinv = 1.0 / A.diagonal() if dinv is None else dinv
    x = np.zeros(n) if x0 is None else x0.copy()
    nb = np.linalg.norm(b)
    rep = Report(iterations=0, converged=False)
    if nb == 0:
        rep.update(converged=True, rel_res_true=0.0)
        return x, rep
    r = b - A @ x
    z = dinv * r
    p = z.copy()
    rho = r @ z
    it = 0
    while it < max_iter:
        q = A @ p
        pq = p @ q
        if pq <= 0:
            rep.update(status="breakdown")
            break
        alpha = rho / pq
        x += alpha * p
        r -= alpha * q
        it += 1
        if np.linalg.norm(r) <= rtol * nb:
            r = b - A @ x
            if np.linalg.norm(r) <= rtol * nb:
                rep.update(converged=True)
                break
        z = dinv * r
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    rep.update(iterations=it, rel_res_true=_true_rel(A, x, b, nb))
    return x, rep


def minres(A, b, rtol=1e-10, max_iter=10**7, minv=None, check_every=50):
    """Preconditioned MINRES (Paige-Saunders recurrences in the form of Elman,
    Silvester & Wathen), SPD preconditioner M = |diag(A)| (reading 11);
    stops on the true residual, checked every ``check_every`` iterations and
    when the preconditioned estimate drops below rtol."""
    n = len(b)
    minv = 1.0 / np.abs(A.diagonal()) if minv is None else minv
    x = np.zeros(n)
    nb = np.linalg.norm(b)
    rep = Report(iterations=0, converged=False)
    if nb == 0:
        rep.update(converged=True, rel_res_true=0.0)
        return x, rep
    v_old = np.zeros(n)
    v = b.copy()
    z = minv * v
    gamma = math.sqrt(v @ z)
    gamma_old = 1.0
    eta = gamma
    eta0 = gamma
    s_old = s = 0.0
    c_old = c = 1.0
    w_old = np.zeros(n)
    w = np.zeros(n)
    it = 0
    while it < max_iter:
        z = z / gamma
        Az = A @ z
        delta = Az @ z
        v_new = Az - (delta / gamma) * v - (gamma / gamma_old) * v_old
        z_new = minv * v_new
        gamma_new = math.sqrt(max(v_new @ z_new, 0.0))
        a0 = c * delta - c_old * s * gamma
        a1 = math.sqrt(a0 * a0 + gamma_new * gamma_new)
        a2 = s * delta + c_old * c * gamma
        a3 = s_old * gamma
        c_new = a0 / a1
        s_new = gamma_new / a1
        w_new = (z - a3 * w_old - a2 * w) / a1
        x += c_new * eta * w_new
        eta = -s_new * eta
        it += 1
        v_old, v = v, v_new
        z = z_new
        gamma_old, gamma = gamma, gamma_new
        c_old, c = c, c_new
        s_old, s = s, s_new
        w_old, w = w, w_new
        if abs(eta) <= rtol * eta0 or it % check_every == 0 or gamma == 0.0:
            if _true_rel(A, x, b, nb) <= rtol:
                rep.update(converged=True)
                break
            if gamma == 0.0:
                break
    rep.update(iterations=it, rel_res_true=_true_rel(A, x, b, nb))
    return x, rep


def bicgstab(A, b, rtol=1e-10, max_iter=10**7, dinv=None):
    """Right-Jacobi-preconditioned BiCGStab (van der Vorst), shadow residual r0."""
    n = len(b)
    dinv = 1.0 / A.diagonal() if dinv is None else dinv
    x = np.zeros(n)
    nb = np.linalg.norm(b)
    rep = Report(iterations=0, converged=False)
    if nb == 0:
        rep.update(converged=True, rel_res_true=0.0)
        return x, rep
    r = b.copy()
    rhat = r.copy()
    rho = alpha = omega = 1.0
    v = np.zeros(n); p = np.zeros(n)
    it = 0
    while it < max_iter:
        rho_new = rhat @ r
        if rho_new == 0.0:
            rep.update(status="breakdown")
            break
        beta = (rho_new / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        y = dinv * p
        v = A @ y
        alpha = rho_new / (rhat @ v)
        s = r - alpha * v
        zz = dinv * s
        t = A @ zz
        tt = t @ t
        omega = (t @ s) / tt if tt > 0 else 0.0
        x += alpha * y + omega * zz
        r = s - omega * t
        rho = rho_new
        it += 1
        if np.linalg.norm(r) <= rtol * nb:
            r = b - A @ x
            if np.linalg.norm(r) <= rtol * nb:
                rep.update(converged=True)
                break
        if omega == 0.0:
            rep.update(status="breakdown")
            break
    rep.update(iterations=it, rel_res_true=_true_rel(A, x, b, nb))
    return x, rep


def gmres(A, b, rtol=1e-10, restart=50, max_iter=10**6, dinv=None):
    """Restarted right-Jacobi-preconditioned GMRES(m), modified Gram-Schmidt
    Arnoldi with Givens rotations (Saad & Schultz)."""
    n = len(b)
    dinv = 1.0 / A.diagonal() if dinv is None else dinv
    x = np.zeros(n)
    nb = np.linalg.norm(b)
    rep = Report(iterations=0, converged=False)
    if nb == 0:
        rep.update(converged=True, rel_res_true=0.0)
        return x, rep
    it = 0
    best = np.inf
    while it < max_iter:
        r = b - A @ x
        beta = np.linalg.norm(r)
        if beta <= rtol * nb:
            rep.update(converged=True)
            break
        if beta >= best * (1 - 1e-12) and it > 0:
            rep.update(status="stagnation")
            break
        best = min(best, beta)
        m = restart
        V = np.zeros((m + 1, n)); H = np.zeros((m + 1, m))
        cs = np.zeros(m); sn = np.zeros(m); g = np.zeros(m + 1)
        V[0] = r / beta
        g[0] = beta
        k = 0
        for k in range(m):
            w = A @ (dinv * V[k])
            for j in range(k + 1):
                H[j, k] = w @ V[j]
                w = w - H[j, k] * V[j]
            H[k + 1, k] = np.linalg.norm(w)
            if H[k + 1, k] > 0:
                V[k + 1] = w / H[k + 1, k]
            for j in range(k):
                t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = t
            den = math.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / den
            sn[k] = H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            it += 1
            if abs(g[k + 1]) <= rtol * nb or H[k, k] == 0 or it >= max_iter:
                break
        kk = k + 1
        y = np.linalg.solve(np.triu(H[:kk, :kk]), g[:kk])
        x = x + dinv * (V[:kk].T @ y)
    rep.update(iterations=it, rel_res_true=_true_rel(A, x, b, nb))
    if rep["rel_res_true"] <= rtol:
        rep.update(converged=True)
    return x, rep
