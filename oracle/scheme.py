"""ORACLE (test infrastructure only) — C-2..C-5, C-7: local blocks, shift E_K,
coupled assembly, hybridisation, recovery.  Follows PAPER.md §3.

Per-cell arithmetic (S_K, A_K, D_K, R_K, Ahat_K^{-1}, B_K, G_K, S_K, recovery) is
done in binary128 by ``cell_f128.c``; this module only gathers per-cell inputs
and scatters with the paper's maps H_K, F_K, Hhat_K.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .mesh import Mesh

_dp = ctypes.POINTER(ctypes.c_double)


def _p(x):
    if x is None:
        return None
    return x.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Params:
    """mu = 1/dt (transient) or 0 (steady), nu = 1/Re."""
    mu: float = 1.0
    nu: float = 1.0
    physics: str = "stokes"       # "stokes" | "ns_step"
    shift: str = "none"           # "none" (mu > 0, E = 0) | "mis"
    mis_seed: int = 0
    lambda_factor: float = 1.1
    k0: int = 0                   # gauge cell K0


@dataclass
class Data:
    fbar: np.ndarray                     # [nc, d] cell-averaged force
    dirichlet: np.ndarray | None = None  # [nc, d+1, d] per local face (boundary faces read)
    u_iter: np.ndarray | None = None     # [nc, d+1, d] NS Newton iterate (all faces)
    p_iter: np.ndarray | None = None     # [nc]


def cell_arrays(m: Mesh, data: Data) -> dict:
    """Per-cell fp64 inputs of the local algebra."""
    f64 = lambda x: None if x is None else np.ascontiguousarray(x, dtype=np.float64)
    return dict(
        a=f64(m.a), vol=f64(m.vol), xK=f64(m.xK),
        xs=f64(m.xs[m.cell_faces]),
        intr=np.ascontiguousarray(m.interior_local.astype(np.int8)),
        fbar=f64(data.fbar), dir=f64(data.dirichlet), uit=f64(data.u_iter),
        pit=f64(data.p_iter),
    )


def _lib():
    from . import lib
    return lib()


def local_blocks(m: Mesh, prm: Params, data: Data):
    """A_K, R_K, D_K (interior-restricted, [(d+1)d] local indexing) and g_K.
    P:L261-306 (+ Dirichlet fold / NS increment form, DESIGN.md readings)."""
    d, nc = m.dim, m.nc
    n = (d + 1) * d
    c = cell_arrays(m, data)
    A = np.zeros((nc, n, n)); R = np.zeros((nc, n)); D = np.zeros((nc, n)); g = np.zeros(nc)
    _lib().or_cell_blocks(
        ctypes.c_int(d), ctypes.c_int64(nc), ctypes.c_double(prm.mu), ctypes.c_double(prm.nu),
        ctypes.c_int(prm.physics == "ns_step"),
        _p(c["a"]), _p(c["vol"]), _p(c["xK"]), _p(c["xs"]), _p(c["intr"]), _p(c["fbar"]),
        _p(c["dir"]), _p(c["uit"]), _p(c["pit"]), _p(A), _p(R), _p(D), _p(g))
    return A, R, D, g


def _splitmix64(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def mis_priority(nc: int, seed: int) -> np.ndarray:
    """priority(K) = splitmix64(seed xor K) (reading of P:L539 "partitioning")."""
    return _splitmix64(np.uint64(seed) ^ np.arange(nc, dtype=np.uint64))


def mis_greedy(m: Mesh, seed: int) -> np.ndarray:
    """M_1 = greedy maximal independent set of the face-adjacency graph, visiting cells
    in ascending (priority, K) order (M_2 = all neighbours of M_1)."""
    nc = m.nc
    pr = mis_priority(nc, seed)
    order = np.lexsort((np.arange(nc), pr))
    fc = m.face_cells[m.face_cells[:, 1] >= 0]
    nbr = [[] for _ in range(nc)]
    for K, L in fc.tolist():
        nbr[K].append(L)
        nbr[L].append(K)
    inM1 = np.zeros(nc, dtype=bool)
    blocked = np.zeros(nc, dtype=bool)
    for K in order.tolist():
        if blocked[K]:
            continue
        inM1[K] = True
        for L in nbr[K]:
            blocked[L] = True
    return inM1


def shift_E(m: Mesh, prm: Params, A: np.ndarray):
    """E_K per (cell, local face).  mu > 0: E = 0.  Otherwise
    E_K = -lambda_K I on M_1 cells, +lambda_L on an M_2 face shared with L in M_1, 0 else;
    lambda_K = lambda_factor * max row sum |A_K| (Gershgorin bound > all eigenvalues)."""
    nc, d = m.nc, m.dim
    if prm.shift == "none":
        return np.zeros((nc, d + 1)), np.zeros(nc, dtype=bool), np.zeros(nc)
    inM1 = mis_greedy(m, prm.mis_seed)
    lam = prm.lambda_factor * np.abs(A).sum(axis=2).max(axis=1)
    E = np.zeros((nc, d + 1))
    intr = m.interior_local
    E[inM1] = -lam[inM1, None]
    E[~intr] = 0.0
    other = np.where(m.face_cells[m.cell_faces, 0] == np.arange(nc)[:, None],
                     m.face_cells[m.cell_faces, 1], m.face_cells[m.cell_faces, 0])
    for K in np.nonzero(~inM1)[0]:
        for s in range(d + 1):
            L = other[K, s]
            if intr[K, s] and L >= 0 and inM1[L]:
                E[K, s] = lam[L]
    return E, inM1, lam


def _gidx(m: Mesh):
    """Global unknown of local (l, i): d * face_dof(cell_faces[K, l]) + i (-1 boundary)."""
    d = m.dim
    dof = m.face_dof[m.cell_faces]                            # [nc, d+1]
    gi = dof[:, :, None] * d + np.arange(d)[None, None, :]
    gi[dof < 0] = -1
    return gi.reshape(m.nc, -1)                               # [nc, (d+1)d]


def _scatter_matrix(gi, blocks, N):
    """sum_K H_K X_K H_K^t over interior entries."""
    nc, n = gi.shape
    r = np.repeat(gi, n, axis=1).ravel()
    c = np.tile(gi, (1, n)).ravel()
    v = blocks.reshape(nc, n * n).ravel()
    keep = (r >= 0) & (c >= 0)
    return sp.coo_matrix((v[keep], (r[keep], c[keep])), shape=(N, N)).tocsr()


def _scatter_vector(gi, vecs, N):
    out = np.zeros(N)
    keep = gi >= 0
    np.add.at(out, gi[keep], vecs[keep])
    return out


def assemble_coupled(m: Mesh, prm: Params, data: Data):
    """Coupled system eq. (syslin): returns (M, rhs, nU) with
    M = [[A, D^t], [D, 0]], rhs = [R; g]; pressure unknowns P_K, K != K0, in
    increasing K."""
    d = m.dim
    A_K, R_K, D_K, g_K = local_blocks(m, prm, data)
    nU = d * m.nf_int
    gi = _gidx(m)
    A = _scatter_matrix(gi, A_K, nU)
    R = _scatter_vector(gi, R_K, nU)
    cellsP = np.array([K for K in range(m.nc) if K != prm.k0], dtype=np.int64)
    rows, cols, vals = [], [], []
    for pi, K in enumerate(cellsP):
        sel = gi[K] >= 0
        rows.append(np.full(sel.sum(), pi)); cols.append(gi[K][sel]); vals.append(D_K[K][sel])
    D = sp.coo_matrix((np.concatenate(vals) if vals else np.zeros(0),
                       (np.concatenate(rows) if rows else np.zeros(0, int),
                        np.concatenate(cols) if cols else np.zeros(0, int))),
                      shape=(len(cellsP), nU)).tocsr()
    M = sp.bmat([[A, D.T], [D, None]], format="csr")
    M.sort_indices()
    rhs = np.concatenate([R, g_K[cellsP]])
    return M, rhs, nU


def _elim_call(fn, m, prm, data, E, extra_in=(), extra_out=()):
    c = cell_arrays(m, data)
    E = np.ascontiguousarray(E, dtype=np.float64)
    cs = np.ascontiguousarray(m.csign)
    return fn(ctypes.c_int(m.dim), ctypes.c_int64(m.nc), ctypes.c_double(prm.mu),
              ctypes.c_double(prm.nu), ctypes.c_int(prm.physics == "ns_step"),
              _p(c["a"]), _p(c["vol"]), _p(c["xK"]), _p(c["xs"]), _p(c["intr"]), _p(c["fbar"]),
              _p(c["dir"]), _p(c["uit"]), _p(c["pit"]), _p(E), _p(cs), ctypes.c_int64(prm.k0),
              *[_p(x) for x in extra_in], *[_p(x) for x in extra_out])


class LocalFailure(RuntimeError):
    pass


def hybridise(m: Mesh, prm: Params, data: Data):
    """G and S of G W = S: G = sum_K H_K G_K H_K^t.
    Returns dict(G csr, S, E, inM1, B, G_loc, S_loc)."""
    d = m.dim
    n = (d + 1) * d
    A_K, _, _, _ = local_blocks(m, prm, data)
    E, inM1, lam = shift_E(m, prm, A_K)
    G_loc = np.zeros((m.nc, n, n)); S_loc = np.zeros((m.nc, n)); B = np.zeros(m.nc)
    status = np.zeros(m.nc, dtype=np.int32)
    from . import lib
    nbad = _elim_call(lib().or_cell_eliminate, m, prm, data, E,
                      extra_out=(G_loc, S_loc, B, status))
    if nbad:
        raise LocalFailure(f"{nbad} cells failed local elimination (status {np.unique(status)})")
    gi = _gidx(m)
    N = d * m.nf_int
    G = _scatter_matrix(gi, G_loc, N)
    G.sort_indices()
    S = _scatter_vector(gi, S_loc, N)
    return dict(G=G, S=S, E=E, inM1=inM1, lam=lam, B=B, G_loc=G_loc, S_loc=S_loc)


def recover(m: Mesh, prm: Params, data: Data, E: np.ndarray, W: np.ndarray):
    """P and U from W; U_sigma taken from the copy of
    face_cells[sigma][0] ("this common value").  Returns (U [nf_int, d],
    P [nc], Uhat [nc, d+1, d], max copy disagreement)."""
    d = m.dim
    n = (d + 1) * d
    gi = _gidx(m)
    Wl = np.where(gi >= 0, W[np.maximum(gi, 0)], 0.0)
    Wl = np.ascontiguousarray(Wl)
    P = np.zeros(m.nc); Uh = np.zeros((m.nc, n)); status = np.zeros(m.nc, dtype=np.int32)
    from . import lib
    nbad = _elim_call(lib().or_cell_recover, m, prm, data, E, extra_in=(Wl,),
                      extra_out=(P, Uh, status))
    if nbad:
        raise LocalFailure(f"{nbad} cells failed recovery")
    Uh = Uh.reshape(m.nc, d + 1, d)
    dofs = m.dof_face
    K0 = m.face_cells[dofs, 0]
    K1 = m.face_cells[dofs, 1]
    l0 = np.argmax(m.cell_faces[K0] == dofs[:, None], axis=1)
    l1 = np.argmax(m.cell_faces[K1] == dofs[:, None], axis=1)
    U = Uh[K0, l0]
    U1 = Uh[K1, l1]
    disagree = float(np.max(np.abs(U - U1))) if len(dofs) else 0.0
    return U, P, Uh, disagree


def _subset_call(fn, m, prm, data, E, cells, extra_in=(), extra_out=()):
    c = cell_arrays(m, data)
    cells = np.asarray(cells, dtype=np.int64)
    sub = {k: (None if v is None else np.ascontiguousarray(v[cells])) for k, v in c.items()}
    Es = np.ascontiguousarray(np.asarray(E, dtype=np.float64)[cells])
    cs = np.ascontiguousarray(m.csign[cells])
    hit = np.nonzero(cells == prm.k0)[0]
    k0 = int(hit[0]) if len(hit) else -1
    return fn(ctypes.c_int(m.dim), ctypes.c_int64(len(cells)), ctypes.c_double(prm.mu),
              ctypes.c_double(prm.nu), ctypes.c_int(prm.physics == "ns_step"),
              _p(sub["a"]), _p(sub["vol"]), _p(sub["xK"]), _p(sub["xs"]), _p(sub["intr"]), _p(sub["fbar"]),
              _p(sub["dir"]), _p(sub["uit"]), _p(sub["pit"]), _p(Es), _p(cs), ctypes.c_int64(k0),
              *[_p(x) for x in extra_in], *[_p(x) for x in extra_out])


def eliminate_cells(m: Mesh, prm: Params, data: Data, E: np.ndarray, cells):
    """G_K, S_K, B_K of a SUBSET of cells (same binary128 algebra as ``hybridise``), for
    sampled parity checks at sizes where the full oracle is too slow."""
    from . import lib
    n = (m.dim + 1) * m.dim
    k = len(cells)
    G = np.zeros((k, n, n)); S = np.zeros((k, n)); B = np.zeros(k); st = np.zeros(k, dtype=np.int32)
    nbad = _subset_call(lib().or_cell_eliminate, m, prm, data, E, cells, extra_out=(G, S, B, st))
    if nbad:
        raise LocalFailure(f"{nbad} cells failed local elimination")
    return G, S, B


def recover_cells(m: Mesh, prm: Params, data: Data, E: np.ndarray, W: np.ndarray, cells):
    """P_K and Uhat_K of a SUBSET of cells given W."""
    from . import lib
    d = m.dim
    n = (d + 1) * d
    cells = np.asarray(cells, dtype=np.int64)
    gi = _gidx(m)[cells]
    Wl = np.ascontiguousarray(np.where(gi >= 0, W[np.maximum(gi, 0)], 0.0))
    k = len(cells)
    P = np.zeros(k); Uh = np.zeros((k, n)); st = np.zeros(k, dtype=np.int32)
    nbad = _subset_call(lib().or_cell_recover, m, prm, data, E, cells, extra_in=(Wl,), extra_out=(P, Uh, st))
    if nbad:
        raise LocalFailure(f"{nbad} cells failed recovery")
    return P, Uh.reshape(k, d + 1, d)


def hybrid_pipeline(m: Mesh, prm: Params, data: Data, solve=None):
    """The paper's 'hybrid method': (1) G, S; (2) solve G W = S;
    (3) recover P, U.  ``solve`` defaults to the refined direct solve."""
    from .krylov import direct_refined
    h = hybridise(m, prm, data)
    if solve is None:
        W = direct_refined(h["G"], h["S"])
    else:
        W = solve(h["G"], h["S"])
    U, P, Uh, dis = recover(m, prm, data, h["E"], W)
    h.update(W=W, U=U, P=P, Uhat=Uh, disagree=dis)
    return h
