"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no mesh connectivity, no
geometry of the scheme, no local blocks, no elimination). It only produces the
raw inputs a user of the method would hand to it:

* vertex coordinates and cell->vertex tables of structured simplicial meshes
  (stand-ins for the paper's external FVCA "Mesh1" family, and
  for the Kuhn 6-tetrahedra cube split);
* cell-averaged forces ``fbar[nc][d]`` ("1/|K| int_K f", PAPER.md L300 eq.
  defrhs), computed from a manufactured solution with a degree-2 rule;
* i.i.d. N(0,1) forces (config 3) and a seeded discretely divergence-free
  Navier-Stokes iterate (config 4), both per (cell, local face).

Randomness is counter based (splitmix64 over (seed, stream, index)), so any
consumer can regenerate any entry independently.

Per-(cell, local face) layout: local face ``s`` of a cell is the face opposite
its local vertex ``s`` (the ABI convention, include/cr.h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "splitmix64", "uniform01", "normal01",
    "square_mesh", "cube_mesh",
    "manufactured_2d", "manufactured_3d", "cell_average",
    "gaussian_force", "ns_iterate_2d", "lid_dirichlet_2d",
    "Config", "CONFIGS", "make_inputs",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """splitmix64 finaliser of (x + golden gamma), vectorised over uint64."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _counter(seed: int, stream: int, index):
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        k = splitmix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ splitmix64(np.uint64(stream)))
        return splitmix64(k ^ idx)


def uniform01(seed: int, stream: int, index) -> np.ndarray:
    """U[0,1): top 53 bits of the counter hash times 2^-53."""
    h = _counter(seed, stream, index)
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal01(seed: int, stream: int, index) -> np.ndarray:
    """N(0,1) by Box-Muller on two counter streams (2*stream, 2*stream+1)."""
    u1 = uniform01(seed, 2 * stream, index)
    u2 = uniform01(seed, 2 * stream + 1, index)
    u1 = 1.0 - u1  # (0, 1]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


# ----------------------------------------------------------------------------- meshes

def square_mesh(n: int, jitter: float = 0.0, seed: int = 0, flip_seed: int | None = None):
    """Unit square, n x n squares, each split along a diagonal into two triangles.

    vertex (i, j) -> j*(n+1)+i ; square (i, j) -> cells 2(jn+i) and 2(jn+i)+1.
    Default (``flip_seed`` None, SPEC.md L38 layout): every square is split along its
    lower-left -> upper-right diagonal: {(i,j),(i+1,j),(i+1,j+1)}, {(i,j),(i+1,j+1),(i,j+1)}.
    ``flip_seed`` given: each square independently (counter-based coin of stream 21) takes
    the other diagonal, {(i,j),(i+1,j),(i,j+1)}, {(i+1,j),(i+1,j+1),(i,j+1)} — an
    unstructured-topology stand-in for the paper's Mesh1 family: interior vertex
    valences then range over 4..8 instead of a fixed 6.
    ``jitter`` is the amplitude relative to h: interior vertices move by independent
    U(-jitter*h, jitter*h) per coordinate (BASELINE.json configs[2] "up to 0.2h").
    Returns coords [nv,2] f64, cells [nc,3] i32.
    """
    h = 1.0 / n
    j, i = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    coords = np.stack([i.ravel() * h, j.ravel() * h], axis=1).astype(np.float64)
    # exact endpoints
    coords[i.ravel() == n, 0] = 1.0
    coords[j.ravel() == n, 1] = 1.0
    if jitter > 0.0:
        vid = np.arange((n + 1) ** 2, dtype=np.uint64)
        interior = (i.ravel() > 0) & (i.ravel() < n) & (j.ravel() > 0) & (j.ravel() < n)
        for c in range(2):
            dx = (2.0 * uniform01(seed, c, vid) - 1.0) * (jitter * h)
            coords[interior, c] += dx[interior]
    sj, si = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    si = si.ravel(); sj = sj.ravel()
    v00 = sj * (n + 1) + si
    v10 = v00 + 1
    v11 = v00 + (n + 1) + 1
    v01 = v00 + (n + 1)
    cells = np.empty((2 * n * n, 3), dtype=np.int32)
    cells[0::2] = np.stack([v00, v10, v11], axis=1)
    cells[1::2] = np.stack([v00, v11, v01], axis=1)
    if flip_seed is not None:
        flip = uniform01(flip_seed, 21, np.arange(n * n, dtype=np.uint64)) < 0.5
        cells[0::2][flip] = np.stack([v00, v10, v01], axis=1)[flip]
        cells[1::2][flip] = np.stack([v10, v11, v01], axis=1)[flip]
    return coords, cells


_PERMS3 = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def cube_mesh(n: int, flip_seed: int | None = None, jitter: float = 0.0, seed: int = 0):
    """Unit cube, n^3 cubes, each split into the 6 Kuhn tetrahedra sharing a main
    diagonal ("splitting in 6 tetrahedra each cube").

    vertex (i,j,k) -> (k(n+1)+j)(n+1)+i ; cube (i,j,k) -> tets 6(kn^2+jn+i)+p for the
    axis permutations p in lexicographic order; tet vertices: corner, corner+e_p0,
    corner+e_p0+e_p1, corner+e_p0+e_p1+e_p2 (corner = the cube's lowest vertex).
    ``flip_seed`` given: the Kuhn split of cube (i,j,k) is mirrored in x iff bx[i], in y iff
    by[j], in z iff bz[k] (counter-based coins, streams 31..33) — i.e. it runs along one of
    the 4 main diagonals.  The triangulation a cube induces on a square face depends only
    on the mirror bits of the two axes spanning that face, which the neighbour across the
    face shares, so the mesh stays conforming while edge valences vary (an unstructured
    stand-in, as in ``square_mesh``).  ``jitter``: interior vertices move by independent
    U(-jitter*h, jitter*h) per coordinate (seed ``seed``, streams 0..2).
    """
    h = 1.0 / n
    k, j, i = np.meshgrid(np.arange(n + 1), np.arange(n + 1), np.arange(n + 1), indexing="ij")
    coords = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], axis=1).astype(np.float64)
    for c, g in enumerate((i, j, k)):
        coords[g.ravel() == n, c] = 1.0
    if jitter > 0.0:
        vid = np.arange((n + 1) ** 3, dtype=np.uint64)
        interior = np.ones(vid.shape, dtype=bool)
        for g in (i, j, k):
            interior &= (g.ravel() > 0) & (g.ravel() < n)
        for c in range(3):
            dx = (2.0 * uniform01(seed, c, vid) - 1.0) * (jitter * h)
            coords[interior, c] += dx[interior]
    ck, cj, ci = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    ci = ci.ravel(); cj = cj.ravel(); ck = ck.ravel()
    stride = (1, n + 1, (n + 1) ** 2)
    if flip_seed is None:
        mir = [np.zeros(ci.shape, dtype=np.int64)] * 3
    else:
        line = np.arange(n, dtype=np.uint64)
        mir = [(uniform01(flip_seed, 31 + a, line) < 0.5).astype(np.int64)[g]
               for a, g in enumerate((ci, cj, ck))]
    # start corner of the (possibly mirrored) diagonal; steps of -1 along mirrored axes
    corner = ((ck + mir[2]) * (n + 1) + (cj + mir[1])) * (n + 1) + (ci + mir[0])
    step = [stride[a] * (1 - 2 * mir[a]) for a in range(3)]
    cells = np.empty((6 * n ** 3, 4), dtype=np.int32)
    for p, perm in enumerate(_PERMS3):
        v0 = corner
        v1 = v0 + step[perm[0]]
        v2 = v1 + step[perm[1]]
        v3 = v2 + step[perm[2]]
        cells[p::6] = np.stack([v0, v1, v2, v3], axis=1)
    return coords, cells


# ----------------------------------------------------------------------------- data

def manufactured_2d(mu: float, nu: float):
    """2D manufactured Stokes solution (BASELINE.json configs[0]: stream function
    sin^2(pi x) sin^2(pi y), pressure cos(pi x)cos(pi y)).  Returns (u, p, f) callables
    of x [.., 2]; f = mu u - nu Lap u + grad p."""
    pi = math.pi

    def u(x):
        X, Y = x[..., 0], x[..., 1]
        return np.stack([pi * np.sin(pi * X) ** 2 * np.sin(2 * pi * Y),
                         -pi * np.sin(2 * pi * X) * np.sin(pi * Y) ** 2], axis=-1)

    def p(x):
        return np.cos(pi * x[..., 0]) * np.cos(pi * x[..., 1])

    def f(x):
        X, Y = x[..., 0], x[..., 1]
        uu = u(x)
        f1 = mu * uu[..., 0] - 2 * nu * pi ** 3 * np.sin(2 * pi * Y) * (2 * np.cos(2 * pi * X) - 1) \
            - pi * np.sin(pi * X) * np.cos(pi * Y)
        f2 = mu * uu[..., 1] + 2 * nu * pi ** 3 * np.sin(2 * pi * X) * (2 * np.cos(2 * pi * Y) - 1) \
            - pi * np.cos(pi * X) * np.sin(pi * Y)
        return np.stack([f1, f2], axis=-1)

    return u, p, f


def manufactured_3d(mu: float, nu: float):
    """3D manufactured Stokes solution u = curl(psi, psi, psi), psi = s(x)s(y)s(z),
    s(t) = sin^2(pi t); p = cos(pi x)cos(pi y)cos(pi z).  (BASELINE.json configs[4]
    "manufactured smooth solution"; reading in DESIGN.md.)"""
    pi = math.pi
    s = lambda t: np.sin(pi * t) ** 2
    s1 = lambda t: pi * np.sin(2 * pi * t)
    s2 = lambda t: 2 * pi ** 2 * np.cos(2 * pi * t)
    s3 = lambda t: -4 * pi ** 3 * np.sin(2 * pi * t)

    def grad_psi(X, Y, Z):
        return (s1(X) * s(Y) * s(Z), s(X) * s1(Y) * s(Z), s(X) * s(Y) * s1(Z))

    def lap_grad_psi(X, Y, Z):
        lx = s3(X) * s(Y) * s(Z) + s1(X) * s2(Y) * s(Z) + s1(X) * s(Y) * s2(Z)
        ly = s2(X) * s1(Y) * s(Z) + s(X) * s3(Y) * s(Z) + s(X) * s1(Y) * s2(Z)
        lz = s2(X) * s(Y) * s1(Z) + s(X) * s2(Y) * s1(Z) + s(X) * s(Y) * s3(Z)
        return lx, ly, lz

    def u(x):
        px, py, pz = grad_psi(x[..., 0], x[..., 1], x[..., 2])
        return np.stack([py - pz, pz - px, px - py], axis=-1)

    def p(x):
        return np.cos(pi * x[..., 0]) * np.cos(pi * x[..., 1]) * np.cos(pi * x[..., 2])

    def f(x):
        X, Y, Z = x[..., 0], x[..., 1], x[..., 2]
        lx, ly, lz = lap_grad_psi(X, Y, Z)
        lap_u = np.stack([ly - lz, lz - lx, lx - ly], axis=-1)
        gp = np.stack([-pi * np.sin(pi * X) * np.cos(pi * Y) * np.cos(pi * Z),
                       -pi * np.cos(pi * X) * np.sin(pi * Y) * np.cos(pi * Z),
                       -pi * np.cos(pi * X) * np.cos(pi * Y) * np.sin(pi * Z)], axis=-1)
        return mu * u(x) - nu * lap_u + gp

    return u, p, f


def cell_average(func, coords: np.ndarray, cells: np.ndarray) -> np.ndarray:
    """Cell average (1/|K|) int_K func by the degree-2 vertex+centroid rule
    (2D: 1/12 per vertex + 3/4 at the centroid; 3D: 1/20 per vertex + 4/5 at the
    centroid; both exact for quadratics).  Returns [nc, d]."""
    d = cells.shape[1] - 1
    wv, wc = (1.0 / 12.0, 0.75) if d == 2 else (1.0 / 20.0, 0.8)
    X = coords[cells]                      # [nc, d+1, d]
    cen = X.mean(axis=1)
    out = wc * func(cen)
    for v in range(d + 1):
        out = out + wv * func(X[:, v, :])
    return np.ascontiguousarray(out, dtype=np.float64)


def gaussian_force(nc: int, d: int, seed: int) -> np.ndarray:
    """f_K ~ N(0,1) i.i.d. per cell and component (BASELINE.json configs[2])."""
    idx = np.arange(nc * d, dtype=np.uint64)
    return normal01(seed, 7, idx).reshape(nc, d).astype(np.float64)


def _local_faces(cells):
    d = cells.shape[1] - 1
    out = []
    for s in range(d + 1):
        others = [c for c in range(d + 1) if c != s]
        out.append(np.sort(cells[:, others], axis=1))
    return np.stack(out, axis=1)           # [nc, d+1, d] sorted vertex tuples


def lid_dirichlet_2d(coords: np.ndarray, cells: np.ndarray, lid=(1.0, 0.0)) -> np.ndarray:
    """Per (cell, local face) Dirichlet values: ``lid`` on faces lying on y = 1, zero
    elsewhere (BASELINE.json configs[3]).  Only boundary faces are read."""
    lf = _local_faces(cells)
    y = coords[:, 1]
    top = (y[lf[..., 0]] == 1.0) & (y[lf[..., 1]] == 1.0)
    out = np.zeros(lf.shape[:2] + (2,), dtype=np.float64)
    out[top] = np.asarray(lid, dtype=np.float64)
    return out


def ns_iterate_2d(coords: np.ndarray, cells: np.ndarray, n: int, seed: int,
                  lid=(1.0, 0.0)) -> np.ndarray:
    """Seeded discretely divergence-free 2D velocity per (cell, local face):
    psi_v ~ U(-1/2,1/2)/n at interior vertices (0 on the boundary); on an edge
    a<b: U = (psi_b - psi_a)/|e| * n_right(a->b) + beta_e * t(a->b),
    beta_e ~ U(-1/2,1/2) keyed by (a, b).  Faces on the boundary carry the
    wall/lid value (``lid`` on y = 1, zero elsewhere).  Both cells of an edge get
    the same value (it is a function of the vertex pair only)."""
    nv = coords.shape[0]
    x, y = coords[:, 0], coords[:, 1]
    bnd_v = (x == 0.0) | (x == 1.0) | (y == 0.0) | (y == 1.0)
    psi = (uniform01(seed, 11, np.arange(nv, dtype=np.uint64)) - 0.5) / n
    psi[bnd_v] = 0.0
    lf = _local_faces(cells)
    a, b = lf[..., 0].astype(np.int64), lf[..., 1].astype(np.int64)
    e = coords[b] - coords[a]
    L = np.sqrt(e[..., 0] ** 2 + e[..., 1] ** 2)
    t = e / L[..., None]
    nr = np.stack([t[..., 1], -t[..., 0]], axis=-1)
    beta = uniform01(seed, 12, (a * nv + b).astype(np.uint64)) - 0.5
    U = ((psi[b] - psi[a]) / L)[..., None] * nr + beta[..., None] * t
    on_bnd = bnd_v[a] & bnd_v[b] & (
        ((x[a] == 0) & (x[b] == 0)) | ((x[a] == 1) & (x[b] == 1)) |
        ((y[a] == 0) & (y[b] == 0)) | ((y[a] == 1) & (y[b] == 1)))
    U[on_bnd] = 0.0
    top = on_bnd & (y[a] == 1.0) & (y[b] == 1.0)
    U[top] = np.asarray(lid, dtype=np.float64)
    return np.ascontiguousarray(U)


# ----------------------------------------------------------------------------- configs

@dataclass
class Config:
    """One BASELINE.json config (0-based index ``idx``)."""
    idx: int
    dim: int
    n: int
    jitter: float
    mu: float
    nu: float
    physics: str          # "stokes" | "ns_step"
    shift: str            # "none" | "mis"
    force: str            # "manufactured" | "gaussian" | "zero"
    solver: str           # "pcg" | "minres" | "bicgstab" | "gmres"
    seed: int = 0
    mis_seed: int = 0
    rtol: float = 1e-10
    extra: dict = field(default_factory=dict)


CONFIGS = {
    0: Config(0, 2, 8, 0.0, 1.0, 1.0, "stokes", "none", "manufactured", "pcg"),
    1: Config(1, 2, 1024, 0.2, 1.0, 1.0, "stokes", "none", "manufactured", "pcg", seed=2),
    2: Config(2, 2, 1024, 0.2, 0.0, 1.0, "stokes", "mis", "gaussian", "minres", seed=2,
              mis_seed=33, extra={"force_seed": 3}),
    3: Config(3, 2, 512, 0.0, 0.0, 0.01, "ns_step", "mis", "zero", "bicgstab", seed=4,
              mis_seed=44),
    4: Config(4, 3, 128, 0.0, 1.0, 1.0, "stokes", "none", "manufactured", "pcg"),
}


def make_inputs(cfg: Config, n: int | None = None) -> dict:
    """Materialise the raw inputs of ``cfg`` (optionally at another mesh size n,
    used for the small parity cases).  Returns dict with coords, cells, fbar,
    dirichlet (per cell-local face or None), u_iter (NS, per cell-local face or None)."""
    n = cfg.n if n is None else n
    if cfg.dim == 2:
        coords, cells = square_mesh(n, cfg.jitter, cfg.seed)
    else:
        coords, cells = cube_mesh(n)
    nc, d = cells.shape[0], cfg.dim
    out = {"coords": coords, "cells": cells, "dirichlet": None, "u_iter": None}
    if cfg.force == "manufactured":
        _, _, f = (manufactured_2d if d == 2 else manufactured_3d)(cfg.mu, cfg.nu)
        out["fbar"] = cell_average(f, coords, cells)
    elif cfg.force == "gaussian":
        out["fbar"] = gaussian_force(nc, d, cfg.extra.get("force_seed", cfg.seed))
    else:
        out["fbar"] = np.zeros((nc, d), dtype=np.float64)
    if cfg.physics == "ns_step":
        out["u_iter"] = ns_iterate_2d(coords, cells, n, cfg.seed)
    return out
