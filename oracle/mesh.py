"""ORACLE (test infrastructure only) — C-1: simplicial mesh, faces, geometry.

Follows PAPER.md §2 item 1: faces F = F_int u F_ext, F_K, M_sigma,
x_K (centre of gravity), x_sigma, a_{K,sigma} = |sigma| n_{K,sigma} (outward).

Conventions:
* face identity = sorted vertex tuple; faces numbered in lexicographic order of
  that tuple; ``face_cells[f] = (lower cell, higher cell)`` (-1 if boundary);
* local face s of a cell = the face opposite its local vertex s;
* interior face dof = rank among interior faces in face order;
* a_{K,s} is computed from the face's sorted vertex tuple (p, q[, r]) and then
  signed to point away from the opposite vertex.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class MeshError(ValueError):
    pass


@dataclass
class Mesh:
    dim: int
    coords: np.ndarray      # [nv, d] f64
    cells: np.ndarray       # [nc, d+1] i32
    faces: np.ndarray       # [nf, d] i32 sorted tuples, lexicographic order
    face_cells: np.ndarray  # [nf, 2] i32, second = -1 on boundary faces
    cell_faces: np.ndarray  # [nc, d+1] i32, local s = face opposite local vertex s
    face_dof: np.ndarray    # [nf] i32, -1 on boundary faces
    vol: np.ndarray         # [nc] |K|
    xK: np.ndarray          # [nc, d]
    xs: np.ndarray          # [nf, d]
    a: np.ndarray           # [nc, d+1, d]

    @property
    def nc(self):
        return self.cells.shape[0]

    @property
    def nf(self):
        return self.faces.shape[0]

    @property
    def nf_int(self):
        return int((self.face_dof >= 0).sum())

    @property
    def dof_face(self):
        return np.nonzero(self.face_dof >= 0)[0].astype(np.int64)

    @property
    def interior_local(self):
        """[nc, d+1] bool: local face interior (P:L117 F_{K,int})."""
        return self.face_dof[self.cell_faces] >= 0

    @property
    def csign(self):
        """C_K diagonal: +1 on face_cells[f][0], -1 on the other cell."""
        own = self.face_cells[self.cell_faces, 0] == np.arange(self.nc)[:, None]
        return np.where(own, 1, -1).astype(np.int8)


def build_mesh(coords: np.ndarray, cells: np.ndarray) -> Mesh:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    nc, d1 = cells.shape
    d = d1 - 1
    if d not in (2, 3) or coords.shape[1] != d:
        raise MeshError("dimension must be 2 or 3")
    if nc and (cells.min() < 0 or cells.max() >= coords.shape[0]):
        raise MeshError("cell references a vertex out of range")

    # all (cell, local face) sorted vertex tuples; local face s = opposite vertex s
    loc = np.stack([np.sort(np.delete(cells, s, axis=1), axis=1) for s in range(d + 1)], axis=1)
    flat = loc.reshape(-1, d)
    order = np.lexsort(flat.T[::-1])         # stable; primary key = first vertex
    srt = flat[order]
    new = np.ones(len(srt), dtype=bool)
    if len(srt) > 1:
        new[1:] = np.any(srt[1:] != srt[:-1], axis=1)
    fid_sorted = np.cumsum(new) - 1
    nf = int(fid_sorted[-1]) + 1 if len(srt) else 0
    runlen = np.bincount(fid_sorted, minlength=nf)
    if np.any(runlen > 2):
        raise MeshError("non-manifold input: a face shared by more than two cells")
    faces = srt[new].astype(np.int32)
    cell_faces = np.empty(nc * (d + 1), dtype=np.int32)
    cell_faces[order] = fid_sorted
    cell_faces = cell_faces.reshape(nc, d + 1)
    owner = (order // (d + 1)).astype(np.int32)   # cell of each sorted entry
    face_cells = np.full((nf, 2), -1, dtype=np.int32)
    first = np.nonzero(new)[0]
    face_cells[:, 0] = owner[first]
    second = np.nonzero(~new)[0]
    face_cells[fid_sorted[second], 1] = owner[second]
    interior = face_cells[:, 1] >= 0
    face_dof = np.full(nf, -1, dtype=np.int32)
    face_dof[interior] = np.arange(int(interior.sum()), dtype=np.int32)

    X = coords[cells]                                   # [nc, d+1, d]
    E = X[:, 1:, :] - X[:, :1, :]
    det = np.linalg.det(E) if nc else np.zeros(0)
    vol = np.abs(det) / (2.0 if d == 2 else 6.0)
    edges = [np.linalg.norm(X[:, i] - X[:, j], axis=1) for i in range(d + 1) for j in range(i)]
    hmax = np.max(np.stack(edges, axis=1), axis=1) if nc else np.zeros(0)
    if np.any(vol <= 1e-14 * hmax ** d):
        raise MeshError("degenerate cell")
    xK = X.sum(axis=1) / (d + 1)
    FX = coords[faces]                                  # [nf, d, d]
    xs = FX.sum(axis=1) / d

    # a_{K,s}: from the sorted tuple of local face s, signed away from vertex s
    a = np.empty((nc, d + 1, d))
    for s in range(d + 1):
        P = coords[loc[:, s, 0]]
        Qv = coords[loc[:, s, 1]]
        if d == 2:
            e = Qv - P
            nvec = np.stack([e[:, 1], -e[:, 0]], axis=1)
        else:
            Rv = coords[loc[:, s, 2]]
            nvec = 0.5 * np.cross(Qv - P, Rv - P)
        opp = X[:, s, :]
        sgn = np.where(np.einsum("ij,ij->i", nvec, P - opp) < 0, -1.0, 1.0)
        a[:, s, :] = nvec * sgn[:, None]
    return Mesh(d, coords, cells, faces, face_cells, cell_faces, face_dof, vol, xK, xs, a)
