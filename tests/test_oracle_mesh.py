"""Pins of oracle C-1 (mesh, faces, geometry) against
closed-form counts, hand-derived SPEC examples, brute-force enumeration and
geometric identities (divergence theorem)."""
import itertools
import math

import numpy as np
import pytest

import cr_inputs as ci
import oracle as O
from oracle.mesh import MeshError


def brute_faces(cells):
    """Independent face enumeration: dict of sorted tuple -> list of cells."""
    faces = {}
    for k, c in enumerate(cells.tolist()):
        for comb in itertools.combinations(sorted(c), len(c) - 1):
            faces.setdefault(comb, []).append(k)
    return faces


@pytest.mark.parametrize("n", range(1, 9))
def test_counts_2d_closed_form(n):
    m = O.build_mesh(*ci.square_mesh(n))
    assert m.nc == 2 * n * n
    assert m.coords.shape[0] == (n + 1) ** 2
    assert m.nf == 3 * n * n + 2 * n
    assert m.nf_int == 3 * n * n - 2 * n
    sK = m.interior_local.sum(1)
    hist = {s: int((sK == s).sum()) for s in (1, 2, 3)}
    assert hist == {1: 2, 2: 4 * n - 4, 3: 2 * (n - 1) ** 2}


@pytest.mark.parametrize("n", range(1, 5))
def test_counts_3d_closed_form(n):
    m = O.build_mesh(*ci.cube_mesh(n))
    assert m.nc == 6 * n ** 3
    assert m.nf == 12 * n ** 3 + 6 * n ** 2
    assert m.nf_int == 12 * n ** 3 - 6 * n ** 2
    sK = m.interior_local.sum(1)
    hist = {s: int((sK == s).sum()) for s in (1, 2, 3, 4)}
    assert hist == {1: 0, 2: 6 * n, 3: 12 * n * (n - 1), 4: 6 * n * (n - 1) ** 2}
    np.testing.assert_allclose(m.vol, 1.0 / (6 * n ** 3), rtol=1e-12)


def test_spec_examples_2d():
    m1 = O.build_mesh(*ci.square_mesh(1))
    assert (m1.nc, m1.nf, m1.nf_int) == (2, 5, 1)
    m2 = O.build_mesh(*ci.square_mesh(2))
    assert (m2.nc, m2.nf, m2.nf_int) == (8, 16, 8)
    # unit right triangle {(0,0),(1,0),(1,1)}: a-vectors (0,-1), (1,0), (-1,1)
    coords = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]])
    m = O.build_mesh(coords, np.array([[0, 1, 2]], dtype=np.int32))
    # local face s is opposite local vertex s
    np.testing.assert_array_equal(m.a[0, 2], [0.0, -1.0])
    np.testing.assert_array_equal(m.a[0, 0], [1.0, 0.0])
    np.testing.assert_array_equal(m.a[0, 1], [-1.0, 1.0])
    assert m.vol[0] == 0.5
    # grad phi = a/|K| = (-2, 2) on the diagonal face
    np.testing.assert_array_equal(m.a[0, 1] / m.vol[0], [-2.0, 2.0])


@pytest.mark.parametrize("maker", [lambda: ci.square_mesh(6, 0.2, seed=9), lambda: ci.cube_mesh(3)])
def test_connectivity_against_brute_force(maker):
    coords, cells = maker()
    m = O.build_mesh(coords, cells)
    bf = brute_faces(cells)
    keys = sorted(bf)                                  # lexicographic order
    assert m.nf == len(keys)
    np.testing.assert_array_equal(m.faces, np.array(keys, dtype=np.int32))
    for f, k in enumerate(keys):
        cl = bf[k]
        assert m.face_cells[f, 0] == cl[0]
        assert m.face_cells[f, 1] == (cl[1] if len(cl) == 2 else -1)
    d = cells.shape[1] - 1
    for K in range(len(cells)):
        for s in range(d + 1):
            t = tuple(sorted(np.delete(cells[K], s)))
            assert tuple(m.faces[m.cell_faces[K, s]]) == t
    dofs = m.face_dof[m.face_dof >= 0]
    np.testing.assert_array_equal(dofs, np.arange(m.nf_int))
    assert np.all(np.diff(np.nonzero(m.face_dof >= 0)[0]) > 0)


@pytest.mark.parametrize("maker", [lambda: ci.square_mesh(7, 0.2, seed=3), lambda: ci.cube_mesh(3)])
def test_geometric_identities(maker):
    coords, cells = maker()
    m = O.build_mesh(coords, cells)
    d = m.dim
    # closed surface: sum_s a_{K,s} = 0
    s = m.a.sum(1)
    assert np.abs(s).max() <= 1e-12 * np.abs(m.a).max()
    # a_{K,s} + a_{L,s} = 0 exactly (same sorted tuple, opposite sign)
    intr = m.face_dof >= 0
    f = np.nonzero(intr)[0]
    K, L = m.face_cells[f, 0], m.face_cells[f, 1]
    lK = np.argmax(m.cell_faces[K] == f[:, None], 1)
    lL = np.argmax(m.cell_faces[L] == f[:, None], 1)
    assert np.array_equal(m.a[K, lK], -m.a[L, lL])
    assert abs(m.vol.sum() - 1.0) < 1e-12
    # divergence theorem on x: sum_s a_{K,s} x_s^t = |K| I   (catches sign / scale / centroid errors)
    xsK = m.xs[m.cell_faces]
    T = np.einsum("ksi,ksj->kij", m.a, xsK)
    np.testing.assert_allclose(T, m.vol[:, None, None] * np.eye(d)[None], atol=1e-14)
    # outward: a_{K,s} . (x_s - x_K) > 0
    assert np.all(np.einsum("ksi,ksi->ks", m.a, xsK - m.xK[:, None, :]) > 0)
    # |a| = face measure computed independently
    X = coords[cells]
    for sl in range(d + 1):
        o = [v for v in range(d + 1) if v != sl]
        if d == 2:
            meas = np.linalg.norm(X[:, o[0]] - X[:, o[1]], axis=1)
        else:
            u1, u2 = X[:, o[1]] - X[:, o[0]], X[:, o[2]] - X[:, o[0]]
            g = np.einsum("ki,ki->k", u1, u1) * np.einsum("ki,ki->k", u2, u2) \
                - np.einsum("ki,ki->k", u1, u2) ** 2
            meas = 0.5 * np.sqrt(g)
        np.testing.assert_allclose(np.linalg.norm(m.a[:, sl], axis=1), meas, rtol=1e-13)
    # centroids are vertex means
    np.testing.assert_allclose(m.xK, X.mean(1), rtol=0, atol=1e-15)


def test_error_paths():
    coords, cells = ci.square_mesh(2)
    with pytest.raises(MeshError):
        O.build_mesh(coords, np.concatenate([cells, cells[:1]]))          # non-manifold
    bad = cells.copy(); bad[0, 2] = 999
    with pytest.raises(MeshError):
        O.build_mesh(coords, bad)
    col = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    with pytest.raises(MeshError):
        O.build_mesh(col, np.array([[0, 1, 2]], dtype=np.int32))          # degenerate
