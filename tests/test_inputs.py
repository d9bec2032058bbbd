"""Seeded input generators (cr_inputs): shapes, determinism, and the manufactured
forces checked by finite differences (independent of the generator's closed forms)."""
import numpy as np
import pytest

import cr_inputs as ci


def test_splitmix_reference_values():
    # splitmix64 with state 0: first outputs of the reference generator (Vigna)
    assert int(ci.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(ci.splitmix64(np.uint64(0x9E3779B97F4A7C15))) == 0x6E789E6AA1B965F4


def test_square_mesh_layout_and_jitter_bounds():
    n = 16
    c0, cells = ci.square_mesh(n)
    c1, cells1 = ci.square_mesh(n, 0.2, seed=5)
    assert np.array_equal(cells, cells1)
    assert cells.shape == (2 * n * n, 3) and c0.shape == ((n + 1) ** 2, 2)
    dx = np.abs(c1 - c0)
    assert dx.max() <= 0.2 / n + 1e-15 and dx.max() > 0.15 / n
    bnd = (c0[:, 0] == 0) | (c0[:, 0] == 1) | (c0[:, 1] == 0) | (c0[:, 1] == 1)
    assert np.all(dx[bnd] == 0)
    c2, _ = ci.square_mesh(n, 0.2, seed=5)
    assert np.array_equal(c1, c2)
    # all triangles positively oriented with area >= 0.1 h^2 (reading 8)
    X = c1[cells]
    e1, e2 = X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]
    area = 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    assert area.min() >= 0.1 / n ** 2 - 1e-15


def test_cube_mesh_kuhn():
    n = 3
    coords, cells = ci.cube_mesh(n)
    X = coords[cells]
    E = X[:, 1:] - X[:, :1]
    vol = np.abs(np.linalg.det(E)) / 6
    np.testing.assert_allclose(vol, 1 / (6 * n ** 3), rtol=1e-12)
    assert abs(vol.sum() - 1) < 1e-12


@pytest.mark.parametrize("dim", [2, 3])
def test_manufactured_force_by_finite_differences(dim):
    mu, nu = 0.7, 1.3
    u, p, f = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(mu, nu)
    rng = np.random.default_rng(1)
    x = rng.uniform(0.1, 0.9, size=(20, dim))
    h = 1e-4
    lap = np.zeros((20, dim))
    gp = np.zeros((20, dim))
    div = np.zeros(20)
    for k in range(dim):
        e = np.zeros(dim); e[k] = h
        lap += (u(x + e) - 2 * u(x) + u(x - e)) / h ** 2
        gp[:, k] = (p(x + e) - p(x - e)) / (2 * h)
        div += (u(x + e)[:, k] - u(x - e)[:, k]) / (2 * h)
    fd = mu * u(x) - nu * lap + gp
    np.testing.assert_allclose(f(x), fd, atol=1e-5 * np.abs(fd).max())
    assert np.abs(div).max() < 1e-6
    # homogeneous Dirichlet on the boundary
    xb = x.copy(); xb[:, 0] = 0.0
    assert np.abs(u(xb)).max() < 1e-14


def test_cell_average_exact_for_quadratics():
    coords, cells = ci.square_mesh(3, 0.2, seed=1)
    q = lambda x: np.stack([x[..., 0] ** 2 + 3 * x[..., 0] * x[..., 1], x[..., 1] ** 2], -1)
    avg = ci.cell_average(q, coords, cells)
    # exact average of x^2, xy, y^2 over a triangle via the edge-midpoint rule
    X = coords[cells]
    mids = [(X[:, i] + X[:, j]) / 2 for i, j in ((0, 1), (1, 2), (0, 2))]
    ex = sum(q(mm) for mm in mids) / 3
    np.testing.assert_allclose(avg, ex, rtol=1e-13)


def test_gaussian_force_stats():
    f = ci.gaussian_force(200000, 2, seed=3)
    assert abs(f.mean()) < 0.01 and abs(f.std() - 1) < 0.01


def test_ns_iterate_discretely_divergence_free_and_consistent():
    n = 8
    coords, cells = ci.square_mesh(n)
    U = ci.ns_iterate_2d(coords, cells, n, seed=4)
    # independent flux computation: outward normal*length per local face
    X = coords[cells]
    div = np.zeros(len(cells))
    for s in range(3):
        o = [v for v in range(3) if v != s]
        P, Q = X[:, o[0]], X[:, o[1]]
        e = Q - P
        nv = np.stack([e[:, 1], -e[:, 0]], 1)
        sgn = np.sign(np.einsum("ij,ij->i", nv, P - X[:, s]))
        div += np.einsum("ij,ij->i", nv * sgn[:, None], U[:, s])
    assert np.abs(div).max() < 1e-15
    # same value seen from both cells of an edge
    key = {}
    for k in range(len(cells)):
        for s in range(3):
            t = tuple(sorted(v for i, v in enumerate(cells[k]) if i != s))
            if t in key:
                assert np.array_equal(key[t], U[k, s])
            key[t] = U[k, s]


def _conforming(cells, d):
    """Every (d-1)-face of a conforming simplicial mesh is shared by 1 or 2 cells; on a
    structured box the interior/boundary face counts are the closed forms of SURVEY A.3."""
    keys = {}
    for k in range(len(cells)):
        for s in range(d + 1):
            t = tuple(sorted(v for i, v in enumerate(cells[k]) if i != s))
            keys[t] = keys.get(t, 0) + 1
    cnt = np.array(list(keys.values()))
    return cnt.max() <= 2, int((cnt == 2).sum()), int((cnt == 1).sum())


def test_flipped_square_mesh_unstructured_and_conforming():
    n = 12
    c0, k0 = ci.square_mesh(n, 0.2, 5)
    c1, k1 = ci.square_mesh(n, 0.2, 5, flip_seed=9)
    assert np.array_equal(c0, c1) and not np.array_equal(k0, k1)
    assert np.array_equal(ci.square_mesh(n, 0.2, 5, flip_seed=9)[1], k1)   # deterministic
    ok, nint, nbnd = _conforming(k1, 2)
    assert ok and nint == 3 * n * n - 2 * n and nbnd == 4 * n
    # interior vertex valences vary (the structured split has valence 6 everywhere)
    val = np.bincount(np.concatenate([k1[:, [0, 1]].ravel(), k1[:, [1, 2]].ravel(), k1[:, [0, 2]].ravel()]))
    inner = [(j * (n + 1) + i) for j in range(1, n) for i in range(1, n)]
    edges = {tuple(sorted(e)) for t in k1.tolist() for e in ((t[0], t[1]), (t[1], t[2]), (t[0], t[2]))}
    deg = np.zeros(len(c1), int)
    for a, b in edges:
        deg[a] += 1; deg[b] += 1
    assert set(deg[inner]) >= {4, 6, 8}
    X = c1[k1]
    e1, e2 = X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]
    area = 0.5 * (e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    assert area.min() >= 0.1 / n ** 2 - 1e-15     # same corner bound as the unflipped split


def test_mirrored_kuhn_cube_mesh_unstructured_and_conforming():
    n = 4
    c0, k0 = ci.cube_mesh(n)
    assert np.array_equal(ci.cube_mesh(n, None)[1], k0)
    c1, k1 = ci.cube_mesh(n, flip_seed=5)
    assert not np.array_equal(k0, k1)
    ok, nint, nbnd = _conforming(k1, 3)
    assert ok and nint == 12 * n ** 3 - 6 * n * n and nbnd == 12 * n * n
    vol = np.abs(np.linalg.det(c1[k1][:, 1:] - c1[k1][:, :1])) / 6
    np.testing.assert_allclose(vol, 1 / (6 * n ** 3), rtol=1e-12)
    # edge valences (tets around an edge) vary beyond the structured {4, 6}
    edges = {}
    for t in k1.tolist():
        for a in range(4):
            for b in range(a + 1, 4):
                e = tuple(sorted((t[a], t[b])))
                edges[e] = edges.get(e, 0) + 1
    assert len(set(edges.values())) > len(set(_kuhn_edge_valences(k0)))


def _kuhn_edge_valences(cells):
    edges = {}
    for t in cells.tolist():
        for a in range(4):
            for b in range(a + 1, 4):
                e = tuple(sorted((t[a], t[b])))
                edges[e] = edges.get(e, 0) + 1
    return edges.values()


def test_cube_jitter_keeps_volumes_positive():
    """|det| of a Kuhn tet is affine in each vertex, so its minimum over the jitter box is at a
    corner of the 12-dimensional box: exhaustive over the 4096 corners for every tet shape
    gives |K| >= 0.37 h^3/6 at 0.1 h."""
    import itertools
    S = np.array(list(itertools.product((-1, 1), repeat=12)), float).reshape(-1, 4, 3)
    for p in [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]:
        v = [np.zeros(3)]
        for a in p:
            w = v[-1].copy(); w[a] += 1; v.append(w)
        d = np.linalg.det((np.array(v)[None] + 0.1 * S)[:, 1:] - (np.array(v)[None] + 0.1 * S)[:, :1])
        assert np.abs(d).min() >= 0.37 and np.all(np.sign(d) == np.sign(d[0]))
    n = 5
    c, k = ci.cube_mesh(n, flip_seed=2, jitter=0.1, seed=3)
    vol = np.abs(np.linalg.det(c[k][:, 1:] - c[k][:, :1])) / 6
    assert vol.min() >= 0.37 / (6 * n ** 3) and abs(vol.sum() - 1) < 1e-12
