"""Pins of oracle C-2 (local blocks S_K, A_K, D_K, R_K, convection; PAPER.md
P:L129-235, L261-306) against hand examples, independent derivations
from the paper's definitions (CR basis from its mean-value conditions, exact
quadrature, Raviart-Thomas reconstruction, co-volume geometry) and finite
differences."""
import ctypes

import numpy as np
import pytest

import cr_inputs as ci
import oracle as O


def _p(x):
    return None if x is None else x.ctypes.data_as(ctypes.c_void_p)


def cell_blocks(coords, mu, nu, fbar=None, intr=None, dirichlet=None, uit=None, is_ns=False):
    """Run the oracle's local_system on ONE cell, faces flagged interior by ``intr``."""
    d = coords.shape[1]
    m = O.build_mesh(coords, np.arange(d + 1, dtype=np.int32)[None])
    n = (d + 1) * d
    intr = np.ones((1, d + 1), np.int8) if intr is None else np.asarray(intr, np.int8).reshape(1, -1)
    fbar = np.zeros((1, d)) if fbar is None else np.asarray(fbar, float).reshape(1, d)
    xs = np.ascontiguousarray(m.xs[m.cell_faces])
    A = np.zeros((1, n, n)); R = np.zeros((1, n)); D = np.zeros((1, n)); g = np.zeros(1)
    dirichlet = None if dirichlet is None else np.ascontiguousarray(dirichlet, float).reshape(1, d + 1, d)
    uit = None if uit is None else np.ascontiguousarray(uit, float).reshape(1, d + 1, d)
    O.lib().or_cell_blocks(ctypes.c_int(d), ctypes.c_int64(1), ctypes.c_double(mu), ctypes.c_double(nu),
                           ctypes.c_int(int(is_ns)), _p(np.ascontiguousarray(m.a)), _p(m.vol),
                           _p(np.ascontiguousarray(m.xK)), _p(xs), _p(intr), _p(fbar),
                           _p(dirichlet), _p(uit), None, _p(A), _p(R), _p(D), _p(g))
    return m, A[0], R[0], D[0], g[0]


def cr_basis_gradients(X):
    """Affine phi_s with mean 1 on face s and 0 on the others.  For an affine
    function the face mean is the value at the face centroid, so solve for
    phi(x) = c0 + c.x at the d+1 face centroids.  Returns grads [d+1, d]."""
    d = X.shape[1]
    xs = np.array([np.delete(X, s, axis=0).mean(0) for s in range(d + 1)])
    M = np.hstack([np.ones((d + 1, 1)), xs])
    C = np.linalg.solve(M, np.eye(d + 1))        # column s = coefficients of phi_s
    return C[1:, :].T


TRI = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]])


def test_spec_mass_only_block():
    # mu = 1, nu = 0, unit right triangle: S_K = |K|/3 I = I/6
    _, A, _, _, _ = cell_blocks(TRI, 1.0, 0.0)
    np.testing.assert_allclose(A, np.eye(6) / 6, atol=1e-17)


def test_spec_rhs_example():
    # fbar = (1,0); diagonal face (local 1): a = (-1,1), x_s - x_K = (1/2,1/2)-(2/3,1/3) -> entries (1/6,-1/6)
    _, _, R, D, _ = cell_blocks(TRI, 1.0, 1.0, fbar=[1.0, 0.0])
    np.testing.assert_allclose(R[2:4], [1 / 6, -1 / 6], rtol=1e-15)
    np.testing.assert_array_equal(D[2:4], [1.0, -1.0])                    # D_K = -a


@pytest.mark.parametrize("dim", [2, 3])
def test_stiffness_matches_cr_basis_from_definition(dim):
    rng = np.random.default_rng(dim)
    X = rng.uniform(0, 1, size=(dim + 1, dim))
    if dim == 2 and np.linalg.det(X[1:] - X[0]) < 0:
        X = X[[0, 2, 1]]
    vol = abs(np.linalg.det(X[1:] - X[0])) / (2 if dim == 2 else 6)
    gr = cr_basis_gradients(X)
    Sstiff = vol * gr @ gr.T                        # int_K grad phi_s . grad phi_s'
    _, A, _, _, _ = cell_blocks(X, 0.0, 1.0)
    S = A[0::dim, 0::dim]
    np.testing.assert_allclose(S, Sstiff, rtol=1e-11, atol=1e-13)
    # component-block-diagonal Stokes A_K
    for i in range(dim):
        for j in range(dim):
            blk = A[i::dim, j::dim]
            if i == j:
                np.testing.assert_array_equal(blk, S)
            else:
                assert np.all(blk == 0)
    # S_K 1 = 0 when mu = 0 and all faces interior
    assert np.abs(S.sum(1)).max() < 1e-12 * np.abs(S).max()


def test_2d_exact_cr_mass_is_lumped_diagonal():
    """in 2D int_K phi_s phi_s' is already diagonal = |K|/3 (the oracle
    uses |K|/(d+1)); exact via the edge-midpoint rule (exact for quadratics)."""
    rng = np.random.default_rng(5)
    X = rng.uniform(0, 1, size=(3, 2))
    vol = abs(np.linalg.det(X[1:] - X[0])) / 2
    xs = np.array([np.delete(X, s, axis=0).mean(0) for s in range(3)])
    Mx = np.hstack([np.ones((3, 1)), xs])
    C = np.linalg.solve(Mx, np.eye(3))
    mids = np.array([(X[i] + X[j]) / 2 for i, j in ((0, 1), (1, 2), (0, 2))])
    phi = np.hstack([np.ones((3, 1)), mids]) @ C    # [mid, s]
    mass = vol / 3 * phi.T @ phi
    np.testing.assert_allclose(mass, vol / 3 * np.eye(3), atol=1e-15)
    _, A, _, _, _ = cell_blocks(X, 1.0, 0.0)
    np.testing.assert_allclose(A[0::2, 0::2], mass, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_rhs_equals_raviart_thomas_pairing(dim):
    """R_K(i,s) = int_K fbar . Pi_hat(phi_s e_i) with the RT basis psi_{K,s} =
    |s|/(d|K|)(x - s_s); the integral of an affine field is |K| times its
    value at x_K.  Independent of eq. (defrhs)'s rewritten form."""
    rng = np.random.default_rng(10 + dim)
    X = rng.uniform(0, 1, size=(dim + 1, dim))
    fbar = rng.normal(size=dim)
    m, _, R, _, _ = cell_blocks(X, 1.0, 1.0, fbar=fbar)
    vol = m.vol[0]
    for s in range(dim + 1):
        for i in range(dim):
            V = np.zeros((dim + 1, dim)); V[s, i] = 1.0
            # Pi_hat v (x_K) = sum_s' (V_s'.a_s')/(d|K|) (x_K - s_s')
            pv = sum((V[t] @ m.a[0, t]) / (dim * vol) * (m.xK[0] - X[t]) for t in range(dim + 1))
            np.testing.assert_allclose(R[s * dim + i], vol * fbar @ pv, rtol=1e-12, atol=1e-15)


def _u_affine(X, U, x):
    """CR interpolant u_K(x) = sum_s U_s phi_s(x), phi from the definition."""
    d = X.shape[1]
    xs = np.array([np.delete(X, s, axis=0).mean(0) for s in range(d + 1)])
    C = np.linalg.solve(np.hstack([np.ones((d + 1, 1)), xs]), np.eye(d + 1))
    phi = np.hstack([1.0, x]) @ C
    return phi @ U


def covolume_flux(X, U):
    """F_{s,s'} = int_{tau_{ss'}} u_K . n_{ss'} from the co-volume geometry
    (P:L189-203): tau_{ss'} is the facet through x_K and the vertices shared by faces
    s and s' (all vertices but s, s'); n oriented from D_{K,s} to D_{K,s'}."""
    d = X.shape[1]
    xK = X.mean(0)
    F = np.zeros((d + 1, d + 1))
    for s in range(d + 1):
        for t in range(d + 1):
            if s == t:
                continue
            shared = [X[v] for v in range(d + 1) if v not in (s, t)]
            pts = [xK] + shared
            if d == 2:
                e = pts[1] - pts[0]
                nvec = np.array([e[1], -e[0]])
            else:
                nvec = 0.5 * np.cross(pts[1] - pts[0], pts[2] - pts[0])
            xt = np.delete(X, t, axis=0).mean(0)        # x_{s'} lies on the D_{s'} side
            if nvec @ (xt - xK) < 0:
                nvec = -nvec
            cen = np.mean(pts, axis=0)                  # u affine: exact midpoint/centroid rule
            F[s, t] = _u_affine(X, U, cen) @ nvec
    return F


@pytest.mark.parametrize("dim", [2, 3])
def test_convection_residual_pair_form_and_covolume_geometry(dim):
    """r from cell_f128.c (single-sum form, flux closed form P:L214) equals the
    gradient in V of the PAIR form b_h (eq. defbh) evaluated with fluxes from
    the co-volume geometry."""
    rng = np.random.default_rng(20 + dim)
    X = rng.uniform(0, 1, size=(dim + 1, dim))
    U = rng.normal(size=(dim + 1, dim))
    m = O.build_mesh(X, np.arange(dim + 1, dtype=np.int32)[None])
    n = (dim + 1) * dim
    r = np.zeros(n); J = np.zeros(n * n)
    O.lib().or_cell_convection(ctypes.c_int(dim), ctypes.c_int64(1), _p(np.ascontiguousarray(m.a)),
                               _p(np.ascontiguousarray(U)), _p(r), _p(J))
    F = covolume_flux(X, U)
    np.testing.assert_allclose(F, -F.T, atol=1e-14)
    grad = np.zeros((dim + 1, dim))
    for s in range(dim + 1):
        for t in range(s + 1, dim + 1):          # unordered pairs {s, t}
            contrib = F[s, t] * (U[t] - U[s]) / 2
            grad[s] += contrib
            grad[t] += contrib
    np.testing.assert_allclose(r.reshape(dim + 1, dim), grad, rtol=1e-11, atol=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_convection_jacobian_matches_central_differences(dim):
    rng = np.random.default_rng(30 + dim)
    X = rng.uniform(0, 1, size=(dim + 1, dim))
    U = rng.normal(size=(dim + 1, dim))
    m = O.build_mesh(X, np.arange(dim + 1, dtype=np.int32)[None])
    a = np.ascontiguousarray(m.a)
    n = (dim + 1) * dim

    def call(Uv):
        r = np.zeros(n); J = np.zeros(n * n)
        O.lib().or_cell_convection(ctypes.c_int(dim), ctypes.c_int64(1), _p(a),
                                   _p(np.ascontiguousarray(Uv)), _p(r), _p(J))
        return r, J.reshape(n, n)

    _, J = call(U)
    h = 1e-3
    Jfd = np.zeros((n, n))
    for c in range(n):
        e = np.zeros(n); e[c] = h
        Jfd[:, c] = (call((U.ravel() + e).reshape(U.shape))[0] - call((U.ravel() - e).reshape(U.shape))[0]) / (2 * h)
    np.testing.assert_allclose(J, Jfd, atol=1e-11 * max(1, np.abs(J).max()))   # quadratic: FD exact
    _, J0 = call(np.zeros_like(U))
    assert np.all(J0 == 0)


def test_flux_telescoping_when_cell_divergence_free():
    """sum_s' a_s'.U_s' = 0 implies sum_{s'} F_{s,s'} = -U_s . a_s."""
    rng = np.random.default_rng(7)
    X = rng.uniform(0, 1, size=(3, 2))
    m = O.build_mesh(X, np.array([[0, 1, 2]], dtype=np.int32))
    U = rng.normal(size=(3, 2))
    a = m.a[0]
    # project U onto {sum a.U = 0}
    flux = sum(a[s] @ U[s] for s in range(3))
    U[0] -= flux * a[0] / (a[0] @ a[0])
    F = covolume_flux(X, U)
    for s in range(3):
        assert abs(F[s].sum() + U[s] @ a[s]) < 1e-14


def test_dirichlet_fold_and_g_sign():
    """Inhomogeneous Dirichlet on face 2 of the unit right triangle (faces 0,1 interior):
    R_I = R - A_IE U^D, g = +a_E . U^D (full-face constraint with D_K = -a)."""
    UD = np.zeros((3, 2)); UD[2] = [0.3, -0.7]
    _, A_full, _, _, _ = cell_blocks(TRI, 1.0, 1.0)
    _, A, R, D, g = cell_blocks(TRI, 1.0, 1.0, intr=[1, 1, 0], dirichlet=UD)
    expR = -(A_full[:, 4:6] @ UD[2])
    expR[4:6] = 0
    np.testing.assert_allclose(R, expR, rtol=1e-15, atol=1e-17)
    assert g == pytest.approx(0.3 * 0.0 + (-0.7) * (-1.0))
    assert np.all(A[4:6] == 0) and np.all(A[:, 4:6] == 0) and np.all(D[4:6] == 0)
