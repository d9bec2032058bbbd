"""Pins of oracle C-8 (post-processing) and of the subset entry points the
full-size GPU checks rely on (oracle.scheme.eliminate_cells / recover_cells / _subset_call).

* errors(): closed forms — a constant velocity offset c on the interior faces gives
  errl2U^2 = c^2 * sum_K |K|/(d+1) * #interior faces of K, a zero-mean pressure offset g gives
  errl2P^2 = sum_K |K| g_K^2 and a constant pressure offset gives 0 (zero-mean) — and
  the absolute values of the scratch ladder in SURVEY.md A.4 (an implementation independent of
  this oracle: n = 8 errl2U = 1.8322e-01, errl2P = 1.0520e+00; n = 16 4.7105e-02 / 4.3976e-01).
* eliminate_cells / recover_cells: on a random cell subset that contains K0 they return the
  very same binary128-rounded G_K, S_K, B_K, P_K, Uhat_K as the whole-mesh hybridise / recover
  (steady + MIS shift with an interior K0, so a wrong K0 remap or E gather changes bits).
"""
import numpy as np
import pytest

import cr_inputs as ci
import oracle as O


def _mesh(dim, n, flip=None):
    coords, cells = ci.square_mesh(n, 0.2, 3, flip_seed=flip) if dim == 2 else ci.cube_mesh(n, flip_seed=flip)
    return coords, cells, O.build_mesh(coords, cells)


@pytest.mark.parametrize("dim,n", [(2, 6), (3, 2)])
def test_errors_closed_forms(dim, n):
    coords, cells, m = _mesh(dim, n, flip=4)
    u, p, _ = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(1.0, 1.0)
    Uex = u(m.xs[m.dof_face])
    Pex = p(m.xK)
    eu, ep = O.errors(m, Uex, Pex, u, p)
    # u vanishes on the boundary (homogeneous Dirichlet) -> the exact interpolant has no error
    assert eu < 1e-14 and ep < 1e-14
    c = np.array([0.3, -0.4, 0.5][:dim])
    nint = (m.face_dof[m.cell_faces] >= 0).sum(axis=1)
    expect_u = np.sqrt(np.sum(m.vol / (dim + 1) * nint) * np.dot(c, c))
    eu, ep = O.errors(m, Uex + c, Pex + 7.0, u, p)
    assert abs(eu - expect_u) <= 1e-13 * expect_u
    assert ep < 1e-12                               # constant pressure offset: zero-mean removes it
    g = np.sin(np.arange(m.nc) * 1.7)
    g = g - np.sum(m.vol * g) / np.sum(m.vol)
    eu, ep = O.errors(m, Uex, Pex + g, u, p)
    assert abs(ep - np.sqrt(np.sum(m.vol * g * g))) <= 1e-13 * ep


@pytest.mark.parametrize("n,eu_ref,ep_ref", [(8, 1.8322e-01, 1.0520e+00), (16, 4.7105e-02, 4.3976e-01)])
def test_errors_absolute_values_survey_a4(n, eu_ref, ep_ref):
    """SURVEY.md A.4 (unjittered 2D, mu = nu = 1, degree-2 force rule, K0 = 0)."""
    u, p, f = ci.manufactured_2d(1.0, 1.0)
    coords, cells = ci.square_mesh(n)
    m = O.build_mesh(coords, cells)
    h = O.hybrid_pipeline(m, O.Params(1.0, 1.0), O.Data(fbar=ci.cell_average(f, coords, cells)))
    eu, ep = O.errors(m, h["U"], h["P"], u, p)
    assert abs(eu - eu_ref) <= 1e-4 * eu_ref and abs(ep - ep_ref) <= 1e-4 * ep_ref, (eu, ep)


CASES = {
    "2d-steady-mis-interiorK0": dict(dim=2, n=7, mu=0.0, shift="mis", k0=41, force="gaussian"),
    "2d-transient-dirichlet": dict(dim=2, n=6, mu=1.0, dirichlet=True),
    "2d-ns-step": dict(dim=2, n=6, mu=0.0, nu=0.01, shift="mis", ns=True),
    "3d-steady-mis-flipped": dict(dim=3, n=2, mu=0.0, shift="mis", k0=13, force="gaussian", flip=6),
}


def _case(dim, n, mu=1.0, nu=1.0, shift="none", k0=0, force="manufactured", dirichlet=False, ns=False, flip=None):
    coords, cells, m = _mesh(dim, n, flip)
    if force == "gaussian":
        fbar = ci.gaussian_force(m.nc, dim, 11)
    else:
        _, _, f = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(mu, nu)
        fbar = ci.cell_average(f, coords, cells)
    dirv = None
    if dirichlet:
        X = coords[cells]
        xs = np.stack([np.delete(X, s, axis=1).mean(1) for s in range(dim + 1)], 1)
        dirv = np.stack([xs[..., 0] - 0.3 + xs[..., 1] ** 2, 0.5 - xs[..., 1]], -1)
    data = O.Data(fbar=fbar, dirichlet=dirv, u_iter=ci.ns_iterate_2d(coords, cells, n, 2) if ns else None)
    prm = O.Params(mu=mu, nu=nu, shift=shift, mis_seed=9, k0=k0, physics="ns_step" if ns else "stokes")
    return m, prm, data


@pytest.mark.parametrize("name", list(CASES))
def test_subset_elimination_and_recovery_equal_whole_mesh(name):
    m, prm, data = _case(**CASES[name])
    h = O.hybridise(m, prm, data)
    rng = np.random.default_rng(7)
    cells = rng.choice(m.nc, size=min(m.nc, 23), replace=False)
    cells = np.unique(np.concatenate([cells, [prm.k0], [m.nc - 1]]))
    rng.shuffle(cells)                        # the subset order must not matter either
    G, S, B = O.eliminate_cells(m, prm, data, h["E"], cells)
    assert np.array_equal(G, h["G_loc"][cells])
    assert np.array_equal(S, h["S_loc"][cells])
    assert np.array_equal(B, h["B"][cells])
    W = rng.normal(size=len(h["S"]))
    U, P, Uh, _ = O.recover(m, prm, data, h["E"], W)
    Ps, Uhs = O.recover_cells(m, prm, data, h["E"], W, cells)
    assert np.array_equal(Ps, P[cells]) and np.array_equal(Uhs, Uh[cells])
    assert Ps[list(cells).index(prm.k0)] == 0.0           # P_K0 = 0
