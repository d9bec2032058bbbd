"""Pins of the Newton oracle (oracle/newton.py), independent of its formulas:
  * quadratic convergence (a wrong or incomplete Jacobian converges linearly at best);
  * the Stokes limit: as nu grows the relative effect of convection falls like 1/nu (Re -> 0),
    against the steady Stokes solution from the independently pinned Stokes assembly with the
    same wall data;
  * the converged velocity is discretely divergence-free on every cell, wall faces included."""
import numpy as np

import cr_inputs as ci
import oracle as O


def _cavity(n):
    coords, cells = ci.square_mesh(n, 0.0, 4)
    m = O.build_mesh(coords, cells)
    return m, ci.lid_dirichlet_2d(coords, cells), np.zeros((m.nc, 2))


def test_newton_converges_quadratically():
    m, wall, f = _cavity(8)
    U, P, h = O.newton_ns(m, O.Params(mu=0.0, nu=0.1, physics="ns_step"), f, wall, max_newton=10, tol=1e-13)
    assert h[-1] <= 1e-13 and len(h) <= 6, h
    for k in range(1, len(h) - 1):
        if h[k] > 1e-6:
            assert h[k + 1] <= 1.0 * h[k] ** 2, h


def test_stokes_limit():
    m, wall, f = _cavity(8)
    Ms, rhs, nU = O.assemble_coupled(m, O.Params(mu=0.0, nu=1.0), O.Data(fbar=f, dirichlet=wall))
    Us = O.direct_refined(Ms, rhs)[:nU].reshape(m.nf_int, 2)
    diffs = []
    for nu in (100.0, 1000.0):
        U, _, _ = O.newton_ns(m, O.Params(mu=0.0, nu=nu, physics="ns_step"), f, wall, tol=1e-13)
        diffs.append(np.linalg.norm(U - Us) / np.linalg.norm(Us))
    assert diffs[1] <= 1e-3
    assert 5.0 <= diffs[0] / diffs[1] <= 20.0, diffs


def test_converged_velocity_is_divergence_free():
    m, wall, f = _cavity(8)
    U, _, _ = O.newton_ns(m, O.Params(mu=0.0, nu=0.01, physics="ns_step"), f, wall, tol=1e-12)
    Uc = O.cell_face_values(m, U, wall)
    div = np.einsum("kli,kli->k", m.a, Uc)
    assert np.abs(div).max() <= 1e-12 * np.abs(m.a).max()


def test_damped_newton_reaches_the_re1000_cavity():
    """P:L783-799 (Table 7 right: lid-driven cavity, Re = 1000, Newton tolerance 5e-7): full
    Newton steps from rest do not converge on this mesh (n = 16), the Armijo-damped iteration does,
    ends with full steps and quadratic decay, and its limit satisfies the discrete equations: the
    nonlinear residual ||F|| at the limit is at rounding level and U is divergence-free per cell."""
    m, wall, f = _cavity(16)
    prm = O.Params(mu=0.0, nu=1e-3, physics="ns_step")
    _, _, h_full = O.newton_ns(m, prm, f, wall, max_newton=25, tol=5e-7)
    assert h_full[-1] > 1e-3                       # undamped: no convergence in 25 steps
    U, P, h = O.newton_ns(m, prm, f, wall, max_newton=40, tol=5e-7, damped=True)
    assert h[-1] <= 5e-7 and len(h) <= 25, h
    assert h[-2] <= 1e-2 and h[-1] <= 10 * h[-2] ** 2, h  # final steps are full Newton steps
    from oracle.newton import residual_norm
    r = residual_norm(m, prm, f, wall, U, P)
    r0 = residual_norm(m, prm, f, wall, 0 * U, 0 * P)
    assert r <= 1e-9 * r0, (r, r0)
    Uc = O.cell_face_values(m, U, wall)
    assert np.abs(np.einsum("kli,kli->k", m.a, Uc)).max() <= 1e-12 * np.abs(m.a).max()
