"""Pins of the backward-Euler oracle (oracle/timestep.py) against what the
mathematics fixes, not against its own formulas:
  * the lumped mass of a structured mesh in closed form;
  * step 1 from U = 0 is the single transient solve (same data, independent assembly path:
    the hybrid method);
  * energy stability with zero data: ||U^{n+1}||_M <= ||U^n||_M for a divergence-free U^n;
  * the steady limit: with time-independent data the iterates converge to the STEADY coupled
    solution (mu = 0), whose fixed-point property holds only if the mass term enters both
    sides with the same sign and size (a dropped or mis-scaled term fails)."""
import numpy as np

import cr_inputs as ci
import oracle as O


def _case(n, jitter=0.2, mu=1.0, nu=1.0, force="gaussian", seed=3):
    coords, cells = ci.square_mesh(n, jitter, seed)
    m = O.build_mesh(coords, cells)
    fbar = ci.gaussian_force(m.nc, 2, seed) if force == "gaussian" else np.zeros((m.nc, 2))
    return m, O.Params(mu=mu, nu=nu), O.Data(fbar=fbar)


def test_lumped_mass_closed_form():
    n = 6
    m, _, _ = _case(n, jitter=0.0)
    # unit square, n x n squares split in 2: every interior edge has two triangles of area
    # 1/(2 n^2), each contributing |K|/3
    assert np.allclose(O.lumped_mass(m), 2 * (1.0 / (2 * n * n)) / 3.0, rtol=1e-14)


def test_first_step_is_the_transient_solve():
    m, prm, data = _case(8)
    Us, Ps = O.backward_euler(m, prm, data, 1)
    h = O.hybrid_pipeline(m, prm, data)
    assert np.abs(Us[0] - h["U"]).max() <= 1e-10 * np.abs(h["U"]).max()
    assert np.abs(Ps[0] - h["P"]).max() <= 1e-9 * np.abs(h["P"]).max()


def test_energy_decays_without_data():
    m, prm, data = _case(8, force="zero")
    U0 = np.random.default_rng(1).normal(size=(m.nf_int, 2))
    Us, _ = O.backward_euler(m, prm, data, 4, U0=U0)
    Ml = O.lumped_mass(m)
    e = [float(np.sum(Ml * u.reshape(-1) ** 2)) for u in Us]
    assert all(e[k + 1] < e[k] for k in range(len(e) - 1)), e
    assert e[-1] < 0.5 * e[0]


def test_steady_limit():
    m, prm, data = _case(8, mu=10.0)
    Us, Ps = O.backward_euler(m, prm, data, 60)
    Ms, rhs, nU = O.assemble_coupled(m, O.Params(mu=0.0, nu=1.0), data)
    x = O.direct_refined(Ms, rhs)
    Uss = x[:nU].reshape(m.nf_int, 2)
    assert np.abs(Us[-1] - Uss).max() <= 1e-9 * np.abs(Uss).max()
    # and not already at step 1 (the mass term matters)
    assert np.abs(Us[0] - Uss).max() > 1e-3 * np.abs(Uss).max()
