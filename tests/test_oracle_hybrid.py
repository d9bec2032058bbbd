"""Pins of oracle C-3..C-5, C-7 (shift E_K, coupled system, hybridisation, recovery;
PAPER.md §3) against the paper's theorems and closed forms:
hybrid = coupled, SPD / symmetric-invertible G,
stencil, G_K C D = 0, explicit enlarged system eq. (syslinhyb)
(P:L354-356), well-balanced constant force, E_K + E_L = 0."""
import numpy as np
import pytest
import scipy.sparse as sp

import cr_inputs as ci
import oracle as O


def relL2(x, y):
    return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)


def setup(dim, n, mu=1.0, nu=1.0, shift="none", jitter=0.2, seed=1, force="manufactured",
          dirichlet=None, ns=False):
    if dim == 2:
        coords, cells = ci.square_mesh(n, jitter, seed)
    else:
        coords, cells = ci.cube_mesh(n)
    m = O.build_mesh(coords, cells)
    if force == "manufactured":
        _, _, f = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(mu, nu)
        fbar = ci.cell_average(f, coords, cells)
    elif force == "gaussian":
        fbar = ci.gaussian_force(m.nc, dim, seed)
    elif force == "zero":
        fbar = np.zeros((m.nc, dim))
    else:
        fbar = np.tile(np.asarray(force, float), (m.nc, 1))
    prm = O.Params(mu=mu, nu=nu, shift=shift, mis_seed=seed + 100,
                   physics="ns_step" if ns else "stokes")
    data = O.Data(fbar=fbar, dirichlet=dirichlet)
    if ns:
        data.u_iter = ci.ns_iterate_2d(coords, cells, n, seed)
    return m, prm, data


def coupled_solution(m, prm, data):
    M, rhs, nU = O.assemble_coupled(m, prm, data)
    x = O.direct_refined(M, rhs)
    U = x[:nU].reshape(-1, m.dim)
    P = np.insert(x[nU:], prm.k0, 0.0)
    return U, P, M, rhs, nU


CASES = [
    ("2d-transient", dict(dim=2, n=6)),
    ("2d-steady-mis", dict(dim=2, n=6, mu=0.0, shift="mis", force="gaussian")),
    ("2d-ns-step", dict(dim=2, n=6, mu=0.0, nu=0.01, shift="mis", force="zero", ns=True, jitter=0.0)),
    ("3d-transient", dict(dim=3, n=2)),
    ("3d-steady-mis", dict(dim=3, n=2, mu=0.0, shift="mis", force="gaussian")),
]


@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_hybrid_equals_coupled(name, kw):
    m, prm, data = setup(**kw)
    Uc, Pc, *_ = coupled_solution(m, prm, data)
    h = O.hybrid_pipeline(m, prm, data)
    assert relL2(h["U"], Uc) < 1e-11
    assert relL2(h["P"], Pc) < 1e-11
    assert h["disagree"] <= 1e-11 * np.abs(Uc).max()                 # P:L393 common value


def test_inhomogeneous_dirichlet_exactness_and_cell_divergence():
    """Dirichlet fold + g_K = +sum_ext a.U^D (reading 7): hybrid = coupled and
    the FULL-face divergence sum_{s in F_K} a_s.U_s (boundary values included) vanishes."""
    coords, cells = ci.square_mesh(5, 0.2, 2)
    m = O.build_mesh(coords, cells)
    # u^D = (x - 0.3, 0.5 - y) + (y^2, x^2): divergence free, non-zero net flux per edge
    uD = lambda x: np.stack([x[..., 0] - 0.3 + x[..., 1] ** 2, 0.5 - x[..., 1] + x[..., 0] ** 2], -1)
    dirichlet = uD(m.xs[m.cell_faces])
    prm = O.Params(mu=1.0, nu=1.0)
    data = O.Data(fbar=np.zeros((m.nc, 2)), dirichlet=dirichlet)
    Uc, Pc, *_ = coupled_solution(m, prm, data)
    h = O.hybrid_pipeline(m, prm, data)
    assert relL2(h["U"], Uc) < 1e-11 and relL2(h["P"], Pc) < 1e-11
    Uf = np.zeros((m.nf, 2))
    Uf[m.face_dof >= 0] = h["U"]
    bnd = m.face_dof[m.cell_faces] < 0
    Ul = Uf[m.cell_faces]
    Ul[bnd] = dirichlet[bnd]
    div = np.einsum("ksi,ksi->k", m.a, Ul)
    assert np.abs(div).max() < 1e-13


def test_transient_G_is_spd_and_symmetric():
    m, prm, data = setup(2, 6)
    h = O.hybridise(m, prm, data)
    G = h["G"].toarray()
    assert np.abs(G - G.T).max() <= 1e-15 * np.abs(G).max()
    np.linalg.cholesky(G)
    m3, prm3, data3 = setup(3, 2)
    np.linalg.cholesky(O.hybridise(m3, prm3, data3)["G"].toarray())


def test_steady_G_symmetric_indefinite_invertible():
    m, prm, data = setup(2, 6, mu=0.0, shift="mis", force="gaussian")
    h = O.hybridise(m, prm, data)
    G = h["G"].toarray()
    assert np.abs(G - G.T).max() <= 1e-14 * np.abs(G).max()
    ev = np.linalg.eigvalsh(0.5 * (G + G.T))
    assert ev.min() < 0 < ev.max()                                   # P:L64 "no longer positive definite"
    assert np.abs(ev).min() > 1e-10 * np.abs(ev).max()


def test_ns_G_nonsymmetric():
    m, prm, data = setup(2, 6, mu=0.0, nu=0.01, shift="mis", force="zero", ns=True, jitter=0.0)
    G = O.hybridise(m, prm, data)["G"].toarray()
    assert np.abs(G - G.T).max() > 1e-6 * np.abs(G).max()


@pytest.mark.parametrize("dim,n", [(2, 5), (3, 2)])
def test_stencil_of_G_is_full_component_stencil_of_A(dim, n):
    """pattern(G) = pattern of sum_K H_K A_K H_K^t with FULL d x d blocks."""
    m, prm, data = setup(dim, n)
    G = O.hybridise(m, prm, data)["G"]
    pat = set()
    for K in range(m.nc):
        dofs = [m.face_dof[f] for f in m.cell_faces[K] if m.face_dof[f] >= 0]
        for p in dofs:
            for q in dofs:
                for i in range(dim):
                    for j in range(dim):
                        pat.add((dim * p + i, dim * q + j))
    Gc = G.tocoo()
    assert set(zip(Gc.row.tolist(), Gc.col.tolist())) == pat


def test_local_projection_identity_GK_C_D_zero():
    """G_K (C_K D_K) = 0 for K != K0 (projection annihilates D_K)."""
    m, prm, data = setup(2, 4)
    h = O.hybridise(m, prm, data)
    _, _, D, _ = O.local_blocks(m, prm, data)
    cs = np.repeat(m.csign, 2, axis=1).astype(float)
    for K in range(1, m.nc):
        v = h["G_loc"][K] @ (cs[K] * D[K])
        assert np.abs(v).max() <= 1e-14 * np.abs(h["G_loc"][K]).max() * np.abs(D[K]).max()


def test_zero_data_gives_zero():
    m, prm, data = setup(2, 4, force="zero")
    h = O.hybrid_pipeline(m, prm, data)
    assert np.all(h["S"] == 0) and np.all(h["W"] == 0) and np.all(h["P"] == 0)


def test_enlarged_system_syslinhyb_explicit():
    """Assemble eq. (syslinhyb) explicitly from A_K, E_K, C_K, D_K, R_K and
    solve it: its (U_hat, P_hat, W_hat) must equal the oracle's eliminated G W = S solve
    and recovery; and J-summing its momentum rows reproduces eq. (syslin)."""
    for kw in (dict(dim=2, n=3), dict(dim=2, n=3, mu=0.0, shift="mis", force="gaussian")):
        m, prm, data = setup(**kw)
        d = m.dim
        n = (d + 1) * d
        A_K, R_K, D_K, g_K = O.local_blocks(m, prm, data)
        h = O.hybrid_pipeline(m, prm, data)
        E = h["E"]
        intr = np.repeat(m.interior_local, d, axis=1)          # [nc, n]
        # hat unknowns: (K, local interior (l,i)) in cell order
        hat_idx = -np.ones((m.nc, n), dtype=int)
        cnt = 0
        for K in range(m.nc):
            for r in range(n):
                if intr[K, r]:
                    hat_idx[K, r] = cnt; cnt += 1
        nU = d * m.nf_int
        nP = m.nc - 1
        Ahat = sp.lil_matrix((cnt, cnt)); Dhat = sp.lil_matrix((nP, cnt)); Chat = sp.lil_matrix((nU, cnt))
        Rhat = np.zeros(cnt)
        for K in range(m.nc):
            for r in range(n):
                if not intr[K, r]:
                    continue
                hr = hat_idx[K, r]
                Rhat[hr] = R_K[K, r]
                for c in range(n):
                    if intr[K, c]:
                        Ahat[hr, hat_idx[K, c]] = A_K[K, r, c] + (E[K, r // d] if r == c else 0.0)
                if K != 0:
                    Dhat[K - 1, hr] = D_K[K, r]
                gdof = d * m.face_dof[m.cell_faces[K, r // d]] + r % d
                Chat[gdof, hr] = m.csign[K, r // d]
        big = sp.bmat([[Ahat, Dhat.T, Chat.T], [Dhat, None, None], [Chat, None, None]], format="csr")
        rhs = np.concatenate([Rhat, g_K[1:], np.zeros(nU)])
        x = O.direct_refined(big, rhs)
        Uh, Ph, Wh = x[:cnt], x[cnt:cnt + nP], x[cnt + nP:]
        assert relL2(Wh, h["W"]) < 1e-10
        assert relL2(np.insert(Ph, 0, 0.0), h["P"]) < 1e-10
        Uh_or = h["Uhat"].reshape(m.nc, n)
        assert relL2(Uh, Uh_or[intr]) < 1e-10
        # J-row sums of the momentum block give A U + D^t P = R
        J = (Chat != 0).astype(float)
        Uc, Pc, M, crhs, _ = coupled_solution(m, prm, data)
        lhs = J @ (Ahat @ Uh + Dhat.T @ Ph + Chat.T @ Wh)
        np.testing.assert_allclose(lhs, J @ Rhat, atol=1e-12 * np.abs(J @ Rhat).max())
        # J Ahat Uhat + J Dhat^t Phat = A U + D^t P evaluated at the hybrid (U, P)
        xu = np.concatenate([h["U"].ravel(), h["P"][1:]])
        np.testing.assert_allclose(J @ (Ahat @ Uh + Dhat.T @ Ph), M[:nU] @ xu,
                                   atol=1e-11 * np.abs(M[:nU] @ xu).max())


@pytest.mark.parametrize("kw", [dict(dim=2, n=6), dict(dim=2, n=6, mu=0.0, shift="mis"),
                                dict(dim=3, n=2), dict(dim=3, n=2, mu=0.0, shift="mis")])
def test_well_balanced_constant_force(kw):
    """constant f gives U = 0 and the exact pressure.  Closed form of the
    discrete pressure with K0 gauge: P_K = f . (x_K - x_K0)."""
    f = [0.7, -1.3] if kw["dim"] == 2 else [0.7, -1.3, 0.4]
    m, prm, data = setup(force=f, **kw)
    h = O.hybrid_pipeline(m, prm, data)
    assert np.abs(h["U"]).max() < 1e-12
    Pex = (m.xK - m.xK[0]) @ np.asarray(f)
    assert np.abs(h["P"] - Pex).max() < 1e-12
    Uc, Pc, *_ = coupled_solution(m, prm, data)
    assert np.abs(Uc).max() < 1e-12 and np.abs(Pc - Pex).max() < 1e-12


def test_mis_shift_properties():
    """M_1 independent and maximal (M_2 = neighbours of M_1), E_K + E_L = 0,
    Ahat_K negative definite on M_1, positive definite on M_2 (Stokes)."""
    m, prm, data = setup(2, 8, mu=0.0, shift="mis", force="gaussian")
    A_K, *_ = O.local_blocks(m, prm, data)
    E, inM1, lam = O.shift_E(m, prm, A_K)
    fi = m.face_cells[m.face_cells[:, 1] >= 0]
    assert not np.any(inM1[fi[:, 0]] & inM1[fi[:, 1]])
    has = np.zeros(m.nc, bool)
    has[fi[inM1[fi[:, 1]], 0]] = True
    has[fi[inM1[fi[:, 0]], 1]] = True
    assert np.all(inM1 | has)
    f = np.nonzero(m.face_dof >= 0)[0]
    K, L = m.face_cells[f, 0], m.face_cells[f, 1]
    lK = np.argmax(m.cell_faces[K] == f[:, None], 1)
    lL = np.argmax(m.cell_faces[L] == f[:, None], 1)
    assert np.all(E[K, lK] + E[L, lL] == 0)
    d = 2
    for Kc in range(m.nc):
        idx = [r for r in range((d + 1) * d) if m.interior_local[Kc, r // d]]
        Ah = A_K[Kc][np.ix_(idx, idx)] + np.diag([E[Kc, r // d] for r in idx])
        ev = np.linalg.eigvalsh(Ah)
        if inM1[Kc]:
            assert ev.max() < 0
        else:
            assert ev.min() > 0
    # greedy MIS is deterministic in the seed and changes with it
    assert np.array_equal(O.scheme.mis_greedy(m, prm.mis_seed), inM1)
    assert not np.array_equal(O.scheme.mis_greedy(m, prm.mis_seed + 1), inM1)


def test_transient_BK_limit():
    """B_K nu/|K| -> d as mu|K|^2/nu -> 0 (interior cells; closed form of
    D^t (I(x)S_K)^{-1} D with P_1 a = 0)."""
    m, prm, data = setup(2, 6, mu=1e-9)
    h = O.hybridise(m, prm, data)
    full = m.interior_local.all(1)
    np.testing.assert_allclose(h["B"][full] * prm.nu / m.vol[full], 2.0, rtol=1e-6)
