"""GPU parity: the CUDA path (through the C ABI, via the thin binding) against the CPU
oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * connectivity, face numbering, MIS membership, sparsity patterns: bit-exact;
  * assembled entries (G, S, coupled A/D/R/g): |dG_ij| <= 1e-12 max_j |G_ij| (row-relative);
  * solved U and P: relative L2 <= 1e-8 against the oracle's refined direct solution,
    solves driven to a true relative residual of 1e-12 (small cases) / 1e-10 (full size).
"""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

import cr_inputs as ci
import oracle as O

pytestmark = pytest.mark.gpu

import paper_2101_03777_b200 as P  # noqa: E402

DEV = torch.device("cuda")


def tg(x, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def relL2(x, y):
    return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))


def to_scipy(rp, ci_, v, n):
    return sp.csr_matrix((v.cpu().numpy(), ci_.cpu().numpy(), rp.cpu().numpy()), shape=(n, n))


def row_rel_err(Ag, Ao):
    """max_i max_j |Ag_ij - Ao_ij| / max_j |Ao_ij|"""
    Ag, Ao = Ag.tocsr(), Ao.tocsr()
    Dm = (Ag - Ao).tocsr()
    Dm.data = np.abs(Dm.data)
    Aa = Ao.copy()
    Aa.data = np.abs(Aa.data)
    dm = np.asarray(Dm.max(axis=1).todense()).ravel()
    am = np.asarray(Aa.max(axis=1).todense()).ravel()
    return float(np.max(dm / np.where(am > 0, am, 1.0)))


def same_pattern(Ag, Ao):
    Ag, Ao = Ag.tocsr(), Ao.tocsr()
    Ag.sort_indices(); Ao.sort_indices()
    return np.array_equal(Ag.indptr, Ao.indptr) and np.array_equal(Ag.indices, Ao.indices)


# ------------------------------------------------------------------ cases
def make_case(dim, n, mu=1.0, nu=1.0, shift="none", jitter=0.2, seed=1, force="manufactured",
              ns=False, dirichlet=False, k0=0, flip=None):
    """flip: seed of the unstructured variants (random diagonals in 2D, mirrored Kuhn splits in 3D)"""
    if dim == 2:
        coords, cells = ci.square_mesh(n, jitter, seed, flip_seed=flip)
    else:
        coords, cells = ci.cube_mesh(n, flip_seed=flip)
    nc = cells.shape[0]
    if force == "manufactured":
        _, _, f = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(mu, nu)
        fbar = ci.cell_average(f, coords, cells)
    elif force == "gaussian":
        fbar = ci.gaussian_force(nc, dim, seed)
    elif force == "zero":
        fbar = np.zeros((nc, dim))
    else:
        fbar = np.tile(np.asarray(force, float), (nc, 1))
    dirv = None
    if dirichlet:
        X = coords[cells]
        xs = np.stack([np.delete(X, s, axis=1).mean(1) for s in range(dim + 1)], 1)
        dirv = np.stack([xs[..., 0] - 0.3 + xs[..., 1] ** 2, 0.5 - xs[..., 1] + xs[..., 0] ** 2], -1)
    uit = ci.ns_iterate_2d(coords, cells, n, seed) if ns else None
    prm = O.Params(mu=mu, nu=nu, shift=shift, mis_seed=seed + 100, physics="ns_step" if ns else "stokes", k0=k0)
    data = O.Data(fbar=fbar, dirichlet=dirv, u_iter=uit)
    prob = P.Problem(mu=mu, nu=nu, fbar=tg(fbar), physics=P.CR_NS_NEWTON_STEP if ns else P.CR_STOKES,
                     shift=P.CR_SHIFT_MIS if shift == "mis" else P.CR_SHIFT_NONE, mis_seed=seed + 100,
                     gauge_cell=k0, dirichlet=None if dirv is None else tg(dirv),
                     u_iter=None if uit is None else tg(uit))
    return coords, cells, prm, data, prob


# ------------------------------------------------------------------ mesh
def _wide_id_cube(n, spread):
    coords, cells = ci.cube_mesh(n)
    nv = coords.shape[0]
    big = np.zeros((nv * spread, 3))
    big[np.arange(nv) * spread] = coords
    return big, (cells.astype(np.int64) * spread).astype(np.int32)


MESHES = {
    "2d-n8": lambda: ci.square_mesh(8),
    "2d-jit-n33": lambda: ci.square_mesh(33, 0.2, 7),
    "3d-n3": lambda: ci.cube_mesh(3),
    "3d-n5": lambda: ci.cube_mesh(5),
    "3d-two-pass-keys": lambda: _wide_id_cube(3, 40000),   # nv > 2^21 -> 3*22 bits > 64
}


@pytest.mark.parametrize("name", list(MESHES))
def test_mesh_parity(name):
    coords, cells = MESHES[name]()
    mo = O.build_mesh(coords, cells)
    mg = P.cr_build_mesh(tg(coords), tg(cells))
    ex = {k: v.cpu().numpy() for k, v in mg.export().items()}
    assert (mg.nf, mg.nf_int) == (mo.nf, mo.nf_int)
    for k in ("faces", "face_cells", "cell_faces", "face_dof"):
        assert np.array_equal(ex[k], getattr(mo, k)), k
    for k in ("xK", "xs", "a"):
        ref = getattr(mo, k)
        assert np.abs(ex[k] - ref).max() <= 1e-15 * np.abs(ref).max(), k
    assert np.abs(ex["vol"] - mo.vol).max() <= 1e-14 * mo.vol.max()


def test_mesh_errors():
    coords, cells = ci.square_mesh(3)
    with pytest.raises(P.CrError) as e:
        P.cr_build_mesh(tg(coords), tg(np.concatenate([cells, cells[:1]])))
    assert e.value.status == -4
    bad = cells.copy(); bad[2, 1] = 10 ** 6
    with pytest.raises(P.CrError):
        P.cr_build_mesh(tg(coords), tg(bad))


# ------------------------------------------------------------------ hybridisation
HYB_CASES = {
    "2d-config0": dict(dim=2, n=8, jitter=0.0),
    "2d-transient-jit-n17": dict(dim=2, n=17),
    "2d-steady-mis-n16": dict(dim=2, n=16, mu=0.0, shift="mis", force="gaussian"),
    "2d-ns-n12": dict(dim=2, n=12, mu=0.0, nu=0.01, shift="mis", force="zero", ns=True, jitter=0.0),
    "2d-dirichlet-n10": dict(dim=2, n=10, dirichlet=True),
    "2d-k0-interior": dict(dim=2, n=9, k0=77),
    "3d-transient-n3": dict(dim=3, n=3),
    "3d-steady-mis-n3": dict(dim=3, n=3, mu=0.0, shift="mis", force="gaussian"),
    # unstructured topologies (vertex valences 4..8 in 2D, varying edge valences in 3D)
    "2d-flip-transient-n14": dict(dim=2, n=14, flip=3),
    "2d-flip-steady-mis-n12": dict(dim=2, n=12, mu=0.0, shift="mis", force="gaussian", flip=4),
    "3d-flip-transient-n4": dict(dim=3, n=4, flip=5),
}


@pytest.mark.parametrize("name", list(HYB_CASES))
def test_hybridise_parity(name):
    coords, cells, prm, data, prob = make_case(**HYB_CASES[name])
    mo = O.build_mesh(coords, cells)
    ho = O.hybridise(mo, prm, data)
    mg = P.cr_build_mesh(tg(coords), tg(cells))
    hg = P.cr_hybridise(mg, prob)
    rp, cols, vals, S = hg.export_csr()
    Gg = to_scipy(rp, cols, vals, hg.n_rows)
    assert hg.nnz == ho["G"].nnz
    assert same_pattern(Gg, ho["G"])
    assert row_rel_err(Gg, ho["G"]) <= 1e-12
    Sg = S.cpu().numpy()
    assert np.abs(Sg - ho["S"]).max() <= 1e-12 * np.abs(ho["S"]).max()
    if prm.shift == "mis":
        inM1, E = hg.export_shift()
        assert np.array_equal(inM1.cpu().numpy().astype(bool), ho["inM1"])
        Eg = E.cpu().numpy()
        assert np.abs(Eg - ho["E"]).max() <= 1e-15 * np.abs(ho["E"]).max()


@pytest.mark.parametrize("name", ["2d-config0", "3d-transient-n3", "2d-ns-n12"])
def test_spmv_parity(name):
    coords, cells, prm, data, prob = make_case(**HYB_CASES[name])
    mo = O.build_mesh(coords, cells)
    ho = O.hybridise(mo, prm, data)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    x = np.random.default_rng(3).normal(size=hg.n_rows)
    y = torch.empty(hg.n_rows, dtype=torch.float64, device=DEV)
    hg.spmv(tg(x), y)
    yo = ho["G"] @ x
    assert np.abs(y.cpu().numpy() - yo).max() <= 1e-13 * np.abs(ho["G"]).max() * np.abs(x).max() * 10


# larger meshes (many 32-cell slices: faces whose two cells sit in different warps take the atomic
# path; ragged last slices), structured, Dirichlet and unstructured
MF_BLOCK_CASES = {
    "2d-jit-n48": dict(dim=2, n=48),
    "2d-dirichlet-n41": dict(dim=2, n=41, dirichlet=True),
    "2d-flip-n40": dict(dim=2, n=40, flip=3),
    "3d-n8": dict(dim=3, n=8),
    "3d-flip-n7": dict(dim=3, n=7, flip=5),
}


@pytest.mark.parametrize("name", ["2d-config0", "2d-transient-jit-n17", "2d-dirichlet-n10", "2d-k0-interior",
                                  "3d-transient-n3", "2d-flip-transient-n14", "3d-flip-transient-n4"]
                         + list(MF_BLOCK_CASES))
def test_matrix_free_spmv_parity(name):
    """y = sum_K H_K G_K H_K^t x from per-cell factors (Shat^{-1} split as 1/(mu|K|) 11^t + T,
    u = w/sqrt(B)) against the oracle's assembled G (entries rounded once from binary128); two
    applications are bitwise equal (exactly two contributions meet at a face: 0 + a + b)."""
    coords, cells, prm, data, prob = make_case(**(HYB_CASES.get(name) or MF_BLOCK_CASES[name]))
    mo = O.build_mesh(coords, cells)
    ho = O.hybridise(mo, prm, data)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    x = np.random.default_rng(7).normal(size=hg.n_rows)
    y = torch.empty(hg.n_rows, dtype=torch.float64, device=DEV)
    hg.spmv_mf(tg(x), y)
    yo = ho["G"] @ x
    Ga = abs(ho["G"])
    bound = 1e-14 * (Ga @ np.abs(x))            # rounding of G's entries, row by row
    assert np.all(np.abs(y.cpu().numpy() - yo) <= 4 * bound + 1e-300)
    y2 = torch.full_like(y, np.nan)
    hg.spmv_mf(tg(x), y2)
    assert torch.equal(y, y2)
    info = hg.mf_info()
    assert info["ncells"] >= mo.nc and info["bytes"] > 0


@pytest.mark.parametrize("name", ["2d-config0", "2d-ns-n12", "2d-dirichlet-n10", "3d-transient-n3"])
def test_coupled_parity(name):
    coords, cells, prm, data, prob = make_case(**HYB_CASES[name])
    mo = O.build_mesh(coords, cells)
    M, rhs, nU = O.assemble_coupled(mo, prm, data)
    cg = P.cr_assemble_coupled(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    rp, cols, vals, rg = cg.export_csr()
    Mg = to_scipy(rp, cols, vals, cg.n_rows)
    assert Mg.shape == M.shape and same_pattern(Mg, M)
    assert row_rel_err(Mg, M) <= 1e-12
    assert np.abs(rg.cpu().numpy() - rhs).max() <= 1e-12 * max(np.abs(rhs).max(), 1e-300)


# ------------------------------------------------------------------ solve + recover
SOLVE_CASES = {
    "config0-pcg": (dict(dim=2, n=8, jitter=0.0), "pcg", 1e-12),
    "2d-jit-n24-pcg-block": (dict(dim=2, n=24), "pcg_block", 1e-12),
    "2d-steady-n16-minres": (dict(dim=2, n=16, mu=0.0, shift="mis", force="gaussian"), "minres", 1e-12),
    "2d-ns-nu1-n8-bicgstab": (dict(dim=2, n=8, mu=0.0, nu=1.0, shift="mis", force="zero", ns=True, jitter=0.0),
                              "bicgstab", 1e-11),
    "2d-ns-nu1-n4-gmres": (dict(dim=2, n=4, mu=0.0, nu=1.0, shift="mis", force="zero", ns=True, jitter=0.0),
                           "gmres", 1e-12),
    "3d-n3-pcg": (dict(dim=3, n=3), "pcg", 1e-12),
    "2d-dirichlet-n10-pcg": (dict(dim=2, n=10, dirichlet=True), "pcg", 1e-12),
    "config0-pcg-afw": (dict(dim=2, n=8, jitter=0.0), "pcg_afw", 1e-12),
    "2d-jit-n24-pcg-afw": (dict(dim=2, n=24), "pcg_afw", 1e-12),
    "3d-n3-pcg-afw": (dict(dim=3, n=3), "pcg_afw", 1e-12),
    "2d-steady-n16-minres-afw": (dict(dim=2, n=16, mu=0.0, shift="mis", force="gaussian"), "minres_afw", 1e-12),
}


MF_CASES = {   # the matrix-free factored operator (transient Stokes)
    "config0-pcg-mf": (dict(dim=2, n=8, jitter=0.0), "pcg", 1e-12),
    "2d-jit-n24-pcg-afw-mf": (dict(dim=2, n=24), "pcg_afw", 1e-12),
    "3d-n3-pcg-afw-mf": (dict(dim=3, n=3), "pcg_afw", 1e-12),
    "2d-dirichlet-n10-pcg-afw-mf": (dict(dim=2, n=10, dirichlet=True), "pcg_afw", 1e-12),
    "2d-k0-interior-pcg-mf": (dict(dim=2, n=9, k0=77), "pcg", 1e-12),
    "2d-jit-n24-pcg-afw2-mf": (dict(dim=2, n=24), "pcg_afw2", 1e-12),
    "3d-n4-pcg-afw2-mf": (dict(dim=3, n=4), "pcg_afw2", 1e-12),
    "2d-dirichlet-n16-pcg-afw2-mf": (dict(dim=2, n=16, dirichlet=True), "pcg_afw2", 1e-12),
}
SOLVE_CASES["2d-jit-n24-pcg-afw2"] = (dict(dim=2, n=24), "pcg_afw2", 1e-12)
# unstructured topologies: patch (KMAX 8 / 16 paths) and two-level solves, assembled and matrix-free
SOLVE_CASES.update({
    "2d-flip-n20-pcg-afw": (dict(dim=2, n=20, flip=3), "pcg_afw", 1e-12),
    "3d-flip-n4-pcg-afw": (dict(dim=3, n=4, flip=5), "pcg_afw", 1e-12),
    "2d-flip-steady-n12-minres-afw": (dict(dim=2, n=12, mu=0.0, shift="mis", force="gaussian", flip=4), "minres_afw",
                                      1e-12),
    # MINRES with |patch| + the coarse |E|^-1 (SPD two-level preconditioner of the indefinite G)
    "2d-steady-n16-minres-afw2": (dict(dim=2, n=16, mu=0.0, shift="mis", force="gaussian"), "minres_afw2", 1e-12),
    "2d-flip-steady-n12-minres-afw2": (dict(dim=2, n=12, mu=0.0, shift="mis", force="gaussian", flip=4),
                                       "minres_afw2", 1e-12),
    "3d-steady-n3-minres-afw2": (dict(dim=3, n=3, mu=0.0, shift="mis", force="gaussian"), "minres_afw2", 1e-12),
})
MF_CASES.update({
    "2d-flip-n20-pcg-afw2-mf": (dict(dim=2, n=20, flip=3), "pcg_afw2", 1e-12),
    "3d-flip-n4-pcg-afw2-mf": (dict(dim=3, n=4, flip=5), "pcg_afw2", 1e-12),
})
# coupled defect correction (CR_DC_FGMRES): steady Stokes and NS steps, target residual 1e-11
SOLVE_CASES.update({
    "2d-steady-n16-dc": (dict(dim=2, n=16, mu=0.0, shift="mis", force="gaussian"), "dc", 1e-11),
    "2d-steady-dirichlet-n12-dc": (dict(dim=2, n=12, mu=0.0, shift="mis", force="gaussian", dirichlet=True),
                                   "dc", 1e-11),
    "2d-steady-k0-interior-dc": (dict(dim=2, n=10, mu=0.0, shift="mis", force="gaussian", k0=57), "dc", 1e-11),
    "3d-steady-n3-dc": (dict(dim=3, n=3, mu=0.0, shift="mis", force="gaussian"), "dc", 1e-11),
    "2d-ns-nu001-n12-dc": (dict(dim=2, n=12, mu=0.0, nu=0.01, shift="mis", force="zero", ns=True, jitter=0.0),
                           "dc", 1e-11),
    "2d-ns-nu1-n8-dc": (dict(dim=2, n=8, mu=0.0, nu=1.0, shift="mis", force="zero", ns=True, jitter=0.0),
                        "dc", 1e-11),
    "2d-transient-n16-dc": (dict(dim=2, n=16, mu=1.0), "dc", 1e-11),
})


@pytest.mark.parametrize("name", list(SOLVE_CASES) + list(MF_CASES))
def test_solve_recover_parity(name):
    mf = name in MF_CASES
    kw, method, rtol = MF_CASES[name] if mf else SOLVE_CASES[name]
    coords, cells, prm, data, prob = make_case(**kw)
    mo = O.build_mesh(coords, cells)
    ho = O.hybrid_pipeline(mo, prm, data)
    mg = P.cr_build_mesh(tg(coords), tg(cells))
    hg = P.cr_hybridise(mg, prob)
    W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
    extra = dict(restart=128) if method == "gmres" else {}
    rep = P.cr_solve(hg, W, method, rtol=rtol, check_every=16, matrix_free=int(mf), **extra)
    assert rep["converged"] and rep["rel_res_true"] <= rtol, rep
    if method == "dc":
        # outer iterations: mesh-independent for Stokes; the coarse nu = 0.01
        # NS mesh (cell Reynolds number ~ 8) needs more
        assert 0 < rep["iterations"] <= (150 if "nu001" in name else 30) and rep["inner_iterations"] > 0, rep
    # the oracle recomputes the true residual of the GPU solution in binary128
    r = O.residual_f128(ho["G"], W.cpu().numpy(), ho["S"])
    assert np.linalg.norm(r) <= 1.5 * rtol * np.linalg.norm(ho["S"])
    U, Pp, diag = P.cr_recover(hg, W)
    assert relL2(U.cpu().numpy(), ho["U"]) <= 1e-8
    assert relL2(Pp.cpu().numpy(), ho["P"]) <= 1e-8
    d = diag.cpu().numpy()
    umax = max(np.abs(ho["U"]).max(), 1.0)
    amax = np.abs(mo.a).max()
    assert d[0] <= 1e-9 * umax                                   # the two copies agree
    # full-face divergence of the assembled U: per copy it is D_K^t Uhat_K - g_K = B_K dP_K, i.e.
    # the rounding of P_K times B_K; across copies add sum_sigma sum_i |a_sigma^i| |dU| <=
    # (d+1) d amax * copy disagreement.  Factor 2 covers the per-copy rounding term.
    assert d[1] <= 2 * (mo.dim + 1) * mo.dim * amax * d[0] + 1e-12 * amax * umax


def test_recover_is_exact_given_W():
    """Recovery alone: oracle per-cell recovery from the GPU's own W (bit-level agreement)."""
    coords, cells, prm, data, prob = make_case(dim=2, n=12, mu=0.0, shift="mis", force="gaussian")
    mo = O.build_mesh(coords, cells)
    ho = O.hybridise(mo, prm, data)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    W = np.random.default_rng(5).normal(size=hg.n_rows)
    U, Pp, _ = P.cr_recover(hg, tg(W))
    Uo, Po, _, _ = O.recover(mo, prm, data, ho["E"], W)
    assert np.abs(Pp.cpu().numpy() - Po).max() <= 1e-13 * np.abs(Po).max()
    assert np.abs(U.cpu().numpy() - Uo).max() <= 1e-13 * np.abs(Uo).max()


@pytest.mark.parametrize("dim,n", [(2, 256), (3, 10)])
def test_well_balanced_closed_form_gpu(dim, n):
    """constant force -> U = 0 and P_K = f.(x_K - x_K0), on the GPU alone."""
    f = [0.7, -1.3] if dim == 2 else [0.7, -1.3, 0.4]
    coords, cells, prm, data, prob = make_case(dim=dim, n=n, force=f)
    out = P.hybrid_method(tg(coords), tg(cells), prob, "pcg", rtol=1e-12)
    xK = out["mesh"].export()["xK"].cpu().numpy()
    Pex = (xK - xK[0]) @ np.asarray(f)
    assert out["U"].abs().max().item() < 1e-10
    # P is kappa(G)-limited: relative 1e-8 (the north star's U/P bar)
    assert np.abs(out["P"].cpu().numpy() - Pex).max() <= 1e-8 * np.abs(Pex).max()


def test_zero_rhs_gives_zero():
    coords, cells, prm, data, prob = make_case(dim=2, n=6, force="zero")
    out = P.hybrid_method(tg(coords), tg(cells), prob, "pcg")
    assert out["W"].abs().max().item() == 0.0 and out["P"].abs().max().item() == 0.0


def test_host_entry_point_matches_device_path():
    coords, cells, prm, data, prob = make_case(dim=2, n=8)
    out = P.hybrid_method_host(torch.from_numpy(coords).pin_memory(), torch.from_numpy(cells).pin_memory(),
                               torch.from_numpy(data.fbar).pin_memory(), 1.0, 1.0, rtol=1e-12)
    ho = O.hybrid_pipeline(O.build_mesh(coords, cells), prm, data)
    assert relL2(out["U_host"].numpy(), ho["U"]) <= 1e-8 and relL2(out["P_host"].numpy(), ho["P"]) <= 1e-8


# ------------------------------------------------------------------ patch preconditioner
def _patches(mo):
    """Independent construction of the patches: interior faces around each vertex (2D) or
    around each edge (3D), faces in ascending dof order."""
    from collections import defaultdict
    import itertools
    pt = defaultdict(list)
    for f in np.nonzero(mo.face_dof >= 0)[0]:
        t = sorted(mo.faces[f])
        keys = t if mo.dim == 2 else list(itertools.combinations(t, 2))
        for k in keys:
            pt[tuple(np.atleast_1d(k))].append(mo.face_dof[f])
    return [np.array(sorted(v)) for _, v in sorted(pt.items())]


def _afw_numpy(G, pats, d, r, kind):
    """kind "inv" (PCG): one block per patch, the mean of the d component blocks R_p G^(ii) R_p^t,
    inverted and applied to every component; "abs" (MINRES): |block| per component."""
    G = G.tocsr()
    z = np.zeros_like(r)
    for p in pats:
        if kind == "inv":
            Bm = sum(G[p * d + i][:, p * d + i].toarray() for i in range(d)) / d
            Bi = np.linalg.inv(Bm)
        for i in range(d):
            ii = p * d + i
            if kind == "abs":
                B = G[ii][:, ii].toarray()
                w, V = np.linalg.eigh(0.5 * (B + B.T))
                Bi = (V / np.abs(w)) @ V.T
            z[ii] += Bi @ r[ii]
    return z


@pytest.mark.parametrize("name,method,kind", [("2d-transient-jit-n17", "pcg_afw", "inv"),
                                              ("3d-transient-n3", "pcg_afw", "inv"),
                                              ("2d-steady-mis-n16", "minres_afw", "abs"),
                                              ("2d-flip-transient-n14", "pcg_afw", "inv"),
                                              ("2d-flip-steady-mis-n12", "minres_afw", "abs"),
                                              ("3d-flip-transient-n4", "pcg_afw", "inv"),
                                              # larger meshes (many slices, ragged last slice)
                                              ("2d-jit-n48", "pcg_afw", "inv"),
                                              ("2d-flip-n40", "pcg_afw", "inv"),
                                              ("3d-n8", "pcg_afw", "inv"),
                                              ("3d-flip-n7", "pcg_afw", "inv")])
def test_patch_preconditioner_apply(name, method, kind):
    """z = sum_p R_p^t B_p^{-1} R_p r on the GPU vs numpy from the oracle's G; bitwise reproducible
    (each face's SLOTS patch contributions are summed in slot order)."""
    coords, cells, prm, data, prob = make_case(**(HYB_CASES.get(name) or MF_BLOCK_CASES[name]))
    mo = O.build_mesh(coords, cells)
    ho = O.hybridise(mo, prm, data)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    r = np.random.default_rng(11).normal(size=hg.n_rows)
    z = torch.empty(hg.n_rows, dtype=torch.float64, device=DEV)
    hg.apply_precond(method, tg(r), z)
    pats = _patches(mo)
    info = hg.precond_info()
    assert info["npatch"] == len(pats) and info["nfallback"] == 0
    assert info["kmax"] == max(len(p) for p in pats)
    if "flip" in name:
        assert info["kmax"] == 8          # the KMAX = 8 kernels (structured meshes stop at 6)
    zo = _afw_numpy(ho["G"], pats, mo.dim, r, kind)
    assert relL2(z.cpu().numpy(), zo) <= 1e-9
    z2 = torch.full_like(z, np.nan)
    hg.apply_precond(method, tg(r), z2)
    assert torch.equal(z, z2)


@pytest.mark.parametrize("dim,n,method", [(2, 40, "pcg_afw2"), (3, 8, "pcg_afw2"), (3, 6, "pcg_afw"),
                                          (2, 33, "pcg_afw")])
def test_solve_order_matches_mesh_order(dim, n, method, monkeypatch):
    """The matrix-free patch-preconditioned PCG runs on the rows renumbered in the cells' visiting
    order (h->so): same operator, same preconditioner, only the reductions' order
    differs — W agrees with the mesh-order solve (CR_SOLVE_ORDER=0) and the counts match."""
    coords, cells, prm, data, prob = make_case(dim=dim, n=n, seed=3)
    mesh = P.cr_build_mesh(tg(coords), tg(cells))
    out = {}
    for so in ("1", "0"):
        monkeypatch.setenv("CR_SOLVE_ORDER", so)
        hg = P.cr_hybridise(mesh, prob)
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        rep = P.cr_solve(hg, W, method, rtol=1e-11, matrix_free=1)
        assert rep["converged"] and rep["rel_res_true"] <= 1e-11
        out[so] = (W.cpu().numpy(), rep["iterations"])
    assert abs(out["1"][1] - out["0"][1]) <= 2, (out["1"][1], out["0"][1])
    assert relL2(out["1"][0], out["0"][0]) <= 1e-9


def test_solve_profile_times_the_iteration_and_leaves_the_solve_unchanged():
    """cr_solve_profile launches the iteration's kernel groups on the handle's buffers (after a solve)
    and times them; a later solve from the same W reproduces the first one bit for bit."""
    coords, cells, prm, data, prob = make_case(dim=3, n=6, seed=5)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    sols = []
    for k in range(2):
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        rep = P.cr_solve(hg, W, "pcg_afw2", rtol=1e-11, matrix_free=1, coarse=2)
        sols.append((W.cpu().numpy(), rep["iterations"]))
        if k == 0:
            ms = P.cr_solve_profile(hg, "pcg_afw2", nrep=3, coarse=2)
            assert set(ms) == set(P.SOLVE_PROFILE_KERNELS) and all(v > 0 for v in ms.values()), ms
    assert sols[0][1] == sols[1][1] and np.array_equal(sols[0][0], sols[1][0])
    with pytest.raises(P.CrError):
        P.cr_solve_profile(P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob), "pcg_afw2")


def test_two_level_cuts_pcg_iterations():
    """The coarse 'stress x area' space removes the h-dependence left by the patches: at n = 64
    (numpy on the oracle's G: 882 -> 109 iterations with 16 coarse intervals)."""
    coords, cells, prm, data, prob = make_case(dim=2, n=64, seed=2)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    its = {}
    for m in ("pcg_afw", "pcg_afw2"):
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        its[m] = P.cr_solve(hg, W, m, rtol=1e-10, matrix_free=1)["iterations"]
    assert its["pcg_afw2"] * 4 <= its["pcg_afw"], its


@pytest.mark.parametrize("dim,n,H", [(2, 64, 8), (2, 96, 24), (3, 8, 4), (3, 12, 6)])
def test_coarse_nd_matches_dense_inverse(dim, n, H, monkeypatch):
    """The nested-dissection coarse solve (multifrontal, explicit front inverses) against the
    dense Gauss-Jordan E^{-1} on the same E = Z^t G Z: the two-level preconditioner applied to
    one vector, and the PCG iteration counts."""
    coords, cells, prm, data, prob = make_case(dim=dim, n=n, seed=4)
    mesh = P.cr_build_mesh(tg(coords), tg(cells))
    r = tg(np.random.default_rng(9).normal(size=dim * int(mesh.nf_int)))
    out = {}
    for mode in ("CR_COARSE_DENSE", "CR_COARSE_ND"):
        monkeypatch.delenv("CR_COARSE_DENSE", raising=False)
        monkeypatch.delenv("CR_COARSE_ND", raising=False)
        monkeypatch.setenv(mode, "1")
        hg = P.cr_hybridise(mesh, prob)
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        rep = P.cr_solve(hg, W, "pcg_afw2", rtol=1e-10, matrix_free=1, coarse=H)
        z = torch.empty_like(r)
        hg.apply_precond("pcg_afw2", r, z)
        out[mode] = (z.cpu().numpy(), rep["iterations"])
    # E is SPD but ill-conditioned (its fp32 rounding already stalls PCG): the two exact
    # inverses agree to kappa(E) * eps
    assert relL2(out["CR_COARSE_ND"][0], out["CR_COARSE_DENSE"][0]) <= 1e-9
    assert abs(out["CR_COARSE_ND"][1] - out["CR_COARSE_DENSE"][1]) <= 1


@pytest.mark.parametrize("dim,n,H,mode", [(2, 48, 8, "CR_COARSE_DENSE"), (2, 64, 8, "CR_COARSE_ND"),
                                          (3, 8, 4, "CR_COARSE_ND")])
def test_coarse_weight_is_linear_in_the_coarse_term(dim, n, H, mode, monkeypatch):
    """CR_COARSE_WEIGHT = theta scales E by 1/theta before it is inverted / factorised:
    M2(theta)^-1 r = M_patch^-1 r + theta Z E^-1 Z^t r, so z(2) = 2 z(1) - z_patch, and the weighted
    two-level PCG still reaches the same solution."""
    coords, cells, prm, data, prob = make_case(dim=dim, n=n, seed=6)
    mesh = P.cr_build_mesh(tg(coords), tg(cells))
    r = tg(np.random.default_rng(11).normal(size=dim * int(mesh.nf_int)))
    monkeypatch.setenv(mode, "1")
    z, Ws = {}, {}
    for th in ("1", "2"):
        monkeypatch.setenv("CR_COARSE_WEIGHT", th)
        hg = P.cr_hybridise(mesh, prob)
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        rep = P.cr_solve(hg, W, "pcg_afw2", rtol=1e-11, matrix_free=1, coarse=H)
        assert rep["converged"]
        zz = torch.empty_like(r)
        hg.apply_precond("pcg_afw2", r, zz)
        z[th], Ws[th] = zz.cpu().numpy(), W.cpu().numpy()
        if th == "1":
            zp = torch.empty_like(r)
            hg.apply_precond("pcg_afw", r, zp)
            zp = zp.cpu().numpy()
    assert relL2(z["2"], 2.0 * z["1"] - zp) <= 1e-9
    assert np.linalg.norm(z["1"] - zp) > 1e-3 * np.linalg.norm(zp)   # the coarse term is not negligible
    assert relL2(Ws["2"], Ws["1"]) <= 1e-8


def test_patch_preconditioner_cuts_pcg_iterations():
    """The patch preconditioner resolves the two scales of G: >= 4x fewer PCG iterations than
    Jacobi at n = 32 (numpy experiment: 3186 vs 429)."""
    coords, cells, prm, data, prob = make_case(dim=2, n=32, seed=2)
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    its = {}
    for m in ("pcg", "pcg_afw"):
        W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
        its[m] = P.cr_solve(hg, W, m, rtol=1e-10)["iterations"]
    assert its["pcg_afw"] * 4 <= its["pcg"], its


# ------------------------------------------------------------------ partitioned path (multi-GPU)
@pytest.mark.timeout(600)
@pytest.mark.parametrize("dim,n,nranks,method", [(2, 12, 2, "pcg"), (2, 12, 3, "pcg_afw"), (2, 10, 2, "pcg_block"),
                                                 (3, 3, 2, "pcg_afw"), (3, 4, 4, "pcg"), (2, 12, 3, "pcg_afw_mf"),
                                                 (3, 3, 2, "pcg_mf"), (2, 16, 3, "pcg_afw2_mf"), (3, 4, 2, "pcg_afw2")])
def test_partitioned_loopback(dim, n, nranks, method):
    """The row-partitioned path (local assembly with renumbered columns, halo exchange before
    every SpMV, allreduced dot products, W gathered for the recovery) with `nranks` ranks as
    threads of this process on one GPU (loopback communicator): each rank's rows of
    G and S equal the oracle's, and every rank recovers the oracle's U and P."""
    import threading
    coords, cells, prm, data, prob = make_case(dim=dim, n=n)
    mo = O.build_mesh(coords, cells)
    ho = O.hybrid_pipeline(mo, prm, data)
    grp = P.LoopbackGroup(nranks)
    res, errs = [None] * nranks, []
    xglob = np.random.default_rng(12).normal(size=mo.nf_int * mo.dim)

    def run(rank):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = P.Comm.loopback(grp, rank)
                c, k = tg(coords), tg(cells)
                mf = method.endswith("_mf")
                out = P.hybrid_method(c, k, prob, method[:-3] if mf else method, rtol=1e-12, stream=st, comm=comm,
                                      check_every=16, matrix_free=int(mf))
                rp, cols, vals, S = out["hybrid"].export_csr(st)
                inf = out["hybrid"].partition_info()
                ymf = None
                if mf:   # cr_spmv_mf on a partitioned handle: halo exchange inside (collective)
                    xl = tg(xglob[inf["row0"] * mo.dim:inf["row1"] * mo.dim])
                    ymf = torch.empty_like(xl)
                    out["hybrid"].spmv_mf(xl, ymf, st)
                st.synchronize()
                res[rank] = dict(out=out, info=inf, ymf=None if ymf is None else ymf.cpu().numpy(), rp=rp.cpu().numpy(),
                                 cols=cols.cpu().numpy(), vals=vals.cpu().numpy(), S=S.cpu().numpy(),
                                 U=out["U"].cpu().numpy(), P=out["P"].cpu().numpy())
        except Exception as e:   # pragma: no cover
            errs.append(repr(e))

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    d = mo.dim
    Go = ho["G"].tocsr()
    rows_seen = 0
    for rank, r in enumerate(res):
        inf = r["info"]
        assert inf["nglobal"] == mo.nf_int
        r0, r1 = inf["row0"], inf["row1"]
        rows_seen += r1 - r0
        Gl = sp.csr_matrix((r["vals"], r["cols"], r["rp"]), shape=((r1 - r0) * d, mo.nf_int * d))
        Gref = Go[r0 * d:r1 * d]
        assert same_pattern(Gl, Gref)
        assert row_rel_err(Gl, Gref) <= 1e-12
        assert np.abs(r["S"] - ho["S"][r0 * d:r1 * d]).max() <= 1e-12 * np.abs(ho["S"]).max()
        assert relL2(r["U"], ho["U"]) <= 1e-8 and relL2(r["P"], ho["P"]) <= 1e-8
        assert np.array_equal(r["U"], res[0]["U"]) and np.array_equal(r["P"], res[0]["P"])
        assert r["out"]["report"]["converged"]
        if r["ymf"] is not None:
            yref = (Go @ xglob)[r0 * d:r1 * d]
            assert np.abs(r["ymf"] - yref).max() <= 1e-11 * np.abs(Go).max() * np.abs(xglob).max()
    assert rows_seen == mo.nf_int


def test_nccl_single_rank_partitioned_path():
    """The NCCL communicator (dlopen'ed libnccl, allreduce + send/recv enqueued inside the
    solver's CUDA graphs) on one rank: same answer as the unpartitioned solve."""
    coords, cells, prm, data, prob = make_case(dim=2, n=12)
    comm = P.Comm.nccl(P.nccl_unique_id(), 0, 1)
    out = P.hybrid_method(tg(coords), tg(cells), prob, "pcg_afw", rtol=1e-12, comm=comm, check_every=8)
    ref = P.hybrid_method(tg(coords), tg(cells), prob, "pcg_afw", rtol=1e-12, check_every=8)
    assert out["hybrid"].partition_info()["nghost"] == 0
    assert out["report"]["iterations"] == ref["report"]["iterations"]
    assert relL2(out["U"].cpu().numpy(), ref["U"].cpu().numpy()) <= 1e-12
    assert relL2(out["P"].cpu().numpy(), ref["P"].cpu().numpy()) <= 1e-10


# ------------------------------------------------------------------ time stepping
@pytest.mark.parametrize("dim,n,nsteps", [(2, 16, 3), (3, 3, 2)])
def test_time_march_matches_oracle(dim, n, nsteps):
    """Backward Euler with the same G every step (cr_transient_rhs + cr_hybrid_set_cell_rhs,
    warm-started two-level PCG) against the oracle's per-step refined direct solves."""
    coords, cells, prm, data, prob = make_case(dim=dim, n=n, force="gaussian", seed=5)
    mo = O.build_mesh(coords, cells)
    U0 = np.random.default_rng(6).normal(size=(mo.nf_int, dim))
    Uo, Po = O.backward_euler(mo, prm, data, nsteps, U0=U0)
    out = P.time_march(tg(coords), tg(cells), prob, nsteps, U0=tg(U0), method="pcg_afw2", rtol=1e-12,
                       matrix_free=1, check_every=16)
    for k in range(nsteps):
        assert relL2(out["U"][k].cpu().numpy(), Uo[k]) <= 1e-8, k
        assert relL2(out["P"][k].cpu().numpy(), Po[k]) <= 1e-8, k
        assert out["reports"][k]["converged"]
    # restoring the data-derived right-hand side gives back the original S
    hg = out["hybrid"]
    S1 = hg.export_csr()[3].clone()
    R, g = hg.transient_rhs(torch.zeros((mo.nf_int, dim), dtype=torch.float64, device=DEV))
    hg.set_cell_rhs(R, g)          # mu M 0 = 0: the same S from explicit cell terms
    S2 = hg.export_csr()[3].clone()
    hg.set_cell_rhs()
    S3 = hg.export_csr()[3]
    ho = O.hybridise(mo, prm, data)
    assert np.abs(S2.cpu().numpy() - ho["S"]).max() <= 1e-12 * np.abs(ho["S"]).max()
    assert np.abs(S3.cpu().numpy() - ho["S"]).max() <= 1e-12 * np.abs(ho["S"]).max()
    assert S1.shape == S3.shape


def test_time_march_warm_start_cuts_iterations():
    """Later steps start from the previous W: fewer iterations than a cold start."""
    coords, cells, prm, data, prob = make_case(dim=2, n=48, force="gaussian", seed=7)
    kw = dict(method="pcg_afw2", rtol=1e-12, matrix_free=1, check_every=8)
    warm = P.time_march(tg(coords), tg(cells), prob, 4, **kw)
    cold = P.time_march(tg(coords), tg(cells), prob, 4, warm_start=False, **kw)
    wi = [r["iterations"] for r in warm["reports"]]
    ci_ = [r["iterations"] for r in cold["reports"]]
    assert sum(wi[1:]) < sum(ci_[1:]), (wi, ci_)
    for a, b in zip(warm["U"], cold["U"]):
        assert relL2(a.cpu().numpy(), b.cpu().numpy()) <= 1e-8


# ------------------------------------------------------------------ Newton for steady NS
@pytest.mark.parametrize("n,nu", [(8, 0.1), (12, 0.01)])
def test_newton_ns_matches_oracle(n, nu):
    """Lid-driven cavity: Newton steps through cr_cell_face_values + cr_hybridise (NS step, MIS
    shift) + CR_DC_FGMRES + cr_recover, against the oracle's Newton with refined direct solves."""
    coords, cells = ci.square_mesh(n, 0.0, 4)
    mo = O.build_mesh(coords, cells)
    wall = ci.lid_dirichlet_2d(coords, cells)
    f = np.zeros((mo.nc, 2))
    Uo, Po, ho = O.newton_ns(mo, O.Params(mu=0.0, nu=nu, physics="ns_step"), f, wall, tol=1e-10)
    out = P.newton_ns(tg(coords), tg(cells), nu, tg(f), tg(wall), tol=1e-10, mis_seed=11, rtol=1e-12)
    assert abs(len(out["history"]) - len(ho)) <= 1, (out["history"], ho)
    assert relL2(out["U"].cpu().numpy(), Uo) <= 1e-8
    assert relL2(out["P"].cpu().numpy(), Po) <= 1e-8


# ------------------------------------------------------------------ direct solvers
@pytest.mark.parametrize("n", [2, 3])
def test_sparse_direct_hybrid_and_coupled(n):
    """Table 4's comparison on the GPU: sparse Cholesky of the hybrid G and sparse QR of the coupled
    matrix both give the oracle's (U, P) on a 3D Kuhn mesh (transient, dt = 5e-4)."""
    coords, cells, prm, data, prob = make_case(dim=3, n=n, mu=2000.0)
    mo = O.build_mesh(coords, cells)
    ho = O.hybrid_pipeline(mo, prm, data)
    mg = P.cr_build_mesh(tg(coords), tg(cells))
    hg = P.cr_hybridise(mg, prob)
    rp, ci_, v, S = hg.export_csr()
    W = P.sparse_direct_solve(rp, ci_, v, S, "chol")
    U, Pp, _ = P.cr_recover(hg, W)
    assert relL2(U.cpu().numpy(), ho["U"]) <= 1e-8 and relL2(Pp.cpu().numpy(), ho["P"]) <= 1e-8
    cg = P.cr_assemble_coupled(mg, prob)
    rp2, ci2, v2, rhs = cg.export_csr()
    x = P.sparse_direct_solve(rp2, ci2, v2, rhs, "qr").cpu().numpy()
    nU = 3 * mo.nf_int
    assert relL2(x[:nU].reshape(-1, 3), ho["U"]) <= 1e-8
    assert relL2(np.insert(x[nU:], 0, 0.0), ho["P"]) <= 1e-8


def test_damped_newton_re1000_matches_oracle():
    """The paper's steady lid-driven cavity at Re = 1000 (Table 7 right) by Armijo-damped
    Newton from rest: the GPU iteration (cr_coupled_rhs_norm line search, cr_newton_update with the
    step length, CR_DC_FGMRES linear solves) takes the oracle's steps and reaches its solution."""
    n, nu = 16, 1e-3
    coords, cells = ci.square_mesh(n, 0.0, 4)
    mo = O.build_mesh(coords, cells)
    wall = ci.lid_dirichlet_2d(coords, cells)
    f = np.zeros((mo.nc, 2))
    Uo, Po, ho = O.newton_ns(mo, O.Params(mu=0.0, nu=nu, physics="ns_step"), f, wall, tol=1e-10, damped=True,
                             max_newton=40)
    out = P.newton_ns(tg(coords), tg(cells), nu, tg(f), tg(wall), tol=1e-10, damped=True, max_newton=40, mis_seed=11,
                      rtol=1e-12)
    assert abs(len(out["history"]) - len(ho)) <= 1, (out["history"], ho)
    assert out["history"][-1] <= 1e-10
    assert relL2(out["U"].cpu().numpy(), Uo) <= 1e-8
    assert relL2(out["P"].cpu().numpy(), Po) <= 1e-8


def test_pool_and_launch_counter():
    """libcr's own memory pool (cr_pool_reserve / cr_pool_trim) and the launch counter: torch's
    allocator is untouched by a reservation, and a solve advances cr_kernel_launches by at least
    its reported kernel launches."""
    before = torch.cuda.memory_reserved()
    P.pool_reserve(256 << 20)
    assert torch.cuda.memory_reserved() == before          # the library's pool, not torch's
    coords, cells, prm, data, prob = make_case(dim=2, n=10)
    n0 = P.kernel_launches()
    out = P.hybrid_method(tg(coords), tg(cells), prob, "pcg_afw2", rtol=1e-12, matrix_free=1, check_every=8)
    n1 = P.kernel_launches()
    assert out["report"]["kernel_launches"] > 0 and n1 - n0 >= 0.5 * out["report"]["kernel_launches"]
    del out
    P.pool_trim(0)
