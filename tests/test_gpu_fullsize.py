"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

The oracle cannot solve these systems, so each stage is checked where the oracle CAN compute
the answer one item at a time, or by a property that holds at any size:
  * mesh: closed-form counts and the whole connectivity bit-exact vs the oracle;
  * hybridisation: sampled rows of G and S vs the oracle's binary128 elimination of the two
    cells of each sampled face (row-relative 1e-12); the steady shift (MIS membership, E)
    bit-exact / 1e-15 on every cell;
  * solve: the GPU's true residual <= 1e-10 (its G is the oracle's, by the sampled rows);
  * recovery: sampled cells recovered by the oracle from the GPU's own W;
  * well-balanced closed form at full size: constant force -> U = 0, P = f.(x_K - x_K0).
"""
import numpy as np
import pytest
import torch

import bench
import cr_inputs as ci
import oracle as O
from oracle.scheme import _gidx, shift_E, local_blocks

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

import paper_2101_03777_b200 as P  # noqa: E402

DEV = torch.device("cuda")
RNG = np.random.default_rng(2024)


def tg(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def counts(dim, n):
    if dim == 2:
        nb = (3 * n * n - 2 * n) + 12 * (n - 1) ** 2 + 8 * (n - 1)
        return dict(nc=2 * n * n, nf=3 * n * n + 2 * n, nf_int=3 * n * n - 2 * n, nb=nb)
    nb = (12 * n ** 3 - 6 * n * n) + 72 * n * (n - 1) ** 2 + 72 * n * (n - 1) + 12 * n
    return dict(nc=6 * n ** 3, nf=12 * n ** 3 + 6 * n * n, nf_int=12 * n ** 3 - 6 * n * n, nb=nb)


def problem(cfg, inp, prm_only=False):
    kw = {}
    if cfg.shift == "mis":
        kw.update(shift=P.CR_SHIFT_MIS, mis_seed=cfg.mis_seed)
    if cfg.physics == "ns_step":
        kw.update(physics=P.CR_NS_NEWTON_STEP, u_iter=tg(inp["u_iter"]))
    prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=tg(inp["fbar"]), **kw)
    prm = O.Params(mu=cfg.mu, nu=cfg.nu, shift=cfg.shift, mis_seed=cfg.mis_seed, physics=cfg.physics)
    data = O.Data(fbar=inp["fbar"], u_iter=inp["u_iter"])
    return prob, prm, data


def check_mesh(mo, mg, dim, n):
    c = counts(dim, n)
    assert (mg.nc, mg.nf, mg.nf_int) == (c["nc"], c["nf"], c["nf_int"])
    ex = mg.export()
    for k in ("faces", "face_cells", "cell_faces", "face_dof"):
        assert torch.equal(ex[k].cpu(), torch.from_numpy(getattr(mo, k))), k
    for k in ("vol", "xK", "a"):
        ref = getattr(mo, k)
        assert np.abs(ex[k].cpu().numpy() - ref).max() <= 1e-14 * np.abs(ref).max(), k


def sampled_rows(mo, prm, data, E, hg, nsample):
    """Rows of G (and S) for sampled block rows: GPU export vs oracle per-cell elimination."""
    d = mo.dim
    rp, cols, vals, S = hg.export_csr()
    rows = np.unique(np.concatenate([RNG.choice(mo.nf_int, nsample, replace=False), [0, mo.nf_int - 1]]))
    faces = mo.dof_face[rows]
    cells = np.unique(mo.face_cells[faces].ravel())
    cells = cells[cells >= 0]
    Gc, Sc, _ = O.eliminate_cells(mo, prm, data, E, cells)
    gi = _gidx(mo)[cells]
    pos = {int(K): j for j, K in enumerate(cells)}
    rp_h = rp.cpu().numpy()
    worst, worst_s, smax = 0.0, 0.0, 0.0
    for r, f in zip(rows, faces):
        ref = {}
        sref = np.zeros(d)
        for K in mo.face_cells[f]:
            if K < 0:
                continue
            j = pos[int(K)]
            l = int(np.nonzero(mo.cell_faces[K] == f)[0][0])
            for i in range(d):
                lr = l * d + i
                sref[i] += Sc[j, lr]
                for q in range(gi.shape[1]):
                    c = gi[j, q]
                    if c >= 0:
                        ref[(i, int(c))] = ref.get((i, int(c)), 0.0) + Gc[j, lr, q]
        for i in range(d):
            a, b = rp_h[r * d + i], rp_h[r * d + i + 1]
            gc = cols[a:b].cpu().numpy()
            gv = vals[a:b].cpu().numpy()
            refc = sorted(c for (ii, c) in ref if ii == i)
            assert list(gc) == refc                                        # pattern bit-exact
            rv = np.array([ref[(i, c)] for c in refc])
            worst = max(worst, np.abs(gv - rv).max() / np.abs(rv).max())
        worst_s = max(worst_s, np.abs(S[r * d:(r + 1) * d].cpu().numpy() - sref).max())
        smax = max(smax, np.abs(sref).max())
    return worst, worst_s / max(smax, 1e-300)     # S: relative to max |S| (as the small-mesh tests)


def sampled_recovery(mo, prm, data, E, W, U, Pg, nsample):
    cells = np.sort(RNG.choice(mo.nc, nsample, replace=False))
    Po, Uh = O.recover_cells(mo, prm, data, E, W, cells)
    Pg = Pg[cells]
    eP = np.abs(Pg - Po).max() / max(np.abs(Po).max(), 1e-300)
    eU, umax = 0.0, 0.0
    for j, K in enumerate(cells):
        for l in range(mo.dim + 1):
            f = mo.cell_faces[K, l]
            dof = mo.face_dof[f]
            if dof >= 0 and mo.face_cells[f, 0] == K:
                eU = max(eU, np.abs(U[dof] - Uh[j, l]).max())
                umax = max(umax, np.abs(Uh[j, l]).max())
    return eP, eU / max(umax, 1e-300)


# ------------------------------------------------------------------ configs[1]: the bench workload
def test_config1_full_size():
    cfg = ci.CONFIGS[1]
    inp = ci.make_inputs(cfg)
    prob, prm, data = problem(cfg, inp)
    mo = O.build_mesh(inp["coords"], inp["cells"])
    mg = P.cr_build_mesh(tg(inp["coords"]), tg(inp["cells"]))
    check_mesh(mo, mg, 2, cfg.n)
    hg = P.cr_hybridise(mg, prob)
    assert hg.nblocks == counts(2, cfg.n)["nb"]
    E = np.zeros((mo.nc, 3))
    eG, eS = sampled_rows(mo, prm, data, E, hg, 200)
    assert eG <= 1e-12 and eS <= 1e-12, (eG, eS)
    W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
    # the bench's solver (bench.SOLVERS[1]): two-level PCG on the matrix-free factored G
    sol = dict(bench.SOLVERS[1])
    rtol = sol.pop("rtol")
    rep = P.cr_solve(hg, W, rtol=rtol, check_every=64, **sol)
    assert rep["converged"] and rep["rel_res_true"] <= rtol
    U, Pp, diag = P.cr_recover(hg, W)
    eP, eU = sampled_recovery(mo, prm, data, E, W.cpu().numpy(), U.cpu().numpy(), Pp.cpu().numpy(), 400)
    assert eP <= 1e-11 and eU <= 1e-11, (eP, eU)
    # the discrete solution keeps the scheme's orders up to the full size (jittered
    # n = 128 gives errl2U 8.628e-4, errl2P 5.949e-2; U ~ h^2, P ~ h -> n = 1024: /64 and /8)
    u, p, _ = ci.manufactured_2d(cfg.mu, cfg.nu)
    eu, ep = O.errors(mo, U.cpu().numpy(), Pp.cpu().numpy(), u, p)
    assert 0.5 * 8.628e-4 / 64 < eu < 1.5 * 8.628e-4 / 64, eu
    assert 0.5 * 5.949e-2 / 8 < ep < 1.5 * 5.949e-2 / 8, ep


@pytest.mark.parametrize("dim,n", [(2, 1024)])
def test_well_balanced_full_size(dim, n):
    """P:L559 at the bench size: constant f -> U = 0 and P_K = f.(x_K - x_K0), through the
    bench's solver (two-level PCG, matrix-free G).  The factored G keeps the O(|K|) part of each
    Shat_K^{-1} exact, so P reaches the 1e-8 bar; the assembled fp64 G stalls at ~8e-7 here
    (DESIGN.md §5.2)."""
    coords, cells = ci.square_mesh(n, 0.2, 2)
    f = np.array([0.7, -1.3])
    prob = P.Problem(mu=1.0, nu=1.0, fbar=tg(np.tile(f, (cells.shape[0], 1))))
    sol = dict(bench.SOLVERS[1])
    rtol = sol.pop("rtol")
    out = P.hybrid_method(tg(coords), tg(cells), prob, rtol=rtol, **sol)
    xK = out["mesh"].export()["xK"].cpu().numpy()
    Pex = (xK - xK[0]) @ f
    assert out["U"].abs().max().item() <= 1e-8
    assert np.abs(out["P"].cpu().numpy() - Pex).max() <= 1e-8 * np.abs(Pex).max()


# ------------------------------------------------------------------ configs[2], configs[3]: shifted systems
@pytest.mark.parametrize("idx", [2, 3])
def test_shifted_configs_full_size_assembly(idx):
    """Steady Stokes (n = 1024) and one Navier-Stokes step (n = 512): the MIS shift on every
    cell and sampled rows of G and S at full size.  (Their Krylov solves do not reach 1e-10 at
    these sizes with a pointwise / patch preconditioner: DESIGN.md "Findings".)"""
    cfg = ci.CONFIGS[idx]
    inp = ci.make_inputs(cfg)
    prob, prm, data = problem(cfg, inp)
    mo = O.build_mesh(inp["coords"], inp["cells"])
    mg = P.cr_build_mesh(tg(inp["coords"]), tg(inp["cells"]))
    hg = P.cr_hybridise(mg, prob)
    A, _, _, _ = local_blocks(mo, prm, data)
    E, inM1, lam = shift_E(mo, prm, A)
    inM1g, Eg = hg.export_shift()
    assert np.array_equal(inM1g.cpu().numpy().astype(bool), inM1)
    # lambda_K comes from |K| and a_K, which agree with the oracle to 1e-14 (different but
    # equally exact determinant / cross-product orders), so E does too
    assert np.abs(Eg.cpu().numpy() - E).max() <= 1e-14 * np.abs(E).max()
    eG, eS = sampled_rows(mo, prm, data, E, hg, 150)
    assert eG <= 1e-12 and eS <= 1e-12, (eG, eS)
    # the solve: coupled FGMRES preconditioned by the transient hybrid solve (CR_DC_FGMRES),
    # stopped on the TARGET's true residual ||S - G W|| / ||S|| <= 1e-10 (G checked above)
    W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
    rep = P.cr_solve(hg, W, "dc", rtol=cfg.rtol, coarse=32, mu_inner=1.0 if idx == 2 else 0.5)
    assert rep["converged"] and rep["rel_res_true"] <= cfg.rtol, rep
    assert rep["iterations"] <= 30, rep
    U, Pp, diag = P.cr_recover(hg, W)
    eP, eU = sampled_recovery(mo, prm, data, E, W.cpu().numpy(), U.cpu().numpy(), Pp.cpu().numpy(), 200)
    assert eP <= 1e-11 and eU <= 1e-11, (eP, eU)


# ------------------------------------------------------------------ configs[4]: 3D
def test_config4_3d_full_size():
    cfg = ci.CONFIGS[4]
    inp = ci.make_inputs(cfg)
    prob, prm, data = problem(cfg, inp)
    mo = O.build_mesh(inp["coords"], inp["cells"])
    mg = P.cr_build_mesh(tg(inp["coords"]), tg(inp["cells"]))
    check_mesh(mo, mg, 3, cfg.n)
    hg = P.cr_hybridise(mg, prob)
    assert hg.nblocks == counts(3, cfg.n)["nb"]
    E = np.zeros((mo.nc, 4))
    eG, eS = sampled_rows(mo, prm, data, E, hg, 100)
    assert eG <= 1e-12 and eS <= 1e-12, (eG, eS)
    W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
    sol = dict(bench.SOLVERS[4])   # the bench's solver: two-level PCG, ND coarse solve, matrix-free G
    rtol = sol.pop("rtol")
    rep = P.cr_solve(hg, W, rtol=rtol, check_every=64, **sol)
    assert rep["converged"] and rep["rel_res_true"] <= rtol
    U, Pp, diag = P.cr_recover(hg, W)
    eP, eU = sampled_recovery(mo, prm, data, E, W.cpu().numpy(), U.cpu().numpy(), Pp.cpu().numpy(), 200)
    assert eP <= 1e-11 and eU <= 1e-11, (eP, eU)
