"""U and P of the BENCH's own solver against the oracle's coupled solution.

The hybrid method reaches exactly the solution of the coupled system eq. (syslin) (abstract
P:L13; "we get P_hat = P"), so the reference for U and P is oracle.assemble_coupled +
oracle.direct_refined (SuperLU + binary128-residual refinement).  The GPU side runs exactly what
bench.py times: bench.SOLVERS[cfg] (two-level PCG on the matrix-free factored G, the bench's
coarse grid and stopping tolerance), through the C ABI.  Bar (BASELINE.json north_star): relative
L2 <= 1e-8 for U and P.

Sizes: 2D n = 256 (configs[1] family: jittered 0.2h, manufactured force; reference computed here,
~30-45 s), 2D n = 512 and 3D n = 16 (configs[4] family; references written by
tests/golden/make_refs.py, which calls only oracle/ — the sparse LU takes minutes there), and
unstructured variants (random diagonals / mirrored Kuhn splits) at sizes the oracle solves here.
"""
import functools
import os

import numpy as np
import pytest
import torch

import bench
import cr_inputs as ci
import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1800)]

import paper_2101_03777_b200 as P  # noqa: E402

DEV = torch.device("cuda")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def tg(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def relL2(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


@functools.lru_cache(maxsize=2)
def configs1_family(n, flip=None):
    """inputs and coupled reference of the configs[1] family at size n (cached: several tests)"""
    cfg = ci.CONFIGS[1]
    coords, cells = ci.square_mesh(n, cfg.jitter, cfg.seed, flip_seed=flip)
    _, _, f = ci.manufactured_2d(cfg.mu, cfg.nu)
    fbar = ci.cell_average(f, coords, cells)
    Uc, Pc = coupled_reference(coords, cells, fbar, cfg.mu, cfg.nu)
    return coords, cells, fbar, Uc, Pc


def coupled_reference(coords, cells, fbar, mu, nu):
    m = O.build_mesh(coords, cells)
    M, rhs, nU = O.assemble_coupled(m, O.Params(mu=mu, nu=nu), O.Data(fbar=fbar))
    x = O.direct_refined(M, rhs)
    return x[:nU].reshape(-1, m.dim), np.insert(x[nU:], 0, 0.0)


def gpu_bench_solve(cfg_idx, coords, cells, fbar, cfg, **over):
    sol = dict(bench.SOLVERS[cfg_idx])
    sol.update(over)
    rtol = sol.pop("rtol")
    prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=tg(fbar))
    out = P.hybrid_method(tg(coords), tg(cells), prob, rtol=rtol, check_every=64, **sol)
    rep = out["report"]
    assert rep["converged"] and rep["rel_res_true"] <= rtol, rep
    return out["U"].cpu().numpy(), out["P"].cpu().numpy(), rep


@pytest.mark.parametrize("n,flip", [(256, None), (128, 7)])
def test_configs1_family_bench_solver_vs_coupled(n, flip):
    cfg = ci.CONFIGS[1]
    coords, cells, fbar, Uc, Pc = configs1_family(n, flip)
    U, Pp, rep = gpu_bench_solve(1, coords, cells, fbar, cfg)
    eu, ep = relL2(U, Uc), relL2(Pp, Pc)
    print(f"2D n={n} flip={flip}: {rep['iterations']} it, residual {rep['rel_res_true']:.2e}, U {eu:.2e}, P {ep:.2e}, "
          f"kappa {rep['kappa_lanczos_est']:.3g}")
    assert eu <= 1e-8 and ep <= 1e-8, (eu, ep)


@pytest.mark.parametrize("name", ["coupled_2d_n512", "coupled_3d_n16"])
def test_stored_reference_bench_solver(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (python tests/golden/make_refs.py {name})")
    ref = np.load(path)
    idx, n = int(ref["config"]), int(ref["n"])
    cfg = ci.CONFIGS[idx]
    inp = ci.make_inputs(cfg, n=n)
    U, Pp, rep = gpu_bench_solve(idx, inp["coords"], inp["cells"], inp["fbar"], cfg)
    eu, ep = relL2(U, ref["U"]), relL2(Pp, ref["P"])
    print(f"{name}: {rep['iterations']} it, residual {rep['rel_res_true']:.2e}, U {eu:.2e}, P {ep:.2e}")
    assert eu <= 1e-8 and ep <= 1e-8, (eu, ep)


def test_configs4_family_unstructured_bench_solver_vs_coupled():
    cfg = ci.CONFIGS[4]
    coords, cells = ci.cube_mesh(8, flip_seed=9)
    _, _, f = ci.manufactured_3d(cfg.mu, cfg.nu)
    fbar = ci.cell_average(f, coords, cells)
    Uc, Pc = coupled_reference(coords, cells, fbar, cfg.mu, cfg.nu)
    U, Pp, rep = gpu_bench_solve(4, coords, cells, fbar, cfg)
    eu, ep = relL2(U, Uc), relL2(Pp, Pc)
    assert eu <= 1e-8 and ep <= 1e-8, (eu, ep)


def test_refine_dd_reaches_below_the_fp64_floor():
    """Parity mode (cr_solver_opts.refine_dd): the double-double residual of the factored operator
    is driven to 2e-13 at 2D n = 256, where the fp64 recursion stalls at 4.6e-13,
    and U, P stay within the bar of the coupled solution."""
    cfg = ci.CONFIGS[1]
    coords, cells, fbar, Uc, Pc = configs1_family(256)
    U, Pp, rep = gpu_bench_solve(1, coords, cells, fbar, cfg, rtol=2e-13, refine_dd=1)
    print(f"refine_dd: residual {rep['rel_res_true']:.2e} after {rep['refine_rounds']} rounds "
          f"({rep['iterations']} + {rep['inner_iterations']} iterations); U {relL2(U, Uc):.2e} P {relL2(Pp, Pc):.2e}")
    assert rep["refine_rounds"] >= 1 and rep["rel_res_true"] <= 2e-13, rep
    assert relL2(U, Uc) <= 1e-9 and relL2(Pp, Pc) <= 1e-8


def test_report_kappa_and_bytes():
    """cr_solve_report: the Lanczos kappa estimate of Jacobi-PCG agrees with numpy's eigenvalues of
    D^-1/2 G D^-1/2 on the oracle's G (within the Lanczos under-estimate of lambda_min), and the
    algorithmic bytes are per-iteration bytes x iterations."""
    coords, cells = ci.square_mesh(10, 0.2, 1)
    _, _, f = ci.manufactured_2d(1.0, 1.0)
    fbar = ci.cell_average(f, coords, cells)
    m = O.build_mesh(coords, cells)
    G = O.hybridise(m, O.Params(1.0, 1.0), O.Data(fbar=fbar))["G"].toarray()
    dm = 1.0 / np.sqrt(np.diag(G))
    ev = np.linalg.eigvalsh(dm[:, None] * G * dm[None, :])
    prob = P.Problem(mu=1.0, nu=1.0, fbar=tg(fbar))
    hg = P.cr_hybridise(P.cr_build_mesh(tg(coords), tg(cells)), prob)
    W = torch.zeros(hg.n_rows, dtype=torch.float64, device=DEV)
    rep = P.cr_solve(hg, W, "pcg", rtol=1e-12)
    assert abs(rep["lambda_max_est"] / ev[-1] - 1) <= 1e-3
    assert 0.5 <= rep["kappa_lanczos_est"] / (ev[-1] / ev[0]) <= 1.0 + 1e-3
    per_it = 8 * hg.nnz + 4 * hg.nblocks + 2 * 8 * hg.n_rows + 7 * 8 * hg.n_rows
    assert abs(rep["bytes_moved"] - per_it * rep["iterations"]) <= 1e-9 * rep["bytes_moved"]


def test_newton_update_abi():
    rng = np.random.default_rng(3)
    U, dU, Pv, dP = (rng.normal(size=k) for k in (1000, 1000, 300, 300))
    Ut, Pt = tg(U), tg(Pv)
    a, b = P.newton_update(Ut, tg(dU), Pt, tg(dP))
    assert np.array_equal(Ut.cpu().numpy(), U + dU) and np.array_equal(Pt.cpu().numpy(), Pv + dP)
    assert abs(a - np.linalg.norm(dU)) <= 1e-14 * a and abs(b - np.linalg.norm(U + dU)) <= 1e-14 * b
