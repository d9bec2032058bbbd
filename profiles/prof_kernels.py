"""Standalone launches of the iteration's kernels on the headline workload (configs[4], or --n) for
CUDA-event timing and for `ncu --set full -k regex:...` captures.

    python profiles/prof_kernels.py [--config 4] [--n N] [--reps 20] [--solve-iters 64] [--ncu]

Builds the mesh, hybridises, runs a short two-level PCG solve (it sets up the patch preconditioner,
the coarse space and the matrix-free factors), then re-launches on the bench's stream:
  mf       y = G x   (k_mf_spmv)
  afw      z = M^-1 r (k_afw_apply_sh + k_afw_zsum)
  afw2     z = M2^-1 r (coarse restrict / ND solve / patch apply / combine)
  spmv     y = G x   (assembled k_spmv)
and prints ms per launch and algorithmic GB/s (the byte counts of bench.kernel_rooflines).
With --ncu each is launched --reps times after one warm-up (keep --reps small under ncu).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--solve-iters", type=int, default=64)
    ap.add_argument("--full-solve", action="store_true", help="solve to the bench's rtol and report iterations")
    ap.add_argument("--only", default="mf,afw,afw2,spmv")
    args = ap.parse_args()

    import torch
    import cr_inputs as ci
    import paper_2101_03777_b200 as P
    import bench

    dev = torch.device("cuda:0")
    cfg = ci.CONFIGS[args.config]
    sol, rtol = bench._solver(args.config)
    P.pool_reserve(int(min(60 * 2 ** 30, 0.6 * torch.cuda.mem_get_info(dev)[0])))
    inp = ci.make_inputs(cfg, n=args.n)
    coords, cells = torch.from_numpy(inp["coords"]).to(dev), torch.from_numpy(inp["cells"]).to(dev)
    fbar = torch.from_numpy(inp["fbar"]).to(dev)
    stream = torch.cuda.current_stream()
    prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar)
    mesh = P.cr_build_mesh(coords, cells)
    hyb = P.cr_hybridise(mesh, prob)
    W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=dev)
    if args.full_solve:
        rep = P.cr_solve(hyb, W, rtol=rtol, check_every=64, max_iter=20000, **sol)
    else:
        rep = P.cr_solve(hyb, W, rtol=1e-30, check_every=args.solve_iters, max_iter=args.solve_iters,
                         raise_on_fail=False, **sol)
    torch.cuda.synchronize()
    N = hyb.n_rows
    N8 = 8 * N
    pinfo, minfo, cinfo = hyb.precond_info(), hyb.mf_info(), hyb.coarse_info()
    slots = 2 if mesh.dim == 2 else 3
    x = torch.randn(N, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    prec_bytes = pinfo["bytes"] + N8 + 2 * slots * N8 + N8
    cases = {
        "mf": (lambda: hyb.spmv_mf(x, y), minfo["bytes"] + 2 * N8),
        "afw": (lambda: hyb.apply_precond("pcg_afw", x, y), prec_bytes),
        "afw2": (lambda: hyb.apply_precond(sol["method"], x, y),
                 prec_bytes + N8 + 8 * N + cinfo["solve_bytes"] + 8 * N),
        "spmv": (lambda: hyb.spmv(x, y), 8 * hyb.nnz + 4 * hyb.nblocks + 2 * N8),
    }
    out = {"n_rows": N, "iterations": rep["iterations"], "solve_s": rep["seconds"],
           "setup_s": rep["setup_seconds"], "rel_res_true": rep["rel_res_true"],
           "ms_per_iter": (rep["seconds"] - rep["setup_seconds"]) / max(rep["iterations"], 1) * 1e3,
           "iter_gbs": rep["bytes_moved"] / max(rep["seconds"] - rep["setup_seconds"], 1e-9) / 1e9,
           "precond": pinfo, "mf": minfo, "coarse": cinfo}
    out["in_solve_ms"] = P.cr_solve_profile(hyb, sol["method"], nrep=10, matrix_free=sol["matrix_free"],
                                            coarse=sol["coarse"])
    for name in args.only.split(","):
        fn, nbytes = cases[name]
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        med = ts[len(ts) // 2]
        out[name] = {"ms_median": med, "ms_min": ts[0], "bytes": nbytes, "gbs": nbytes / med / 1e6,
                     "frac": nbytes / med / 1e6 / 6550.4}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
