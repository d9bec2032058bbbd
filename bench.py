#!/usr/bin/env python
"""Benchmark of the hybrid method's hot path on B200 (BASELINE.json metric:
"hybridised-system PCG time-to-solution; SpMV GB/s as % of B200 HBM peak").

Headline workload (one "step"): BASELINE.json configs[4] — the largest single-GPU config:
3D transient Stokes, unit cube, 128^3 cubes x 6 Kuhn tetrahedra (12,582,912 cells, 75,202,560
face unknowns), mu = nu = 1, manufactured fp64 force — through the whole hot path:
cr_build_mesh -> cr_hybridise -> cr_solve (PCG to a TRUE relative residual of 1e-10 with the
two-level preconditioner (edge-patch additive Schwarz + coarse "stress x area" space, nested-
dissection coarse solve) on the matrix-free factored G) -> cr_recover,
inputs resident in HBM.  value = seconds per step (time to solution, lower is better).
`--config 1` times configs[1] (2D n = 1024) instead; configs[1..3], time stepping, Newton and
the Table 4 analogue are reported inside the same line (`other_configs`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4|1]

For N > 1 (torchrun, one rank per GPU) the SAME problem is partitioned: each rank owns a slab
of face rows of G, exchanges SpMV ghosts with its neighbours (NCCL send/recv) and allreduces
the Krylov dot products (strong scaling); timed on the device, max over ranks.
--impl reference times the CPU oracle (oracle/, numpy/scipy + binary128 C) on the host cores on
a bounded sample of the same workload family and extrapolates per unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "hybridised-system PCG time-to-solution; SpMV GB/s as % of B200 HBM peak"
HEADLINE = 4         # BASELINE.json configs[4]: the largest config that fits one GPU
# The solver bench.py times, per config (tests/test_gpu_bench_parity.py runs exactly these):
# two-level PCG (patch additive Schwarz + coarse "stress x area" space)
# on the matrix-free factored G (§5.2); coarse = intervals per direction of the coarse grid.
# rtol: the TRUE relative residual; 2D needs 1e-11 for relL2(P) <= 1e-8 against the coupled
# solution (2.5e-8 at 1e-10, 3.9e-9 at 1e-11 on n = 256; DESIGN.md §2 reading 13), 3D meets it
# at the north star's 1e-10.
SOLVERS = {1: dict(method="pcg_afw2", matrix_free=1, coarse=64, rtol=1e-11),
           4: dict(method="pcg_afw2", matrix_free=1, coarse=16, rtol=1e-10)}
COARSE_MULTI = 12    # configs[4] coarse intervals at 4+ GPUs (replicated coarse solve)
MAX_ITER = 20000     # a cap (the solves take ~500): a regression fails loudly instead of running on
# Jacobi-PCG iterations to a true 1e-10 residual, measured on the B200 (the oracle's own solver;
# used to extrapolate the CPU oracle's time): configs[1] by the r01 driver run (BENCH_r01.json
# pcg_jacobi), configs[4] by `python bench.py --jacobi` (profiles/r02_jacobi_configs4.log).
JACOBI_ITERS = {1: 161758, 4: 48569}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled every 200 ms DURING the timed region, in-process
    through NVML (the nvidia-smi subprocess stalled the host thread's CUDA calls for up to
    0.7 s at some of its queries); nvidia-smi -lms is the fallback when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.lines = []
        self.proc = None
        self.nv = None
        self.stop = threading.Event()

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]

            def loop():
                while not self.stop.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.lines.append(", ".join([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]))
                    self.stop.wait(0.2)

            self.nv = nv
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) stalls the driver for a few hundred ms: let it
            # finish before the timed region opens, so only its cheap periodic queries overlap
            t0 = time.time()
            while len(self.lines) < 2 and time.time() - t0 < 10:
                time.sleep(0.02)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle arm
# bounded samples of each config family the oracle times (mesh size n_sample, PCG iterations)
ORACLE_SAMPLE = {1: (256, 200), 4: (12, 200)}


def oracle_sample(cfg_idx: int):
    """Time the oracle, as it stands, on a bounded sample of the configs[cfg_idx] family (same
    generator, jitter, mu, nu; smaller n) and return per-unit costs."""
    import numpy as np
    import cr_inputs as ci
    import oracle as O
    n_sample, iters = ORACLE_SAMPLE[cfg_idx]
    cfg = ci.CONFIGS[cfg_idx]
    inp = ci.make_inputs(cfg, n=n_sample)
    t0 = time.perf_counter()
    m = O.build_mesh(inp["coords"], inp["cells"])
    t1 = time.perf_counter()
    prm, data = O.Params(mu=cfg.mu, nu=cfg.nu), O.Data(fbar=inp["fbar"])
    h = O.hybridise(m, prm, data)
    t2 = time.perf_counter()
    _, rep = O.pcg(h["G"], h["S"], rtol=1e-30, max_iter=iters)
    t3 = time.perf_counter()
    O.recover(m, prm, data, h["E"], np.zeros(len(h["S"])))
    t4 = time.perf_counter()
    return dict(nc=m.nc, nnz=h["G"].nnz, mesh_s=t1 - t0, hyb_s=t2 - t1, iter_s=(t3 - t2) / rep["iterations"],
                rec_s=t4 - t3, iters=rep["iterations"], n=n_sample, dim=m.dim)


def oracle_extrapolate(s: dict, nc_full: int, nnz_full: int, iters_full: int) -> float:
    f = nc_full / s["nc"]
    return (s["mesh_s"] + s["hyb_s"] + s["rec_s"]) * f + s["iter_s"] * (nnz_full / s["nnz"]) * iters_full


def full_sizes(cfg_idx):
    """Closed-form sizes of the structured meshes: cells, nnz(G), blocks, unknowns."""
    import cr_inputs as ci
    n = ci.CONFIGS[cfg_idx].n
    if ci.CONFIGS[cfg_idx].dim == 2:
        nc, nf_int = 2 * n * n, 3 * n * n - 2 * n
        nb = nf_int + 12 * (n - 1) ** 2 + 8 * (n - 1)
        return nc, 4 * nb, nb, 2 * nf_int
    nc, nf_int = 6 * n ** 3, 12 * n ** 3 - 6 * n * n
    nb = nf_int + 72 * n * (n - 1) ** 2 + 72 * n * (n - 1) + 12 * n
    return nc, 9 * nb, nb, 3 * nf_int


def jacobi_iters(cfg_idx):
    """Jacobi-PCG iteration count of the config (measured on the B200; see JACOBI_ITERS).  For
    configs[4] without a measurement: the SURVEY A.5 fit (n^1.35 from n <= 32), labelled."""
    it = JACOBI_ITERS.get(cfg_idx)
    if it:
        return it, "measured on the B200"
    return 70000, "SURVEY A.5 fit (not measured)"


def workload_config(cfg_idx, world):
    """The `config` object of both arms (identical by construction)."""
    import cr_inputs as ci
    cfg = ci.CONFIGS[cfg_idx]
    nc, nnz, nb, N = full_sizes(cfg_idx)
    sol = SOLVERS[cfg_idx]
    if cfg.dim == 2:
        what = f"configs[1] 2D transient Stokes n={cfg.n} jittered 0.2h (triangles)"
    else:
        what = f"configs[4] 3D transient Stokes n={cfg.n} Kuhn cubes (6 tetrahedra each)"
    return {"workload": what + f", two-level-preconditioned PCG on the matrix-free G to true {sol['rtol']:g}",
            "cells": nc, "unknowns": N, "nnz_G": nnz, "blocks_G": nb,
            "parallelism": (f"face rows partitioned over {world} GPUs (NCCL halo send/recv + allreduce)"
                            if world > 1 else "1 GPU"),
            "l2": "working set > L2 (G = %.2f GB assembled; per-iteration streams > 1 GB) and a 256 MB L2 flush "
                  "before each step" % (8 * nnz / 1e9),
            "memory": "libcr pool reserved up front (cr_pool_reserve, --pool-reserve-gb; DESIGN.md §1)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg_idx = args.config
    nc, nnz, nb, N = full_sizes(cfg_idx)
    iters_full, src = jacobi_iters(cfg_idx)
    vals, samples = [], []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(cfg_idx)
        if i >= args.warmup:
            vals.append(oracle_extrapolate(s, nc, nnz, iters_full))
            samples.append(s)
    v = statistics.mean(vals)
    s = samples[-1]
    sample_desc = (f"oracle on the configs[{cfg_idx}] family at n={s['n']} ({s['nc']} cells): mesh+hybridise+recover "
                   f"timed in full, Jacobi PCG (the oracle's solver) timed over {s['iters']} iterations; extrapolated "
                   f"per cell and per nnz x {iters_full} iterations ({src}) to the full workload")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg_idx, args.gpus),
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "oracle", "sample": sample_desc},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
# solvers of the configs without a transient hybrid system
OTHER_SOLVERS = {2: dict(method="dc", coarse=64, mu_inner=1.0),
                 3: dict(method="dc", coarse=64, mu_inner=0.5, inner_rtol=1e-7)}


def _ev(torch, stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def _solver(cfg_idx):
    sol = dict(SOLVERS[cfg_idx])
    rtol = sol.pop("rtol")
    return sol, rtol


def stage_times(P, cfg_idx, coords, cells, fbar, stream):
    """One step with CUDA events between the four C-ABI calls."""
    import torch
    import cr_inputs as ci
    cfg = ci.CONFIGS[cfg_idx]
    sol, rtol = _solver(cfg_idx)
    torch.cuda.synchronize()
    e = [_ev(torch, stream)]
    mesh = P.cr_build_mesh(coords, cells)
    e.append(_ev(torch, stream))
    hyb = P.cr_hybridise(mesh, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar))
    e.append(_ev(torch, stream))
    W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=coords.device)
    rep = P.cr_solve(hyb, W, rtol=rtol, check_every=64, max_iter=MAX_ITER, **sol)
    e.append(_ev(torch, stream))
    P.cr_recover(hyb, W)
    e.append(_ev(torch, stream))
    torch.cuda.synchronize()
    t = [e[i].elapsed_time(e[i + 1]) * 1e-3 for i in range(4)]
    return {"mesh_s": t[0], "hybridise_s": t[1], "solve_s": t[2], "recover_s": t[3],
            "assembly_cells_per_s": mesh.nc / t[1], "mesh_cells_per_s": mesh.nc / t[0],
            "recover_cells_per_s": mesh.nc / t[3], "iterations": rep["iterations"]}


def time_stepping(P, cfg, coords, cells, fbar, stream, nsteps=5):
    """configs[1] as nsteps backward-Euler steps (mu = 1/dt) with G and its preconditioners built
    once: per-step iterations (warm start) and solve times."""
    import torch
    sol, rtol = _solver(1)
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.time_march(coords, cells, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar), nsteps, rtol=rtol, check_every=64,
                       max_iter=MAX_ITER, **sol)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    reps = out["reports"]
    return {"steps": nsteps, "total_s": a.elapsed_time(b) * 1e-3, "iterations": [r["iterations"] for r in reps],
            "solve_s": [r["seconds"] for r in reps], "rel_res_true": [r["rel_res_true"] for r in reps],
            "note": "step 1 includes the preconditioner / coarse-space setup; later steps reuse them"}


def newton_cavity(P, ci, dev, stream, n=256, nu=0.01, tol=5e-7, damped=False):
    """Steady lid-driven cavity (Re = 1/nu) by Newton's method (tolerance of P:L783-799
    Table 7), each step through the hybrid path (NS step + CR_DC_FGMRES); damped: Armijo line search
    on the nonlinear residual (Re = 1000 from rest, the paper's case)."""
    import torch
    coords, cells = ci.square_mesh(n, 0.0, 4)
    wall = ci.lid_dirichlet_2d(coords, cells)
    tg = lambda a: torch.from_numpy(a).to(dev)
    f = torch.zeros((cells.shape[0], 2), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.newton_ns(tg(coords), tg(cells), nu, f, tg(wall), tol=tol, mis_seed=44, coarse=32, mu_inner=0.5,
                      inner_rtol=1e-7, damped=damped, max_newton=40, restart=100, max_iter=2000)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    return {"workload": f"2D lid-driven cavity n={n} Re={1 / nu:g}, {'damped ' if damped else ''}Newton from rest "
                        f"to ||dU|| <= {tol:g} ||U||",
            "newton_steps": len(out["history"]), "converged": bool(out["history"][-1] <= tol),
            "history": out["history"], "step_lengths": out["step_lengths"], "total_s": a.elapsed_time(b) * 1e-3,
            "outer_iterations": [r["iterations"] for r in out["reports"]],
            "inner_iterations": [r["inner_iterations"] for r in out["reports"]]}


def direct_table4(P, ci, dev, stream, ns=(2, 4, 8)):
    """The paper's direct-solver comparison (Table 4: 3D Kuhn meshes, transient Stokes
    with dt = 5e-4, one linear system): the hybrid G by sparse Cholesky + recovery against the
    coupled saddle system by sparse QR (cuSOLVER, METIS ordering), seconds per linear system."""
    import numpy as np
    import torch
    rows = []
    for n in ns:
        coords, cells = ci.cube_mesh(n)
        _, _, f = ci.manufactured_3d(2000.0, 1.0)
        fbar = ci.cell_average(f, coords, cells)
        tg = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        prob = P.Problem(mu=2000.0, nu=1.0, fbar=tg(fbar))
        mesh = P.cr_build_mesh(tg(coords), tg(cells))
        torch.cuda.synchronize()
        a = _ev(torch, stream)
        hyb = P.cr_hybridise(mesh, prob)
        rp, cidx, v, S = hyb.export_csr()
        W = P.sparse_direct_solve(rp, cidx, v, S, "chol")
        U, Pp, _ = P.cr_recover(hyb, W)
        b = _ev(torch, stream)
        cpl = P.cr_assemble_coupled(mesh, prob)
        rp2, ci2, v2, rhs = cpl.export_csr()
        x = P.sparse_direct_solve(rp2, ci2, v2, rhs, "qr")
        c = _ev(torch, stream)
        torch.cuda.synchronize()
        nU = U.numel()
        du = float(torch.linalg.norm(x[:nU] - U.reshape(-1)) / torch.linalg.norm(U))
        rows.append({"n": n, "Ncv": int(mesh.nc), "hybrid_unknowns": int(hyb.n_rows), "coupled_unknowns": int(rhs.numel()),
                     "hybrid_s": a.elapsed_time(b) * 1e-3, "coupled_s": b.elapsed_time(c) * 1e-3, "relL2_U": du})
    return {"workload": "Table 4 analogue: 3D Kuhn n^3 x 6 tets, transient Stokes dt = 5e-4, one system",
            "solvers": "hybrid: cuSOLVER sparse Cholesky of G + recovery; coupled: cuSOLVER sparse QR (METIS)",
            "rows": rows}


def other_config(P, ci, idx, dev, stream):
    """Time-to-solution (mesh + hybridise + solve + recover, inputs in HBM) of configs[idx]."""
    import torch
    cfg = ci.CONFIGS[idx]
    inp = ci.make_inputs(cfg)
    tg = lambda a: torch.from_numpy(a).to(dev)
    kw = {}
    if cfg.shift == "mis":
        kw.update(shift=P.CR_SHIFT_MIS, mis_seed=cfg.mis_seed)
    if cfg.physics == "ns_step":
        kw.update(physics=P.CR_NS_NEWTON_STEP, u_iter=tg(inp["u_iter"]))
    prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=tg(inp["fbar"]), **kw)
    coords, cells = tg(inp["coords"]), tg(inp["cells"])
    if idx in SOLVERS:
        sol, rtol = _solver(idx)
    else:
        sol, rtol = OTHER_SOLVERS[idx], cfg.rtol
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.hybrid_method(coords, cells, prob, rtol=rtol, check_every=64, **sol)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    rep = out["report"]
    kind = {"stokes": "transient Stokes" if cfg.mu > 0 else "steady Stokes", "ns_step": "Navier-Stokes Newton step"}
    r = {"workload": f"configs[{idx}] {cfg.dim}D {kind[cfg.physics]} n={cfg.n} (nu={cfg.nu})", "solver": sol,
         "rtol": rtol, "time_to_solution_s": a.elapsed_time(b) * 1e-3, "solve_s": rep["seconds"],
         "iterations": rep["iterations"], "rel_res_true": rep["rel_res_true"],
         "unknowns": out["hybrid"].n_rows, "cells": out["mesh"].nc}
    if sol["method"] == "dc":
        r["inner_iterations"] = rep["inner_iterations"]
    del out
    return r


def kernel_rooflines(P, torch, hyb, mesh, rep, stream, dev, peak, peak_src, cfg_idx):
    """Per-kernel algorithmic GB/s of the solve's iteration.  Each kernel group is launched by
    cr_solve_profile on the handle's own solver buffers exactly as the solve launches it (same row
    order, grids) and timed alone with CUDA events on the bench's stream; share = its time / the
    solve's ms per iteration (the coarse path overlaps the patch solves on a side stream in the solve,
    so the shares can add up to slightly more than 1).  The dominant kernel is the one with the
    largest share.  The assembled SpMV (not used by the solve) is timed through cr_spmv for
    reference."""
    N, nnz, nb = hyb.n_rows, hyb.nnz, hyb.nblocks
    N8 = 8 * N
    pinfo, minfo, cinfo = hyb.precond_info(), hyb.mf_info(), hyb.coarse_info()
    slots = 2 if mesh.dim == 2 else 3
    D = mesh.dim
    sol = SOLVERS[cfg_idx]
    prof = P.cr_solve_profile(hyb, sol["method"], nrep=20, matrix_free=sol["matrix_free"], coarse=sol["coarse"],
                              stream=stream)
    s_ = {k: v * 1e-3 for k, v in prof.items()}

    x = torch.randn(N, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        hyb.spmv(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        hyb.spmv(x, y)
    e1.record(stream)
    torch.cuda.synchronize()
    spmv_s = e0.elapsed_time(e1) / 20 * 1e-3

    # algorithmic bytes per launch (DESIGN.md §5 table)
    b_mf = minfo["bytes"] + N8 + N8                                        # cell factors + p once + q once
    b_upd = 3 * N8                                                         # r, q read; r written
    b_coarse = N8 + 8 * N + 4 * (N // D) + cinfo["solve_bytes"]            # r, fp32 basis, perm, E^-1 / ND fronts
    b_patch = pinfo["bytes"] + N8 + slots * N8                             # operator + r + slot contributions
    b_pdir = slots * N8 + 2 * N8 + 2 * N8 + 8 * N                          # slots, p and x read + written, basis
    b_spmv = 8 * nnz + 4 * nb + N8 + N8                                    # values + block cols + x + y

    def traffic(tag):
        f = os.path.join(ROOT, "profiles", f"r02_dram_bytes_c{cfg_idx}_{tag}.json")
        try:
            return json.load(open(f)).get("dram_bytes_per_launch")
        except Exception:
            return None

    def roof(kernel, bytes_, sec, tr=None):
        return {"kernel": kernel, "bound": "hbm", "achieved": bytes_ / sec / 1e9, "peak": peak, "unit": "GB/s",
                "frac": bytes_ / sec / 1e9 / peak, "traffic": tr, "peak_source": peak_src,
                "algorithmic_bytes": bytes_, "launch_s": sec, "timing": "in-solve launch (cr_solve_profile)"}

    kernels = {
        "mf": roof(f"k_mf_spmv<{D},1> + memset(q) (matrix-free factored G p with p.q: the in-solve G apply)", b_mf,
                   s_["mf"], traffic("mf")),
        "update_r": roof("k_pcg_update_r<false> (r -= alpha q, r.r)", b_upd, s_["update_r"]),
        "coarse": roof("k_coarse_restrict3c / k_coarse_restrict + k_coarse_gather + k_nd_solve (nested dissection) / dense E^-1 "
                       "(y = E^-1 Z^t r)", b_coarse, s_["coarse"]) if s_["coarse"] > 0 else None,
        "precond": roof("k_afw_apply_sc (patch additive Schwarz solves, one warp per (slice, component), slot contributions)", b_patch, s_["patch"],
                        traffic("afw_apply")),
        "pdir": roof("k_pcg_pdir_afw2 (p = z + Z y + beta p, x += alpha p)", b_pdir, s_["pdir"]),
    }
    kernels["precond_two_level"] = roof("coarse path + patch solves (z = M2^-1 r)", b_coarse + b_patch,
                                        s_["coarse"] + s_["patch"])
    kernels["spmv_assembled"] = roof("k_spmv (assembled sliced block-ELL G x; not used by the bench's solve; "
                                     "timed through cr_spmv)", b_spmv, spmv_s, traffic("spmv"))
    kernels["spmv_assembled"]["timing"] = "standalone cr_spmv launches"
    kernels = {k: v for k, v in kernels.items() if v is not None}
    it_s = (rep["seconds"] - rep["setup_seconds"]) / max(rep["iterations"], 1)
    shares = {k: s_[k] / it_s for k in ("mf", "update_r", "coarse", "patch", "pdir")}
    groups = {"mf": "mf", "update_r": "update_r", "coarse": "coarse", "patch": "precond", "pdir": "pdir"}
    dominant = groups[max(shares, key=shares.get)]
    return kernels, dominant, shares


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=HEADLINE, choices=sorted(SOLVERS))
    ap.add_argument("--n", type=int, default=None, help="override mesh size (debug only; not a bench value)")
    ap.add_argument("--jacobi", action="store_true", help="also solve the headline config with Jacobi PCG (minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--profile-run", action="store_true",
                    help="profiler runs only (ncu launch list): keep --warmup as given (< 3 allowed) and skip the "
                         "Jacobi-PCG sample; the printed numbers are not bench values")
    ap.add_argument("--force-comm", action="store_true",
                    help="debug: run the partitioned (--gpus N > 1) code path on one GPU through a one-rank NCCL "
                         "communicator (not a bench value)")
    ap.add_argument("--pool-reserve-gb", type=float, default=None,
                    help="map this much into libcr's memory pool before the first step (cr_pool_reserve); default "
                         "120 for configs[4], 24 for configs[1]: without it the pool maps new memory in the middle of "
                         "some steps (3D: 3.5-6.1 s per step instead of 3.47 +- 0.01 s)")
    args = ap.parse_args()
    if not args.profile_run:
        args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import cr_inputs as ci
    import paper_2101_03777_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        # libcr's own NCCL communicator (halo send/recv + allreduce inside its CUDA graphs)
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = P.Comm.nccl(uid[0], rank, world)
    elif args.force_comm:
        comm = P.Comm.nccl(P.nccl_unique_id(), 0, 1)
    multi = comm is not None   # the partitioned path: no single-GPU extras

    def barrier():
        if world > 1:
            dist.barrier()

    cfg_idx = args.config
    cfg = ci.CONFIGS[cfg_idx]
    sol, rtol = _solver(cfg_idx)
    if world >= 4 and cfg.dim == 3:
        # the coarse solve is replicated on every rank: at 4+ ranks the smaller H = 12 coarse space
        # (0.70 GB of fronts per solve instead of 2.45 GB, 560 instead of 441 iterations on one GPU)
        # gives the shorter time to solution (DESIGN.md §8 model)
        sol["coarse"] = COARSE_MULTI
    if args.pool_reserve_gb is None:
        args.pool_reserve_gb = 120.0 if cfg.dim == 3 else 24.0
    if args.pool_reserve_gb > 0:
        free = torch.cuda.mem_get_info(dev)[0]
        P.pool_reserve(int(min(args.pool_reserve_gb * 2 ** 30, 0.8 * free)))
    inp = ci.make_inputs(cfg, n=args.n)
    coords_h = torch.from_numpy(inp["coords"]).pin_memory()
    cells_h = torch.from_numpy(inp["cells"]).pin_memory()
    fbar_h = torch.from_numpy(inp["fbar"]).pin_memory()
    coords, cells, fbar = coords_h.to(dev), cells_h.to(dev), fbar_h.to(dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2

    def step():
        prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar)
        mesh = P.cr_build_mesh(coords, cells)
        hyb = P.cr_hybridise(mesh, prob, comm=comm)
        W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=dev)
        rep = P.cr_solve(hyb, W, rtol=rtol, check_every=64, max_iter=MAX_ITER, **sol)
        U, Pp, diag = P.cr_recover(hyb, W)
        return mesh, hyb, rep, U, Pp, diag

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    barrier()
    torch.cuda.synchronize()
    l0 = P.kernel_launches()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            new = step()
            evs[k][1].record(stream)
            reps.append(new[2])
            out = new   # the previous step's handles are released after its end event
            del new
        torch.cuda.synchronize()
    launches = P.kernel_launches() - l0
    barrier()
    ms = [a.elapsed_time(b) for a, b in evs]
    ms_per_step = sum(ms) / len(ms)
    t = torch.tensor([ms_per_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item())
    mesh, hyb, rep = out[0], out[1], reps[-1]
    nnz, nb, nrows = hyb.nnz, hyb.nblocks, hyb.n_rows

    peak, peak_src = measured_peaks()
    cinfo, pinfo, minfo = hyb.coarse_info(), hyb.precond_info(), hyb.mf_info()
    iter_s = rep["seconds"] - rep["setup_seconds"]
    iter_gbs = rep["bytes_moved"] / iter_s / 1e9 if iter_s > 0 else None
    if not multi:
        kernels, dominant, shares = kernel_rooflines(P, torch, hyb, mesh, rep, stream, dev, peak, peak_src, cfg_idx)
    else:
        # partitioned runs: cr_solve_profile times single-GPU handles only; report this rank's whole
        # iteration (its algorithmic bytes / its iteration time) against the same peak
        dominant, shares = "iteration", None
        kernels = {"iteration": {
            "kernel": "two-level PCG iteration, all kernels of rank 0's partition (per-kernel profile: single GPU only)",
            "bound": "hbm", "achieved": iter_gbs, "peak": peak, "unit": "GB/s",
            "frac": iter_gbs / peak if iter_gbs else None, "traffic": None, "peak_source": peak_src,
            "algorithmic_bytes": rep["bytes_moved"] / max(rep["iterations"], 1),
            "launch_s": iter_s / max(rep["iterations"], 1), "timing": "solve report (CUDA events around the iterations)"}}

    # the north star's baseline solver (Jacobi PCG) on the same G: to solution with --jacobi, else
    # a sample of 2,000 iterations for its time per iteration
    jac = None
    if not multi and not args.profile_run:
        Wj = torch.zeros(nrows, dtype=torch.float64, device=dev)
        if args.jacobi:
            rj = P.cr_solve(hyb, Wj, "pcg", rtol=rtol, check_every=256, raise_on_fail=False)
            jac = {"iterations": rj["iterations"], "rel_res_true": rj["rel_res_true"], "solve_s": rj["seconds"],
                   "converged": bool(rj["converged"]), "kappa_lanczos_est": rj["kappa_lanczos_est"]}
        else:
            rj = P.cr_solve(hyb, Wj, "pcg", rtol=rtol, check_every=256, max_iter=2000, raise_on_fail=False)
            jac = {"sampled_iterations": rj["iterations"], "ms_per_iter": rj["seconds"] / max(rj["iterations"], 1) * 1e3,
                   "iter_gbs": rj["bytes_moved"] / (rj["seconds"] - rj["setup_seconds"]) / 1e9 if rj["seconds"] > 0 else None,
                   "kappa_lanczos_est_partial": rj["kappa_lanczos_est"],
                   "iterations_to_1e-10": jacobi_iters(cfg_idx)[0], "iterations_source": jacobi_iters(cfg_idx)[1]}
        del Wj

    # ---- e2e through the C ABI from HOST buffers (cr_hybrid_method_host: pinned host -> device,
    # the whole method, device -> host of U and P), caller-owned pinned result buffers
    nc_full, ndim = mesh.nc, mesh.dim
    nf_int = mesh.nf_int
    del out, hyb, mesh
    e2e = None
    if not args.no_e2e and not multi:
        Uh = torch.empty(nf_int * ndim, dtype=torch.float64, pin_memory=True)
        Ph = torch.empty(nc_full, dtype=torch.float64, pin_memory=True)

        def e2e_step():
            return P.hybrid_method_host(coords_h, cells_h, fbar_h, cfg.mu, cfg.nu, rtol=rtol, out=(Uh, Ph),
                                        stream=stream, max_iter=MAX_ITER, **sol)

        e2e_step()   # warm-up
        e2e_ms = []
        for _ in range(min(args.steps, 5)):   # each with its own host -> device -> host copies
            torch.cuda.synchronize()
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        h2d = coords_h.numel() * 8 + cells_h.numel() * 4 + fbar_h.numel() * 8
        d2h = res["U_host"].numel() * 8 + res["P_host"].numel() * 8
        e2e = {"value": sum(e2e_ms) / len(e2e_ms) * 1e-3, "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": len(e2e_ms), "api": "cr_hybrid_method_host (C ABI)"}

    # ---- stage times of one step and time-to-solution of the other configs (single GPU only)
    stages, others, tstep, newton, table4 = None, None, None, None, None
    if not multi and not args.no_other_configs:
        stages = stage_times(P, cfg_idx, coords, cells, fbar, stream)
        del coords, cells, fbar
        torch.cuda.empty_cache()
        others = {}
        for idx in (1, 2, 3, 4):
            if idx == cfg_idx:
                continue
            others[f"configs[{idx}]"] = other_config(P, ci, idx, dev, stream)
            torch.cuda.empty_cache()
        c1 = ci.CONFIGS[1]
        i1 = ci.make_inputs(c1)
        tg = lambda a: torch.from_numpy(a).to(dev)
        tstep = time_stepping(P, c1, tg(i1["coords"]), tg(i1["cells"]), tg(i1["fbar"]), stream)
        newton = {"re100": newton_cavity(P, ci, dev, stream),
                  # the paper's Table 7 case (Re = 1000) from rest, Armijo-damped
                  "re1000": newton_cavity(P, ci, dev, stream, n=64, nu=1e-3, damped=True)}
        table4 = direct_table4(P, ci, dev, stream)

    cpu = None
    if rank == 0 and not multi and not args.no_cpu_baseline:
        s = oracle_sample(cfg_idx)
        it_full, src = jacobi_iters(cfg_idx)
        v = oracle_extrapolate(s, nc_full, nnz, it_full)
        cpu = {"value": v, "unit": "s", "cores": 1, "kind": "oracle",
               "sample": (f"oracle on the configs[{cfg_idx}] family at n={s['n']} ({s['nc']} cells): mesh+hybridise+"
                          f"recover timed in full ({s['mesh_s'] + s['hyb_s'] + s['rec_s']:.1f} s), Jacobi PCG (the "
                          f"oracle's solver) over {s['iters']} iterations ({s['iter_s'] * 1e3:.2f} ms/it); "
                          f"extrapolated per cell and per nnz x {it_full} Jacobi-PCG iterations ({src}) to the "
                          f"full workload")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_steps_rank0": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg_idx, world),
            "pcg": {**sol, "rtol": rtol, "coarse": cinfo, "precond": pinfo, "mf": minfo,
                    "iterations": rep["iterations"], "rel_res_true": rep["rel_res_true"], "solve_s": rep["seconds"],
                    "setup_s": rep["setup_seconds"], "ms_per_iter": iter_s / max(rep["iterations"], 1) * 1e3,
                    "iter_gbs": iter_gbs, "bytes_moved": rep["bytes_moved"],
                    "kappa_lanczos_est": rep["kappa_lanczos_est"], "kernel_shares_of_iteration": shares},
            "pcg_jacobi": jac,
            "roofline": kernels[dominant],
            "roofline_kernels": kernels,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "gpu_launches_note": "libcr kernels launched in the timed region (cr_kernel_launches: direct launches + "
                                 "kernel nodes of every replayed solver graph; CUB / cuBLAS / cuSOLVER excluded)",
            "e2e": e2e,
            "stages": stages,
            "other_configs": others,
            "time_stepping_configs1": tstep,
            "newton_cavity": newton,
            "direct_table4": table4,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
