#!/usr/bin/env python
"""Benchmark of the hybrid method's hot path on B200 (BASELINE.json metric:
"hybridised-system PCG time-to-solution; SpMV GB/s as % of B200 HBM peak").

Workload (one "step"): BASELINE.json configs[1] — 2D transient Stokes, unit square,
1024 x 1024 squares split into 2,097,152 triangles, interior vertices jittered by up to
0.2h (seed 2), mu = nu = 1, manufactured fp64 force — run through the whole hot path:
cr_build_mesh -> cr_hybridise -> cr_solve (PCG to a TRUE relative residual of 1e-10, with
the two-level preconditioner (patch additive Schwarz + a coarse "stress x area vector" space)
and the matrix-free factored G)
-> cr_recover, inputs resident in HBM.  value = seconds per step (time to solution, lower is better).
The same step with Jacobi PCG (the north star's baseline solver) is timed once and reported
under "pcg_jacobi".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

For N > 1 (torchrun, one rank per GPU) the SAME problem is partitioned: each rank owns a slab
of face rows of G, exchanges SpMV ghosts with its neighbours (NCCL send/recv) and allreduces
the Krylov dot products (strong scaling); timed on the device, max over
ranks.
--impl reference times the CPU oracle (oracle/, numpy/scipy + binary128 C) on the host
cores on a bounded sample of the same workload and extrapolates per unit.
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
CONFIG_IDX = 1
METHOD = "pcg_afw2"  # patch additive Schwarz + coarse "stress x area" correction
MATRIX_FREE = 1      # G applied from per-cell factors
COARSE = 64          # coarse grid intervals per direction (flat nested-dissection coarse solve)
MAX_ITER = 20000     # a cap (the solve takes ~800): a regression fails loudly instead of running on
# Jacobi-PCG iterations of configs[1] to a true 1e-10 residual, measured on B200 by this
# bench (used only by --impl reference to extrapolate the oracle's per-iteration time).
ITERS_CONFIG1_MEASURED = 162221   # Jacobi PCG, configs[1], B200 bench r01 (profiles/r01_bench_*.log)


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
def oracle_sample(n_sample: int = 256, iters: int = 200):
    """Time the oracle, as it stands, on a bounded sample of the configs[1] family (same
    generator, jitter, mu, nu; n = n_sample) and return per-unit costs."""
    import numpy as np
    import cr_inputs as ci
    import oracle as O
    cfg = ci.CONFIGS[CONFIG_IDX]
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
                rec_s=t4 - t3, iters=rep["iterations"], n=n_sample)


def oracle_extrapolate(s: dict, nc_full: int, nnz_full: int, iters_full: int) -> float:
    f = nc_full / s["nc"]
    return (s["mesh_s"] + s["hyb_s"] + s["rec_s"]) * f + s["iter_s"] * (nnz_full / s["nnz"]) * iters_full


def workload_config(n, world):
    """The `config` object of both arms (identical by construction; closed-form sizes of the
    structured n x n triangulation)."""
    nc, nnz, nb, N = full_sizes(n)
    return {"workload": "configs[1] 2D transient Stokes n=%d jittered 0.2h, two-level-preconditioned PCG to "
                        "true 1e-10" % n,
            "cells": nc, "unknowns": N, "nnz_G": nnz, "blocks_G": nb,
            "parallelism": (f"face rows partitioned over {world} GPUs (NCCL halo send/recv + allreduce)"
                            if world > 1 else "1 GPU"),
            "l2": "working set > L2 (G = %.2f GB per SpMV) and a 256 MB L2 flush before each step" % (8 * nnz / 1e9)}


def full_sizes(n=1024):
    nc = 2 * n * n
    nf_int = 3 * n * n - 2 * n
    nb = nf_int + 12 * (n - 1) ** 2 + 8 * (n - 1)
    return nc, 4 * nb, nb, 2 * nf_int


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    nc, nnz, nb, N = full_sizes()
    iters_full = ITERS_CONFIG1_MEASURED or 170000
    vals = []
    samples = []
    for i in range(args.warmup + args.steps):
        s = oracle_sample()
        if i >= args.warmup:
            vals.append(oracle_extrapolate(s, nc, nnz, iters_full))
            samples.append(s)
    v = statistics.mean(vals)
    s = samples[-1]
    sample_desc = (f"oracle on configs[1]-family mesh n={s['n']} ({s['nc']} cells): mesh+hybridise+recover "
                   f"timed in full, PCG timed over {s['iters']} iterations; extrapolated per cell and per "
                   f"nnz x {iters_full} iterations (B200-measured count) to n=1024")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(1024, args.gpus),
            "cpu_baseline": {"value": v, "unit": "s", "cores": 1, "kind": "oracle", "sample": sample_desc},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
# solver per config
OTHER_SOLVERS = {2: dict(method="dc", coarse=64, mu_inner=1.0),
                 3: dict(method="dc", coarse=64, mu_inner=0.5, inner_rtol=1e-7),
                 4: dict(method="pcg_afw2", matrix_free=1, coarse=16)}


def _ev(torch, stream):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


def stage_times(P, cfg, coords, cells, fbar, stream):
    """One configs[1] step with CUDA events between the four C-ABI calls."""
    import torch
    torch.cuda.synchronize()
    e = [_ev(torch, stream)]
    mesh = P.cr_build_mesh(coords, cells)
    e.append(_ev(torch, stream))
    hyb = P.cr_hybridise(mesh, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar))
    e.append(_ev(torch, stream))
    W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=coords.device)
    rep = P.cr_solve(hyb, W, METHOD, rtol=cfg.rtol, check_every=64, matrix_free=MATRIX_FREE, coarse=COARSE,
                     max_iter=MAX_ITER)
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
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.time_march(coords, cells, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar), nsteps, method=METHOD,
                       rtol=cfg.rtol, matrix_free=MATRIX_FREE, coarse=COARSE, check_every=64, max_iter=MAX_ITER)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    reps = out["reports"]
    return {"steps": nsteps, "total_s": a.elapsed_time(b) * 1e-3, "iterations": [r["iterations"] for r in reps],
            "solve_s": [r["seconds"] for r in reps], "rel_res_true": [r["rel_res_true"] for r in reps],
            "note": "step 1 includes the preconditioner / coarse-space setup; later steps reuse them"}


def newton_cavity(P, ci, dev, stream, n=256, nu=0.01, tol=5e-7):
    """Steady lid-driven cavity (Re = 1/nu) by Newton's method (tolerance of P:L783-799
    Table 7), each step through the hybrid path (NS step + CR_DC_FGMRES)."""
    import torch
    coords, cells = ci.square_mesh(n, 0.0, 4)
    wall = ci.lid_dirichlet_2d(coords, cells)
    tg = lambda a: torch.from_numpy(a).to(dev)
    f = torch.zeros((cells.shape[0], 2), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.newton_ns(tg(coords), tg(cells), nu, f, tg(wall), tol=tol, mis_seed=44, coarse=32, mu_inner=0.5,
                      inner_rtol=1e-7)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    return {"workload": f"2D lid-driven cavity n={n} Re={1 / nu:g}, Newton to ||dU|| <= {tol:g} ||U||",
            "newton_steps": len(out["history"]), "history": out["history"], "total_s": a.elapsed_time(b) * 1e-3,
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
    sol = OTHER_SOLVERS[idx]
    torch.cuda.synchronize()
    a = _ev(torch, stream)
    out = P.hybrid_method(coords, cells, prob, rtol=cfg.rtol, check_every=64, **sol)
    b = _ev(torch, stream)
    torch.cuda.synchronize()
    rep = out["report"]
    kind = {"stokes": "transient Stokes" if cfg.mu > 0 else "steady Stokes", "ns_step": "Navier-Stokes Newton step"}
    r = {"workload": f"configs[{idx}] {cfg.dim}D {kind[cfg.physics]} n={cfg.n} (nu={cfg.nu})", "solver": sol,
         "time_to_solution_s": a.elapsed_time(b) * 1e-3, "solve_s": rep["seconds"],
         "iterations": rep["iterations"], "rel_res_true": rep["rel_res_true"],
         "unknowns": out["hybrid"].n_rows, "cells": out["mesh"].nc}
    if sol["method"] == "dc":
        r["inner_iterations"] = rep["inner_iterations"]
    del out
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override mesh size (debug only; not a bench value)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    args = ap.parse_args()
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

    def barrier():
        if world > 1:
            dist.barrier()

    cfg = ci.CONFIGS[CONFIG_IDX]
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
        rep = P.cr_solve(hyb, W, METHOD, rtol=cfg.rtol, check_every=64, matrix_free=MATRIX_FREE, coarse=COARSE,
                         max_iter=MAX_ITER)
        U, Pp, diag = P.cr_recover(hyb, W)
        return mesh, hyb, rep, U, Pp, diag

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    barrier()
    torch.cuda.synchronize()
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
    barrier()
    ms = [a.elapsed_time(b) for a, b in evs]
    ms_per_step = sum(ms) / len(ms)
    t = torch.tensor([ms_per_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item())
    mesh, hyb, rep = out[0], out[1], reps[-1]
    N, nnz, nb = hyb.n_rows, hyb.nnz, hyb.nblocks

    # ---- per-kernel rooflines: each kernel of the PCG step re-launched standalone on the same
    # stream and timed with CUDA events (the in-solve launches live inside a CUDA graph)
    peak, peak_src = measured_peaks()
    N8 = 8 * N
    pinfo = hyb.precond_info()
    slots = 2 if mesh.dim == 2 else 3

    def time_launch(fn, nrep=50):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nrep):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / nrep * 1e-3

    x = torch.randn(N, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    spmv_s = time_launch(lambda: hyb.spmv(x, y))
    spmv_bytes = 8 * nnz + 4 * nb + N8 + N8          # values + block cols + x once + y
    mf_s = time_launch(lambda: hyb.spmv_mf(x, y))
    minfo = hyb.mf_info()
    mf_bytes = minfo["bytes"] + N8 + N8              # per-cell factors + x once + q once
    prec_s = time_launch(lambda: hyb.apply_precond("pcg_afw", x, y))
    prec2_s = time_launch(lambda: hyb.apply_precond(METHOD, x, y))
    # patch operator + r read + slot contributions written, then read back and z written
    prec_bytes = pinfo["bytes"] + N8 + slots * N8 + slots * N8 + N8
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "spmv_dram_bytes.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # PCG-two-level iteration: G apply + update (x,p,r,q read; x,r write) + patch apply + coarse
    # (restriction reads r and the fp32 row basis, E^-1 once) + p update (+ basis again)
    g_bytes = mf_bytes if MATRIX_FREE else spmv_bytes
    cinfo = hyb.coarse_info()
    coarse_bytes = N8 + 8 * N + cinfo["solve_bytes"] + 8 * N   # r, (x, a) fp32, E^-1 or ND fronts, (x, a) again
    iter_bytes = g_bytes + 6 * N8 + (pinfo["bytes"] + N8 + slots * N8) + coarse_bytes + (slots * N8 + 2 * N8)
    iter_gbs = iter_bytes * rep["iterations"] / rep["seconds"] / 1e9 if rep["seconds"] > 0 else None

    def roof(kernel, bytes_, sec, traffic_=None):
        return {"kernel": kernel, "bound": "hbm", "achieved": bytes_ / sec / 1e9, "peak": peak, "unit": "GB/s",
                "frac": bytes_ / sec / 1e9 / peak, "traffic": traffic_, "peak_source": peak_src,
                "algorithmic_bytes": bytes_, "launch_s": sec}

    prec_traffic = None   # ncu --set full DRAM bytes of k_afw_apply (the zsum's slot read-back is not in it)
    afile = os.path.join(ROOT, "profiles", "afw_dram_bytes.json")
    if os.path.exists(afile) and mesh.dim == 2:
        try:
            prec_traffic = json.load(open(afile)).get("dram_bytes_per_launch")
        except Exception:
            prec_traffic = None
    prec2_bytes = prec_bytes + coarse_bytes
    kernels = {
        "mf": roof("k_mf_spmv (matrix-free factored G x, per-cell factors, the in-solve G apply)", mf_bytes, mf_s),
        "precond": roof("k_afw_apply + k_afw_zsum (patch additive Schwarz z = M^-1 r)", prec_bytes, prec_s, prec_traffic),
        "precond_two_level": roof("coarse restrict + gather + E^-1 solve (nested dissection) + patch apply + combine (z = M2^-1 r)",
                                  prec2_bytes, prec2_s),
        "spmv": roof("k_spmv (assembled sliced block-ELL G x, same row code as the assembled PCG SpMV)",
                     spmv_bytes, spmv_s, traffic),
    }
    dominant = "mf" if mf_s >= prec_s else "precond"

    # ---- one-level patch PCG (assembled G), and the north star's baseline solver (Jacobi PCG)
    Wa = torch.zeros(N, dtype=torch.float64, device=dev)
    repa = P.cr_solve(hyb, Wa, "pcg_afw", rtol=cfg.rtol, check_every=64, matrix_free=0)
    Wj = torch.zeros(N, dtype=torch.float64, device=dev)
    repj = P.cr_solve(hyb, Wj, "pcg", rtol=cfg.rtol, check_every=64)

    # ---- e2e through the public API from HOST buffers (pinned host -> device -> host)
    # (the handles of the timed steps are released first, as a caller's next solve would)
    nc_full, ndim = mesh.nc, mesh.dim
    del out, hyb, mesh, Wa, Wj, x, y
    e2e = None
    if not args.no_e2e:
        def e2e_step():
            return P.hybrid_method_host(coords_h, cells_h, fbar_h, cfg.mu, cfg.nu, METHOD, cfg.rtol, comm=comm,
                                        matrix_free=MATRIX_FREE, coarse=COARSE)

        o2 = e2e_step()   # warm-up
        del o2
        e2e_ms = []
        for _ in range(args.steps):   # K steps, each with its own host -> device -> host copies
            torch.cuda.synchronize()
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            res = e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(a.elapsed_time(b))
            o2 = res   # the previous step's handles are released outside the timed region
            del res
        e2e_s = sum(e2e_ms) / len(e2e_ms) * 1e-3
        t2 = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        h2d = coords_h.numel() * 8 + cells_h.numel() * 4 + fbar_h.numel() * 8
        d2h = o2["U_host"].numel() * 8 + o2["P_host"].numel() * 8
        e2e = {"value": float(t2.item()), "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- stage times of one configs[1] step (assembly cells/s) and time-to-solution of the
    # other configs (one run each, not part of the timed step; single GPU only)
    stages, others, tstep, newton, table4 = None, None, None, None, None
    if world == 1 and not args.no_other_configs:
        stages = stage_times(P, cfg, coords, cells, fbar, stream)
        tstep = time_stepping(P, cfg, coords, cells, fbar, stream)
        newton = newton_cavity(P, ci, dev, stream)
        table4 = direct_table4(P, ci, dev, stream)
        others = {}
        for idx in (2, 3, 4):
            others[f"configs[{idx}]"] = other_config(P, ci, idx, dev, stream)
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s = oracle_sample()
        v = oracle_extrapolate(s, nc_full, nnz, repj["iterations"])
        cpu = {"value": v, "unit": "s", "cores": 1, "kind": "oracle",
               "sample": (f"oracle on configs[1]-family mesh n={s['n']} ({s['nc']} cells): mesh+hybridise+recover "
                          f"timed in full ({s['mesh_s'] + s['hyb_s'] + s['rec_s']:.1f} s), PCG over {s['iters']} "
                          f"iterations ({s['iter_s'] * 1e3:.2f} ms/it); extrapolated per cell and per nnz x "
                          f"{repj['iterations']} Jacobi-PCG iterations (the oracle's solver, count measured on the B200 in this run) to the full workload")}

    launches = rep["kernel_launches"] + 25     # mesh (sort/scan/geometry ~15), hybridise 1, recover 3, copies
    launches += 12   # patch build (pairs, sort, scans, setup)
    launches += (5 ** ndim) * ndim ** 2 * 8 + 200   # coarse E assembly (colour passes) + ND factorisation
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_per_step / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_steps_rank0": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.n or cfg.n, world),
            "pcg": {"method": METHOD, "matrix_free": MATRIX_FREE, "coarse_intervals": COARSE, "coarse": cinfo,
                    "iterations": rep["iterations"],
                    "rel_res_true": rep["rel_res_true"], "solve_s": rep["seconds"],
                    "ms_per_iter": rep["seconds"] / max(rep["iterations"], 1) * 1e3,
                    "iter_gbs": iter_gbs, "iter_bytes": iter_bytes, "precond": pinfo, "mf": minfo},
            "pcg_patch_assembled_G": {"iterations": repa["iterations"], "rel_res_true": repa["rel_res_true"],
                                "solve_s": repa["seconds"],
                                "ms_per_iter": repa["seconds"] / max(repa["iterations"], 1) * 1e3},
            "pcg_jacobi": {"iterations": repj["iterations"], "rel_res_true": repj["rel_res_true"],
                           "solve_s": repj["seconds"],
                           "ms_per_iter": repj["seconds"] / max(repj["iterations"], 1) * 1e3},
            "roofline": kernels[dominant],
            "roofline_kernels": kernels,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "stages_configs1": stages,
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
