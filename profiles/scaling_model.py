"""Strong-scaling model of configs[4] (3D n = 128) over 1..8 GPUs from MEASURED single-GPU times.

    python profiles/scaling_model.py profiles/r02_launches_bench.csv BENCH_LINE.json > profiles/r02_scaling_model.md

Inputs
  * an ncu launch list of the bench command (gpu__time_duration.sum per launch, serialised and cold:
    used for the SHARE of each kernel in one PCG iteration, then scaled to the measured ms/iteration);
  * the bench JSON line (stage times, iterations, setup time of the solve).

Model: rank q of N owns 1/N of the face rows (z-slabs).  Per iteration, the kernels
over rows or cells (matrix-free G, vector updates, patch solves, direction update, restriction) take
1/N of their single-GPU time; the coarse gather and the nested-dissection coarse solve are
replicated on every rank; communication adds 3 scalar allreduces, one allreduce of the coarse
vector c (nE doubles) and one halo exchange (two neighbours, one vertex plane of faces each).  Setup:
hybridisation, matrix-free factors, patch blocks and the coarse E assembly divide by N (E: plus one
allreduce of D^2 nE doubles per colour); the mesh, the ND factorisation and the recovery are
replicated (plus the allgather of W).  Variant "overlap": the coarse path on its own stream and
communicator (CR_DIST_OVERLAP=1) runs concurrently with the rank's fine-level kernels.

Communication constants (B200_PROFILING.md measured NVLink references; latency assumed):
  allreduce of a few doubles: 15 us; bandwidth terms at 725 GB/s (allreduce bus) / 770 GB/s (peer copy).
"""
import csv
import json
import sys

LAT = 15e-6          # small collective latency on 8 x B200 NVLink (assumed)
BW_AR = 725e9        # measured 8-rank allreduce bus bandwidth
BW_P2P = 770e9       # measured peer copy per direction

import re

# the iteration's kernels (exact base names; setup variants such as k_mf_spmv_colour,
# k_coarse_restrict3m or k_coarse_gather_all excluded)
DIST = re.compile(r"(k_mf_spmv<3, 1>|k_pcg_update_r|k_afw_apply(_sh)?<3, 3, \d+, (1, )?5>|k_pcg_pdir_afw2<3, 3>|"
                  r"cr::k_coarse_restrict3$)")
REPL = re.compile(r"(k_coarse_gather<3>|cr::k_nd_solve$|cr::k_nd_phase$|cr::k_nd_cdot$)")


def iteration_split(path):
    """(distributed, replicated) fractions of one PCG iteration from an ncu launch list."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    dist = repl = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name, t = r[ki].split("(")[0].replace("void ", "").strip(), float(r[vi].replace(",", ""))
        if DIST.search(name):
            dist += t
        elif REPL.search(name):
            repl += t
    tot = dist + repl
    return dist / tot, repl / tot


def main():
    # optional overrides key=value (another coarse grid measured on one GPU): iterations, ms_per_iter,
    # repl_ms (replicated coarse ms per iteration), nd_fact (s), setup (s), nE, label
    ov = dict(a.split("=", 1) for a in sys.argv[3:])
    fd, fr = iteration_split(sys.argv[1])
    line = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    pcg, st = line["pcg"], line.get("stages")
    if not st:   # a bench line without stage times: the r02 CR_TRACE values
        st = {"mesh_s": 0.009, "hybridise_s": 0.089, "recover_s": 0.028}
    it = int(ov.get("iterations", pcg["iterations"]))
    ms_it = float(ov.get("ms_per_iter", pcg["ms_per_iter"])) * 1e-3
    setup = float(ov.get("setup", pcg["setup_s"]))
    nE = int(ov.get("nE", pcg["coarse"]["nE"]))
    N1 = line["config"]["unknowns"]
    n = round((line["config"]["cells"] / 6) ** (1 / 3))
    t_dist, t_repl = fd * ms_it, fr * ms_it
    if "repl_ms" in ov:
        t_repl = float(ov["repl_ms"]) * 1e-3
        t_dist = ms_it - t_repl
        fd, fr = t_dist / ms_it, t_repl / ms_it
    if "label" in ov:
        print(f"**{ov['label']}**\n")
    # setup split (single-GPU trace): ND factorisation replicated, the rest distributed
    nd_fact = float(ov.get("nd_fact", line.get("nd_factorisation_s", 0.2)))
    setup_dist = max(setup - nd_fact, 0.0)
    halo_bytes = 2 * 12 * (n + 1) ** 2 * 3 * 8         # two neighbours, one vertex plane of faces each
    print("| N | per-iteration (ms) | iterations (s) | setup (s) | step (s) | efficiency | overlap: step (s) | overlap: efficiency |")
    print("|---|---|---|---|---|---|---|---|")
    t1 = None
    for N in (1, 2, 4, 8):
        comm = 0.0 if N == 1 else 3 * LAT + (LAT + 8 * nE / BW_AR) + (LAT + halo_bytes / BW_P2P)
        per_it = t_dist / N + t_repl + comm
        per_it_ov = (max(t_dist / N, t_repl) if N > 1 else per_it) + comm
        e_setup = 0.0 if N == 1 else 125 * (LAT + 8 * 9 * nE / BW_AR)
        s_setup = setup_dist / N + nd_fact + e_setup
        other = st["mesh_s"] + st["hybridise_s"] / N + st["recover_s"] + (0 if N == 1 else 8 * N1 / BW_P2P)
        step = other + s_setup + it * per_it
        step_ov = other + s_setup + it * per_it_ov
        if t1 is None:
            t1 = step
        print(f"| {N} | {per_it * 1e3:.3f} | {it * per_it:.3f} | {s_setup:.3f} | {step:.3f} | {t1 / (N * step):.2f} | "
              f"{step_ov:.3f} | {t1 / (N * step_ov):.2f} |")
    print(f"\nsingle-GPU iteration {ms_it * 1e3:.3f} ms: {fd:.2f} distributed (rows / cells), {fr:.2f} replicated "
          f"(coarse gather + nested-dissection solve), from the launch list's kernel shares")


if __name__ == "__main__":
    main()
