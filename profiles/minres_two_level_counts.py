"""MINRES iteration counts on the steady Stokes hybrid system (configs[2] family): |patch| vs |patch| +
coarse |E|^-1, true residual 1e-10, n = 32 .. 256 (CR_MINRES_AFW vs CR_MINRES_AFW2).

    python profiles/minres_two_level_counts.py 32 64 128 256
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import cr_inputs as ci
import paper_2101_03777_b200 as P
dev = torch.device("cuda:0")
cfg = ci.CONFIGS[2]
out = []
for n in [int(a) for a in sys.argv[1:]] or (32, 64, 128):
    inp = ci.make_inputs(cfg, n=n)
    prob = P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=torch.from_numpy(inp["fbar"]).to(dev), shift=P.CR_SHIFT_MIS,
                     mis_seed=cfg.mis_seed)
    mesh = P.cr_build_mesh(torch.from_numpy(inp["coords"]).to(dev), torch.from_numpy(inp["cells"]).to(dev))
    for method, H in (("minres_afw", 0), ("minres_afw2", 8), ("minres_afw2", 16), ("minres_afw2", 32)):
        hyb = P.cr_hybridise(mesh, prob)
        W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=dev)
        t0 = time.time()
        rep = P.cr_solve(hyb, W, method, rtol=1e-10, max_iter=min(400000, 2000 * n), check_every=256, coarse=H,
                         raise_on_fail=False)
        torch.cuda.synchronize()
        r = dict(n=n, method=method, H=H, iterations=rep["iterations"], rel_res_true=rep["rel_res_true"],
                 converged=bool(rep["converged"]), seconds=rep["seconds"], coarse=hyb.coarse_info())
        print(json.dumps(r), flush=True)
