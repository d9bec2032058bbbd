"""Iteration counts of the two-level PCG (patch additive Schwarz + theta * coarse correction) against
the relative weight theta of the coarse term (CR_COARSE_WEIGHT).
Usage: python profiles/coarse_weight_sweep.py [config idx ...]   (default 1 4)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
import cr_inputs as ci  # noqa: E402
import paper_2101_03777_b200 as P  # noqa: E402

dev = torch.device("cuda:0")
idxs = [int(a) for a in sys.argv[1:]] or [1, 4]
thetas = [float(t) for t in os.environ.get("THETAS", "1 0.5 2 3 4 6 8").split()]
for idx in idxs:
    cfg = ci.CONFIGS[idx]
    inp = ci.make_inputs(cfg)
    tg = lambda a: torch.from_numpy(a).to(dev)
    coords, cells, fbar = tg(inp["coords"]), tg(inp["cells"]), tg(inp["fbar"])
    sol, rtol = B._solver(idx)
    for th in thetas:
        os.environ["CR_COARSE_WEIGHT"] = repr(th)
        out = P.hybrid_method(coords, cells, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar), rtol=rtol, check_every=64, **sol)
        torch.cuda.synchronize()
        r = out["report"]
        print(f"configs[{idx}] theta={th:g}: iterations={r['iterations']} solve_s={r['seconds']:.4f} "
              f"rel_res_true={r['rel_res_true']:.3e} converged={r['converged']}", flush=True)
        del out
