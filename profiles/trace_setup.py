import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench as B, cr_inputs as ci, paper_2101_03777_b200 as P
dev = torch.device("cuda:0")
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = ci.CONFIGS[idx]
inp = ci.make_inputs(cfg)
tg = lambda a: torch.from_numpy(a).to(dev)
coords, cells, fbar = tg(inp["coords"]), tg(inp["cells"]), tg(inp["fbar"])
sol, rtol = B._solver(idx)
for rep in range(3):
    print(f"--- pass {rep}", file=sys.stderr, flush=True)
    out = P.hybrid_method(coords, cells, P.Problem(mu=cfg.mu, nu=cfg.nu, fbar=fbar), rtol=rtol, check_every=64, **sol)
    torch.cuda.synchronize()
    r = out["report"]
    print(r["iterations"], r["seconds"], r.get("setup_seconds"), file=sys.stderr, flush=True)
    del out
