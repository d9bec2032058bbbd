"""Writes the stored U/P references of the bench-setting parity tests (tests/test_gpu_bench_parity.py).

Calls ONLY oracle/ (and the seeded generators in cr_inputs): the coupled saddle system
eq. (syslin) assembled by oracle.assemble_coupled and solved by
oracle.direct_refined (SuperLU + iterative refinement with a binary128 residual).  The hybrid
method reaches exactly this solution (abstract P:L13; "we get P_hat = P"), so it is
the reference for U and P at any size the direct solve can handle.  Stored here because the
sparse LU of these sizes takes minutes (3D n = 16: ~8 min, 2D n = 512: ~15 min on one core).

    python tests/golden/make_refs.py [name ...]
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import cr_inputs as ci  # noqa: E402
import oracle as O  # noqa: E402

# name -> (BASELINE.json config family, mesh size); inputs = cr_inputs.make_inputs(CONFIGS[idx], n)
REFS = {"coupled_2d_n512": (1, 512), "coupled_3d_n16": (4, 16)}


def reference(idx, n):
    cfg = ci.CONFIGS[idx]
    inp = ci.make_inputs(cfg, n=n)
    m = O.build_mesh(inp["coords"], inp["cells"])
    prm, data = O.Params(mu=cfg.mu, nu=cfg.nu), O.Data(fbar=inp["fbar"])
    M, rhs, nU = O.assemble_coupled(m, prm, data)
    info = {}
    x = O.direct_refined(M, rhs, info=info)
    U = x[:nU].reshape(-1, m.dim)
    P = np.insert(x[nU:], prm.k0, 0.0)
    return U, P, info["refine_hist"]


def main(names):
    for name in names:
        idx, n = REFS[name]
        t = time.time()
        U, P, hist = reference(idx, n)
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, U=U, P=P, refine_hist=np.asarray(hist), config=idx, n=n)
        print(f"{name}: {time.time() - t:.0f} s, refinement residuals {hist} -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(REFS))
