"""ORACLE — TEST INFRASTRUCTURE ONLY (not part of the product path).

A plain, slow, obviously-correct CPU implementation of what the hybrid method of
Chenier & Eymard (arXiv 2101.03777, /root/reference/PAPER.md) computes, written
from the paper.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code
with the CUDA path (``paper_2101_03777_b200``) and never imports it; both only
share the seeded input generators in ``cr_inputs``.

Layout
  mesh.py      C-1  mesh, faces, geometry
  scheme.py    C-2..C-5, C-7  local blocks, shift, coupled and hybrid
               assembly, recovery
  krylov.py    C-6  direct solve + refinement, CPU Krylov      (§4)
  post.py      C-8  error norms, zero-mean pressure
  timestep.py  backward-Euler steps with one coupled matrix
  newton.py    Newton's method for steady Navier-Stokes
  cell_f128.c  per-cell algebra in binary128 (libquadmath)

Every function cites the PAPER.md lines it follows ("P:Lnnn").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_f128.so")
_SRC = os.path.join(_HERE, "cell_f128.c")

_lib = None


def build(force: bool = False) -> str:
    """Compile the binary128 cell-algebra helper (gcc, -ffp-contract=off)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11",
               _SRC, "-o", _SO, "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
        _lib.or_dot_f128.restype = ctypes.c_double
    return _lib


from .mesh import Mesh, build_mesh  # noqa: E402
from .scheme import (Params, Data, cell_arrays, local_blocks, mis_priority, shift_E,  # noqa: E402
                     assemble_coupled, hybridise, recover, hybrid_pipeline, eliminate_cells,
                     recover_cells)
from .krylov import (residual_f128, direct_refined, pcg, minres, bicgstab, gmres)  # noqa: E402
from .post import zero_mean, errors  # noqa: E402
from .timestep import lumped_mass, backward_euler  # noqa: E402
from .newton import cell_face_values, newton_ns  # noqa: E402

__all__ = ["build", "lib", "Mesh", "build_mesh", "Params", "Data", "cell_arrays",
           "local_blocks", "mis_priority", "shift_E", "assemble_coupled", "hybridise",
           "recover", "hybrid_pipeline", "eliminate_cells", "recover_cells", "residual_f128", "direct_refined", "pcg",
           "minres", "bicgstab", "gmres", "zero_mean", "errors", "lumped_mass", "backward_euler", "cell_face_values", "newton_ns"]
