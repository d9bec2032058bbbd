"""paper_2101_03777_b200 — B200-native hybrid method for the Crouzeix-Raviart Stokes /
Navier-Stokes systems (Chenier & Eymard, arXiv 2101.03777).

Thin Python binding of the C ABI ``include/cr.h`` (libcr.so, built in-tree for sm_100a).
Every function here only marshals torch CUDA tensors into device pointers and calls the
library; all arithmetic runs in the CUDA kernels.  There is no CPU fallback: importing
this package fails loudly when libcr.so is missing, and every call checks that its
tensors live on a CUDA device.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcr.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libcr.so not found at {LIB_PATH}: build it with `python -m paper_2101_03777_b200.build` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ ABI mirror (include/cr.h)
CR_OK = 0
STATUS = {0: "CR_OK", -1: "CR_ERR_INVALID_ARG", -2: "CR_ERR_CUDA", -3: "CR_ERR_OOM",
          -4: "CR_ERR_NONMANIFOLD", -5: "CR_ERR_DEGENERATE_CELL", -6: "CR_ERR_NO_INTERIOR_FACE",
          -7: "CR_ERR_SINGULAR_LOCAL", -8: "CR_ERR_NOT_CONVERGED", -9: "CR_ERR_BREAKDOWN",
          -10: "CR_ERR_STAGNATION", -11: "CR_ERR_NCCL"}
CR_STOKES, CR_NS_NEWTON_STEP = 0, 1
CR_SHIFT_NONE, CR_SHIFT_MIS = 0, 1
(CR_PCG_JACOBI, CR_PCG_BLOCKJACOBI, CR_MINRES_ABSJACOBI, CR_BICGSTAB_JACOBI, CR_GMRES_JACOBI,
 CR_PCG_AFW, CR_MINRES_AFW, CR_PCG_AFW2, CR_DC_FGMRES, CR_MINRES_AFW2) = range(10)
METHODS = {"pcg": CR_PCG_JACOBI, "pcg_block": CR_PCG_BLOCKJACOBI, "minres": CR_MINRES_ABSJACOBI,
           "bicgstab": CR_BICGSTAB_JACOBI, "gmres": CR_GMRES_JACOBI, "pcg_afw": CR_PCG_AFW,
           "minres_afw": CR_MINRES_AFW, "pcg_afw2": CR_PCG_AFW2, "dc": CR_DC_FGMRES, "minres_afw2": CR_MINRES_AFW2}


class CrError(RuntimeError):
    def __init__(self, status: int, msg: str, report=None):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.report = report


class MeshInfo(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nv", ctypes.c_int64), ("nc", ctypes.c_int64),
                ("nf", ctypes.c_int64), ("nf_int", ctypes.c_int64), ("n_unknowns", ctypes.c_int64)]


class Params(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_double), ("nu", ctypes.c_double), ("gauge_cell", ctypes.c_int32),
                ("physics", ctypes.c_int32), ("shift", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("mis_seed", ctypes.c_uint64), ("lambda_factor", ctypes.c_double)]


class Data(ctypes.Structure):
    _fields_ = [("fbar_d", ctypes.c_void_p), ("dirichlet_d", ctypes.c_void_p),
                ("u_iter_d", ctypes.c_void_p), ("p_iter_d", ctypes.c_void_p)]


class SolverOpts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("restart", ctypes.c_int32), ("rtol", ctypes.c_double),
                ("max_iter", ctypes.c_int64), ("check_every", ctypes.c_int32), ("matrix_free", ctypes.c_int32),
                ("coarse", ctypes.c_int32), ("mu_inner", ctypes.c_double), ("inner_rtol", ctypes.c_double),
                ("refine_dd", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("rel_res_true", ctypes.c_double),
                ("rel_res_recursive", ctypes.c_double), ("converged", ctypes.c_int32),
                ("status", ctypes.c_int32), ("seconds", ctypes.c_double), ("spmv_calls", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("inner_iterations", ctypes.c_int64),
                ("kappa_lanczos_est", ctypes.c_double), ("lambda_min_est", ctypes.c_double),
                ("lambda_max_est", ctypes.c_double), ("bytes_moved", ctypes.c_double),
                ("refine_rounds", ctypes.c_int32), ("reserved", ctypes.c_int32), ("setup_seconds", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp, _i32, _i64, _st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
_P = ctypes.POINTER
_sig = {
    "cr_build_mesh": [_i32, _i64, _vp, _i64, _vp, _vp, _P(_vp)],
    "cr_mesh_info": [_vp, _P(MeshInfo)],
    "cr_mesh_export": [_vp] + [_vp] * 8 + [_vp],
    "cr_assemble_coupled": [_vp, _P(Params), _P(Data), _vp, _P(_vp)],
    "cr_coupled_info": [_vp, _P(_i64), _P(_i64)],
    "cr_coupled_export_csr": [_vp, _vp, _vp, _vp, _vp, _vp],
    "cr_hybridise": [_vp, _P(Params), _P(Data), _vp, _vp, _P(_vp)],
    "cr_hybrid_info": [_vp, _P(_i64), _P(_i64), _P(_i64)],
    "cr_hybrid_export_csr": [_vp, _vp, _vp, _vp, _vp, _vp],
    "cr_hybrid_export_shift": [_vp, _vp, _vp, _vp],
    "cr_spmv": [_vp, _vp, _vp, _vp],
    "cr_spmv_mf": [_vp, _vp, _vp, _vp],
    "cr_hybrid_mf_info": [_vp, _P(_i64), _P(_i64)],
    "cr_solve": [_vp, _P(SolverOpts), _vp, _vp, _P(SolveReport)],
    "cr_recover": [_vp, _vp, _vp, _vp, _vp, _vp],
    "cr_comm_init": [_vp, _i32, _i32, _P(_vp)],
    "cr_nccl_unique_id": [_vp],
    "cr_loopback_create": [_i32, _P(_vp)],
    "cr_comm_init_loopback": [_vp, _i32, _P(_vp)],
    "cr_hybrid_partition_info": [_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64)],
    "cr_partition_plan": [_i32, _i64, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp],
    "cr_apply_precond": [_vp, _i32, _vp, _vp, _vp],
    "cr_hybrid_precond_info": [_vp, _P(_i64), _P(_i32), _P(_i64), _P(_i64)],
    "cr_solve_profile": [_vp, _P(SolverOpts), _i32, _vp, _vp],
    "cr_transient_rhs": [_vp, _vp, _vp, _vp, _vp],
    "cr_hybrid_set_cell_rhs": [_vp, _vp, _vp, _vp],
    "cr_cell_face_values": [_vp, _vp, _vp, _vp, _vp],
    "cr_coarse_nd_plan": [_i32, _i32, _i32, _P(_i64), _P(_i32), _P(_i64), _P(_i64), _vp, _vp, _vp, _vp, _vp, _vp],
    "cr_sparse_direct_solve": [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _P(_i32)],
    "cr_hybrid_coarse_info": [_vp, _P(_i32), _P(_i64), _P(_i32), _P(_i64)],
    "cr_newton_update": [_i64, _vp, _vp, _i64, _vp, _vp, ctypes.c_double, _vp, _vp],
    "cr_coupled_rhs_norm": [_vp, _P(Params), _P(Data), _vp, _vp],
    "cr_hybrid_method_host": [_i32, _i64, _vp, _i64, _vp, _P(Params), _vp, _vp, _P(SolverOpts), _vp, _vp, _vp,
                              _P(MeshInfo), _P(SolveReport), _vp],
    "cr_pool_reserve": [_i64, _vp],
    "cr_pool_trim": [_i64],
}
for _name, _args in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _st
for _name in ("cr_destroy_mesh", "cr_destroy_coupled", "cr_destroy_hybrid", "cr_comm_destroy", "cr_loopback_destroy"):
    getattr(_lib, _name).argtypes = [_vp]
    getattr(_lib, _name).restype = None
_lib.cr_last_error.restype = ctypes.c_char_p
_lib.cr_version.restype = ctypes.c_char_p
_lib.cr_kernel_launches.restype = ctypes.c_int64
_lib.cr_kernel_launches.argtypes = []

ABI_SYMBOLS = sorted(list(_sig) + ["cr_destroy_mesh", "cr_destroy_coupled", "cr_destroy_hybrid",
                                   "cr_comm_destroy", "cr_loopback_destroy", "cr_last_error", "cr_version",
                                   "cr_kernel_launches"])


def _check(status: int, report=None):
    if status != CR_OK:
        raise CrError(status, _lib.cr_last_error().decode(), report)


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t: torch.Tensor | None, dtype=None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("libcr takes CUDA tensors only (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def version() -> str:
    return _lib.cr_version().decode()


def kernel_launches() -> int:
    """Kernels libcr launched in this process so far (cr_kernel_launches)."""
    return int(_lib.cr_kernel_launches())


def pool_reserve(nbytes: int, stream=None):
    """Map nbytes into libcr's own memory pool now (cr_pool_reserve; opt-in)."""
    _check(_lib.cr_pool_reserve(int(nbytes), _stream(stream)))


def pool_trim(keep_bytes: int = 0):
    """Return unused pool memory beyond keep_bytes to the device (cr_pool_trim)."""
    _check(_lib.cr_pool_trim(int(keep_bytes)))


# ------------------------------------------------------------------ handles
class Mesh:
    """cr_mesh handle (owns its device memory)."""

    def __init__(self, handle):
        self._h = handle
        info = MeshInfo()
        _check(_lib.cr_mesh_info(self._h, ctypes.byref(info)))
        self.dim, self.nv, self.nc = info.dim, info.nv, info.nc
        self.nf, self.nf_int, self.n_unknowns = info.nf, info.nf_int, info.n_unknowns

    def export(self, stream=None) -> dict:
        d, dev = self.dim, torch.device("cuda")
        out = dict(
            faces=torch.empty((self.nf, d), dtype=torch.int32, device=dev),
            face_cells=torch.empty((self.nf, 2), dtype=torch.int32, device=dev),
            cell_faces=torch.empty((self.nc, d + 1), dtype=torch.int32, device=dev),
            face_dof=torch.empty(self.nf, dtype=torch.int32, device=dev),
            vol=torch.empty(self.nc, dtype=torch.float64, device=dev),
            xK=torch.empty((self.nc, d), dtype=torch.float64, device=dev),
            xs=torch.empty((self.nf, d), dtype=torch.float64, device=dev),
            a=torch.empty((self.nc, d + 1, d), dtype=torch.float64, device=dev),
        )
        _check(_lib.cr_mesh_export(self._h, *[_ptr(out[k]) for k in
                                              ("faces", "face_cells", "cell_faces", "face_dof", "vol", "xK", "xs", "a")],
                                   _stream(stream)))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cr_destroy_mesh(self._h)
            self._h = None


def cr_build_mesh(coords: torch.Tensor, cells: torch.Tensor, stream=None) -> Mesh:
    """coords [nv, d] f64 CUDA, cells [nc, d+1] i32 CUDA -> Mesh."""
    d = coords.shape[1]
    h = ctypes.c_void_p()
    _check(_lib.cr_build_mesh(d, coords.shape[0], _ptr(coords, torch.float64), cells.shape[0],
                              _ptr(cells, torch.int32), _stream(stream), ctypes.byref(h)))
    return Mesh(h)


@dataclass
class Problem:
    """cr_params + cr_data (tensors stay alive as long as this object)."""
    mu: float
    nu: float
    fbar: torch.Tensor
    physics: int = CR_STOKES
    shift: int = CR_SHIFT_NONE
    mis_seed: int = 0
    lambda_factor: float = 1.1
    gauge_cell: int = 0
    dirichlet: torch.Tensor | None = None
    u_iter: torch.Tensor | None = None
    p_iter: torch.Tensor | None = None

    def params(self) -> Params:
        return Params(self.mu, self.nu, self.gauge_cell, self.physics, self.shift, 0,
                      self.mis_seed & 0xFFFFFFFFFFFFFFFF, self.lambda_factor)

    def data(self) -> Data:
        return Data(_ptr(self.fbar, torch.float64), _ptr(self.dirichlet, torch.float64),
                    _ptr(self.u_iter, torch.float64), _ptr(self.p_iter, torch.float64))


class Hybrid:
    """cr_hybrid handle: G (sliced block-ELL), S, shift, preconditioners."""

    def __init__(self, handle, mesh: Mesh):
        self._h = handle
        self.mesh = mesh
        nr, nnz, nb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.cr_hybrid_info(self._h, ctypes.byref(nr), ctypes.byref(nnz), ctypes.byref(nb)))
        self.n_rows, self.nnz, self.nblocks = nr.value, nnz.value, nb.value

    def partition_info(self) -> dict:
        r0, r1, ng, nglob = (ctypes.c_int64() for _ in range(4))
        _check(_lib.cr_hybrid_partition_info(self._h, ctypes.byref(r0), ctypes.byref(r1), ctypes.byref(ng),
                                             ctypes.byref(nglob)))
        return dict(row0=r0.value, row1=r1.value, nghost=ng.value, nglobal=nglob.value)

    def export_csr(self, stream=None):
        dev = torch.device("cuda")
        rp = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        v = torch.empty(self.nnz, dtype=torch.float64, device=dev)
        S = torch.empty(self.n_rows, dtype=torch.float64, device=dev)
        _check(_lib.cr_hybrid_export_csr(self._h, _ptr(rp), _ptr(ci), _ptr(v), _ptr(S), _stream(stream)))
        return rp, ci, v, S

    def export_shift(self, stream=None):
        dev = torch.device("cuda")
        inM1 = torch.empty(self.mesh.nc, dtype=torch.uint8, device=dev)
        E = torch.empty((self.mesh.nc, self.mesh.dim + 1), dtype=torch.float64, device=dev)
        _check(_lib.cr_hybrid_export_shift(self._h, _ptr(inM1), _ptr(E), _stream(stream)))
        return inM1, E

    def spmv(self, x: torch.Tensor, y: torch.Tensor, stream=None):
        _check(_lib.cr_spmv(self._h, _ptr(x, torch.float64), _ptr(y, torch.float64), _stream(stream)))
        return y

    def spmv_mf(self, x: torch.Tensor, y: torch.Tensor, stream=None):
        """y = G x with the matrix-free factored operator."""
        _check(_lib.cr_spmv_mf(self._h, _ptr(x, torch.float64), _ptr(y, torch.float64), _stream(stream)))
        return y

    def mf_info(self) -> dict:
        nc, nb = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.cr_hybrid_mf_info(self._h, ctypes.byref(nc), ctypes.byref(nb)))
        return dict(ncells=nc.value, bytes=nb.value)

    def apply_precond(self, method: str | int, r: torch.Tensor, z: torch.Tensor, stream=None):
        """z = M^{-1} r for the preconditioner of `method`."""
        m = METHODS[method] if isinstance(method, str) else int(method)
        _check(_lib.cr_apply_precond(self._h, m, _ptr(r, torch.float64), _ptr(z, torch.float64), _stream(stream)))
        return z

    def coarse_info(self) -> dict:
        H, nE, nd, nb = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
        _check(_lib.cr_hybrid_coarse_info(self._h, ctypes.byref(H), ctypes.byref(nE), ctypes.byref(nd), ctypes.byref(nb)))
        return dict(H=H.value, nE=nE.value, nested_dissection=bool(nd.value), solve_bytes=nb.value)

    def precond_info(self) -> dict:
        npatch, kmax, nfb, nby = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.cr_hybrid_precond_info(self._h, ctypes.byref(npatch), ctypes.byref(kmax), ctypes.byref(nfb),
                                           ctypes.byref(nby)))
        return dict(npatch=npatch.value, kmax=kmax.value, nfallback=nfb.value, bytes=nby.value)

    def transient_rhs(self, U_prev: torch.Tensor, stream=None):
        """Cell right-hand sides (R [nc, d+1, d], g [nc]) of the backward-Euler step from U_prev
        [nf_int, d] (lumped mass P:L129)."""
        m = self.mesh
        dev = U_prev.device
        R = torch.empty((m.nc, m.dim + 1, m.dim), dtype=torch.float64, device=dev)
        g = torch.empty(m.nc, dtype=torch.float64, device=dev)
        _check(_lib.cr_transient_rhs(self._h, _ptr(U_prev, torch.float64), _ptr(R), _ptr(g), _stream(stream)))
        return R, g

    def set_cell_rhs(self, R: torch.Tensor | None = None, g: torch.Tensor | None = None, stream=None):
        """S of the same G for explicit cell right-hand sides (None: the data-derived S)."""
        _check(_lib.cr_hybrid_set_cell_rhs(self._h, None if R is None else _ptr(R, torch.float64),
                                           None if g is None else _ptr(g, torch.float64), _stream(stream)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cr_destroy_hybrid(self._h)
            self._h = None


def cr_hybridise(mesh: Mesh, prob: Problem, stream=None, comm: "Comm | None" = None) -> Hybrid:
    """G and S of G W = S.  With a multi-rank ``comm`` only this rank's rows."""
    h = ctypes.c_void_p()
    prm, data = prob.params(), prob.data()
    _check(_lib.cr_hybridise(mesh._h, ctypes.byref(prm), ctypes.byref(data), comm._h if comm else None,
                             _stream(stream), ctypes.byref(h)))
    hy = Hybrid(h, mesh)
    hy.comm = comm          # keep the communicator alive as long as the handle
    return hy


# ------------------------------------------------------------------ multi-GPU
def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (call on rank 0, broadcast to the others)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.cr_nccl_unique_id(buf))
    return buf.raw


class LoopbackGroup:
    """In-process group of ``n`` ranks sharing one GPU (testing the partitioned path)."""

    def __init__(self, n: int):
        self._h = ctypes.c_void_p()
        _check(_lib.cr_loopback_create(n, ctypes.byref(self._h)))
        self.n = n

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cr_loopback_destroy(self._h)
            self._h = None


class Comm:
    """cr_comm handle: NCCL (one process per GPU) or in-process loopback."""

    def __init__(self, handle, rank: int, nranks: int, keep=None):
        self._h, self.rank, self.nranks, self._keep = handle, rank, nranks, keep

    @classmethod
    def nccl(cls, unique_id: bytes, rank: int, nranks: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(_lib.cr_comm_init(ctypes.c_char_p(unique_id), rank, nranks, ctypes.byref(h)))
        return cls(h, rank, nranks)

    @classmethod
    def loopback(cls, group: LoopbackGroup, rank: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(_lib.cr_comm_init_loopback(group._h, rank, ctypes.byref(h)))
        return cls(h, rank, group.n, keep=group)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cr_comm_destroy(self._h)
            self._h = None


def partition_plan(dim: int, cell_faces, face_cells, face_dof, rank: int, nranks: int) -> dict:
    """Host partition plan (no GPU): numpy int32 arrays as exported by the mesh."""
    import numpy as np
    cf = np.ascontiguousarray(cell_faces, dtype=np.int32)
    fc = np.ascontiguousarray(face_cells, dtype=np.int32)
    fd = np.ascontiguousarray(face_dof, dtype=np.int32)
    df = np.ascontiguousarray(np.nonzero(fd >= 0)[0], dtype=np.int32)
    nf_int = len(df)
    rr = np.zeros(2, np.int64)
    rc = np.zeros(nranks, np.int64)
    sc = np.zeros(nranks, np.int64)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    args = (dim, nf_int, p(cf), p(fc), p(fd), p(df), rank, nranks, p(rr), p(rc), p(sc))
    _check(_lib.cr_partition_plan(*args, None, None))
    gh = np.zeros(int(rc.sum()), np.int32)
    sr = np.zeros(int(sc.sum()), np.int32)
    _check(_lib.cr_partition_plan(*args, p(gh), p(sr)))
    return dict(row0=int(rr[0]), row1=int(rr[1]), recv_counts=rc, send_counts=sc, ghosts=gh, send_rows=sr)


def _opts(method, rtol, max_iter, check_every, restart, matrix_free, coarse, mu_inner, inner_rtol, refine_dd):
    m = METHODS[method] if isinstance(method, str) else int(method)
    if m == CR_DC_FGMRES and max_iter == 10**7:
        max_iter = 0
    return SolverOpts(m, restart, rtol, max_iter, check_every, int(matrix_free), int(coarse), float(mu_inner),
                      float(inner_rtol), int(refine_dd), 0)


def cr_solve(hyb: Hybrid, W: torch.Tensor, method: str | int = "pcg", rtol: float = 1e-10,
             max_iter: int = 10**7, check_every: int = 64, restart: int = 50, matrix_free: int = 0, coarse: int = 0,
             mu_inner: float = 0.0, inner_rtol: float = 0.0, refine_dd: int = 0, stream=None,
             raise_on_fail: bool = True) -> dict:
    """Krylov solve of G W = S in place.  Returns the cr_solve_report as a dict.
    method "dc" (CR_DC_FGMRES): outer FGMRES on the coupled system preconditioned by the
    transient hybrid solve (mu_inner, inner_rtol); max_iter then caps the outer iterations.
    refine_dd = 1: double-double residual + iterative refinement (parity mode, PCG methods)."""
    opts = _opts(method, rtol, max_iter, check_every, restart, matrix_free, coarse, mu_inner, inner_rtol, refine_dd)
    rep = SolveReport()
    st = _lib.cr_solve(hyb._h, ctypes.byref(opts), _ptr(W, torch.float64), _stream(stream), ctypes.byref(rep))
    out = rep.as_dict()
    if raise_on_fail:
        _check(st, out)
    out["status_name"] = STATUS.get(st, st)
    return out


SOLVE_PROFILE_KERNELS = ("mf", "update_r", "coarse", "patch", "pdir")


def cr_solve_profile(hyb: Hybrid, method: str | int = "pcg_afw2", nrep: int = 20, matrix_free: int = 1,
                     coarse: int = 0, stream=None) -> dict:
    """Mean device ms per launch of each kernel group of the patch-preconditioned PCG iteration,
    launched on the handle's solver buffers as cr_solve launches them (after a cr_solve with the
    same options): G p + p.q, r update, coarse path, patch solves, direction + solution update."""
    opts = _opts(method, 1e-10, 1, 64, 50, matrix_free, coarse, 0.0, 0.0, 0)
    ms = (ctypes.c_double * 5)()
    _check(_lib.cr_solve_profile(hyb._h, ctypes.byref(opts), int(nrep), ctypes.cast(ms, ctypes.c_void_p),
                                 _stream(stream)))
    return dict(zip(SOLVE_PROFILE_KERNELS, list(ms)))


def cr_recover(hyb: Hybrid, W: torch.Tensor, stream=None):
    """P and U from W.  Returns U [nf_int, d], P [nc], diag [2]
    (global arrays on every rank of a partitioned handle; W holds this rank's rows)."""
    mesh = hyb.mesh
    dev = W.device
    U = torch.empty((mesh.nf_int, mesh.dim), dtype=torch.float64, device=dev)
    P = torch.empty(mesh.nc, dtype=torch.float64, device=dev)
    diag = torch.empty(2, dtype=torch.float64, device=dev)
    _check(_lib.cr_recover(hyb._h, _ptr(W, torch.float64), _ptr(U), _ptr(P), _ptr(diag), _stream(stream)))
    return U, P, diag


class Coupled:
    def __init__(self, handle):
        self._h = handle
        nr, nnz = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.cr_coupled_info(self._h, ctypes.byref(nr), ctypes.byref(nnz)))
        self.n_rows, self.nnz = nr.value, nnz.value

    def export_csr(self, stream=None):
        dev = torch.device("cuda")
        rp = torch.empty(self.n_rows + 1, dtype=torch.int64, device=dev)
        ci = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        v = torch.empty(self.nnz, dtype=torch.float64, device=dev)
        rhs = torch.empty(self.n_rows, dtype=torch.float64, device=dev)
        _check(_lib.cr_coupled_export_csr(self._h, _ptr(rp), _ptr(ci), _ptr(v), _ptr(rhs), _stream(stream)))
        return rp, ci, v, rhs

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.cr_destroy_coupled(self._h)
            self._h = None


def cr_assemble_coupled(mesh: Mesh, prob: Problem, stream=None) -> Coupled:
    """The coupled saddle system eq. (syslin), for parity/export."""
    h = ctypes.c_void_p()
    prm, data = prob.params(), prob.data()
    _check(_lib.cr_assemble_coupled(mesh._h, ctypes.byref(prm), ctypes.byref(data), _stream(stream),
                                    ctypes.byref(h)))
    return Coupled(h)


# ------------------------------------------------------------------ the paper's "hybrid method"
def hybrid_method(coords: torch.Tensor, cells: torch.Tensor, prob: Problem, method: str = "pcg",
                  rtol: float = 1e-10, stream=None, comm: Comm | None = None, **solve_kw) -> dict:
    """(1) mesh, G and S; (2) solve G W = S; (3) recover P and U.
    All tensors must already be on the GPU.  With a multi-rank ``comm`` (one call per rank)
    each rank holds and solves its rows of G; U and P come back whole on every rank."""
    mesh = cr_build_mesh(coords, cells, stream)
    hyb = cr_hybridise(mesh, prob, stream, comm)
    W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=coords.device)
    rep = cr_solve(hyb, W, method, rtol, stream=stream, **solve_kw)
    U, P, diag = cr_recover(hyb, W, stream)
    return dict(mesh=mesh, hybrid=hyb, W=W, U=U, P=P, diag=diag, report=rep)


def time_march(coords: torch.Tensor, cells: torch.Tensor, prob: Problem, nsteps: int, U0: torch.Tensor | None = None,
               method: str = "pcg_afw2", rtol: float = 1e-10, warm_start: bool = True, stream=None,
               **solve_kw) -> dict:
    """Backward Euler for transient Stokes (mu = 1/dt) with the hybrid method: G, its
    patch / coarse preconditioners and matrix-free factors are built once and reused by every
    step; per step only S (cr_transient_rhs + cr_hybrid_set_cell_rhs), the solve
    (warm-started from the previous W) and the recovery run."""
    mesh = cr_build_mesh(coords, cells, stream)
    hyb = cr_hybridise(mesh, prob, stream)
    dev = coords.device
    U = torch.zeros((mesh.nf_int, mesh.dim), dtype=torch.float64, device=dev) if U0 is None else U0
    W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=dev)
    Us, Ps, reps = [], [], []
    for _ in range(nsteps):
        R, g = hyb.transient_rhs(U, stream)
        hyb.set_cell_rhs(R, g, stream)
        if not warm_start:
            W.zero_()
        reps.append(cr_solve(hyb, W, method, rtol, stream=stream, **solve_kw))
        U, P, _ = cr_recover(hyb, W, stream)
        Us.append(U)
        Ps.append(P)
    return dict(mesh=mesh, hybrid=hyb, U=Us, P=Ps, reports=reps)


def cell_face_values(mesh: "Mesh", U: torch.Tensor, bnd: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """[nc, d+1, d]: U on interior faces, bnd (wall values, or 0) on boundary faces."""
    out = torch.empty((mesh.nc, mesh.dim + 1, mesh.dim), dtype=torch.float64, device=U.device)
    _check(_lib.cr_cell_face_values(mesh._h, _ptr(U, torch.float64), _ptr(bnd, torch.float64), _ptr(out),
                                    _stream(stream)))
    return out


def newton_ns(coords: torch.Tensor, cells: torch.Tensor, nu: float, fbar: torch.Tensor, wall: torch.Tensor | None,
              max_newton: int = 30, tol: float = 5e-7, mis_seed: int = 0, method: str = "dc", rtol: float = 1e-10,
              damped: bool = False, lam_min: float = 1.0 / 64, stream=None, **solve_kw) -> dict:
    """Newton's method for steady Navier-Stokes from U^0 = 0, P^0 = 0: each
    step hybridises the linearised problem at (U^k, P^k) (MIS shift), solves it (default: coupled
    FGMRES preconditioned by the transient hybrid solve) and recovers the increments; stops when
    ||lam dU|| <= tol ||U^{k+1}||.  damped: Armijo backtracking lam = 1, 1/2, ... >= lam_min on the
    nonlinear residual ||F|| (cr_coupled_rhs_norm), the rule of oracle.newton_ns(damped=True)."""
    mesh = cr_build_mesh(coords, cells, stream)
    dev = coords.device
    U = torch.zeros((mesh.nf_int, mesh.dim), dtype=torch.float64, device=dev)
    Pk = torch.zeros(mesh.nc, dtype=torch.float64, device=dev)
    hist, reps, lams = [], [], []

    def ns_problem(Uv, Pv):
        return Problem(mu=0.0, nu=nu, fbar=fbar, physics=CR_NS_NEWTON_STEP, shift=CR_SHIFT_MIS, mis_seed=mis_seed,
                       u_iter=cell_face_values(mesh, Uv, wall, stream), p_iter=Pv)

    for _ in range(max_newton):
        prob = ns_problem(U, Pk)
        hyb = cr_hybridise(mesh, prob, stream)
        W = torch.zeros(hyb.n_rows, dtype=torch.float64, device=dev)
        reps.append(cr_solve(hyb, W, method, rtol, stream=stream, **solve_kw))
        dU, dP, _ = cr_recover(hyb, W, stream)
        del hyb
        lam = 1.0
        if damped:
            r0 = coupled_rhs_norm(mesh, prob, stream)
            while lam > lam_min:
                Ut, Pt = U.clone(), Pk.clone()
                newton_update(Ut, dU, Pt, dP, lam, stream)
                if coupled_rhs_norm(mesh, ns_problem(Ut, Pt), stream) < (1.0 - 1e-4 * lam) * r0:
                    break
                lam *= 0.5
        du, un = newton_update(U, dU, Pk, dP, lam, stream)
        rel = du / max(un, 1e-300)
        hist.append(rel)
        lams.append(lam)
        if rel <= tol:
            break
    return dict(mesh=mesh, U=U, P=Pk, history=hist, step_lengths=lams, reports=reps)


def newton_update(U: torch.Tensor, dU: torch.Tensor, P: torch.Tensor | None = None, dP: torch.Tensor | None = None,
                  lam: float = 1.0, stream=None):
    """U += lam dU, P += lam dP in place on the device (cr_newton_update); returns
    (||lam dU||, ||U_new||)."""
    norms = (ctypes.c_double * 2)()
    _check(_lib.cr_newton_update(U.numel(), _ptr(U, torch.float64), _ptr(dU, torch.float64),
                                 0 if P is None else P.numel(), _ptr(P, torch.float64), _ptr(dP, torch.float64),
                                 float(lam), ctypes.cast(norms, ctypes.c_void_p), _stream(stream)))
    return norms[0], norms[1]


def coupled_rhs_norm(mesh: "Mesh", prob: Problem, stream=None) -> float:
    """||[R; g]||_2 of the coupled system (cr_coupled_rhs_norm): for a Navier-Stokes step, the
    nonlinear residual ||F(U^k, P^k)|| (the merit function of the damped Newton line search)."""
    out = ctypes.c_double()
    prm, data = prob.params(), prob.data()
    _check(_lib.cr_coupled_rhs_norm(mesh._h, ctypes.byref(prm), ctypes.byref(data), ctypes.byref(out),
                                    _stream(stream)))
    return out.value


def sparse_direct_solve(rp: torch.Tensor, ci: torch.Tensor, v: torch.Tensor, b: torch.Tensor, method: str = "chol",
                        reorder: int = 3, stream=None) -> torch.Tensor:
    """x = A^{-1} b for a canonical CSR (as exported) by cuSOLVER sparse Cholesky ("chol") or QR ("qr")."""
    x = torch.empty_like(b)
    sing = ctypes.c_int32()
    _check(_lib.cr_sparse_direct_solve(rp.numel() - 1, ci.numel(), _ptr(rp, torch.int64), _ptr(ci, torch.int32),
                                       _ptr(v, torch.float64), _ptr(b, torch.float64), _ptr(x, torch.float64),
                                       0 if method == "chol" else 1, reorder, _stream(stream), ctypes.byref(sing)))
    return x


def coarse_nd_plan(H: int, dim: int, box: int = 0) -> dict:
    """The host nested-dissection plan of the coarse solve (no GPU): per front depth, parent, I and
    B node lists (numpy).  box > 0: the flat two-level plan."""
    import numpy as np
    nf, md, ti, tb = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.cr_coarse_nd_plan(H, dim, box, ctypes.byref(nf), ctypes.byref(md), ctypes.byref(ti),
                                  ctypes.byref(tb), None, None, None, None, None, None))
    n = nf.value
    depth, kids = np.zeros(n, np.int32), np.full(n, -1, np.int32)
    nI, nB = np.zeros(n, np.int32), np.zeros(n, np.int32)
    In, Bn = np.zeros(max(ti.value, 1), np.int32), np.zeros(max(tb.value, 1), np.int32)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(_lib.cr_coarse_nd_plan(H, dim, box, ctypes.byref(nf), ctypes.byref(md), ctypes.byref(ti),
                                  ctypes.byref(tb), p(depth), p(kids), p(nI), p(nB), p(In), p(Bn)))
    oi, ob = np.concatenate([[0], np.cumsum(nI)]), np.concatenate([[0], np.cumsum(nB)])
    return dict(maxdepth=md.value, depth=depth, parent=kids,
                I=[In[oi[f]:oi[f + 1]] for f in range(n)], B=[Bn[ob[f]:ob[f + 1]] for f in range(n)])


def _hptr(a, dtype):
    """Host pointer of a contiguous CPU tensor / numpy array of the given torch dtype."""
    import numpy as np
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise ValueError("host buffers expected (cr_hybrid_method_host copies them to the device)")
        if a.dtype != dtype or not a.is_contiguous():
            raise TypeError(f"expected a contiguous {dtype} CPU tensor")
        return ctypes.c_void_p(a.data_ptr())
    npd = {torch.float64: np.float64, torch.int32: np.int32}[dtype]
    if not isinstance(a, np.ndarray) or a.dtype != npd or not a.flags.c_contiguous:
        raise TypeError(f"expected a C-contiguous {npd.__name__} array")
    return a.ctypes.data_as(ctypes.c_void_p)


def hybrid_method_host(coords, cells, fbar, mu: float, nu: float, method: str = "pcg", rtol: float = 1e-10,
                       stream=None, dirichlet=None, out: tuple | None = None, matrix_free: int = 0, coarse: int = 0,
                       max_iter: int = 10**7, check_every: int = 64, restart: int = 50, mu_inner: float = 0.0,
                       inner_rtol: float = 0.0, refine_dd: int = 0, gauge_cell: int = 0, **prob_kw) -> dict:
    """The hybrid method end to end from HOST buffers through the C ABI (cr_hybrid_method_host):
    host -> device copies, mesh, hybridisation, solve, recovery and device -> host copies of U and
    P, all on `stream` (synchronised before returning).  coords [nv, d] f64, cells [nc, d+1] i32,
    fbar [nc, d] f64 (CPU tensors or numpy; pinned memory makes the copies asynchronous DMA).
    out = (U_h, P_h): caller-owned host buffers with capacity >= d * nf_int and >= nc (default:
    fresh pinned tensors, owned by the caller).  Returns U_host [nf_int, d], P_host [nc] (views of
    out), the solve report and the mesh counts."""
    d = int(coords.shape[1])
    nv, nc = int(coords.shape[0]), int(cells.shape[0])
    if out is None:
        cap = (d + 1) * nc // 2 + (d + 1) * nc % 2   # nf_int <= (d+1) nc / 2
        out = (torch.empty(cap * d, dtype=torch.float64, pin_memory=True),
               torch.empty(nc, dtype=torch.float64, pin_memory=True))
    Uh, Ph = out
    sizes = (ctypes.c_int64 * 2)(Uh.numel(), Ph.numel())
    prob = Problem(mu=mu, nu=nu, fbar=None, gauge_cell=gauge_cell, **prob_kw)
    prm = prob.params()
    opts = _opts(method, rtol, max_iter, check_every, restart, matrix_free, coarse, mu_inner, inner_rtol, refine_dd)
    info, rep = MeshInfo(), SolveReport()
    _check(_lib.cr_hybrid_method_host(d, nv, _hptr(coords, torch.float64), nc, _hptr(cells, torch.int32),
                                      ctypes.byref(prm), _hptr(fbar, torch.float64),
                                      None if dirichlet is None else _hptr(dirichlet, torch.float64),
                                      ctypes.byref(opts), _hptr(Uh, torch.float64), _hptr(Ph, torch.float64),
                                      ctypes.cast(sizes, ctypes.c_void_p), ctypes.byref(info), ctypes.byref(rep),
                                      _stream(stream)), rep.as_dict())
    nU = int(info.n_unknowns)
    return dict(U_host=Uh[:nU].view(-1, d), P_host=Ph[:nc], report=rep.as_dict(), nf_int=int(info.nf_int),
                nf=int(info.nf), n_unknowns=nU)
