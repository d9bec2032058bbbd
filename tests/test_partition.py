"""Multi-GPU host logic on the CPU.

* the host partition planner of libcr (cr_partition_plan) against a brute-force reading of
  the stencil of the oracle's G: ranges tile the rows, ghosts are exactly the
  off-range stencil columns, send lists are what the peers' rows reference;
* world_size-2 `gloo` run: each process plans its own rank, the two halves of every halo
  agree, and a distributed Jacobi PCG that exchanges ghosts with send/recv and sums its dot
  products with all_reduce (the same sequence the NCCL path runs on the GPU) reproduces the
  single-process solution of the oracle's G.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cr_inputs as ci
import oracle as O


def _binding():
    # the binding loads libcr.so (a CPU box can call its host-only functions)
    import paper_2101_03777_b200 as P
    return P


def _case(n=6, dim=2):
    coords, cells = ci.square_mesh(n, 0.2, 3) if dim == 2 else ci.cube_mesh(n)
    m = O.build_mesh(coords, cells)
    _, _, f = (ci.manufactured_2d if dim == 2 else ci.manufactured_3d)(1.0, 1.0)
    data = O.Data(fbar=ci.cell_average(f, coords, cells))
    h = O.hybridise(m, O.Params(mu=1.0, nu=1.0), data)
    return m, h


def _block_pattern(m, G):
    d = m.dim
    Gb = sp.csr_matrix((np.ones(G.nnz), G.indices // d, G.indptr[::d]), shape=(m.nf_int, m.nf_int))
    Gb.sum_duplicates()
    return Gb


@pytest.mark.parametrize("dim,n,nranks", [(2, 6, 1), (2, 6, 2), (2, 7, 3), (3, 2, 4)])
def test_plan_matches_stencil(dim, n, nranks):
    P = _binding()
    m, h = _case(n, dim)
    Gb = _block_pattern(m, h["G"])
    plans = [P.partition_plan(dim, m.cell_faces, m.face_cells, m.face_dof, q, nranks) for q in range(nranks)]
    # ranges tile [0, nf_int) in order, balanced to one row
    assert plans[0]["row0"] == 0 and plans[-1]["row1"] == m.nf_int
    for a, b in zip(plans, plans[1:]):
        assert a["row1"] == b["row0"]
    sizes = [p["row1"] - p["row0"] for p in plans]
    assert max(sizes) - min(sizes) <= 1
    owner = np.concatenate([np.full(s, q) for q, s in enumerate(sizes)])
    for q, p in enumerate(plans):
        rows = np.arange(p["row0"], p["row1"])
        cols = np.unique(Gb[rows].indices)
        ghosts = cols[(cols < p["row0"]) | (cols >= p["row1"])]
        assert np.array_equal(p["ghosts"], ghosts)
        assert np.array_equal(p["recv_counts"], np.bincount(owner[ghosts], minlength=nranks))
        # send list to peer r = my rows that r's rows reference, ascending, grouped by r
        off = 0
        for r in range(nranks):
            cnt = int(p["send_counts"][r])
            got = p["send_rows"][off:off + cnt]
            off += cnt
            if r == q:
                assert cnt == 0
                continue
            rr = np.arange(plans[r]["row0"], plans[r]["row1"])
            need = np.unique(Gb[rr].indices)
            need = need[(need >= p["row0"]) & (need < p["row1"])]
            assert np.array_equal(got, need)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        P = _binding()
        m, h = _case(8, 2)
        G, S, d = h["G"].tocsr(), h["S"], m.dim
        pl = P.partition_plan(d, m.cell_faces, m.face_cells, m.face_dof, rank, world)
        r0, r1 = pl["row0"], pl["row1"]
        nloc, ghosts = r1 - r0, pl["ghosts"].astype(np.int64)
        # 1. both halves of the halo agree: my send list to the peer == the peer's ghosts from me
        peer = 1 - rank
        mine = torch.from_numpy(pl["send_rows"][pl["send_counts"][:peer].sum():][:pl["send_counts"][peer]].astype(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(ghosts)], dtype=torch.int64))
        theirs = torch.zeros(int(sizes[peer]), dtype=torch.int64)
        reqs = [dist.isend(torch.from_numpy(ghosts), peer), dist.irecv(theirs, peer)]
        for rq in reqs:
            rq.wait()
        theirs = theirs.numpy()
        lo, hi = r0, r1
        assert np.array_equal(mine.numpy(), theirs[(theirs >= lo) & (theirs < hi)])
        # 2. distributed Jacobi PCG with local numbering [owned | ghosts]
        gidx = np.concatenate([np.arange(r0, r1), ghosts])
        sc = lambda rows: (rows[:, None] * d + np.arange(d)).ravel()
        Gl = G[sc(np.arange(r0, r1))][:, sc(gidx)].tocsr()
        b = S[sc(np.arange(r0, r1))]
        dinv = 1.0 / G.diagonal()[sc(np.arange(r0, r1))]
        send_loc = mine.numpy() - r0
        nrecv = len(ghosts)

        def halo(v):   # v: [(nloc + nghost) d]
            sbuf = torch.from_numpy(v.reshape(-1, d)[send_loc].ravel().copy())
            rbuf = torch.zeros(nrecv * d, dtype=torch.float64)
            rq = [dist.isend(sbuf, peer), dist.irecv(rbuf, peer)]
            for x in rq:
                x.wait()
            v[nloc * d:] = rbuf.numpy()

        def dot(a, b_):
            t = torch.tensor([float(a @ b_)], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t)

        x = np.zeros((nloc + nrecv) * d)
        r = b.copy()
        z = dinv * r
        p = np.zeros_like(x)
        p[:nloc * d] = z
        rho = dot(r, z)
        bn = np.sqrt(dot(b, b))
        it = 0
        while it < 20000:
            halo(p)
            qv = Gl @ p
            alpha = rho / dot(p[:nloc * d], qv)
            x[:nloc * d] += alpha * p[:nloc * d]
            r -= alpha * qv
            it += 1
            if np.sqrt(dot(r, r)) <= 1e-11 * bn:
                break
            z = dinv * r
            rn = dot(r, z)
            p[:nloc * d] = z + (rn / rho) * p[:nloc * d]
            rho = rn
        locs = torch.from_numpy(x[:nloc * d].copy())
        lens = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(lens, torch.tensor([nloc * d], dtype=torch.int64))
        parts = [torch.zeros(int(l), dtype=torch.float64) for l in lens]
        dist.all_gather(parts, locs)
        W = torch.cat(parts).numpy()
        if rank == 0:
            Wref, rep = O.pcg(G, S, rtol=1e-11)
            q.put(("ok", float(np.linalg.norm(W - Wref) / np.linalg.norm(Wref)), it, rep["iterations"]))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(("err", traceback.format_exc(), 0, 0))


def test_gloo_two_ranks_halo_and_distributed_pcg():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    status, err, it, it_ref = q.get(timeout=10)
    assert status == "ok", err
    assert err <= 1e-8
    assert abs(it - it_ref) <= 2      # same algorithm, only the dot-product summation order differs
