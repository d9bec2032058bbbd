// Row partition of G across ranks.  Host code.
//
// Rank q of P owns the contiguous block rows [row0(q), row1(q)) of the lexicographic face
// order, row0(q) = floor(q nf_int / P): the faces are sorted by their smallest vertex and the
// vertices are numbered x-fastest, so a range is (close to) a y-slab in 2D / a z-slab in 3D.
// The stencil of row sigma is every interior face of the two cells of M_sigma,
// so the pattern of G is symmetric: q needs row tau of rank p (a ghost) exactly when tau needs
// a row of q.  Hence each rank derives BOTH directions of its halo from its own rows:
//   ghosts(q)       = stencil columns of q's rows owned by another rank, ascending;
//   send(q -> p)    = q's rows whose stencil touches p's range, ascending,
// and send(q -> p) == the part of ghosts(p) owned by q, in the same order (checked by the
// world-size-2 gloo test).  Nothing here needs a GPU.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace cr {

int64_t part_row0(int64_t nrows, int rank, int nranks) { return (int64_t)((__int128)nrows * rank / nranks); }

int part_owner(int64_t nrows, int nranks, int64_t row) {
    // largest q with row0(q) <= row
    int q = (int)((__int128)row * nranks / nrows);
    while (q + 1 < nranks && part_row0(nrows, q + 1, nranks) <= row) ++q;
    while (q > 0 && part_row0(nrows, q, nranks) > row) --q;
    return q;
}

void plan_partition(int dim, int64_t nf_int, const int32_t *cell_faces, const int32_t *face_cells,
                    const int32_t *face_dof, const int32_t *dof_face, int rank, int nranks, PartPlan &pl) {
    CR_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, CR_ERR_INVALID_ARG, "bad rank / nranks");
    CR_REQUIRE(nf_int >= nranks, CR_ERR_INVALID_ARG, "fewer interior faces than ranks");
    const int NF = dim + 1;
    pl.rank = rank;
    pl.nranks = nranks;
    pl.row0 = part_row0(nf_int, rank, nranks);
    pl.row1 = part_row0(nf_int, rank + 1, nranks);
    std::vector<int64_t> ghosts;
    std::vector<std::vector<int32_t>> send(nranks);
    std::vector<int> touched(nranks, -1);
    for (int64_t r = pl.row0; r < pl.row1; ++r) {
        const int64_t f = dof_face[r];
        for (int side = 0; side < 2; ++side) {
            const int64_t K = face_cells[2 * f + side];
            if (K < 0) continue;
            for (int l = 0; l < NF; ++l) {
                const int64_t c = face_dof[cell_faces[K * NF + l]];
                if (c < 0 || (c >= pl.row0 && c < pl.row1)) continue;
                ghosts.push_back(c);
                const int q = part_owner(nf_int, nranks, c);
                if (touched[q] != (int)(r - pl.row0)) {   // rows are visited in order: one entry per (q, r)
                    touched[q] = (int)(r - pl.row0);
                    send[q].push_back((int32_t)r);
                }
            }
        }
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    pl.ghosts.assign(ghosts.begin(), ghosts.end());
    pl.recv_counts.assign(nranks, 0);
    for (int64_t g : ghosts) pl.recv_counts[part_owner(nf_int, nranks, g)]++;
    pl.send_counts.assign(nranks, 0);
    pl.send_rows.clear();
    for (int q = 0; q < nranks; ++q) {
        pl.send_counts[q] = (int64_t)send[q].size();
        pl.send_rows.insert(pl.send_rows.end(), send[q].begin(), send[q].end());
    }
}

// Partition of a hybrid handle for comm's rank: host plan from the mesh connectivity, then
// the device maps (global -> local numbering, send rows) and halo tables.
void setup_part(cr_hybrid_s *h, const cr_mesh_s *m, cr_comm_s *comm, cudaStream_t s) {
    const int NF = m->dim + 1;
    std::vector<int32_t> cf(m->nc * NF), fc(m->nf * 2), fd(m->nf), df(m->nf_int);
    CR_CUDA(cudaMemcpyAsync(cf.data(), m->cell_faces.get(), cf.size() * 4, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(fc.data(), m->face_cells.get(), fc.size() * 4, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(fd.data(), m->face_dof.get(), fd.size() * 4, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(df.data(), m->dof_face.get(), df.size() * 4, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    PartPlan pl;
    plan_partition(m->dim, m->nf_int, cf.data(), fc.data(), fd.data(), df.data(), comm->rank, comm->nranks, pl);
    Part &P = h->part;
    P.on = true;
    P.rank = comm->rank;
    P.nranks = comm->nranks;
    P.row0 = pl.row0;
    P.row1 = pl.row1;
    P.nloc = pl.row1 - pl.row0;
    P.nghost = (int64_t)pl.ghosts.size();
    P.nglobal = m->nf_int;
    P.rcount = pl.recv_counts;
    P.scount = pl.send_counts;
    P.roff.assign(P.nranks, 0);
    P.soff.assign(P.nranks, 0);
    for (int q = 1; q < P.nranks; ++q) {
        P.roff[q] = P.roff[q - 1] + P.rcount[q - 1];
        P.soff[q] = P.soff[q - 1] + P.scount[q - 1];
    }
    P.all_row0.resize(P.nranks + 1);
    for (int q = 0; q <= P.nranks; ++q) P.all_row0[q] = part_row0(m->nf_int, q, P.nranks);
    std::vector<int32_t> g2l(m->nf_int, -1), l2g(P.nloc + P.nghost);
    for (int64_t i = 0; i < P.nloc; ++i) {
        g2l[P.row0 + i] = (int32_t)i;
        l2g[i] = (int32_t)(P.row0 + i);
    }
    for (int64_t j = 0; j < P.nghost; ++j) {
        g2l[pl.ghosts[j]] = (int32_t)(P.nloc + j);
        l2g[P.nloc + j] = (int32_t)pl.ghosts[j];
    }
    P.nsend = (int64_t)pl.send_rows.size();
    std::vector<int32_t> sr(P.nsend);
    for (int64_t k = 0; k < P.nsend; ++k) sr[k] = (int32_t)(pl.send_rows[k] - P.row0);
    P.g2l.alloc(g2l.size(), s);
    P.l2g.alloc(l2g.size(), s);
    P.send_rows.alloc(sr.size() > 0 ? sr.size() : 1, s);
    P.sendbuf.alloc((P.nsend > 0 ? P.nsend : 1) * m->dim, s);
    CR_CUDA(cudaMemcpyAsync(P.g2l.get(), g2l.data(), g2l.size() * 4, cudaMemcpyHostToDevice, s));
    CR_CUDA(cudaMemcpyAsync(P.l2g.get(), l2g.data(), l2g.size() * 4, cudaMemcpyHostToDevice, s));
    if (P.nsend) CR_CUDA(cudaMemcpyAsync(P.send_rows.get(), sr.data(), sr.size() * 4, cudaMemcpyHostToDevice, s));
    CR_CUDA(cudaStreamSynchronize(s));   // host vectors go out of scope
}

}  // namespace cr

extern "C" cr_status cr_partition_plan(int32_t dim, int64_t nf_int, const int32_t *cell_faces_h,
                                       const int32_t *face_cells_h, const int32_t *face_dof_h,
                                       const int32_t *dof_face_h, int32_t rank, int32_t nranks,
                                       int64_t *row_range, int64_t *recv_counts, int64_t *send_counts,
                                       int32_t *ghosts, int32_t *send_rows) {
    try {
        CR_REQUIRE(dim == 2 || dim == 3, CR_ERR_INVALID_ARG, "dim must be 2 or 3");
        CR_REQUIRE(cell_faces_h && face_cells_h && face_dof_h && dof_face_h && row_range && recv_counts && send_counts,
                   CR_ERR_INVALID_ARG, "null argument");
        cr::PartPlan pl;
        cr::plan_partition(dim, nf_int, cell_faces_h, face_cells_h, face_dof_h, dof_face_h, rank, nranks, pl);
        row_range[0] = pl.row0;
        row_range[1] = pl.row1;
        for (int q = 0; q < nranks; ++q) {
            recv_counts[q] = pl.recv_counts[q];
            send_counts[q] = pl.send_counts[q];
        }
        if (ghosts)
            for (size_t i = 0; i < pl.ghosts.size(); ++i) ghosts[i] = (int32_t)pl.ghosts[i];
        if (send_rows)
            for (size_t i = 0; i < pl.send_rows.size(); ++i) send_rows[i] = pl.send_rows[i];
        return CR_OK;
    } catch (const cr::Error &e) {
        cr::set_last_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        cr::set_last_error(e.what());
        return CR_ERR_INVALID_ARG;
    }
}
