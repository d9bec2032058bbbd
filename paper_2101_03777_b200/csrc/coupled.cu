// cr_assemble_coupled: the coupled saddle-point system eq. (syslin) on the device
// (PAPER.md P:L253-306), exported as a canonical CSR for parity checks.
//   A = sum_K H_K A_K H_K^t   (full d x d blocks on the face stencil, as G)
//   D = sum_{K != K0} F_K D_K^t H_K^t,  D_K = -a
//   R = sum_K H_K R_K  (+ Dirichlet fold / NS increment form), g
// Rows: d*nf_int momentum rows (face-major, component-minor), then nc-1 divergence rows
// (K != K0 in increasing K).  Columns sorted; explicit zeros of the d x d blocks kept.
#include <cub/cub.cuh>

#include "local.cuh"
#include "spmv.cuh"

namespace cr {

__device__ __forceinline__ int64_t pidx(int64_t K, int k0) { return K < k0 ? K : K - 1; }

// rounded A_K row (l, i) -> block (l, q) entries; returns rounded R_K(l, i), g
template <int D>
__device__ __forceinline__ void coupled_cell_row(const Cell<D> &c, const ProbView &p, int l,
                                                 double (&Arow)[D + 1][D][D], double (&Rl)[D], double &gK) {
    constexpr int NF = D + 1, N = NF * D;
    if (!p.is_ns) {
        dd R[NF][D], g;
        stokes_rhs<D>(c, p, R, g);
        for (int q = 0; q < NF; ++q) {
            double sv = (c.dof[q] >= 0) ? dd_round(S_entry<D>(c, p.mu, p.nu, l, q)) : 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) Arow[q][i][j] = (i == j) ? sv : 0.0;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) Rl[i] = dd_round(R[l][i]);
        gK = dd_round(g);
    } else {
        dd A[N][N], R[N], g;
        ns_local_system<D>(c, p, A, R, g);
        for (int q = 0; q < NF; ++q)
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    Arow[q][i][j] = (c.dof[q] >= 0) ? dd_round(A[l * D + i][q * D + j]) : 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) Rl[i] = dd_round(R[l * D + i]);
        gK = dd_round(g);
    }
}

// counts per block row (momentum) and per cell (divergence rows)
template <int D>
__global__ void k_coupled_counts(MeshView mv, const int32_t *dof_face, int64_t nrows, int64_t nc, int k0,
                                 int64_t *cnt_rows, int64_t *cnt_cells) {
    constexpr int NF = D + 1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int f = dof_face[r];
        int nb = 1, np = 0;
        for (int side = 0; side < 2; ++side) {
            const int64_t K = mv.face_cells[2 * (int64_t)f + side];
            if (K != k0) ++np;
            for (int l = 0; l < NF; ++l) {
                int g = mv.cell_faces[K * NF + l];
                if (g != f && mv.face_dof[g] >= 0) ++nb;
            }
        }
        cnt_rows[r] = (int64_t)D * (nb * D + np);   // D scalar rows per block row
    }
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        if (K == k0) { cnt_cells[K] = 0; continue; }
        int s = 0;
        for (int l = 0; l < NF; ++l) if (mv.face_dof[mv.cell_faces[K * NF + l]] >= 0) ++s;
        cnt_cells[K] = (int64_t)D * s;
    }
}

template <int D>
__global__ void __launch_bounds__(64) k_coupled_rows(MeshView mv, ProbView p, const int32_t *dof_face, int64_t nrows,
                                                     int64_t nU, const int64_t *base, int64_t *row_ptr, int32_t *cols,
                                                     double *vals, double *rhs) {
    constexpr int NF = D + 1, W = 2 * D + 1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int f = dof_face[r];
        int bc[W];
        double bv[W][D][D];
        int nb = 1;
        bc[0] = (int)r;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) bv[0][i][j] = 0.0;
        double Rsum[D] = {};
        int64_t pc[2];
        double pv[2][D];
        int np = 0;
        for (int side = 0; side < 2; ++side) {
            const int64_t K = mv.face_cells[2 * (int64_t)f + side];
            Cell<D> c;
            load_cell<D>(mv, K, c);
            int l = 0;
            for (int q = 0; q < NF; ++q) if (c.face[q] == f) l = q;
            double Arow[NF][D][D], Rl[D], gK;
            coupled_cell_row<D>(c, p, l, Arow, Rl, gK);
#pragma unroll
            for (int i = 0; i < D; ++i) Rsum[i] += Rl[i];
            for (int q = 0; q < NF; ++q) {
                if (c.dof[q] < 0) continue;
                if (q == l) {
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int j = 0; j < D; ++j) bv[0][i][j] += Arow[q][i][j];
                } else {
                    bc[nb] = c.dof[q];
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int j = 0; j < D; ++j) bv[nb][i][j] = Arow[q][i][j];
                    ++nb;
                }
            }
            if (K != p.k0) {
                pc[np] = nU + pidx(K, p.k0);
#pragma unroll
                for (int i = 0; i < D; ++i) pv[np][i] = -c.a[l][i];    // D^t entry = D_K(l, i) = -a
                ++np;
            }
        }
        // sort blocks by column
        int ord[W];
        for (int k = 0; k < nb; ++k) ord[k] = k;
        for (int a = 1; a < nb; ++a)
            for (int b = a; b > 0 && bc[ord[b - 1]] > bc[ord[b]]; --b) { int t = ord[b]; ord[b] = ord[b - 1]; ord[b - 1] = t; }
        if (np == 2 && pc[0] > pc[1]) {
            int64_t t = pc[0]; pc[0] = pc[1]; pc[1] = t;
            for (int i = 0; i < D; ++i) { double u = pv[0][i]; pv[0][i] = pv[1][i]; pv[1][i] = u; }
        }
        const int64_t per = (int64_t)nb * D + np;
        for (int i = 0; i < D; ++i) {
            int64_t pos = base[r] + i * per;
            row_ptr[r * D + i] = pos;
            for (int k = 0; k < nb; ++k)
                for (int j = 0; j < D; ++j) {
                    cols[pos] = bc[ord[k]] * D + j;
                    vals[pos] = bv[ord[k]][i][j];
                    ++pos;
                }
            for (int k = 0; k < np; ++k) {
                cols[pos] = (int32_t)pc[k];
                vals[pos] = pv[k][i];
                ++pos;
            }
            rhs[r * D + i] = Rsum[i];
        }
    }
}

template <int D>
__global__ void k_coupled_div_rows(MeshView mv, ProbView p, int64_t nc, int64_t nU, const int64_t *base_cells,
                                   int64_t *row_ptr, int32_t *cols, double *vals, double *rhs) {
    constexpr int NF = D + 1;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        if (K == p.k0) continue;
        Cell<D> c;
        load_cell<D>(mv, K, c);
        // interior faces sorted by dof
        int ord[NF];
        for (int q = 0; q < c.s; ++q) ord[q] = c.map[q];
        for (int a = 1; a < c.s; ++a)
            for (int b = a; b > 0 && c.dof[ord[b - 1]] > c.dof[ord[b]]; --b) { int t = ord[b]; ord[b] = ord[b - 1]; ord[b - 1] = t; }
        const int64_t row = nU + pidx(K, p.k0);
        int64_t pos = base_cells[K];
        row_ptr[row] = pos;
        for (int q = 0; q < c.s; ++q)
            for (int i = 0; i < D; ++i) {
                cols[pos] = c.dof[ord[q]] * D + i;
                vals[pos] = -c.a[ord[q]][i];
                ++pos;
            }
        double Rl[D], gK;
        double Arow[NF][D][D];
        coupled_cell_row<D>(c, p, c.map[0], Arow, Rl, gK);
        rhs[row] = gK;
    }
}

template <int D>
static void assemble_coupled_t(cr_coupled_s *c, const cr_mesh_s *m, const ProbView &p, cudaStream_t s) {
    const int64_t nrows = m->nf_int, nc = m->nc, nU = D * nrows;
    MeshView mv = mesh_view(m);
    DevBuf<int64_t> cnt_rows, cnt_cells, base_rows, base_cells;
    cnt_rows.alloc(nrows, s); cnt_cells.alloc(nc, s); base_rows.alloc(nrows, s); base_cells.alloc(nc, s);
    const int T = 256;
    k_coupled_counts<D><<<grid_for(std::max(nrows, nc), T), T, 0, s>>>(mv, m->dof_face.get(), nrows, nc, p.k0,
                                                                        cnt_rows.get(), cnt_cells.get());
    CR_CHECK_LAUNCH();
    size_t tb = 0, tb2 = 0;
    CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt_rows.get(), base_rows.get(), (int)nrows, s));
    CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt_cells.get(), base_cells.get(), (int)nc, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(std::max(tb, tb2), s);
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt_rows.get(), base_rows.get(), (int)nrows, s));
    int64_t last_base = 0, last_cnt = 0;
    CR_CUDA(cudaMemcpyAsync(&last_base, base_rows.get() + nrows - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&last_cnt, cnt_rows.get() + nrows - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    const int64_t nnzA = last_base + last_cnt;
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb2, cnt_cells.get(), base_cells.get(), (int)nc, s));
    int64_t lb2 = 0, lc2 = 0;
    CR_CUDA(cudaMemcpyAsync(&lb2, base_cells.get() + nc - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&lc2, cnt_cells.get() + nc - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    const int64_t nnzD = lb2 + lc2;
    c->n_rows = nU + nc - 1;
    c->nnz = nnzA + nnzD;
    c->row_ptr.alloc(c->n_rows + 1, s);
    c->cols.alloc(c->nnz, s);
    c->vals.alloc(c->nnz, s);
    c->rhs.alloc(c->n_rows, s);
    // shift the divergence-row bases by nnzA
    DevBuf<int64_t> bc2;
    bc2.alloc(nc, s);
    {
        std::vector<int64_t> hb(nc);
        CR_CUDA(cudaMemcpyAsync(hb.data(), base_cells.get(), nc * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        for (auto &v : hb) v += nnzA;
        CR_CUDA(cudaMemcpyAsync(bc2.get(), hb.data(), nc * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaStreamSynchronize(s));
    }
    k_coupled_rows<D><<<grid_for(nrows, 64, 16), 64, 0, s>>>(mv, p, m->dof_face.get(), nrows, nU, base_rows.get(),
                                                              c->row_ptr.get(), c->cols.get(), c->vals.get(), c->rhs.get());
    CR_CHECK_LAUNCH();
    k_coupled_div_rows<D><<<grid_for(nc, 64, 16), 64, 0, s>>>(mv, p, nc, nU, bc2.get(), c->row_ptr.get(), c->cols.get(),
                                                               c->vals.get(), c->rhs.get());
    CR_CHECK_LAUNCH();
    int64_t nnz = c->nnz;
    CR_CUDA(cudaMemcpyAsync(c->row_ptr.get() + c->n_rows, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    CR_CUDA(cudaStreamSynchronize(s));
}

void assemble_coupled(cr_coupled_s *c, const cr_mesh_s *m, const cr_params &prm, const cr_data &data, cudaStream_t s) {
    CR_REQUIRE(prm.gauge_cell >= 0 && prm.gauge_cell < m->nc, CR_ERR_INVALID_ARG, "gauge cell out of range");
    CR_REQUIRE(m->nf_int > 0, CR_ERR_NO_INTERIOR_FACE, "mesh has no interior face");
    // reuse the hybrid's data-copy helper through a scratch hybrid handle
    cr_hybrid_s tmp;
    tmp.mesh = m;
    tmp.prm = prm;
    tmp.prm.shift = CR_SHIFT_NONE;
    tmp.is_ns = prm.physics == CR_NS_NEWTON_STEP;
    CR_REQUIRE(!tmp.is_ns || data.u_iter_d, CR_ERR_INVALID_ARG, "NS step needs u_iter_d");
    copy_problem_data(&tmp, m, data, s);
    ProbView p = prob_view(&tmp);
    if (m->dim == 2) assemble_coupled_t<2>(c, m, p, s);
    else assemble_coupled_t<3>(c, m, p, s);
}

}  // namespace cr
