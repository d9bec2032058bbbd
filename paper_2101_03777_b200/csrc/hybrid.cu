// cr_hybridise: shift E_K (K5), pattern + local elimination + scatter of G and S
// (K6-K8 fused, face-centric), preconditioner diagonals, canonical CSR export, SpMV.
//
// Face-centric assembly: one thread per interior face sigma = one block row of G.  For each
// of the two cells K of M_sigma it recomputes the cell's elimination (double-double) and
// emits row sigma of G_K: the off-diagonal blocks (sigma, sigma') of a cell have exactly one
// contributor (two distinct faces share at most one simplex), the diagonal block and S_sigma
// have two (K and L) and are summed in registers.  So G is written once, coalesced, with no
// atomics and no staging; each cell is recomputed d+1 times (cheap ALU vs. HBM).
#include <cub/cub.cuh>

#include "local.cuh"
#include "spmv.cuh"

namespace cr {

// ------------------------------------------------------------------ K5: greedy-equivalent MIS
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

enum : uint8_t { MIS_UNDECIDED = 0, MIS_IN = 1, MIS_OUT = 2 };

// A cell joins M1 once every lower-(priority, K) neighbour is OUT; it leaves once any
// neighbour is IN.  Every decision is final and agrees with the sequential greedy MIS in
// ascending (priority, K) order, so in-place updates are race-benign and deterministic.
template <int D>
__global__ void k_mis_round(MeshView mv, int64_t nc, uint64_t seed, volatile uint8_t *state, unsigned *undecided) {
    unsigned cnt = 0;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        if (state[K] != MIS_UNDECIDED) continue;
        const uint64_t pK = splitmix64(seed ^ (uint64_t)K);
        bool out = false, can_in = true;
#pragma unroll
        for (int l = 0; l < D + 1; ++l) {
            int f = mv.cell_faces[K * (D + 1) + l];
            int32_t c0 = mv.face_cells[2 * (int64_t)f], c1 = mv.face_cells[2 * (int64_t)f + 1];
            if (c1 < 0) continue;
            int64_t L = (c0 == (int32_t)K) ? c1 : c0;
            uint8_t sL = state[L];
            if (sL == MIS_IN) { out = true; break; }
            uint64_t pL = splitmix64(seed ^ (uint64_t)L);
            bool lower = (pL < pK) || (pL == pK && L < K);
            if (lower && sL != MIS_OUT) can_in = false;
        }
        if (out) state[K] = MIS_OUT;
        else if (can_in) state[K] = MIS_IN;
        else ++cnt;
    }
    cnt = (unsigned)warp_sum((double)cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(undecided, cnt);
}

// numpy's pairwise sum order for a short contiguous row (the oracle's np.abs(A).sum(axis=2))
template <int N>
__device__ __forceinline__ double np_rowsum(const double (&a)[N]) {
    if constexpr (N < 8) {
        double r = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) r = __dadd_rn(r, a[i]);
        return r;
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        for (; i < N - (N % 8); i += 8)
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < N; ++i) res = __dadd_rn(res, a[i]);
        return res;
    }
}

// lambda_K = factor * max_row sum_col |A_K| (interior-restricted, fp64-rounded entries)
template <int D>
__global__ void k_lambda(MeshView mv, ProbView p, int64_t nc, double factor, double *lam, int *err) {
    constexpr int NF = D + 1, N = NF * D;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        Cell<D> c;
        load_cell<D>(mv, K, c);
        double best = 0.0;
        if (!p.is_ns) {
            for (int l = 0; l < NF; ++l) {
                if (c.dof[l] < 0) continue;
                double row[N];
#pragma unroll
                for (int q = 0; q < N; ++q) row[q] = 0.0;
                for (int t = 0; t < NF; ++t)
                    if (c.dof[t] >= 0) row[t * D] = fabs(dd_round(S_entry<D>(c, p.mu, p.nu, l, t)));
                // every component row of I (x) S has the same entries (shifted by i): same sum
                best = fmax(best, np_rowsum<N>(row));
            }
        } else {
            dd A[N][N], R[N], g;
            ns_local_system<D>(c, p, A, R, g);
            for (int r = 0; r < N; ++r) {
                if (c.dof[r / D] < 0) continue;
                double row[N];
#pragma unroll
                for (int q = 0; q < N; ++q) row[q] = (c.dof[q / D] >= 0) ? fabs(dd_round(A[r][q])) : 0.0;
                best = fmax(best, np_rowsum<N>(row));
            }
        }
        lam[K] = __dmul_rn(factor, best);
    }
}

template <int D>
__global__ void k_shift(MeshView mv, int64_t nc, const uint8_t *state, const double *lam, double *E, uint8_t *inM1) {
    constexpr int NF = D + 1;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        bool in = state[K] == MIS_IN;
        inM1[K] = in ? 1 : 0;
        for (int l = 0; l < NF; ++l) {
            int f = mv.cell_faces[K * NF + l];
            int32_t c0 = mv.face_cells[2 * (int64_t)f], c1 = mv.face_cells[2 * (int64_t)f + 1];
            double e = 0.0;
            if (c1 >= 0) {
                if (in) e = -lam[K];
                else {
                    int64_t L = (c0 == (int32_t)K) ? c1 : c0;
                    if (state[L] == MIS_IN) e = lam[L];
                }
            }
            E[K * NF + l] = e;
        }
    }
}

// ------------------------------------------------------------------ K6-K8: face-centric assembly
struct AsmOut {
    int32_t *cols;
    double *vals;
    uint8_t *rowlen;
    double *S, *dinv, *absdinv, *bdinv;
    unsigned long long *nblocks;
    int *err;
};

template <int D>
__device__ __forceinline__ void write_block(const AsmOut &o, int64_t r, int slot, int32_t col, const double (&b)[D][D]) {
    constexpr int W = 2 * D + 1, B2 = D * D;
    const int64_t slice = r >> 5;
    const int lane = (int)(r & 31);
    o.cols[slice * (W * 32) + slot * 32 + lane] = col;
    double *vp = o.vals + slice * ((int64_t)W * B2 * 32) + lane;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) vp[(slot * B2 + i * D + j) * 32] = b[i][j];
}

template <int D>
__device__ __forceinline__ void finish_row(const AsmOut &o, int64_t r, int slot, double (&diag)[D][D], const double (&Sr)[D]) {
    constexpr int W = 2 * D + 1;
    double z[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) z[i][j] = 0.0;
    write_block<D>(o, r, 0, (int32_t)r, diag);
    o.rowlen[r] = (uint8_t)slot;
    for (int k = slot; k < W; ++k) write_block<D>(o, r, k, (int32_t)r, z);
#pragma unroll
    for (int i = 0; i < D; ++i) {
        o.S[r * D + i] = Sr[i];
        o.dinv[r * D + i] = 1.0 / diag[i][i];
        o.absdinv[r * D + i] = 1.0 / fabs(diag[i][i]);
    }
    // inverse of the diagonal block (face-block Jacobi), Gauss-Jordan in fp64
    double Mx[D][2 * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) { Mx[i][j] = diag[i][j]; Mx[i][D + j] = (i == j) ? 1.0 : 0.0; }
#pragma unroll
    for (int k = 0; k < D; ++k) {
        int pv = k;
        for (int i = k + 1; i < D; ++i) if (fabs(Mx[i][k]) > fabs(Mx[pv][k])) pv = i;
        if (pv != k)
#pragma unroll
            for (int j = 0; j < 2 * D; ++j) { double t = Mx[k][j]; Mx[k][j] = Mx[pv][j]; Mx[pv][j] = t; }
        double inv = 1.0 / Mx[k][k];
#pragma unroll
        for (int j = 0; j < 2 * D; ++j) Mx[k][j] *= inv;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            if (i == k) continue;
            double f = Mx[i][k];
#pragma unroll
            for (int j = 0; j < 2 * D; ++j) Mx[i][j] -= f * Mx[k][j];
        }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) o.bdinv[(r * D + i) * D + j] = Mx[i][D + j];
}

template <int D>
__global__ void __launch_bounds__(128) k_assemble_stokes(MeshView mv, ProbView p, const int32_t *dof_face,
                                                         int64_t nrows, int64_t row0, const int32_t *g2l, AsmOut o,
                                                         int sonly = 0) {
    constexpr int NF = D + 1;
    unsigned long long nb_local = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int f = dof_face[row0 + r];
        double diag[D][D], Sr[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            Sr[i] = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) diag[i][j] = 0.0;
        }
        int slot = 1;
        for (int side = 0; side < 2; ++side) {
            const int64_t K = mv.face_cells[2 * (int64_t)f + side];
            Cell<D> c;
            load_cell<D>(mv, K, c);
            StokesElim<D> e;
            stokes_eliminate<D>(c, p, e);
            if (e.status != DE_OK) { atomicCAS(o.err, DE_OK, e.status); continue; }
            int pr = 0;
            for (int q = 0; q < c.s; ++q) if (c.face[c.map[q]] == f) pr = q;
            const int lr = c.map[pr];
            const bool k0 = (K == p.k0);
            // row pr of Shat^{-1}
            dd srow[NF];
            for (int q = 0; q < c.s; ++q) srow[q] = dd_of(q == pr ? 1.0 : 0.0);
            ldl_solve<D>(e, c.s, srow);
            // S_K row: C_l (t_i - w_i[p] (sum_i w_i^t R_i - g)/B)
            dd R[NF][D], g;
            stokes_rhs<D>(c, p, R, g);
            dd wR = dd_of(0.0);
            dd ti[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                ti[i] = dd_of(0.0);
                for (int q = 0; q < c.s; ++q) {
                    wR = wR + e.w[i][q] * R[c.map[q]][i];
                    ti[i] = ti[i] + srow[q] * R[c.map[q]][i];
                }
            }
            dd coef = k0 ? dd_of(0.0) : (wR - g) / e.B;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                dd v = k0 ? ti[i] : ti[i] - e.w[i][pr] * coef;
                Sr[i] += dd_round(v * c.C[lr]);
            }
            // G row blocks
            dd wpB[D];
#pragma unroll
            for (int i = 0; i < D; ++i) wpB[i] = k0 ? dd_of(0.0) : e.w[i][pr] / e.B;
            for (int q = 0; q < c.s; ++q) {
                const int lq = c.map[q];
                const double cc = c.C[lr] * c.C[lq];
                double b[D][D];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        dd v = (i == j) ? srow[q] : dd_of(0.0);
                        if (!k0) v = v - wpB[i] * e.w[j][q];
                        b[i][j] = dd_round(v * cc);
                    }
                if (q == pr) {
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int j = 0; j < D; ++j) diag[i][j] += b[i][j];
                } else if (!sonly) {
                    write_block<D>(o, r, slot++, g2l ? g2l[c.dof[lq]] : (int32_t)c.dof[lq], b);
                }
            }
        }
        if (sonly) {
#pragma unroll
            for (int i = 0; i < D; ++i) o.S[r * D + i] = Sr[i];
            continue;
        }
        finish_row<D>(o, r, slot, diag, Sr);
        nb_local += (unsigned long long)slot;
    }
    nb_local = (unsigned long long)warp_sum((double)nb_local);
    if ((threadIdx.x & 31) == 0) atomicAdd(o.nblocks, nb_local);
}

template <int D>
__global__ void __launch_bounds__(64) k_assemble_ns(MeshView mv, ProbView p, const int32_t *dof_face,
                                                         int64_t nrows, int64_t row0, const int32_t *g2l, AsmOut o) {
    unsigned long long nb_local = 0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int f = dof_face[row0 + r];
        double diag[D][D], Sr[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            Sr[i] = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) diag[i][j] = 0.0;
        }
        int slot = 1;
        for (int side = 0; side < 2; ++side) {
            const int64_t K = mv.face_cells[2 * (int64_t)f + side];
            Cell<D> c;
            load_cell<D>(mv, K, c);
            NSElim<D> e;
            ns_eliminate<D>(c, p, e);
            if (e.status != DE_OK) { atomicCAS(o.err, DE_OK, e.status); continue; }
            const bool k0 = (K == p.k0);
            int pr = 0;
            for (int q = 0; q < c.s; ++q) if (c.face[c.map[q]] == f) pr = q;
            const int lr = c.map[pr];
            dd vR = dd_of(0.0);
            for (int q = 0; q < e.m; ++q) vR = vR + e.v[q] * e.R[q];
            dd coef = k0 ? dd_of(0.0) : (vR - e.g) / e.B;
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const int rr = pr * D + i;
                dd t = dd_of(0.0);
                for (int q = 0; q < e.m; ++q) t = t + e.Ainv[rr][q] * e.R[q];
                if (!k0) t = t - e.w[rr] * coef;
                Sr[i] += dd_round(t * c.C[lr]);
            }
            for (int q = 0; q < c.s; ++q) {
                const int lq = c.map[q];
                const double cc = c.C[lr] * c.C[lq];
                double b[D][D];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        const int rr = pr * D + i, qq = q * D + j;
                        dd v = e.Ainv[rr][qq];
                        if (!k0) v = v - e.w[rr] * e.v[qq] / e.B;
                        b[i][j] = dd_round(v * cc);
                    }
                if (q == pr) {
#pragma unroll
                    for (int i = 0; i < D; ++i)
#pragma unroll
                        for (int j = 0; j < D; ++j) diag[i][j] += b[i][j];
                } else {
                    write_block<D>(o, r, slot++, g2l ? g2l[c.dof[lq]] : (int32_t)c.dof[lq], b);
                }
            }
        }
        finish_row<D>(o, r, slot, diag, Sr);
        nb_local += (unsigned long long)slot;
    }
    nb_local = (unsigned long long)warp_sum((double)nb_local);
    if ((threadIdx.x & 31) == 0) atomicAdd(o.nblocks, nb_local);
}

// ------------------------------------------------------------------ data copies
void copy_problem_data(cr_hybrid_s *h, const cr_mesh_s *m, const cr_data &data, cudaStream_t s) {
    const int D = m->dim;
    CR_REQUIRE(data.fbar_d, CR_ERR_INVALID_ARG, "fbar_d is required");
    h->fbar.alloc(m->nc * D, s);
    CR_CUDA(cudaMemcpyAsync(h->fbar.get(), data.fbar_d, m->nc * D * sizeof(double), cudaMemcpyDeviceToDevice, s));
    h->has_dir = data.dirichlet_d != nullptr;
    if (h->has_dir) {
        h->dir.alloc(m->nc * (D + 1) * D, s);
        CR_CUDA(cudaMemcpyAsync(h->dir.get(), data.dirichlet_d, m->nc * (D + 1) * D * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    }
    h->has_uit = data.u_iter_d != nullptr;
    if (h->has_uit) {
        h->uit.alloc(m->nc * (D + 1) * D, s);
        CR_CUDA(cudaMemcpyAsync(h->uit.get(), data.u_iter_d, m->nc * (D + 1) * D * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    }
    h->has_pit = data.p_iter_d != nullptr;
    if (h->has_pit) {
        h->pit.alloc(m->nc, s);
        CR_CUDA(cudaMemcpyAsync(h->pit.get(), data.p_iter_d, m->nc * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
}

ProbView prob_view(const cr_hybrid_s *h) {
    ProbView p;
    p.mu = h->prm.mu;
    p.nu = h->prm.nu;
    p.k0 = h->prm.gauge_cell;
    p.is_ns = h->is_ns;
    p.fbar = h->fbar.get();
    p.dir = h->has_dir ? h->dir.get() : nullptr;
    p.uit = h->has_uit ? h->uit.get() : nullptr;
    p.pit = h->has_pit ? h->pit.get() : nullptr;
    p.E = h->prm.shift == CR_SHIFT_MIS ? h->E.get() : nullptr;
    p.rcell = h->rcell.n ? h->rcell.get() : nullptr;
    p.gcell = h->gcell.n ? h->gcell.get() : nullptr;
    return p;
}

static int read_int(const int *d, cudaStream_t s) {
    int h = 0;
    CR_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    return h;
}

static cr_status status_of(int e) {
    switch (e) {
        case DE_NOINTERIOR: return CR_ERR_NO_INTERIOR_FACE;
        case DE_SINGULAR:
        case DE_BZERO: return CR_ERR_SINGULAR_LOCAL;
        default: return CR_ERR_CUDA;
    }
}

template <int D>
static void hybridise_t(cr_hybrid_s *h, const cr_mesh_s *m, cudaStream_t s) {
    const int T = 256;
    const int64_t nc = m->nc;
    const int64_t nrows = h->part.on ? h->part.nloc : m->nf_int;
    const int64_t row0 = h->part.on ? h->part.row0 : 0;
    const int32_t *g2l = h->part.on ? h->part.g2l.get() : nullptr;
    MeshView mv = mesh_view(m);
    DevBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    // ---- shift E_K
    h->inM1.alloc(nc, s);
    h->inM1.zero(s);
    h->E.alloc(nc * (D + 1), s);
    h->E.zero(s);
    h->lam.alloc(nc, s);
    h->lam.zero(s);
    if (h->prm.shift == CR_SHIFT_MIS) {
        DevBuf<uint8_t> state;
        state.alloc(nc, s);
        state.zero(s);
        DevBuf<unsigned> und;
        und.alloc(1, s);
        unsigned hu = 1;
        for (int round = 0; round < 10000 && hu; ++round) {
            und.zero(s);
            k_mis_round<D><<<grid_for(nc, T), T, 0, s>>>(mv, nc, h->prm.mis_seed, state.get(), und.get());
            CR_CHECK_LAUNCH();
            CR_CUDA(cudaMemcpyAsync(&hu, und.get(), sizeof(unsigned), cudaMemcpyDeviceToHost, s));
            CR_CUDA(cudaStreamSynchronize(s));
        }
        CR_REQUIRE(hu == 0, CR_ERR_CUDA, "MIS did not terminate");
        ProbView p0 = prob_view(h);
        p0.E = nullptr;
        k_lambda<D><<<grid_for(nc, 128), 128, 0, s>>>(mv, p0, nc, h->prm.lambda_factor, h->lam.get(), err.get());
        CR_CHECK_LAUNCH();
        k_shift<D><<<grid_for(nc, T), T, 0, s>>>(mv, nc, state.get(), h->lam.get(), h->E.get(), h->inM1.get());
        CR_CHECK_LAUNCH();
    }
    // ---- G, S
    BlockEll &G = h->G;
    G.d = D;
    G.W = 2 * D + 1;
    G.nrows = nrows;
    G.nslices = (nrows + 31) / 32;
    G.cols.alloc(G.nslices * G.W * 32, s);
    G.vals.alloc(G.nslices * G.W * D * D * 32, s);
    // padded rows of the last slice: zero values, column 0
    G.cols.zero(s);
    G.vals.zero(s);
    h->S.alloc(nrows * D, s);
    h->dinv.alloc(nrows * D, s);
    h->absdinv.alloc(nrows * D, s);
    h->bdinv.alloc(nrows * D * D, s);
    DevBuf<unsigned long long> nb;
    nb.alloc(1, s);
    nb.zero(s);
    h->rowlen.alloc(nrows, s);
    AsmOut o{G.cols.get(), G.vals.get(), h->rowlen.get(), h->S.get(), h->dinv.get(), h->absdinv.get(),
             h->bdinv.get(), nb.get(), err.get()};
    ProbView p = prob_view(h);
    if (!h->is_ns) {
        k_assemble_stokes<D><<<grid_for(nrows, 128, 16), 128, 0, s>>>(mv, p, m->dof_face.get(), nrows, row0, g2l, o);
    } else {
        k_assemble_ns<D><<<grid_for(nrows, 64, 16), 64, 0, s>>>(mv, p, m->dof_face.get(), nrows, row0, g2l, o);
    }
    CR_CHECK_LAUNCH();
    int e = read_int(err.get(), s);
    CR_REQUIRE(e == DE_OK, status_of(e), "local elimination failed (singular Ahat_K, B_K ~ 0 or cell without interior face)");
    unsigned long long hnb = 0;
    CR_CUDA(cudaMemcpyAsync(&hnb, nb.get(), sizeof(hnb), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    G.nblocks = (int64_t)hnb;
}

// backward-Euler step right-hand side per cell (mu = 1/dt; lumped mass |K|/(d+1) per local
// face): R_K(l) = data terms (force, Dirichlet fold) + mu |K|/(d+1) U^n_sigma(l),
// g_K = data term.  Rounded once from double-double.
template <int D>
__global__ void __launch_bounds__(128) k_transient_rhs(MeshView mv, ProbView p, int64_t nc, const double *Uprev,
                                                       double *Rout, double *gout) {
    constexpr int NF = D + 1;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        Cell<D> c;
        load_cell<D>(mv, K, c);
        dd R[NF][D], g;
        stokes_rhs<D>(c, p, R, g);
        const dd mK = two_prod(p.mu, c.vol) / (double)NF;
#pragma unroll
        for (int l = 0; l < NF; ++l)
#pragma unroll
            for (int i = 0; i < D; ++i) {
                dd v = R[l][i];
                if (c.dof[l] >= 0) v = v + mK * Uprev[(int64_t)c.dof[l] * D + i];
                Rout[(K * NF + l) * D + i] = dd_round(v);
            }
        gout[K] = dd_round(g);
    }
}

void transient_rhs(const cr_hybrid_s *h, const double *Uprev, double *R, double *g, cudaStream_t s) {
    const cr_mesh_s *m = h->mesh;
    CR_REQUIRE(!h->is_ns, CR_ERR_INVALID_ARG, "transient right-hand side: Stokes handles only");
    ProbView p = prob_view(h);
    p.rcell = p.gcell = nullptr;   // the data-derived terms
    MeshView mv = mesh_view(m);
    if (m->dim == 2)
        k_transient_rhs<2><<<grid_for(m->nc, 128, 16), 128, 0, s>>>(mv, p, m->nc, Uprev, R, g);
    else
        k_transient_rhs<3><<<grid_for(m->nc, 128, 16), 128, 0, s>>>(mv, p, m->nc, Uprev, R, g);
    CR_CHECK_LAUNCH();
}

// S of the same G for new cell right-hand sides (h->rcell / h->gcell): the Stokes assembly kernel with
// its G writes disabled
void hybrid_update_rhs(cr_hybrid_s *h, cudaStream_t s) {
    const cr_mesh_s *m = h->mesh;
    CR_REQUIRE(!h->is_ns, CR_ERR_INVALID_ARG, "hybrid_update_rhs: Stokes handles only");
    const int64_t nrows = h->G.nrows;
    const int64_t row0 = h->part.on ? h->part.row0 : 0;
    const int32_t *g2l = h->part.on ? h->part.g2l.get() : nullptr;
    DevBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    DevBuf<unsigned long long> nb;
    nb.alloc(1, s);
    nb.zero(s);
    AsmOut o{h->G.cols.get(), h->G.vals.get(), h->rowlen.get(), h->S.get(), h->dinv.get(), h->absdinv.get(),
             h->bdinv.get(), nb.get(), err.get()};
    MeshView mv = mesh_view(m);
    ProbView p = prob_view(h);
    if (m->dim == 2)
        k_assemble_stokes<2><<<grid_for(nrows, 128, 16), 128, 0, s>>>(mv, p, m->dof_face.get(), nrows, row0, g2l, o, 1);
    else
        k_assemble_stokes<3><<<grid_for(nrows, 128, 16), 128, 0, s>>>(mv, p, m->dof_face.get(), nrows, row0, g2l, o, 1);
    CR_CHECK_LAUNCH();
}

void hybridise(cr_hybrid_s *h, const cr_mesh_s *m, const cr_params &prm, const cr_data &data, cr_comm_s *comm,
               cudaStream_t s) {
    CR_REQUIRE(prm.physics == CR_STOKES || prm.physics == CR_NS_NEWTON_STEP, CR_ERR_INVALID_ARG, "bad physics");
    CR_REQUIRE(prm.shift == CR_SHIFT_NONE || prm.shift == CR_SHIFT_MIS, CR_ERR_INVALID_ARG, "bad shift");
    CR_REQUIRE(prm.gauge_cell >= 0 && prm.gauge_cell < m->nc, CR_ERR_INVALID_ARG, "gauge cell out of range");
    CR_REQUIRE(prm.nu > 0.0 && prm.mu >= 0.0, CR_ERR_INVALID_ARG, "need nu > 0, mu >= 0");
    CR_REQUIRE(m->nf_int > 0, CR_ERR_NO_INTERIOR_FACE, "mesh has no interior face");
    h->mesh = m;
    h->prm = prm;
    if (h->prm.lambda_factor <= 0.0) h->prm.lambda_factor = 1.1;
    h->is_ns = prm.physics == CR_NS_NEWTON_STEP;
    CR_REQUIRE(!h->is_ns || data.u_iter_d, CR_ERR_INVALID_ARG, "NS step needs u_iter_d");
    copy_problem_data(h, m, data, s);
    h->comm = comm;
    if (comm && comm->impl) setup_part(h, m, comm, s);
    if (m->dim == 2) hybridise_t<2>(h, m, s);
    else hybridise_t<3>(h, m, s);
}

// ------------------------------------------------------------------ canonical CSR export
template <int D>
__global__ void k_csr_counts(int64_t nrows, const uint8_t *rowlen, int64_t *cnt) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x)
        cnt[r] = (int64_t)rowlen[r] * D * D;
}

template <int D>
__global__ void k_csr_fill(EllView<D> G, const uint8_t *rowlen, const int64_t *base, const double *S,
                           const int32_t *l2g, int64_t *row_ptr, int32_t *cols, double *vals, double *Sout) {
    constexpr int W = 2 * D + 1, B2 = D * D;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < G.nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int nb = rowlen[r];
        const int64_t slice = r >> 5;
        const int lane = (int)(r & 31);
        int bc[W], bs[W];
        for (int k = 0; k < nb; ++k) {
            const int32_t c = G.cols[slice * (W * 32) + k * 32 + lane];
            bc[k] = l2g ? l2g[c] : c;   // partitioned: export GLOBAL block columns
            bs[k] = k;
        }
        for (int i = 1; i < nb; ++i)            // insertion sort by block column
            for (int j = i; j > 0 && bc[j - 1] > bc[j]; --j) {
                int t = bc[j]; bc[j] = bc[j - 1]; bc[j - 1] = t;
                t = bs[j]; bs[j] = bs[j - 1]; bs[j - 1] = t;
            }
        for (int i = 0; i < D; ++i) {
            int64_t pos = base[r] + (int64_t)i * nb * D;
            row_ptr[r * D + i] = pos;
            for (int k = 0; k < nb; ++k)
                for (int j = 0; j < D; ++j) {
                    cols[pos] = bc[k] * D + j;
                    vals[pos] = G.vals[slice * ((int64_t)W * B2 * 32) + (bs[k] * B2 + i * D + j) * 32 + lane];
                    ++pos;
                }
            if (Sout) Sout[r * D + i] = S[r * D + i];
        }
    }
}

void hybrid_export_csr(const cr_hybrid_s *h, int64_t *row_ptr, int32_t *cols, double *vals, double *S,
                       cudaStream_t s) {
    const int D = h->G.d;
    const int64_t nrows = h->G.nrows;
    const int32_t *l2g = h->part.on ? h->part.l2g.get() : nullptr;
    DevBuf<int64_t> cnt, base;
    cnt.alloc(nrows, s);
    base.alloc(nrows, s);
    const int T = 256;
    if (D == 2) k_csr_counts<2><<<grid_for(nrows, T), T, 0, s>>>(nrows, h->rowlen.get(), cnt.get());
    else k_csr_counts<3><<<grid_for(nrows, T), T, 0, s>>>(nrows, h->rowlen.get(), cnt.get());
    CR_CHECK_LAUNCH();
    size_t tb = 0;
    CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), base.get(), (int)nrows, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, s);
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), base.get(), (int)nrows, s));
    if (D == 2) {
        EllView<2> G{h->G.cols.get(), h->G.vals.get(), nrows};
        k_csr_fill<2><<<grid_for(nrows, T), T, 0, s>>>(G, h->rowlen.get(), base.get(), h->S.get(), l2g, row_ptr, cols, vals, S);
    } else {
        EllView<3> G{h->G.cols.get(), h->G.vals.get(), nrows};
        k_csr_fill<3><<<grid_for(nrows, T), T, 0, s>>>(G, h->rowlen.get(), base.get(), h->S.get(), l2g, row_ptr, cols, vals, S);
    }
    CR_CHECK_LAUNCH();
    int64_t nnz = h->G.nblocks * D * D;
    CR_CUDA(cudaMemcpyAsync(row_ptr + nrows * D, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    CR_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ plain SpMV y = G x
template <int D>
__global__ void __launch_bounds__(256) k_spmv(EllView<D> G, const double *__restrict__ x, double *__restrict__ y) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < G.nrows; r += (int64_t)gridDim.x * blockDim.x) {
        double v[D];
        spmv_row<D>(G, r, x, v);
#pragma unroll
        for (int i = 0; i < D; ++i) y[r * D + i] = v[i];
    }
}

void spmv(const BlockEll &G, const double *x, double *y, cudaStream_t s) {
    const int T = 256;
    if (G.d == 2) {
        EllView<2> v{G.cols.get(), G.vals.get(), G.nrows};
        k_spmv<2><<<grid_for(G.nrows, T), T, 0, s>>>(v, x, y);
    } else {
        EllView<3> v{G.cols.get(), G.vals.get(), G.nrows};
        k_spmv<3><<<grid_for(G.nrows, T), T, 0, s>>>(v, x, y);
    }
    CR_CHECK_LAUNCH();
}

}  // namespace cr
