// cr_recover: per-cell recovery of P and U from W.
//   K16a cell kernel : elimination recomputed (double-double), P_K, Uhat_K at every interior
//                      local face -> Uhat[nc][d+1][d]
//   K16b face kernel : U_sigma = copy of face_cells[sigma][0]; max |Uhat_K - Uhat_L|
//   K16c cell kernel : max_K |sum_{sigma in F_K} a_{K,sigma} . U_sigma| (Dirichlet values on
//                      boundary faces) — the discrete divergence of the assembled U
#include <vector>
#include "local.cuh"
#include "spmv.cuh"

namespace cr {

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

template <int D>
__global__ void __launch_bounds__(128) k_recover_cells(MeshView mv, ProbView p, int64_t nc, const double *W,
                                                       double *P, double *Uhat, int *err) {
    constexpr int NF = D + 1;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        Cell<D> c;
        load_cell<D>(mv, K, c);
        const bool k0 = (K == p.k0);
        double *Uo = Uhat + K * NF * D;
#pragma unroll
        for (int q = 0; q < NF * D; ++q) Uo[q] = 0.0;
        if (!p.is_ns) {
            StokesElim<D> e;
            stokes_eliminate<D>(c, p, e);
            if (e.status != DE_OK) { atomicCAS(err, DE_OK, e.status); P[K] = 0.0; continue; }
            dd R[NF][D], g;
            stokes_rhs<D>(c, p, R, g);
            // rhs_i = R_i - C W_i ; P = (sum_i w_i^t rhs_i - g)/B ; Uhat_i = Shat^{-1} rhs_i - P w_i
            dd rhs[D][NF];
            dd wr = dd_of(0.0);
#pragma unroll
            for (int i = 0; i < D; ++i)
                for (int q = 0; q < c.s; ++q) {
                    const int l = c.map[q];
                    rhs[i][q] = R[l][i] - dd_of(c.C[l] * W[(int64_t)c.dof[l] * D + i]);
                    wr = wr + e.w[i][q] * rhs[i][q];
                }
            dd PK = k0 ? dd_of(0.0) : (wr - g) / e.B;
            P[K] = dd_round(PK);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                ldl_solve<D>(e, c.s, rhs[i]);
                for (int q = 0; q < c.s; ++q) Uo[c.map[q] * D + i] = dd_round(rhs[i][q] - e.w[i][q] * PK);
            }
        } else {
            NSElim<D> e;
            ns_eliminate<D>(c, p, e);
            if (e.status != DE_OK) { atomicCAS(err, DE_OK, e.status); P[K] = 0.0; continue; }
            dd rhs[NF * D];
            dd vr = dd_of(0.0);
            for (int q = 0; q < e.m; ++q) {
                const int l = e.map[q] / D, i = e.map[q] % D;
                rhs[q] = e.R[q] - dd_of(c.C[l] * W[(int64_t)c.dof[l] * D + i]);
                vr = vr + e.v[q] * rhs[q];
            }
            dd PK = k0 ? dd_of(0.0) : (vr - e.g) / e.B;
            P[K] = dd_round(PK);
            for (int q = 0; q < e.m; ++q) {
                const int l = e.map[q] / D, i = e.map[q] % D;
                rhs[q] = rhs[q] + dd_of(c.a[l][i]) * PK;   // - D P with D = -a
            }
            for (int r = 0; r < e.m; ++r) {
                dd acc = dd_of(0.0);
                for (int q = 0; q < e.m; ++q) acc = acc + e.Ainv[r][q] * rhs[q];
                Uo[e.map[r]] = dd_round(acc);
            }
        }
    }
}

template <int D>
__global__ void k_recover_faces(const int32_t *dof_face, const int32_t *face_cells, const int32_t *cell_faces,
                                int64_t nrows, const double *Uhat, double *U, double *diag) {
    constexpr int NF = D + 1;
    double mx = 0.0;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int f = dof_face[r];
        const int64_t K = face_cells[2 * (int64_t)f], L = face_cells[2 * (int64_t)f + 1];
        int lK = 0, lL = 0;
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            if (cell_faces[K * NF + l] == f) lK = l;
            if (cell_faces[L * NF + l] == f) lL = l;
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double uK = Uhat[(K * NF + lK) * D + i], uL = Uhat[(L * NF + lL) * D + i];
            U[r * D + i] = uK;
            mx = fmax(mx, fabs(uK - uL));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && diag) atomic_max_nonneg(diag, mx);
}

template <int D>
__global__ void k_cell_divergence(MeshView mv, const double *dir, int64_t nc, const double *U, double *diag) {
    constexpr int NF = D + 1;
    double mx = 0.0;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            const int f = mv.cell_faces[K * NF + l];
            const int dof = mv.face_dof[f];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double u = dof >= 0 ? U[(int64_t)dof * D + i] : (dir ? dir[(K * NF + l) * D + i] : 0.0);
                s += mv.a[(K * NF + l) * D + i] * u;
            }
        }
        mx = fmax(mx, fabs(s));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(diag, mx);
}

// per (cell, local face) values of a face field: U on interior faces, bnd (or 0) on boundary faces
template <int D>
__global__ void k_cell_face_values(const int32_t *cell_faces, const int32_t *face_dof, int64_t nc, const double *U,
                                   const double *bnd, double *out) {
    constexpr int NF = D + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc * NF; t += (int64_t)gridDim.x * blockDim.x) {
        const int dof = face_dof[cell_faces[t]];
#pragma unroll
        for (int i = 0; i < D; ++i)
            out[t * D + i] = dof >= 0 ? U[(int64_t)dof * D + i] : (bnd ? bnd[t * D + i] : 0.0);
    }
}

void cell_face_values(const cr_mesh_s *m, const double *U, const double *bnd, double *out, cudaStream_t s) {
    const int64_t n = m->nc * (m->dim + 1);
    if (m->dim == 2)
        k_cell_face_values<2><<<grid_for(n, 256), 256, 0, s>>>(m->cell_faces.get(), m->face_dof.get(), m->nc, U, bnd, out);
    else
        k_cell_face_values<3><<<grid_for(n, 256), 256, 0, s>>>(m->cell_faces.get(), m->face_dof.get(), m->nc, U, bnd, out);
    CR_CHECK_LAUNCH();
}

void recover(const cr_hybrid_s *h, const double *W, double *U, double *P, double *diag, cudaStream_t s) {
    const cr_mesh_s *m = h->mesh;
    const int D = m->dim;
    DevBuf<double> Wfull;
    if (h->part.on) {   // every rank recovers the whole mesh from the gathered W (once per solve)
        const Part &Pt = h->part;
        std::vector<int64_t> cnt(Pt.nranks), dsp(Pt.nranks);
        for (int q = 0; q < Pt.nranks; ++q) {
            dsp[q] = Pt.all_row0[q] * D;
            cnt[q] = (Pt.all_row0[q + 1] - Pt.all_row0[q]) * D;
        }
        Wfull.alloc(Pt.nglobal * D, s);
        h->comm->impl->allgatherv(W, Wfull.get(), cnt, dsp, s);
        W = Wfull.get();
    }
    const int64_t nc = m->nc, nrows = m->nf_int;
    MeshView mv = mesh_view(m);
    ProbView p = prob_view(h);
    // the per-cell copies live in the handle (allocated once: no pool traffic per recovery)
    DevBuf<double> &Uhat = const_cast<cr_hybrid_s *>(h)->uhat;
    if (Uhat.n != (size_t)(nc * (D + 1) * D)) Uhat.alloc(nc * (D + 1) * D, s);
    DevBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    DevBuf<double> dg;
    dg.alloc(2, s);
    dg.zero(s);
    const int T = 256;
    if (D == 2) {
        k_recover_cells<2><<<grid_for(nc, 128, 16), 128, 0, s>>>(mv, p, nc, W, P, Uhat.get(), err.get());
        CR_CHECK_LAUNCH();
        k_recover_faces<2><<<grid_for(nrows, T), T, 0, s>>>(m->dof_face.get(), m->face_cells.get(), m->cell_faces.get(),
                                                            nrows, Uhat.get(), U, dg.get());
        CR_CHECK_LAUNCH();
        k_cell_divergence<2><<<grid_for(nc, T), T, 0, s>>>(mv, p.dir, nc, U, dg.get() + 1);
    } else {
        k_recover_cells<3><<<grid_for(nc, 128, 16), 128, 0, s>>>(mv, p, nc, W, P, Uhat.get(), err.get());
        CR_CHECK_LAUNCH();
        k_recover_faces<3><<<grid_for(nrows, T), T, 0, s>>>(m->dof_face.get(), m->face_cells.get(), m->cell_faces.get(),
                                                            nrows, Uhat.get(), U, dg.get());
        CR_CHECK_LAUNCH();
        k_cell_divergence<3><<<grid_for(nc, T), T, 0, s>>>(mv, p.dir, nc, U, dg.get() + 1);
    }
    CR_CHECK_LAUNCH();
    if (diag) CR_CUDA(cudaMemcpyAsync(diag, dg.get(), 2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
    int he = 0;
    CR_CUDA(cudaMemcpyAsync(&he, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    CR_REQUIRE(he == DE_OK, CR_ERR_SINGULAR_LOCAL, "local elimination failed during recovery");
}

// Newton update: U += dU, P += dP, per-block partials of |dU|^2 and |U + dU|^2
__global__ void __launch_bounds__(256) k_newton_update(int64_t nU, double *U, const double *dU, int64_t nP, double *P,
                                                       const double *dP, double lam, double *part) {
    __shared__ double s0[256], s1[256];
    double a = 0.0, b = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nU; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = lam * dU[i], u = U[i] + d;
        U[i] = u;
        a = fma(d, d, a);
        b = fma(u, u, b);
    }
    if (dP)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nP; i += (int64_t)gridDim.x * blockDim.x)
            P[i] += lam * dP[i];
    s0[threadIdx.x] = a;
    s1[threadIdx.x] = b;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s0[threadIdx.x] += s0[threadIdx.x + o];
            s1[threadIdx.x] += s1[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = s0[0];
        part[2 * blockIdx.x + 1] = s1[0];
    }
}

void newton_update(int64_t nU, double *U, const double *dU, int64_t nP, double *P, const double *dP, double lam,
                   double *norms, cudaStream_t s) {
    const int G = num_sms() * 4;
    DevBuf<double> part;
    part.alloc(2 * G, s);
    k_newton_update<<<G, 256, 0, s>>>(nU, U, dU, nP, P, dP, lam, part.get());
    CR_CHECK_LAUNCH();
    std::vector<double> h(2 * G);
    CR_CUDA(cudaMemcpyAsync(h.data(), part.get(), 2 * G * sizeof(double), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    double a = 0.0, b = 0.0;
    for (int k = 0; k < G; ++k) {   // fixed order: deterministic
        a += h[2 * k];
        b += h[2 * k + 1];
    }
    norms[0] = sqrt(a);
    norms[1] = sqrt(b);
}

}  // namespace cr
