// CR_DC_FGMRES: steady Stokes and Navier-Stokes-step solves by flexible GMRES on the coupled
// system [[A, D^t],[D, 0]] (eq. (syslin)), right-preconditioned by the exact inverse
// of the TRANSIENT Stokes coupled operator K_mu (mass coefficient mu_inner, same viscosity),
// which the hybrid method applies (G_mu is SPD, solved by the two-level PCG on the
// matrix-free G_mu).  DESIGN.md §7.1.
//
// Why: the hybrid matrices of the steady / NS problems (shift E) are indefinite and
// their Krylov iteration counts grow like h^-1.2 (measured); K_mu^{-1} K0 has a
// mesh-independent spectrum (K0 - K_mu = -mu_inner M, a compact perturbation relative to the
// viscous operator), so the outer iteration count stays flat.
//
// One application of K_mu^{-1} to v = [v_U; v_P]:
//   R_K(l, i) = v_U(sigma, i) on the first cell of each interior face sigma (0 on the other),
//   g_K = v_P(K) (K != K0): any split with sum_K H_K R_K = v_U is admissible;
//   S_mu from these cell right-hand sides (hybrid_update_rhs), G_mu W = S_mu, recovery of
//   (U, P) = K_mu^{-1} v.
// At the end (and at every check) the target's W follows from (U, P) through the local
// relation on the first cell K of each face (C_{K,sigma} = 1):
//   W_sigma = R_K(l) - (Ahat_K U_K)(l) + a_{K,l} P_K          (Ahat_K = A_K + E_K, D_K = -a)
// which is exactly the W that the target hybrid system G W = S has for that (U, P), and the
// stopping rule is the TARGET's true ||S - G W|| / ||S|| <= rtol.
#include <cmath>
#include <vector>

#include "local.cuh"
#include "spmv.cuh"

#define GRID_STRIDE(r, n) \
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < (n); r += (int64_t)gridDim.x * blockDim.x)

namespace cr {

namespace {

__device__ __forceinline__ int64_t pidx(int64_t K, int k0) { return K < k0 ? K : K - 1; }

constexpr int kDotBlocks = 1184;   // 8 x 148: fixed, so the reduction order is fixed
constexpr int kDotThreads = 256;

__global__ void __launch_bounds__(kDotThreads) k_dot_partial(int64_t n, const double *a, const double *b,
                                                             double *partials) {
    __shared__ double sh[kDotThreads / 32];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc = fma(a[i], b[i], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < kDotThreads / 32; ++w) s += sh[w];
        partials[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(1024) k_dot_final(const double *partials, int np, double *out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
        *out = s;
    }
}

__global__ void k_axpy(int64_t n, double alpha, const double *x, double *y) {
    GRID_STRIDE(i, n) y[i] = fma(alpha, x[i], y[i]);
}
__global__ void k_scale(int64_t n, double alpha, const double *x, double *y) {
    GRID_STRIDE(i, n) y[i] = alpha * x[i];
}
__global__ void k_sub(int64_t n, const double *b, const double *y, double *r) {
    GRID_STRIDE(i, n) r[i] = b[i] - y[i];
}

// y = K x, canonical CSR, 8 lanes per row (rows have <= 3*(2d+1)*d + 2 entries)
constexpr int kTPR = 8;
__global__ void __launch_bounds__(256) k_csr_spmv(int64_t nrows, const int64_t *rp, const int32_t *cols,
                                                  const double *vals, const double *x, double *y) {
    const int lane = threadIdx.x % kTPR;
    const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kTPR;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x / kTPR;
    for (int64_t r = g0; r < nrows + ((nrows % gs) ? gs - nrows % gs : 0); r += gs) {
        double acc = 0.0;
        if (r < nrows)
            for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += kTPR) acc = fma(vals[k], x[cols[k]], acc);
#pragma unroll
        for (int o = kTPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, kTPR);
        if (r < nrows && lane == 0) y[r] = acc;
    }
}

// cell right-hand sides of one K_mu^{-1} application
template <int D>
__global__ void k_dc_split(MeshView mv, int64_t nc, int k0, int64_t nU, const double *v, double *rcell, double *gcell) {
    constexpr int NF = D + 1;
    GRID_STRIDE(K, nc) {
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            const int f = mv.cell_faces[K * NF + l];
            const int dof = mv.face_dof[f];
            const bool own = dof >= 0 && mv.face_cells[2 * (int64_t)f] == (int32_t)K;
#pragma unroll
            for (int i = 0; i < D; ++i) rcell[(K * NF + l) * D + i] = own ? v[(int64_t)dof * D + i] : 0.0;
        }
        gcell[K] = (K == k0) ? 0.0 : v[nU + pidx(K, k0)];
    }
}

__global__ void k_dc_pack(int64_t nU, int64_t nc, int k0, const double *U, const double *P, double *z) {
    GRID_STRIDE(i, nU) z[i] = U[i];
    GRID_STRIDE(K, nc) if (K != k0) z[nU + pidx(K, k0)] = P[K];
}

// target W from coupled (U, P): W_sigma = C_l (R_K(l) - (Ahat_K U_K)(l) + a_l P_K), K = first cell
template <int D>
__global__ void __launch_bounds__(64) k_dc_w(MeshView mv, ProbView p, const int32_t *dof_face, int64_t nrows,
                                             int64_t nU, const double *x, double *W) {
    constexpr int NF = D + 1, N = NF * D;
    GRID_STRIDE(r, nrows) {
        const int f = dof_face[r];
        const int64_t K = mv.face_cells[2 * (int64_t)f];
        Cell<D> c;
        load_cell<D>(mv, K, c);
        int l = 0;
#pragma unroll
        for (int q = 0; q < NF; ++q)
            if (c.face[q] == f) l = q;
        const double PK = (K == p.k0) ? 0.0 : x[nU + pidx(K, p.k0)];
        dd acc[D];
        if (!p.is_ns) {
            dd R[NF][D], g;
            stokes_rhs<D>(c, p, R, g);
#pragma unroll
            for (int i = 0; i < D; ++i) acc[i] = R[l][i] + two_prod(c.a[l][i], PK);
            for (int q = 0; q < c.s; ++q) {
                const int lq = c.map[q];
                dd sv = S_entry<D>(c, p.mu, p.nu, l, lq);
                if (lq == l && p.E) sv = sv + p.E[K * NF + l];
#pragma unroll
                for (int i = 0; i < D; ++i) acc[i] = acc[i] - sv * x[(int64_t)c.dof[lq] * D + i];
            }
        } else {
            dd A[N][N], R[N], g;
            ns_local_system<D>(c, p, A, R, g);
#pragma unroll
            for (int i = 0; i < D; ++i) acc[i] = R[l * D + i] + two_prod(c.a[l][i], PK);
            for (int q = 0; q < c.s; ++q) {
                const int lq = c.map[q];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        dd av = A[l * D + i][lq * D + j];
                        if (lq == l && i == j && p.E) av = av + p.E[K * NF + l];
                        acc[i] = acc[i] - av * x[(int64_t)c.dof[lq] * D + j];
                    }
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) W[r * D + i] = c.C[l] * dd_round(acc[i]);
    }
}

struct DotBuf {
    DevBuf<double> partials, out;
    explicit DotBuf(cudaStream_t s) {
        partials.alloc(kDotBlocks, s);
        out.alloc(1, s);
    }
};

double dot(DotBuf &db, int64_t n, const double *a, const double *b, cudaStream_t s) {
    k_dot_partial<<<kDotBlocks, kDotThreads, 0, s>>>(n, a, b, db.partials.get());
    CR_CHECK_LAUNCH();
    k_dot_final<<<1, 1024, 0, s>>>(db.partials.get(), kDotBlocks, db.out.get());
    CR_CHECK_LAUNCH();
    double h = 0.0;
    CR_CUDA(cudaMemcpyAsync(&h, db.out.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    return h;
}

int vgrid(int64_t n) { return grid_for(n, 256, 8); }

}  // namespace

void coupled_spmv(const cr_coupled_s *c, const double *x, double *y, cudaStream_t s) {
    k_csr_spmv<<<grid_for(c->n_rows * kTPR, 256, 8), 256, 0, s>>>(c->n_rows, c->row_ptr.get(), c->cols.get(),
                                                                   c->vals.get(), x, y);
    CR_CHECK_LAUNCH();
}

void solve_dc(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep) {
    const cr_mesh_s *m = h->mesh;
    CR_REQUIRE(!h->part.on, CR_ERR_INVALID_ARG, "CR_DC_FGMRES: single-rank handles only");
    const int D = m->dim;
    const int64_t nrows = m->nf_int, nc = m->nc, nU = (int64_t)D * nrows;
    const double rtol = o.rtol > 0 ? o.rtol : 1e-10;
    const double mu_in = o.mu_inner > 0 ? o.mu_inner : 1.0;
    const double in_rtol = o.inner_rtol > 0 ? o.inner_rtol : 1e-11;
    const int mres = o.restart > 0 ? std::min(o.restart, 200) : 30;
    const int64_t max_outer = o.max_iter > 0 ? o.max_iter : 500;
    cudaEvent_t e0, e1;
    CR_CUDA(cudaEventCreate(&e0));
    CR_CUDA(cudaEventCreate(&e1));
    CR_CUDA(cudaEventRecord(e0, s));

    // target coupled system K0 x = b (same data the target hybrid owns)
    cr_data td{};
    td.fbar_d = h->fbar.get();
    td.dirichlet_d = h->has_dir ? h->dir.get() : nullptr;
    td.u_iter_d = h->has_uit ? h->uit.get() : nullptr;
    td.p_iter_d = h->has_pit ? h->pit.get() : nullptr;
    cr_coupled_s K0;
    assemble_coupled(&K0, m, h->prm, td, s);
    const int64_t n = K0.n_rows;

    // inner transient Stokes hybrid (mu_inner, same nu and gauge cell, no shift)
    cr_hybrid_s hin;
    {
        cr_params pin = h->prm;
        pin.mu = mu_in;
        pin.physics = CR_STOKES;
        pin.shift = CR_SHIFT_NONE;
        DevBuf<double> zf;
        zf.alloc(nc * D, s);
        zf.zero(s);
        cr_data din{};
        din.fbar_d = zf.get();
        hybridise(&hin, m, pin, din, nullptr, s);
        CR_CUDA(cudaStreamSynchronize(s));
    }
    hin.rcell.alloc(nc * (D + 1) * D, s);
    hin.gcell.alloc(nc, s);
    cr_solver_opts io{};
    io.method = CR_PCG_AFW2;
    io.rtol = in_rtol;
    io.max_iter = 200000;
    io.check_every = o.check_every;
    io.matrix_free = 1;
    io.coarse = o.coarse;
    DevBuf<double> Win, Uin, Pin;
    Win.alloc(nU, s);
    Uin.alloc(nU, s);
    Pin.alloc(nc, s);
    int64_t inner_its = 0, inner_calls = 0;
    const MeshView mv = mesh_view(m);
    const int k0 = h->prm.gauge_cell;
    auto apply_minv = [&](const double *v, double *z) {
        if (D == 2) k_dc_split<2><<<vgrid(nc), 256, 0, s>>>(mv, nc, k0, nU, v, hin.rcell.get(), hin.gcell.get());
        else k_dc_split<3><<<vgrid(nc), 256, 0, s>>>(mv, nc, k0, nU, v, hin.rcell.get(), hin.gcell.get());
        CR_CHECK_LAUNCH();
        hybrid_update_rhs(&hin, s);
        Win.zero(s);
        cr_solve_report ir{};
        try {
            solve(&hin, io, Win.get(), s, &ir);
        } catch (const Error &e) {
            if (e.code != CR_ERR_NOT_CONVERGED) throw;   // an inexact inner solve is still a preconditioner
        }
        inner_its += ir.iterations;
        ++inner_calls;
        recover(&hin, Win.get(), Uin.get(), Pin.get(), nullptr, s);
        k_dc_pack<<<vgrid(nU), 256, 0, s>>>(nU, nc, k0, Uin.get(), Pin.get(), z);
        CR_CHECK_LAUNCH();
    };

    // target hybrid residual of the W that a coupled iterate x defines
    DotBuf db(s);
    DevBuf<double> GW, rW;
    GW.alloc(nU, s);
    rW.alloc(nU, s);
    const ProbView pt = prob_view(h);
    const double Snorm = std::sqrt(dot(db, nU, h->S.get(), h->S.get(), s));
    auto target_res = [&](const double *x) {
        if (D == 2) k_dc_w<2><<<grid_for(nrows, 64, 16), 64, 0, s>>>(mv, pt, m->dof_face.get(), nrows, nU, x, W);
        else k_dc_w<3><<<grid_for(nrows, 64, 16), 64, 0, s>>>(mv, pt, m->dof_face.get(), nrows, nU, x, W);
        CR_CHECK_LAUNCH();
        spmv(h->G, W, GW.get(), s);
        k_sub<<<vgrid(nU), 256, 0, s>>>(nU, h->S.get(), GW.get(), rW.get());
        CR_CHECK_LAUNCH();
        const double rr = dot(db, nU, rW.get(), rW.get(), s);
        return Snorm > 0 ? std::sqrt(rr) / Snorm : std::sqrt(rr);
    };

    // FGMRES(m), x0 = 0
    DevBuf<double> x, r, xt;
    x.alloc(n, s);
    r.alloc(n, s);
    xt.alloc(n, s);
    x.zero(s);
    std::vector<DevBuf<double>> V(mres + 1), Z(mres);
    for (auto &v : V) v.alloc(n, s);
    for (auto &z : Z) z.alloc(n, s);
    std::vector<double> Hs((mres + 1) * mres), cs(mres), sn(mres), gv(mres + 1), y(mres);
    auto Hm = [&](int i, int j) -> double & { return Hs[j * (mres + 1) + i]; };
    const double bnorm = std::sqrt(dot(db, n, K0.rhs.get(), K0.rhs.get(), s));
    int64_t outer = 0;
    double tres = target_res(x.get());
    int status = CR_OK;
    int64_t spmvs = 0;
    double est = bnorm;
    bool done = !(tres > rtol) || bnorm == 0.0;
    // form xt = x + sum_{i<=j} y_i Z_i from the current least-squares problem
    auto form = [&](int j) {
        for (int i = j; i >= 0; --i) {
            double t = gv[i];
            for (int k = i + 1; k <= j; ++k) t -= Hm(i, k) * y[k];
            y[i] = t / Hm(i, i);
        }
        CR_CUDA(cudaMemcpyAsync(xt.get(), x.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        for (int i = 0; i <= j; ++i) {
            k_axpy<<<vgrid(n), 256, 0, s>>>(n, y[i], Z[i].get(), xt.get());
            CR_CHECK_LAUNCH();
        }
    };
    while (!done) {
        coupled_spmv(&K0, x.get(), r.get(), s);
        ++spmvs;
        k_sub<<<vgrid(n), 256, 0, s>>>(n, K0.rhs.get(), r.get(), r.get());
        CR_CHECK_LAUNCH();
        const double beta = std::sqrt(dot(db, n, r.get(), r.get(), s));
        if (!(beta > 0)) break;
        k_scale<<<vgrid(n), 256, 0, s>>>(n, 1.0 / beta, r.get(), V[0].get());
        CR_CHECK_LAUNCH();
        std::fill(gv.begin(), gv.end(), 0.0);
        gv[0] = beta;
        int j = 0;
        bool cycle_end = false;
        for (; j < mres && !cycle_end; ++j) {
            apply_minv(V[j].get(), Z[j].get());
            coupled_spmv(&K0, Z[j].get(), V[j + 1].get(), s);
            ++spmvs;
            ++outer;
            for (int i = 0; i <= j; ++i) {   // modified Gram-Schmidt
                const double hij = dot(db, n, V[j + 1].get(), V[i].get(), s);
                Hm(i, j) = hij;
                k_axpy<<<vgrid(n), 256, 0, s>>>(n, -hij, V[i].get(), V[j + 1].get());
                CR_CHECK_LAUNCH();
            }
            const double hn = std::sqrt(dot(db, n, V[j + 1].get(), V[j + 1].get(), s));
            Hm(j + 1, j) = hn;
            if (hn > 0) {
                k_scale<<<vgrid(n), 256, 0, s>>>(n, 1.0 / hn, V[j + 1].get(), V[j + 1].get());
                CR_CHECK_LAUNCH();
            }
            for (int i = 0; i < j; ++i) {   // previous Givens rotations
                const double a = Hm(i, j), b = Hm(i + 1, j);
                Hm(i, j) = cs[i] * a + sn[i] * b;
                Hm(i + 1, j) = -sn[i] * a + cs[i] * b;
            }
            const double a = Hm(j, j), b = Hm(j + 1, j);
            const double rho = std::hypot(a, b);
            cs[j] = rho > 0 ? a / rho : 1.0;
            sn[j] = rho > 0 ? b / rho : 0.0;
            Hm(j, j) = rho;
            Hm(j + 1, j) = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            est = std::fabs(gv[j + 1]);
            // the target's own stopping rule on the W of the current iterate
            form(j);
            tres = target_res(xt.get());
            if (!(tres > rtol)) { done = true; cycle_end = true; }
            else if (outer >= max_outer || hn == 0.0) cycle_end = true;
        }
        CR_CUDA(cudaMemcpyAsync(x.get(), xt.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        if (!done && outer >= max_outer) { status = CR_ERR_NOT_CONVERGED; break; }
    }
    if (done) tres = target_res(x.get());   // W holds the W of the returned iterate
    CR_CUDA(cudaEventRecord(e1, s));
    CR_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    CR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (status == CR_OK && !(tres <= rtol)) status = CR_ERR_NOT_CONVERGED;
    if (rep) {
        rep->iterations = outer;
        rep->rel_res_true = tres;
        rep->rel_res_recursive = bnorm > 0 ? est / bnorm : 0.0;   // coupled residual estimate
        rep->converged = status == CR_OK;
        rep->status = status;
        rep->seconds = ms * 1e-3;
        rep->spmv_calls = spmvs;
        rep->kernel_launches = 0;
        rep->inner_iterations = inner_its;
    }
    if (status != CR_OK) throw Error((cr_status)status, "CR_DC_FGMRES did not converge (see report)");
}

}  // namespace cr
