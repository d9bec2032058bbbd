// Parity mode of cr_solve (cr_solver_opts.refine_dd): the residual S - G W evaluated in
// double-double and iterative refinement on top of the fp64 Krylov solve.
//
// Why: the fp64 PCG recursion cannot certify residuals below ~u * ||G|| ||W|| / ||S||
// (measured floor 4e-13 at 2D n = 256).  The matrix-free G_K = C_K[c_K 1 1^t + T_K - u_K u_K^t]C_K
// (mf.cuh) has a large part c_K = 1/(mu|K|) acting on the cell sum sum_l C_l x_l, which nearly
// cancels for a converged W; summing it in fp64 loses ~|log10 h| digits.  Here every cell
// contribution and the sum of the two contributions of a face are carried in double-double
// (dd.cuh: error-free two_sum / two_prod), so r is the correctly rounded residual of the stored
// operator (the fp64 factors, or the assembled fp64 G).  Refinement (W += G^{-1} r with the fp64
// solver on r) then converges to the solution of that operator ("G W = S").
#include <cmath>
#include <vector>

#include "dd.cuh"
#include "internal.cuh"
#include "local.cuh"
#include "mf.cuh"
#include "spmv.cuh"

namespace cr {

// per (slot t, local face a, component i): the cell's contribution (C_K G_K C_K x_K)_a^i in dd
template <int D>
__global__ void __launch_bounds__(256) k_mf_contrib_dd(MfView M, const double *__restrict__ x, double2 *contrib) {
    using LY = MfLayout<D>;
    constexpr int NF = LY::NF, NT = LY::NT;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M.ncells; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slice = t >> 5;
        const int lane = (int)(t & 31);
        const int32_t *ip = M.ids + slice * (NF * 32) + lane;
        const double *vp = M.v + slice * ((int64_t)LY::NE * 32) + lane;
        const unsigned sg = M.sg[t];
        int id[NF];
        double cs[NF], xs[D][NF];
        for (int l = 0; l < NF; ++l) {
            id[l] = ip[l * 32];
            cs[l] = ((sg >> l) & 1u) ? -1.0 : 1.0;
            for (int i = 0; i < D; ++i) xs[i][l] = id[l] >= 0 ? cs[l] * x[(int64_t)id[l] * D + i] : 0.0;
        }
        const double c = vp[0];
        double T[NT], u[D][NF];
        for (int e = 0; e < NT; ++e) T[e] = vp[(1 + e) * 32];
        for (int i = 0; i < D; ++i)
            for (int l = 0; l < NF; ++l) u[i][l] = vp[(1 + NT + i * NF + l) * 32];
        dd pu = dd_of(0.0);
        for (int i = 0; i < D; ++i)
            for (int l = 0; l < NF; ++l) pu = pu + two_prod(u[i][l], xs[i][l]);
        for (int i = 0; i < D; ++i) {
            dd sum = dd_of(0.0);
            for (int l = 0; l < NF; ++l) sum = sum + xs[i][l];
            const dd cb = sum * c;
            for (int a = 0; a < NF; ++a) {
                dd y = cb;
                for (int b = 0; b < NF; ++b) {
                    const int e = a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
                    y = y + two_prod(T[e], xs[i][b]);
                }
                y = y - pu * u[i][a];
                contrib[(t * NF + a) * D + i] = cs[a] > 0 ? make_double2(y.hi, y.lo) : make_double2(-y.hi, -y.lo);
            }
        }
    }
}

// r = S - (sum of the two cells' contributions of each interior face), in dd, rounded once
template <int D>
__global__ void __launch_bounds__(256) k_mf_resid_dd(MeshView mv, const int32_t *dof_face, const int32_t *slot, const double2 *contrib,
                                                     const double *S, int64_t nrows, double *r) {
    constexpr int NF = D + 1;
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < nrows; row += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = dof_face[row];
        dd acc[D];
        for (int i = 0; i < D; ++i) acc[i] = dd_of(0.0);
        for (int side = 0; side < 2; ++side) {
            const int64_t K = mv.face_cells[2 * f + side];
            if (K < 0) continue;
            int l = 0;
            for (int q = 0; q < NF; ++q)
                if (mv.cell_faces[K * NF + q] == (int32_t)f) l = q;
            const int64_t t = slot[K];
            for (int i = 0; i < D; ++i) {
                const double2 v = contrib[(t * NF + l) * D + i];
                acc[i] = acc[i] + dd{v.x, v.y};
            }
        }
        for (int i = 0; i < D; ++i) r[row * D + i] = dd_round(dd_of(S[row * D + i]) - acc[i]);
    }
}

// r = S - G x with the assembled sliced block-ELL G, products and sums in dd
template <int D>
__global__ void __launch_bounds__(256) k_ell_resid_dd(EllView<D> G, const double *__restrict__ x, const double *S,
                                                      double *r) {
    constexpr int W = 2 * D + 1, B2 = D * D;
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < G.nrows; row += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slice = row >> 5;
        const int lane = (int)(row & 31);
        const int32_t *cp = G.cols + slice * (W * 32) + lane;
        const double *vp = G.vals + slice * ((int64_t)W * B2 * 32) + lane;
        dd y[D];
        for (int i = 0; i < D; ++i) y[i] = dd_of(0.0);
        for (int k = 0; k < W; ++k) {
            const int64_t c = cp[k * 32];
            for (int i = 0; i < D; ++i)
                for (int j = 0; j < D; ++j) y[i] = y[i] + two_prod(vp[(k * B2 + i * D + j) * 32], x[c * D + j]);
        }
        for (int i = 0; i < D; ++i) r[row * D + i] = dd_round(dd_of(S[row * D + i]) - y[i]);
    }
}

// per-block partial sums of a[i]^2 (fixed grid: deterministic)
__global__ void __launch_bounds__(256) k_sumsq_partials(int64_t n, const double *a, double *partials) {
    __shared__ double sh[256];
    double v = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v = fma(a[i], a[i], v);
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

__global__ void k_axpy1(int64_t n, double *y, const double *x) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) y[i] += x[i];
}

double norm2(const double *a, int64_t n, cudaStream_t s) {
    const int G = num_sms() * 4;
    DevBuf<double> part;
    part.alloc(G, s);
    k_sumsq_partials<<<G, 256, 0, s>>>(n, a, part.get());
    CR_CHECK_LAUNCH();
    std::vector<double> h(G);
    CR_CUDA(cudaMemcpyAsync(h.data(), part.get(), G * sizeof(double), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double v : h) t += v;
    return sqrt(t);
}

template <int D>
static void residual_dd_t(cr_hybrid_s *h, bool mf, const double *W, double *r, cudaStream_t s) {
    const int64_t nrows = h->G.nrows;
    if (mf) {
        build_mf(h, s);
        constexpr int NF = D + 1;
        DevBuf<double2> contrib;
        contrib.alloc((size_t)h->mf.ncells * NF * D, s);
        MfView M{h->mf.ids.get(), h->mf.sg.get(), h->mf.v.get(), h->mf.nb.get(), h->mf.ncells};
        k_mf_contrib_dd<D><<<grid_for(h->mf.ncells, 256), 256, 0, s>>>(M, W, contrib.get());
        CR_CHECK_LAUNCH();
        k_mf_resid_dd<D><<<grid_for(nrows, 256), 256, 0, s>>>(mesh_view(h->mesh), h->mesh->dof_face.get(), h->mf.slot.get(), contrib.get(),
                                                              h->S.get(), nrows, r);
        CR_CHECK_LAUNCH();
    } else {
        EllView<D> G{h->G.cols.get(), h->G.vals.get(), nrows};
        k_ell_resid_dd<D><<<grid_for(nrows, 256), 256, 0, s>>>(G, W, h->S.get(), r);
        CR_CHECK_LAUNCH();
    }
}

void residual_dd(cr_hybrid_s *h, bool mf, const double *W, double *r, double *rnorm, double *snorm, cudaStream_t s) {
    CR_REQUIRE(!h->part.on, CR_ERR_INVALID_ARG, "the double-double residual covers unpartitioned handles");
    if (h->G.d == 2) residual_dd_t<2>(h, mf, W, r, s);
    else residual_dd_t<3>(h, mf, W, r, s);
    const int64_t N = h->G.nrows * h->G.d;
    *rnorm = norm2(r, N, s);
    *snorm = norm2(h->S.get(), N, s);
}

// cr_solve: the fp64 solvers (solve.cu), plus the refinement of the parity mode
void solve(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep) {
    if (!o.refine_dd) {
        solve_rhs(h, o, W, s, rep, nullptr);
        return;
    }
    const bool pcg = o.method == CR_PCG_JACOBI || o.method == CR_PCG_BLOCKJACOBI || o.method == CR_PCG_AFW ||
                     o.method == CR_PCG_AFW2;
    CR_REQUIRE(pcg && !h->part.on, CR_ERR_INVALID_ARG, "refine_dd covers the PCG methods on one GPU");
    const double rtol = o.rtol > 0 ? o.rtol : 1e-10;
    const int64_t N = h->G.nrows * h->G.d;
    cudaEvent_t e0, e1;
    CR_CUDA(cudaEventCreate(&e0));
    CR_CUDA(cudaEventCreate(&e1));
    CR_CUDA(cudaEventRecord(e0, s));
    cr_solver_opts o1 = o;
    o1.refine_dd = 0;
    o1.rtol = std::max(rtol, 1e-11);   // the fp64 recursion certifies residuals down to ~1e-12
    cr_solve_report r1{};
    try {
        solve_rhs(h, o1, W, s, &r1, nullptr);
    } catch (const Error &e) {
        if (e.code != CR_ERR_NOT_CONVERGED) {
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            throw;
        }
    }
    DevBuf<double> r, dW;
    r.alloc(N, s);
    dW.alloc(N, s);
    double rn = 0.0, sn = 0.0;
    const bool mf = o.matrix_free != 0;
    residual_dd(h, mf, W, r.get(), &rn, &sn, s);
    int rounds = 0;
    int64_t inner = 0, launches = r1.kernel_launches, spmvs = r1.spmv_calls;
    double prev = INFINITY;
    while (sn > 0 && rn > rtol * sn && rounds < 8 && rn < 0.5 * prev) {
        prev = rn;
        cr_solver_opts oi = o1;
        // aim 10x below the target, but not below what fp64 certifies for the correction
        oi.rtol = std::min(0.5, std::max(0.1 * rtol * sn / rn, 1e-6));
        oi.max_iter = o.max_iter;
        dW.zero(s);
        cr_solve_report ri{};
        try {
            solve_rhs(h, oi, dW.get(), s, &ri, r.get());
        } catch (const Error &e) {
            if (e.code != CR_ERR_NOT_CONVERGED) throw;
        }
        inner += ri.iterations;
        launches += ri.kernel_launches;
        spmvs += ri.spmv_calls;
        k_axpy1<<<grid_for(N, 256), 256, 0, s>>>(N, W, dW.get());
        CR_CHECK_LAUNCH();
        residual_dd(h, mf, W, r.get(), &rn, &sn, s);
        ++rounds;
    }
    CR_CUDA(cudaEventRecord(e1, s));
    CR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double rel = sn > 0 ? rn / sn : 0.0;
    const bool ok = rel <= rtol;
    if (rep) {
        *rep = r1;
        rep->rel_res_true = rel;
        rep->inner_iterations = inner;
        rep->refine_rounds = rounds;
        if (r1.iterations > 0) rep->bytes_moved = r1.bytes_moved * (double)(r1.iterations + inner) / (double)r1.iterations;
        rep->kernel_launches = launches;
        rep->spmv_calls = spmvs;
        rep->seconds = ms * 1e-3;
        rep->converged = ok;
        rep->status = ok ? CR_OK : CR_ERR_NOT_CONVERGED;
    }
    if (!ok) throw Error(CR_ERR_NOT_CONVERGED, "refine_dd: the double-double residual did not reach rtol (see report)");
}

}  // namespace cr
