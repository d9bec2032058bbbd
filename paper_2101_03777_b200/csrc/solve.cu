// cr_solve: Krylov solvers for G W = S on the device (§4.2-4.3).
//
// Every solver keeps its scalars in a device-resident KState; each reduction is a
// deterministic two-level sum (fixed grid, per-block partials, last block sums in block
// order) whose last block also performs the scalar recurrence (alpha, beta, Givens, ...).
// `check_every` iterations are captured once into a CUDA graph and replayed; after each
// replay the host reads the state (one 128-byte D2H) to test convergence.  Kernels return
// immediately once the state flag is set, so a converged graph replay costs ~launch time.
//
//   PCG       (SPD G, mu > 0):  3 kernels/iter: spmv+p.q | x,r update + z=M r + r.z, r.r | p = z + beta p
//   MINRES    (symmetric, steady): spmv+z.q | Lanczos v, z=M v, z.v + Givens | w, x update
//   BiCGStab  (nonsymmetric, NS): p,y | spmv+rhat.v | s,z | spmv+t.s,t.t | x,r update + rhat.r, r.r
//   GMRES(m)  (nonsymmetric): Arnoldi with classical Gram-Schmidt twice, Givens on device
// Stopping rule: TRUE relative residual ||S - G W|| / ||S|| <= rtol (reading 12).
#include <cub/cub.cuh>
#include <cstdlib>

#include <cmath>
#include <cstddef>
#include <cstring>

#include "afw.cuh"
#include "internal.cuh"
#include "mf.cuh"
#include "spmv.cuh"

namespace cr {

enum { FLAG_RUN = 0, FLAG_CONV = 1, FLAG_BREAK = 2 };
constexpr int kMaxRestart = 128;
constexpr int kLanczos = 1024;   // CG coefficients kept for the kappa estimate (cr_solve_report)

struct KState {
    // ---- header: read back by the host after every graph replay
    long long iters;
    long long wx_iter;   // MINRES: last iteration whose w/x update ran
    int flag;
    int k;               // GMRES: Arnoldi steps done in the current cycle
    unsigned tickets[8];
    double red[4];       // distributed mode: this rank's reduction values, allreduced in place
    double qc;           // two-level: c^t E^{-1} c of the coarse correction (global)
    double qf;           // two-level: r^t M_patch^{-1} r of the patch part (global)
    double rho, alpha, beta, pq, rr, bb, tol2;
    // MINRES
    double gamma, gamma_old, delta, eta, eta0, c, c_old, s, s_old;
    double a1, a2, a3, cn, eta_w, gz;
    // BiCGStab
    double omega, rho_new, rv, ts, tt;
    double hnorm;
    // ---- GMRES arrays (device only)
    double H[(kMaxRestart + 1) * kMaxRestart];
    double cs[kMaxRestart], sn[kMaxRestart], g[kMaxRestart + 1], h[kMaxRestart + 1], y[kMaxRestart];
    // PCG: (rho_k, p_k^t G p_k) of iteration k < kLanczos -> alpha_k = rho_k / pq_k,
    // beta_k = rho_{k+1} / rho_k: the Lanczos tridiagonal of the preconditioned G
    double lz[2 * kLanczos];
};
constexpr size_t kStateHeader = offsetof(KState, H);

struct SolverWork {
    int64_t N = 0, Nalloc = 0;
    int D = 0;
    DevBuf<double> x, b, r, p, q, z, z2, v, v2, w, w2, y, t, rhat;
    DevBuf<double> V;           // GMRES basis (m+1) x N
    DevBuf<double> zs;          // patch preconditioner: per-(face, slot) contributions
    DevBuf<double> partials;
    DevBuf<KState> st;
    KState *hst = nullptr;      // pinned
    cudaGraphExec_t graph = nullptr;
    int graph_key = -1;
    int64_t graph_kernels = 0;  // kernel nodes of `graph` (launch accounting)
    cudaEvent_t e0 = nullptr, e1 = nullptr, es = nullptr;   // solve start / end, preconditioner setup done
    cudaStream_t cap = nullptr;   // private capture stream
    cudaStream_t side = nullptr;  // two-level: the coarse path runs here, concurrently with the patches
    cudaEvent_t fork = nullptr, join = nullptr;
    ~SolverWork() {
        if (side) cudaStreamDestroy(side);
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (cap) cudaStreamDestroy(cap);
        if (graph) cudaGraphExecDestroy(graph);
        if (hst) cudaFreeHost(hst);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (es) cudaEventDestroy(es);
    }
};

void free_solver_work(SolverWork *w) { delete w; }

constexpr int kT = 256;
constexpr int kMaxPartials = 8;   // values per block

#define GRID_STRIDE(r, n) for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < (n); r += (int64_t)gridDim.x * blockDim.x)

// preconditioner application on one block row: z = M r
template <int D, int PREC>
__device__ __forceinline__ void apply_prec(const double *M, int64_t r, const double (&rv)[D], double (&zv)[D]) {
    if constexpr (PREC == 1) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) acc = fma(M[(r * D + i) * D + j], rv[j], acc);
            zv[i] = acc;
        }
    } else {
#pragma unroll
        for (int i = 0; i < D; ++i) zv[i] = M[r * D + i] * rv[i];
    }
}

template <int D>
__device__ __forceinline__ void ld(const double *a, int64_t r, double (&v)[D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = a[r * D + i];
}
template <int D>
__device__ __forceinline__ void stv(double *a, int64_t r, const double (&v)[D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) a[r * D + i] = v[i];
}

// ------------------------------------------------------------------ scalar recurrences
// Applied by the last block of a reduction on one GPU, or by k_fin after the allreduce of
// the per-rank values in st->red on several (the same code either way).
enum FinKind { FIN_BB, FIN_RR, FIN_PCG_INIT, FIN_PQ, FIN_UPD_PC, FIN_UPD_R, FIN_AFW_PCG_INIT, FIN_AFW_PCG,
               FIN_AFW2_PCG_INIT, FIN_AFW2_PCG, FIN_AFW2_QF_INIT, FIN_AFW2_QF, FIN_PQ2 };

__device__ __forceinline__ void apply_fin(KState *st, int kind, const double *t, double rtol) {
    switch (kind) {
        case FIN_BB: st->bb = t[0]; break;
        case FIN_RR: st->rr = t[0]; break;
        case FIN_PCG_INIT:   // t = (r.z, r.r)
            st->rho = t[0];
            st->rr = t[1];
            st->tol2 = rtol * rtol * st->bb;
            st->flag = (t[1] <= st->tol2) ? FLAG_CONV : FLAG_RUN;
            break;
        case FIN_PQ:         // t = p.q
            if (st->iters < kLanczos) { st->lz[2 * st->iters] = st->rho; st->lz[2 * st->iters + 1] = t[0]; }
            st->pq = t[0];
            if (!(t[0] > 0.0)) st->flag = FLAG_BREAK;
            else st->alpha = st->rho / t[0];
            break;
        case FIN_UPD_PC:     // t = (r.z, r.r)
            st->iters += 1;
            st->rr = t[1];
            st->beta = t[0] / st->rho;
            st->rho = t[0];
            if (t[1] <= st->tol2) st->flag = FLAG_CONV;
            break;
        case FIN_UPD_R:      // t = r.r
            st->iters += 1;
            st->rr = t[0];
            if (t[0] <= st->tol2) st->flag = FLAG_CONV;
            break;
        case FIN_AFW_PCG_INIT:   // t = r^t M^{-1} r
            st->rho = t[0];
            st->beta = 0.0;
            st->tol2 = rtol * rtol * st->bb;
            st->flag = (st->rr <= st->tol2) ? FLAG_CONV : FLAG_RUN;
            break;
        case FIN_AFW_PCG:
            st->beta = t[0] / st->rho;
            st->rho = t[0];
            break;
        case FIN_AFW2_PCG_INIT:  // r^t M2^{-1} r = fine part + coarse part
            st->rho = t[0] + st->qc;
            st->beta = 0.0;
            st->tol2 = rtol * rtol * st->bb;
            st->flag = (st->rr <= st->tol2) ? FLAG_CONV : FLAG_RUN;
            break;
        case FIN_AFW2_PCG:
            st->beta = (t[0] + st->qc) / st->rho;
            st->rho = t[0] + st->qc;
            break;
        // two-level with the coarse path on a second stream: the patch and coarse quadratic forms
        // land in qf / qc; the direction update forms beta = (qf + qc) / rho itself and the next
        // p.q reduction makes rho = qf + qc current (FIN_PQ2)
        case FIN_AFW2_QF_INIT:
            st->qf = t[0];
            st->tol2 = rtol * rtol * st->bb;
            st->flag = (st->rr <= st->tol2) ? FLAG_CONV : FLAG_RUN;
            break;
        case FIN_AFW2_QF: st->qf = t[0]; break;
        case FIN_PQ2:
            st->rho = st->qf + st->qc;
            if (st->iters < kLanczos) { st->lz[2 * st->iters] = st->rho; st->lz[2 * st->iters + 1] = t[0]; }
            st->pq = t[0];
            if (!(t[0] > 0.0)) st->flag = FLAG_BREAK;
            else st->alpha = st->rho / t[0];
            break;
    }
}

template <int NV>
__device__ __forceinline__ void fin_or_store(KState *st, int kind, const double *t, double rtol, int dist) {
    if (dist) {
#pragma unroll
        for (int i = 0; i < NV; ++i) st->red[i] = t[i];
    } else {
        apply_fin(st, kind, t, rtol);
    }
}

// distributed mode: the recurrence after the allreduce (a converged state stays frozen)
__global__ void k_fin(KState *st, int kind, double rtol) {
    const bool init = kind == FIN_BB || kind == FIN_RR || kind == FIN_PCG_INIT || kind == FIN_AFW_PCG_INIT ||
                      kind == FIN_AFW2_PCG_INIT || kind == FIN_AFW2_QF_INIT;
    if (!init && st->flag != FLAG_RUN) return;
    apply_fin(st, kind, st->red, rtol);
}

// pack the owned rows peers need: buf[k] = x[send_rows[k]]
template <int D>
__global__ void k_halo_pack(int64_t n, const int32_t *rows, const double *x, double *buf) {
    GRID_STRIDE(k, n) {
#pragma unroll
        for (int i = 0; i < D; ++i) buf[k * D + i] = x[(int64_t)rows[k] * D + i];
    }
}

// ------------------------------------------------------------------ matrix-free G (mf.cuh)
// q += G_mf x over this rank's cells (q pre-zeroed); REDUCE: p.q -> alpha (FIN_PQ)
template <int D, bool REDUCE>
__global__ void __launch_bounds__(kT, D == 2 ? 3 : 2) k_mf_spmv(MfView M, const double *x, double *q, int64_t nown, KState *st,
                                                double *partials, int dist, int pqkind) {
    if (REDUCE && st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    GRID_STRIDE(t, M.ncells) acc[0] += mf_cell<D>(M, t, x, q, nown);
    if (REDUCE)
        reduce_and_finish<1>(acc, partials, &st->tickets[1], [&](double *t) { fin_or_store<1>(st, pqkind, t, 0.0, dist); });
}

// The same operator with the per-slice factor stream staged through shared memory by the
// bulk-copy (TMA) engine: each warp owns a 2-stage ring; while it gathers x, computes and scatters
// slice k, the copy of slice k + 2 warps ahead is in flight, so the factor stream never waits
// behind the dependent id -> x gathers (the latency that bounded k_mf_spmv).
constexpr int kMfTmaWarps = 4;
template <int D>
constexpr int mf_tma_smem() { return kMfTmaWarps * (2 * MfSlice<D>::BYTES + 16); }

template <int D, bool REDUCE>
__global__ void __launch_bounds__(kMfTmaWarps * 32, D == 2 ? 5 : 4)
    k_mf_spmv_tma(MfView M, const double *x, double *q, int64_t nown, KState *st, double *partials, int dist, int pqkind) {
    if (REDUCE && st->flag != FLAG_RUN) return;
    extern __shared__ __align__(128) unsigned char mf_smem[];
    constexpr int SB = MfSlice<D>::BYTES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *ring = mf_smem + warp * (2 * SB + 16);
    uint64_t *bar = reinterpret_cast<uint64_t *>(ring + 2 * SB);
    const int64_t nsl = M.ncells >> 5;
    const int64_t w0 = (int64_t)blockIdx.x * kMfTmaWarps + warp, nw = (int64_t)gridDim.x * kMfTmaWarps;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
        if (w0 < nsl) mf_issue_slice<D>(M, w0, ring, &bar[0]);
        if (w0 + nw < nsl) mf_issue_slice<D>(M, w0 + nw, ring + SB, &bar[1]);
    }
    __syncwarp();
    double acc[1] = {0.0};
    int64_t k = 0;
    for (int64_t sl = w0; sl < nsl; sl += nw, ++k) {
        const int stg = (int)(k & 1);
        const unsigned par = (unsigned)((k >> 1) & 1);
        while (!mbar_try_wait(&bar[stg], par)) {
        }
        acc[0] += mf_cell_staged<D>(ring + stg * SB, lane, x, q, nown);
        __syncwarp();
        if (lane == 0 && sl + 2 * nw < nsl) {
            fence_proxy_async_smem();   // this warp's reads of the stage precede the copy over it
            mf_issue_slice<D>(M, sl + 2 * nw, ring + stg * SB, &bar[stg]);
        }
    }
    if (REDUCE)
        reduce_and_finish<1>(acc, partials, &st->tickets[1], [&](double *t) { fin_or_store<1>(st, pqkind, t, 0.0, dist); });
}

template <int D, bool REDUCE>
static int mf_tma_grid() {
    static thread_local int nb = 0;
    if (nb == 0) {
        CR_CUDA(cudaFuncSetAttribute(k_mf_spmv_tma<D, REDUCE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     mf_tma_smem<D>()));
        CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_mf_spmv_tma<D, REDUCE>, kMfTmaWarps * 32,
                                                              mf_tma_smem<D>()));
        if (nb < 1) nb = 1;
    }
    return num_sms() * nb;
}

// coarse setup: 32-cell slices with a face in a coarse cell that touches a node of `colour`
template <int D>
__global__ void k_mf_slice_flag(MfView M, CoarseView C, int colour, int64_t nslices, uint8_t *flag) {
    constexpr int NF = D + 1;
    for (int64_t sl = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); sl < nslices;
         sl += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int lane = threadIdx.x & 31;
        bool act = false;
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            const int32_t row = M.ids[sl * (NF * 32) + l * 32 + lane];
            if (row >= 0) {
                int ic[D];
                float xi[D];
                coarse_locate<D>(C.g, C.fx + (int64_t)row * D, ic, xi);
                act = act || coarse_cell_active<D>(ic, colour);
            }
        }
        act = __any_sync(0xffffffffu, act);
        if (lane == 0) flag[sl] = act ? 1 : 0;
    }
}

// the colours (base-5 digits of the node indices) of the corners of every face's coarse cell, per
// 32-cell slice, as a 128-bit mask (computed once; the colour passes then test one bit)
template <int D>
__global__ void k_mf_slice_colours(MfView M, CoarseView C, int64_t nslices, unsigned *mask) {
    constexpr int NF = D + 1;
    for (int64_t sl = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); sl < nslices;
         sl += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int lane = threadIdx.x & 31;
        unsigned m[4] = {0u, 0u, 0u, 0u};
        for (int l = 0; l < NF; ++l) {
            const int32_t row = M.ids[sl * (NF * 32) + l * 32 + lane];
            if (row < 0) continue;
            int ic[D];
            float xi[D];
            coarse_locate<D>(C.g, C.fx + (int64_t)row * D, ic, xi);
            for (int n = 0; n < (1 << D); ++n) {
                int col = 0, mul = 1;
                for (int i = 0; i < D; ++i) {
                    col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
                    mul *= 5;
                }
                m[col >> 5] |= 1u << (col & 31);
            }
        }
        for (int w = 0; w < 4; ++w) {
            const unsigned v = __reduce_or_sync(0xffffffffu, m[w]);
            if (lane == 0) mask[sl * 4 + w] = v;
        }
    }
}

__global__ void k_mf_flag_colour(const unsigned *mask, int64_t nslices, int colour, uint8_t *flag) {
    for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nslices; sl += (int64_t)gridDim.x * blockDim.x)
        flag[sl] = (mask[sl * 4 + (colour >> 5)] >> (colour & 31)) & 1u;
}

// q += G_mf x over the listed slices only (coarse setup: x vanishes on every other cell)
template <int D>
__global__ void __launch_bounds__(kT, D == 2 ? 3 : 2) k_mf_spmv_slices(MfView M, const int32_t *slices, const int64_t *nact,
                                                       const double *x, double *q, int64_t nown) {
    const int64_t n = *nact * 32;
    GRID_STRIDE(t, n) {
        const int64_t tt = (int64_t)slices[t >> 5] * 32 + (t & 31);
        mf_cell<D>(M, tt, x, q, nown);
    }
}

// the same for ncol right-hand sides x + c xs -> q + c xs (coarse setup: the D^2 columns of a colour);
// the cell's factors are loaded once for all of them
template <int D>
__global__ void __launch_bounds__(kT, D == 2 ? 3 : 2) k_mf_spmv_slices_all(MfView M, const int32_t *slices, const int64_t *nact,
                                                           const double *x, double *q, int64_t xs, int ncol, int64_t nown) {
    using LY = MfLayout<D>;
    constexpr int NF = LY::NF, NT = LY::NT;
    const int64_t n = *nact * 32;
    GRID_STRIDE(t, n) {
        const int64_t tt = (int64_t)slices[t >> 5] * 32 + (t & 31);
        const int64_t slice = tt >> 5;
        const int lane = (int)(tt & 31);
        const int32_t *ip = M.ids + slice * (NF * 32) + lane;
        const double *vp = M.v + slice * ((int64_t)LY::NE * 32) + lane;
        int id[NF];
        unsigned nbc[NF];
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            id[l] = ip[l * 32];
            nbc[l] = M.nb[slice * (NF * 32) + l * 32 + lane];
        }
        const unsigned sg = M.sg[tt];
        const double c = vp[0];
        double T[NT], u[D][NF];
#pragma unroll
        for (int e = 0; e < NT; ++e) T[e] = vp[(1 + e) * 32];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int l = 0; l < NF; ++l) u[i][l] = vp[(1 + NT + i * NF + l) * 32];
        for (int col = 0; col < ncol; ++col) mf_cell_core<D>(id, sg, c, T, u, nbc, lane, x + col * xs, q + col * xs, nown);
    }
}

// coarse setup without materialising Z: for the listed slices, q = [G z_(k, l)] for the D^2 columns of
// `colour`, interleaved per row (q[row qs + (k D + l) D + i], qs = D^3), the input z_(k,l) at face
// sigma = e_k s_sigma a_sigma^(l) (s_sigma = sum of the colour's hat weights at x_sigma) computed from the
// coarse view's row data on the fly
template <int D>
__global__ void __launch_bounds__(kT, D == 2 ? 2 : 1) k_mf_spmv_colour(MfView M, CoarseView C, int colour,
                                                       const int32_t *slices, const int64_t *nact, double *q, int64_t qs,
                                                       int64_t nown) {
    using LY = MfLayout<D>;
    constexpr int NF = LY::NF, NT = LY::NT, NN = 1 << D;
    const int64_t n = *nact * 32;
    GRID_STRIDE(t, n) {
        const int64_t tt = (int64_t)slices[t >> 5] * 32 + (t & 31);
        const int64_t slice = tt >> 5;
        const int lane = (int)(tt & 31);
        const int32_t *ip = M.ids + slice * (NF * 32) + lane;
        const double *vp = M.v + slice * ((int64_t)LY::NE * 32) + lane;
        int id[NF];
        unsigned nbc[NF];
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            id[l] = ip[l * 32];
            nbc[l] = M.nb[slice * (NF * 32) + l * 32 + lane];
        }
        const unsigned sg = M.sg[tt];
        double cs[NF], sw[NF], fa[NF][D];
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            cs[l] = ((sg >> l) & 1u) ? -1.0 : 1.0;
            sw[l] = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) fa[l][i] = 0.0;
            if (id[l] >= 0) {
                const float *x = C.fx + (int64_t)id[l] * D;
                int ic[D];
                float xi[D];
                coarse_locate<D>(C.g, x, ic, xi);
                double w[NN];
                coarse_weights<D>(C.g, x, w);
                for (int nn = 0; nn < NN; ++nn) {
                    int col = 0, mul = 1;
                    for (int i = 0; i < D; ++i) {
                        col += ((ic[i] + ((nn >> i) & 1)) % 5) * mul;
                        mul *= 5;
                    }
                    if (col == colour) sw[l] += w[nn];
                }
#pragma unroll
                for (int i = 0; i < D; ++i) fa[l][i] = (double)C.fa[(int64_t)id[l] * D + i];
            }
        }
        const double c = vp[0];
        double T[NT], u[D][NF];
#pragma unroll
        for (int e = 0; e < NT; ++e) T[e] = vp[(1 + e) * 32];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int l = 0; l < NF; ++l) u[i][l] = vp[(1 + NT + i * NF + l) * 32];
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int l2 = 0; l2 < D; ++l2) {
                double xk[NF];
#pragma unroll
                for (int l = 0; l < NF; ++l) xk[l] = cs[l] * sw[l] * fa[l][l2];
                mf_cell_core_1c<D>(id, cs, xk, k, c, T, u, nbc, lane, q + (int64_t)(k * D + l2) * D, nown, qs);
            }
    }
}

// r = b - q, |r|^2 (FIN_RR)
__global__ void __launch_bounds__(kT) k_resid_vec(int64_t N, const double *b, const double *q, double *r, KState *st,
                                                  double *partials, int dist) {
    double acc[1] = {0.0};
    GRID_STRIDE(i, N) {
        const double ri = b[i] - q[i];
        r[i] = ri;
        acc[0] = fma(ri, ri, acc[0]);
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[7], [&](double *t) { fin_or_store<1>(st, FIN_RR, t, 0.0, dist); });
}

// ------------------------------------------------------------------ generic
// q = G x ; r = b - q ; partial |r|^2  (true residual)
template <int D>
__global__ void __launch_bounds__(kT) k_true_residual(EllView<D> G, const double *x, const double *b, double *r,
                                                      KState *st, double *partials, int dist) {
    double acc[1] = {0.0};
    GRID_STRIDE(row, G.nrows) {
        double y[D];
        spmv_row<D>(G, row, x, y);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double ri = b[row * D + i] - y[i];
            r[row * D + i] = ri;
            acc[0] += ri * ri;
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[7], [&](double *t) { fin_or_store<1>(st, FIN_RR, t, 0.0, dist); });
}

__global__ void k_norm2(const double *a, int64_t n, KState *st, double *partials, int dist) {
    double acc[1] = {0.0};
    GRID_STRIDE(i, n) acc[0] += a[i] * a[i];
    reduce_and_finish<1>(acc, partials, &st->tickets[6], [&](double *t) { fin_or_store<1>(st, FIN_BB, t, 0.0, dist); });
}

// ------------------------------------------------------------------ PCG
template <int D, int PREC>
__global__ void __launch_bounds__(kT) k_pcg_init(int64_t nrows, const double *b, const double *r, double *p,
                                                 const double *M, double rtol, KState *st, double *partials, int dist) {
    // r already holds b - G x (k_true_residual); z = M r ; p = z ; rho = r.z
    double acc[2] = {0.0, 0.0};
    GRID_STRIDE(row, nrows) {
        double rv[D], zv[D];
        ld<D>(r, row, rv);
        apply_prec<D, PREC>(M, row, rv, zv);
        stv<D>(p, row, zv);
#pragma unroll
        for (int i = 0; i < D; ++i) { acc[0] += rv[i] * zv[i]; acc[1] += rv[i] * rv[i]; }
    }
    reduce_and_finish<2>(acc, partials, &st->tickets[0], [&](double *t) { fin_or_store<2>(st, FIN_PCG_INIT, t, rtol, dist); });
}

template <int D>
__global__ void __launch_bounds__(kT) k_pcg_spmv(EllView<D> G, const double *p, double *q, KState *st, double *partials, int dist,
                                                int pqkind = FIN_PQ) {
    if (st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    GRID_STRIDE(row, G.nrows) {
        double y[D];
        spmv_row<D>(G, row, p, y);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            q[row * D + i] = y[i];
            acc[0] += p[row * D + i] * y[i];
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[1], [&](double *t) { fin_or_store<1>(st, pqkind, t, 0.0, dist); });
}

template <int D, int PREC>
__global__ void __launch_bounds__(kT) k_pcg_update(int64_t nrows, double *x, double *r, const double *p, const double *q,
                                                   const double *M, KState *st, double *partials, int dist) {
    if (st->flag != FLAG_RUN) return;
    const double alpha = st->alpha;
    double acc[2] = {0.0, 0.0};
    GRID_STRIDE(row, nrows) {
        double rv[D], zv[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            x[row * D + i] = fma(alpha, p[row * D + i], x[row * D + i]);
            rv[i] = fma(-alpha, q[row * D + i], r[row * D + i]);
            r[row * D + i] = rv[i];
        }
        apply_prec<D, PREC>(M, row, rv, zv);
#pragma unroll
        for (int i = 0; i < D; ++i) { acc[0] += rv[i] * zv[i]; acc[1] += rv[i] * rv[i]; }
    }
    reduce_and_finish<2>(acc, partials, &st->tickets[2], [&](double *t) { fin_or_store<2>(st, FIN_UPD_PC, t, 0.0, dist); });
}

// Jacobi PCG, flat double2 form: x += alpha p ; r -= alpha q ; z = dinv r ; r.z, r.r
__global__ void __launch_bounds__(kT, 4) k_pcg_update_jac(int64_t N, double *__restrict__ x, double *__restrict__ r,
                                                       const double *__restrict__ p, const double *__restrict__ q,
                                                       const double *__restrict__ dinv, KState *st, double *partials,
                                                       int dist) {
    if (st->flag != FLAG_RUN) return;
    const double alpha = st->alpha;
    double acc[2] = {0.0, 0.0};
    const int64_t n2 = N >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    double2 *x2 = reinterpret_cast<double2 *>(x), *r2 = reinterpret_cast<double2 *>(r);
    const double2 *p2 = reinterpret_cast<const double2 *>(p), *q2 = reinterpret_cast<const double2 *>(q);
    const double2 *d2 = reinterpret_cast<const double2 *>(dinv);
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 pv[4], qv[4], xv[4], rv[4], dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pv[u] = __ldcs(p2 + i + u * stride);
            qv[u] = __ldcs(q2 + i + u * stride);
            xv[u] = __ldcs(x2 + i + u * stride);
            rv[u] = __ldcs(r2 + i + u * stride);
            dv[u] = d2[i + u * stride];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xv[u].x = fma(alpha, pv[u].x, xv[u].x);
            xv[u].y = fma(alpha, pv[u].y, xv[u].y);
            rv[u].x = fma(-alpha, qv[u].x, rv[u].x);
            rv[u].y = fma(-alpha, qv[u].y, rv[u].y);
            acc[0] = fma(rv[u].x, dv[u].x * rv[u].x, acc[0]);
            acc[0] = fma(rv[u].y, dv[u].y * rv[u].y, acc[0]);
            acc[1] = fma(rv[u].x, rv[u].x, acc[1]);
            acc[1] = fma(rv[u].y, rv[u].y, acc[1]);
            __stcs(x2 + i + u * stride, xv[u]);
            r2[i + u * stride] = rv[u];
        }
    }
    for (; i < n2; i += stride) {
        double2 pv = p2[i], qv = q2[i], xv = x2[i], rv = r2[i], dv = d2[i];
        xv.x = fma(alpha, pv.x, xv.x);
        xv.y = fma(alpha, pv.y, xv.y);
        rv.x = fma(-alpha, qv.x, rv.x);
        rv.y = fma(-alpha, qv.y, rv.y);
        acc[0] = fma(rv.x, dv.x * rv.x, acc[0]);
        acc[0] = fma(rv.y, dv.y * rv.y, acc[0]);
        acc[1] = fma(rv.x, rv.x, acc[1]);
        acc[1] = fma(rv.y, rv.y, acc[1]);
        x2[i] = xv;
        r2[i] = rv;
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t k = N - 1;
        x[k] = fma(alpha, p[k], x[k]);
        const double rk = fma(-alpha, q[k], r[k]);
        r[k] = rk;
        acc[0] = fma(rk, dinv[k] * rk, acc[0]);
        acc[1] = fma(rk, rk, acc[1]);
    }
    reduce_and_finish<2>(acc, partials, &st->tickets[2], [&](double *t) { fin_or_store<2>(st, FIN_UPD_PC, t, 0.0, dist); });
}

// Jacobi PCG, flat double2 form: p = dinv r + beta p
__global__ void __launch_bounds__(kT) k_pcg_pdir_jac(int64_t N, double *__restrict__ p, const double *__restrict__ r,
                                                     const double *__restrict__ dinv, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double beta = st->beta;
    const int64_t n2 = N >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    double2 *p2 = reinterpret_cast<double2 *>(p);
    const double2 *r2 = reinterpret_cast<const double2 *>(r), *d2 = reinterpret_cast<const double2 *>(dinv);
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 pv[4], rv[4], dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pv[u] = __ldcs(p2 + i + u * stride);
            rv[u] = r2[i + u * stride];
            dv[u] = d2[i + u * stride];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pv[u].x = fma(beta, pv[u].x, dv[u].x * rv[u].x);
            pv[u].y = fma(beta, pv[u].y, dv[u].y * rv[u].y);
            p2[i + u * stride] = pv[u];
        }
    }
    for (; i < n2; i += stride) {
        double2 pv = p2[i], rv = r2[i], dv = d2[i];
        pv.x = fma(beta, pv.x, dv.x * rv.x);
        pv.y = fma(beta, pv.y, dv.y * rv.y);
        p2[i] = pv;
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[N - 1] = fma(beta, p[N - 1], dinv[N - 1] * r[N - 1]);
}

template <int D, int PREC>
__global__ void __launch_bounds__(kT) k_pcg_pdir(int64_t nrows, double *p, const double *r, const double *M, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double beta = st->beta;
    GRID_STRIDE(row, nrows) {
        double rv[D], zv[D];
        ld<D>(r, row, rv);
        apply_prec<D, PREC>(M, row, rv, zv);
#pragma unroll
        for (int i = 0; i < D; ++i) p[row * D + i] = fma(beta, p[row * D + i], zv[i]);
    }
}

// ------------------------------------------------------------------ MINRES scalar recurrences
// gamma_1 = sqrt(v_1^t M v_1) and the Givens state (called by the last block of a reduction)
__device__ __forceinline__ void minres_start(KState *st, double vMv) {
    double gm = sqrt(fmax(vMv, 0.0));
    st->gamma = gm;
    st->gamma_old = 1.0;
    st->eta = gm;
    st->eta0 = gm;
    st->s = st->s_old = 0.0;
    st->c = st->c_old = 1.0;
    st->flag = (gm == 0.0) ? FLAG_CONV : FLAG_RUN;
}

// new gamma = sqrt(v_{j+1}^t M v_{j+1}); QR of the tridiagonal by Givens rotations
__device__ __forceinline__ void minres_givens(KState *st, double vMv) {
    const double gn = sqrt(fmax(vMv, 0.0));
    const double gmo = st->gamma, dlo = st->delta;
    const double a0 = st->c * dlo - st->c_old * st->s * gmo;
    const double a1 = sqrt(a0 * a0 + gn * gn);
    const double a2 = st->s * dlo + st->c_old * st->c * gmo;
    const double a3 = st->s_old * gmo;
    const double cn = a0 / a1, sn = gn / a1;
    st->a1 = a1; st->a2 = a2; st->a3 = a3; st->cn = cn;
    st->eta_w = st->eta;
    st->gz = gmo;
    st->eta = -sn * st->eta;
    st->gamma_old = gmo;
    st->gamma = gn;
    st->c_old = st->c; st->c = cn;
    st->s_old = st->s; st->s = sn;
    st->iters += 1;
    if (gn == 0.0) st->flag = FLAG_CONV;          // exact invariant subspace
}

// ------------------------------------------------------------------ MINRES (preconditioned, SPD M)
// Paige-Saunders recurrences in the Elman-Silvester-Wathen form (oracle/krylov.py minres):
// z_j = M v_j / gamma_j; delta = z_j^t G z_j; v_{j+1} = G z_j - delta/gamma v_j - gamma/gamma_old v_{j-1}
template <int D>
__global__ void __launch_bounds__(kT) k_minres_init(int64_t nrows, const double *v, double *z, const double *M,
                                                    double *w, double *w2, double *vold, KState *st, double *partials) {
    double acc[1] = {0.0};
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double vi = v[row * D + i], zi = M[row * D + i] * vi;
            z[row * D + i] = zi;
            w[row * D + i] = 0.0;
            w2[row * D + i] = 0.0;
            vold[row * D + i] = 0.0;
            acc[0] += zi * vi;
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[0], [&](double *t) { minres_start(st, t[0]); });
}

template <int D>
__global__ void __launch_bounds__(kT) k_minres_spmv(EllView<D> G, const double *z, double *q, KState *st, double *partials) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->wx_iter = st->iters;   // previous w/x update has completed
    if (st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    GRID_STRIDE(row, G.nrows) {
        double y[D];
        spmv_row<D>(G, row, z, y);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            q[row * D + i] = y[i];
            acc[0] += z[row * D + i] * y[i];
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[1], [&](double *t) {
        st->delta = t[0] / (st->gamma * st->gamma);
    });
}

// v_new (written over v_old) = q/gamma - delta/gamma v - gamma/gamma_old v_old ; z_new = M v_new
template <int D>
__global__ void __launch_bounds__(kT) k_minres_lanczos(int64_t nrows, const double *q, const double *v, double *vold_new,
                                                       double *znew, const double *M, KState *st, double *partials) {
    if (st->flag != FLAG_RUN) return;
    const double gm = st->gamma, go = st->gamma_old, dl = st->delta;
    const double c1 = 1.0 / gm, c2 = dl / gm, c3 = gm / go;
    double acc[1] = {0.0};
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            double vn = q[k] * c1 - c2 * v[k] - c3 * vold_new[k];
            double zn = M[k] * vn;
            vold_new[k] = vn;
            znew[k] = zn;
            acc[0] += zn * vn;
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[2], [&](double *t) { minres_givens(st, t[0]); });
}

// w_new (written over w_old) = (z/gz - a3 w_old - a2 w)/a1 ; x += cn eta_w w_new
template <int D>
__global__ void __launch_bounds__(kT) k_minres_wx(int64_t nrows, const double *z, const double *w, double *wold_new,
                                                  double *x, const KState *st) {
    if (st->flag == FLAG_BREAK) return;
    if (st->wx_iter >= st->iters) return;   // no pending Lanczos step
    const double inv_gz = 1.0 / st->gz, a1 = st->a1, a2 = st->a2, a3 = st->a3, f = st->cn * st->eta_w;
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            double wn = (z[k] * inv_gz - a3 * wold_new[k] - a2 * w[k]) / a1;
            wold_new[k] = wn;
            x[k] = fma(f, wn, x[k]);
        }
    }
}

// ------------------------------------------------------------------ patch (AFW) preconditioner
// What the last block does with q = sum_p r_p^t B_p^{-1} r_p  (= r^t M^{-1} r)
enum { AFW_PCG_INIT = 0, AFW_PCG = 1, AFW_MINRES_INIT = 2, AFW_MINRES = 3, AFW_PCG2_INIT = 4, AFW_PCG2 = 5,
       AFW_MINRES2_INIT = 6, AFW_MINRES2 = 7 };

// zs (per face slot) = patch contributions of M^{-1} r
template <int D, int SLOTS, int KMAX, bool SYM, int WHAT>
__global__ void __launch_bounds__(kT, 4) k_afw_apply(AfwView A, const double *r, double *zs, double rtol, KState *st,
                                                  double *partials, int dist) {
    if (WHAT != AFW_PCG_INIT && WHAT != AFW_MINRES_INIT && WHAT != AFW_PCG2_INIT && WHAT != AFW_MINRES2_INIT &&
        st->flag != FLAG_RUN)
        return;
    double acc[1] = {0.0};
    const int64_t nt = ((A.npatch + 31) >> 5) * 32 * D;     // one thread per (patch, component)
    GRID_STRIDE(t, nt) acc[0] += afw_patch_comp<D, SLOTS, KMAX, SYM>(A, t, r, zs);
    reduce_and_finish<1>(acc, partials, &st->tickets[3], [&](double *t) {
        if (WHAT == AFW_PCG_INIT) {
            fin_or_store<1>(st, FIN_AFW_PCG_INIT, t, rtol, dist);
        } else if (WHAT == AFW_PCG) {
            fin_or_store<1>(st, FIN_AFW_PCG, t, rtol, dist);
        } else if (WHAT == AFW_PCG2_INIT) {
            fin_or_store<1>(st, FIN_AFW2_QF_INIT, t, rtol, dist);
        } else if (WHAT == AFW_PCG2) {
            fin_or_store<1>(st, FIN_AFW2_QF, t, rtol, dist);
        } else if (WHAT == AFW_MINRES_INIT) {
            minres_start(st, t[0]);
        } else if (WHAT == AFW_MINRES2_INIT) {   // v^t M v = patch part + coarse part c^t |E|^-1 c
            minres_start(st, t[0] + st->qc);
        } else if (WHAT == AFW_MINRES2) {
            minres_givens(st, t[0] + st->qc);
        } else {
            minres_givens(st, t[0]);
        }
    });
}

// the shared-block variant (afw_patch_shared): one thread per patch for all components
template <int D, int SLOTS, int KMAX, int WHAT>
__global__ void __launch_bounds__(kT, 2) k_afw_apply_sh(AfwView A, const double *r, double *zs, double rtol, KState *st,
                                                     double *partials, int dist) {
    if (WHAT != AFW_PCG_INIT && WHAT != AFW_PCG2_INIT && st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    const int64_t nt = ((A.npatch + 31) >> 5) * 32;
    GRID_STRIDE(t, nt) acc[0] += afw_patch_shared<D, SLOTS, KMAX>(A, t, r, zs);
    reduce_and_finish<1>(acc, partials, &st->tickets[3], [&](double *t) {
        if (WHAT == AFW_PCG_INIT) fin_or_store<1>(st, FIN_AFW_PCG_INIT, t, rtol, dist);
        else if (WHAT == AFW_PCG) fin_or_store<1>(st, FIN_AFW_PCG, t, rtol, dist);
        else if (WHAT == AFW_PCG2_INIT) fin_or_store<1>(st, FIN_AFW2_QF_INIT, t, rtol, dist);
        else if (WHAT == AFW_PCG2) fin_or_store<1>(st, FIN_AFW2_QF, t, rtol, dist);
    });
}

// the shared-block variant split over components (afw_patch_split): blocks of 4 slices x D warps
constexpr int kAfwSpb = 4;
template <int D, int SLOTS, int KMAX, int WHAT>
__global__ void __launch_bounds__(32 * D * kAfwSpb, D == 3 ? 2 : 3) k_afw_apply_sc(AfwView A, const double *r, double *zs,
                                                                                 double rtol, KState *st, double *partials,
                                                                                 int dist) {
    if (WHAT != AFW_PCG_INIT && WHAT != AFW_PCG2_INIT && st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = warp % D;
    const int64_t nslices = (A.npatch + 31) >> 5;
    for (int64_t slice = (int64_t)blockIdx.x * kAfwSpb + warp / D; slice < nslices; slice += (int64_t)gridDim.x * kAfwSpb)
        acc[0] += afw_patch_split<D, SLOTS, KMAX>(A, slice, i, lane, r, zs);
    reduce_and_finish<1>(acc, partials, &st->tickets[3], [&](double *t) {
        if (WHAT == AFW_PCG_INIT) fin_or_store<1>(st, FIN_AFW_PCG_INIT, t, rtol, dist);
        else if (WHAT == AFW_PCG) fin_or_store<1>(st, FIN_AFW_PCG, t, rtol, dist);
        else if (WHAT == AFW_PCG2_INIT) fin_or_store<1>(st, FIN_AFW2_QF_INIT, t, rtol, dist);
        else if (WHAT == AFW_PCG2) fin_or_store<1>(st, FIN_AFW2_QF, t, rtol, dist);
    });
}

// x += alpha p (XUPD; else the direction update does it: k_pcg_pdir_afw*) ; r -= alpha q ; |r|^2
// (convergence).  Flat over the N = D*nrows entries in 16-byte double2 units, 4 independent units
// in flight per thread (memory-level parallelism).
template <bool XUPD>
__global__ void __launch_bounds__(kT, 4) k_pcg_update_r(int64_t N, double *__restrict__ x, double *__restrict__ r,
                                                     const double *__restrict__ p, const double *__restrict__ q,
                                                     KState *st, double *partials, int dist) {
    if (st->flag != FLAG_RUN) return;
    const double alpha = st->alpha;
    double acc[1] = {0.0};
    const int64_t n2 = N >> 1, stride = (int64_t)gridDim.x * blockDim.x;
    double2 *x2 = reinterpret_cast<double2 *>(x), *r2 = reinterpret_cast<double2 *>(r);
    const double2 *p2 = reinterpret_cast<const double2 *>(p), *q2 = reinterpret_cast<const double2 *>(q);
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n2; i += 4 * stride) {
        double2 pv[4], qv[4], xv[4], rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (XUPD) {
                pv[u] = __ldcs(p2 + i + u * stride);
                xv[u] = __ldcs(x2 + i + u * stride);
            }
            qv[u] = __ldcs(q2 + i + u * stride);
            rv[u] = __ldcs(r2 + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (XUPD) {
                xv[u].x = fma(alpha, pv[u].x, xv[u].x);
                xv[u].y = fma(alpha, pv[u].y, xv[u].y);
                __stcs(x2 + i + u * stride, xv[u]);
            }
            rv[u].x = fma(-alpha, qv[u].x, rv[u].x);
            rv[u].y = fma(-alpha, qv[u].y, rv[u].y);
            acc[0] = fma(rv[u].x, rv[u].x, acc[0]);
            acc[0] = fma(rv[u].y, rv[u].y, acc[0]);
            r2[i + u * stride] = rv[u];
        }
    }
    for (; i < n2; i += stride) {
        double2 qv = q2[i], rv = r2[i];
        if (XUPD) {
            double2 pv = p2[i], xv = x2[i];
            xv.x = fma(alpha, pv.x, xv.x);
            xv.y = fma(alpha, pv.y, xv.y);
            x2[i] = xv;
        }
        rv.x = fma(-alpha, qv.x, rv.x);
        rv.y = fma(-alpha, qv.y, rv.y);
        acc[0] = fma(rv.x, rv.x, acc[0]);
        acc[0] = fma(rv.y, rv.y, acc[0]);
        r2[i] = rv;
    }
    if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t k = N - 1;
        if (XUPD) x[k] = fma(alpha, p[k], x[k]);
        const double rk = fma(-alpha, q[k], r[k]);
        r[k] = rk;
        acc[0] = fma(rk, rk, acc[0]);
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[2], [&](double *t) { fin_or_store<1>(st, FIN_UPD_R, t, 0.0, dist); });
}

// x += alpha p of the iteration whose residual update met the tolerance (its direction update,
// which carries the x update, returned early)
__global__ void k_pcg_x_final(int64_t N, double *__restrict__ x, const double *__restrict__ p, const KState *st) {
    const double alpha = st->alpha;
    GRID_STRIDE(i, N) x[i] = fma(alpha, p[i], x[i]);
}

// p = z + beta p, z = sum of the slot contributions (beta = 0: p = z); x (non-null): x += alpha p
// first, with the old p (the iteration's solution update, moved here from k_pcg_update_r: p is read
// here anyway)
template <int D, int SLOTS>
__global__ void __launch_bounds__(kT) k_pcg_pdir_afw(int64_t nrows, double *__restrict__ p, const double *__restrict__ zs,
                                                     const KState *st, double *__restrict__ x) {
    if (st->flag != FLAG_RUN) return;
    const double beta = st->beta, alpha = st->alpha;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (D == 2 && !x) {
        double2 *p2 = reinterpret_cast<double2 *>(p);
        int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        for (; row + 3 * stride < nrows; row += 4 * stride) {
            double2 pv[4];
            double z0[4], z1[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t r = row + u * stride;
                pv[u] = __ldcs(p2 + r);
                z0[u] = __ldcs(zs + r);
                z1[u] = __ldcs(zs + nrows + r);
#pragma unroll
                for (int sl = 1; sl < SLOTS; ++sl) {
                    z0[u] += __ldcs(zs + (int64_t)(sl * 2) * nrows + r);
                    z1[u] += __ldcs(zs + (int64_t)(sl * 2 + 1) * nrows + r);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                pv[u].x = (beta == 0.0) ? z0[u] : fma(beta, pv[u].x, z0[u]);
                pv[u].y = (beta == 0.0) ? z1[u] : fma(beta, pv[u].y, z1[u]);
                p2[row + u * stride] = pv[u];
            }
        }
        for (; row < nrows; row += stride) {
            double z[2];
            afw_sum<2, SLOTS>(zs, nrows, row, z);
            double2 pv = p2[row];
            pv.x = (beta == 0.0) ? z[0] : fma(beta, pv.x, z[0]);
            pv.y = (beta == 0.0) ? z[1] : fma(beta, pv.y, z[1]);
            p2[row] = pv;
        }
    } else {
        GRID_STRIDE(row, nrows) {
            double z[D];
            afw_sum<D, SLOTS>(zs, nrows, row, z);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const double po = p[row * D + i];
                if (x) x[row * D + i] = fma(alpha, po, x[row * D + i]);
                p[row * D + i] = (beta == 0.0) ? z[i] : fma(beta, po, z[i]);
            }
        }
    }
}

// two-level: p = (sum of the slot contributions) + Z y + beta p
template <int D, int SLOTS>
__global__ void __launch_bounds__(kT) k_pcg_pdir_afw2(int64_t nrows, double *__restrict__ p, const double *__restrict__ zs,
                                                      CoarseView C, const double *__restrict__ y, const KState *st,
                                                      int first, double *__restrict__ x) {
    if (st->flag != FLAG_RUN) return;
    const double beta = first ? 0.0 : (st->qf + st->qc) / st->rho;
    const double alpha = st->alpha;
    GRID_STRIDE(row, nrows) {
        double z[D], zc[D];
        afw_sum<D, SLOTS>(zs, nrows, row, z);
        coarse_prolong<D>(C, row, y, zc);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const double zi = z[i] + zc[i];
            const double po = p[row * D + i];
            if (x) x[row * D + i] = fma(alpha, po, x[row * D + i]);
            p[row * D + i] = (beta == 0.0) ? zi : fma(beta, po, zi);
        }
    }
}

// z = sum of the slot contributions (MINRES); `guard` skips after convergence
template <int D, int SLOTS>
__global__ void __launch_bounds__(kT) k_afw_zsum(int64_t nrows, double *z, const double *zs, const KState *st, int guard) {
    if (guard && st->flag != FLAG_RUN) return;
    GRID_STRIDE(row, nrows) {
        double zv[D];
        afw_sum<D, SLOTS>(zs, nrows, row, zv);
#pragma unroll
        for (int i = 0; i < D; ++i) z[row * D + i] = zv[i];
    }
}

// z = sum of the slot contributions + Z y (MINRES with the coarse |E|^-1 part); `guard` as k_afw_zsum
template <int D, int SLOTS>
__global__ void __launch_bounds__(kT) k_afw_zsum2(int64_t nrows, double *z, const double *zs, CoarseView C,
                                                  const double *__restrict__ y, const KState *st, int guard) {
    if (guard && st->flag != FLAG_RUN) return;
    GRID_STRIDE(row, nrows) {
        double zv[D], zc[D];
        afw_sum<D, SLOTS>(zs, nrows, row, zv);
        coarse_prolong<D>(C, row, y, zc);
#pragma unroll
        for (int i = 0; i < D; ++i) z[row * D + i] = zv[i] + zc[i];
    }
}

// MINRES Lanczos vector only: v_new (over v_old) = q/gamma - delta/gamma v - gamma/gamma_old v_old
template <int D>
__global__ void __launch_bounds__(kT) k_minres_lanczos_v(int64_t nrows, const double *q, const double *v, double *vold_new,
                                                         const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double gm = st->gamma, go = st->gamma_old, dl = st->delta;
    const double c1 = 1.0 / gm, c2 = dl / gm, c3 = gm / go;
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            vold_new[k] = q[k] * c1 - c2 * v[k] - c3 * vold_new[k];
        }
    }
}

__global__ void k_zero3(int64_t n, double *a, double *b, double *c) {
    GRID_STRIDE(i, n) { a[i] = 0.0; b[i] = 0.0; c[i] = 0.0; }
}

// ------------------------------------------------------------------ BiCGStab (right Jacobi)
template <int D>
__global__ void __launch_bounds__(kT) k_bicg_init(int64_t nrows, const double *r, double *rhat, double *p, double *v,
                                                  double rtol, KState *st, double *partials) {
    double acc[1] = {0.0};
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            rhat[k] = r[k];
            p[k] = 0.0;
            v[k] = 0.0;
            acc[0] += r[k] * r[k];
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[0], [&](double *t) {
        st->rho = 1.0; st->alpha = 1.0; st->omega = 1.0;
        st->rho_new = t[0];
        st->rr = t[0];
        st->tol2 = rtol * rtol * st->bb;
        st->flag = (t[0] <= st->tol2) ? FLAG_CONV : (t[0] == 0.0 ? FLAG_BREAK : FLAG_RUN);
    });
}

template <int D>
__global__ void __launch_bounds__(kT) k_bicg_pdir(int64_t nrows, const double *r, double *p, const double *v,
                                                  double *y, const double *M, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double beta = (st->rho_new / st->rho) * (st->alpha / st->omega), om = st->omega;
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            double pk = r[k] + beta * (p[k] - om * v[k]);
            p[k] = pk;
            y[k] = M[k] * pk;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kT) k_bicg_spmv1(EllView<D> G, const double *y, double *v, const double *rhat,
                                                   KState *st, double *partials) {
    if (st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    GRID_STRIDE(row, G.nrows) {
        double o[D];
        spmv_row<D>(G, row, y, o);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            v[row * D + i] = o[i];
            acc[0] += rhat[row * D + i] * o[i];
        }
    }
    reduce_and_finish<1>(acc, partials, &st->tickets[1], [&](double *t) {
        st->rv = t[0];
        if (t[0] == 0.0) st->flag = FLAG_BREAK;
        else st->alpha = st->rho_new / t[0];
    });
}

template <int D>
__global__ void __launch_bounds__(kT) k_bicg_s(int64_t nrows, double *r, const double *v, double *z, const double *M,
                                               const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double al = st->alpha;
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            double sk = fma(-al, v[k], r[k]);
            r[k] = sk;                 // r now holds s
            z[k] = M[k] * sk;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kT) k_bicg_spmv2(EllView<D> G, const double *z, double *t, const double *s,
                                                   KState *st, double *partials) {
    if (st->flag != FLAG_RUN) return;
    double acc[2] = {0.0, 0.0};
    GRID_STRIDE(row, G.nrows) {
        double o[D];
        spmv_row<D>(G, row, z, o);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            t[row * D + i] = o[i];
            acc[0] += o[i] * s[row * D + i];
            acc[1] += o[i] * o[i];
        }
    }
    reduce_and_finish<2>(acc, partials, &st->tickets[3], [&](double *t2) {
        st->ts = t2[0];
        st->tt = t2[1];
        st->omega = t2[1] > 0.0 ? t2[0] / t2[1] : 0.0;
    });
}

template <int D>
__global__ void __launch_bounds__(kT) k_bicg_xr(int64_t nrows, double *x, double *r, const double *y, const double *z,
                                                const double *t, const double *rhat, KState *st, double *partials) {
    if (st->flag != FLAG_RUN) return;
    const double al = st->alpha, om = st->omega;
    double acc[2] = {0.0, 0.0};
    GRID_STRIDE(row, nrows) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const int64_t k = row * D + i;
            x[k] = x[k] + al * y[k] + om * z[k];
            double rk = fma(-om, t[k], r[k]);
            r[k] = rk;
            acc[0] += rhat[k] * rk;
            acc[1] += rk * rk;
        }
    }
    reduce_and_finish<2>(acc, partials, &st->tickets[4], [&](double *t2) {
        st->iters += 1;
        st->rho = st->rho_new;
        st->rho_new = t2[0];
        st->rr = t2[1];
        if (t2[1] <= st->tol2) st->flag = FLAG_CONV;
        else if (t2[0] == 0.0 || st->omega == 0.0) st->flag = FLAG_BREAK;
    });
}

// ------------------------------------------------------------------ GMRES(m), right Jacobi
__global__ void k_gmres_start(int64_t n, const double *r, double *V0, KState *st) {
    // V0 = r / ||r|| (||r||^2 in st->rr); g = (beta, 0, ...)
    const double beta = sqrt(st->rr);
    const double inv = beta > 0 ? 1.0 / beta : 0.0;
    GRID_STRIDE(i, n) V0[i] = r[i] * inv;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->g[0] = beta;
        st->k = 0;
        st->flag = (st->rr <= st->tol2) ? FLAG_CONV : FLAG_RUN;
    }
}

__global__ void k_scale(int64_t n, const double *M, const double *a, double *out, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    GRID_STRIDE(i, n) out[i] = M[i] * a[i];
}

template <int D>
__global__ void __launch_bounds__(kT) k_spmv_guard(EllView<D> G, const double *x, double *y, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    GRID_STRIDE(row, G.nrows) {
        double o[D];
        spmv_row<D>(G, row, x, o);
#pragma unroll
        for (int i = 0; i < D; ++i) y[row * D + i] = o[i];
    }
}

// h[j] (+)= V_j . w for j = 0..k  (classical Gram-Schmidt pass), block-level partials per j
__global__ void __launch_bounds__(kT) k_gmres_dots(int64_t n, int k, const double *V, const double *w, KState *st,
                                                   double *partials, int accumulate) {
    if (st->flag != FLAG_RUN) return;
    __shared__ double sh[32];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = 0; j <= k; ++j) {
        double acc = 0.0;
        GRID_STRIDE(i, n) acc += V[(int64_t)j * n + i] * w[i];
        acc = warp_sum(acc);
        if (lane == 0) sh[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < nw; ++q) t += sh[q];
            partials[(int64_t)blockIdx.x * (kMaxRestart + 1) + j] = t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned tk = atomicAdd(&st->tickets[5], 1u);
        s_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int j = 0; j <= k; ++j) {
        double acc = 0.0;
        for (int bidx = threadIdx.x; bidx < (int)gridDim.x; bidx += blockDim.x)
            acc += __ldcg(partials + (int64_t)bidx * (kMaxRestart + 1) + j);
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) sh[warp] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < nw; ++q) t += sh[q];
            st->h[j] = accumulate ? st->h[j] + t : t;
        }
    }
    if (threadIdx.x == 0) st->tickets[5] = 0u;
}

// w -= sum_j h_j V_j (only the increment of this pass: hnew - hold kept in y[])
__global__ void __launch_bounds__(kT) k_gmres_orth(int64_t n, int k, const double *V, double *w, const KState *st, int pass) {
    if (st->flag != FLAG_RUN) return;
    GRID_STRIDE(i, n) {
        double acc = w[i];
        for (int j = 0; j <= k; ++j) acc -= (pass == 0 ? st->h[j] : st->h[j] - st->y[j]) * V[(int64_t)j * n + i];
        w[i] = acc;
    }
}

__global__ void k_gmres_keep_h(KState *st, int k) {
    if (st->flag != FLAG_RUN) return;
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int j = 0; j <= k; ++j) st->y[j] = st->h[j];
}

// ||w|| then Givens update of column k (thread 0 of the last block)
__global__ void __launch_bounds__(kT) k_gmres_norm_givens(int64_t n, int k, const double *w, KState *st, double *partials) {
    if (st->flag != FLAG_RUN) return;
    double acc[1] = {0.0};
    GRID_STRIDE(i, n) acc[0] += w[i] * w[i];
    reduce_and_finish<1>(acc, partials, &st->tickets[6], [&](double *t) {
        const int m1 = kMaxRestart;
        double hk1 = sqrt(t[0]);
        st->hnorm = hk1;
        double col[kMaxRestart + 1];
        for (int j = 0; j <= k; ++j) col[j] = st->h[j];
        col[k + 1] = hk1;
        for (int j = 0; j < k; ++j) {
            double a = st->cs[j] * col[j] + st->sn[j] * col[j + 1];
            col[j + 1] = -st->sn[j] * col[j] + st->cs[j] * col[j + 1];
            col[j] = a;
        }
        double den = hypot(col[k], col[k + 1]);
        double cs = den > 0 ? col[k] / den : 1.0, sn = den > 0 ? col[k + 1] / den : 0.0;
        st->cs[k] = cs;
        st->sn[k] = sn;
        col[k] = den;
        for (int j = 0; j <= k; ++j) st->H[j * m1 + k] = col[j];
        st->g[k + 1] = -sn * st->g[k];
        st->g[k] = cs * st->g[k];
        st->k = k + 1;
        st->iters += 1;
        if (fabs(st->g[k + 1]) * fabs(st->g[k + 1]) <= st->tol2 || hk1 == 0.0 || den == 0.0) st->flag = FLAG_CONV;
    });
}

__global__ void k_gmres_next(int64_t n, const double *w, double *Vk1, const KState *st) {
    if (st->flag != FLAG_RUN) return;
    const double inv = 1.0 / st->hnorm;
    GRID_STRIDE(i, n) Vk1[i] = w[i] * inv;
}

// y = H^{-1} g (upper triangular, st->k columns) ; x += M (V y)
__global__ void k_gmres_solve_y(KState *st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int k = st->k, m1 = kMaxRestart;
    for (int i = k - 1; i >= 0; --i) {
        double acc = st->g[i];
        for (int j = i + 1; j < k; ++j) acc -= st->H[i * m1 + j] * st->y[j];
        st->y[i] = acc / st->H[i * m1 + i];
    }
}

__global__ void __launch_bounds__(kT) k_gmres_update_x(int64_t n, const double *V, const double *M, double *x, const KState *st) {
    const int k = st->k;
    GRID_STRIDE(i, n) {
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc += st->y[j] * V[(int64_t)j * n + i];
        x[i] = fma(M[i], acc, x[i]);
    }
}

// ------------------------------------------------------------------ host driver
static void ensure_work(cr_hybrid_s *h, cudaStream_t s) {
    const int D = h->G.d;
    const int64_t N = h->G.nrows * D;
    // SpMV inputs carry the ghost rows of a partitioned system after the owned ones
    const int64_t Nalloc = (h->G.nrows + (h->part.on ? h->part.nghost : 0)) * D;
    if (h->work && h->work->N == N) return;
    delete h->work;
    SolverWork *w = new SolverWork();
    h->work = w;
    w->N = N;
    w->D = D;
    // the PCG methods' vectors; MINRES / BiCGStab / GMRES add theirs on first use (ensure_extra)
    for (DevBuf<double> *b : {&w->x, &w->b, &w->r, &w->p, &w->q, &w->z, &w->t}) {
        b->alloc(Nalloc, s);
        b->zero(s);
    }
    w->Nalloc = Nalloc;
    w->partials.alloc((size_t)num_sms() * 16 * (kMaxRestart + 1), s);
    w->st.alloc(1, s);
    w->st.zero(s);
    CR_CUDA(cudaMallocHost((void **)&w->hst, sizeof(KState)));
    CR_CUDA(cudaEventCreate(&w->e0));
    CR_CUDA(cudaEventCreate(&w->e1));
    CR_CUDA(cudaEventCreate(&w->es));
    CR_CUDA(cudaStreamCreateWithFlags(&w->cap, cudaStreamNonBlocking));
    CR_CUDA(cudaStreamCreateWithFlags(&w->side, cudaStreamNonBlocking));
    CR_CUDA(cudaEventCreateWithFlags(&w->fork, cudaEventDisableTiming));
    CR_CUDA(cudaEventCreateWithFlags(&w->join, cudaEventDisableTiming));
}

// vectors of the non-PCG methods (MINRES, BiCGStab, GMRES), allocated on first use
static void ensure_extra(SolverWork *w, cudaStream_t s) {
    if (w->v.n) return;
    for (DevBuf<double> *b : {&w->z2, &w->v, &w->v2, &w->w, &w->w2, &w->y, &w->rhat}) {
        b->alloc(w->Nalloc, s);
        b->zero(s);
    }
}

struct Launcher {
    cr_hybrid_s *h;
    SolverWork *w;
    cudaStream_t s;
    int64_t launches = 0;
    int64_t spmvs = 0;
    int D;
    int64_t nrows, N;
    int grid_rows, grid_vec;
    int dist = 0;           // partitioned over several ranks
    Comm *comm = nullptr;
    int mf = 0;             // matrix-free factored G
    int so = 0;             // vectors in the solve order (h->so): mf / patch / coarse views in that order

    // after a reducing kernel: allreduce this rank's values and apply the recurrence
    void reduced(cudaStream_t ks, int nv, int kind, double rtol) {
        if (!dist) return;
        comm->allreduce(w->st.get()->red, nv, false, ks);
        k_fin<<<1, 32, 0, ks>>>(w->st.get(), kind, rtol);
        CR_CHECK_LAUNCH();
        ++launches;
    }
    // ghost rows of an SpMV input from the ranks that own them
    void halo(cudaStream_t ks, double *v) {
        if (!dist) return;
        const Part &P = h->part;
        if (P.nsend) {
            if (D == 2) k_halo_pack<2><<<grid_for(P.nsend, kT), kT, 0, ks>>>(P.nsend, P.send_rows.get(), v, P.sendbuf.get());
            else k_halo_pack<3><<<grid_for(P.nsend, kT), kT, 0, ks>>>(P.nsend, P.send_rows.get(), v, P.sendbuf.get());
            CR_CHECK_LAUNCH();
            ++launches;
        }
        comm->halo(P, P.sendbuf.get(), v + P.nloc * D, D, ks);
    }
};

template <int D>
static EllView<D> ell(const cr_hybrid_s *h) { return EllView<D>{h->G.cols.get(), h->G.vals.get(), h->G.nrows}; }

static void read_state(SolverWork *w, cudaStream_t s) {
    CR_CUDA(cudaMemcpyAsync(w->hst, w->st.get(), kStateHeader, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
}

// out[i] = in[perm[i]] / out[perm[i]] = in[i] by block rows of D (the solve order's permutation)
template <int D>
__global__ void k_so_gather(int64_t nrows, const int32_t *perm, const double *in, double *out) {
    GRID_STRIDE(i, nrows) {
        const int64_t r = perm[i];
#pragma unroll
        for (int k = 0; k < D; ++k) out[i * D + k] = in[r * D + k];
    }
}
template <int D>
__global__ void k_so_scatter(int64_t nrows, const int32_t *perm, const double *in, double *out) {
    GRID_STRIDE(i, nrows) {
        const int64_t r = perm[i];
#pragma unroll
        for (int k = 0; k < D; ++k) out[r * D + k] = in[i * D + k];
    }
}

template <int D>
static MfView mf_view(const cr_hybrid_s *h, int so = 0) {
    return MfView{so ? h->mf.ids_so.get() : h->mf.ids.get(), h->mf.sg.get(), h->mf.v.get(), h->mf.nb.get(), h->mf.ncells};
}

// q = G_mf x (q zeroed first); REDUCE also reduces x.q -> alpha
template <int D, bool REDUCE>
static void mf_apply(Launcher &L, cudaStream_t ks, const double *x, double *q, double rtol, int pqkind = FIN_PQ) {
    CR_CUDA(cudaMemsetAsync(q, 0, L.N * sizeof(double), ks));
    // CR_MF_TMA=1: the bulk-copy-staged variant (measured slower in-solve: 6.97 vs 6.62 ms per 3D
    // iteration, the factor stream is not what bounds this kernel)
    static const char *et = std::getenv("CR_MF_TMA");
    if (!et || atoi(et) == 0) {
        k_mf_spmv<D, REDUCE><<<occ_grid(k_mf_spmv<D, REDUCE>, kT, L.h->mf.ncells), kT, 0, ks>>>(
            mf_view<D>(L.h, L.so), x, q, L.nrows, L.w->st.get(), L.w->partials.get(), L.dist, pqkind);
    } else {
        const int64_t nsl = L.h->mf.ncells / 32;
        const int grid = (int)std::min<int64_t>(mf_tma_grid<D, REDUCE>(), (nsl + kMfTmaWarps - 1) / kMfTmaWarps);
        k_mf_spmv_tma<D, REDUCE><<<std::max(grid, 1), kMfTmaWarps * 32, mf_tma_smem<D>(), ks>>>(
            mf_view<D>(L.h, L.so), x, q, L.nrows, L.w->st.get(), L.w->partials.get(), L.dist, pqkind);
    }
    CR_CHECK_LAUNCH();
    ++L.launches;
    if (REDUCE) L.reduced(ks, 1, pqkind, rtol);
}

template <int D>
static void true_residual(Launcher &L, double *x, double *r) {
    if (L.mf) {
        L.halo(L.s, x);
        mf_apply<D, false>(L, L.s, x, L.w->q.get(), 0.0);
        k_resid_vec<<<L.grid_vec, kT, 0, L.s>>>(L.N, L.w->b.get(), L.w->q.get(), r, L.w->st.get(), L.w->partials.get(),
                                               L.dist);
        CR_CHECK_LAUNCH();
        L.reduced(L.s, 1, FIN_RR, 0.0);
        ++L.launches;
        ++L.spmvs;
        return;
    }
    L.halo(L.s, x);
    k_true_residual<D><<<L.grid_rows, kT, 0, L.s>>>(ell<D>(L.h), x, L.w->b.get(), r, L.w->st.get(), L.w->partials.get(),
                                                   L.dist);
    CR_CHECK_LAUNCH();
    L.reduced(L.s, 1, FIN_RR, 0.0);
    ++L.launches;
    ++L.spmvs;
}

// run `body` k times inside a CUDA graph (captured once per (method, k)), replay until done
// The body launches on `ks`; it is captured on the work's private non-blocking stream (the
// caller's stream may be the legacy default stream, which cannot capture) and the graph is
// then launched on the caller's stream.
template <int D, int WHAT>
static void launch_afw(Launcher &L, cudaStream_t ks, const double *r, double *zs, double rtol) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    const AfwPrec &P = L.h->afw;
    AfwView A{P.ioff.get(), P.voff.get(), P.kl.get(), L.so ? P.ids_so.get() : P.ids.get(), P.vals.get(), P.npatch,
              L.h->G.nrows, P.shared};
    const int64_t nt = P.nslices * 32 * D;
    const bool sym = P.built != AFW_GEN;
    // two-level: leave one block per SM to the coarse kernels that run concurrently on the side stream
    // two-level in 2D: leave 2 of the 4 block slots per SM to the concurrent coarse path (its
    // latency-bound nested-dissection phases then overlap the patch solves: -3 % per iteration at
    // H = 64; in 3D and with the dense E^-1 reserving measured slower).  CR_AFW_RSV overrides.
    static const char *er = std::getenv("CR_AFW_RSV");
    const bool two_level = WHAT == AFW_PCG2 || WHAT == AFW_PCG2_INIT;
    const int rsv = er ? atoi(er) : (D == 2 && two_level && !L.dist && L.h->coarse.nd.on ? 2 : 0);
    KState *st = L.w->st.get();
    double *part = L.w->partials.get();
    if (P.shared && (WHAT == AFW_PCG || WHAT == AFW_PCG_INIT || WHAT == AFW_PCG2 || WHAT == AFW_PCG2_INIT)) {
        const int64_t nts = P.nslices * 32;
        // default: one warp per (slice, component) (k_afw_apply_sc, 1.39 vs 1.54 ms on configs[4]);
        // CR_AFW_SPLIT=0: one thread per patch for all components (k_afw_apply_sh)
        static const char *es = std::getenv("CR_AFW_SPLIT");
        if (!(es && atoi(es) == 0) && P.kmax <= 6) {
            constexpr int NT = 32 * D * kAfwSpb;
            k_afw_apply_sc<D, SLOTS, 6, WHAT><<<occ_grid(k_afw_apply_sc<D, SLOTS, 6, WHAT>, NT, nts * D, rsv), NT, 0, ks>>>(
                A, r, zs, rtol, st, part, L.dist);
        } else if (P.kmax <= 6) k_afw_apply_sh<D, SLOTS, 6, WHAT><<<occ_grid(k_afw_apply_sh<D, SLOTS, 6, WHAT>, kT, nts, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
        else if (P.kmax <= 8) k_afw_apply_sh<D, SLOTS, 8, WHAT><<<occ_grid(k_afw_apply_sh<D, SLOTS, 8, WHAT>, kT, nts, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
        else k_afw_apply_sh<D, SLOTS, 16, WHAT><<<occ_grid(k_afw_apply_sh<D, SLOTS, 16, WHAT>, kT, nts, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
    } else if (P.kmax <= 6) {
        if (sym) k_afw_apply<D, SLOTS, 6, true, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 6, true, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
        else k_afw_apply<D, SLOTS, 6, false, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 6, false, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
    } else if (P.kmax <= 8) {
        if (sym) k_afw_apply<D, SLOTS, 8, true, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 8, true, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
        else k_afw_apply<D, SLOTS, 8, false, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 8, false, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
    } else {
        if (sym) k_afw_apply<D, SLOTS, 16, true, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 16, true, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
        else k_afw_apply<D, SLOTS, 16, false, WHAT><<<occ_grid(k_afw_apply<D, SLOTS, 16, false, WHAT>, kT, nt, rsv), kT, 0, ks>>>(A, r, zs, rtol, st, part, L.dist);
    }
    CR_CHECK_LAUNCH();
    ++L.launches;
    if (WHAT == AFW_PCG_INIT) L.reduced(ks, 1, FIN_AFW_PCG_INIT, rtol);
    if (WHAT == AFW_PCG) L.reduced(ks, 1, FIN_AFW_PCG, rtol);
    if (WHAT == AFW_PCG2_INIT) L.reduced(ks, 1, FIN_AFW2_QF_INIT, rtol);
    if (WHAT == AFW_PCG2) L.reduced(ks, 1, FIN_AFW2_QF, rtol);
}

template <class Body, class Done>
static void graph_loop(Launcher &L, cudaStream_t &ks, int key, int k, Body body, Done done) {
    SolverWork *w = L.w;
    if (L.dist && !L.comm->capturable()) {   // host-synchronising collectives: no graph
        ks = L.s;
        while (true) {
            for (int i = 0; i < k; ++i) body(i);
            read_state(w, L.s);
            if (done()) break;
        }
        return;
    }
    if (w->graph_key != key) {
        if (w->graph) { cudaGraphExecDestroy(w->graph); w->graph = nullptr; }
        cudaGraph_t g;
        ks = w->cap;
        CR_CUDA(cudaStreamBeginCapture(w->cap, cudaStreamCaptureModeThreadLocal));
        int64_t l0 = L.launches, s0 = L.spmvs;
        g_capturing = true;   // captured launches are counted when the graph replays
        try {
            for (int i = 0; i < k; ++i) body(i);
        } catch (...) {
            g_capturing = false;
            cudaGraph_t junk;
            cudaStreamEndCapture(w->cap, &junk);
            if (junk) cudaGraphDestroy(junk);
            throw;
        }
        g_capturing = false;
        L.launches = l0;
        L.spmvs = s0;
        CR_CUDA(cudaStreamEndCapture(w->cap, &g));
        ks = L.s;
        size_t nn = 0;
        CR_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        if (nn) CR_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        w->graph_kernels = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CR_CUDA(cudaGraphNodeGetType(nd, &ty));
            if (ty == cudaGraphNodeTypeKernel) ++w->graph_kernels;
        }
        CR_CUDA(cudaGraphInstantiate(&w->graph, g, 0));
        CR_CUDA(cudaGraphDestroy(g));
        w->graph_key = key;
    }
    while (true) {
        CR_CUDA(cudaGraphLaunch(w->graph, L.s));
        count_launches(w->graph_kernels);
        read_state(w, L.s);
        if (done()) break;
    }
}

// extreme eigenvalues of the symmetric tridiagonal T (diag a, off-diagonal b) by bisection on
// the Sturm count (host; m <= kLanczos)
static double tri_eig(const std::vector<double> &a, const std::vector<double> &b, int k) {
    const int m = (int)a.size();
    double lo = INFINITY, hi = -INFINITY;
    for (int i = 0; i < m; ++i) {   // Gershgorin bounds
        const double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < m ? fabs(b[i]) : 0.0);
        lo = fmin(lo, a[i] - r);
        hi = fmax(hi, a[i] + r);
    }
    auto count_below = [&](double x) {   // eigenvalues < x
        int c = 0;
        double q = a[0] - x;
        if (q < 0) ++c;
        for (int i = 1; i < m; ++i) {
            const double qq = q != 0.0 ? q : 1e-300;
            q = a[i] - x - b[i - 1] * b[i - 1] / qq;
            if (q < 0) ++c;
        }
        return c;
    };
    for (int it = 0; it < 200; ++it) {   // k-th smallest eigenvalue (0-based)
        const double mid = 0.5 * (lo + hi);
        if (count_below(mid) > k) hi = mid;
        else lo = mid;
        if (hi - lo <= 1e-14 * fmax(fabs(lo), fabs(hi))) break;
    }
    return 0.5 * (lo + hi);
}

// kappa of the preconditioned G from the CG coefficients: T_kk = 1/alpha_k + beta_{k-1}/alpha_{k-1},
// T_{k,k+1} = sqrt(beta_k)/alpha_k (the Lanczos matrix CG builds implicitly)
static void lanczos_kappa(SolverWork *w, cudaStream_t s, int64_t iters, cr_solve_report *rep) {
    const int m = (int)std::min<int64_t>(iters, kLanczos) - 1;
    if (m < 2) return;
    std::vector<double> lz(2 * (m + 1));
    CR_CUDA(cudaMemcpyAsync(lz.data(), reinterpret_cast<const char *>(w->st.get()) + offsetof(KState, lz),
                            lz.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    std::vector<double> a(m), b(m > 0 ? m - 1 : 0);
    double alpha_prev = 0.0, beta_prev = 0.0;
    for (int k = 0; k < m; ++k) {
        const double rho = lz[2 * k], pq = lz[2 * k + 1], rho1 = lz[2 * (k + 1)];
        if (!(rho > 0 && pq > 0 && rho1 > 0)) return;
        const double alpha = rho / pq, beta = rho1 / rho;
        a[k] = 1.0 / alpha + (k > 0 ? beta_prev / alpha_prev : 0.0);
        if (k + 1 < m) b[k] = sqrt(beta) / alpha;
        alpha_prev = alpha;
        beta_prev = beta;
    }
    const double lmin = tri_eig(a, b, 0), lmax = tri_eig(a, b, m - 1);
    rep->lambda_min_est = lmin;
    rep->lambda_max_est = lmax;
    rep->kappa_lanczos_est = lmin > 0 ? lmax / lmin : 0.0;
}

// algorithmic HBM bytes of one iteration of `o.method`:
// G apply (assembled: values + block cols + x + y; matrix-free: cell factors + x + q), the
// vector updates, and the preconditioner's operator and vectors
static double iter_bytes(const cr_hybrid_s *h, const cr_solver_opts &o) {
    const double N8 = 8.0 * (double)h->G.nrows * h->G.d;
    const int d = h->G.d, slots = d == 2 ? 2 : 3;
    const double nnz = (double)h->G.nblocks * d * d;
    const double g_asm = 8.0 * nnz + 4.0 * (double)h->G.nblocks + 2 * N8;
    const double g_mf = h->mf.built ? (double)(h->mf.v.n * sizeof(double) + h->mf.ids.n * sizeof(int32_t) + h->mf.sg.n +
                                               h->mf.nb.n) + 2 * N8
                                    : g_asm;
    const double g = o.matrix_free ? g_mf : g_asm;
    const double afw = h->afw.built >= 0 ? (double)(h->afw.vals.n * sizeof(double) + h->afw.ids.n * sizeof(int32_t) +
                                                    h->afw.kl.n + 2 * h->afw.ioff.n * sizeof(int64_t))
                                         : 0.0;
    switch (o.method) {
        case CR_PCG_JACOBI: return g + 7 * N8;                 // x, r, p, q, dinv read; x, r write (+ p rewrite)
        case CR_PCG_BLOCKJACOBI: return g + 6 * N8 + N8 * d;   // + inverse diagonal blocks
        // r update (r, q read, r written); patch apply; direction update with the x update (slots, p,
        // x read, p, x written)
        case CR_PCG_AFW: return g + 3 * N8 + (afw + N8 + slots * N8) + (slots * N8 + 4 * N8);
        case CR_PCG_AFW2: {
            const double coarse = 2 * N8 + (double)(h->coarse.nd.on ? h->coarse.nd.bytes : 8 * h->coarse.nE * h->coarse.nE);
            return g + 3 * N8 + (afw + N8 + slots * N8) + coarse + (slots * N8 + 4 * N8 + N8);
        }
        case CR_MINRES_ABSJACOBI: return g + 10 * N8;
        case CR_MINRES_AFW: return g + 10 * N8 + afw + 2 * slots * N8;
        case CR_MINRES_AFW2:
            return g + 10 * N8 + afw + 2 * slots * N8 + 3 * N8 + (double)(8 * h->coarse.nE * h->coarse.nE);
        case CR_BICGSTAB_JACOBI: return 2 * g + 12 * N8;
        default: return 0.0;
    }
}

template <int D>
static void solve_t(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep,
                    const double *rhs) {
    ensure_work(h, s);
    SolverWork *w = h->work;
    Launcher L{h, w, s};
    cudaStream_t ks = s;   // stream the captured bodies launch on (swapped during capture)
    L.D = D;
    L.nrows = h->G.nrows;
    L.N = w->N;
    L.grid_rows = grid_for(L.nrows, kT);
    L.grid_vec = grid_for(L.N, kT);
    L.dist = h->part.on ? 1 : 0;
    L.comm = h->part.on ? h->comm->impl : nullptr;
    const bool pcg_family = o.method == CR_PCG_JACOBI || o.method == CR_PCG_BLOCKJACOBI || o.method == CR_PCG_AFW ||
                            o.method == CR_PCG_AFW2;
    CR_REQUIRE(!L.dist || pcg_family, CR_ERR_INVALID_ARG, "a partitioned (multi-GPU) solve supports the PCG methods only");
    L.mf = o.matrix_free ? 1 : 0;
    CR_REQUIRE(!L.mf || pcg_family, CR_ERR_INVALID_ARG, "matrix_free supports the PCG methods only");
    Trace trc(s);
    if (L.mf) build_mf(h, s);
    trc.mark("matrix-free factors");
    const int64_t N = w->N, nrows = L.nrows;
    const double rtol = o.rtol > 0 ? o.rtol : 1e-10;
    const int64_t max_iter = o.max_iter > 0 ? o.max_iter : 10000000;
    int kk = o.check_every > 0 ? o.check_every : 64;
    kk = (kk + 1) & ~1;   // even: MINRES buffer rotation has period 2
    double *x = w->x.get();
    // solve order (h->so): the matrix-free patch-preconditioned PCG on one GPU runs on
    // S, W permuted into it (CR_SOLVE_ORDER=0: the mesh's face order)
    const char *eso = std::getenv("CR_SOLVE_ORDER");   // read per solve (tests compare both orders)
    const bool so_on = L.mf && !L.dist && (o.method == CR_PCG_AFW || o.method == CR_PCG_AFW2) && !(eso && atoi(eso) == 0);
    if (so_on) {
        build_so(h, s);
        k_so_gather<D><<<L.grid_rows, kT, 0, s>>>(nrows, h->so.perm.get(), W, x);
        CR_CHECK_LAUNCH();
        k_so_gather<D><<<L.grid_rows, kT, 0, s>>>(nrows, h->so.perm.get(), rhs ? rhs : h->S.get(), w->b.get());
        CR_CHECK_LAUNCH();
    } else {
        CR_CUDA(cudaMemcpyAsync(x, W, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
        CR_CUDA(cudaMemcpyAsync(w->b.get(), rhs ? rhs : h->S.get(), N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    CR_CUDA(cudaMemsetAsync(w->st.get(), 0, sizeof(KState), s));
    CR_CUDA(cudaEventRecord(w->e0, s));
    CR_CUDA(cudaEventRecord(w->es, s));   // re-recorded once a preconditioner / coarse space is built
    double *part = w->partials.get();
    KState *st = w->st.get();
    k_norm2<<<L.grid_vec, kT, 0, s>>>(w->b.get(), N, st, part, L.dist);
    CR_CHECK_LAUNCH();
    L.reduced(s, 1, FIN_BB, 0.0);
    ++L.launches;
    cr_status status = CR_OK;
    int replacements = 0;
    const int method = o.method;

    if (method == CR_PCG_JACOBI || method == CR_PCG_BLOCKJACOBI) {
        const bool blk = method == CR_PCG_BLOCKJACOBI;
        const double *M = blk ? h->bdinv.get() : h->dinv.get();
        auto init = [&]() {
            true_residual<D>(L, x, w->r.get());
            if (blk) k_pcg_init<D, 1><<<L.grid_rows, kT, 0, s>>>(nrows, w->b.get(), w->r.get(), w->p.get(), M, rtol, st, part, L.dist);
            else k_pcg_init<D, 0><<<L.grid_rows, kT, 0, s>>>(nrows, w->b.get(), w->r.get(), w->p.get(), M, rtol, st, part, L.dist);
            CR_CHECK_LAUNCH();
            L.reduced(s, 2, FIN_PCG_INIT, rtol);
            ++L.launches;
        };
        init();
        read_state(w, s);
        if (w->hst->bb == 0.0) { CR_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), s)); }
        while (w->hst->flag == FLAG_RUN) {
            auto body = [&](int) {
                L.halo(ks, w->p.get());
                if (L.mf) {
                    mf_apply<D, true>(L, ks, w->p.get(), w->q.get(), rtol);
                } else {
                    k_pcg_spmv<D><<<occ_grid(k_pcg_spmv<D>, kT, L.nrows), kT, 0, ks>>>(ell<D>(h), w->p.get(), w->q.get(), st, part, L.dist);
                    CR_CHECK_LAUNCH();
                    L.reduced(ks, 1, FIN_PQ, rtol);
                }
                if (blk) {
                    k_pcg_update<D, 1><<<L.grid_rows, kT, 0, ks>>>(nrows, x, w->r.get(), w->p.get(), w->q.get(), M, st, part, L.dist);
                    CR_CHECK_LAUNCH();
                    L.reduced(ks, 2, FIN_UPD_PC, rtol);
                    k_pcg_pdir<D, 1><<<L.grid_rows, kT, 0, ks>>>(nrows, w->p.get(), w->r.get(), M, st);
                } else {
                    k_pcg_update_jac<<<occ_grid(k_pcg_update_jac, kT, L.N / 2), kT, 0, ks>>>(N, x, w->r.get(), w->p.get(), w->q.get(), M, st, part, L.dist);
                    CR_CHECK_LAUNCH();
                    L.reduced(ks, 2, FIN_UPD_PC, rtol);
                    k_pcg_pdir_jac<<<occ_grid(k_pcg_pdir_jac, kT, L.N / 2), kT, 0, ks>>>(N, w->p.get(), w->r.get(), M, st);
                }
                CR_CHECK_LAUNCH();
            };
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() {
                return w->hst->flag != FLAG_RUN || w->hst->iters >= max_iter;
            });
            int64_t dit = w->hst->iters - it0;
            L.launches += 3 * ((dit + kk - 1) / kk) * kk;
            L.spmvs += dit;
            if (w->hst->flag == FLAG_CONV) {
                // recursive residual converged: check the true residual (residual replacement)
                init();
                read_state(w, s);
                if (w->hst->flag == FLAG_CONV || replacements >= 8) break;
                ++replacements;
            }
            if (w->hst->flag == FLAG_BREAK) { status = CR_ERR_BREAKDOWN; break; }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_PCG_AFW) {
        constexpr int SLOTS = D == 2 ? 2 : 3;
        build_afw(h, AFW_SPD, s);
        L.so = so_on ? 1 : 0;
        if (L.so) afw_so(h, s);
        CR_CUDA(cudaEventRecord(w->es, s));
        if (w->zs.n < (size_t)SLOTS * N) w->zs.alloc((size_t)SLOTS * N, s);
        double *zs = w->zs.get();
        auto init = [&]() {
            true_residual<D>(L, x, w->r.get());
            launch_afw<D, AFW_PCG_INIT>(L, s, w->r.get(), zs, rtol);
            k_pcg_pdir_afw<D, SLOTS><<<L.grid_rows, kT, 0, s>>>(nrows, w->p.get(), zs, st, nullptr);
            CR_CHECK_LAUNCH();
            ++L.launches;
        };
        init();
        read_state(w, s);
        if (w->hst->bb == 0.0) { CR_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), s)); }
        while (w->hst->flag == FLAG_RUN) {
            auto body = [&](int) {
                L.halo(ks, w->p.get());
                if (L.mf) {
                    mf_apply<D, true>(L, ks, w->p.get(), w->q.get(), rtol);
                } else {
                    k_pcg_spmv<D><<<occ_grid(k_pcg_spmv<D>, kT, L.nrows), kT, 0, ks>>>(ell<D>(h), w->p.get(), w->q.get(), st, part, L.dist);
                    CR_CHECK_LAUNCH();
                    L.reduced(ks, 1, FIN_PQ, rtol);
                }
                k_pcg_update_r<false><<<occ_grid(k_pcg_update_r<false>, kT, L.N / 2), kT, 0, ks>>>(N, x, w->r.get(), w->p.get(), w->q.get(), st, part, L.dist);
                CR_CHECK_LAUNCH();
                L.reduced(ks, 1, FIN_UPD_R, rtol);
                launch_afw<D, AFW_PCG>(L, ks, w->r.get(), zs, rtol);
                k_pcg_pdir_afw<D, SLOTS><<<occ_grid(k_pcg_pdir_afw<D, SLOTS>, kT, nrows), kT, 0, ks>>>(nrows, w->p.get(), zs, st, x);
                CR_CHECK_LAUNCH();
            };
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() {
                return w->hst->flag != FLAG_RUN || w->hst->iters >= max_iter;
            });
            int64_t dit = w->hst->iters - it0;
            L.launches += 4 * ((dit + kk - 1) / kk) * kk;
            L.spmvs += dit;
            if (w->hst->flag == FLAG_CONV && dit > 0) {   // the converged iteration's x update
                k_pcg_x_final<<<L.grid_vec, kT, 0, s>>>(N, x, w->p.get(), st);
                CR_CHECK_LAUNCH();
                ++L.launches;
            }
            if (w->hst->flag == FLAG_CONV) {
                init();
                read_state(w, s);
                if (w->hst->flag == FLAG_CONV || replacements >= 8) break;
                ++replacements;
            }
            if (w->hst->flag == FLAG_BREAK) { status = CR_ERR_BREAKDOWN; break; }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_PCG_AFW2) {
        constexpr int SLOTS = D == 2 ? 2 : 3;
        build_afw(h, AFW_SPD, s);
        CR_CUDA(cudaEventRecord(w->es, s));
        trc.mark("patch preconditioner");
        const int H = o.coarse > 0 ? o.coarse : (D == 2 ? 64 : 16);
        // E = Z^t G Z needs G applied to colour sums of coarse columns; with the matrix-free G only
        // the 32-cell slices touching the colour's support are applied (the rest of z is zero)
        DevBuf<uint8_t> sflag;
        DevBuf<int32_t> slist;
        DevBuf<int64_t> snum;
        DevBuf<uint8_t> stmp;
        int last_colour = -1;
        // the 32-cell slices touching the coarse cells around `colour`'s nodes (x vanishes elsewhere)
        DevBuf<unsigned> smask;
        int mask_H = -1;   // coarse grid the mask was computed for (a retry with a halved H recomputes it)
        auto select_slices = [&](int colour) {
            const int64_t nsl = h->mf.ncells / 32;
            if (sflag.n == 0) {
                sflag.alloc(nsl, s);
                slist.alloc(nsl, s);
                snum.alloc(1, s);
                size_t tb = 0;
                cub::CountingInputIterator<int32_t> it(0);
                CR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, sflag.get(), slist.get(), snum.get(), nsl, s));
                stmp.alloc(tb, s);
                smask.alloc((size_t)nsl * 4, s);
            }
            if (mask_H != h->coarse.g.H) {
                k_mf_slice_colours<D><<<grid_for(nsl * 32, kT), kT, 0, s>>>(mf_view<D>(h), h->coarse.view(), nsl,
                                                                           smask.get());
                CR_CHECK_LAUNCH();
                mask_H = h->coarse.g.H;
                last_colour = -1;
            }
            if (colour == last_colour) return;
            k_mf_flag_colour<<<grid_for(nsl, kT), kT, 0, s>>>(smask.get(), nsl, colour, sflag.get());
            CR_CHECK_LAUNCH();
            size_t tb = stmp.n;
            cub::CountingInputIterator<int32_t> it(0);
            CR_CUDA(cub::DeviceSelect::Flagged(stmp.get(), tb, it, sflag.get(), slist.get(), snum.get(), nsl, s));
            last_colour = colour;
        };
        build_coarse(h, H, [&](const double *z, double *Y, int colour, int ncol, int64_t stride) {
            for (int c = 0; c < ncol; ++c) L.halo(s, const_cast<double *>(z) + c * stride);
            if (L.mf && colour >= 0 && !L.dist) {
                select_slices(colour);
                // Y arrives zero (build_coarse clears the rows it touched after each pass)
                if (ncol == 1) {
                    k_mf_spmv_slices<D><<<occ_grid(k_mf_spmv_slices<D>, kT, h->mf.ncells), kT, 0, s>>>(
                        mf_view<D>(h), slist.get(), snum.get(), z, Y, L.nrows);
                } else {
                    k_mf_spmv_slices_all<D><<<occ_grid(k_mf_spmv_slices_all<D>, kT, h->mf.ncells), kT, 0, s>>>(
                        mf_view<D>(h), slist.get(), snum.get(), z, Y, stride, ncol, L.nrows);
                }
                CR_CHECK_LAUNCH();
            } else {
                for (int c = 0; c < ncol; ++c) {
                    if (L.mf) mf_apply<D, false>(L, s, z + c * stride, Y + c * stride, 0.0);
                    else spmv(h->G, z + c * stride, Y + c * stride, s);
                }
            }
        }, (L.mf && !L.dist) ? ApplyGColour([&](int colour, double *Y, int64_t stride) {
            select_slices(colour);
            k_mf_spmv_colour<D><<<occ_grid(k_mf_spmv_colour<D>, kT, h->mf.ncells), kT, 0, s>>>(
                mf_view<D>(h), h->coarse.view(), colour, slist.get(), snum.get(), Y, stride, L.nrows);
            CR_CHECK_LAUNCH();
        }) : ApplyGColour(), s);
        trc.mark("coarse space (E, E^-1)");
        CR_CUDA(cudaEventRecord(w->es, s));
        if (w->zs.n < (size_t)SLOTS * N) w->zs.alloc((size_t)SLOTS * N, s);
        double *zs = w->zs.get();
        L.so = so_on ? 1 : 0;
        if (L.so) {
            afw_so(h, s);
            coarse_so(h, s);
        }
        const CoarseView CV = L.so ? h->coarse.view_so() : h->coarse.view();
        double *yc = h->coarse.y.get();
        // coarse path (restriction, gather, E^-1 GEMV) forked onto a side stream so it overlaps the
        // patch solves; joined before the direction update.  Partitioned runs fork only with a
        // second communicator for the coarse allreduce (NCCL collectives of one communicator must
        // not be reordered between ranks); its replicated coarse solve then hides behind the
        // rank's share of the fine-level work.
        // (opt-in, CR_DIST_OVERLAP=1: concurrent collectives of two communicators are only safe when
        // every rank's GPU can run both NCCL kernels at once; not measurable with one GPU per call)
        static const char *eov = std::getenv("CR_DIST_OVERLAP");
        const bool fork = !L.dist || (eov && atoi(eov) == 1 && L.comm->capturable() && L.comm->has_side());
        double *cpart = h->coarse.gpart.get();
        auto coarse_begin = [&](cudaStream_t q) {
            cudaStream_t cs = q;
            if (fork) {
                CR_CUDA(cudaEventRecord(w->fork, q));
                CR_CUDA(cudaStreamWaitEvent(w->side, w->fork, 0));
                cs = w->side;
            }
            coarse_restrict_solve(h, w->r.get(), &st->qc, fork ? cpart : part, &st->tickets[4], cs, fork && L.dist, L.so);
            if (fork) CR_CUDA(cudaEventRecord(w->join, w->side));
            L.launches += 3;
        };
        auto coarse_end = [&](cudaStream_t q) {
            if (fork) CR_CUDA(cudaStreamWaitEvent(q, w->join, 0));
        };
        auto init = [&]() {
            true_residual<D>(L, x, w->r.get());
            coarse_begin(s);
            launch_afw<D, AFW_PCG2_INIT>(L, s, w->r.get(), zs, rtol);
            coarse_end(s);
            k_pcg_pdir_afw2<D, SLOTS><<<L.grid_rows, kT, 0, s>>>(nrows, w->p.get(), zs, CV, yc, st, 1, nullptr);
            CR_CHECK_LAUNCH();
            ++L.launches;
        };
        init();
        read_state(w, s);
        trc.mark("initial residual");
        if (w->hst->bb == 0.0) { CR_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double), s)); }
        bool first_replay = true;
        while (w->hst->flag == FLAG_RUN) {
            auto body = [&](int) {
                L.halo(ks, w->p.get());
                if (L.mf) {
                    mf_apply<D, true>(L, ks, w->p.get(), w->q.get(), rtol, FIN_PQ2);
                } else {
                    k_pcg_spmv<D><<<occ_grid(k_pcg_spmv<D>, kT, L.nrows), kT, 0, ks>>>(ell<D>(h), w->p.get(), w->q.get(), st, part,
                                                                                     L.dist, FIN_PQ2);
                    CR_CHECK_LAUNCH();
                    L.reduced(ks, 1, FIN_PQ2, rtol);
                }
                k_pcg_update_r<false><<<occ_grid(k_pcg_update_r<false>, kT, L.N / 2), kT, 0, ks>>>(N, x, w->r.get(), w->p.get(), w->q.get(), st, part, L.dist);
                CR_CHECK_LAUNCH();
                L.reduced(ks, 1, FIN_UPD_R, rtol);
                coarse_begin(ks);
                launch_afw<D, AFW_PCG2>(L, ks, w->r.get(), zs, rtol);
                coarse_end(ks);
                k_pcg_pdir_afw2<D, SLOTS><<<occ_grid(k_pcg_pdir_afw2<D, SLOTS>, kT, nrows), kT, 0, ks>>>(nrows, w->p.get(), zs, CV, yc, st, 0, x);
                CR_CHECK_LAUNCH();
            };
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() {
                return w->hst->flag != FLAG_RUN || w->hst->iters >= max_iter;
            });
            if (first_replay) { trc.mark("iterations (incl. graph capture)"); first_replay = false; }
            int64_t dit = w->hst->iters - it0;
            L.launches += 7 * ((dit + kk - 1) / kk) * kk;
            L.spmvs += dit;
            if (w->hst->flag == FLAG_CONV && dit > 0) {   // the converged iteration's x update
                k_pcg_x_final<<<L.grid_vec, kT, 0, s>>>(N, x, w->p.get(), st);
                CR_CHECK_LAUNCH();
                ++L.launches;
            }
            if (w->hst->flag == FLAG_CONV) {
                init();
                read_state(w, s);
                if (w->hst->flag == FLAG_CONV || replacements >= 8) break;
                ++replacements;
            }
            if (w->hst->flag == FLAG_BREAK) { status = CR_ERR_BREAKDOWN; break; }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_MINRES_AFW || method == CR_MINRES_AFW2) {
        ensure_extra(w, s);
        constexpr int SLOTS = D == 2 ? 2 : 3;
        const bool two = method == CR_MINRES_AFW2;
        build_afw(h, AFW_ABS, s);
        if (two) {
            // coarse |E|^{-1}: E = Z^t G Z of the shifted G by the assembled G, dense eigendecomposition
            const int H = o.coarse > 0 ? o.coarse : (D == 2 ? 32 : 8);
            build_coarse(h, H, [&](const double *z, double *Y, int, int ncol, int64_t stride) {
                for (int c = 0; c < ncol; ++c) spmv(h->G, z + c * stride, Y + c * stride, s);
            }, ApplyGColour(), s, true);
        }
        CR_CUDA(cudaEventRecord(w->es, s));
        if (w->zs.n < (size_t)SLOTS * N) w->zs.alloc((size_t)SLOTS * N, s);
        double *zs = w->zs.get();
        double *va = w->v.get(), *vb = w->v2.get(), *za = w->z.get(), *zb = w->z2.get();
        double *wa = w->w.get(), *wb = w->w2.get();
        const CoarseView CV = h->coarse.view();
        double *yc = h->coarse.y.get();
        // z = M v: the |patch| part, plus Z |E|^{-1} Z^t v (its c^t y lands in st->qc before the patch
        // kernel's last block forms v^t M v)
        auto precond = [&](cudaStream_t q, const double *v, double *zout, bool init) {
            if (two) coarse_restrict_solve(h, v, &st->qc, part, &st->tickets[4], q);
            if (init) {
                if (two) launch_afw<D, AFW_MINRES2_INIT>(L, q, v, zs, rtol);
                else launch_afw<D, AFW_MINRES_INIT>(L, q, v, zs, rtol);
            } else {
                if (two) launch_afw<D, AFW_MINRES2>(L, q, v, zs, rtol);
                else launch_afw<D, AFW_MINRES>(L, q, v, zs, rtol);
            }
            if (two) k_afw_zsum2<D, SLOTS><<<L.grid_rows, kT, 0, q>>>(nrows, zout, zs, CV, yc, st, init ? 0 : 1);
            else k_afw_zsum<D, SLOTS><<<L.grid_rows, kT, 0, q>>>(nrows, zout, zs, st, init ? 0 : 1);
            CR_CHECK_LAUNCH();
        };
        true_residual<D>(L, x, va);
        k_zero3<<<L.grid_vec, kT, 0, s>>>(N, wa, wb, vb);
        CR_CHECK_LAUNCH();
        precond(s, va, za, true);
        L.launches += 2;
        read_state(w, s);
        const double bnorm = sqrt(w->hst->bb);
        auto body = [&](int i) {
            double *v = (i & 1) ? vb : va, *vold = (i & 1) ? va : vb;
            double *z = (i & 1) ? zb : za, *zn = (i & 1) ? za : zb;
            double *ww = (i & 1) ? wb : wa, *wold = (i & 1) ? wa : wb;
            k_minres_spmv<D><<<L.grid_rows, kT, 0, ks>>>(ell<D>(h), z, w->q.get(), st, part);
            k_minres_lanczos_v<D><<<L.grid_rows, kT, 0, ks>>>(nrows, w->q.get(), v, vold, st);
            CR_CHECK_LAUNCH();
            precond(ks, vold, zn, false);
            k_minres_wx<D><<<L.grid_rows, kT, 0, ks>>>(nrows, z, ww, wold, x, st);
            CR_CHECK_LAUNCH();
        };
        while (w->hst->flag == FLAG_RUN) {
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() { return true; });
            int64_t dit = w->hst->iters - it0;
            L.launches += 5 * kk;
            L.spmvs += dit;
            true_residual<D>(L, x, w->t.get());
            read_state(w, s);
            const double tr = sqrt(w->hst->rr);
            if (tr <= rtol * bnorm) { w->hst->flag = FLAG_CONV; break; }
            if (w->hst->flag != FLAG_RUN) {
                status = w->hst->flag == FLAG_BREAK ? CR_ERR_BREAKDOWN : CR_ERR_STAGNATION;
                break;
            }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_MINRES_ABSJACOBI) {
        ensure_extra(w, s);
        const double *M = h->absdinv.get();
        double *va = w->v.get(), *vb = w->v2.get(), *za = w->z.get(), *zb = w->z2.get();
        double *wa = w->w.get(), *wb = w->w2.get();
        // v = b - G x
        true_residual<D>(L, x, va);
        k_minres_init<D><<<L.grid_rows, kT, 0, s>>>(nrows, va, za, M, wa, wb, vb, st, part);
        CR_CHECK_LAUNCH();
        ++L.launches;
        read_state(w, s);
        const double bnorm = sqrt(w->hst->bb);
        // iteration j uses (v=va, vold=vb, z=za, znew->zb, w=wa, wold->wb) then swaps
        auto body = [&](int i) {
            double *v = (i & 1) ? vb : va, *vold = (i & 1) ? va : vb;
            double *z = (i & 1) ? zb : za, *zn = (i & 1) ? za : zb;
            double *ww = (i & 1) ? wb : wa, *wold = (i & 1) ? wa : wb;
            k_minres_spmv<D><<<L.grid_rows, kT, 0, ks>>>(ell<D>(h), z, w->q.get(), st, part);
            k_minres_lanczos<D><<<L.grid_rows, kT, 0, ks>>>(nrows, w->q.get(), v, vold, zn, M, st, part);
            k_minres_wx<D><<<L.grid_rows, kT, 0, ks>>>(nrows, z, ww, wold, x, st);
            CR_CHECK_LAUNCH();
        };
        while (w->hst->flag == FLAG_RUN) {
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() { return true; });
            int64_t dit = w->hst->iters - it0;
            L.launches += 3 * kk;
            L.spmvs += dit;
            // true residual check every graph replay (r goes to the scratch t buffer)
            true_residual<D>(L, x, w->t.get());
            read_state(w, s);
            const double tr = sqrt(w->hst->rr);
            if (tr <= rtol * bnorm) { w->hst->flag = FLAG_CONV; break; }
            if (w->hst->flag != FLAG_RUN) {
                status = w->hst->flag == FLAG_BREAK ? CR_ERR_BREAKDOWN : CR_ERR_STAGNATION;
                break;
            }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_BICGSTAB_JACOBI) {
        ensure_extra(w, s);
        const double *M = h->dinv.get();
        true_residual<D>(L, x, w->r.get());
        k_bicg_init<D><<<L.grid_rows, kT, 0, s>>>(nrows, w->r.get(), w->rhat.get(), w->p.get(), w->v.get(), rtol, st, part);
        CR_CHECK_LAUNCH();
        ++L.launches;
        read_state(w, s);
        auto body = [&](int) {
            k_bicg_pdir<D><<<L.grid_rows, kT, 0, ks>>>(nrows, w->r.get(), w->p.get(), w->v.get(), w->y.get(), M, st);
            k_bicg_spmv1<D><<<L.grid_rows, kT, 0, ks>>>(ell<D>(h), w->y.get(), w->v.get(), w->rhat.get(), st, part);
            k_bicg_s<D><<<L.grid_rows, kT, 0, ks>>>(nrows, w->r.get(), w->v.get(), w->z.get(), M, st);
            k_bicg_spmv2<D><<<L.grid_rows, kT, 0, ks>>>(ell<D>(h), w->z.get(), w->t.get(), w->r.get(), st, part);
            k_bicg_xr<D><<<L.grid_rows, kT, 0, ks>>>(nrows, x, w->r.get(), w->y.get(), w->z.get(), w->t.get(),
                                                   w->rhat.get(), st, part);
            CR_CHECK_LAUNCH();
        };
        while (w->hst->flag == FLAG_RUN) {
            int64_t it0 = w->hst->iters;
            graph_loop(L, ks, method * 100000 + L.mf * 50000 + kk, kk, body, [&]() {
                return w->hst->flag != FLAG_RUN || w->hst->iters >= max_iter;
            });
            int64_t dit = w->hst->iters - it0;
            L.launches += 5 * ((dit + kk - 1) / kk) * kk;
            L.spmvs += 2 * dit;
            if (w->hst->flag == FLAG_CONV) {
                true_residual<D>(L, x, w->t.get());
                read_state(w, s);
                if (w->hst->rr <= w->hst->tol2 || replacements >= 8) { w->hst->flag = FLAG_CONV; break; }
                ++replacements;   // restart from the true residual
                true_residual<D>(L, x, w->r.get());
                k_bicg_init<D><<<L.grid_rows, kT, 0, s>>>(nrows, w->r.get(), w->rhat.get(), w->p.get(), w->v.get(), rtol, st, part);
                CR_CHECK_LAUNCH();
                read_state(w, s);
                continue;
            }
            if (w->hst->flag == FLAG_BREAK) { status = CR_ERR_BREAKDOWN; break; }
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
        }
    } else if (method == CR_GMRES_JACOBI) {
        ensure_extra(w, s);
        const double *M = h->dinv.get();
        int m = o.restart > 0 ? o.restart : 50;
        CR_REQUIRE(m <= kMaxRestart, CR_ERR_INVALID_ARG, "GMRES restart must be <= 128");
        if (w->V.n < (size_t)(m + 1) * N) w->V.alloc((size_t)(m + 1) * N, s);
        double *V = w->V.get();
        double best = INFINITY;
        int stagn = 0;
        auto cycle = [&](int) {
            for (int k = 0; k < m; ++k) {
                double *Vk = V + (int64_t)k * N;
                k_scale<<<L.grid_vec, kT, 0, ks>>>(N, M, Vk, w->y.get(), st);
                k_spmv_guard<D><<<L.grid_rows, kT, 0, ks>>>(ell<D>(h), w->y.get(), w->w.get(), st);
                k_gmres_dots<<<L.grid_vec, kT, 0, ks>>>(N, k, V, w->w.get(), st, part, 0);
                k_gmres_orth<<<L.grid_vec, kT, 0, ks>>>(N, k, V, w->w.get(), st, 0);
                k_gmres_keep_h<<<1, 32, 0, ks>>>(st, k);
                k_gmres_dots<<<L.grid_vec, kT, 0, ks>>>(N, k, V, w->w.get(), st, part, 1);
                k_gmres_orth<<<L.grid_vec, kT, 0, ks>>>(N, k, V, w->w.get(), st, 1);
                k_gmres_norm_givens<<<L.grid_vec, kT, 0, ks>>>(N, k, w->w.get(), st, part);
                k_gmres_next<<<L.grid_vec, kT, 0, ks>>>(N, w->w.get(), V + (int64_t)(k + 1) * N, st);
                CR_CHECK_LAUNCH();
            }
        };
        while (true) {
            true_residual<D>(L, x, w->r.get());
            read_state(w, s);
            const double rn = sqrt(w->hst->rr);
            if (w->hst->bb == 0.0 || rn <= rtol * sqrt(w->hst->bb)) break;
            if (rn >= best * (1.0 - 1e-12)) { if (++stagn >= 2) { status = CR_ERR_STAGNATION; break; } }
            else stagn = 0;
            best = fmin(best, rn);
            if (w->hst->iters >= max_iter) { status = CR_ERR_NOT_CONVERGED; break; }
            // set tol2 then start the cycle
            KState tmp = *w->hst;
            tmp.tol2 = rtol * rtol * tmp.bb;
            CR_CUDA(cudaMemcpyAsync(&st->tol2, &tmp.tol2, sizeof(double), cudaMemcpyHostToDevice, s));
            k_gmres_start<<<L.grid_vec, kT, 0, s>>>(N, w->r.get(), V, st);
            CR_CHECK_LAUNCH();
            graph_loop(L, ks, method * 100000 + m, 1, cycle, [&]() { return true; });
            k_gmres_solve_y<<<1, 32, 0, s>>>(st);
            k_gmres_update_x<<<L.grid_vec, kT, 0, s>>>(N, V, M, x, st);
            CR_CHECK_LAUNCH();
            read_state(w, s);
            L.launches += 9 * m + 3;
            L.spmvs += w->hst->k + 1;
        }
    } else {
        throw Error(CR_ERR_INVALID_ARG, "unknown solver method");
    }
    CR_CUDA(cudaEventRecord(w->e1, s));
    // final true residual
    true_residual<D>(L, x, w->t.get());
    read_state(w, s);
    float ms = 0.f;
    CR_CUDA(cudaEventElapsedTime(&ms, w->e0, w->e1));
    float ms_setup = 0.f;
    CR_CUDA(cudaEventElapsedTime(&ms_setup, w->e0, w->es));
    const double bn = sqrt(w->hst->bb);
    const double tr = bn > 0 ? sqrt(w->hst->rr) / bn : 0.0;
    if (L.so) {
        k_so_scatter<D><<<L.grid_rows, kT, 0, s>>>(nrows, h->so.perm.get(), x, W);
        CR_CHECK_LAUNCH();
    } else {
        CR_CUDA(cudaMemcpyAsync(W, x, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    CR_CUDA(cudaStreamSynchronize(s));
    if (status == CR_OK && !(tr <= rtol)) status = CR_ERR_NOT_CONVERGED;
    if (rep) {
        rep->iterations = w->hst->iters;
        rep->rel_res_true = tr;
        rep->rel_res_recursive = (method == CR_MINRES_ABSJACOBI || method == CR_MINRES_AFW || method == CR_MINRES_AFW2)
                                     ? fabs(w->hst->eta) / (w->hst->eta0 > 0 ? w->hst->eta0 : 1.0)
                                     : tr;
        rep->converged = status == CR_OK;
        rep->status = status;
        rep->seconds = ms * 1e-3;
        rep->spmv_calls = L.spmvs;
        rep->kernel_launches = L.launches;
        rep->inner_iterations = 0;
        rep->kappa_lanczos_est = rep->lambda_min_est = rep->lambda_max_est = 0.0;
        rep->refine_rounds = 0;
        rep->setup_seconds = ms_setup * 1e-3;
        rep->bytes_moved = iter_bytes(h, o) * (double)w->hst->iters;
        if (pcg_family && w->hst->iters > 1) lanczos_kappa(w, s, w->hst->iters, rep);
    }
    if (status != CR_OK) throw Error(status, "solver did not converge (see report)");
}

__global__ void k_scale_plain(int64_t n, const double *M, const double *a, double *out) {
    GRID_STRIDE(i, n) out[i] = M[i] * a[i];
}

template <int D>
__global__ void k_block_apply(int64_t nrows, const double *M, const double *r, double *z) {
    GRID_STRIDE(row, nrows) {
        double rv[D], zv[D];
        ld<D>(r, row, rv);
        apply_prec<D, 1>(M, row, rv, zv);
        stv<D>(z, row, zv);
    }
}

// z = M^{-1} r for the preconditioner of `method` (cr_apply_precond)
template <int D>
static void apply_precond_t(cr_hybrid_s *h, int method, const double *r, double *z, cudaStream_t s) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    ensure_work(h, s);
    SolverWork *w = h->work;
    const int64_t nrows = h->G.nrows, N = w->N;
    Launcher L{h, w, s};
    const int grid = grid_for(nrows, kT);
    switch (method) {
        case CR_PCG_JACOBI:
        case CR_BICGSTAB_JACOBI:
        case CR_GMRES_JACOBI:
            k_scale_plain<<<grid_for(N, kT), kT, 0, s>>>(N, h->dinv.get(), r, z);
            break;
        case CR_MINRES_ABSJACOBI:
            k_scale_plain<<<grid_for(N, kT), kT, 0, s>>>(N, h->absdinv.get(), r, z);
            break;
        case CR_PCG_BLOCKJACOBI:
            k_block_apply<D><<<grid, kT, 0, s>>>(nrows, h->bdinv.get(), r, z);
            break;
        case CR_PCG_AFW2: {
            build_afw(h, AFW_SPD, s);
            // the coarse grid of the last two-level solve, else the default
            const int Hc = h->coarse.requested > 0 ? h->coarse.requested : (D == 2 ? 64 : 16);
            build_coarse(h, Hc, [&](const double *zz, double *Y, int, int ncol, int64_t stride) {
                for (int c = 0; c < ncol; ++c) spmv(h->G, zz + c * stride, Y + c * stride, s);
            }, ApplyGColour(), s);
            if (w->zs.n < (size_t)SLOTS * N) w->zs.alloc((size_t)SLOTS * N, s);
            CR_CUDA(cudaMemsetAsync(w->st.get(), 0, sizeof(KState), s));
            coarse_restrict_solve(h, r, &w->st.get()->qc, w->partials.get(), &w->st.get()->tickets[4], s);
            launch_afw<D, AFW_PCG_INIT>(L, s, r, w->zs.get(), 1e-10);
            CR_CUDA(cudaMemsetAsync(w->st.get(), 0, sizeof(KState), s));   // flag RUN, beta 0: p = z
            k_pcg_pdir_afw2<D, SLOTS><<<grid, kT, 0, s>>>(nrows, z, w->zs.get(), h->coarse.view(), h->coarse.y.get(),
                                                         w->st.get(), 1, nullptr);
            break;
        }
        case CR_PCG_AFW:
        case CR_MINRES_AFW: {
            build_afw(h, method == CR_PCG_AFW ? AFW_SPD : AFW_ABS, s);
            if (w->zs.n < (size_t)SLOTS * N) w->zs.alloc((size_t)SLOTS * N, s);
            CR_CUDA(cudaMemsetAsync(w->st.get(), 0, sizeof(KState), s));
            launch_afw<D, AFW_PCG_INIT>(L, s, r, w->zs.get(), 1e-10);
            k_afw_zsum<D, SLOTS><<<grid, kT, 0, s>>>(nrows, z, w->zs.get(), w->st.get(), 0);
            break;
        }
        default:
            throw Error(CR_ERR_INVALID_ARG, "unknown preconditioner method");
    }
    CR_CHECK_LAUNCH();
}

// y = G x on a partitioned handle: x (owned rows) -> work vector, halo, SpMV of the owned rows
template <int D>
static void spmv_part_t(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s) {
    ensure_work(h, s);
    SolverWork *w = h->work;
    Launcher L{h, w, s};
    L.D = D;
    L.dist = 1;
    L.comm = h->comm->impl;
    double *xt = w->t.get();
    CR_CUDA(cudaMemcpyAsync(xt, x, w->N * sizeof(double), cudaMemcpyDeviceToDevice, s));
    L.halo(s, xt);
    spmv(h->G, xt, y, s);
}

void spmv_part(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s) {
    if (h->G.d == 2) spmv_part_t<2>(h, x, y, s);
    else spmv_part_t<3>(h, x, y, s);
}

// y = G_mf x (matrix-free factored operator); on a partitioned handle x holds the owned rows and
// the ghosts come by the halo exchange (a collective: every rank calls it)
template <int D>
static void spmv_mf_t(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s) {
    ensure_work(h, s);
    build_mf(h, s);
    SolverWork *w = h->work;
    Launcher L{h, w, s};
    L.D = D;
    L.nrows = h->G.nrows;
    L.N = w->N;
    const double *xin = x;
    if (h->part.on) {
        L.dist = 1;
        L.comm = h->comm->impl;
        double *xt = w->t.get();
        CR_CUDA(cudaMemcpyAsync(xt, x, w->N * sizeof(double), cudaMemcpyDeviceToDevice, s));
        L.halo(s, xt);
        xin = xt;
    }
    mf_apply<D, false>(L, s, xin, y, 0.0);
}

void spmv_mf(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s) {
    if (h->G.d == 2) spmv_mf_t<2>(h, x, y, s);
    else spmv_mf_t<3>(h, x, y, s);
}

void apply_precond(cr_hybrid_s *h, int method, const double *r, double *z, cudaStream_t s) {
    if (h->G.d == 2) apply_precond_t<2>(h, method, r, z, s);
    else apply_precond_t<3>(h, method, r, z, s);
}

// Per-kernel device times of the patch-preconditioned PCG iteration (cr_solve_profile): the kernels
// of one iteration launched on the handle's own buffers exactly as the solve launches them (same
// row order, same grids), each timed alone with CUDA events on s.  The solver state is zeroed
// before every launch (flag RUN), so every launch does its full work; the numbers it computes are
// discarded.
template <int D>
static void profile_t(cr_hybrid_s *h, const cr_solver_opts &o, int nrep, double *ms, cudaStream_t s) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    SolverWork *w = h->work;
    CR_REQUIRE(w && w->zs.n >= (size_t)SLOTS * w->N && h->afw.built == AFW_SPD && o.matrix_free && h->mf.built &&
                   !h->part.on && (o.method == CR_PCG_AFW2 ? h->coarse.built > 0 : o.method == CR_PCG_AFW),
               CR_ERR_INVALID_ARG, "cr_solve_profile: run cr_solve with the same (matrix-free, patch PCG) options first");
    Launcher L{h, w, s};
    L.D = D;
    L.nrows = h->G.nrows;
    L.N = w->N;
    L.grid_rows = grid_for(L.nrows, kT);
    L.grid_vec = grid_for(L.N, kT);
    L.mf = 1;
    const char *eso = std::getenv("CR_SOLVE_ORDER");
    L.so = (h->so.built && !(eso && atoi(eso) == 0)) ? 1 : 0;
    if (L.so) {
        afw_so(h, s);
        coarse_so(h, s);
    }
    const int64_t N = w->N, nrows = L.nrows;
    KState *st = w->st.get();
    double *part = w->partials.get(), *x = w->x.get(), *zs = w->zs.get();
    const CoarseView CV = L.so ? h->coarse.view_so() : h->coarse.view();
    double *yc = h->coarse.y.get();
    const bool two = o.method == CR_PCG_AFW2;
    const double rtol = 1e-30;
    cudaEvent_t a, b;
    CR_CUDA(cudaEventCreate(&a));
    CR_CUDA(cudaEventCreate(&b));
    auto timed = [&](auto launch) {
        double tot = 0.0;
        for (int k = 0; k < nrep; ++k) {
            CR_CUDA(cudaMemsetAsync(st, 0, kStateHeader, s));
            CR_CUDA(cudaEventRecord(a, s));
            launch();
            CR_CUDA(cudaEventRecord(b, s));
            CR_CUDA(cudaEventSynchronize(b));
            float t = 0.f;
            CR_CUDA(cudaEventElapsedTime(&t, a, b));
            tot += t;
        }
        return tot / nrep;
    };
    ms[0] = timed([&] { mf_apply<D, true>(L, s, w->p.get(), w->q.get(), rtol, two ? FIN_PQ2 : FIN_PQ); });
    ms[1] = timed([&] {
        k_pcg_update_r<false><<<occ_grid(k_pcg_update_r<false>, kT, L.N / 2), kT, 0, s>>>(N, x, w->r.get(), w->p.get(),
                                                                                         w->q.get(), st, part, 0);
        CR_CHECK_LAUNCH();
    });
    ms[2] = two ? timed([&] { coarse_restrict_solve(h, w->r.get(), &st->qc, part, &st->tickets[4], s, false, L.so); })
                : 0.0;
    if (two) ms[3] = timed([&] { launch_afw<D, AFW_PCG2>(L, s, w->r.get(), zs, rtol); });
    else ms[3] = timed([&] { launch_afw<D, AFW_PCG>(L, s, w->r.get(), zs, rtol); });
    if (two)
        ms[4] = timed([&] {
            k_pcg_pdir_afw2<D, SLOTS><<<occ_grid(k_pcg_pdir_afw2<D, SLOTS>, kT, nrows), kT, 0, s>>>(nrows, w->p.get(), zs, CV,
                                                                                                 yc, st, 0, x);
            CR_CHECK_LAUNCH();
        });
    else
        ms[4] = timed([&] {
            k_pcg_pdir_afw<D, SLOTS><<<occ_grid(k_pcg_pdir_afw<D, SLOTS>, kT, nrows), kT, 0, s>>>(nrows, w->p.get(), zs, st, x);
            CR_CHECK_LAUNCH();
        });
    CR_CUDA(cudaEventDestroy(a));
    CR_CUDA(cudaEventDestroy(b));
    CR_CUDA(cudaMemsetAsync(st, 0, sizeof(KState), s));
    CR_CUDA(cudaStreamSynchronize(s));
}

void solve_profile(cr_hybrid_s *h, const cr_solver_opts &o, int nrep, double *ms, cudaStream_t s) {
    if (h->G.d == 2) profile_t<2>(h, o, nrep, ms, s);
    else profile_t<3>(h, o, nrep, ms, s);
}

void solve_rhs(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep,
               const double *rhs) {
    if (h->G.d == 2) solve_t<2>(h, o, W, s, rep, rhs);
    else solve_t<3>(h, o, W, s, rep, rhs);
}

}  // namespace cr
