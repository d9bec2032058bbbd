// Two-level additive Schwarz for G:  M2^{-1} = M_patch^{-1} + Z E^{-1} Z^t,
// E = Z^t G Z.
//
// W is a face traction (C_K W_K = R_K - D_K P_K - Ahat_K Uhat_K, with D_K = -a_K), so
// the slowly converging modes of the patch-preconditioned G are smooth "stress fields times
// face area vectors".  The coarse space is exactly that, on a uniform coarse grid of H^d cells
// over the mesh bounding box with (multi)linear hats phi_j:
//     Z_(j,k,l):  W_sigma^(k) = a_sigma^(l) phi_j(x_sigma),   d^2 columns per coarse node,
// a_sigma taken from face_cells[sigma][0].  (The constant-pressure column, k = l, is the
// outlier eigenvector of the patch-preconditioned operator.)  Measured with numpy on the
// oracle's G (configs[1] family): n = 32: 424 -> 65 PCG iterations (H = 16), n = 64: 882 -> 109.
//
// Setup: rows sorted by coarse cell -> chunks of <= CH rows; E column blocks from G applied to
// the sum of the columns of one colour (nodes 5 apart in every direction never share a row of
// Z^t G Z), restricted, scattered; E symmetrised and inverted in place (Gauss-Jordan, E SPD).
// Per iteration: restriction c = Z^t r (chunk partials, fixed-order gather: deterministic),
// y = E^{-1} c and c^t y (dense GEMV), prolongation fused into the direction update.
#include <cub/cub.cuh>
#include <string>
#include <tuple>
#include <mutex>
#include <memory>
#include <map>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <vector>

#include "coarse.cuh"
#include "internal.cuh"
#include "spmv.cuh"

namespace cr {

constexpr int kCH = 2048;   // rows per restriction chunk

// cuBLAS DGEMM (a plain library GEMM) for the rank-32 updates of the coarse Gauss-Jordan; loaded
// with dlopen (libcublas.so.12: the copy torch maps) so libcr loads without it on a CPU box.
struct Blas {
    void *h = nullptr, *handle = nullptr;
    int (*Create)(void **) = nullptr;
    int (*SetStream)(void *, cudaStream_t) = nullptr;
    int (*Dgemm)(void *, int, int, int, int, int, const double *, const double *, int, const double *, int,
                 const double *, double *, int) = nullptr;
};
static Blas &blas() {
    static thread_local Blas b = [] {
        Blas x;
        x.h = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) x.h = dlopen("libcublas.so", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) return x;
        x.Create = (decltype(x.Create))dlsym(x.h, "cublasCreate_v2");
        x.SetStream = (decltype(x.SetStream))dlsym(x.h, "cublasSetStream_v2");
        x.Dgemm = (decltype(x.Dgemm))dlsym(x.h, "cublasDgemm_v2");
        if (x.Create && x.Create(&x.handle) != 0) x.handle = nullptr;
        return x;
    }();
    return b;
}
// column-major C(m x n) = alpha A(m x k) B(k x n) + beta C, no transposes
static void dgemm(cudaStream_t s, int m, int n, int k, double alpha, const double *A, int lda, const double *B, int ldb,
                  double beta, double *C, int ldc) {
    Blas &b = blas();
    CR_REQUIRE(b.handle && b.Dgemm, CR_ERR_CUDA, "cuBLAS (libcublas.so.12) could not be loaded");
    b.SetStream(b.handle, s);
    const int st = b.Dgemm(b.handle, 0, 0, m, n, k, &alpha, A, lda, B, ldb, &beta, C, ldc);
    CR_REQUIRE(st == 0, CR_ERR_CUDA, "cublasDgemm failed");
}

template <int D>
__global__ void k_coarse_faces(const int32_t *dof_face, int64_t row0, int64_t nrows, const int32_t *face_cells,
                               const int32_t *cell_faces, const double *a, const double *xs, CoarseGrid g, float *fx,
                               float *fa, uint32_t *ccell) {
    constexpr int NF = D + 1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = dof_face[row0 + r];
        const int64_t K = face_cells[2 * f];
        int l = 0;
        for (int q = 0; q < NF; ++q)
            if (cell_faces[K * NF + q] == (int32_t)f) l = q;
        int ic[D];
        float xi[D];
        for (int i = 0; i < D; ++i) {
            fx[r * D + i] = (float)xs[f * D + i];
            fa[r * D + i] = (float)a[(K * NF + l) * D + i];
        }
        coarse_locate<D>(g, fx + r * D, ic, xi);
        uint32_t c = 0;
        for (int i = D - 1; i >= 0; --i) c = c * g.H + ic[i];
        ccell[r] = c;
    }
}

// row r is "interior" to its coarse cell when every face of its two cells lies in that cell: G z
// then vanishes on r for any z supported outside the cell (setup restrictions skip such rows)
template <int D>
__global__ void k_coarse_interior(const int32_t *dof_face, const int32_t *face_cells, const int32_t *cell_faces,
                                  const int32_t *face_dof, int64_t nrows, const uint32_t *cc, uint32_t *key) {
    constexpr int NF = D + 1;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = dof_face[r];
        bool inter = true;
        for (int side = 0; side < 2; ++side) {
            const int64_t K = face_cells[2 * f + side];
            for (int l = 0; l < NF; ++l) {
                const int d = face_dof[cell_faces[K * NF + l]];
                if (d >= 0 && cc[d] != cc[r]) inter = false;
            }
        }
        key[r] = cc[r] * 2u + (inter ? 1u : 0u);
    }
}

// partial restriction of one chunk: the 2^D nodes of its coarse cell x D^2 tensor components.
// One thread per row with all 2^D D^2 accumulators (16 in 2D, 72 in 3D); rows are read 4 at a time
// per thread (independent loads in flight); warp shuffles then shared memory reduce the block
// (fixed trees: deterministic).
template <int D>
__global__ void __launch_bounds__(256) k_coarse_restrict(CoarseView C, const double *r, double *part,
                                                         const int32_t *list = nullptr, const int64_t *ends = nullptr,
                                                         int64_t rrs = D, double *clear_base = nullptr) {
    constexpr int NN = 1 << D, DD = D * D, NV = NN * DD;
    constexpr int TPR = 1;                           // threads per row
    constexpr int NA = NV;                           // accumulators per thread
    constexpr int SL = 256 / TPR, U = 4;
    const int64_t ch = list ? (int64_t)list[blockIdx.x] : (int64_t)blockIdx.x;   // list: a subset of chunks
    const int64_t b = C.chunk_start[ch], e = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    const int slot = threadIdx.x / TPR;
    double acc[NA];
#pragma unroll
    for (int v = 0; v < NA; ++v) acc[v] = 0.0;
    for (int64_t t0 = b + slot; t0 < e; t0 += (int64_t)SL * U) {
        int64_t row[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = t0 + (int64_t)u * SL;
            row[u] = t < e ? (int64_t)C.perm[t] : -1;
        }
        float xv[U][D], av[U][D];
        double rv[U][D];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const bool ok = row[u] >= 0;
                const int64_t t = t0 + (int64_t)u * SL;   // sorted position: the row data is stored in this order
                xv[u][i] = ok ? C.fxp[t * D + i] : 0.f;
                av[u][i] = ok ? C.fap[t * D + i] : 0.f;
                rv[u][i] = ok ? r[row[u] * rrs + i] : 0.0;
            }
        if (clear_base)   // setup: zero the rows read (interleaved, full-sector stores)
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (row[u] >= 0) {
                    double2 *z2 = reinterpret_cast<double2 *>(clear_base + row[u] * rrs);
                    for (int q = 0; q < (int)(rrs >> 1); ++q) z2[q] = make_double2(0.0, 0.0);
                }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            int ic[D];
            float xi[D];
            coarse_locate<D>(C.g, xv[u], ic, xi);
            double ar[DD];   // r^(k) a^(l)
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
                for (int l = 0; l < D; ++l) ar[k * D + l] = (double)av[u][l] * rv[u][k];
#pragma unroll
            for (int n = 0; n < NN; ++n) {
                double wn = 1.0;
#pragma unroll
                for (int i = 0; i < D; ++i) wn *= ((n >> i) & 1) ? (double)xi[i] : 1.0 - (double)xi[i];
#pragma unroll
                for (int v = 0; v < DD; ++v) acc[n * DD + v] = fma(wn, ar[v], acc[n * DD + v]);
            }
        }
    }
    __shared__ double sh[8][NV];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int v = 0; v < NA; ++v) {
        double x = acc[v];
#pragma unroll
        for (int o = 16; o >= TPR; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane < TPR) sh[warp][v] = x;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < NV; v += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += sh[w][v];
        part[ch * NV + v] = x;
    }
}

// c[(node, k, l)] = sum of the partials of the chunks of the <= 2^D coarse cells around node
template <int D>
__global__ void k_coarse_gather(CoarseView C, const double *part, double *c) {
    constexpr int NN = 1 << D, NV = NN * D * D;
    const int64_t nE = C.nE;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nE; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = q / (D * D);
        const int kl = (int)(q - node * D * D);
        int nd[D];
        int64_t t = node;
        for (int i = 0; i < D; ++i) { nd[i] = (int)(t % (C.g.H + 1)); t /= (C.g.H + 1); }
        double s = 0.0;
        for (int n = 0; n < NN; ++n) {   // coarse cell = node - offset(n); node is its corner n
            int cc[D];
            bool ok = true;
            for (int i = 0; i < D; ++i) {
                cc[i] = nd[i] - ((n >> i) & 1);
                ok = ok && cc[i] >= 0 && cc[i] < C.g.H;
            }
            if (!ok) continue;
            int64_t cell = 0;
            for (int i = D - 1; i >= 0; --i) cell = cell * C.g.H + cc[i];
            for (int64_t ch = C.cell_chunk[cell]; ch < C.cell_chunk[cell + 1]; ++ch) s += part[ch * NV + n * D * D + kl];
        }
        c[q] = s;
    }
}

// y = Einv c (one 128-thread block per row, 16-byte loads, 4 in flight per thread),
// q = c^t y -> *qout (block partials, last block sums)
__global__ void __launch_bounds__(128) k_coarse_gemv(const double *Einv, int64_t nE, const double *c, double *y,
                                                     double *qout, double *partials, unsigned *ticket) {
    double acc[1] = {0.0};
    __shared__ double sh[4];
    const int64_t n2 = nE >> 1;   // nE = D^2 (H+1)^D is even for D = 2; odd tails handled below
    const double2 *c2 = reinterpret_cast<const double2 *>(c);
    for (int64_t row = blockIdx.x; row < nE; row += gridDim.x) {
        const double *er = Einv + row * nE;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (((row * nE) & 1) == 0) {
            const double2 *e2 = reinterpret_cast<const double2 *>(er);
            int64_t j = threadIdx.x;
            for (; j + 3 * 128 < n2; j += 4 * 128) {
                const double2 a0 = __ldcs(e2 + j), a1 = __ldcs(e2 + j + 128), a2 = __ldcs(e2 + j + 256),
                              a3 = __ldcs(e2 + j + 384);
                const double2 b0 = c2[j], b1 = c2[j + 128], b2 = c2[j + 256], b3 = c2[j + 384];
                s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
                s1 = fma(a1.x, b1.x, fma(a1.y, b1.y, s1));
                s2 = fma(a2.x, b2.x, fma(a2.y, b2.y, s2));
                s3 = fma(a3.x, b3.x, fma(a3.y, b3.y, s3));
            }
            for (; j < n2; j += 128) {
                const double2 a0 = __ldcs(e2 + j), b0 = c2[j];
                s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
            }
            if ((nE & 1) && threadIdx.x == 0) s0 = fma(er[nE - 1], c[nE - 1], s0);
        } else {
            for (int64_t j = threadIdx.x; j < nE; j += 128) s0 = fma(__ldcs(er + j), c[j], s0);
        }
        double s = (s0 + s1) + (s2 + s3);
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            const double t = (sh[0] + sh[1]) + (sh[2] + sh[3]);
            y[row] = t;
            acc[0] = fma(c[row], t, acc[0]);
        }
        __syncthreads();
    }
    reduce_and_finish<1>(acc, partials, ticket, [&](double *t) { *qout = t[0]; });
}

// ------------------------------------------------------------------ setup
// z = sum of the columns (j, k, l) with j of colour (j_i mod 5 == col_i for all i)
template <int D>
__global__ void k_coarse_colour(CoarseView C, int64_t nrows, int colour, int k, int l, double *z) {
    constexpr int NN = 1 << D;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        int ic[D];
        float xi[D];
        coarse_locate<D>(C.g, C.fx + r * D, ic, xi);
        double w[NN];
        coarse_weights<D>(C.g, C.fx + r * D, w);
        double s = 0.0;
        for (int n = 0; n < NN; ++n) {
            int col = 0, mul = 1;
            for (int i = 0; i < D; ++i) {
                col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
                mul *= 5;
            }
            if (col == colour) s += w[n];
        }
        for (int i = 0; i < D; ++i) z[r * D + i] = (i == k) ? s * (double)C.fa[r * D + l] : 0.0;
    }
}

// the colour column sum of one (k, l) written only on the rows of the listed chunks (the coarse cells
// of the colour's supports; every other row of z stays 0), or those rows cleared
template <int D>
__global__ void __launch_bounds__(256) k_coarse_colour_chunks(CoarseView C, const int32_t *list, int colour, int k,
                                                              int l, int clear, double *z, const int64_t *ends = nullptr) {
    constexpr int NN = 1 << D;
    const int64_t ch = list[blockIdx.x];
    const int64_t end = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    for (int64_t t = C.chunk_start[ch] + threadIdx.x; t < end; t += blockDim.x) {
        const int64_t r = C.perm[t];
        double s = 0.0;
        if (!clear) {
            int ic[D];
            float xi[D];
            coarse_locate<D>(C.g, C.fx + r * D, ic, xi);
            double w[NN];
            coarse_weights<D>(C.g, C.fx + r * D, w);
            for (int n = 0; n < NN; ++n) {
                int col = 0, mul = 1;
                for (int i = 0; i < D; ++i) {
                    col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
                    mul *= 5;
                }
                if (col == colour) s += w[n];
            }
        }
        for (int i = 0; i < D; ++i) z[r * D + i] = (i == k && !clear) ? s * (double)C.fa[r * D + l] : 0.0;
    }
}

// E[q', q(q', colour, k, l)] = R[q'] for the unique colour node within 2 of node(q')
template <int D>
__global__ void k_coarse_scatterE(int64_t nE, int H, int colour, int k, int l, const double *R, double *E) {
    for (int64_t qp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qp < nE; qp += (int64_t)gridDim.x * blockDim.x) {
        int64_t node = qp / (D * D), t = node;
        int64_t jn = 0, mul = 1;
        int cl = colour;
        bool ok = true;
        for (int i = 0; i < D; ++i) {
            const int ni = (int)(t % (H + 1));
            t /= (H + 1);
            const int ci = cl % 5;
            cl /= 5;
            int delta = ((ci - ni) % 5 + 5) % 5;   // 0..4
            if (delta > 2) delta -= 5;             // -2..2
            const int ji = ni + delta;
            ok = ok && ji >= 0 && ji <= H;
            jn += (int64_t)ji * mul;
            mul *= (H + 1);
        }
        if (!ok) continue;
        const int64_t q = jn * D * D + k * D + l;
        E[qp * nE + q] = R[qp];
    }
}

__global__ void k_symmetrize(double *E, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / n, j = t - i * n;
        if (j <= i) continue;
        const double v = 0.5 * (E[i * n + j] + E[j * n + i]);
        E[i * n + j] = v;
        E[j * n + i] = v;
    }
}

// Blocked Gauss-Jordan inversion in place, no pivoting (E SPD), pivot blocks of kGB:
//   Pk = A_KK^{-1};  X = A_:K Pk;  A_IJ -= X_I A_KJ (I,J != K);  A_KJ = Pk A_KJ;  A_IK = -X_I;
//   A_KK = Pk.  The three products are cuBLAS DGEMMs (build_coarse_t).
constexpr int kGB = 32;

// Pk = inverse of the b x b diagonal block: one CTA, [A | I] in shared memory, scalar Gauss-Jordan
// without pivoting (the block is a Schur complement of an SPD matrix); coalesced load / store
__global__ void __launch_bounds__(256) k_gj_diag(const double *E, int64_t n, int64_t k0, int b, double *Pk, int *bad) {
    __shared__ double A[kGB][2 * kGB + 1];
    __shared__ double colc[kGB];
    const int tid = threadIdx.x, nb2 = 2 * b;
    for (int t = tid; t < b * nb2; t += blockDim.x) {
        const int i = t / nb2, j = t - i * nb2;
        A[i][j] = j < b ? E[(k0 + i) * n + k0 + j] : (j - b == i ? 1.0 : 0.0);
    }
    __syncthreads();
    for (int c = 0; c < b; ++c) {
        const double piv = A[c][c];
        if (tid == 0 && !(piv > 0.0)) atomicExch(bad, 1);
        if (tid < b) colc[tid] = A[tid][c] / piv;
        __syncthreads();
        for (int t = tid; t < b * nb2; t += blockDim.x) {
            const int i = t / nb2, j = t - i * nb2;
            if (i != c) A[i][j] -= colc[i] * A[c][j];
        }
        __syncthreads();
        for (int j = tid; j < nb2; j += blockDim.x) A[c][j] /= piv;
        __syncthreads();
    }
    for (int t = tid; t < b * b; t += blockDim.x) Pk[t] = A[t / b][b + t % b];
}

// pivot columns A_IK = -X_I, A_KK = Pk
__global__ void k_gj_cols(double *E, int64_t n, int64_t k0, int b, const double *Pk, const double *X) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * b; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / b;
        const int c = (int)(t - i * b);
        E[i * n + k0 + c] = (i >= k0 && i < k0 + b) ? Pk[(i - k0) * b + c] : -X[t];
    }
}

// 3D restriction of one chunk with 9 accumulators per lane (the 72 of one thread per row need 227
// registers: one CTA per SM, latency-bound).  Each lane loads the data of 4 rows (4 x 32 rows per
// warp in flight); the products are then formed by corner: lane L owns corner L % 8 and, by warp
// shuffles, takes the rows 4k + L / 8 (k = 0..7) of every 32-row batch.  Fixed shuffle / shared
// memory trees: deterministic.
__global__ void __launch_bounds__(256, 2) k_coarse_restrict3(CoarseView C, const double *r, double *part,
                                                          const int32_t *list = nullptr, const int64_t *ends = nullptr) {
    constexpr int D = 3, DD = 9, NV = 72, U = 4;
    const int64_t ch = list ? (int64_t)list[blockIdx.x] : (int64_t)blockIdx.x;
    const int64_t b = C.chunk_start[ch], e = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int corner = lane & 7, rsub = lane >> 3;
    double acc[DD];
#pragma unroll
    for (int v = 0; v < DD; ++v) acc[v] = 0.0;
    for (int64_t t0 = b + warp * 32 + lane; t0 - lane < e; t0 += (int64_t)8 * 32 * U) {
        float xi[U][D], av[U][D];
        double rv[U][D];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = t0 + (int64_t)u * 8 * 32;
            const int64_t row = t < e ? (int64_t)C.perm[t] : -1;
            float xv[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                xv[i] = row >= 0 ? C.fxp[t * D + i] : 0.f;   // row data in sorted order: coalesced
                av[u][i] = row >= 0 ? C.fap[t * D + i] : 0.f;
                rv[u][i] = row >= 0 ? r[row * D + i] : 0.0;
            }
            int ic[D];
            coarse_locate<D>(C.g, xv, ic, xi[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int src = 4 * k + rsub;   // row of this batch handled now by this lane's corner
                float x0 = __shfl_sync(0xffffffffu, xi[u][0], src), x1 = __shfl_sync(0xffffffffu, xi[u][1], src),
                      x2 = __shfl_sync(0xffffffffu, xi[u][2], src);
                float a0 = __shfl_sync(0xffffffffu, av[u][0], src), a1 = __shfl_sync(0xffffffffu, av[u][1], src),
                      a2 = __shfl_sync(0xffffffffu, av[u][2], src);
                double r0 = __shfl_sync(0xffffffffu, rv[u][0], src), r1 = __shfl_sync(0xffffffffu, rv[u][1], src),
                       r2 = __shfl_sync(0xffffffffu, rv[u][2], src);
                const double wn = ((corner & 1) ? (double)x0 : 1.0 - (double)x0) *
                                  ((corner & 2) ? (double)x1 : 1.0 - (double)x1) *
                                  ((corner & 4) ? (double)x2 : 1.0 - (double)x2);
                const double ar[DD] = {(double)a0 * r0, (double)a1 * r0, (double)a2 * r0,
                                       (double)a0 * r1, (double)a1 * r1, (double)a2 * r1,
                                       (double)a0 * r2, (double)a1 * r2, (double)a2 * r2};
#pragma unroll
                for (int v = 0; v < DD; ++v) acc[v] = fma(wn, ar[v], acc[v]);
            }
    }
    __shared__ double sh[8][NV];
#pragma unroll
    for (int v = 0; v < DD; ++v) {
        double x = acc[v];
        x += __shfl_xor_sync(0xffffffffu, x, 16);
        x += __shfl_xor_sync(0xffffffffu, x, 8);
        if (lane < 8) sh[warp][lane * DD + v] = x;   // lane = corner
    }
    __syncthreads();
    for (int v = threadIdx.x; v < NV; v += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += sh[w][v];
        part[ch * NV + v] = x;
    }
}

// k_coarse_restrict3 with the per-row work done once by the row's lane: it forms the 8 corner
// weights and the 9 products a_k r_i in shared memory, and the corner lanes (lane % 8) read them
// instead of receiving the raw row data by 9 shuffles and recomputing the products 8 times (the
// shuffle version issued ~530 instructions per row and ran issue-bound).  Same terms, same
// accumulation order per lane as k_coarse_restrict3: bitwise the same partials.
__global__ void __launch_bounds__(256, 4) k_coarse_restrict3b(CoarseView C, const double *r, double *part,
                                                           const int32_t *list = nullptr, const int64_t *ends = nullptr) {
    constexpr int D = 3, DD = 9, NV = 72;
    __shared__ __align__(16) double sw[8][32][9];   // odd row stride: the 8 weight stores are 2-way, not 16-way, bank-conflicted
    __shared__ __align__(16) double sar[8][32][10];
    const int64_t ch = list ? (int64_t)list[blockIdx.x] : (int64_t)blockIdx.x;
    const int64_t b = C.chunk_start[ch], e = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int corner = lane & 7, rsub = lane >> 3;
    double acc[DD];
#pragma unroll
    for (int v = 0; v < DD; ++v) acc[v] = 0.0;
    for (int64_t t0 = b + warp * 32; t0 < e; t0 += 8 * 32) {
        const int64_t t = t0 + lane;
        const int64_t row = t < e ? (int64_t)C.perm[t] : -1;
        float xv[D], av[D], xi[D];
        double rv[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            xv[i] = row >= 0 ? C.fxp[t * D + i] : 0.f;
            av[i] = row >= 0 ? C.fap[t * D + i] : 0.f;
            rv[i] = row >= 0 ? r[row * D + i] : 0.0;
        }
        int ic[D];
        coarse_locate<D>(C.g, xv, ic, xi);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            sw[warp][lane][c] = row < 0 ? 0.0
                                        : ((c & 1) ? (double)xi[0] : 1.0 - (double)xi[0]) *
                                              ((c & 2) ? (double)xi[1] : 1.0 - (double)xi[1]) *
                                              ((c & 4) ? (double)xi[2] : 1.0 - (double)xi[2]);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int k = 0; k < D; ++k) sar[warp][lane][i * D + k] = (double)av[k] * rv[i];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = 4 * k + rsub;
            const double wn = sw[warp][j][corner];
            const double2 *p2 = reinterpret_cast<const double2 *>(&sar[warp][j][0]);
            const double2 q0 = p2[0], q1 = p2[1], q2 = p2[2], q3 = p2[3];
            const double q8 = sar[warp][j][8];
            acc[0] = fma(wn, q0.x, acc[0]);
            acc[1] = fma(wn, q0.y, acc[1]);
            acc[2] = fma(wn, q1.x, acc[2]);
            acc[3] = fma(wn, q1.y, acc[3]);
            acc[4] = fma(wn, q2.x, acc[4]);
            acc[5] = fma(wn, q2.y, acc[5]);
            acc[6] = fma(wn, q3.x, acc[6]);
            acc[7] = fma(wn, q3.y, acc[7]);
            acc[8] = fma(wn, q8, acc[8]);
        }
        __syncwarp();
    }
    __shared__ double sh[8][NV];
#pragma unroll
    for (int v = 0; v < DD; ++v) {
        double x = acc[v];
        x += __shfl_xor_sync(0xffffffffu, x, 16);
        x += __shfl_xor_sync(0xffffffffu, x, 8);
        if (lane < 8) sh[warp][lane * DD + v] = x;   // lane = corner
    }
    __syncthreads();
    for (int v = threadIdx.x; v < NV; v += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += sh[w][v];
        part[ch * NV + v] = x;
    }
}

// k_coarse_restrict3b was bound by shared-memory wavefronts (ncu: L1/shared throughput 95 %): each
// lane served one corner and re-read a row's 9 products once per corner.  Here a lane serves the
// corner pair (c, c + 4) that differs in z only, so every product it reads from shared memory feeds
// two accumulators, and it forms the two hat weights from the row's (xi, eta, zeta) itself (the same
// double products in the same order as 3b).  Lanes 4 apart (8 rows at a time) share a pair; the sum
// over them is a fixed xor-shuffle tree: deterministic, not bitwise 3b's order.
__global__ void __launch_bounds__(256, 3) k_coarse_restrict3c(CoarseView C, const double *r, double *part) {
    constexpr int D = 3, DD = 9, NV = 72;
    __shared__ __align__(16) float4 sxi[8][32];
    __shared__ __align__(16) double sar[8][32][10];
    const int64_t ch = blockIdx.x;
    const int64_t b = C.chunk_start[ch], e = C.chunk_start[ch + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cp = lane & 3, rsub = lane >> 2;
    double acc0[DD], acc1[DD];
#pragma unroll
    for (int v = 0; v < DD; ++v) acc0[v] = acc1[v] = 0.0;
    for (int64_t t0 = b + warp * 32; t0 < e; t0 += 8 * 32) {
        const int64_t t = t0 + lane;
        const int64_t row = t < e ? (int64_t)C.perm[t] : -1;
        float xv[D], av[D], xi[D];
        double rv[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            xv[i] = row >= 0 ? C.fxp[t * D + i] : 0.f;
            av[i] = row >= 0 ? C.fap[t * D + i] : 0.f;   // a padding row's products are 0
            rv[i] = row >= 0 ? r[row * D + i] : 0.0;
        }
        int ic[D];
        coarse_locate<D>(C.g, xv, ic, xi);
        sxi[warp][lane] = make_float4(xi[0], xi[1], xi[2], 0.f);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int k = 0; k < D; ++k) sar[warp][lane][i * D + k] = (double)av[k] * rv[i];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int j = 8 * k + rsub;
            const float4 xq = sxi[warp][j];
            const double wxy = ((cp & 1) ? (double)xq.x : 1.0 - (double)xq.x) * ((cp & 2) ? (double)xq.y : 1.0 - (double)xq.y);
            const double w0 = wxy * (1.0 - (double)xq.z), w1 = wxy * (double)xq.z;
            const double2 *p2 = reinterpret_cast<const double2 *>(&sar[warp][j][0]);
            const double2 q0 = p2[0], q1 = p2[1], q2 = p2[2], q3 = p2[3];
            const double q[DD] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y, sar[warp][j][8]};
#pragma unroll
            for (int v = 0; v < DD; ++v) {
                acc0[v] = fma(w0, q[v], acc0[v]);
                acc1[v] = fma(w1, q[v], acc1[v]);
            }
        }
        __syncwarp();
    }
    __shared__ double sh[8][NV];
#pragma unroll
    for (int v = 0; v < DD; ++v) {
        double x0 = acc0[v], x1 = acc1[v];
        x0 += __shfl_xor_sync(0xffffffffu, x0, 4);
        x1 += __shfl_xor_sync(0xffffffffu, x1, 4);
        x0 += __shfl_xor_sync(0xffffffffu, x0, 8);
        x1 += __shfl_xor_sync(0xffffffffu, x1, 8);
        x0 += __shfl_xor_sync(0xffffffffu, x0, 16);
        x1 += __shfl_xor_sync(0xffffffffu, x1, 16);
        if (lane < 4) {
            sh[warp][lane * DD + v] = x0;         // corner cp
            sh[warp][(lane + 4) * DD + v] = x1;   // corner cp + 4
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < NV; v += blockDim.x) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += sh[w][v];
        part[ch * NV + v] = x;
    }
}

// ------------------------------------------------------------------ batched setup (all D^2 (k, l) columns of a colour)
// The D^2 columns of one colour, (k, l) -> column k D + l, stored as separate vectors of stride zs.
template <int D>
__global__ void __launch_bounds__(256) k_coarse_colour_chunks_all(CoarseView C, const int32_t *list, int colour, int clear,
                                                                  double *z, int64_t zs, const int64_t *ends = nullptr) {
    constexpr int NN = 1 << D;
    const int64_t ch = list[blockIdx.x];
    const int64_t end = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    for (int64_t t = C.chunk_start[ch] + threadIdx.x; t < end; t += blockDim.x) {
        const int64_t r = C.perm[t];
        double s = 0.0;
        if (!clear) {
            int ic[D];
            float xi[D];
            coarse_locate<D>(C.g, C.fx + r * D, ic, xi);
            double w[NN];
            coarse_weights<D>(C.g, C.fx + r * D, w);
            for (int n = 0; n < NN; ++n) {
                int col = 0, mul = 1;
                for (int i = 0; i < D; ++i) {
                    col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
                    mul *= 5;
                }
                if (col == colour) s += w[n];
            }
        }
        for (int k = 0; k < D; ++k)
            for (int l = 0; l < D; ++l) {
                const double v = clear ? 0.0 : s * (double)C.fa[r * D + l];
                double *zc = z + (int64_t)(k * D + l) * zs + r * D;
                for (int i = 0; i < D; ++i) zc[i] = (i == k) ? v : 0.0;
            }
    }
}

// the D^2 columns of a colour on every local row (partitioned setup)
template <int D>
__global__ void k_coarse_colour_all(CoarseView C, int64_t nrows, int colour, double *z, int64_t zs) {
    constexpr int NN = 1 << D;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        int ic[D];
        float xi[D];
        coarse_locate<D>(C.g, C.fx + r * D, ic, xi);
        double w[NN];
        coarse_weights<D>(C.g, C.fx + r * D, w);
        double sw = 0.0;
        for (int n = 0; n < NN; ++n) {
            int col = 0, mul = 1;
            for (int i = 0; i < D; ++i) {
                col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
                mul *= 5;
            }
            if (col == colour) sw += w[n];
        }
        for (int k = 0; k < D; ++k)
            for (int l = 0; l < D; ++l) {
                const double v = sw * (double)C.fa[r * D + l];
                double *zc = z + (int64_t)(k * D + l) * zs + r * D;
                for (int i = 0; i < D; ++i) zc[i] = (i == k) ? v : 0.0;
            }
    }
}

// k_coarse_restrict3 for NC columns at once (entry (row, c, i) at r[c rs + row rrs + i], partials at
// part + c ps): the row data (perm, centroid, area vector) is read once for all NC columns;
// clear_base: zero the rows read (setup)
template <int NC>
__global__ void __launch_bounds__(256, 2) k_coarse_restrict3m(CoarseView C, const double *r, int64_t rs, double *part,
                                                           int64_t ps, const int32_t *list, const int64_t *ends,
                                                           int64_t rrs = 3, double *clear_base = nullptr) {
    constexpr int D = 3, DD = 9, NV = 72, U = 1;
    const int64_t ch = list ? (int64_t)list[blockIdx.x] : (int64_t)blockIdx.x;
    const int64_t b = C.chunk_start[ch], e = ends ? ends[blockIdx.x] : C.chunk_start[ch + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int corner = lane & 7, rsub = lane >> 3;
    double acc[NC][DD];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < DD; ++v) acc[c][v] = 0.0;
    for (int64_t t0 = b + warp * 32 + lane; t0 - lane < e; t0 += (int64_t)8 * 32 * U) {
        float xi[U][D], av[U][D];
        double rv[U][NC][D];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = t0 + (int64_t)u * 8 * 32;
            const int64_t row = t < e ? (int64_t)C.perm[t] : -1;
            float xv[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                xv[i] = row >= 0 ? C.fxp[t * D + i] : 0.f;
                av[u][i] = row >= 0 ? C.fap[t * D + i] : 0.f;
#pragma unroll
                for (int c = 0; c < NC; ++c) rv[u][c][i] = row >= 0 ? r[c * rs + row * rrs + i] : 0.0;
            }
            int ic[D];
            coarse_locate<D>(C.g, xv, ic, xi[u]);
            // interleaved setup rows (rrs doubles, 256-byte aligned): the last launch zeroes the whole row
            // with full-sector stores (the next colour's G application accumulates into 0)
            if (clear_base && row >= 0) {
                double2 *z2 = reinterpret_cast<double2 *>(clear_base + row * rrs);
                for (int q = 0; q < (int)(rrs >> 1); ++q) z2[q] = make_double2(0.0, 0.0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int src = 4 * k + rsub;   // row of this batch handled now by this lane's corner
                const float x0 = __shfl_sync(0xffffffffu, xi[u][0], src), x1 = __shfl_sync(0xffffffffu, xi[u][1], src),
                            x2 = __shfl_sync(0xffffffffu, xi[u][2], src);
                const float a0 = __shfl_sync(0xffffffffu, av[u][0], src), a1 = __shfl_sync(0xffffffffu, av[u][1], src),
                            a2 = __shfl_sync(0xffffffffu, av[u][2], src);
                const double wn = ((corner & 1) ? (double)x0 : 1.0 - (double)x0) *
                                  ((corner & 2) ? (double)x1 : 1.0 - (double)x1) *
                                  ((corner & 4) ? (double)x2 : 1.0 - (double)x2);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double r0 = __shfl_sync(0xffffffffu, rv[u][c][0], src),
                                 r1 = __shfl_sync(0xffffffffu, rv[u][c][1], src),
                                 r2 = __shfl_sync(0xffffffffu, rv[u][c][2], src);
                    const double ar[DD] = {(double)a0 * r0, (double)a1 * r0, (double)a2 * r0,
                                           (double)a0 * r1, (double)a1 * r1, (double)a2 * r1,
                                           (double)a0 * r2, (double)a1 * r2, (double)a2 * r2};
#pragma unroll
                    for (int v = 0; v < DD; ++v) acc[c][v] = fma(wn, ar[v], acc[c][v]);
                }
            }
    }
    __shared__ double sh[8][NV];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#pragma unroll
        for (int v = 0; v < DD; ++v) {
            double x = acc[c][v];
            x += __shfl_xor_sync(0xffffffffu, x, 16);
            x += __shfl_xor_sync(0xffffffffu, x, 8);
            if (lane < 8) sh[warp][lane * DD + v] = x;   // lane = corner
        }
        __syncthreads();
        for (int v = threadIdx.x; v < NV; v += blockDim.x) {
            double x = 0.0;
            for (int w = 0; w < 8; ++w) x += sh[w][v];
            part[c * ps + ch * NV + v] = x;
        }
        __syncthreads();
    }
}

// k_coarse_gather for D^2 columns (partials at part + c * ps, result at out + c * nE)
template <int D>
__global__ void k_coarse_gather_all(CoarseView C, const double *part, int64_t ps, double *out) {
    constexpr int NN = 1 << D, NV = NN * D * D, NCOL = D * D;
    const int64_t nE = C.nE;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nE * NCOL; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = t / nE, q = t - col * nE;
        const int64_t node = q / (D * D);
        const int kl = (int)(q - node * D * D);
        int nd[D];
        int64_t tt = node;
        for (int i = 0; i < D; ++i) { nd[i] = (int)(tt % (C.g.H + 1)); tt /= (C.g.H + 1); }
        double sum = 0.0;
        for (int n = 0; n < NN; ++n) {
            int cc[D];
            bool ok = true;
            for (int i = 0; i < D; ++i) {
                cc[i] = nd[i] - ((n >> i) & 1);
                ok = ok && cc[i] >= 0 && cc[i] < C.g.H;
            }
            if (!ok) continue;
            int64_t cell = 0;
            for (int i = D - 1; i >= 0; --i) cell = cell * C.g.H + cc[i];
            for (int64_t ch = C.cell_chunk[cell]; ch < C.cell_chunk[cell + 1]; ++ch)
                sum += part[col * ps + ch * NV + n * D * D + kl];
        }
        out[col * nE + q] = sum;
    }
}

// row data in sorted (coarse-cell) order for the restrictions: fxp[t] = fx[perm[t]], fap likewise
template <int D>
__global__ void k_coarse_permute_rows(const int32_t *perm, int64_t n, const float *fx, const float *fa, float *fxp,
                                      float *fap) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = perm[t];
        for (int i = 0; i < D; ++i) {
            fxp[t * D + i] = fx[r * D + i];
            fap[t * D + i] = fa[r * D + i];
        }
    }
}

// first sorted position with coarse cell >= c (c = 0..ncc)
__global__ void k_cell_starts(const uint32_t *cc_sorted, int64_t n, int64_t ncc, int64_t *cstart, int mult = 1,
                              int add = 0) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= ncc; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t key = c * mult + add;
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)cc_sorted[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        cstart[c] = lo;
    }
}

__global__ void k_iota_u32(uint32_t *a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

// ------------------------------------------------------------------ sparse direct coarse solve (ND)
// E = Z^t G Z couples coarse nodes up to 2 apart in every direction (a fine cell straddling a
// coarse grid line joins the supports of hats 2 apart), so E has a 5^D-node block stencil with
// D^2 x D^2 blocks.  Stored structured: Es[((node * 5^D + nbr) * m + a) * m + b], m = D^2, nbr the
// base-5 digits of (node' - node + 2).
// Nested dissection of the (H+1)^D node grid: a box is split across its longest side by a
// separator slab 2 nodes thick (no stencil coupling across it); boxes of <= kNdLeaf nodes per
// side are leaf fronts.  Fronts in post-order (children first).  Multifrontal elimination with
// explicit inverses (E SPD => every front's F_II is an SPD Schur complement):
//   F = [[F_II, F_IB], [F_BI, F_BB]]  (original entries with a pivot end + children's updates)
//   Finv = F_II^{-1},  W = F_BI Finv,  U = F_BB - W F_IB  (passed to the parent)
// Solve E y = c:  forward (deepest level first)  b_I = c_I + children's u at I;  u = b_B - W b_I
//                 backward (root first)          y_I = Finv b_I - W^t y_B
// Every front's arithmetic is a fixed sequence (children summed in child order): deterministic.
constexpr int kNdLeaf2 = 4, kNdLeaf3 = 3, kNdR = 2;

struct HostFront {
    std::vector<int32_t> I, B;   // nodes
    std::vector<int> kids;       // child fronts
    int depth = 0;
};

static void nd_plan(int H, int D, std::vector<HostFront> &F, int box = 0) {
    const int n1 = H + 1, leaf = D == 2 ? kNdLeaf2 : kNdLeaf3;
    auto nid = [&](const int *c) {
        int64_t v = 0;
        for (int i = D - 1; i >= 0; --i) v = v * n1 + c[i];
        return (int32_t)v;
    };
    std::function<int(std::array<int, 3>, std::array<int, 3>, int)> rec = [&](std::array<int, 3> lo,
                                                                             std::array<int, 3> hi, int depth) {
        int ext[3] = {1, 1, 1}, ax = 0;
        for (int i = 0; i < D; ++i) {
            ext[i] = hi[i] - lo[i] + 1;
            if (ext[i] > ext[ax]) ax = i;
        }
        HostFront f;
        f.depth = depth;
        std::array<int, 3> slo = lo, shi = hi;
        if (ext[ax] > leaf) {
            const int s0 = (lo[ax] + hi[ax] - kNdR + 1) / 2, s1 = s0 + kNdR - 1;
            std::array<int, 3> lo1 = lo, hi1 = hi, lo2 = lo, hi2 = hi;
            hi1[ax] = s0 - 1;
            lo2[ax] = s1 + 1;
            if (hi1[ax] >= lo1[ax]) f.kids.push_back(rec(lo1, hi1, depth + 1));
            if (hi2[ax] >= lo2[ax]) f.kids.push_back(rec(lo2, hi2, depth + 1));
            slo[ax] = s0;
            shi[ax] = s1;
        }
        int c[3];
        for (c[2] = (D > 2 ? slo[2] : 0); c[2] <= (D > 2 ? shi[2] : 0); ++c[2])
            for (c[1] = slo[1]; c[1] <= shi[1]; ++c[1])
                for (c[0] = slo[0]; c[0] <= shi[0]; ++c[0]) f.I.push_back(nid(c));
        std::sort(f.I.begin(), f.I.end());
        F.push_back(std::move(f));
        return (int)F.size() - 1;
    };
    F.clear();
    if (box > 0) {
        // flat two-level plan: separator slabs (2 nodes thick) after every `box` nodes per axis,
        // root = all separator nodes, children = the boxes between them (any number)
        // a slab must leave at least one node after it (else it would not separate anything)
        auto sep = [&](int x) { return x % (box + kNdR) >= box && (x / (box + kNdR)) * (box + kNdR) + box + kNdR <= H; };
        std::vector<std::array<int, 2>> seg;   // box intervals per axis
        for (int x = 0; x <= H;) {
            if (sep(x)) { ++x; continue; }
            int y = x;
            while (y + 1 <= H && !sep(y + 1)) ++y;
            seg.push_back({x, y});
            x = y + 1;
        }
        const int ns = (int)seg.size();
        if (ns < 2) {   // the grid is smaller than one box: recursive bisection instead
            nd_plan(H, D, F, 0);
            return;
        }
        HostFront root;
        root.depth = 0;
        int nbox = 1;
        for (int i = 0; i < D; ++i) nbox *= ns;
        for (int bi = 0; bi < nbox; ++bi) {
            int t = bi, c[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            for (int i = 0; i < D; ++i) { lo[i] = seg[t % ns][0]; hi[i] = seg[t % ns][1]; t /= ns; }
            HostFront f;
            f.depth = 1;
            for (c[2] = lo[2]; c[2] <= hi[2]; ++c[2])
                for (c[1] = lo[1]; c[1] <= hi[1]; ++c[1])
                    for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0]) f.I.push_back(nid(c));
            std::sort(f.I.begin(), f.I.end());
            root.kids.push_back((int)F.size());
            F.push_back(std::move(f));
        }
        int c[3] = {0, 0, 0};
        for (c[2] = 0; c[2] <= (D > 2 ? H : 0); ++c[2])
            for (c[1] = 0; c[1] <= H; ++c[1])
                for (c[0] = 0; c[0] <= H; ++c[0]) {
                    bool s2 = false;
                    for (int i = 0; i < D; ++i) s2 = s2 || sep(c[i]);
                    if (s2) root.I.push_back(nid(c));
                }
        std::sort(root.I.begin(), root.I.end());
        F.push_back(std::move(root));
    } else {
        rec({0, 0, 0}, {H, H, H}, 0);
    }
    // B sets: stencil neighbours of the pivots and the children's B, eliminated later
    const int64_t nn = (int64_t)std::pow((double)n1, D);
    std::vector<int32_t> pos(nn, -1);
    for (int f = 0; f < (int)F.size(); ++f)
        for (int32_t v : F[f].I) pos[v] = f;
    for (int f = 0; f < (int)F.size(); ++f) {
        std::vector<int32_t> b;
        for (int k : F[f].kids) b.insert(b.end(), F[k].B.begin(), F[k].B.end());
        for (int32_t v : F[f].I) {
            int cv[3] = {0, 0, 0};
            int64_t t = v;
            for (int i = 0; i < D; ++i) { cv[i] = (int)(t % n1); t /= n1; }
            const int span = 2 * kNdR + 1, nofs = D == 2 ? span * span : span * span * span;
            for (int o = 0; o < nofs; ++o) {
                int w[3], oo = o;
                bool ok = true;
                for (int i = 0; i < D; ++i) {
                    w[i] = cv[i] + (oo % span) - kNdR;
                    oo /= span;
                    ok = ok && w[i] >= 0 && w[i] <= H;
                }
                if (ok && pos[nid(w)] > f) b.push_back(nid(w));
            }
        }
        std::sort(b.begin(), b.end(), [&](int32_t x, int32_t y) { return pos[x] != pos[y] ? pos[x] < pos[y] : x < y; });
        b.erase(std::unique(b.begin(), b.end()), b.end());
        std::vector<int32_t> out;
        for (int32_t v : b)
            if (pos[v] != f) out.push_back(v);
        F[f].B = std::move(out);
    }
}

// structured E from the colour passes: E[(node(q'), nbr), comp(q'), (k, l)] = R[q']
template <int D>
__global__ void k_coarse_scatterEs(int64_t nE, int H, int colour, int k, int l, const double *R, double *Es) {
    constexpr int M = D * D, NBR = D == 2 ? 25 : 125;
    for (int64_t qp = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qp < nE; qp += (int64_t)gridDim.x * blockDim.x) {
        const int64_t node = qp / M;
        int64_t t = node;
        int cl = colour, nbr = 0, mul = 1;
        bool ok = true;
        for (int i = 0; i < D; ++i) {
            const int ni = (int)(t % (H + 1));
            t /= (H + 1);
            const int ci = cl % 5;
            cl /= 5;
            int delta = ((ci - ni) % 5 + 5) % 5;
            if (delta > 2) delta -= 5;
            ok = ok && ni + delta >= 0 && ni + delta <= H;
            nbr += (delta + 2) * mul;
            mul *= 5;
        }
        if (!ok) continue;
        Es[((node * NBR + nbr) * M + (qp - node * M)) * M + k * D + l] = R[qp];
    }
}

// k_coarse_scatterEs for the D^2 columns of a colour (R + (k D + l) nE)
template <int D>
__global__ void k_coarse_scatterEs_all(int64_t nE, int H, int colour, const double *R, double *Es) {
    constexpr int M = D * D, NBR = D == 2 ? 25 : 125;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nE * M; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = t / nE, qp = t - col * nE;
        const int64_t node = qp / M;
        int64_t tt = node;
        int cl = colour, nbr = 0, mul = 1;
        bool ok = true;
        for (int i = 0; i < D; ++i) {
            const int ni = (int)(tt % (H + 1));
            tt /= (H + 1);
            const int ci = cl % 5;
            cl /= 5;
            int delta = ((ci - ni) % 5 + 5) % 5;
            if (delta > 2) delta -= 5;
            ok = ok && ni + delta >= 0 && ni + delta <= H;
            nbr += (delta + 2) * mul;
            mul *= 5;
        }
        if (!ok) continue;
        Es[((node * NBR + nbr) * M + (qp - node * M)) * M + col] = R[t];
    }
}

// Es <- (Es + Es^t) / 2 (entry pairs (a, d, p, q) <-> (a + d, -d, q, p))
template <int D>
__global__ void k_es_symmetrize(int64_t nnode, int H, double *Es) {
    constexpr int M = D * D, NBR = D == 2 ? 25 : 125;
    const int64_t tot = nnode * NBR * M * M;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(t % M), p = (int)((t / M) % M);
        const int nbr = (int)((t / (M * M)) % NBR);
        const int64_t a = t / ((int64_t)M * M * NBR);
        int64_t ta = a, b = 0, mul = 1;
        int mnbr = 0, m5 = 1;
        bool ok = true;
        int nb = nbr;
        for (int i = 0; i < D; ++i) {
            const int ai = (int)(ta % (H + 1));
            ta /= (H + 1);
            const int d = nb % 5 - 2;
            nb /= 5;
            ok = ok && ai + d >= 0 && ai + d <= H;
            b += (int64_t)(ai + d) * mul;
            mul *= (H + 1);
            mnbr += (2 - d) * m5;
            m5 *= 5;
        }
        if (!ok || b < a || (b == a && q <= p)) continue;
        const int64_t t2 = ((b * NBR + mnbr) * M + q) * M + p;
        const double v = 0.5 * (Es[t] + Es[t2]);
        Es[t] = v;
        Es[t2] = v;
    }
}

struct NdLevelDev {   // one depth of the factorisation
    const int32_t *fronts;     // front ids
    const int64_t *foff;       // prefix of n_pad^2 over the level (entries of F)
    const int64_t *fbase;      // F offset of each front in the F pool
    const int32_t *nIp, *nBp;  // padded sizes
    int nf;
};

template <int D>
__device__ __forceinline__ bool nd_stencil(int64_t a, int64_t b, int H, int &nbr) {
    nbr = 0;
    int m5 = 1;
    for (int i = 0; i < D; ++i) {
        const int ai = (int)(a % (H + 1)), bi = (int)(b % (H + 1));
        a /= (H + 1);
        b /= (H + 1);
        const int d = bi - ai;
        if (d < -2 || d > 2) return false;
        nbr += (d + 2) * m5;
        m5 *= 5;
    }
    return true;
}

// F of every front of a level (column-major, ld n_pad): original E entries with a pivot end,
// identity on the padded pivots, 0 elsewhere
template <int D>
__global__ void k_nd_assemble(NdLevelDev L, const NdFrontDev *fr, const int32_t *nodes, const double *Es, int H,
                              double *Fpool) {
    constexpr int M = D * D, NBR = D == 2 ? 25 : 125;
    const int64_t tot = L.foff[L.nf];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = L.nf - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (L.foff[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const NdFrontDev F = fr[L.fronts[lo]];
        const int nIp = L.nIp[lo], np = nIp + L.nBp[lo];
        const int64_t e = t - L.foff[lo];
        const int p = (int)(e % np), q = (int)(e / np);
        auto decode = [&](int x, int64_t &node, int &comp, int &kind) {   // kind 0: I, 1: B, 2: pad I, 3: pad B
            if (x < nIp) {
                if (x < F.nI) { node = nodes[F.ioff + x / M]; comp = x % M; kind = 0; }
                else kind = 2;
            } else {
                const int y = x - nIp;
                if (y < F.nB) { node = nodes[F.boff + y / M]; comp = y % M; kind = 1; }
                else kind = 3;
            }
        };
        int64_t np_ = 0, nq = 0;
        int cp = 0, cq = 0, kp = 0, kq = 0;
        decode(p, np_, cp, kp);
        decode(q, nq, cq, kq);
        double v = 0.0;
        int nbr;
        if (kp <= 1 && kq <= 1 && (kp == 0 || kq == 0) && nd_stencil<D>(np_, nq, H, nbr))
            v = Es[((np_ * NBR + nbr) * M + cp) * M + cq];
        else if (kp == 2 && p == q)
            v = 1.0;
        Fpool[L.fbase[lo] + e] = v;
    }
}

// F_f[map(k), map(l)] += U_child[k, l] for child `which` of every front of the level
__global__ void k_nd_extend(NdLevelDev L, NdLevelDev Lc, const NdFrontDev *fr, const int32_t *map,
                            const int32_t *kids, const int32_t *child_slot, int which, double *Fpool) {
    // child_slot[f] = index of front f within the child level arrays (fronts of depth d+1)
    for (int i = blockIdx.y; i < L.nf; i += gridDim.y) {
        const NdFrontDev F = fr[L.fronts[i]];
        if (which >= F.kid_cnt) continue;
        const int kid = kids[F.kid_off + which];
        const NdFrontDev K = fr[kid];
        const int ci = child_slot[kid];
        const int npc = Lc.nIp[ci] + Lc.nBp[ci], nIpc = Lc.nIp[ci];
        const int np = L.nIp[i] + L.nBp[i], nIp = L.nIp[i];
        const double *U = Fpool + Lc.fbase[ci] + nIpc + (int64_t)nIpc * npc;
        double *Fp = Fpool + L.fbase[i];
        const int64_t tot = (int64_t)K.nB * K.nB;
        for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
            const int k = (int)(t % K.nB), l = (int)(t / K.nB);
            int pk = map[K.map + k], pl = map[K.map + l];
            pk = pk < F.nI ? pk : nIp + (pk - F.nI);
            pl = pl < F.nI ? pl : nIp + (pl - F.nI);
            Fp[pk + (int64_t)pl * np] += U[k + (int64_t)l * npc];
        }
    }
}

// copy the pivot block F_II (ld n_pad) into Finv (ld nIp)
__global__ void k_nd_copy_pivots(const double *Fp, int np, int nIp, double *Fi) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nIp * nIp; t += (int64_t)gridDim.x * blockDim.x)
        Fi[t] = Fp[(t % nIp) + (t / nIp) * (int64_t)np];
}

__global__ void k_nd_transpose(const NdFrontDev *fr, const int64_t *pre, int nf, const double *W, double *Wt) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pre[nf]; t += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nf - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const NdFrontDev F = fr[lo];
        const int64_t e = t - pre[lo];
        const int i = (int)(e % F.nI), b = (int)(e / F.nI);
        Wt[F.wt + e] = W[F.w + b + (int64_t)i * F.ldW];
    }
}


// solve layouts (NdFrontDev fs / wts / ws) from the factorisation's Finv (ld ldFi) and column-major W
// (ld ldW); kind 0: Finv rows, 1: W rows, 2: W columns; padding entries 0
__global__ void k_nd_relayout(const NdFrontDev *fr, const int64_t *pre, int nf, int kind, const double *Finv,
                              const double *W, double *out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pre[nf]; t += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = nf - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const NdFrontDev F = fr[lo];
        const int64_t e = t - pre[lo];
        double v = 0.0;
        if (kind == 0) {            // row i, column j of Finv
            const int i = (int)(e / F.ldFs), j = (int)(e % F.ldFs);
            if (j < F.nI) v = Finv[F.finv + (int64_t)i * F.ldFi + j];
        } else if (kind == 1) {     // row b of W (over pivots i)
            const int b = (int)(e / F.ldWts), i = (int)(e % F.ldWts);
            if (i < F.nI) v = W[F.w + b + (int64_t)i * F.ldW];
        } else {                    // column i of W (over B rows b)
            const int i = (int)(e / F.ldWs), b = (int)(e % F.ldWs);
            if (b < F.nB) v = W[F.w + b + (int64_t)i * F.ldW];
        }
        out[t] = v;
    }
}

// software grid barrier (all CTAs of the launch are co-resident: grid <= one wave).  Polls with
// gpu-scope acquire loads (a volatile load is a system-scope strong load: far slower).
__device__ __forceinline__ unsigned nd_ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void nd_grid_barrier(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = nd_ld_acquire(bar + 1);
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (nd_ld_acquire(bar + 1) == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// lane's share of sum_i a[i] x[i] (i = lane, lane + 32, ...): 4 independent loads in flight
__device__ __forceinline__ double nd_dot_lane(const double *__restrict__ a, const double *x, int n, int lane) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lane;
    for (; i + 96 < n; i += 128) {
        s0 = fma(a[i], __ldcg(x + i), s0);
        s1 = fma(a[i + 32], __ldcg(x + i + 32), s1);
        s2 = fma(a[i + 64], __ldcg(x + i + 64), s2);
        s3 = fma(a[i + 96], __ldcg(x + i + 96), s3);
    }
    for (; i < n; i += 32) s0 = fma(a[i], __ldcg(x + i), s0);
    return (s0 + s1) + (s2 + s3);
}
// 16-byte variant (a and x 16-byte aligned, n even): 8 doubles of a in flight per lane
__device__ __forceinline__ double nd_dot_lane2(const double *__restrict__ a, const double *x, int n, int lane) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a), *x2 = reinterpret_cast<const double2 *>(x);
    const int n2 = n >> 1;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lane;
    for (; i + 96 < n2; i += 128) {
        const double2 a0 = a2[i], a1 = a2[i + 32], a2v = a2[i + 64], a3 = a2[i + 96];
        const double2 b0 = __ldcg(x2 + i), b1 = __ldcg(x2 + i + 32), b2 = __ldcg(x2 + i + 64), b3 = __ldcg(x2 + i + 96);
        s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
        s1 = fma(a1.x, b1.x, fma(a1.y, b1.y, s1));
        s2 = fma(a2v.x, b2.x, fma(a2v.y, b2.y, s2));
        s3 = fma(a3.x, b3.x, fma(a3.y, b3.y, s3));
    }
    for (; i < n2; i += 32) {
        const double2 a0 = a2[i], b0 = __ldcg(x2 + i);
        s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
    }
    return (s0 + s1) + (s2 + s3);
}
__device__ __forceinline__ double nd_dot(const double *__restrict__ a, const double *x, int n, int lane) {
    const bool al = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(x)) & 15) == 0 && (n & 1) == 0;
    return al ? nd_dot_lane2(a, x, n, lane) : nd_dot_lane(a, x, n, lane);
}

// the same with x gathered: sum_i a[i] x[idx[i]]
__device__ __forceinline__ double nd_dot_lane_g(const double *__restrict__ a, const double *x, const int32_t *idx, int n,
                                                int lane) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lane;
    for (; i + 96 < n; i += 128) {
        const int j0 = idx[i], j1 = idx[i + 32], j2 = idx[i + 64], j3 = idx[i + 96];
        s0 = fma(a[i], __ldcg(x + j0), s0);
        s1 = fma(a[i + 32], __ldcg(x + j1), s1);
        s2 = fma(a[i + 64], __ldcg(x + j2), s2);
        s3 = fma(a[i + 96], __ldcg(x + j3), s3);
    }
    for (; i < n; i += 32) s0 = fma(a[i], __ldcg(x + idx[i]), s0);
    return (s0 + s1) + (s2 + s3);
}

// 16-byte variant of nd_dot_lane_g (a 16-byte aligned; n may be odd: the tail element by lane 0)
__device__ __forceinline__ double nd_dot_lane2_g(const double *__restrict__ a, const double *x, const int32_t *idx, int n,
                                                 int lane) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a);
    const int n2 = n >> 1;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = lane;
    for (; i + 32 < n2; i += 64) {
        const double2 a0 = a2[i], a1 = a2[i + 32];
        const int j0 = idx[2 * i], j1 = idx[2 * i + 1], j2 = idx[2 * i + 64], j3 = idx[2 * i + 65];
        s0 = fma(a0.x, __ldcg(x + j0), s0);
        s1 = fma(a0.y, __ldcg(x + j1), s1);
        s2 = fma(a1.x, __ldcg(x + j2), s2);
        s3 = fma(a1.y, __ldcg(x + j3), s3);
    }
    for (; i < n2; i += 32) {
        const double2 a0 = a2[i];
        s0 = fma(a0.x, __ldcg(x + idx[2 * i]), s0);
        s1 = fma(a0.y, __ldcg(x + idx[2 * i + 1]), s1);
    }
    if ((n & 1) && lane == 0) s2 = fma(a[n - 1], __ldcg(x + idx[n - 1]), s2);
    return (s0 + s1) + (s2 + s3);
}

constexpr int kNdMaxLev = 48;
struct NdSched {
    int nlev;
    int aoff[kNdMaxLev + 1];   // forward level L (depth maxd - L): local rhs assembly entries
    int boff[kNdMaxLev + 1];   //                                   B rows
    int coff[kNdMaxLev + 1];   // backward depth L: I rows
    int8_t gb[kNdMaxLev];      // lanes per B row of forward level L (8, 16 or 32)
    int goff[kNdMaxLev + 1];   // backward depth L: y_B gather entries
};

// lanes [sub] of a G-lane group: their share of sum_i a[i] x[i] (16-byte aligned, n even), then the
// group's sum in every lane of the group (fixed shuffle tree)
template <int G>
__device__ __forceinline__ double nd_dot_group2(const double *__restrict__ a, const double *x, int n, int sub) {
    const double2 *a2 = reinterpret_cast<const double2 *>(a), *x2 = reinterpret_cast<const double2 *>(x);
    const int n2 = n >> 1;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = sub;
    for (; i + 3 * G < n2; i += 4 * G) {
        const double2 a0 = a2[i], a1 = a2[i + G], a2v = a2[i + 2 * G], a3 = a2[i + 3 * G];
        const double2 b0 = __ldcg(x2 + i), b1 = __ldcg(x2 + i + G), b2 = __ldcg(x2 + i + 2 * G), b3 = __ldcg(x2 + i + 3 * G);
        s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
        s1 = fma(a1.x, b1.x, fma(a1.y, b1.y, s1));
        s2 = fma(a2v.x, b2.x, fma(a2v.y, b2.y, s2));
        s3 = fma(a3.x, b3.x, fma(a3.y, b3.y, s3));
    }
    for (; i < n2; i += G) {
        const double2 a0 = a2[i], b0 = __ldcg(x2 + i);
        s0 = fma(a0.x, b0.x, fma(a0.y, b0.y, s0));
    }
    return (s0 + s1) + (s2 + s3);
}

// forward phase B of one level with G lanes per B row (32 / G rows per warp in flight: the deep
// levels' rows are short, nI = 72 .. 243)
template <int G, class View>
__device__ __forceinline__ void nd_phase_b(const View &V, int64_t k0, int64_t k1, int64_t gw, int64_t nw, int lane) {
    constexpr int R = 32 / G;
    const int sub = lane % G, grp = lane / G;
    for (int64_t kb = k0 + gw * R; kb < k1; kb += nw * R) {
        const int64_t k = kb + grp;
        double a = 0.0;
        int2 e = make_int2(0, 0);
        const bool ok = k < k1;
        if (ok) {
            e = V.lbr[k];
            const NdFrontDev &F = V.fr[e.x];
            a = nd_dot_group2<G>(V.wt + F.wts + (int64_t)e.y * F.ldWts, V.bi + F.bi, F.ldWts, sub);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (ok && sub == 0) {
            const NdFrontDev &F = V.fr[e.x];
            V.u[F.u + e.y] = __ldcg(V.lb + F.lb + e.y) - a;
        }
    }
}

struct NdSolveView {
    const NdFrontDev *fr;
    const int64_t *invp;
    const int32_t *invl;
    const int32_t *uidx;
    const double *finv, *w, *wt;
    double *bi, *lb, *u;
    const int2 *la, *lbr, *lc;
    double *yb;
    const int2 *lg;
};

// The whole solve E y = c in one persistent launch.  Per forward level: (A) every local
// unknown of the level's fronts: b = c (pivots) + child 0's u + child 1's u (fixed order);
// (B) a warp per B row: u = b_B - W b_I.  Per backward level: (C) a warp per pivot row:
// y_I = Finv b_I - W^t y_B.  Levels and phases are separated by grid barriers; data written
// by other CTAs is read through L2 (__ldcg).  Then q = c^t y.
__global__ void __launch_bounds__(256) k_nd_solve(NdSolveView V, NdSched S, const double *c, double *y, unsigned *bar,
                                                  int64_t nE, double *qout, double *partials, unsigned *ticket) {
    const int lane = threadIdx.x & 31;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    const int64_t gw = gt >> 5, nw = gs >> 5;
    for (int L = 0; L < S.nlev; ++L) {
        for (int64_t k = S.aoff[L] + gt; k < S.aoff[L + 1]; k += gs) {
            const int2 e = V.la[k];
            const NdFrontDev F = V.fr[e.x];
            double v = e.y < F.nI ? c[V.uidx[F.uoff + e.y]] : 0.0;
            for (int64_t q = V.invp[F.inv + e.y]; q < V.invp[F.inv + e.y + 1]; ++q) v += __ldcg(V.u + V.invl[q]);
            if (e.y < F.nI) V.bi[F.bi + e.y] = v;
            else V.lb[F.lb + e.y - F.nI] = v;
        }
        nd_grid_barrier(bar);
        if (S.boff[L + 1] > S.boff[L]) {
            if (S.gb[L] == 8) nd_phase_b<8>(V, S.boff[L], S.boff[L + 1], gw, nw, lane);
            else if (S.gb[L] == 16) nd_phase_b<16>(V, S.boff[L], S.boff[L + 1], gw, nw, lane);
            else nd_phase_b<32>(V, S.boff[L], S.boff[L + 1], gw, nw, lane);
            nd_grid_barrier(bar);
        }
    }
    for (int L = 0; L < S.nlev; ++L) {
        // (G) the level's y_B gathered once into a contiguous, zero-padded copy per front, so the
        // pivot rows below stream it instead of an index -> y gather per element of W
        if (S.goff[L + 1] > S.goff[L]) {
            for (int64_t k = S.goff[L] + gt; k < S.goff[L + 1]; k += gs) {
                const int2 e = V.lg[k];
                const NdFrontDev &F = V.fr[e.x];
                V.yb[F.yb + e.y] = e.y < F.nB ? __ldcg(y + V.uidx[F.uoff + F.nI + e.y]) : 0.0;
            }
            nd_grid_barrier(bar);
        }
        for (int64_t k = S.coff[L] + gw; k < S.coff[L + 1]; k += nw) {
            const int2 e = V.lc[k];
            const NdFrontDev F = V.fr[e.x];
            const double pa = nd_dot_lane2(V.finv + F.fs + (int64_t)e.y * F.ldFs, V.bi + F.bi, F.ldFs, lane);
            const double pb = nd_dot_lane2(V.w + F.ws + (int64_t)e.y * F.ldWs, V.yb + F.yb, F.ldWs, lane);
            const double a = warp_sum(pa - pb);
            if (lane == 0) y[V.uidx[F.uoff + e.y]] = a;
        }
        nd_grid_barrier(bar);
    }
    double acc[1] = {0.0};
    for (int64_t i = gt; i < nE; i += gs) acc[0] = fma(c[i], __ldcg(y + i), acc[0]);
    reduce_and_finish<1>(acc, partials, ticket, [&](double *t) { *qout = t[0]; });
}

// One phase of one level as its own launch (shallow trees: the flat plan has 2 levels, so 5 short
// launches replace the persistent kernel and its spin barriers).  kind 0: A, 1: B, 2: C.
__global__ void __launch_bounds__(256) k_nd_phase(NdSolveView V, int kind, int64_t k0, int64_t k1, const double *c,
                                                  double *y) {
    const int lane = threadIdx.x & 31;
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    if (kind == 0) {
        for (int64_t k = k0 + gt; k < k1; k += gs) {
            const int2 e = V.la[k];
            const NdFrontDev F = V.fr[e.x];
            double v = e.y < F.nI ? c[V.uidx[F.uoff + e.y]] : 0.0;
            for (int64_t q = V.invp[F.inv + e.y]; q < V.invp[F.inv + e.y + 1]; ++q) v += V.u[V.invl[q]];
            if (e.y < F.nI) V.bi[F.bi + e.y] = v;
            else V.lb[F.lb + e.y - F.nI] = v;
        }
        return;
    }
    for (int64_t k = k0 + (gt >> 5); k < k1; k += gs >> 5) {
        if (kind == 1) {
            const int2 e = V.lbr[k];
            const NdFrontDev F = V.fr[e.x];
            const double a = warp_sum(nd_dot_lane2(V.wt + F.wts + (int64_t)e.y * F.ldWts, V.bi + F.bi, F.ldWts, lane));
            if (lane == 0) V.u[F.u + e.y] = V.lb[F.lb + e.y] - a;
        } else {
            const int2 e = V.lc[k];
            const NdFrontDev F = V.fr[e.x];
            const double pa = nd_dot_lane2(V.finv + F.fs + (int64_t)e.y * F.ldFs, V.bi + F.bi, F.ldFs, lane);
            const double pb = nd_dot_lane2_g(V.w + F.ws + (int64_t)e.y * F.ldWs, y, V.uidx + F.uoff + F.nI, F.nB, lane);
            const double a = warp_sum(pa - pb);
            if (lane == 0) y[V.uidx[F.uoff + e.y]] = a;
        }
    }
}

__global__ void __launch_bounds__(256) k_nd_cdot(int64_t n, const double *c, const double *y, double *qout,
                                                 double *partials, unsigned *ticket) {
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc[0] = fma(c[i], y[i], acc[0]);
    reduce_and_finish<1>(acc, partials, ticket, [&](double *t) { *qout = t[0]; });
}

static void gj_invert(double *A, int64_t n, cudaStream_t s);   // below (blocked Gauss-Jordan, SPD)
static void spd_invert(double *A, int64_t n, cudaStream_t s, int *info_d = nullptr);   // below (cuSOLVER Cholesky)

struct BlasBatched {
    int (*TrsmB)(void *, int, int, int, int, int, int, const double *, const double *const[], int, double *const[], int,
                 int) = nullptr;
    int (*GetrfB)(void *, int, double *const[], int, int *, int *, int) = nullptr;
    int (*GetriB)(void *, int, const double *const[], int, const int *, double *const[], int, int *, int) = nullptr;
    int (*GemmB)(void *, int, int, int, int, int, const double *, const double *const[], int, const double *const[], int,
                 const double *, double *const[], int, int) = nullptr;
};
static BlasBatched &blas_batched() {
    static thread_local BlasBatched b = [] {
        BlasBatched x;
        Blas &bl = blas();
        if (!bl.h) return x;
        x.GetrfB = (decltype(x.GetrfB))dlsym(bl.h, "cublasDgetrfBatched");
        x.TrsmB = (decltype(x.TrsmB))dlsym(bl.h, "cublasDtrsmBatched");
        x.GetriB = (decltype(x.GetriB))dlsym(bl.h, "cublasDgetriBatched");
        x.GemmB = (decltype(x.GemmB))dlsym(bl.h, "cublasDgemmBatched");
        return x;
    }();
    return b;
}

template <class T>
static void upload(DevBuf<T> &d, const std::vector<T> &h, cudaStream_t s) {
    d.alloc(h.size(), s);
    if (!h.empty()) CR_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}

struct Lapack;
static Lapack &lapack();
static bool lapack_potrf_batched(int n, int lda, int nb, double **A, int *info, cudaStream_t s);

__global__ void k_identity_batched(double *const *X, int n, int nb) {
    const int64_t tot = (int64_t)n * n * nb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(t / ((int64_t)n * n));
        const int64_t e = t - (int64_t)b * n * n;
        X[b][e] = (e % n) == (e / n) ? 1.0 : 0.0;
    }
}

// Finv = A^{-1} for a batch of SPD pivot blocks (in place factor of A, ld lda; Finv ld n):
// Cholesky (cusolverDnDpotrfBatched), X = I, L X = I, L^t X' = X (two cublasDtrsmBatched).
// Returns false when a routine is unavailable (the caller then uses batched LU + inverse).
static bool nd_batched_cholesky_inverse(int n, int lda, int nb, double **dA, double **dX, const std::vector<double *> &,
                                        int *info, cudaStream_t s) {
    BlasBatched &bb = blas_batched();
    Blas &bl = blas();
    if (!bb.TrsmB || !bl.handle) return false;
    if (!lapack_potrf_batched(n, lda, nb, dA, info, s)) return false;
    k_identity_batched<<<grid_for((int64_t)n * n * nb, 256, 16), 256, 0, s>>>(dX, n, nb);
    CR_CHECK_LAUNCH();
    bl.SetStream(bl.handle, s);
    const double one = 1.0;
    // column-major: side left (0), lower (0), no-trans (0) / trans (1), non-unit diagonal (0)
    CR_REQUIRE(bb.TrsmB(bl.handle, 0, 0, 0, 0, n, n, &one, dA, lda, dX, n, nb) == 0, CR_ERR_CUDA, "cublasDtrsmBatched failed");
    CR_REQUIRE(bb.TrsmB(bl.handle, 0, 0, 1, 0, n, n, &one, dA, lda, dX, n, nb) == 0, CR_ERR_CUDA, "cublasDtrsmBatched failed");
    return true;
}

// host-side plan of nd_setup (depends only on H, D and the plan variant)
struct NdHost {
    std::vector<HostFront> F;
    int nf = 0, maxd = 0;
    std::vector<std::vector<int>> lev;
    std::vector<int> parent, slot, nIp, nBp;
    std::vector<char> batched;
    std::vector<NdFrontDev> fr;
    std::vector<int32_t> nodes, map, uidx, kidl;
    std::vector<int64_t> fbase, invp;
    std::vector<int32_t> invl;
    int64_t ofi = 0, ow = 0, owt = 0, obi = 0, ou = 0, olb = 0, oinv = 0, fpool = 0, maxn = 0, bytes = 0;
};

template <int D>
static void nd_setup(CoarseOp &C, const double *Es, int H, cudaStream_t s) {
    constexpr int M = D * D;
    CoarseNd &N = C.nd;
    Trace tr(s);
    // the host-side plan and index maps depend only on (H, D, box): built once per process and reused
    // (the 3D bisection plan with its B sets and CSR maps took ~21 ms per solve)
    const char *eb = std::getenv("CR_ND_BOX");
    const int box = eb ? std::max(0, atoi(eb)) : (D == 2 ? 12 : 0);
    static std::mutex plan_mu;
    static std::map<std::tuple<int, int, int>, std::shared_ptr<NdHost>> plan_cache;
    std::shared_ptr<NdHost> PH;
    {
        std::lock_guard<std::mutex> lk(plan_mu);
        auto it = plan_cache.find(std::make_tuple(H, D, box));
        if (it != plan_cache.end()) PH = it->second;
    }
    if (!PH) {
        PH = std::make_shared<NdHost>();
        NdHost &Q = *PH;
        auto &F = Q.F;
        nd_plan(H, D, F, box);
        const int nf = (int)F.size();
        int maxd = 0;
        for (auto &f : F) maxd = std::max(maxd, f.depth);
        Q.nf = nf;
        Q.maxd = maxd;
        auto &lev = Q.lev;
        lev.assign(maxd + 1, {});
        for (int f = 0; f < nf; ++f) lev[F[f].depth].push_back(f);
        auto &parent = Q.parent;
        auto &slot = Q.slot;
        parent.assign(nf, -1);
        slot.assign(nf, 0);
        for (int f = 0; f < nf; ++f)
            for (int k : F[f].kids) parent[k] = f;
        // padded sizes: levels with many small fronts are factorised by batched cuBLAS calls
        auto &nIp = Q.nIp;
        auto &nBp = Q.nBp;
        auto &batched = Q.batched;
        nIp.assign(nf, 0);
        nBp.assign(nf, 0);
        batched.assign(maxd + 1, 0);
        for (int d = 0; d <= maxd; ++d) {
            int mi = 0, mb = 0;
            for (int f : lev[d]) { mi = std::max(mi, (int)F[f].I.size() * M); mb = std::max(mb, (int)F[f].B.size() * M); }
            batched[d] = lev[d].size() >= 4 && mi <= 640;
            for (size_t k = 0; k < lev[d].size(); ++k) {
                const int f = lev[d][k];
                slot[f] = (int)k;
                nIp[f] = batched[d] ? mi : (int)F[f].I.size() * M;
                nBp[f] = batched[d] ? mb : (int)F[f].B.size() * M;
            }
        }
        auto &fr = Q.fr;
        fr.assign(nf, NdFrontDev{});
        auto &nodes = Q.nodes;
        auto &map = Q.map;
        int64_t ofi = 0, ow = 0, owt = 0, obi = 0, ou = 0, olb = 0, oinv = 0, fpool = 0, maxn = 0, bytes = 0;
        auto &uidx = Q.uidx;
        auto &kidl = Q.kidl;
        auto &fbase = Q.fbase;
        fbase.assign(nf, 0);
        for (int f = 0; f < nf; ++f) {
            NdFrontDev &x = fr[f];
            x.ioff = (int64_t)nodes.size();
            nodes.insert(nodes.end(), F[f].I.begin(), F[f].I.end());
            x.boff = (int64_t)nodes.size();
            nodes.insert(nodes.end(), F[f].B.begin(), F[f].B.end());
            x.nI = (int32_t)F[f].I.size() * M;
            x.nB = (int32_t)F[f].B.size() * M;
            x.kid_off = (int32_t)kidl.size();
            x.kid_cnt = (int32_t)F[f].kids.size();
            kidl.insert(kidl.end(), F[f].kids.begin(), F[f].kids.end());
            x.ldFi = nIp[f];
            x.ldW = std::max(nBp[f], 1);
            x.finv = ofi; ofi += (int64_t)nIp[f] * nIp[f];
            x.w = ow; ow += (int64_t)nBp[f] * nIp[f];
            x.wt = owt; owt += (int64_t)x.nB * x.nI;
            x.bi = obi; obi += (x.nI + 1) & ~1;   // even: 16-byte aligned, zero pad entry
            x.u = ou; ou += x.nB;
            x.lb = olb; olb += x.nB;
            x.inv = oinv; oinv += x.nI + x.nB;
            x.uoff = (int64_t)uidx.size();
            for (int32_t v : F[f].I)
                for (int cc = 0; cc < M; ++cc) uidx.push_back(v * M + cc);
            for (int32_t v : F[f].B)
                for (int cc = 0; cc < M; ++cc) uidx.push_back(v * M + cc);
            fbase[f] = fpool;
            fpool += (int64_t)(nIp[f] + nBp[f]) * (nIp[f] + nBp[f]);
            maxn = std::max<int64_t>(maxn, x.nI + x.nB);
            bytes += 8 * ((int64_t)x.nI * x.nI + 2 * (int64_t)x.nB * x.nI);
            // this front's B unknowns -> local unknowns of the parent
            x.map = (int64_t)map.size();
            if (parent[f] >= 0) {
                const HostFront &P = F[parent[f]];
                for (int32_t v : F[f].B) {
                    int pos;
                    auto it = std::lower_bound(P.I.begin(), P.I.end(), v);
                    if (it != P.I.end() && *it == v) {
                        pos = (int)(it - P.I.begin());
                    } else {
                        auto jt = std::find(P.B.begin(), P.B.end(), v);
                        CR_REQUIRE(jt != P.B.end(), CR_ERR_INVALID_ARG, "coarse ND plan: child boundary node missing in parent");
                        pos = (int)P.I.size() + (int)(jt - P.B.begin());
                    }
                    for (int c = 0; c < M; ++c) map.push_back(pos * M + c);
                }
            }
        }
        // children's u entries landing on each local unknown of their parent (absolute u indices, in
        // child order: a fixed summation order), as CSR rows
        std::vector<std::vector<int32_t>> invr(oinv);
        for (int f = 0; f < nf; ++f)
            for (int kid : F[f].kids)
                for (int q = 0; q < fr[kid].nB; ++q) invr[fr[f].inv + map[fr[kid].map + q]].push_back((int32_t)(fr[kid].u + q));
        std::vector<int64_t> invp(oinv + 1, 0);
        std::vector<int32_t> invl;
        for (int64_t g = 0; g < oinv; ++g) {
            invl.insert(invl.end(), invr[g].begin(), invr[g].end());
            invp[g + 1] = (int64_t)invl.size();
        }
        Q.ofi = ofi; Q.ow = ow; Q.owt = owt; Q.obi = obi; Q.ou = ou; Q.olb = olb; Q.oinv = oinv;
        Q.fpool = fpool; Q.maxn = maxn; Q.bytes = bytes;
        Q.invp = std::move(invp);
        Q.invl = std::move(invl);
        std::lock_guard<std::mutex> lk(plan_mu);
        plan_cache[std::make_tuple(H, D, box)] = PH;
    }
    const NdHost &Q = *PH;
    const auto &F = Q.F;
    const int nf = Q.nf, maxd = Q.maxd;
    const auto &lev = Q.lev;
    const auto &slot = Q.slot;
    const auto &nIp = Q.nIp;
    const auto &nBp = Q.nBp;
    const auto &batched = Q.batched;
    std::vector<NdFrontDev> fr = Q.fr;   // copied: the solve layouts are filled in below
    const auto &nodes = Q.nodes;
    const auto &map = Q.map;
    const auto &uidx = Q.uidx;
    std::vector<int32_t> kidl = Q.kidl;
    const auto &fbase = Q.fbase;
    const int64_t ofi = Q.ofi, ow = Q.ow, obi = Q.obi, ou = Q.ou, olb = Q.olb, fpool = Q.fpool, bytes = Q.bytes;
    std::vector<int64_t> invp = Q.invp;
    std::vector<int32_t> invl = Q.invl;
    tr.mark("  nd: plan + maps (host)");
    upload(N.fr, fr, s);
    upload(N.nodes, nodes, s);
    upload(N.map, map, s);
    upload(N.invp, invp, s);
    if (invl.empty()) invl.push_back(0);
    upload(N.invl, invl, s);
    if (kidl.empty()) kidl.push_back(0);
    upload(N.kids, kidl, s);
    upload(N.uidx, uidx, s);
    N.lb.alloc(std::max<int64_t>(olb, 1), s);
    N.finv.alloc(std::max<int64_t>(ofi, 1), s);
    N.w.alloc(std::max<int64_t>(ow, 1), s);
    N.w.zero(s);
    N.bi.alloc(std::max<int64_t>(obi, 2), s);
    N.bi.zero(s);   // pad entries stay 0 (the 16-byte dot products read them)
    N.u.alloc(std::max<int64_t>(ou, 1), s);
    N.m = M;
    N.maxdepth = maxd;
    N.nfront = nf;
    N.bytes = bytes;
    // work lists: forward by level deepest first (A: local unknowns, B: B rows), backward root
    // first (C: pivot rows)
    CR_REQUIRE(maxd + 1 <= kNdMaxLev, CR_ERR_INVALID_ARG, "coarse ND tree too deep");
    {
        std::vector<int2> la, lbr, lc;
        N.aoff.assign(maxd + 2, 0);
        N.boff.assign(maxd + 2, 0);
        N.coff.assign(maxd + 2, 0);
        N.gb.assign(maxd + 1, 32);
        for (int L = 0; L <= maxd; ++L) {
            double rows = 0.0, len = 0.0;
            for (int f : lev[maxd - L]) {
                for (int p = 0; p < fr[f].nI + fr[f].nB; ++p) la.push_back(make_int2(f, p));
                for (int b = 0; b < fr[f].nB; ++b) lbr.push_back(make_int2(f, b));
                rows += fr[f].nB;
                len += (double)fr[f].nB * fr[f].nI;
            }
            // lanes per B row: the level's mean row length in 16-byte units, >= 4 per lane
            const double n2 = rows > 0 ? 0.5 * len / rows : 0.0;
            static const char *eg = std::getenv("CR_ND_GROUPS");   // 0: a warp per B row everywhere
            N.gb[L] = (eg && atoi(eg) == 0) ? 32 : (n2 < 64 ? 8 : (n2 < 128 ? 16 : 32));
            for (int f : lev[L])
                for (int i = 0; i < fr[f].nI; ++i) lc.push_back(make_int2(f, i));
            N.aoff[L + 1] = (int)la.size();
            N.boff[L + 1] = (int)lbr.size();
            N.coff[L + 1] = (int)lc.size();
        }
        upload(N.la, la, s);
        upload(N.lbr, lbr, s);
        upload(N.lc, lc, s);
        N.bar.alloc(2, s);
        N.bar.zero(s);
        int occ = 0, dev = 0, coop = 0;
        CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_nd_solve, 256, 0));
        CR_CUDA(cudaGetDevice(&dev));
        CR_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        // one co-resident wave (more resident warps: the phases are latency-bound); 0 = no
        // persistent kernel (per-phase launches)
        // CR_ND_GRID = CTAs per SM (tuning: a small grid can run beside the patch solves when they
        // leave block slots free, CR_AFW_RSV)
        static const char *eg = std::getenv("CR_ND_GRID");
        const int per_sm = eg ? std::max(1, std::min(atoi(eg), occ)) : std::min(occ, 8);
        N.grid = (coop && occ >= 1) ? num_sms() * per_sm : 0;
    }
    tr.mark("  nd: uploads + work lists");
    // numeric factorisation, deepest level first
    DevBuf<double> Fp;
    Fp.alloc(std::max<int64_t>(fpool, 1), s);
    tr.mark("  nd: F pool alloc");
    std::vector<DevBuf<int32_t>> lfronts(maxd + 2), lnIp(maxd + 2), lnBp(maxd + 2);
    std::vector<DevBuf<int64_t>> lfoff(maxd + 2), lfbase(maxd + 2);
    std::vector<NdLevelDev> LV(maxd + 2);
    std::vector<int32_t> hslot(slot.begin(), slot.end());
    DevBuf<int32_t> dslot;
    upload(dslot, hslot, s);
    DevBuf<int> finfo;   // cuSOLVER infos of the fronts inverted one by one, checked once at the end
    finfo.alloc(2 * (size_t)nf, s);
    finfo.zero(s);
    BlasBatched &bb = blas_batched();
    Blas &bl = blas();
    CR_REQUIRE(bl.handle && bb.GemmB && bb.GetrfB && bb.GetriB, CR_ERR_CUDA, "cuBLAS batched routines unavailable");
    const int T = 256;
    for (int d = maxd; d >= 0; --d) {
        const auto &L = lev[d];
        std::vector<int32_t> hf(L.begin(), L.end()), hi(L.size()), hb(L.size());
        std::vector<int64_t> hoff(L.size() + 1, 0), hbase(L.size());
        for (size_t k = 0; k < L.size(); ++k) {
            const int f = L[k];
            hi[k] = nIp[f];
            hb[k] = nBp[f];
            const int64_t np = nIp[f] + nBp[f];
            hoff[k + 1] = hoff[k] + np * np;
            hbase[k] = fbase[f];
        }
        upload(lfronts[d], hf, s); upload(lnIp[d], hi, s); upload(lnBp[d], hb, s);
        upload(lfoff[d], hoff, s); upload(lfbase[d], hbase, s);
        LV[d] = NdLevelDev{lfronts[d].get(), lfoff[d].get(), lfbase[d].get(), lnIp[d].get(), lnBp[d].get(), (int)L.size()};
        k_nd_assemble<D><<<grid_for(hoff.back(), T, 16), T, 0, s>>>(LV[d], N.fr.get(), N.nodes.get(), Es, H, Fp.get());
        CR_CHECK_LAUNCH();
        tr.mark("  nd: level assemble");
        if (d < maxd) {
            int64_t mxb = 1;
            int maxk = 0;
            for (int f : L) {
                maxk = std::max(maxk, (int)F[f].kids.size());
                for (int k : F[f].kids) mxb = std::max<int64_t>(mxb, (int64_t)fr[k].nB * fr[k].nB);
            }
            dim3 g((unsigned)std::min<int64_t>((mxb + T - 1) / T, 4096), (unsigned)std::min<size_t>(L.size(), 65535));
            for (int which = 0; which < maxk; ++which) {   // one child at a time: fixed summation order
                k_nd_extend<<<g, T, 0, s>>>(LV[d], LV[d + 1], N.fr.get(), N.map.get(), N.kids.get(), dslot.get(), which,
                                           Fp.get());
                CR_CHECK_LAUNCH();
            }
        }
        const double one = 1.0, zero = 0.0, mone = -1.0;
        bl.SetStream(bl.handle, s);
        if (batched[d]) {
            const int nb = (int)L.size(), ni = nIp[L[0]], nbp = nBp[L[0]], np = ni + nbp;
            std::vector<double *> pA(nb), pFi(nb), pFB(nb), pW(nb), pFIB(nb), pFBB(nb);
            for (int k = 0; k < nb; ++k) {
                const int f = L[k];
                double *base = Fp.get() + fbase[f];
                pA[k] = base;
                pFi[k] = N.finv.get() + fr[f].finv;
                pFB[k] = base + ni;
                pW[k] = N.w.get() + fr[f].w;
                pFIB[k] = base + (int64_t)ni * np;
                pFBB[k] = base + ni + (int64_t)ni * np;
            }
            DevBuf<double *> dA, dFi, dFB, dW, dFIB, dFBB;
            upload(dA, pA, s); upload(dFi, pFi, s); upload(dFB, pFB, s);
            upload(dW, pW, s); upload(dFIB, pFIB, s); upload(dFBB, pFBB, s);
            DevBuf<int> piv, info;
            piv.alloc((size_t)ni * nb, s);
            info.alloc(nb, s);
            info.zero(s);
            if (!nd_batched_cholesky_inverse(ni, np, nb, dA.get(), dFi.get(), pFi, info.get(), s)) {
                CR_REQUIRE(bb.GetrfB(bl.handle, ni, dA.get(), np, piv.get(), info.get(), nb) == 0, CR_ERR_CUDA,
                           "cublasDgetrfBatched failed");
                CR_REQUIRE(bb.GetriB(bl.handle, ni, dA.get(), np, piv.get(), dFi.get(), ni, info.get(), nb) == 0, CR_ERR_CUDA,
                           "cublasDgetriBatched failed");
            }
            std::vector<int> hinfo(nb);
            CR_CUDA(cudaMemcpyAsync(hinfo.data(), info.get(), nb * sizeof(int), cudaMemcpyDeviceToHost, s));
            CR_CUDA(cudaStreamSynchronize(s));
            for (int v : hinfo) CR_REQUIRE(v == 0, CR_ERR_SINGULAR_LOCAL, "coarse ND front is singular");
            if (nbp > 0) {
                CR_REQUIRE(bb.GemmB(bl.handle, 0, 0, nbp, ni, ni, &one, dFB.get(), np, dFi.get(), ni, &zero, dW.get(), nbp, nb) == 0,
                           CR_ERR_CUDA, "cublasDgemmBatched failed");
                CR_REQUIRE(bb.GemmB(bl.handle, 0, 0, nbp, nbp, ni, &mone, dW.get(), nbp, dFIB.get(), np, &one, dFBB.get(), np, nb) == 0,
                           CR_ERR_CUDA, "cublasDgemmBatched failed");
            }
            CR_CUDA(cudaStreamSynchronize(s));   // the pointer arrays are freed at scope exit
        } else {
            for (int f : L) {
                const int ni = nIp[f], nbp = nBp[f], np = ni + nbp;
                double *base = Fp.get() + fbase[f];
                double *Fi = N.finv.get() + fr[f].finv;
                k_nd_copy_pivots<<<grid_for((int64_t)ni * ni, T, 16), T, 0, s>>>(base, np, ni, Fi);
                CR_CHECK_LAUNCH();
                spd_invert(Fi, ni, s, finfo.get() + 2 * f);
                if (nbp > 0) {
                    dgemm(s, nbp, ni, ni, 1.0, base + ni, np, Fi, ni, 0.0, N.w.get() + fr[f].w, nbp);
                    dgemm(s, nbp, nbp, ni, -1.0, N.w.get() + fr[f].w, nbp, base + (int64_t)ni * np, np, 1.0,
                          base + ni + (int64_t)ni * np, np);
                }
            }
        }
    }
    tr.mark("  nd: level factorisations");
    {
        std::vector<int> hinfo(2 * (size_t)nf);
        CR_CUDA(cudaMemcpyAsync(hinfo.data(), finfo.get(), hinfo.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        for (int v : hinfo) CR_REQUIRE(v == 0, CR_ERR_SINGULAR_LOCAL, "coarse ND front is not positive definite");
    }
    // solve layouts: rows 16-byte aligned with even leading dimensions and zero padding, so every
    // dot product of the solve streams double2 (the odd D^2 = 9 unknowns per node made nI, nB odd)
    {
        auto ev = [](int64_t v) { return (v + 1) & ~(int64_t)1; };
        int64_t ofs = 0, owts = 0, ows = 0, oyb = 0;
        std::vector<int64_t> pf(nf + 1, 0), pwt(nf + 1, 0), pw(nf + 1, 0);
        for (int f = 0; f < nf; ++f) {
            NdFrontDev &x = fr[f];
            x.ldFs = (int32_t)ev(x.nI);
            x.ldWts = (int32_t)ev(x.nI);
            x.ldWs = (int32_t)std::max<int64_t>(ev(x.nB), 2);
            x.fs = ofs; ofs += (int64_t)x.nI * x.ldFs;
            x.wts = owts; owts += (int64_t)x.nB * x.ldWts;
            x.ws = ows; ows += (int64_t)x.nI * x.ldWs;
            x.yb = oyb; oyb += x.ldWs;
            pf[f + 1] = ofs; pwt[f + 1] = owts; pw[f + 1] = ows;
        }
        upload(N.fr, fr, s);
        N.yb.alloc(std::max<int64_t>(oyb, 2), s);
        {   // backward y_B gathers by depth (root first, like the pivot rows)
            std::vector<int2> lg;
            N.goff.assign(maxd + 2, 0);
            for (int L = 0; L <= maxd; ++L) {
                for (int f : lev[L])
                    for (int b = 0; b < fr[f].ldWs; ++b) lg.push_back(make_int2(f, b));
                N.goff[L + 1] = (int)lg.size();
            }
            upload(N.lg, lg, s);
        }
        N.fs.alloc(std::max<int64_t>(ofs, 2), s);
        N.wts.alloc(std::max<int64_t>(owts, 2), s);
        N.ws.alloc(std::max<int64_t>(ows, 2), s);
        DevBuf<int64_t> dpf, dpwt, dpw;
        upload(dpf, pf, s);
        upload(dpwt, pwt, s);
        upload(dpw, pw, s);
        if (ofs) k_nd_relayout<<<grid_for(ofs, T, 16), T, 0, s>>>(N.fr.get(), dpf.get(), nf, 0, N.finv.get(), N.w.get(), N.fs.get());
        if (owts) k_nd_relayout<<<grid_for(owts, T, 16), T, 0, s>>>(N.fr.get(), dpwt.get(), nf, 1, N.finv.get(), N.w.get(), N.wts.get());
        if (ows) k_nd_relayout<<<grid_for(ows, T, 16), T, 0, s>>>(N.fr.get(), dpw.get(), nf, 2, N.finv.get(), N.w.get(), N.ws.get());
        CR_CHECK_LAUNCH();
        CR_CUDA(cudaStreamSynchronize(s));
        N.finv.release();
        N.w.release();
        N.wt.release();
    }
    N.on = true;
}

// y = E^{-1} c by the ND fronts, q = c^t y
static void nd_solve(const CoarseOp &C, const double *c, double *y, double *qout, double *partials, unsigned *ticket,
                     cudaStream_t s) {
    const CoarseNd &N = C.nd;
    NdSolveView V{N.fr.get(), N.invp.get(), N.invl.get(), N.uidx.get(), N.fs.get(), N.ws.get(), N.wts.get(),
                  const_cast<double *>(N.bi.get()), const_cast<double *>(N.lb.get()), const_cast<double *>(N.u.get()),
                  N.la.get(), N.lbr.get(), N.lc.get(), const_cast<double *>(N.yb.get()), N.lg.get()};
    NdSched S;
    S.nlev = N.maxdepth + 1;
    for (int L = 0; L <= S.nlev; ++L) {
        S.aoff[L] = N.aoff[L];
        S.boff[L] = N.boff[L];
        S.coff[L] = N.coff[L];
    }
    for (int L = 0; L < S.nlev; ++L) S.gb[L] = (int8_t)N.gb[L];
    for (int L = 0; L <= S.nlev; ++L) S.goff[L] = N.goff[L];
    static const char *ep = std::getenv("CR_ND_PERSIST");
    const bool persistent = (ep ? atoi(ep) != 0 : N.maxdepth > 1) && N.grid > 0;
    if (persistent) {
        // cooperative launch: the runtime guarantees that all N.grid CTAs are co-resident (the
        // software grid barrier needs it), or fails the launch — then the per-phase launches
        // below take over.  N.grid = SMs x occupancy of this device (0 when cooperative launches
        // are unsupported).
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(N.grid);
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CR_CUDA(cudaLaunchKernelEx(&cfg, k_nd_solve, V, S, c, y, const_cast<unsigned *>(N.bar.get()), C.nE, qout,
                                   partials, ticket));
        CR_CHECK_LAUNCH();
        return;
    }
    auto launch = [&](int kind, int64_t k0, int64_t k1) {
        if (k1 <= k0) return;
        const int64_t work = kind == 0 ? (k1 - k0) : (k1 - k0) * 32;
        k_nd_phase<<<grid_for(work, 256, 8), 256, 0, s>>>(V, kind, k0, k1, c, y);
        CR_CHECK_LAUNCH();
    };
    for (int L = 0; L < S.nlev; ++L) {
        launch(0, S.aoff[L], S.aoff[L + 1]);
        launch(1, S.boff[L], S.boff[L + 1]);
    }
    for (int L = 0; L < S.nlev; ++L) launch(2, S.coff[L], S.coff[L + 1]);
    k_nd_cdot<<<occ_grid(k_nd_cdot, 256, C.nE), 256, 0, s>>>(C.nE, c, y, qout, partials, ticket);
    CR_CHECK_LAUNCH();
}


// blocked Gauss-Jordan inversion in place of an SPD n x n matrix (row- or column-major: a
// row-major M is the column-major M^t for cuBLAS):
//   Y = A[K,:];  X = A[:,K] Pk;  A -= X Y;  A[K,:] = Pk Y;  A[:,K] = -X, A[K,K] = Pk
static void gj_invert(double *A, int64_t n64, cudaStream_t s) {
    const int T = 256;
    DevBuf<double> Pk, X, Yb;
    Pk.alloc(kGB * kGB, s);
    X.alloc(n64 * kGB, s);
    Yb.alloc(n64 * kGB, s);
    DevBuf<int> bad;
    bad.alloc(1, s);
    bad.zero(s);
    const int n = (int)n64;
    for (int64_t k0 = 0; k0 < n64; k0 += kGB) {
        const int b = (int)std::min<int64_t>(kGB, n64 - k0);
        k_gj_diag<<<1, 256, 0, s>>>(A, n64, k0, b, Pk.get(), bad.get());
        CR_CUDA(cudaMemcpyAsync(Yb.get(), A + k0 * n64, (size_t)b * n64 * sizeof(double), cudaMemcpyDeviceToDevice, s));
        dgemm(s, b, n, b, 1.0, Pk.get(), b, A + k0, n, 0.0, X.get(), b);            // X^t = Pk^t A[:,K]^t
        dgemm(s, n, n, b, -1.0, Yb.get(), n, X.get(), b, 1.0, A, n);                 // A^t -= Y^t X^t
        dgemm(s, n, b, b, 1.0, Yb.get(), n, Pk.get(), b, 0.0, A + k0 * n64, n);     // A[K,:]^t = Y^t Pk^t
        k_gj_cols<<<grid_for(n64 * b, T), T, 0, s>>>(A, n64, k0, b, Pk.get(), X.get());
    }
    CR_CHECK_LAUNCH();
    int hb = 0;
    CR_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    CR_REQUIRE(hb == 0, CR_ERR_SINGULAR_LOCAL, "coarse matrix Z^t G Z is not positive definite");
}

// Dense SPD inverse by cuSOLVER (dlopen'ed libcusolver.so.11): Cholesky potrf + potri on the lower
// triangle, then the upper triangle mirrored.  ~3x fewer flops than Gauss-Jordan and LAPACK-size
// panels (the coarse setup is part of every solve); Gauss-Jordan is the fallback when the library
// is missing.  A non-positive pivot (info > 0) throws CR_ERR_SINGULAR_LOCAL (build_coarse halves H).
struct Lapack {
    void *h = nullptr, *handle = nullptr;
    int (*Create)(void **) = nullptr;
    int (*SetStream)(void *, cudaStream_t) = nullptr;
    int (*PotrfBS)(void *, int, int, double *, int, int *) = nullptr;
    int (*Potrf)(void *, int, int, double *, int, double *, int, int *) = nullptr;
    int (*PotriBS)(void *, int, int, double *, int, int *) = nullptr;
    int (*Potri)(void *, int, int, double *, int, double *, int, int *) = nullptr;
    int (*SyevdBS)(void *, int, int, int, const double *, int, const double *, int *) = nullptr;
    int (*Syevd)(void *, int, int, int, double *, int, double *, double *, int, int *) = nullptr;
    int (*PotrfB)(void *, int, int, double *[], int, int *, int) = nullptr;
};
static Lapack &lapack() {
    static thread_local Lapack L = [] {
        Lapack x;
        x.h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) return x;
        x.Create = (decltype(x.Create))dlsym(x.h, "cusolverDnCreate");
        x.SetStream = (decltype(x.SetStream))dlsym(x.h, "cusolverDnSetStream");
        x.PotrfBS = (decltype(x.PotrfBS))dlsym(x.h, "cusolverDnDpotrf_bufferSize");
        x.Potrf = (decltype(x.Potrf))dlsym(x.h, "cusolverDnDpotrf");
        x.PotriBS = (decltype(x.PotriBS))dlsym(x.h, "cusolverDnDpotri_bufferSize");
        x.Potri = (decltype(x.Potri))dlsym(x.h, "cusolverDnDpotri");
        x.SyevdBS = (decltype(x.SyevdBS))dlsym(x.h, "cusolverDnDsyevd_bufferSize");
        x.Syevd = (decltype(x.Syevd))dlsym(x.h, "cusolverDnDsyevd");
        x.PotrfB = (decltype(x.PotrfB))dlsym(x.h, "cusolverDnDpotrfBatched");
        if (!(x.Create && x.SetStream && x.PotrfBS && x.Potrf && x.PotriBS && x.Potri) || x.Create(&x.handle) != 0)
            x.handle = nullptr;
        return x;
    }();
    return L;
}

__global__ void k_mirror_lower(double *A, int64_t n) {   // column-major: A(j, i) = A(i, j), i > j
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / n, i = t - j * n;
        if (i > j) A[j + i * n] = A[i + j * n];
    }
}

// info_d != nullptr: no host synchronisation; the two cuSOLVER infos are written to info_d[0..1]
// for the caller to check once (the ND setup inverts many fronts back to back)
static void spd_invert(double *A, int64_t n64, cudaStream_t s, int *info_d) {
    Lapack &L = lapack();
    if (!L.handle) {
        gj_invert(A, n64, s);
        if (info_d) CR_CUDA(cudaMemsetAsync(info_d, 0, 2 * sizeof(int), s));
        return;
    }
    const int n = (int)n64, lower = 0;
    L.SetStream(L.handle, s);
    int lw1 = 0, lw2 = 0;
    CR_REQUIRE(L.PotrfBS(L.handle, lower, n, A, n, &lw1) == 0 && L.PotriBS(L.handle, lower, n, A, n, &lw2) == 0,
               CR_ERR_CUDA, "cusolverDn buffer size query failed");
    DevBuf<double> work;
    work.alloc(std::max(std::max(lw1, lw2), 1), s);
    DevBuf<int> info;
    int *inf = info_d;
    if (!inf) {
        info.alloc(2, s);
        inf = info.get();
    }
    CR_CUDA(cudaMemsetAsync(inf, 0, 2 * sizeof(int), s));
    CR_REQUIRE(L.Potrf(L.handle, lower, n, A, n, work.get(), lw1, inf) == 0, CR_ERR_CUDA, "cusolverDnDpotrf failed");
    CR_REQUIRE(L.Potri(L.handle, lower, n, A, n, work.get(), lw2, inf + 1) == 0, CR_ERR_CUDA, "cusolverDnDpotri failed");
    k_mirror_lower<<<grid_for(n64 * n64, 256, 16), 256, 0, s>>>(A, n64);
    CR_CHECK_LAUNCH();
    if (info_d) return;
    int hi[2] = {0, 0};
    CR_CUDA(cudaMemcpyAsync(hi, inf, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    CR_REQUIRE(hi[0] == 0 && hi[1] == 0, CR_ERR_SINGULAR_LOCAL, "coarse matrix is not positive definite (potrf/potri)");
}

// |A|^{-1} = V |Lambda|^{-1} V^t in place for a symmetric (indefinite) A: cuSOLVER syevd (plain
// library eigendecomposition), columns of V scaled by 1 / max(|lambda|, 1e-13 max|lambda|), one DGEMM
__global__ void k_scale_cols_absinv(const double *V, const double *w, int64_t n, double wmax, double *B) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / n;   // column-major: column j
        B[t] = V[t] / fmax(fabs(w[j]), 1e-13 * wmax);
    }
}

static void abs_invert(double *A, int64_t n64, cudaStream_t s) {
    Lapack &L = lapack();
    Blas &bl = blas();
    CR_REQUIRE(L.handle && L.SyevdBS && L.Syevd && bl.handle && bl.Dgemm, CR_ERR_CUDA,
               "cuSOLVER syevd / cuBLAS DGEMM unavailable for the coarse |E|^{-1}");
    const int n = (int)n64;
    L.SetStream(L.handle, s);
    DevBuf<double> w, B;
    w.alloc(n, s);
    B.alloc((size_t)n * n, s);
    int lw = 0;
    CR_REQUIRE(L.SyevdBS(L.handle, 1, 0, n, A, n, w.get(), &lw) == 0, CR_ERR_CUDA, "cusolverDnDsyevd_bufferSize failed");
    DevBuf<double> work;
    work.alloc(std::max(lw, 1), s);
    DevBuf<int> info;
    info.alloc(1, s);
    CR_REQUIRE(L.Syevd(L.handle, 1, 0, n, A, n, w.get(), work.get(), lw, info.get()) == 0, CR_ERR_CUDA,
               "cusolverDnDsyevd failed");
    std::vector<double> hw(n);
    int hi = 0;
    CR_CUDA(cudaMemcpyAsync(hw.data(), w.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&hi, info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    CR_REQUIRE(hi == 0, CR_ERR_CUDA, "cusolverDnDsyevd did not converge");
    double wmax = 0.0;
    for (double v : hw) wmax = std::max(wmax, std::fabs(v));
    CR_REQUIRE(wmax > 0.0, CR_ERR_SINGULAR_LOCAL, "coarse matrix is zero");
    k_scale_cols_absinv<<<grid_for(n64 * n64, 256, 16), 256, 0, s>>>(A, w.get(), n64, wmax, B.get());
    CR_CHECK_LAUNCH();
    // A <- B V^t (column-major, symmetric up to rounding; symmetrised below)
    DevBuf<double> V;
    V.alloc((size_t)n * n, s);
    CR_CUDA(cudaMemcpyAsync(V.get(), A, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    bl.SetStream(bl.handle, s);
    const double one = 1.0, zero = 0.0;
    CR_REQUIRE(bl.Dgemm(bl.handle, 0, 1, n, n, n, &one, B.get(), n, V.get(), n, &zero, A, n) == 0, CR_ERR_CUDA,
               "cublasDgemm failed");
    k_symmetrize<<<grid_for(n64 * n64, 256, 64), 256, 0, s>>>(A, n64);
    CR_CHECK_LAUNCH();
}

static bool lapack_potrf_batched(int n, int lda, int nb, double **A, int *info, cudaStream_t s) {
    Lapack &L = lapack();
    if (!L.handle || !L.PotrfB) return false;
    L.SetStream(L.handle, s);
    CR_REQUIRE(L.PotrfB(L.handle, 0, n, A, lda, info, nb) == 0, CR_ERR_CUDA, "cusolverDnDpotrfBatched failed");
    return true;
}

__global__ void k_coarse_scale(double *a, int64_t n, double f) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] *= f;
}

template <int D>
static void build_coarse_t(cr_hybrid_s *h, int H, const ApplyG &applyG, const ApplyGColour &applyGc, cudaStream_t s) {
    constexpr int NN = 1 << D, NV = NN * D * D;
    const cr_mesh_s *m = h->mesh;
    CoarseOp &C = h->coarse;
    const int64_t nrows = h->G.nrows, row0 = h->part.on ? h->part.row0 : 0;
    const int T = 256;
    C.g.H = H;
    Trace tr(s);
    {
        // min / max of the vertex coordinates by CUB
        DevBuf<double> lo, hi;
        lo.alloc(D, s); hi.alloc(D, s);
        std::vector<double> hlo(D), hhi(D);
        DevBuf<double> comp;
        comp.alloc(m->nf, s);
        for (int i = 0; i < D; ++i) {
            // face centroids span the hull of the vertices' convex combinations: enough for hats
            CR_CUDA(cudaMemcpy2DAsync(comp.get(), sizeof(double), m->xs.get() + i, D * sizeof(double), sizeof(double),
                                      m->nf, cudaMemcpyDeviceToDevice, s));
            size_t tb = 0;
            CR_CUDA(cub::DeviceReduce::Min(nullptr, tb, comp.get(), lo.get() + i, (int)m->nf, s));
            DevBuf<uint8_t> tmp;
            tmp.alloc(tb, s);
            CR_CUDA(cub::DeviceReduce::Min(tmp.get(), tb, comp.get(), lo.get() + i, (int)m->nf, s));
            CR_CUDA(cub::DeviceReduce::Max(tmp.get(), tb, comp.get(), hi.get() + i, (int)m->nf, s));
        }
        CR_CUDA(cudaMemcpyAsync(hlo.data(), lo.get(), D * sizeof(double), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaMemcpyAsync(hhi.data(), hi.get(), D * sizeof(double), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < D; ++i) {
            const double w = hhi[i] - hlo[i];
            C.g.lo[i] = (float)(hlo[i] - 1e-6 * w);
            C.g.inv[i] = (float)(H / (w * (1.0 + 2e-6)));
        }
    }
    int64_t nnode = 1, ncc = 1;
    for (int i = 0; i < D; ++i) { nnode *= (H + 1); ncc *= H; }
    C.nE = nnode * D * D;
    // per-row data and coarse cell
    C.fx.alloc(nrows * D, s);
    C.fa.alloc(nrows * D, s);
    DevBuf<uint32_t> cc, cc2, idx;
    cc.alloc(nrows, s); cc2.alloc(nrows, s); idx.alloc(nrows, s);
    C.perm.alloc(nrows, s);
    C.perm_so.release();   // solve-order copies follow the new rows (coarse_so)
    C.fx_so.release();
    C.fa_so.release();
    k_coarse_faces<D><<<grid_for(nrows, T), T, 0, s>>>(m->dof_face.get(), row0, nrows, m->face_cells.get(),
                                                       m->cell_faces.get(), m->a.get(), m->xs.get(), C.g, C.fx.get(),
                                                       C.fa.get(), cc.get());
    CR_CHECK_LAUNCH();
    // sort key: coarse cell x 2 + interior bit (single rank), so each cell's rows that G can couple
    // to a neighbouring cell come first
    const bool layered = !h->part.on;
    std::vector<int64_t> cbnd(ncc + 1, 0);   // per cell: first interior row (sorted position)
    {
        DevBuf<uint32_t> key;
        if (layered) {
            key.alloc(nrows, s);
            k_coarse_interior<D><<<grid_for(nrows, T), T, 0, s>>>(m->dof_face.get(), m->face_cells.get(),
                                                                  m->cell_faces.get(), m->face_dof.get(), nrows, cc.get(),
                                                                  key.get());
            CR_CHECK_LAUNCH();
            CR_CUDA(cudaMemcpyAsync(cc.get(), key.get(), nrows * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        }
        k_iota_u32<<<grid_for(nrows, T), T, 0, s>>>(idx.get(), nrows);
        CR_CHECK_LAUNCH();
        int bits = 1;
        while (((int64_t)1 << bits) < ncc * (layered ? 2 : 1)) ++bits;
        size_t tb = 0;
        CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, cc.get(), cc2.get(), idx.get(),
                                                reinterpret_cast<uint32_t *>(C.perm.get()), (int)nrows, 0, bits, s));
        DevBuf<uint8_t> tmp;
        tmp.alloc(tb, s);
        CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, cc.get(), cc2.get(), idx.get(),
                                                reinterpret_cast<uint32_t *>(C.perm.get()), (int)nrows, 0, bits, s));
        C.fxp.alloc(nrows * D, s);
        C.fap.alloc(nrows * D, s);
        k_coarse_permute_rows<D><<<grid_for(nrows, T), T, 0, s>>>(C.perm.get(), nrows, C.fx.get(), C.fa.get(), C.fxp.get(),
                                                                   C.fap.get());
        CR_CHECK_LAUNCH();
        // rows of each coarse cell (device), chunks of <= kCH rows (host: a few thousand entries)
        DevBuf<int64_t> cs;
        cs.alloc(ncc + 1, s);
        k_cell_starts<<<grid_for(ncc + 1, T), T, 0, s>>>(cc2.get(), nrows, ncc, cs.get(), layered ? 2 : 1, 0);
        CR_CHECK_LAUNCH();
        std::vector<int64_t> cstart(ncc + 1);
        CR_CUDA(cudaMemcpyAsync(cstart.data(), cs.get(), (ncc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        if (layered) {
            k_cell_starts<<<grid_for(ncc + 1, T), T, 0, s>>>(cc2.get(), nrows, ncc, cs.get(), 2, 1);
            CR_CHECK_LAUNCH();
            CR_CUDA(cudaMemcpyAsync(cbnd.data(), cs.get(), (ncc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            CR_CUDA(cudaStreamSynchronize(s));
        } else {
            cbnd = std::vector<int64_t>(cstart.begin() + 1, cstart.end());   // every row "boundary"
            cbnd.push_back(nrows);
        }
        std::vector<int64_t> chunk_start, cell_chunk(ncc + 1, 0);
        for (int64_t c = 0; c < ncc; ++c) {
            cell_chunk[c] = (int64_t)chunk_start.size();
            for (int64_t b = cstart[c]; b < cstart[c + 1]; b += kCH) chunk_start.push_back(b);
        }
        cell_chunk[ncc] = (int64_t)chunk_start.size();
        chunk_start.push_back(nrows);
        C.nchunk = (int64_t)chunk_start.size() - 1;
        C.chunk_start.alloc(chunk_start.size(), s);
        C.cell_chunk.alloc(cell_chunk.size(), s);
        CR_CUDA(cudaMemcpyAsync(C.chunk_start.get(), chunk_start.data(), chunk_start.size() * 8, cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaMemcpyAsync(C.cell_chunk.get(), cell_chunk.data(), cell_chunk.size() * 8, cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaStreamSynchronize(s));
    }
    C.part.alloc(std::max<int64_t>(C.nchunk, 1) * NV, s);
    C.c.alloc(C.nE, s);
    C.y.alloc(C.nE, s);
    C.gpart.alloc((size_t)num_sms() * 32, s);
    // dense E^{-1} (one bandwidth-bound GEMV per iteration) while it is at most 8000^2 doubles,
    // the ND sparse direct solve beyond (its ~2 log2(H) dependent levels cost latency, its bytes
    // grow only like nE log nE).  CR_COARSE_DENSE=1 / CR_COARSE_ND=1 force one (tests).
    const bool dense = C.absmode || (std::getenv("CR_COARSE_DENSE") ? true : std::getenv("CR_COARSE_ND") ? false
                                                                                                   : C.nE <= 8000);
    C.nd = CoarseNd();
    constexpr int NBR = D == 2 ? 25 : 125;
    DevBuf<double> Es;
    if (dense) {
        C.Einv.alloc(C.nE * C.nE, s);
        C.Einv.zero(s);
    } else {
        Es.alloc((size_t)nnode * NBR * D * D * D * D, s);
        Es.zero(s);
    }
    // E = Z^t G Z by colours
    CoarseView V = C.view();
    DevBuf<double> z, Y;
    const int64_t Nalloc = (nrows + (h->part.on ? h->part.nghost : 0)) * D;
    z.alloc(Nalloc, s);
    Y.alloc(Nalloc, s);
    z.zero(s);
    int ncol = 1;
    for (int i = 0; i < D; ++i) ncol *= 5;
    // Single rank: per colour, z is written only on the chunks of the coarse cells of its supports
    // (cell index = colour digit - 1 or colour digit, mod 5, in every direction: (2/5)^D of the
    // rows), G z is nonzero only one fine cell around them, so the restriction runs over the
    // chunks of cells at digit - 2 .. digit + 1 ((4/5)^D), and z and Y are cleared on those rows
    // afterwards instead of being rewritten / memset whole.  (Needs fine cells smaller than coarse
    // cells: the H clamp above.)
    const bool restricted = !h->part.on;
    std::vector<int32_t> lsup, lact;
    std::vector<int64_t> osup(ncol + 1, 0), oact(ncol + 1, 0), lend;
    DevBuf<int32_t> dsup, dact;
    DevBuf<int64_t> dend;
    if (restricted) {
        std::vector<int64_t> hcc(ncc + 1), hcs(C.nchunk + 1);
        CR_CUDA(cudaMemcpyAsync(hcc.data(), C.cell_chunk.get(), (ncc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaMemcpyAsync(hcs.data(), C.chunk_start.get(), (C.nchunk + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        for (int colour = 0; colour < ncol; ++colour) {
            for (int64_t cell = 0; cell < ncc; ++cell) {
                int64_t t = cell;
                int cl = colour;
                bool sup = true, act = true;
                for (int i = 0; i < D; ++i) {
                    const int x = (int)(t % H);
                    t /= H;
                    const int dgt = cl % 5;
                    cl /= 5;
                    const int dm = ((x - dgt) % 5 + 5) % 5;   // x - digit mod 5
                    sup = sup && (dm == 0 || dm == 4);
                    act = act && dm != 2;
                }
                for (int64_t ch = hcc[cell]; ch < hcc[cell + 1]; ++ch) {
                    if (sup) lsup.push_back((int32_t)ch);
                    if (sup) {   // the colour's supports: every row
                        lact.push_back((int32_t)ch);
                        lend.push_back(hcs[ch + 1]);
                    } else if (act && hcs[ch] < cbnd[cell]) {   // ring cells: rows G couples outside the cell
                        lact.push_back((int32_t)ch);
                        lend.push_back(std::min(hcs[ch + 1], cbnd[cell]));
                    }
                }
            }
            osup[colour + 1] = (int64_t)lsup.size();
            oact[colour + 1] = (int64_t)lact.size();
        }
        upload(dsup, lsup, s);
        upload(dact, lact, s);
        upload(dend, lend, s);
        Y.zero(s);
    }
    if (restricted) {
        // all D^2 (k, l) columns of a colour at once: one fill, one G application (D^2 right-hand
        // sides, cell factors read once), NC-column restrictions reading the row data once, one
        // gather and one scatter per colour (was one of each per column: 1,125 passes in 3D)
        constexpr int NCOL = D * D;
        const int64_t zs = Nalloc;
        DevBuf<double> zall, Yall, pall, call;
        if (!applyGc) {
            zall.alloc((size_t)NCOL * zs, s);
            zall.zero(s);
        }
        // interleaved rows padded to a multiple of 256 bytes (D^3 = 27 -> 32 doubles, 8 -> 8): whole
        // sectors when a row is cleared
        const int64_t YRS = D == 3 ? 32 : 8;
        Yall.alloc(applyGc ? (size_t)YRS * (zs / D) : (size_t)NCOL * zs, s);
        Yall.zero(s);
        const int64_t ps = C.nchunk * NV;
        pall.alloc((size_t)NCOL * ps, s);
        call.alloc((size_t)NCOL * C.nE, s);
        for (int colour = 0; colour < ncol; ++colour) {
            const unsigned nsup = (unsigned)(osup[colour + 1] - osup[colour]);
            const unsigned nact = (unsigned)(oact[colour + 1] - oact[colour]);
            if (applyGc) {   // G applied to the colour's columns without materialising them (Y interleaved)
                applyGc(colour, Yall.get(), YRS);
            } else {
                if (nsup)
                    k_coarse_colour_chunks_all<D><<<nsup, 256, 0, s>>>(V, dsup.get() + osup[colour], colour, 0, zall.get(), zs);
                CR_CHECK_LAUNCH();
                applyG(zall.get(), Yall.get(), colour, NCOL, zs);
            }
            pall.zero(s);
            if (nact) {
                // entry (row, column c, component i): interleaved rows of YRS doubles (applyGc; the last
                // restriction launch zeroes the rows it read) or column vectors (stride zs)
                const int64_t cstr = applyGc ? D : zs, rstr = applyGc ? YRS : D;
                if (D == 3) {
                    for (int c0 = 0; c0 < NCOL; c0 += 3)
                        k_coarse_restrict3m<3><<<nact, 256, 0, s>>>(
                            V, Yall.get() + c0 * cstr, cstr, pall.get() + c0 * ps, ps, dact.get() + oact[colour],
                            dend.get() + oact[colour], rstr, (applyGc && c0 + 3 == NCOL) ? Yall.get() : nullptr);
                } else {
                    for (int c = 0; c < NCOL; ++c)
                        k_coarse_restrict<D><<<nact, 256, 0, s>>>(V, Yall.get() + c * cstr, pall.get() + c * ps,
                                                                  dact.get() + oact[colour], dend.get() + oact[colour],
                                                                  rstr, (applyGc && c + 1 == NCOL) ? Yall.get() : nullptr);
                }
                CR_CHECK_LAUNCH();
            }
            k_coarse_gather_all<D><<<grid_for(C.nE * NCOL, T), T, 0, s>>>(V, pall.get(), ps, call.get());
            CR_CHECK_LAUNCH();
            // Y was cleared by the restriction that read it (every row G z can reach is read)
            if (!applyGc && nsup)
                k_coarse_colour_chunks_all<D><<<nsup, 256, 0, s>>>(V, dsup.get() + osup[colour], colour, 1, zall.get(), zs);
            CR_CHECK_LAUNCH();
            if (dense) {
                for (int k = 0; k < D; ++k)
                    for (int l = 0; l < D; ++l)
                        k_coarse_scatterE<D><<<grid_for(C.nE, T), T, 0, s>>>(C.nE, H, colour, k, l,
                                                                             call.get() + (k * D + l) * C.nE, C.Einv.get());
            } else {
                k_coarse_scatterEs_all<D><<<grid_for(C.nE * NCOL, T), T, 0, s>>>(C.nE, H, colour, call.get(), Es.get());
            }
            CR_CHECK_LAUNCH();
        }
    } else {
        // partitioned: every rank restricts its own rows (all chunks), the D^2 columns of a colour
        // in one pass and one allreduce of the D^2 restricted vectors per colour
        constexpr int NCOL = D * D;
        const int64_t zs = Nalloc;
        DevBuf<double> zall, Yall, pall, call;
        zall.alloc((size_t)NCOL * zs, s);
        Yall.alloc((size_t)NCOL * zs, s);
        zall.zero(s);
        Yall.zero(s);
        const int64_t ps = C.nchunk * NV;
        pall.alloc((size_t)NCOL * std::max<int64_t>(ps, 1), s);
        call.alloc((size_t)NCOL * C.nE, s);
        for (int colour = 0; colour < ncol; ++colour) {
            k_coarse_colour_all<D><<<grid_for(nrows, T), T, 0, s>>>(V, nrows, colour, zall.get(), zs);
            CR_CHECK_LAUNCH();
            applyG(zall.get(), Yall.get(), -1 - colour, NCOL, zs);
            if (C.nchunk > 0) {
                if (D == 3) {
                    for (int c0 = 0; c0 < NCOL; c0 += 3)
                        k_coarse_restrict3m<3><<<(unsigned)C.nchunk, 256, 0, s>>>(V, Yall.get() + c0 * zs, zs,
                                                                                pall.get() + c0 * ps, ps, nullptr, nullptr);
                } else {
                    for (int c = 0; c < NCOL; ++c)
                        k_coarse_restrict<D><<<(unsigned)C.nchunk, 256, 0, s>>>(V, Yall.get() + c * zs, pall.get() + c * ps);
                }
                CR_CHECK_LAUNCH();
            }
            k_coarse_gather_all<D><<<grid_for(C.nE * NCOL, T), T, 0, s>>>(V, pall.get(), ps, call.get());
            CR_CHECK_LAUNCH();
            h->comm->impl->allreduce(call.get(), (int)(C.nE * NCOL), false, s);
            if (dense) {
                for (int k = 0; k < D; ++k)
                    for (int l = 0; l < D; ++l)
                        k_coarse_scatterE<D><<<grid_for(C.nE, T), T, 0, s>>>(C.nE, H, colour, k, l,
                                                                             call.get() + (k * D + l) * C.nE, C.Einv.get());
            } else {
                k_coarse_scatterEs_all<D><<<grid_for(C.nE * NCOL, T), T, 0, s>>>(C.nE, H, colour, call.get(), Es.get());
            }
            CR_CHECK_LAUNCH();
        }
    }
    tr.mark("coarse: E = Z^t G Z");
    // relative weight theta of the coarse term in M^-1 = sum_p R_p^t B_p^-1 R_p + theta Z E^-1 Z^t
    // (E is scaled by 1/theta before it is factorised)
    if (C.weight != 1.0) {
        const int64_t ne = dense ? C.nE * C.nE : (int64_t)nnode * NBR * D * D * D * D;
        k_coarse_scale<<<grid_for(ne, T, 16), T, 0, s>>>(dense ? C.Einv.get() : Es.get(), ne, 1.0 / C.weight);
        CR_CHECK_LAUNCH();
    }
    if (dense) {
        k_symmetrize<<<grid_for(C.nE * C.nE, T, 64), T, 0, s>>>(C.Einv.get(), C.nE);
        CR_CHECK_LAUNCH();
        if (C.absmode) {
            abs_invert(C.Einv.get(), C.nE, s);
            tr.mark("coarse: |E|^-1 (syevd)");
        } else {
            spd_invert(C.Einv.get(), C.nE, s);
            tr.mark("coarse: E^-1 (Cholesky potrf + potri)");
        }
    } else {
        k_es_symmetrize<D><<<grid_for((int64_t)nnode * NBR * D * D * D * D, T, 16), T, 0, s>>>(nnode, H, Es.get());
        CR_CHECK_LAUNCH();
        nd_setup<D>(C, Es.get(), H, s);
        tr.mark("coarse: E factorised (nested dissection)");
    }
    C.built = H;
}

void build_coarse(cr_hybrid_s *h, int H, const ApplyG &applyG, const ApplyGColour &applyGc,
                  cudaStream_t s, bool absmode) {
    CR_REQUIRE(H >= 1 && H <= 256, CR_ERR_INVALID_ARG, "coarse grid intervals must be in [1, 256]");
    const int D = h->G.d;
    if (absmode) H = std::min(H, D == 2 ? 43 : 8);   // dense eigendecomposition: <= ~8,000 coarse unknowns
    if ((h->coarse.absmode != 0) != absmode) {       // the other inverse: rebuild
        h->coarse.built = 0;
        h->coarse.requested = 0;
    }
    h->coarse.absmode = absmode ? 1 : 0;
    if (const char *ew = std::getenv("CR_COARSE_WEIGHT")) {
        const double w = std::atof(ew);
        if (w > 0.0) h->coarse.weight = w;
    }
    // at least ~4 faces per coarse unknown: a coarse grid finer than the mesh makes Z rank-deficient
    const double nglob = (double)(h->part.on ? h->part.nglobal : h->G.nrows);
    const int hmax = std::max(1, (int)std::floor(std::pow(nglob / (4.0 * D * D), 1.0 / D)));
    H = std::min(H, hmax);
    if (h->coarse.built == H || h->coarse.requested == H) return;
    h->coarse.requested = H;
    while (true) {
        try {
            if (D == 2) build_coarse_t<2>(h, H, applyG, applyGc, s);
            else build_coarse_t<3>(h, H, applyG, applyGc, s);
            return;
        } catch (const Error &e) {
            if (e.code != CR_ERR_SINGULAR_LOCAL || H <= 1) throw;
            H /= 2;    // E not numerically positive definite: coarser grid
        }
    }
}

// per-iteration pieces (called from solve.cu)
__global__ void k_coarse_rows_so(const int32_t *perm, int64_t n, const int32_t *iperm, const float *fx, const float *fa,
                                 int D, int32_t *perm_so, float *fx_so, float *fa_so) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        perm_so[t] = iperm[perm[t]];
        const int64_t nr = iperm[t];   // row t in the solve order
        for (int i = 0; i < D; ++i) {
            fx_so[nr * D + i] = fx[t * D + i];
            fa_so[nr * D + i] = fa[t * D + i];
        }
    }
}

void coarse_so(cr_hybrid_s *h, cudaStream_t s) {
    CoarseOp &C = h->coarse;
    if (!h->so.built || !C.built || C.perm_so.n == C.perm.n) return;
    const int64_t n = (int64_t)C.perm.n;
    const int D = h->G.d;
    C.perm_so.alloc(n, s);
    C.fx_so.alloc((size_t)n * D, s);
    C.fa_so.alloc((size_t)n * D, s);
    k_coarse_rows_so<<<grid_for(n, 256), 256, 0, s>>>(C.perm.get(), n, h->so.iperm.get(), C.fx.get(), C.fa.get(), D,
                                                      C.perm_so.get(), C.fx_so.get(), C.fa_so.get());
    CR_CHECK_LAUNCH();
}

void coarse_restrict_solve(cr_hybrid_s *h, const double *r, double *qout, double *partials, unsigned *ticket,
                           cudaStream_t s, bool side, bool so) {
    CoarseOp &C = h->coarse;
    CoarseView V = so ? C.view_so() : C.view();
    const int T = 256;
    if (h->G.d == 2) {
        k_coarse_restrict<2><<<(unsigned)C.nchunk, 256, 0, s>>>(V, r, C.part.get());
        k_coarse_gather<2><<<grid_for(C.nE, T), T, 0, s>>>(V, C.part.get(), C.c.get());
    } else {
        // CR_RESTRICT=3b: the one-corner-per-lane restriction (measured 0.07 ms slower on configs[4])
        static const char *ep = std::getenv("CR_RESTRICT");
        if (!(ep && std::string(ep) == "3b")) k_coarse_restrict3c<<<(unsigned)C.nchunk, 256, 0, s>>>(V, r, C.part.get());
        else k_coarse_restrict3b<<<(unsigned)C.nchunk, 256, 0, s>>>(V, r, C.part.get());
        k_coarse_gather<3><<<grid_for(C.nE, T), T, 0, s>>>(V, C.part.get(), C.c.get());
    }
    CR_CHECK_LAUNCH();
    if (h->part.on) {
        if (side) h->comm->impl->allreduce_side(C.c.get(), (int)C.nE, s);
        else h->comm->impl->allreduce(C.c.get(), (int)C.nE, false, s);
    }
    if (C.nd.on) {
        nd_solve(C, C.c.get(), C.y.get(), qout, partials, ticket, s);
        return;
    }
    k_coarse_gemv<<<occ_grid(k_coarse_gemv, 128, C.nE * 128), 128, 0, s>>>(C.Einv.get(), C.nE, C.c.get(), C.y.get(),
                                                                           qout, partials, ticket);
    CR_CHECK_LAUNCH();
}

}  // namespace cr

// ------------------------------------------------------------------ host-only plan export (tests)
extern "C" cr_status cr_coarse_nd_plan(int32_t H, int32_t dim, int32_t box, int64_t *nfront, int32_t *maxdepth, int64_t *total_I,
                                       int64_t *total_B, int32_t *depth, int32_t *parent, int32_t *nI, int32_t *nB,
                                       int32_t *I_nodes, int32_t *B_nodes) {
    try {
        CR_REQUIRE(dim == 2 || dim == 3, CR_ERR_INVALID_ARG, "dim must be 2 or 3");
        CR_REQUIRE(H >= 1 && H <= 256, CR_ERR_INVALID_ARG, "H must be in [1, 256]");
        CR_REQUIRE(nfront && maxdepth && total_I && total_B, CR_ERR_INVALID_ARG, "null argument");
        std::vector<cr::HostFront> F;
        CR_REQUIRE(box >= 0, CR_ERR_INVALID_ARG, "box must be >= 0");
        cr::nd_plan(H, dim, F, box);
        int64_t ti = 0, tb = 0;
        int md = 0;
        for (size_t f = 0; f < F.size(); ++f) {
            if (depth) depth[f] = F[f].depth;
            if (parent) {
                if (f + 1 == F.size()) parent[f] = -1;
                for (int k : F[f].kids) parent[k] = (int32_t)f;
            }
            if (nI) nI[f] = (int32_t)F[f].I.size();
            if (nB) nB[f] = (int32_t)F[f].B.size();
            if (I_nodes) std::copy(F[f].I.begin(), F[f].I.end(), I_nodes + ti);
            if (B_nodes) std::copy(F[f].B.begin(), F[f].B.end(), B_nodes + tb);
            ti += (int64_t)F[f].I.size();
            tb += (int64_t)F[f].B.size();
            md = std::max(md, F[f].depth);
        }
        *nfront = (int64_t)F.size();
        *maxdepth = md;
        *total_I = ti;
        *total_B = tb;
        return CR_OK;
    } catch (const cr::Error &e) {
        cr::set_last_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        cr::set_last_error(e.what());
        return CR_ERR_INVALID_ARG;
    }
}
