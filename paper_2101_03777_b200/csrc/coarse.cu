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
#include <dlfcn.h>

#include <algorithm>
#include <cmath>

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

// partial restriction of one chunk: the 2^D nodes of its coarse cell x D^2 tensor components.
// One thread per row with all 2^D D^2 accumulators (16 in 2D, 72 in 3D); rows are read 4 at a time
// per thread (independent loads in flight); warp shuffles then shared memory reduce the block
// (fixed trees: deterministic).
template <int D>
__global__ void __launch_bounds__(256) k_coarse_restrict(CoarseView C, const double *r, double *part) {
    constexpr int NN = 1 << D, DD = D * D, NV = NN * DD;
    constexpr int TPR = 1;                           // threads per row
    constexpr int NA = NV;                           // accumulators per thread
    constexpr int SL = 256 / TPR, U = 4;
    const int64_t ch = blockIdx.x;
    const int64_t b = C.chunk_start[ch], e = C.chunk_start[ch + 1];
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
                xv[u][i] = ok ? C.fx[row[u] * D + i] : 0.f;
                av[u][i] = ok ? C.fa[row[u] * D + i] : 0.f;
                rv[u][i] = ok ? r[row[u] * D + i] : 0.0;
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

// first sorted position with coarse cell >= c (c = 0..ncc)
__global__ void k_cell_starts(const uint32_t *cc_sorted, int64_t n, int64_t ncc, int64_t *cstart) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= ncc; c += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)cc_sorted[mid] < c) lo = mid + 1;
            else hi = mid;
        }
        cstart[c] = lo;
    }
}

__global__ void k_iota_u32(uint32_t *a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

template <int D>
static void build_coarse_t(cr_hybrid_s *h, int H, const std::function<void(const double *, double *, int)> &applyG,
                           cudaStream_t s) {
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
    k_coarse_faces<D><<<grid_for(nrows, T), T, 0, s>>>(m->dof_face.get(), row0, nrows, m->face_cells.get(),
                                                       m->cell_faces.get(), m->a.get(), m->xs.get(), C.g, C.fx.get(),
                                                       C.fa.get(), cc.get());
    CR_CHECK_LAUNCH();
    {
        k_iota_u32<<<grid_for(nrows, T), T, 0, s>>>(idx.get(), nrows);
        CR_CHECK_LAUNCH();
        int bits = 1;
        while (((int64_t)1 << bits) < ncc) ++bits;
        size_t tb = 0;
        CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, cc.get(), cc2.get(), idx.get(),
                                                reinterpret_cast<uint32_t *>(C.perm.get()), (int)nrows, 0, bits, s));
        DevBuf<uint8_t> tmp;
        tmp.alloc(tb, s);
        CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, cc.get(), cc2.get(), idx.get(),
                                                reinterpret_cast<uint32_t *>(C.perm.get()), (int)nrows, 0, bits, s));
        // rows of each coarse cell (device), chunks of <= kCH rows (host: a few thousand entries)
        DevBuf<int64_t> cs;
        cs.alloc(ncc + 1, s);
        k_cell_starts<<<grid_for(ncc + 1, T), T, 0, s>>>(cc2.get(), nrows, ncc, cs.get());
        CR_CHECK_LAUNCH();
        std::vector<int64_t> cstart(ncc + 1);
        CR_CUDA(cudaMemcpyAsync(cstart.data(), cs.get(), (ncc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
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
    C.gpart.alloc((size_t)kSMs * 32, s);
    C.Einv.alloc(C.nE * C.nE, s);
    C.Einv.zero(s);
    // E = Z^t G Z by colours
    CoarseView V = C.view();
    DevBuf<double> z, Y;
    const int64_t Nalloc = (nrows + (h->part.on ? h->part.nghost : 0)) * D;
    z.alloc(Nalloc, s);
    Y.alloc(Nalloc, s);
    z.zero(s);
    int ncol = 1;
    for (int i = 0; i < D; ++i) ncol *= 5;
    for (int colour = 0; colour < ncol; ++colour)
        for (int k = 0; k < D; ++k)
            for (int l = 0; l < D; ++l) {
                k_coarse_colour<D><<<grid_for(nrows, T), T, 0, s>>>(V, nrows, colour, k, l, z.get());
                CR_CHECK_LAUNCH();
                applyG(z.get(), Y.get(), colour);
                k_coarse_restrict<D><<<(unsigned)C.nchunk, 256, 0, s>>>(V, Y.get(), C.part.get());
                k_coarse_gather<D><<<grid_for(C.nE, T), T, 0, s>>>(V, C.part.get(), C.c.get());
                CR_CHECK_LAUNCH();
                if (h->part.on) h->comm->impl->allreduce(C.c.get(), (int)C.nE, false, s);
                k_coarse_scatterE<D><<<grid_for(C.nE, T), T, 0, s>>>(C.nE, H, colour, k, l, C.c.get(), C.Einv.get());
                CR_CHECK_LAUNCH();
            }
    tr.mark("coarse: E = Z^t G Z");
    k_symmetrize<<<grid_for(C.nE * C.nE, T, 64), T, 0, s>>>(C.Einv.get(), C.nE);
    CR_CHECK_LAUNCH();
    // blocked Gauss-Jordan on the row-major E (a row-major M is the column-major M^t for cuBLAS):
    //   Y = E[K,:];  X = E[:,K] Pk;  E -= X Y;  E[K,:] = Pk Y;  E[:,K] = -X, E[K,K] = Pk
    DevBuf<double> Pk, X, Yb;
    Pk.alloc(kGB * kGB, s);
    X.alloc(C.nE * kGB, s);
    Yb.alloc(C.nE * kGB, s);
    DevBuf<int> bad;
    bad.alloc(1, s);
    bad.zero(s);
    const int n = (int)C.nE;
    for (int64_t k0 = 0; k0 < C.nE; k0 += kGB) {
        const int b = (int)std::min<int64_t>(kGB, C.nE - k0);
        double *Ep = C.Einv.get();
        k_gj_diag<<<1, 256, 0, s>>>(Ep, C.nE, k0, b, Pk.get(), bad.get());
        CR_CUDA(cudaMemcpyAsync(Yb.get(), Ep + k0 * C.nE, (size_t)b * C.nE * sizeof(double), cudaMemcpyDeviceToDevice, s));
        dgemm(s, b, n, b, 1.0, Pk.get(), b, Ep + k0, n, 0.0, X.get(), b);            // X^t = Pk^t E[:,K]^t
        dgemm(s, n, n, b, -1.0, Yb.get(), n, X.get(), b, 1.0, Ep, n);                  // E^t -= Y^t X^t
        dgemm(s, n, b, b, 1.0, Yb.get(), n, Pk.get(), b, 0.0, Ep + k0 * C.nE, n);     // E[K,:]^t = Y^t Pk^t
        k_gj_cols<<<grid_for(C.nE * b, T), T, 0, s>>>(Ep, C.nE, k0, b, Pk.get(), X.get());
    }
    CR_CHECK_LAUNCH();
    int hb = 0;
    CR_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    tr.mark("coarse: E^-1 (Gauss-Jordan)");
    CR_REQUIRE(hb == 0, CR_ERR_SINGULAR_LOCAL, "coarse matrix Z^t G Z is not positive definite");
    C.built = H;
}

void build_coarse(cr_hybrid_s *h, int H, const std::function<void(const double *, double *, int)> &applyG,
                  cudaStream_t s) {
    CR_REQUIRE(H >= 1 && H <= 64, CR_ERR_INVALID_ARG, "coarse grid intervals must be in [1, 64]");
    const int D = h->G.d;
    // at least ~4 faces per coarse unknown: a coarse grid finer than the mesh makes Z rank-deficient
    const double nglob = (double)(h->part.on ? h->part.nglobal : h->G.nrows);
    const int hmax = std::max(1, (int)std::floor(std::pow(nglob / (4.0 * D * D), 1.0 / D)));
    H = std::min(H, hmax);
    if (h->coarse.built == H || h->coarse.requested == H) return;
    h->coarse.requested = H;
    while (true) {
        try {
            if (D == 2) build_coarse_t<2>(h, H, applyG, s);
            else build_coarse_t<3>(h, H, applyG, s);
            return;
        } catch (const Error &e) {
            if (e.code != CR_ERR_SINGULAR_LOCAL || H <= 1) throw;
            H /= 2;    // E not numerically positive definite: coarser grid
        }
    }
}

// per-iteration pieces (called from solve.cu)
void coarse_restrict_solve(cr_hybrid_s *h, const double *r, double *qout, double *partials, unsigned *ticket,
                           cudaStream_t s) {
    CoarseOp &C = h->coarse;
    CoarseView V = C.view();
    const int T = 256;
    if (h->G.d == 2) {
        k_coarse_restrict<2><<<(unsigned)C.nchunk, 256, 0, s>>>(V, r, C.part.get());
        k_coarse_gather<2><<<grid_for(C.nE, T), T, 0, s>>>(V, C.part.get(), C.c.get());
    } else {
        k_coarse_restrict<3><<<(unsigned)C.nchunk, 256, 0, s>>>(V, r, C.part.get());
        k_coarse_gather<3><<<grid_for(C.nE, T), T, 0, s>>>(V, C.part.get(), C.c.get());
    }
    CR_CHECK_LAUNCH();
    if (h->part.on) h->comm->impl->allreduce(C.c.get(), (int)C.nE, false, s);
    k_coarse_gemv<<<occ_grid(k_coarse_gemv, 128, C.nE * 128), 128, 0, s>>>(C.Einv.get(), C.nE, C.c.get(), C.y.get(),
                                                                           qout, partials, ticket);
    CR_CHECK_LAUNCH();
}

}  // namespace cr
