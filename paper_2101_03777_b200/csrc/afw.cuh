// Overlapping-patch additive Schwarz preconditioner for G (device side of precond.cu).
//
//   M^{-1} r = sum_p R_p^t  B_p^{-1}  R_p r,     B_p = R_p G R_p^t  (one block per component)
//
// Patches are the interior faces around a vertex (2D) or around an edge (3D): the kernel of
// the cellwise signed sum sigma -> sum_{sigma in F_K} C_{K,sigma} W_sigma (the large 1/mu|K|
// part of G, P:L510-517 with S_K^{-1} of SURVEY A.1) is spanned by circulations around
// interior vertices (2D) / edges (3D), each supported on one patch, so the patch solves
// resolve both scales of G exactly where Jacobi resolves neither (Arnold-Falk-Winther-type
// space decomposition).
//
// Layout (sliced, 32 patches per slice = one warp, so every load is one coalesced 256-B row):
//   kl[slice]                         patch size k of the slice (max over its 32 patches)
//   ids[ioff[slice] + j*32 + lane]    (dof * SLOTS + slot) of patch face j, or -1 (padding)
//   vals[voff[slice] + (i*T + e)*32 + lane]
//        component i, entry e of B_p^{-1}: packed lower triangle (T = k(k+1)/2, symmetric
//        modes) or row-major k x k (T = k^2, general mode)
// A face belongs to exactly SLOTS patches (2 endpoints in 2D, 3 edges of a triangle in 3D);
// slot s of face sigma receives patch s's contribution in zs[(s*D + i)*nrows + dof] (one array per
// slot and component: a vertex's / edge's faces whose first vertex it is are consecutive dofs, so
// half the writes are coalesced), and consumers sum the SLOTS values in slot order, so the result
// is deterministic (no atomics).
#pragma once
#include <cstdint>

namespace cr {

struct AfwView {
    const int64_t *ioff, *voff;
    const uint8_t *kl;
    const int32_t *ids;
    const double *vals;
    int64_t npatch;
    int64_t nrows;   // block rows (zs stride)
    int shared = 0;  // 1: one block per patch for all D components (CR_AFW_SHARED, experiment)
};

// z-contributions of one patch for one velocity component: thread t of a launch covers slice
// t / (32 D), component (t / 32) % D, lane t % 32, so every load of ids / vals is one
// coalesced warp row.  Returns r_p^(i)t B_p^{-1} r_p^(i) (its sum over p, i is r^t M^{-1} r).
template <int D, int SLOTS, int KMAX, bool SYM>
__device__ __forceinline__ double afw_patch_comp(const AfwView &A, int64_t t, const double *__restrict__ r,
                                                 double *__restrict__ zs) {
    const int lane = (int)(t & 31);
    const int64_t w = t >> 5;
    const int64_t slice = w / D;
    const int i = (int)(w - slice * D);
    const int k = A.kl[slice];
    const int32_t *ip = A.ids + A.ioff[slice] + lane;
    int id[KMAX];
    double rv[KMAX], y[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) id[j] = (j < k) ? __ldcs(ip + j * 32) : -1;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        rv[j] = (id[j] >= 0) ? r[(int64_t)(id[j] / SLOTS) * D + i] : 0.0;
        y[j] = 0.0;
    }
    const int T = SYM ? k * (k + 1) / 2 : k * k;
    const double *vi = A.vals + A.voff[slice] + lane + (int64_t)(A.shared ? 0 : i) * T * 32;
    if (SYM && k == KMAX) {
        // full-size slice (nearly all of them): every operator load is issued before the first
        // FMA needs one, instead of one row's worth per (data-dependent) branch
        constexpr int TM = KMAX * (KMAX + 1) / 2;
        double v[TM];
#pragma unroll
        for (int e = 0; e < TM; ++e) v[e] = __ldcs(vi + e * 32);
#pragma unroll
        for (int a = 0; a < KMAX; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) {
                const double w = v[a * (a + 1) / 2 + b];
                y[a] = fma(w, rv[b], y[a]);
                if (a != b) y[b] = fma(w, rv[a], y[b]);
            }
    } else if constexpr (SYM) {
#pragma unroll
        for (int a = 0; a < KMAX; ++a) {
            if (a < k) {
#pragma unroll
                for (int b = 0; b <= a; ++b) {
                    const double v = __ldcs(vi + (a * (a + 1) / 2 + b) * 32);
                    y[a] = fma(v, rv[b], y[a]);
                    if (a != b) y[b] = fma(v, rv[a], y[b]);
                }
            }
        }
    } else {
#pragma unroll
        for (int a = 0; a < KMAX; ++a) {
            if (a < k) {
#pragma unroll
                for (int b = 0; b < KMAX; ++b)
                    if (b < k) y[a] = fma(__ldcs(vi + (a * k + b) * 32), rv[b], y[a]);
            }
        }
    }
    double quad = 0.0;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (id[j] >= 0) {
            quad = fma(rv[j], y[j], quad);
            zs[((int64_t)(id[j] % SLOTS) * D + i) * A.nrows + id[j] / SLOTS] = y[j];
        }
    }
    return quad;
}

// shared mode (one block per patch for all components, PCG): thread t covers patch t (slice t / 32,
// lane t % 32) and all D components, so the block is read once per patch.  Returns the patch's share
// of r^t M^{-1} r.
template <int D, int SLOTS, int KMAX>
__device__ __forceinline__ double afw_patch_shared(const AfwView &A, int64_t t, const double *__restrict__ r,
                                                   double *__restrict__ zs) {
    const int lane = (int)(t & 31);
    const int64_t slice = t >> 5;
    const int k = A.kl[slice];
    const int32_t *ip = A.ids + A.ioff[slice] + lane;
    int id[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) id[j] = (j < k) ? __ldcs(ip + j * 32) : -1;
    const double *vi = A.vals + A.voff[slice] + lane;
    constexpr int TM = KMAX * (KMAX + 1) / 2;
    double v[TM];
    if (k == KMAX) {
#pragma unroll
        for (int e = 0; e < TM; ++e) v[e] = __ldcs(vi + e * 32);
    } else {
#pragma unroll
        for (int a = 0; a < KMAX; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) v[a * (a + 1) / 2 + b] = (a < k) ? __ldcs(vi + (a * (a + 1) / 2 + b) * 32) : 0.0;
    }
    double quad = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double rv[KMAX], y[KMAX];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            rv[j] = (id[j] >= 0) ? r[(int64_t)(id[j] / SLOTS) * D + i] : 0.0;
            y[j] = 0.0;
        }
#pragma unroll
        for (int a = 0; a < KMAX; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) {
                const double w = v[a * (a + 1) / 2 + b];
                y[a] = fma(w, rv[b], y[a]);
                if (a != b) y[b] = fma(w, rv[a], y[b]);
            }
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            if (id[j] >= 0) {
                quad = fma(rv[j], y[j], quad);
                zs[((int64_t)(id[j] % SLOTS) * D + i) * A.nrows + id[j] / SLOTS] = y[j];
            }
        }
    }
    return quad;
}

// shared mode split over components (CR_AFW_SPLIT=1): warp (slice, component i) of a thread block
// whose D warps share the slice; ids and the packed block are read through the read-only path so
// the slice's other component warps find them in L1.  The component's products are the same FMAs
// in the same order as afw_patch_shared: identical slot values.
template <int D, int SLOTS, int KMAX>
__device__ __forceinline__ double afw_patch_split(const AfwView &A, int64_t slice, int i, int lane,
                                                  const double *__restrict__ r, double *__restrict__ zs) {
    const int k = A.kl[slice];
    const int32_t *ip = A.ids + A.ioff[slice] + lane;
    int id[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) id[j] = (j < k) ? __ldg(ip + j * 32) : -1;
    const double *vi = A.vals + A.voff[slice] + lane;
    constexpr int TM = KMAX * (KMAX + 1) / 2;
    double v[TM];
#pragma unroll
    for (int a = 0; a < KMAX; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) v[a * (a + 1) / 2 + b] = (a < k) ? __ldg(vi + (a * (a + 1) / 2 + b) * 32) : 0.0;
    double rv[KMAX], y[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        rv[j] = (id[j] >= 0) ? r[(int64_t)(id[j] / SLOTS) * D + i] : 0.0;
        y[j] = 0.0;
    }
#pragma unroll
    for (int a = 0; a < KMAX; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) {
            const double w = v[a * (a + 1) / 2 + b];
            y[a] = fma(w, rv[b], y[a]);
            if (a != b) y[b] = fma(w, rv[a], y[b]);
        }
    double quad = 0.0;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (id[j] >= 0) {
            quad = fma(rv[j], y[j], quad);
            zs[((int64_t)(id[j] % SLOTS) * D + i) * A.nrows + id[j] / SLOTS] = y[j];
        }
    }
    return quad;
}

// z[row] = sum_s zs[row, s] (slot order)
template <int D, int SLOTS>
__device__ __forceinline__ void afw_sum(const double *__restrict__ zs, int64_t nrows, int64_t row, double (&z)[D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) z[i] = zs[(int64_t)i * nrows + row];
#pragma unroll
    for (int s = 1; s < SLOTS; ++s)
#pragma unroll
        for (int i = 0; i < D; ++i) z[i] += zs[((int64_t)s * D + i) * nrows + row];
}

}  // namespace cr
