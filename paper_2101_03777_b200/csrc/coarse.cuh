// Coarse space of the two-level preconditioner (coarse.cu): uniform grid of H^D cells over the
// mesh bounding box, (multi)linear hats, D^2 "stress" components per node.
#pragma once
#include <cstdint>

namespace cr {

struct CoarseGrid {
    int H = 0;
    float lo[3] = {0, 0, 0};
    float inv[3] = {0, 0, 0};   // H / width
};

struct CoarseView {
    CoarseGrid g;
    const float *fx, *fa;          // [rows][D] face centroid, area vector (fp32: a fixed basis)
    const int32_t *perm;           // rows sorted by coarse cell
    const float *fxp, *fap;        // fx, fa in that sorted order (the restrictions read them coalesced)
    const int64_t *chunk_start;    // [nchunk + 1]
    const int64_t *cell_chunk;     // [ncoarse_cells + 1]
    int64_t nE;                    // (H+1)^D D^2
};

// coarse cell and local coordinates in [0, 1]
template <int D>
__device__ __forceinline__ void coarse_locate(const CoarseGrid &g, const float *x, int (&ic)[D], float (&xi)[D]) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const float t = (x[i] - g.lo[i]) * g.inv[i];
        int c = (int)floorf(t);
        c = c < 0 ? 0 : (c > g.H - 1 ? g.H - 1 : c);
        ic[i] = c;
        float u = t - (float)c;
        xi[i] = u < 0.f ? 0.f : (u > 1.f ? 1.f : u);
    }
}

// hat weights of the 2^D corners of the coarse cell (corner n: bit i = +1 in direction i)
template <int D>
__device__ __forceinline__ void coarse_weights(const CoarseGrid &g, const float *x, double (&w)[1 << D]) {
    int ic[D];
    float xi[D];
    coarse_locate<D>(g, x, ic, xi);
#pragma unroll
    for (int n = 0; n < (1 << D); ++n) {
        double v = 1.0;
#pragma unroll
        for (int i = 0; i < D; ++i) v *= ((n >> i) & 1) ? (double)xi[i] : 1.0 - (double)xi[i];
        w[n] = v;
    }
}

// global coarse node of corner n
template <int D>
__device__ __forceinline__ int64_t coarse_node(const CoarseGrid &g, const int (&ic)[D], int n) {
    int64_t node = 0;
#pragma unroll
    for (int i = D - 1; i >= 0; --i) node = node * (g.H + 1) + ic[i] + ((n >> i) & 1);
    return node;
}

// does coarse cell ic have a corner node of colour `colour` (node indices mod 5, base-5 digits)?
template <int D>
__device__ __forceinline__ bool coarse_cell_active(const int (&ic)[D], int colour) {
#pragma unroll
    for (int n = 0; n < (1 << D); ++n) {
        int col = 0, mul = 1;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            col += ((ic[i] + ((n >> i) & 1)) % 5) * mul;
            mul *= 5;
        }
        if (col == colour) return true;
    }
    return false;
}

// (Z y) at a row: sum_n w_n sum_l a^(l) y[(node_n D + k) D + l]
template <int D>
__device__ __forceinline__ void coarse_prolong(const CoarseView &C, int64_t row, const double *y, double (&z)[D]) {
    int ic[D];
    float xi[D];
    coarse_locate<D>(C.g, C.fx + row * D, ic, xi);
    double w[1 << D];
    coarse_weights<D>(C.g, C.fx + row * D, w);
    double av[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        av[i] = C.fa[row * D + i];
        z[i] = 0.0;
    }
#pragma unroll
    for (int n = 0; n < (1 << D); ++n) {
        const double *yn = y + coarse_node<D>(C.g, ic, n) * D * D;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double s = 0.0;
#pragma unroll
            for (int l = 0; l < D; ++l) s = fma(av[l], yn[k * D + l], s);
            z[k] = fma(w[n], s, z[k]);
        }
    }
}

}  // namespace cr
