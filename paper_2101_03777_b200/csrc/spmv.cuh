// Sliced block-ELL SpMV row kernel for G (d x d blocks, W = 2d+1 blocks per block row).
//
// HBM layout (per slice of 32 consecutive block rows = one warp):
//   cols[slice][k][lane]                 int32 block column (padding: the row itself)
//   vals[slice][k*d*d + i*d + j][lane]   fp64
// so every warp-wide load of one (k, i, j) entry reads 32 consecutive doubles (256 B,
// fully coalesced), and a block row's values stream exactly once per SpMV.
#pragma once
#include <cstdint>

namespace cr {

template <int D>
struct EllView {
    const int32_t *cols;
    const double *vals;
    int64_t nrows;
};

// y = (G x)[row r, 0..D-1]
template <int D>
__device__ __forceinline__ void spmv_row(const EllView<D> &G, int64_t r, const double *__restrict__ x, double y[D]) {
    constexpr int W = 2 * D + 1, B2 = D * D;
    const int64_t slice = r >> 5;
    const int lane = (int)(r & 31);
    const int32_t *cp = G.cols + slice * (W * 32) + lane;
    const double *vp = G.vals + slice * ((int64_t)W * B2 * 32) + lane;
    int c[W];
#pragma unroll
    for (int k = 0; k < W; ++k) c[k] = __ldcs(cp + k * 32);
    double v[W][B2];
#pragma unroll
    for (int k = 0; k < W; ++k)
#pragma unroll
        for (int e = 0; e < B2; ++e) v[k][e] = __ldcs(vp + (k * B2 + e) * 32);
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
        double xv[D];
        if constexpr (D == 2) {
            double2 t = __ldg(reinterpret_cast<const double2 *>(x) + c[k]);
            xv[0] = t.x;
            xv[1] = t.y;
        } else {
#pragma unroll
            for (int j = 0; j < D; ++j) xv[j] = __ldg(x + (int64_t)c[k] * D + j);
        }
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) y[i] = fma(v[k][i * D + j], xv[j], y[i]);
    }
}

// ------------------------------------------------------------------ deterministic reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV values, write this block's partials, and let the LAST block to finish
// (ticket counter) sum all partials in fixed block order and call fin(tot) on thread 0.
// Deterministic: fixed grid, fixed thread->data map, fixed summation trees.
template <int NV, class Fin>
__device__ __forceinline__ void reduce_and_finish(double (&v)[NV], double *partials, unsigned *ticket, Fin fin) {
    __shared__ double sh[NV][32];
    __shared__ int s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[i][warp] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += sh[i][w];
            partials[(int64_t)blockIdx.x * NV + i] = t;
        }
        __threadfence();
        unsigned tk = atomicAdd(ticket, 1u);
        s_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double tot[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
        for (int i = 0; i < NV; ++i) tot[i] += __ldcg(partials + (int64_t)b * NV + i);
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] = warp_sum(tot[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[i][warp] = tot[i];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += sh[i][w];
            tot[i] = t;
        }
        fin(tot);
        *ticket = 0u;
    }
}

}  // namespace cr
