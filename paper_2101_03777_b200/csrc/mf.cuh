// Matrix-free factored application of G.
//
// G = sum_K H_K G_K H_K^t with, for transient Stokes (E_K = 0),
//     G_K = C_K [ I_d (x) Shat_K^{-1} - w w^t / B_K ] C_K,    w_i = Shat_K^{-1} D_K^{(i)},
// so a cell needs Shat_K^{-1} (symmetric, one block shared by the d components) and
// u = w / sqrt(B_K) instead of its (d s_K)^2 entries of G.  For a cell whose d+1 faces are
// all interior, Shat_K^{-1} = (1/(mu|K|)) 1 1^t + T_K (the 1/alpha P_1 part), and T_K
// is stored separately so that its O(|K|/nu) entries keep full relative precision next to the
// O(1/(mu|K|)) part.  Per cell (2D): c, T (6), u (6) = 13 doubles + 3 face ids + sign mask =
// 116 B against 270 B of assembled G per cell; 3D: 23 doubles + 4 ids, 200 B against 1056 B.
//
// Layout (32 cells per slice, lane-contiguous so every load is a coalesced warp row):
//   ids [slice][l][lane]   local dof of local face l (-1: boundary face)
//   sg  [slice*32 + lane]  bit l set <=> C_{K,l} = -1
//   v   [slice][e][lane]   e = 0: c;  1 .. NT: T packed lower triangle;  then u[i][l]
#pragma once
#include <cstdint>

namespace cr {

template <int D>
struct MfLayout {
    static constexpr int NF = D + 1;
    static constexpr int NT = NF * (NF + 1) / 2;
    static constexpr int NE = 1 + NT + D * NF;
};

struct MfView {
    const int32_t *ids;
    const uint8_t *sg;
    const double *v;
    int64_t ncells;     // cells processed (padded to slices of 32 with ids = -1)
};

// y_K = G_K x_K scattered into q (q pre-zeroed: exactly two cells add into each interior face, so
// 0 + a + b rounds the same in either order -> deterministic).  Returns this cell's share of
// p^t G p counted on rows < nown (owned rows).
template <int D>
__device__ __forceinline__ double mf_cell(const MfView &M, int64_t t, const double *__restrict__ x,
                                          double *__restrict__ q, int64_t nown) {
    using LY = MfLayout<D>;
    constexpr int NF = LY::NF, NT = LY::NT;
    const int64_t slice = t >> 5;
    const int lane = (int)(t & 31);
    const int32_t *ip = M.ids + slice * (NF * 32) + lane;
    const double *vp = M.v + slice * ((int64_t)LY::NE * 32) + lane;
    int id[NF];
    double cs[NF];
    const unsigned sg = M.sg[t];
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        id[l] = __ldcs(ip + l * 32);
        cs[l] = ((sg >> l) & 1u) ? -1.0 : 1.0;
    }
    const double c = __ldcs(vp);
    double T[NT], u[D][NF];
#pragma unroll
    for (int e = 0; e < NT; ++e) T[e] = __ldcs(vp + (1 + e) * 32);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int l = 0; l < NF; ++l) u[i][l] = __ldcs(vp + (1 + NT + i * NF + l) * 32);
    double xs[D][NF];
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        if (id[l] >= 0) {
            if constexpr (D == 2) {
                const double2 v2 = __ldg(reinterpret_cast<const double2 *>(x) + id[l]);
                xs[0][l] = cs[l] * v2.x;
                xs[1][l] = cs[l] * v2.y;
            } else {
#pragma unroll
                for (int i = 0; i < D; ++i) xs[i][l] = cs[l] * __ldg(x + (int64_t)id[l] * D + i);
            }
        } else {
#pragma unroll
            for (int i = 0; i < D; ++i) xs[i][l] = 0.0;
        }
    }
    // projection coefficient sum_j u_j^t xs_j
    double pu = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int l = 0; l < NF; ++l) pu = fma(u[i][l], xs[i][l], pu);
    double quad = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double sum = 0.0;
#pragma unroll
        for (int l = 0; l < NF; ++l) sum += xs[i][l];
        const double cb = c * sum;
#pragma unroll
        for (int a = 0; a < NF; ++a) {
            double y = cb;
#pragma unroll
            for (int b = 0; b < NF; ++b) {
                const int e = a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
                y = fma(T[e], xs[i][b], y);
            }
            y = fma(-u[i][a], pu, y);
            if (id[a] >= 0 && id[a] < nown) {
                quad = fma(xs[i][a], y, quad);
                atomicAdd(q + (int64_t)id[a] * D + i, cs[a] * y);
            }
        }
    }
    return quad;
}

}  // namespace cr
