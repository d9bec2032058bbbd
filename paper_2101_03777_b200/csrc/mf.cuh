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
    const uint8_t *nb;  // [slice][l][lane]: 0x80 | l' << 5 | lane' when the other cell of face l is in
                        // the same 32-cell slice (as its local face l'), else 0
    int64_t ncells;     // cells processed (padded to slices of 32 with ids = -1)
};

// y_K = G_K x_K scattered into q (q pre-zeroed).  A face whose two cells sit in the same warp
// (32 consecutive cells: most faces inside a structured row of squares / a Kuhn cube) is summed
// in registers through shuffles and stored once by the lower cell; the others get one atomicAdd
// from each side.  Either way exactly two contributions meet, and 0 + a + b rounds the same in
// either order -> deterministic.  Returns this cell's share of p^t G p on rows < nown (owned).
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
    unsigned nbc[NF];
#pragma unroll
    for (int a = 0; a < NF; ++a) nbc[a] = M.nb[slice * (NF * 32) + a * 32 + lane];
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double sum = 0.0;
#pragma unroll
        for (int l = 0; l < NF; ++l) sum += xs[i][l];
        const double cb = c * sum;
        double out[NF];
#pragma unroll
        for (int a = 0; a < NF; ++a) {
            double y = cb;
#pragma unroll
            for (int b = 0; b < NF; ++b) {
                const int e = a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
                y = fma(T[e], xs[i][b], y);
            }
            y = fma(-u[i][a], pu, y);
            if (id[a] >= 0 && id[a] < nown) quad = fma(xs[i][a], y, quad);
            out[a] = cs[a] * y;
        }
        // the partner's contribution to each in-warp shared face (round b2 publishes face b2)
        double part[NF];
#pragma unroll
        for (int a = 0; a < NF; ++a) part[a] = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < NF; ++b2)
#pragma unroll
            for (int a = 0; a < NF; ++a) {
                const int src = (nbc[a] & 0x80u) ? (int)(nbc[a] & 31u) : lane;
                const double v = __shfl_sync(0xffffffffu, out[b2], src);
                if ((nbc[a] & 0x80u) && (int)((nbc[a] >> 5) & 3u) == b2) part[a] = v;
            }
#pragma unroll
        for (int a = 0; a < NF; ++a) {
            if (id[a] < 0 || id[a] >= nown) continue;
            double *dst = q + (int64_t)id[a] * D + i;
            if (nbc[a] & 0x80u) {
                if ((int)(nbc[a] & 31u) > lane) *dst = out[a] + part[a];   // lower cell stores the pair
            } else {
                atomicAdd(dst, out[a]);
            }
        }
    }
    return quad;
}

}  // namespace cr
