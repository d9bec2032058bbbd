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

// q[i] += v with no return value: red.global (atomicAdd compiles to a returning ATOMG in kernels
// that also fence, e.g. the reducing k_mf_spmv, and each then waits for its L2 round trip)
__device__ __forceinline__ void red_add_f64(double *p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// y_K = G_K x_K scattered into q (q pre-zeroed).  A face whose two cells sit in the same warp
// (32 consecutive cells: most faces inside a structured row of squares / a Kuhn cube) is summed
// in registers through shuffles and stored once by the lower cell; the others get one atomicAdd
// from each side.  Either way exactly two contributions meet, and 0 + a + b rounds the same in
// either order -> deterministic.  Returns this cell's share of p^t G p on rows < nown (owned).
// (factors already loaded: id, sign mask, c, T, u, in-warp partner codes)
// scatter of component i of one cell's contribution y[a] (local face a) into q: the pair of an in-warp
// shared face summed in registers and stored by the lower cell, the others by one atomicAdd per side
template <int D>
__device__ __forceinline__ void mf_scatter(const int (&id)[D + 1], const double (&cs)[D + 1], const double (&y)[D + 1],
                                           const unsigned (&nbc)[D + 1], int lane, int i, double *__restrict__ q,
                                           int64_t nown, int64_t qrs) {
    constexpr int NF = D + 1;
    double out[NF];
#pragma unroll
    for (int a = 0; a < NF; ++a) out[a] = cs[a] * y[a];
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
        double *dst = q + (int64_t)id[a] * qrs + i;   // qrs: row stride of q (D, or interleaved columns)
        if (nbc[a] & 0x80u) {
            if ((int)(nbc[a] & 31u) > lane) *dst = out[a] + part[a];   // lower cell stores the pair
        } else {
            red_add_f64(dst, out[a]);
        }
    }
}

// the cell's contribution for already gathered, sign-applied face values xs[i][l] = C_l x_(l, i)
template <int D>
__device__ __forceinline__ double mf_cell_core_xs(const int (&id)[D + 1], const double (&cs)[D + 1],
                                                  const double (&xs)[D][D + 1], double c,
                                                  const double (&T)[MfLayout<D>::NT], const double (&u)[D][D + 1],
                                                  const unsigned (&nbc)[D + 1], int lane, double *__restrict__ q,
                                                  int64_t nown, int64_t qrs = D) {
    constexpr int NF = D + 1;
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
        double y[NF];
#pragma unroll
        for (int a = 0; a < NF; ++a) {
            double v = cb;
#pragma unroll
            for (int b = 0; b < NF; ++b) {
                const int e = a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
                v = fma(T[e], xs[i][b], v);
            }
            v = fma(-u[i][a], pu, v);
            if (id[a] >= 0 && id[a] < nown) quad = fma(xs[i][a], v, quad);
            y[a] = v;
        }
        mf_scatter<D>(id, cs, y, nbc, lane, i, q, nown, qrs);
    }
    return quad;
}

// input in one velocity component k only (xk[l] = C_l x_(l, k); the coarse setup's columns e_k s a^(l))
template <int D>
__device__ __forceinline__ void mf_cell_core_1c(const int (&id)[D + 1], const double (&cs)[D + 1], const double (&xk)[D + 1],
                                                int k, double c, const double (&T)[MfLayout<D>::NT],
                                                const double (&u)[D][D + 1], const unsigned (&nbc)[D + 1], int lane,
                                                double *__restrict__ q, int64_t nown, int64_t qrs) {
    constexpr int NF = D + 1;
    double pu = 0.0, sum = 0.0;
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        pu = fma(u[k][l], xk[l], pu);
        sum += xk[l];
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double y[NF];
#pragma unroll
        for (int a = 0; a < NF; ++a) {
            double v = -u[i][a] * pu;
            if (i == k) {
                double t = c * sum;
#pragma unroll
                for (int b = 0; b < NF; ++b) {
                    const int e = a >= b ? a * (a + 1) / 2 + b : b * (b + 1) / 2 + a;
                    t = fma(T[e], xk[b], t);
                }
                v = fma(-u[i][a], pu, t);
            }
            y[a] = v;
        }
        mf_scatter<D>(id, cs, y, nbc, lane, i, q, nown, qrs);
    }
}

// (factors already loaded: id, sign mask, c, T, u, in-warp partner codes; x gathered here)
template <int D>
__device__ __forceinline__ double mf_cell_core(const int (&id)[D + 1], unsigned sg, double c,
                                               const double (&T)[MfLayout<D>::NT], const double (&u)[D][D + 1],
                                               const unsigned (&nbc)[D + 1], int lane, const double *__restrict__ x,
                                               double *__restrict__ q, int64_t nown) {
    constexpr int NF = D + 1;
    double cs[NF];
#pragma unroll
    for (int l = 0; l < NF; ++l) cs[l] = ((sg >> l) & 1u) ? -1.0 : 1.0;
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
    return mf_cell_core_xs<D>(id, cs, xs, c, T, u, nbc, lane, q, nown);
}

// the same cell, factors streamed from HBM (coalesced warp rows)
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
#pragma unroll
    for (int l = 0; l < NF; ++l) id[l] = __ldcs(ip + l * 32);
    const unsigned sg = M.sg[t];
    const double c = __ldcs(vp);
    double T[NT], u[D][NF];
#pragma unroll
    for (int e = 0; e < NT; ++e) T[e] = __ldcs(vp + (1 + e) * 32);
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int l = 0; l < NF; ++l) u[i][l] = __ldcs(vp + (1 + NT + i * NF + l) * 32);
    unsigned nbc[NF];
#pragma unroll
    for (int a = 0; a < NF; ++a) nbc[a] = M.nb[slice * (NF * 32) + a * 32 + lane];
    return mf_cell_core<D>(id, sg, c, T, u, nbc, lane, x, q, nown);
}

// ------------------------------------------------------------------ TMA-staged slices
// One 32-cell slice as it lies in HBM, copied whole into shared memory by the bulk-copy engine
// (cp.async.bulk: v, ids, nb, sg are contiguous per slice): v [NE][32] f64, ids [NF][32] i32,
// nb [NF][32] u8, sg [32] u8.  All four sizes and offsets are multiples of 16 bytes.
template <int D>
struct MfSlice {
    static constexpr int NF = D + 1, NE = MfLayout<D>::NE;
    static constexpr int V = NE * 32 * 8, IDS = NF * 32 * 4, NB = NF * 32, SG = 32;
    static constexpr int OFF_IDS = V, OFF_NB = V + IDS, OFF_SG = V + IDS + NB;
    static constexpr int BYTES = V + IDS + NB + SG;
    static_assert(V % 16 == 0 && IDS % 16 == 0 && NB % 16 == 0 && BYTES % 16 == 0, "bulk-copy granularity");
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// the elected lane arms the stage's barrier and issues the four bulk copies of slice `sl`
template <int D>
__device__ __forceinline__ void mf_issue_slice(const MfView &M, int64_t sl, unsigned char *stage, uint64_t *bar) {
    using SL = MfSlice<D>;
    mbar_expect_tx(bar, SL::BYTES);
    bulk_g2s(stage, M.v + sl * (int64_t)(SL::NE * 32), SL::V, bar);
    bulk_g2s(stage + SL::OFF_IDS, M.ids + sl * (int64_t)(SL::NF * 32), SL::IDS, bar);
    bulk_g2s(stage + SL::OFF_NB, M.nb + sl * (int64_t)(SL::NF * 32), SL::NB, bar);
    bulk_g2s(stage + SL::OFF_SG, M.sg + sl * 32, SL::SG, bar);
}

// the cell of `lane` in a staged slice
template <int D>
__device__ __forceinline__ double mf_cell_staged(const unsigned char *stage, int lane, const double *__restrict__ x,
                                                 double *__restrict__ q, int64_t nown) {
    using LY = MfLayout<D>;
    using SL = MfSlice<D>;
    constexpr int NF = LY::NF, NT = LY::NT;
    const double *vp = reinterpret_cast<const double *>(stage) + lane;
    const int32_t *ip = reinterpret_cast<const int32_t *>(stage + SL::OFF_IDS) + lane;
    const uint8_t *np = stage + SL::OFF_NB + lane;
    int id[NF];
    unsigned nbc[NF];
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        id[l] = ip[l * 32];
        nbc[l] = np[l * 32];
    }
    const unsigned sg = stage[SL::OFF_SG + lane];
    const double c = vp[0];
    double T[NT], u[D][NF];
#pragma unroll
    for (int e = 0; e < NT; ++e) T[e] = vp[(1 + e) * 32];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int l = 0; l < NF; ++l) u[i][l] = vp[(1 + NT + i * NF + l) * 32];
    return mf_cell_core<D>(id, sg, c, T, u, nbc, lane, x, q, nown);
}

}  // namespace cr
