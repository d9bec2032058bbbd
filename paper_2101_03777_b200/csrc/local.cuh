// Per-cell local algebra of the hybrid method (device code), double-double.
//
//   S_K[s][t] = mu |K|/(d+1) delta_st + nu a_s . a_t / |K|          P:L261-265 (CR basis
//               gradient a_s/|K|, lumped mass |K|/(d+1))
//   A_K = I_d (x) S_K  (+ convection Jacobian for NS)
//   D_K = -a, R_K = a (fbar . (x_s - x_K))
//   Ahat_K = A_K + E_K; B_K = D^t Ahat^{-1} D
//   G_K = C (Ahat^{-1} - w v^t / B_K) C,  G_K0 = C Ahat^{-1} C
//   S_K = C (Ahat^{-1} R - w (v^t R - g)/B_K)
//
// Stokes (b_h = 0): Ahat_K = I_d (x) Shat_K with Shat_K = S_K + E_K (E_K acts identically
// on every component), so the elimination only needs an LDL^t factorisation of the
// s_K x s_K symmetric definite Shat_K (no pivoting needed for a definite matrix).
// Navier-Stokes step: the full (d s_K) x (d s_K) nonsymmetric Ahat_K, Gauss-Jordan with
// partial pivoting.  Everything is computed in double-double and rounded once.
#pragma once
#include "dd.cuh"
#include "internal.cuh"

namespace cr {

struct MeshView {
    const double *a, *vol, *xK, *xs;
    const int32_t *cell_faces, *face_dof, *face_cells;
};

inline MeshView mesh_view(const cr_mesh_s *m) {
    return {m->a.get(), m->vol.get(), m->xK.get(), m->xs.get(),
            m->cell_faces.get(), m->face_dof.get(), m->face_cells.get()};
}

struct ProbView {
    double mu = 0.0, nu = 0.0;
    int k0 = 0, is_ns = 0;
    const double *fbar = nullptr, *dir = nullptr, *uit = nullptr, *pit = nullptr, *E = nullptr;   // E [nc][d+1]
    // explicit cell right-hand sides (coupled defect correction, dc.cu): R_K [nc][d+1][d], g_K [nc];
    // when set they replace the force / Dirichlet terms of stokes_rhs
    const double *rcell = nullptr, *gcell = nullptr;
};

template <int D>
struct Cell {
    static constexpr int NF = D + 1;
    int64_t K;
    double a[NF][D];
    double vol;
    double xK[D];
    double xs[NF][D];
    int face[NF];
    int dof[NF];
    double C[NF];
    int s;        // number of interior faces s_K
    int map[NF];  // compact index -> local face
};

template <int D>
__device__ __forceinline__ void load_cell(const MeshView &mv, int64_t K, Cell<D> &c) {
    constexpr int NF = D + 1;
    c.K = K;
    c.vol = mv.vol[K];
#pragma unroll
    for (int i = 0; i < D; ++i) c.xK[i] = mv.xK[K * D + i];
    c.s = 0;
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        int f = mv.cell_faces[K * NF + l];
        c.face[l] = f;
        c.dof[l] = mv.face_dof[f];
        c.C[l] = (mv.face_cells[2 * (int64_t)f] == (int32_t)K) ? 1.0 : -1.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            c.a[l][i] = mv.a[(K * NF + l) * D + i];
            c.xs[l][i] = mv.xs[(int64_t)f * D + i];
        }
    }
#pragma unroll
    for (int l = 0; l < NF; ++l)
        if (c.dof[l] >= 0) c.map[c.s++] = l;
}

// S_K over all d+1 local faces, double-double
template <int D>
__device__ __forceinline__ dd S_entry(const Cell<D> &c, double mu, double nu, int s, int t) {
    dd dot = two_prod(c.a[s][0], c.a[t][0]);
#pragma unroll
    for (int i = 1; i < D; ++i) dot = dot + two_prod(c.a[s][i], c.a[t][i]);
    dd v = (dot * nu) / c.vol;
    if (s == t) v = v + two_prod(mu, c.vol) / (double)(D + 1);
    return v;
}

// R_K (all local faces, per component) incl. Dirichlet fold for Stokes, and g_K.
//   R[l][i] = a_l^i (fbar . (x_l - x_K)) - sum_{ext t} S[l][t] UD[t][i];   g = + sum_ext a_t . UD_t
template <int D>
__device__ __forceinline__ void stokes_rhs(const Cell<D> &c, const ProbView &p, dd R[D + 1][D], dd &g) {
    constexpr int NF = D + 1;
    const int64_t K = c.K;
    if (p.rcell) {
#pragma unroll
        for (int l = 0; l < NF; ++l)
#pragma unroll
            for (int i = 0; i < D; ++i) R[l][i] = dd_of(p.rcell[(K * NF + l) * D + i]);
        g = dd_of(p.gcell[K]);
        return;
    }
    dd fdx[NF];
#pragma unroll
    for (int l = 0; l < NF; ++l) {
        fdx[l] = dd_of(0.0);
#pragma unroll
        for (int i = 0; i < D; ++i) fdx[l] = fdx[l] + two_sum(c.xs[l][i], -c.xK[i]) * p.fbar[K * D + i];
    }
#pragma unroll
    for (int l = 0; l < NF; ++l)
#pragma unroll
        for (int i = 0; i < D; ++i) R[l][i] = fdx[l] * c.a[l][i];
    g = dd_of(0.0);
    if (p.dir) {
#pragma unroll
        for (int t = 0; t < NF; ++t) {
            if (c.dof[t] >= 0) continue;
            double ud[D];
#pragma unroll
            for (int j = 0; j < D; ++j) {
                ud[j] = p.dir[(K * NF + t) * D + j];
                g = g + two_prod(c.a[t][j], ud[j]);
            }
#pragma unroll
            for (int l = 0; l < NF; ++l) {
                if (c.dof[l] < 0) continue;
                dd st = S_entry<D>(c, p.mu, p.nu, l, t);
#pragma unroll
                for (int i = 0; i < D; ++i) R[l][i] = R[l][i] - st * ud[i];
            }
        }
    }
}

// --------------------------------------------------------------------------- Stokes path
template <int D>
struct StokesElim {
    static constexpr int NF = D + 1;
    dd L[NF][NF];   // unit lower factor of Shat (compact)
    dd Dg[NF];      // LDL^t diagonal
    dd w[D][NF];    // w_i = Shat^{-1} D_i (compact), D_i[p] = -a[map p][i]
    dd B;
    int status;     // DE_OK / DE_SINGULAR / DE_BZERO / DE_NOINTERIOR
};

template <int D>
__device__ __forceinline__ void ldl_solve(const StokesElim<D> &e, int s, dd x[D + 1]) {
    for (int i = 0; i < s; ++i)
        for (int k = 0; k < i; ++k) x[i] = x[i] - e.L[i][k] * x[k];
    for (int i = 0; i < s; ++i) x[i] = x[i] / e.Dg[i];
    for (int i = s - 1; i >= 0; --i)
        for (int k = i + 1; k < s; ++k) x[i] = x[i] - e.L[k][i] * x[k];
}

template <int D>
__device__ __forceinline__ void stokes_eliminate(const Cell<D> &c, const ProbView &p, StokesElim<D> &e) {
    constexpr int NF = D + 1;
    const int s = c.s;
    e.status = DE_OK;
    if (s == 0) { e.status = DE_NOINTERIOR; return; }
    dd Sh[NF][NF];
    double mx = 0.0;
    for (int q = 0; q < s; ++q)
        for (int r = 0; r <= q; ++r) {
            dd v = S_entry<D>(c, p.mu, p.nu, c.map[q], c.map[r]);
            if (q == r && p.E) v = v + p.E[c.K * NF + c.map[q]];
            Sh[q][r] = v;
            Sh[r][q] = v;
            mx = fmax(mx, fabs(v.hi));
        }
    // LDL^t (Shat is definite: positive on M2 / transient cells, negative on M1 cells)
    for (int j = 0; j < s; ++j) {
        dd dj = Sh[j][j];
        for (int k = 0; k < j; ++k) dj = dj - e.L[j][k] * e.L[j][k] * e.Dg[k];
        e.Dg[j] = dj;
        if (!(fabs(dj.hi) > 1e-30 * mx)) { e.status = DE_SINGULAR; return; }
        for (int i = j + 1; i < s; ++i) {
            dd v = Sh[i][j];
            for (int k = 0; k < j; ++k) v = v - e.L[i][k] * e.L[j][k] * e.Dg[k];
            e.L[i][j] = v / dj;
        }
    }
    e.B = dd_of(0.0);
    double dn = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        dd x[NF];
        for (int q = 0; q < s; ++q) x[q] = dd_of(-c.a[c.map[q]][i]);
        ldl_solve<D>(e, s, x);
        for (int q = 0; q < s; ++q) {
            e.w[i][q] = x[q];
            e.B = e.B + x[q] * (-c.a[c.map[q]][i]);
            dn += c.a[c.map[q]][i] * c.a[c.map[q]][i];
        }
    }
    if (c.K != p.k0) {
        double an = 0.0;   // crude scale of Shat^{-1}
        for (int q = 0; q < s; ++q) an = fmax(an, 1.0 / fabs(e.Dg[q].hi));
        if (!(fabs(e.B.hi) > 1e-30 * dn * an)) e.status = DE_BZERO;
    }
}

// --------------------------------------------------------------------------- NS path
template <int D>
struct NSElim {
    static constexpr int M = D * (D + 1);
    int m;
    int map[M];        // compact -> full local index l*D + i
    dd Ainv[M][M];
    dd w[M], v[M], B;
    dd R[M];           // compact R_K
    dd g;
    int status;
};

// Co-volume convection at the Newton iterate: residual r (all faces) and
// Jacobian J, and the increment-form RHS (reading 6):
//   A = I (x) S + J;  R = -[(I (x) S) U^k + r(U^k) + D P^k - R^f];  g = sum_all a . U^k
template <int D>
__device__ __forceinline__ void ns_local_system(const Cell<D> &c, const ProbView &p,
                                                dd A[D * (D + 1)][D * (D + 1)], dd R[D * (D + 1)], dd &g) {
    constexpr int NF = D + 1, N = NF * D;
    const int64_t K = c.K;
    double U[NF][D];
#pragma unroll
    for (int l = 0; l < NF; ++l)
#pragma unroll
        for (int i = 0; i < D; ++i) U[l][i] = p.uit[(K * NF + l) * D + i];
    dd S[NF][NF];
    for (int s = 0; s < NF; ++s)
        for (int t = 0; t < NF; ++t) S[s][t] = S_entry<D>(c, p.mu, p.nu, s, t);
    dd ubar[D];
    for (int i = 0; i < D; ++i) {
        dd acc = dd_of(0.0);
        for (int l = 0; l < NF; ++l) acc = acc + U[l][i];
        ubar[i] = acc / (double)NF;
    }
    dd F[NF][NF];
    dd nn[NF][NF][D];
    for (int s = 0; s < NF; ++s)
        for (int t = 0; t < NF; ++t) {
            dd f = dd_of(0.0);
            for (int i = 0; i < D; ++i) {
                nn[s][t][i] = two_sum(c.a[t][i], -c.a[s][i]) / (double)NF;
                f = f + (two_sum(U[s][i], U[t][i]) - ubar[i]) * nn[s][t][i];
            }
            F[s][t] = f;
        }
    for (int r = 0; r < N; ++r)
        for (int q = 0; q < N; ++q) A[r][q] = dd_of(0.0);
    for (int s = 0; s < NF; ++s)
        for (int t = 0; t < NF; ++t)
            for (int i = 0; i < D; ++i) A[s * D + i][t * D + i] = S[s][t];
    // Jacobian  dr_{s,i}/dU^j_t = 1/2 sum_{s' != s} [(d_ts + d_ts' - 1/(d+1)) n^j_{ss'} (U^i_s' - U^i_s)
    //                                                 + F_{ss'} d_ij (d_ts' - d_ts)]
    for (int s = 0; s < NF; ++s)
        for (int i = 0; i < D; ++i)
            for (int t = 0; t < NF; ++t)
                for (int j = 0; j < D; ++j) {
                    dd acc = dd_of(0.0);
                    for (int sp = 0; sp < NF; ++sp) {
                        if (sp == s) continue;
                        double coef = (t == s ? 1.0 : 0.0) + (t == sp ? 1.0 : 0.0);
                        dd cf = dd_of(coef) - dd_of(1.0) / (double)NF;
                        acc = acc + cf * nn[s][sp][j] * two_sum(U[sp][i], -U[s][i]);
                        if (i == j) {
                            double dl = (t == sp ? 1.0 : 0.0) - (t == s ? 1.0 : 0.0);
                            if (dl != 0.0) acc = acc + F[s][sp] * dl;
                        }
                    }
                    A[s * D + i][t * D + j] = A[s * D + i][t * D + j] + acc * 0.5;
                }
    // residual r_{s,i} = 1/2 sum_{t != s} F_st (U^i_t - U^i_s) and RHS
    g = dd_of(0.0);
    double pk = p.pit ? p.pit[K] : 0.0;
    for (int s = 0; s < NF; ++s) {
        dd fdx = dd_of(0.0);
        for (int i = 0; i < D; ++i) fdx = fdx + two_sum(c.xs[s][i], -c.xK[i]) * p.fbar[K * D + i];
        for (int i = 0; i < D; ++i) {
            dd rc = dd_of(0.0);
            for (int t = 0; t < NF; ++t)
                if (t != s) rc = rc + F[s][t] * two_sum(U[t][i], -U[s][i]);
            rc = rc * 0.5;
            dd su = dd_of(0.0);
            for (int t = 0; t < NF; ++t) su = su + S[s][t] * U[t][i];
            dd dp = two_prod(-c.a[s][i], pk);
            dd rf = fdx * c.a[s][i];
            R[s * D + i] = -(su + rc + dp - rf);
            g = g + two_prod(c.a[s][i], U[s][i]);
        }
    }
}

template <int D>
__device__ __noinline__ void ns_eliminate(const Cell<D> &c, const ProbView &p, NSElim<D> &e) {
    constexpr int NF = D + 1, N = NF * D;
    e.status = DE_OK;
    e.m = 0;
    for (int q = 0; q < c.s; ++q)
        for (int i = 0; i < D; ++i) e.map[e.m++] = c.map[q] * D + i;
    if (e.m == 0) { e.status = DE_NOINTERIOR; return; }
    dd A[N][N], Rf[N];
    ns_local_system<D>(c, p, A, Rf, e.g);
    const int m = e.m;
    dd W[N][N];
    double mx = 0.0;
    for (int r = 0; r < m; ++r) {
        for (int q = 0; q < m; ++q) {
            W[r][q] = A[e.map[r]][e.map[q]];
            e.Ainv[r][q] = dd_of(r == q ? 1.0 : 0.0);
        }
        if (p.E) W[r][r] = W[r][r] + p.E[c.K * NF + e.map[r] / D];
        for (int q = 0; q < m; ++q) mx = fmax(mx, fabs(W[r][q].hi));
        e.R[r] = Rf[e.map[r]];
    }
    // Gauss-Jordan with partial pivoting
    for (int k = 0; k < m; ++k) {
        int piv = k;
        for (int r = k + 1; r < m; ++r)
            if (fabs(W[r][k].hi) > fabs(W[piv][k].hi)) piv = r;
        if (!(fabs(W[piv][k].hi) > 1e-30 * mx)) { e.status = DE_SINGULAR; return; }
        if (piv != k)
            for (int q = 0; q < m; ++q) {
                dd t = W[k][q]; W[k][q] = W[piv][q]; W[piv][q] = t;
                t = e.Ainv[k][q]; e.Ainv[k][q] = e.Ainv[piv][q]; e.Ainv[piv][q] = t;
            }
        dd inv = dd_of(1.0) / W[k][k];
        for (int q = 0; q < m; ++q) { W[k][q] = W[k][q] * inv; e.Ainv[k][q] = e.Ainv[k][q] * inv; }
        for (int r = 0; r < m; ++r) {
            if (r == k) continue;
            dd f = W[r][k];
            if (f.hi == 0.0) continue;
            for (int q = 0; q < m; ++q) {
                W[r][q] = W[r][q] - f * W[k][q];
                e.Ainv[r][q] = e.Ainv[r][q] - f * e.Ainv[k][q];
            }
        }
    }
    e.B = dd_of(0.0);
    for (int r = 0; r < m; ++r) {
        dd sw = dd_of(0.0), sv = dd_of(0.0);
        for (int q = 0; q < m; ++q) {
            double Dq = -c.a[e.map[q] / D][e.map[q] % D];
            sw = sw + e.Ainv[r][q] * Dq;
            sv = sv + e.Ainv[q][r] * Dq;
        }
        e.w[r] = sw;
        e.v[r] = sv;
    }
    double dn = 0.0, an = 0.0;
    for (int r = 0; r < m; ++r) {
        double Dr = -c.a[e.map[r] / D][e.map[r] % D];
        e.B = e.B + e.w[r] * Dr;
        dn += Dr * Dr;
        for (int q = 0; q < m; ++q) an = fmax(an, fabs(e.Ainv[r][q].hi));
    }
    if (c.K != p.k0 && !(fabs(e.B.hi) > 1e-30 * dn * an)) e.status = DE_BZERO;
}

}  // namespace cr
