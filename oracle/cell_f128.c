/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * helper with the CUDA product path (paper_2101_03777_b200/csrc).
 *
 * Per-cell local algebra of the hybrid method, written out plainly in IEEE
 * binary128 (__float128, libquadmath) and rounded to fp64 only at the end.
 *
 * Why binary128: the transient local block S_K = mu|K|/(d+1) I + nu a a^t/|K|
 * has kappa(S_K) ~ nu (d+1)|a|^2/(mu |K|^2) ~ 1e8 at BASELINE configs[1];
 * a plain fp64 Gauss-Jordan would lose ~8 digits of G_K
 * and could not serve as the 1e-12 reference.  In binary128 the same textbook
 * elimination is exact to far below fp64 rounding.
 *
 * Citations are PAPER.md line numbers ("P:Lnnn").
 *
 * Local unknown ordering: (l, i) -> l*d + i, l = local face (the face opposite
 * local vertex l), i = velocity component.  All (d+1)*d local unknowns are
 * carried; rows/columns of boundary faces are zero in the outputs.
 */
#include <quadmath.h>
#include <stdint.h>
#include <string.h>
#include <math.h>

typedef __float128 Q;

#define MAXD 3
#define MAXF 4
#define MAXN 12

enum { OR_OK = 0, OR_SINGULAR = 1, OR_BZERO = 2, OR_NOINTERIOR = 3 };

typedef struct {
    int d;
    double mu, nu;
    int is_ns;
} cellparams;

/* raw per-cell inputs (fp64 pointers into the batch arrays) */
typedef struct {
    const double *a;     /* [(d+1)][d]  a_{K,sigma} = |sigma| n_{K,sigma} */
    double vol;          /* |K| */
    const double *xK;    /* [d]  centre of gravity */
    const double *xs;    /* [(d+1)][d] face centres of gravity */
    const int8_t *intr;  /* [(d+1)] 1 if the local face is interior */
    const double *fbar;  /* [d] (1/|K|) int_K f */
    const double *dir;   /* [(d+1)][d] Dirichlet values or NULL */
    const double *uit;   /* [(d+1)][d] Newton iterate U^k (NS) or NULL */
    double pit;          /* Newton pressure iterate P^k_K (NS) */
} cellin;

static Q qabs(Q x) { return x < 0 ? -x : x; }

/* ------------------------------------------------------------------ local blocks
 * S_K with the CR basis gradient grad phi_{sigma,K} = a_{K,sigma}/|K|
 * (from the defining mean-value conditions P:L129) and the lumped mass
 * int_K Pi_h phi_s Pi_h phi_s' = |K|/(d+1) delta:
 *     S[s][s'] = mu |K|/(d+1) delta_{ss'} + nu a_s . a_s' / |K|
 * over ALL d+1 local faces (boundary columns feed the Dirichlet fold).
 */
static void local_S(const cellparams *p, const cellin *c, Q S[MAXF][MAXF])
{
    int d = p->d, nf = d + 1;
    Q vol = (Q)c->vol;
    for (int s = 0; s < nf; ++s)
        for (int t = 0; t < nf; ++t) {
            Q dot = 0;
            for (int i = 0; i < d; ++i) dot += (Q)c->a[s * d + i] * (Q)c->a[t * d + i];
            S[s][t] = (Q)p->nu * dot / vol;
            if (s == t) S[s][t] += (Q)p->mu * vol / (Q)(d + 1);
        }
}

/* Co-volume convection, all d+1 faces:
 *   n_{ss'} = (a_{s'} - a_s)/(d+1)
 *   F_{ss'} = (U_s + U_s' - (1/(d+1)) sum_s'' U_s'') . n_{ss'}
 *   r_{s,i} = 1/2 sum_{s' != s} F_{ss'} (U^i_s' - U^i_s)             P:L196 (single-sum form)
 *   J[(s,i),(t,j)] = d r_{s,i} / d U^j_t  (exact derivative, product rule)
 */
static void local_convection(const cellparams *p, const cellin *c,
                             Q r[MAXN], Q J[MAXN][MAXN])
{
    int d = p->d, nf = d + 1, n = nf * d;
    Q U[MAXF][MAXD], nn[MAXF][MAXF][MAXD], F[MAXF][MAXF], ubar[MAXD];
    for (int s = 0; s < nf; ++s)
        for (int i = 0; i < d; ++i) U[s][i] = (Q)c->uit[s * d + i];
    for (int i = 0; i < d; ++i) {
        ubar[i] = 0;
        for (int s = 0; s < nf; ++s) ubar[i] += U[s][i];
        ubar[i] /= (Q)nf;
    }
    for (int s = 0; s < nf; ++s)
        for (int t = 0; t < nf; ++t) {
            F[s][t] = 0;
            for (int i = 0; i < d; ++i) {
                nn[s][t][i] = ((Q)c->a[t * d + i] - (Q)c->a[s * d + i]) / (Q)nf;
                F[s][t] += (U[s][i] + U[t][i] - ubar[i]) * nn[s][t][i];
            }
        }
    for (int s = 0; s < nf; ++s)
        for (int i = 0; i < d; ++i) {
            Q acc = 0;
            for (int t = 0; t < nf; ++t)
                if (t != s) acc += F[s][t] * (U[t][i] - U[s][i]);
            r[s * d + i] = acc / 2;
        }
    for (int row = 0; row < n; ++row)
        for (int col = 0; col < n; ++col) J[row][col] = 0;
    for (int s = 0; s < nf; ++s)
        for (int i = 0; i < d; ++i)
            for (int t = 0; t < nf; ++t)
                for (int j = 0; j < d; ++j) {
                    Q acc = 0;
                    for (int sp = 0; sp < nf; ++sp) {
                        if (sp == s) continue;
                        Q dF = ((t == s ? (Q)1 : (Q)0) + (t == sp ? (Q)1 : (Q)0) - (Q)1 / (Q)nf)
                               * nn[s][sp][j];
                        acc += dF * (U[sp][i] - U[s][i]);
                        if (i == j) acc += F[s][sp] * ((t == sp ? (Q)1 : (Q)0) - (t == s ? (Q)1 : (Q)0));
                    }
                    J[s * d + i][t * d + j] = acc / 2;
                }
}

/* Full (all faces) A_K, R_K restricted to interior rows, g_K, D_K.
 *   A_K[(s,i),(t,j)] = delta_ij S[s][t]  (+ J for NS)
 *   D_K[(s,i)] = -a^{(i)}_s
 *   R_K[(s,i)] = a^{(i)}_s (fbar . (x_s - x_K))
 * Stokes, Dirichlet fold (the paper assumes homogeneous BC; reading in
 * DESIGN.md): R_{K,I} -= A_{K,IE} U^D_E ;  g_K = + sum_{ext s} a_s . U^D_s.
 * NS step, increment form (reading in DESIGN.md):
 *   R_K = -[ (I (x) S) U^k + r(U^k) + D_K P^k - R^f ]  on interior rows,
 *   g_K = sum_{all s} a_s . U^k_s.
 */
static void local_system(const cellparams *p, const cellin *c,
                         Q A[MAXN][MAXN], Q R[MAXN], Q D[MAXN], Q *g)
{
    int d = p->d, nf = d + 1, n = nf * d;
    Q S[MAXF][MAXF];
    local_S(p, c, S);
    for (int r = 0; r < n; ++r)
        for (int cc = 0; cc < n; ++cc) A[r][cc] = 0;
    for (int s = 0; s < nf; ++s)
        for (int t = 0; t < nf; ++t)
            for (int i = 0; i < d; ++i) A[s * d + i][t * d + i] = S[s][t];
    Q rconv[MAXN];
    if (p->is_ns) {
        Q J[MAXN][MAXN];
        local_convection(p, c, rconv, J);
        for (int r = 0; r < n; ++r)
            for (int cc = 0; cc < n; ++cc) A[r][cc] += J[r][cc];
    }
    for (int s = 0; s < nf; ++s) {
        Q fdx = 0;
        for (int i = 0; i < d; ++i) fdx += (Q)c->fbar[i] * ((Q)c->xs[s * d + i] - (Q)c->xK[i]);
        for (int i = 0; i < d; ++i) {
            D[s * d + i] = -(Q)c->a[s * d + i];
            R[s * d + i] = (Q)c->a[s * d + i] * fdx;
        }
    }
    *g = 0;
    if (p->is_ns) {
        for (int s = 0; s < nf; ++s)
            for (int i = 0; i < d; ++i) {
                Q su = 0;
                for (int t = 0; t < nf; ++t) su += S[s][t] * (Q)c->uit[t * d + i];
                R[s * d + i] = -(su + rconv[s * d + i] + D[s * d + i] * (Q)c->pit - R[s * d + i]);
                *g += (Q)c->a[s * d + i] * (Q)c->uit[s * d + i];
            }
    } else if (c->dir) {
        for (int t = 0; t < nf; ++t) {
            if (c->intr[t]) continue;
            for (int j = 0; j < d; ++j) {
                Q ud = (Q)c->dir[t * d + j];
                for (int r = 0; r < n; ++r) R[r] -= A[r][t * d + j] * ud;
                *g += (Q)c->a[t * d + j] * ud;
            }
        }
    }
    /* restrict to interior rows/columns: zero the boundary ones */
    for (int s = 0; s < nf; ++s) {
        if (c->intr[s]) continue;
        for (int i = 0; i < d; ++i) {
            int r = s * d + i;
            R[r] = 0; D[r] = 0;
            for (int cc = 0; cc < n; ++cc) { A[r][cc] = 0; A[cc][r] = 0; }
        }
    }
}

/* Gauss-Jordan with partial pivoting, M (m x m, compact) -> Minv.  Returns 0 or
 * OR_SINGULAR when a pivot falls below 1e-30 * max|M|. */
static int gauss_jordan(int m, Q M[MAXN][MAXN], Q Minv[MAXN][MAXN])
{
    Q W[MAXN][2 * MAXN];
    Q mx = 0;
    for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) {
            W[r][c] = M[r][c];
            W[r][m + c] = (r == c) ? 1 : 0;
            if (qabs(M[r][c]) > mx) mx = qabs(M[r][c]);
        }
    for (int k = 0; k < m; ++k) {
        int piv = k;
        for (int r = k + 1; r < m; ++r)
            if (qabs(W[r][k]) > qabs(W[piv][k])) piv = r;
        if (!(qabs(W[piv][k]) > (Q)1e-30 * mx)) return OR_SINGULAR;
        if (piv != k)
            for (int c = 0; c < 2 * m; ++c) { Q t = W[k][c]; W[k][c] = W[piv][c]; W[piv][c] = t; }
        Q inv = (Q)1 / W[k][k];
        for (int c = 0; c < 2 * m; ++c) W[k][c] *= inv;
        for (int r = 0; r < m; ++r) {
            if (r == k) continue;
            Q f = W[r][k];
            if (f == 0) continue;
            for (int c = 0; c < 2 * m; ++c) W[r][c] -= f * W[k][c];
        }
    }
    for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) Minv[r][c] = W[r][m + c];
    return OR_OK;
}

static void load_cell(int d, int64_t k, const double *a, const double *vol, const double *xK,
                      const double *xs, const int8_t *intr, const double *fbar,
                      const double *dir, const double *uit, const double *pit, cellin *c)
{
    int nf = d + 1;
    c->a = a + k * nf * d;
    c->vol = vol[k];
    c->xK = xK + k * d;
    c->xs = xs + k * nf * d;
    c->intr = intr + k * nf;
    c->fbar = fbar + k * d;
    c->dir = dir ? dir + k * nf * d : NULL;
    c->uit = uit ? uit + k * nf * d : NULL;
    c->pit = pit ? pit[k] : 0.0;
}

/* Exported: per-cell A_K, R_K, D_K, g_K (rounded to fp64), interior-restricted. */
int or_cell_blocks(int d, int64_t nc, double mu, double nu, int is_ns,
                   const double *a, const double *vol, const double *xK, const double *xs,
                   const int8_t *intr, const double *fbar, const double *dir,
                   const double *uit, const double *pit,
                   double *A_out, double *R_out, double *D_out, double *g_out)
{
    cellparams p = { d, mu, nu, is_ns };
    int n = (d + 1) * d;
    for (int64_t k = 0; k < nc; ++k) {
        cellin c;
        load_cell(d, k, a, vol, xK, xs, intr, fbar, dir, uit, pit, &c);
        Q A[MAXN][MAXN], R[MAXN], D[MAXN], g;
        local_system(&p, &c, A, R, D, &g);
        for (int r = 0; r < n; ++r) {
            R_out[k * n + r] = (double)R[r];
            D_out[k * n + r] = (double)D[r];
            for (int cc = 0; cc < n; ++cc) A_out[k * n * n + r * n + cc] = (double)A[r][cc];
        }
        g_out[k] = (double)g;
    }
    return 0;
}

/* Exported: full convection residual and Jacobian over all d+1 faces (test hook). */
int or_cell_convection(int d, int64_t nc, const double *a, const double *uit,
                       double *r_out, double *J_out)
{
    cellparams p = { d, 0.0, 0.0, 1 };
    int n = (d + 1) * d;
    for (int64_t k = 0; k < nc; ++k) {
        cellin c;
        memset(&c, 0, sizeof c);
        c.a = a + k * n;
        c.uit = uit + k * n;
        Q r[MAXN], J[MAXN][MAXN];
        local_convection(&p, &c, r, J);
        for (int i = 0; i < n; ++i) {
            r_out[k * n + i] = (double)r[i];
            for (int j = 0; j < n; ++j) J_out[k * n * n + i * n + j] = (double)J[i][j];
        }
    }
    return 0;
}

/* Local elimination of one cell, compact interior indexing.
 *   Ahat_K = A_K + E_K
 *   w = Ahat^{-1} D ; v = Ahat^{-t} D ; B_K = D^t Ahat^{-1} D
 *   G_K  = C (Ahat^{-1} - w v^t / B_K) C        (K != K0)
 *   G_K0 = C Ahat^{-1} C
 *   S_K  = C (Ahat^{-1} R - w (v^t R - g)/B_K)  (K != K0)          P:L498 (+ g)
 *   S_K0 = C Ahat^{-1} R
 * Also returns what recovery needs: Ahat^{-1}, v, B.
 */
typedef struct {
    int m;                 /* compact size d * s_K */
    int map[MAXN];         /* compact -> full local index */
    Q Ainv[MAXN][MAXN];
    Q w[MAXN], v[MAXN], B;
    Q R[MAXN], D[MAXN], g;
    Q C[MAXN];
} elim;

static int eliminate(const cellparams *p, const cellin *c, const double *E, const int8_t *cs,
                     int is_k0, elim *e)
{
    int d = p->d, nf = d + 1, n = nf * d;
    Q A[MAXN][MAXN], R[MAXN], D[MAXN], g;
    local_system(p, c, A, R, D, &g);
    e->m = 0;
    for (int s = 0; s < nf; ++s)
        if (c->intr[s])
            for (int i = 0; i < d; ++i) e->map[e->m++] = s * d + i;
    (void)n;
    if (e->m == 0) return OR_NOINTERIOR;
    Q Ah[MAXN][MAXN];
    for (int r = 0; r < e->m; ++r) {
        int fr = e->map[r];
        for (int cc = 0; cc < e->m; ++cc) Ah[r][cc] = A[fr][e->map[cc]];
        Ah[r][r] += (Q)E[fr / d];            /* E_K diagonal, same for every component */
        e->R[r] = R[fr];
        e->D[r] = D[fr];
        e->C[r] = (Q)cs[fr / d];
    }
    e->g = g;
    int st = gauss_jordan(e->m, Ah, e->Ainv);
    if (st) return st;
    e->B = 0;
    for (int r = 0; r < e->m; ++r) {
        Q sw = 0, sv = 0;
        for (int cc = 0; cc < e->m; ++cc) {
            sw += e->Ainv[r][cc] * e->D[cc];
            sv += e->Ainv[cc][r] * e->D[cc];
        }
        e->w[r] = sw;
        e->v[r] = sv;
    }
    for (int r = 0; r < e->m; ++r) e->B += e->D[r] * e->w[r];
    if (!is_k0) {
        Q dn = 0, an = 0;
        for (int r = 0; r < e->m; ++r) dn += e->D[r] * e->D[r];
        for (int r = 0; r < e->m; ++r)
            for (int cc = 0; cc < e->m; ++cc)
                if (qabs(e->Ainv[r][cc]) > an) an = qabs(e->Ainv[r][cc]);
        if (!(qabs(e->B) > (Q)1e-30 * dn * an)) return OR_BZERO;
    }
    return OR_OK;
}

int or_cell_eliminate(int d, int64_t nc, double mu, double nu, int is_ns,
                      const double *a, const double *vol, const double *xK, const double *xs,
                      const int8_t *intr, const double *fbar, const double *dir,
                      const double *uit, const double *pit,
                      const double *E, const int8_t *csign, int64_t k0,
                      double *G_out, double *S_out, double *B_out, int32_t *status)
{
    cellparams p = { d, mu, nu, is_ns };
    int nf = d + 1, n = nf * d;
    int nbad = 0;
    for (int64_t k = 0; k < nc; ++k) {
        cellin c;
        load_cell(d, k, a, vol, xK, xs, intr, fbar, dir, uit, pit, &c);
        double *G = G_out + k * n * n, *S = S_out + k * n;
        for (int i = 0; i < n * n; ++i) G[i] = 0.0;
        for (int i = 0; i < n; ++i) S[i] = 0.0;
        elim e;
        int is_k0 = (k == k0);
        int st = eliminate(&p, &c, E + k * nf, csign + k * nf, is_k0, &e);
        status[k] = st;
        B_out[k] = 0.0;
        if (st) { ++nbad; continue; }
        B_out[k] = (double)e.B;
        Q vR = 0;
        for (int r = 0; r < e.m; ++r) vR += e.v[r] * e.R[r];
        for (int r = 0; r < e.m; ++r) {
            Q AR = 0;
            for (int cc = 0; cc < e.m; ++cc) {
                Q val = e.Ainv[r][cc];
                if (!is_k0) val -= e.w[r] * e.v[cc] / e.B;
                G[e.map[r] * n + e.map[cc]] = (double)(e.C[r] * val * e.C[cc]);
                AR += e.Ainv[r][cc] * e.R[cc];
            }
            Q sv = AR;
            if (!is_k0) sv -= e.w[r] * (vR - e.g) / e.B;
            S[e.map[r]] = (double)(e.C[r] * sv);
        }
    }
    return nbad;
}

/* Recovery:
 *   P_K = (v^t (R_K - C_K W_K) - g_K) / B_K   (K != K0),  P_K0 = 0
 *   Uhat_K = Ahat_K^{-1} (R_K - D_K P_K - C_K W_K)
 * W_loc[k][(l,i)] = W at local face l (zero on boundary faces).
 */
int or_cell_recover(int d, int64_t nc, double mu, double nu, int is_ns,
                    const double *a, const double *vol, const double *xK, const double *xs,
                    const int8_t *intr, const double *fbar, const double *dir,
                    const double *uit, const double *pit,
                    const double *E, const int8_t *csign, int64_t k0,
                    const double *W_loc, double *P_out, double *U_out, int32_t *status)
{
    cellparams p = { d, mu, nu, is_ns };
    int nf = d + 1, n = nf * d;
    int nbad = 0;
    for (int64_t k = 0; k < nc; ++k) {
        cellin c;
        load_cell(d, k, a, vol, xK, xs, intr, fbar, dir, uit, pit, &c);
        double *U = U_out + k * n;
        for (int i = 0; i < n; ++i) U[i] = 0.0;
        elim e;
        int is_k0 = (k == k0);
        int st = eliminate(&p, &c, E + k * nf, csign + k * nf, is_k0, &e);
        status[k] = st;
        P_out[k] = 0.0;
        if (st) { ++nbad; continue; }
        Q rhs[MAXN];
        for (int r = 0; r < e.m; ++r) rhs[r] = e.R[r] - e.C[r] * (Q)W_loc[k * n + e.map[r]];
        Q P = 0;
        if (!is_k0) {
            Q vr = 0;
            for (int r = 0; r < e.m; ++r) vr += e.v[r] * rhs[r];
            P = (vr - e.g) / e.B;
        }
        P_out[k] = (double)P;
        for (int r = 0; r < e.m; ++r) {
            Q acc = 0;
            for (int cc = 0; cc < e.m; ++cc) acc += e.Ainv[r][cc] * (rhs[cc] - e.D[cc] * P);
            U[e.map[r]] = (double)acc;
        }
    }
    return nbad;
}

/* r = b - A x with every product and sum in binary128, rounded once (used for
 * iterative refinement of the direct and Krylov reference solves). */
int or_residual_f128(int64_t nrows, const int64_t *rowptr, const int32_t *cols,
                     const double *vals, const double *x, const double *b, double *r)
{
    for (int64_t i = 0; i < nrows; ++i) {
        Q acc = (Q)b[i];
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            acc -= (Q)vals[k] * (Q)x[cols[k]];
        r[i] = (double)acc;
    }
    return 0;
}

/* Exact-ish dot/norm helper: sum_i x_i y_i in binary128. */
double or_dot_f128(int64_t n, const double *x, const double *y)
{
    Q acc = 0;
    for (int64_t i = 0; i < n; ++i) acc += (Q)x[i] * (Q)y[i];
    return (double)acc;
}
