/*
 * cr.h — C ABI of libcr, the B200 (sm_100a) implementation of the hybrid method of
 * Chenier & Eymard, "Exact pressure elimination for the Crouzeix-Raviart scheme
 * applied to the Stokes and Navier-Stokes problems" (arXiv 2101.03777).
 * Citations "P:Lnnn" are lines of /root/reference/PAPER.md.
 *
 * Pipeline (the paper's "hybrid method"):
 *   cr_build_mesh    faces, M_sigma, F_K, x_K, x_sigma, |K|, a_{K,sigma}
 *   cr_hybridise     G = sum_K H_K G_K H_K^t and S of  G W = S
 *   cr_solve         Krylov solve of G W = S (PCG / MINRES / BiCGStab / GMRES)
 *   cr_recover       P and U from W, per cell
 *   cr_assemble_coupled  the coupled saddle system eq. (syslin)
 *
 * Conventions (all calls):
 *   - Pointers suffixed _d are DEVICE pointers on the current CUDA device.  Input
 *     pointers are borrowed for the duration of the (stream-ordered) call; output
 *     buffers are caller-owned and must be sized from cr_mesh_info / *_info.
 *   - All work is enqueued on stream `s` (cudaStream_t; NULL = legacy default stream).
 *     Calls that must return host-visible counts or convergence data synchronise `s`
 *     (documented per call); the others are asynchronous.
 *   - Errors: every call returns a cr_status; no C++ exception crosses the ABI.
 *     cr_last_error() returns a thread-local message for the last non-OK status.
 *   - Local face s of a cell is the face OPPOSITE its local vertex s.  Faces are
 *     numbered in lexicographic order of their sorted vertex tuple; face_cells[f] =
 *     (lower cell, higher cell), -1 in the second slot for a boundary face; interior
 *     faces get dof = rank among interior faces.  Velocity / auxiliary unknowns are
 *     indexed d*dof + i (face-major, component-minor).
 *   - C_K = +1 on face_cells[f][0], -1 on the other cell ("equal to +-1").
 *   - Gauge cell K0: P_{K0} = 0.
 *   - fp64 throughout.  Per-cell eliminations are carried out in double-double
 *     arithmetic and rounded once (kappa(S_K) reaches ~1e8 at 2D n = 1024).
 */
#ifndef CR_H
#define CR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *cr_stream_t; /* == cudaStream_t */

typedef enum {
    CR_OK = 0,
    CR_ERR_INVALID_ARG = -1,      /* bad pointer / size / dimension / option            */
    CR_ERR_CUDA = -2,             /* CUDA runtime error (message in cr_last_error)      */
    CR_ERR_OOM = -3,              /* device allocation failed                           */
    CR_ERR_NONMANIFOLD = -4,      /* a face shared by > 2 cells (1 or 2)        */
    CR_ERR_DEGENERATE_CELL = -5,  /* |K| <= 1e-14 (max edge)^d, or vertex out of range  */
    CR_ERR_NO_INTERIOR_FACE = -6, /* s_K = 0 => D_K = 0, B_K = 0 (P:L486 assumes s_K>0) */
    CR_ERR_SINGULAR_LOCAL = -7,   /* Ahat_K singular or |B_K| ~ 0        */
    CR_ERR_NOT_CONVERGED = -8,    /* max_iter reached                                   */
    CR_ERR_BREAKDOWN = -9,        /* CG p^t G p <= 0, BiCGStab rho or omega = 0         */
    CR_ERR_STAGNATION = -10,      /* GMRES(m) restart cycle made no progress            */
    CR_ERR_NCCL = -11             /* NCCL error                                         */
} cr_status;

typedef struct cr_mesh_s *cr_mesh;
typedef struct cr_coupled_s *cr_coupled;
typedef struct cr_hybrid_s *cr_hybrid;
typedef struct cr_comm_s *cr_comm;
typedef struct cr_loopback_s *cr_loopback;

/* ------------------------------------------------------------------ mesh
 * coords_d [nv][dim] f64, cells_d [nc][dim+1] i32 (0-based vertex ids, any orientation).
 * Builds faces and incidence with a device radix sort of the (dim+1)*nc face tuples,
 * then |K|, x_K, x_sigma and the outward area vectors a_{K,sigma} = |sigma| n_{K,sigma}.
 * Synchronises `s` (counts are returned to the host).  Errors: INVALID_ARG (dim not 2/3,
 * nv or nc <= 0, nc*(dim+1) >= 2^31), DEGENERATE_CELL, NONMANIFOLD, OOM, CUDA.          */
cr_status cr_build_mesh(int32_t dim, int64_t nv, const double *coords_d, int64_t nc,
                        const int32_t *cells_d, cr_stream_t s, cr_mesh *out);

typedef struct {
    int32_t dim;
    int64_t nv, nc, nf, nf_int;
    int64_t n_unknowns;          /* dim * nf_int = size of G, U, W, S                      */
} cr_mesh_info_t;
cr_status cr_mesh_info(cr_mesh m, cr_mesh_info_t *out);

/* Copies the mesh arrays (any pointer may be NULL):
 *   faces_d [nf][dim] i32 sorted vertex tuples (lexicographic face order)
 *   face_cells_d [nf][2] i32, cell_faces_d [nc][dim+1] i32, face_dof_d [nf] i32 (-1 boundary)
 *   vol_d [nc], xK_d [nc][dim], xs_d [nf][dim], a_d [nc][dim+1][dim] f64. Asynchronous. */
cr_status cr_mesh_export(cr_mesh m, int32_t *faces_d, int32_t *face_cells_d, int32_t *cell_faces_d,
                         int32_t *face_dof_d, double *vol_d, double *xK_d, double *xs_d, double *a_d,
                         cr_stream_t s);
void cr_destroy_mesh(cr_mesh m);

/* ------------------------------------------------------------------ problem data */
enum { CR_STOKES = 0, CR_NS_NEWTON_STEP = 1 };  /* b_h = 0 / one Newton step */
enum { CR_SHIFT_NONE = 0, CR_SHIFT_MIS = 1 };   /* E_K = 0 (mu > 0) / M1-M2 shift */

typedef struct {
    double mu;             /* 1/dt (transient) or 0 (steady)                        */
    double nu;             /* 1/Re                                                  */
    int32_t gauge_cell;    /* K0, P:L177 (default 0)                                       */
    int32_t physics;       /* CR_STOKES | CR_NS_NEWTON_STEP                                */
    int32_t shift;         /* CR_SHIFT_NONE | CR_SHIFT_MIS                                 */
    int32_t reserved;
    uint64_t mis_seed;     /* M1 = greedy MIS in ascending (splitmix64(seed ^ K), K) order */
    double lambda_factor;  /* lambda_K = factor * Gershgorin bound of A_K (> all eigenvalues) */
} cr_params;

typedef struct {
    const double *fbar_d;      /* [nc][dim] (1/|K|) int_K f                        */
    const double *dirichlet_d; /* [nc][dim+1][dim] values at the centroid of each LOCAL face;
                                  read on boundary faces only; NULL = homogeneous    */
    const double *u_iter_d;    /* NS: [nc][dim+1][dim] Newton iterate U^k at every local face
                                  (boundary faces carry the wall values); the two copies of an
                                  interior face must agree                                   */
    const double *p_iter_d;    /* NS: [nc] pressure iterate P^k, NULL = 0                     */
} cr_data;

/* ------------------------------------------------------------------ coupled system
 * Assembles A = sum_K H_K A_K H_K^t, D = sum_{K != K0} F_K D_K^t H_K^t, R and g on the device.
 * Synchronises `s` (nnz).  Used for parity / export; the hybrid path never needs it.   */
cr_status cr_assemble_coupled(cr_mesh m, const cr_params *prm, const cr_data *data, cr_stream_t s,
                              cr_coupled *out);
/* saddle matrix [[A, D^t],[D, 0]] of size n_rows = dim*nf_int + nc - 1 (pressures of K != K0 in
 * increasing K), canonical CSR: int64 row_ptr_d [n_rows+1], cols sorted, f64 vals; rhs [R; g]. */
cr_status cr_coupled_info(cr_coupled c, int64_t *n_rows, int64_t *nnz);
cr_status cr_coupled_export_csr(cr_coupled c, int64_t *row_ptr_d, int32_t *cols_d, double *vals_d,
                                double *rhs_d, cr_stream_t s);
void cr_destroy_coupled(cr_coupled c);

/* ------------------------------------------------------------------ hybridisation
 * Per interior face (block row of G), for each of its two cells: Ahat_K = A_K + E_K,
 * Ahat_K^{-1}, w = Ahat^{-1} D_K, B_K = D_K^t w, G_K and S_K in double-double,
 * written straight into a sliced block-ELL G (d x d blocks, width 2d+1) — no atomics, no
 * staging.  shift = MIS runs the M1/M2 construction first (hashed-priority Luby rounds that
 * reproduce the sequential greedy MIS exactly).  `comm`: NULL (or a single-rank communicator
 * without an id) = the whole G on this GPU; a multi-rank communicator = this rank's block rows
 * only (see "multi-GPU" below; the communicator must outlive the handle).
 * Synchronises `s`.  Errors: NO_INTERIOR_FACE, SINGULAR_LOCAL, INVALID_ARG, OOM, CUDA.   */
cr_status cr_hybridise(cr_mesh m, const cr_params *prm, const cr_data *data, cr_comm comm,
                       cr_stream_t s, cr_hybrid *out);
/* n_rows = dim*nf_int (partitioned: dim * owned rows); nnz = scalar nonzeros of G (explicit
 * zeros of the stencil included; partitioned: of the owned rows)                            */
cr_status cr_hybrid_info(cr_hybrid h, int64_t *n_rows, int64_t *nnz, int64_t *nblocks);
/* canonical scalar CSR of G (int64 row_ptr_d [n_rows+1], cols ascending) and S_d [n_rows];
 * partitioned: the owned rows, with GLOBAL column indices                                   */
cr_status cr_hybrid_export_csr(cr_hybrid h, int64_t *row_ptr_d, int32_t *cols_d, double *vals_d,
                               double *S_d, cr_stream_t s);
/* MIS membership inM1_d [nc] (u8) and E_d [nc][dim+1] (shift per local face); either may be NULL */
cr_status cr_hybrid_export_shift(cr_hybrid h, uint8_t *inM1_d, double *E_d, cr_stream_t s);
/* y = G x (the solver's SpMV kernel; x_d, y_d [n_rows], must not alias).  Asynchronous. */
cr_status cr_spmv(cr_hybrid h, const double *x_d, double *y_d, cr_stream_t s);
/* y = G x with the matrix-free factored operator (built on first use; transient Stokes,
 * unpartitioned handles): G = sum_K H_K C_K[I (x) Shat_K^{-1} - u_K u_K^t]C_K H_K^t, u = w/sqrt(B)
 * (P:L508-517); x_d, y_d [n_rows], must not alias.  Asynchronous after the first build.    */
cr_status cr_spmv_mf(cr_hybrid h, const double *x_d, double *y_d, cr_stream_t s);
/* ------------------------------------------------------------------ time stepping
 * Backward Euler for transient Stokes keeps G (and its preconditioners) from step to step:
 * only S changes ("all the linear systems have the same matrix").
 * cr_transient_rhs: per-cell right-hand sides of the step U^n -> U^{n+1}:
 *   R_K(l) = data terms of the handle (force P:L298-301, Dirichlet fold)
 *            + mu |K|/(d+1) U^n_{sigma(l)}   (lumped mass; interior faces)
 *   g_K    = data term.
 *   U_prev_d [nf_int][dim] (global numbering), R_d [nc][dim+1][dim], g_d [nc].  Asynchronous.
 * cr_hybrid_set_cell_rhs: replace the handle's right-hand side by explicit R_K, g_K (any split
 *   with sum_K H_K R_K = the momentum right-hand side is admissible) and recompute S
 *   with the same G; R_d = g_d = NULL restores the data-derived S.  Transient / steady Stokes
 *   handles (not NS).  Asynchronous.                                                          */
cr_status cr_transient_rhs(cr_hybrid h, const double *U_prev_d, double *R_d, double *g_d, cr_stream_t s);
cr_status cr_hybrid_set_cell_rhs(cr_hybrid h, const double *R_d, const double *g_d, cr_stream_t s);

/* two-level coarse space of the handle (0 if not built): intervals H, coarse unknowns nE, nd = 1
 * for the nested-dissection solve (0: dense E^{-1}), bytes one coarse solve reads (E^{-1} or the
 * fronts' Finv + 2 W).  Any pointer may be NULL.                                              */
cr_status cr_hybrid_coarse_info(cr_hybrid h, int32_t *H, int64_t *nE, int32_t *nd, int64_t *solve_bytes);

/* matrix-free operator statistics (0 if not built): cells (padded to 32) and device bytes     */
cr_status cr_hybrid_mf_info(cr_hybrid h, int64_t *ncells, int64_t *bytes);
void cr_destroy_hybrid(cr_hybrid h);

/* ------------------------------------------------------------------ solve
 * Solves G W = S.  W_d [n_rows] holds the initial guess on entry (use zeros) and the solution
 * on exit.  Stopping rule: TRUE relative residual ||S - G W||_2 / ||S||_2 <= rtol (recomputed
 * at exit; recursive-residual convergence triggers a true-residual check and, if it fails, a
 * residual replacement).  matrix_free = 1 applies G as sum_K H_K G_K H_K^t from per-cell factors
 * (Shat_K^{-1}, w_K / sqrt(B_K)) instead of the assembled block-ELL (transient Stokes
 * PCG methods only; the residual is then that of the factored operator).  Synchronises `s`.  */
enum { CR_PCG_JACOBI = 0, CR_PCG_BLOCKJACOBI = 1, CR_MINRES_ABSJACOBI = 2,
       CR_BICGSTAB_JACOBI = 3, CR_GMRES_JACOBI = 4,
       /* overlapping-patch additive Schwarz M^{-1} = sum_p R_p^t (R_p G R_p^t)^{-1} R_p, one
        * block per velocity component, patches = interior faces around a vertex (2D) / an
        * edge (3D); built on the device at the first solve that needs it (DESIGN.md
        * "Preconditioners").  PCG: Cholesky of each patch block (G SPD);
        * MINRES: |patch block|^{-1} (SPD although G is indefinite).                */
       CR_PCG_AFW = 5, CR_MINRES_AFW = 6,
       /* two-level: the patch preconditioner plus the coarse correction Z (Z^t G Z)^{-1} Z^t,
        * Z_(j,k,l): W^(k) = a_sigma^(l) phi_j(x_sigma) on a uniform grid of `coarse` intervals
        * per direction; E = Z^t G Z assembled and inverted on the device.   */
       CR_PCG_AFW2 = 7,
       /* steady Stokes / NS step: flexible GMRES(restart) on the coupled system [[A, D^t],[D, 0]]
        * (P:L253-306), right-preconditioned by the exact transient-Stokes inverse K_mu^{-1}
        * (mass coefficient mu_inner, same nu and K0), applied through the hybrid method: cell
        * right-hand sides -> S_mu -> CR_PCG_AFW2 on the matrix-free G_mu (to inner_rtol) ->
        * recovery.  The W returned is the target's, formed from (U, P) by the local relation
        * W_sigma = R_K - Ahat_K U_K + a_K P_K on the first cell of sigma; the stopping rule is
        * the target's true ||S - G W|| / ||S|| <= rtol (assembled G).  iterations = outer
        * iterations; inner_iterations = total inner PCG iterations; max_iter caps the outer
        * ones (default 500); the initial W is ignored (x0 = 0).  Single rank.  DESIGN.md §7.1. */
       CR_DC_FGMRES = 8,
       /* MINRES preconditioned by |patch| + a coarse |E|^{-1} (E = Z^t G Z of the shifted, indefinite
        * G; |E|^{-1} = V |Lambda|^{-1} V^t by a dense symmetric eigendecomposition, so the coarse grid
        * is capped at ~8,000 coarse unknowns: H <= 43 in 2D, 8 in 3D): the SPD two-level
        * preconditioner MINRES needs for steady Stokes (round-2 measurement). */
       CR_MINRES_AFW2 = 9 };
typedef struct {
    int32_t method;       /* CR_* above                                                        */
    int32_t restart;      /* GMRES m (default 50)                                              */
    double rtol;          /* default 1e-10                                                     */
    int64_t max_iter;     /* total Krylov iterations cap                                       */
    int32_t check_every;  /* iterations per captured CUDA graph between host checks (def 64)   */
    int32_t matrix_free;  /* 0: assembled G; 1: matrix-free factored G (see above)             */
    int32_t coarse;       /* CR_PCG_AFW2: coarse intervals per direction (0: 64 in 2D, 16 in 3D; <= 256);
                           * E^{-1} dense up to 8000 unknowns, else nested-dissection fronts  */
    double mu_inner;      /* CR_DC_FGMRES: mass coefficient of the inner transient operator (0: 1) */
    double inner_rtol;    /* CR_DC_FGMRES: inner PCG tolerance (0: 1e-11)                       */
    int32_t refine_dd;    /* 1: parity mode (PCG methods, one GPU): after the fp64 solve, iterative
                           * refinement W += G^{-1}(S - G W) with the residual S - G W evaluated in
                           * double-double (the operator the solve used: assembled G, or the
                           * factored G_K of every cell, summed in dd) until that residual is
                           * <= rtol (at most 8 rounds; rel_res_true is then the dd residual).
                           * Reaches below the fp64 residual floor of the recursive iteration. */
    int32_t reserved;
} cr_solver_opts;
typedef struct {
    int64_t iterations;
    double rel_res_true;       /* ||S - G W|| / ||S|| at exit (fp64 SpMV)                       */
    double rel_res_recursive;  /* solver's own residual estimate at exit                        */
    int32_t converged;
    int32_t status;            /* cr_status of the solve                                        */
    double seconds;            /* device time of the solve (CUDA events)                        */
    int64_t spmv_calls;
    int64_t kernel_launches;   /* kernels launched by cr_solve                                   */
    int64_t inner_iterations;  /* CR_DC_FGMRES: inner PCG iterations over all outer ones;
                                  refine_dd: PCG iterations of the refinement rounds             */
    double kappa_lanczos_est;  /* PCG methods: lambda_max / lambda_min of the preconditioned G,
                                  estimated from the Lanczos tridiagonal of the first <= 1024 CG
                                  coefficients (alpha_k, beta_k); 0 for other methods            */
    double lambda_min_est, lambda_max_est;
    double bytes_moved;        /* algorithmic HBM bytes of the iterations (per-iteration bytes of
                                  the method's kernels x iterations)               */
    int32_t refine_rounds;     /* refine_dd: refinement rounds run                               */
    int32_t reserved;
    double setup_seconds;      /* part of `seconds` spent building the preconditioner (patch blocks,
                                  coarse space E = Z^t G Z and its factorisation) before the first
                                  iteration; seconds - setup_seconds = the iterations             */
} cr_solve_report;
cr_status cr_solve(cr_hybrid h, const cr_solver_opts *opts, double *W_d, cr_stream_t s,
                   cr_solve_report *rep);

/* Device time of each kernel group of the patch-preconditioned PCG iteration (opts->method =
 * CR_PCG_AFW2 or CR_PCG_AFW, matrix_free = 1, one GPU), launched on the handle's own solver buffers
 * exactly as cr_solve launches them (same row order, grids and streams' kernels), each group timed
 * alone with CUDA events on s over nrep launches (the solver state is reset before each launch, the
 * numbers computed are discarded).  Requires a preceding cr_solve of `h` with the same options (its
 * preconditioner, coarse space and work vectors are reused; a later cr_solve is unaffected).
 * ms[5] (host, caller-owned): mean ms per launch of 0 G p with p.q (k_mf_spmv), 1 r update,
 * 2 coarse restriction + gather + coarse solve (0 for CR_PCG_AFW), 3 patch solves,
 * 4 direction + solution update.  Synchronises s.  (bench.py's rooflines.)          */
cr_status cr_solve_profile(cr_hybrid h, const cr_solver_opts *opts, int32_t nrep, double *ms, cr_stream_t s);

/* z_d = M^{-1} r_d for the preconditioner that `method` (CR_* above) uses: diag(G)^{-1},
 * |diag(G)|^{-1}, inverse diagonal blocks, or the patch additive Schwarz operator (built on
 * first use).  r_d, z_d [n_rows], must not alias.  Asynchronous except for a first patch
 * build (which synchronises `s`).                                                          */
cr_status cr_apply_precond(cr_hybrid h, int32_t method, const double *r_d, double *z_d, cr_stream_t s);
/* patch preconditioner statistics (0 if not built): number of patches, largest patch, patch
 * blocks that were singular and fell back to their diagonal, device bytes of the operator
 * (what one application reads besides the vectors).  Any pointer may be NULL.               */
cr_status cr_hybrid_precond_info(cr_hybrid h, int64_t *npatch, int32_t *kmax, int64_t *nfallback,
                                 int64_t *bytes);

/* ------------------------------------------------------------------ recovery
 * P_K = (v^t (R_K - C_K W_K) - g_K)/B_K (K != K0), P_K0 = 0;  Uhat_K = Ahat^{-1}(R_K - D_K P_K - C_K W_K);
 * U_sigma = the copy of face_cells[sigma][0].  U_d [nf_int][dim], P_d [nc].
 * diag_d (may be NULL) [2]: max |Uhat_K - Uhat_L| over interior faces ("this common value")
 * and max_K |sum_{sigma in F_K} a_{K,sigma} . U_sigma| (boundary faces at their Dirichlet value). */
cr_status cr_recover(cr_hybrid h, const double *W_d, double *U_d, double *P_d, double *diag_d,
                     cr_stream_t s);

/* ------------------------------------------------------------------ Newton update
 * U_d[i] += lam dU_d[i] (i < nU), P_d[k] += lam dP_d[k] (k < nP) on the device, and returns on the
 * host norms_h[0] = ||lam dU||_2, norms_h[1] = ||U + lam dU||_2 (fixed-order reductions:
 * deterministic); Newton's method stops when norms_h[0] <= tol * norms_h[1] (P:L783-799:
 * tol = 5e-7).  lam = 1: the full step; lam < 1: a damped step (line search, see
 * cr_coupled_rhs_norm).  U_d / dU_d [nU], P_d / dP_d [nP] (dP_d may be NULL: P unchanged).
 * Synchronises `s`.                                                                          */
cr_status cr_newton_update(int64_t nU, double *U_d, const double *dU_d, int64_t nP, double *P_d,
                           const double *dP_d, double lam, double *norms_h, cr_stream_t s);
/* ||[R; g]||_2 of the coupled system of (prm, data): for a Navier-Stokes Newton step
 * (physics = CR_NS_NEWTON_STEP, u_iter / p_iter = the iterate) the increment-form right-hand side is
 * minus the nonlinear residual F(U^k, P^k) of the discrete steady equations, so this is ||F||, the
 * merit function of a damped Newton line search.  Returned on the host; synchronises `s`.     */
cr_status cr_coupled_rhs_norm(cr_mesh m, const cr_params *prm, const cr_data *data, double *norm_h, cr_stream_t s);

/* Per (cell, local face) values of a face field (the Newton iterate layout of cr_data.u_iter_d,
 * P:L302): out_d[K][l] = U_d[face_dof(sigma)] on interior faces, bnd_d[K][l] (wall / lid values;
 * NULL = 0) on boundary faces.  U_d [nf_int][dim], bnd_d / out_d [nc][dim+1][dim].  Newton's
 * method for steady Navier-Stokes iterates cr_hybridise(u_iter = this, p_iter = P^k)
 * -> cr_solve -> cr_recover (increments dU, dP).  Asynchronous.                               */
cr_status cr_cell_face_values(cr_mesh m, const double *U_d, const double *bnd_d, double *out_d, cr_stream_t s);

/* ------------------------------------------------------------------ multi-GPU
 * One process per GPU.  Rank q of P owns the contiguous block rows [floor(q F/P), floor((q+1)F/P))
 * of G (F = nf_int, lexicographic face order = slabs); every rank builds the whole mesh, assembles
 * and stores only its rows (columns renumbered: owned rows first, then ghosts in ascending global
 * order) and exchanges ghost entries of the SpMV input with the ranks that own them.  Partitioned
 * handles come from cr_hybridise(..., comm, ...) with an NCCL or loopback comm; then n_rows of
 * cr_hybrid_info, the W_d of cr_solve and the x/y of cr_spmv are LOCAL (owned rows x dim);
 * cr_recover gathers W and returns the GLOBAL U [nf_int][dim] and P [nc] on every rank.
 * Distributed cr_solve supports the PCG methods (CR_PCG_JACOBI, CR_PCG_AFW; the patch
 * preconditioner uses the patches restricted to the owned faces).                            */
/* 128-byte NCCL unique id (rank 0 creates it and broadcasts it, e.g. with torch.distributed) */
cr_status cr_nccl_unique_id(void *out128);
/* NCCL communicator (NCCL is dlopen'ed: import torch first).  nccl_unique_id = NULL with
 * nranks = 1 gives a trivial communicator (unpartitioned handles); with an id, even a single
 * rank takes the partitioned path (all collectives through NCCL).                            */
cr_status cr_comm_init(const void *nccl_unique_id, int32_t rank, int32_t nranks, cr_comm *out);
/* In-process loopback group: nranks host threads of ONE process share one GPU, exchanging
 * through device copies and host barriers (no NCCL, no CUDA graphs).  For testing the
 * partitioned path on a single GPU; each thread uses its own comm from cr_comm_init_loopback. */
cr_status cr_loopback_create(int32_t nranks, cr_loopback *out);
void cr_loopback_destroy(cr_loopback g);
cr_status cr_comm_init_loopback(cr_loopback g, int32_t rank, cr_comm *out);
void cr_comm_destroy(cr_comm c);
/* partition of a hybrid handle: owned global block rows [row0, row1), ghosts, global rows    */
cr_status cr_hybrid_partition_info(cr_hybrid h, int64_t *row0, int64_t *row1, int64_t *nghost,
                                   int64_t *nglobal);
/* The partition plan on the HOST (no GPU): for rank `rank` of `nranks`, row_range [2], per-peer
 * recv_counts / send_counts [nranks] (block rows), then, if non-NULL, ghosts [sum recv_counts]
 * (ascending global block rows) and send_rows [sum send_counts] (global block rows, by peer,
 * ascending).  Arrays as exported by cr_mesh_export plus dof_face [nf_int] (the face of each
 * interior dof).  Call once with ghosts = send_rows = NULL to size them.                    */
cr_status cr_partition_plan(int32_t dim, int64_t nf_int, const int32_t *cell_faces_h,
                            const int32_t *face_cells_h, const int32_t *face_dof_h,
                            const int32_t *dof_face_h, int32_t rank, int32_t nranks,
                            int64_t *row_range, int64_t *recv_counts, int64_t *send_counts,
                            int32_t *ghosts, int32_t *send_rows);

/* The nested-dissection plan of the coarse solve (host only, no GPU; coarse.cu)
 * for an (H+1)^dim node grid: box = 0 recursive bisection, box > 0 the flat two-level plan
 * (separator slabs after every `box` nodes form the root, the boxes are its children).  Fronts
 * in post-order (children before parents), each with its depth, its parent (parent [nf]; -1
 * for the root), pivot nodes I and boundary nodes B (the later-eliminated nodes its subtree
 * couples to through the 5^dim-node stencil of Z^t G Z), the lists concatenated in front order
 * (node = x + (H+1) (y + (H+1) z)).  Call once with the array arguments NULL to size them.     */
cr_status cr_coarse_nd_plan(int32_t H, int32_t dim, int32_t box, int64_t *nfront, int32_t *maxdepth, int64_t *total_I,
                            int64_t *total_B, int32_t *depth, int32_t *parent, int32_t *nI, int32_t *nB,
                            int32_t *I_nodes, int32_t *B_nodes);

/* Sparse direct solve A x = b of a canonical CSR system (int64 row_ptr [n+1], int32 cols, f64
 * vals: the layout of cr_hybrid_export_csr / cr_coupled_export_csr) on the device with cuSOLVER
 * (plain library factorisation): method 0 = sparse Cholesky (SPD: the transient hybrid G,
 * P:L535), 1 = sparse QR (the indefinite coupled matrix); reorder 0 none, 1 symrcm,
 * 2 symamd, 3 metis.  The paper's direct-solver comparison (Table 4).  Synchronises
 * `s`; *singularity (may be NULL) = -1 or the first singular pivot (then CR_ERR_SINGULAR_LOCAL). */
cr_status cr_sparse_direct_solve(int64_t n, int64_t nnz, const int64_t *row_ptr_d, const int32_t *cols_d,
                                 const double *vals_d, const double *b_d, double *x_d, int32_t method,
                                 int32_t reorder, cr_stream_t s, int32_t *singularity);

/* ------------------------------------------------------------------ the whole method from HOST buffers
 * The paper's "hybrid method" end to end for a caller whose data lives in host
 * memory: coords_h [nv][dim], cells_h [nc][dim+1], fbar_h [nc][dim] (and, when non-NULL,
 * dirichlet_h [nc][dim+1][dim]) are copied to the device on `s` (pinned host memory makes the
 * copies asynchronous DMA; pageable memory works, staged by the driver), then cr_build_mesh ->
 * cr_hybridise -> cr_solve -> cr_recover run on the device, and U_h [nf_int][dim] and P_h [nc]
 * (caller-owned HOST buffers; size nf_int from the mesh — pass sizes_h [2] = {nf_int*dim, nc}
 * capacities) receive the result.  The handles and device buffers live only for the call.
 * mesh_info (may be NULL) receives the mesh counts; rep the solve report.  Synchronises `s`.
 * Errors: those of the four calls; INVALID_ARG when a capacity is too small.               */
cr_status cr_hybrid_method_host(int32_t dim, int64_t nv, const double *coords_h, int64_t nc,
                                const int32_t *cells_h, const cr_params *prm, const double *fbar_h,
                                const double *dirichlet_h, const cr_solver_opts *opts, double *U_h,
                                double *P_h, const int64_t *sizes_h, cr_mesh_info_t *mesh_info,
                                cr_solve_report *rep, cr_stream_t s);

/* ------------------------------------------------------------------ memory and accounting
 * All device memory of the handles comes from the library's OWN stream-ordered pool on the
 * current device (cudaMemPoolCreate; the device's default pool is never modified).  The pool
 * keeps freed memory mapped for re-use by the next call (release threshold UINT64_MAX).
 * cr_pool_reserve: map `bytes` into the pool now (opt-in; avoids mapping new memory in the
 * middle of a later solve).  cr_pool_trim: return all but `keep_bytes` of the unused memory.
 * cr_kernel_launches: kernels this process launched from libcr so far (direct launches plus
 * the kernel nodes of every replayed solver graph; CUB, cuBLAS and cuSOLVER launches excluded). */
cr_status cr_pool_reserve(int64_t bytes, cr_stream_t s);
cr_status cr_pool_trim(int64_t keep_bytes);
int64_t cr_kernel_launches(void);

const char *cr_last_error(void);
const char *cr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CR_H */
