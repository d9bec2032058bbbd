// C ABI entry points of libcr (include/cr.h).  Every entry point converts exceptions into a
// cr_status and a thread-local message; no C++ exception crosses the ABI.
#include <cstring>
#include <string>

#include "internal.cuh"

#include <chrono>
#include <cstdlib>

namespace cr {
static thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }

static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
Trace::Trace(cudaStream_t st) : s(st) {
    const char *e = std::getenv("CR_TRACE");
    on = e && e[0] == '1';
    if (on) {
        cudaStreamSynchronize(s);
        t0 = now_s();
    }
}
void Trace::mark(const char *what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = now_s();
    std::fprintf(stderr, "[cr_trace] %-28s %9.3f ms\n", what, (t - t0) * 1e3);
    t0 = t;
}
}  // namespace cr

// Keep freed stream-ordered memory in the device's default pool (no trim to the OS at every
// synchronisation): repeated solves re-use their buffers without remapping.
static void keep_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    static thread_local int done_dev = -1;
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // reserve physical memory for the pool once (CR_POOL_RESERVE_GB, default 16): growing the
        // pool mid-solve (mapping new memory after a burst of frees of mixed sizes) stalled the
        // first allocation after a two-level solve for up to 0.5 s
        const char *e = std::getenv("CR_POOL_RESERVE_GB");
        const double gb = e ? atof(e) : 16.0;
        size_t fr = 0, tot = 0;
        if (gb > 0 && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
            const size_t want = std::min((size_t)(gb * 1073741824.0), fr / 2);
            void *p = nullptr;
            if (want > 0 && cudaMallocAsync(&p, want, 0) == cudaSuccess) {
                cudaFreeAsync(p, 0);
                cudaStreamSynchronize(0);
            }
            cudaGetLastError();
        }
    }
    done_dev = dev;
}

cr_hybrid_s::~cr_hybrid_s() { cr::free_solver_work(work); }

#define CR_API_BEGIN try {
#define CR_API_END                                              \
    return CR_OK;                                               \
    }                                                           \
    catch (const cr::Error &e) {                                \
        cr::set_last_error(e.what());                           \
        return e.code;                                          \
    }                                                           \
    catch (const std::exception &e) {                           \
        cr::set_last_error(e.what());                           \
        return CR_ERR_CUDA;                                     \
    }                                                           \
    catch (...) {                                               \
        cr::set_last_error("unknown error");                    \
        return CR_ERR_CUDA;                                     \
    }

extern "C" {

const char *cr_last_error(void) { return cr::g_last_error.c_str(); }
const char *cr_version(void) { return "libcr 0.1 (sm_100a, fp64, double-double local elimination)"; }

cr_status cr_build_mesh(int32_t dim, int64_t nv, const double *coords_d, int64_t nc, const int32_t *cells_d,
                        cr_stream_t s, cr_mesh *out) {
    CR_API_BEGIN
    CR_REQUIRE(out, CR_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    keep_pool();
    cr_mesh_s *m = new cr_mesh_s();
    try {
        cr::build_mesh(m, dim, nv, coords_d, nc, cells_d, (cudaStream_t)s);
    } catch (...) {
        delete m;
        throw;
    }
    *out = m;
    CR_API_END
}

cr_status cr_mesh_info(cr_mesh m, cr_mesh_info_t *out) {
    CR_API_BEGIN
    CR_REQUIRE(m && out, CR_ERR_INVALID_ARG, "null handle");
    out->dim = m->dim;
    out->nv = m->nv;
    out->nc = m->nc;
    out->nf = m->nf;
    out->nf_int = m->nf_int;
    out->n_unknowns = m->dim * m->nf_int;
    CR_API_END
}

static void copy_d2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (dst && bytes) CR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
}

cr_status cr_mesh_export(cr_mesh m, int32_t *faces_d, int32_t *face_cells_d, int32_t *cell_faces_d,
                         int32_t *face_dof_d, double *vol_d, double *xK_d, double *xs_d, double *a_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(m, CR_ERR_INVALID_ARG, "null handle");
    cudaStream_t st = (cudaStream_t)s;
    const int D = m->dim;
    copy_d2d(faces_d, m->faces.get(), m->nf * D * sizeof(int32_t), st);
    copy_d2d(face_cells_d, m->face_cells.get(), m->nf * 2 * sizeof(int32_t), st);
    copy_d2d(cell_faces_d, m->cell_faces.get(), m->nc * (D + 1) * sizeof(int32_t), st);
    copy_d2d(face_dof_d, m->face_dof.get(), m->nf * sizeof(int32_t), st);
    copy_d2d(vol_d, m->vol.get(), m->nc * sizeof(double), st);
    copy_d2d(xK_d, m->xK.get(), m->nc * D * sizeof(double), st);
    copy_d2d(xs_d, m->xs.get(), m->nf * D * sizeof(double), st);
    copy_d2d(a_d, m->a.get(), m->nc * (D + 1) * D * sizeof(double), st);
    CR_API_END
}

void cr_destroy_mesh(cr_mesh m) {
    cr::SyncFreeScope sync;
    delete m;
}

cr_status cr_assemble_coupled(cr_mesh m, const cr_params *prm, const cr_data *data, cr_stream_t s, cr_coupled *out) {
    CR_API_BEGIN
    CR_REQUIRE(m && prm && data && out, CR_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    cr_coupled_s *c = new cr_coupled_s();
    try {
        cr::assemble_coupled(c, m, *prm, *data, (cudaStream_t)s);
    } catch (...) {
        delete c;
        throw;
    }
    *out = c;
    CR_API_END
}

cr_status cr_coupled_info(cr_coupled c, int64_t *n_rows, int64_t *nnz) {
    CR_API_BEGIN
    CR_REQUIRE(c, CR_ERR_INVALID_ARG, "null handle");
    if (n_rows) *n_rows = c->n_rows;
    if (nnz) *nnz = c->nnz;
    CR_API_END
}

cr_status cr_coupled_export_csr(cr_coupled c, int64_t *row_ptr_d, int32_t *cols_d, double *vals_d, double *rhs_d,
                                cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(c, CR_ERR_INVALID_ARG, "null handle");
    cudaStream_t st = (cudaStream_t)s;
    copy_d2d(row_ptr_d, c->row_ptr.get(), (c->n_rows + 1) * sizeof(int64_t), st);
    copy_d2d(cols_d, c->cols.get(), c->nnz * sizeof(int32_t), st);
    copy_d2d(vals_d, c->vals.get(), c->nnz * sizeof(double), st);
    copy_d2d(rhs_d, c->rhs.get(), c->n_rows * sizeof(double), st);
    CR_API_END
}

void cr_destroy_coupled(cr_coupled c) {
    cr::SyncFreeScope sync;
    delete c;
}

cr_status cr_hybridise(cr_mesh m, const cr_params *prm, const cr_data *data, cr_comm comm, cr_stream_t s,
                       cr_hybrid *out) {
    CR_API_BEGIN
    CR_REQUIRE(m && prm && data && out, CR_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    cr_hybrid_s *h = new cr_hybrid_s();
    try {
        cr::hybridise(h, m, *prm, *data, comm, (cudaStream_t)s);
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
    CR_API_END
}

cr_status cr_hybrid_info(cr_hybrid h, int64_t *n_rows, int64_t *nnz, int64_t *nblocks) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    const int D = h->G.d;
    if (n_rows) *n_rows = h->G.nrows * D;
    if (nnz) *nnz = h->G.nblocks * D * D;
    if (nblocks) *nblocks = h->G.nblocks;
    CR_API_END
}

cr_status cr_hybrid_partition_info(cr_hybrid h, int64_t *row0, int64_t *row1, int64_t *nghost, int64_t *nglobal) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    const bool on = h->part.on;
    if (row0) *row0 = on ? h->part.row0 : 0;
    if (row1) *row1 = on ? h->part.row1 : h->G.nrows;
    if (nghost) *nghost = on ? h->part.nghost : 0;
    if (nglobal) *nglobal = on ? h->part.nglobal : h->G.nrows;
    CR_API_END
}

cr_status cr_hybrid_export_csr(cr_hybrid h, int64_t *row_ptr_d, int32_t *cols_d, double *vals_d, double *S_d,
                               cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && row_ptr_d && cols_d && vals_d, CR_ERR_INVALID_ARG, "null argument");
    cr::hybrid_export_csr(h, row_ptr_d, cols_d, vals_d, S_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_hybrid_export_shift(cr_hybrid h, uint8_t *inM1_d, double *E_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    const cr_mesh_s *m = h->mesh;
    copy_d2d(inM1_d, h->inM1.get(), m->nc, (cudaStream_t)s);
    copy_d2d(E_d, h->E.get(), m->nc * (m->dim + 1) * sizeof(double), (cudaStream_t)s);
    CR_API_END
}

cr_status cr_spmv(cr_hybrid h, const double *x_d, double *y_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && x_d && y_d && x_d != y_d, CR_ERR_INVALID_ARG, "bad arguments");
    if (h->part.on) cr::spmv_part(h, x_d, y_d, (cudaStream_t)s);
    else cr::spmv(h->G, x_d, y_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_spmv_mf(cr_hybrid h, const double *x_d, double *y_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && x_d && y_d && x_d != y_d, CR_ERR_INVALID_ARG, "bad arguments");
    cr::spmv_mf(h, x_d, y_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_hybrid_set_cell_rhs(cr_hybrid h, const double *R_d, const double *g_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && ((R_d == nullptr) == (g_d == nullptr)), CR_ERR_INVALID_ARG, "R_d and g_d: both or neither");
    CR_REQUIRE(!h->is_ns, CR_ERR_INVALID_ARG, "explicit cell right-hand sides: Stokes handles only");
    cudaStream_t st = (cudaStream_t)s;
    const cr_mesh_s *m = h->mesh;
    if (!R_d) {
        h->rcell.release();
        h->gcell.release();
    } else {
        const size_t nr = (size_t)m->nc * (m->dim + 1) * m->dim;
        if (h->rcell.n != nr) h->rcell.alloc(nr, st);
        if (h->gcell.n != (size_t)m->nc) h->gcell.alloc(m->nc, st);
        CR_CUDA(cudaMemcpyAsync(h->rcell.get(), R_d, nr * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CR_CUDA(cudaMemcpyAsync(h->gcell.get(), g_d, m->nc * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    cr::hybrid_update_rhs(h, st);
    CR_API_END
}

cr_status cr_transient_rhs(cr_hybrid h, const double *U_prev_d, double *R_d, double *g_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && U_prev_d && R_d && g_d, CR_ERR_INVALID_ARG, "null argument");
    cr::transient_rhs(h, U_prev_d, R_d, g_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_hybrid_coarse_info(cr_hybrid h, int32_t *H, int64_t *nE, int32_t *nd, int64_t *solve_bytes) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    const auto &C = h->coarse;
    if (H) *H = C.built;
    if (nE) *nE = C.built ? C.nE : 0;
    if (nd) *nd = C.built && C.nd.on ? 1 : 0;
    if (solve_bytes) *solve_bytes = !C.built ? 0 : C.nd.on ? C.nd.bytes : (int64_t)(8 * C.nE * C.nE);
    CR_API_END
}

cr_status cr_hybrid_mf_info(cr_hybrid h, int64_t *ncells, int64_t *bytes) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    const bool b = h->mf.built;
    if (ncells) *ncells = b ? h->mf.ncells : 0;
    if (bytes)
        *bytes = b ? (int64_t)(h->mf.v.n * sizeof(double) + h->mf.ids.n * sizeof(int32_t) + h->mf.sg.n + h->mf.nb.n)
                   : 0;
    CR_API_END
}

void cr_destroy_hybrid(cr_hybrid h) {
    cr::SyncFreeScope sync;
    delete h;
}

cr_status cr_solve(cr_hybrid h, const cr_solver_opts *opts, double *W_d, cr_stream_t s, cr_solve_report *rep) {
    CR_API_BEGIN
    CR_REQUIRE(h && opts && W_d, CR_ERR_INVALID_ARG, "null argument");
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (opts->method == CR_DC_FGMRES) cr::solve_dc(h, *opts, W_d, (cudaStream_t)s, rep);
    else cr::solve(h, *opts, W_d, (cudaStream_t)s, rep);
    CR_API_END
}

cr_status cr_apply_precond(cr_hybrid h, int32_t method, const double *r_d, double *z_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && r_d && z_d && r_d != z_d, CR_ERR_INVALID_ARG, "bad arguments");
    cr::apply_precond(h, method, r_d, z_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_hybrid_precond_info(cr_hybrid h, int64_t *npatch, int32_t *kmax, int64_t *nfallback, int64_t *bytes) {
    CR_API_BEGIN
    CR_REQUIRE(h, CR_ERR_INVALID_ARG, "null handle");
    if (bytes)
        *bytes = h->afw.built >= 0 ? (int64_t)(h->afw.vals.n * sizeof(double) + h->afw.ids.n * sizeof(int32_t) +
                                               h->afw.kl.n + 2 * h->afw.ioff.n * sizeof(int64_t))
                                   : 0;
    if (npatch) *npatch = h->afw.built >= 0 ? h->afw.npatch : 0;
    if (kmax) *kmax = h->afw.built >= 0 ? h->afw.kmax : 0;
    if (nfallback) *nfallback = h->afw.built >= 0 ? h->afw.nfallback : 0;
    CR_API_END
}

cr_status cr_cell_face_values(cr_mesh m, const double *U_d, const double *bnd_d, double *out_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(m && U_d && out_d, CR_ERR_INVALID_ARG, "null argument");
    cr::cell_face_values(m, U_d, bnd_d, out_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_recover(cr_hybrid h, const double *W_d, double *U_d, double *P_d, double *diag_d, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(h && W_d && U_d && P_d, CR_ERR_INVALID_ARG, "null argument");
    cr::recover(h, W_d, U_d, P_d, diag_d, (cudaStream_t)s);
    CR_API_END
}

}  // extern "C"
