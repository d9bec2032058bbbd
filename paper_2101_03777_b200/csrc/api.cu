// C ABI entry points of libcr (include/cr.h).  Every entry point converts exceptions into a
// cr_status and a thread-local message; no C++ exception crosses the ABI.
#include <cstring>
#include <memory>
#include <string>

#include "internal.cuh"

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <nvtx3/nvToolsExt.h>

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
Range::Range(const char *name) { nvtxRangePushA(name); }
Range::~Range() { nvtxRangePop(); }
void Trace::mark(const char *what) {
    nvtxMarkA(what);
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = now_s();
    std::fprintf(stderr, "[cr_trace] %-28s %9.3f ms\n", what, (t - t0) * 1e3);
    t0 = t;
}
}  // namespace cr

namespace cr {
// ------------------------------------------------------------------ memory pool, SM count, launch counter
static std::mutex g_dev_mu;
static cudaMemPool_t g_pool[64] = {};
static int g_sms[64] = {};
static std::atomic<long long> g_launches{0};
thread_local bool g_capturing = false;

static int cur_dev() {
    int dev = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_REQUIRE(dev >= 0 && dev < 64, CR_ERR_INVALID_ARG, "device index out of range");
    return dev;
}

cudaMemPool_t lib_pool() {
    const int dev = cur_dev();
    if (g_pool[dev]) return g_pool[dev];
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        cudaMemPool_t pool;
        CR_CUDA(cudaMemPoolCreate(&pool, &pp));
        // memory freed by one call stays mapped for the next (no trim at synchronisations):
        // repeated solves re-use their buffers without remapping.  cr_pool_trim returns it.
        uint64_t thr = UINT64_MAX;
        CR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        g_pool[dev] = pool;
    }
    return g_pool[dev];
}

int num_sms() {
    const int dev = cur_dev();
    if (!g_sms[dev]) {
        int n = 0;
        CR_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
        g_sms[dev] = n > 0 ? n : 1;
    }
    return g_sms[dev];
}

void count_launches(int64_t n) {
    if (!g_capturing) g_launches.fetch_add(n, std::memory_order_relaxed);
}
}  // namespace cr

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
const char *cr_version(void) { return "libcr 0.2 (sm_100a, fp64, double-double local elimination)"; }

int64_t cr_kernel_launches(void) { return (int64_t)cr::g_launches.load(); }

cr_status cr_pool_reserve(int64_t bytes, cr_stream_t s) {
    CR_API_BEGIN
    CR_REQUIRE(bytes >= 0, CR_ERR_INVALID_ARG, "bytes < 0");
    if (bytes > 0) {
        void *p = nullptr;
        CR_CUDA(cudaMallocFromPoolAsync(&p, (size_t)bytes, cr::lib_pool(), (cudaStream_t)s));
        CR_CUDA(cudaFreeAsync(p, (cudaStream_t)s));
        CR_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    }
    CR_API_END
}

cr_status cr_pool_trim(int64_t keep_bytes) {
    CR_API_BEGIN
    CR_REQUIRE(keep_bytes >= 0, CR_ERR_INVALID_ARG, "keep_bytes < 0");
    CR_CUDA(cudaMemPoolTrimTo(cr::lib_pool(), (size_t)keep_bytes));
    CR_API_END
}

cr_status cr_build_mesh(int32_t dim, int64_t nv, const double *coords_d, int64_t nc, const int32_t *cells_d,
                        cr_stream_t s, cr_mesh *out) {
    cr::Range nvtx_range("cr_build_mesh");
    CR_API_BEGIN
    CR_REQUIRE(out, CR_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
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
    cr::Range nvtx_range("cr_assemble_coupled");
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
    cr::Range nvtx_range("cr_hybridise");
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
    cr::Range nvtx_range("cr_spmv");
    CR_API_BEGIN
    CR_REQUIRE(h && x_d && y_d && x_d != y_d, CR_ERR_INVALID_ARG, "bad arguments");
    if (h->part.on) cr::spmv_part(h, x_d, y_d, (cudaStream_t)s);
    else cr::spmv(h->G, x_d, y_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_spmv_mf(cr_hybrid h, const double *x_d, double *y_d, cr_stream_t s) {
    cr::Range nvtx_range("cr_spmv_mf");
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
    cr::Range nvtx_range("cr_transient_rhs");
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
    cr::Range nvtx_range("cr_solve");
    CR_API_BEGIN
    CR_REQUIRE(h && opts && W_d, CR_ERR_INVALID_ARG, "null argument");
    if (rep) std::memset(rep, 0, sizeof(*rep));
    if (opts->method == CR_DC_FGMRES) cr::solve_dc(h, *opts, W_d, (cudaStream_t)s, rep);
    else cr::solve(h, *opts, W_d, (cudaStream_t)s, rep);
    CR_API_END
}

cr_status cr_solve_profile(cr_hybrid h, const cr_solver_opts *opts, int32_t nrep, double *ms, cr_stream_t s) {
    cr::Range nvtx_range("cr_solve_profile");
    CR_API_BEGIN
    CR_REQUIRE(h && opts && ms && nrep > 0, CR_ERR_INVALID_ARG, "bad arguments");
    for (int k = 0; k < 5; ++k) ms[k] = 0.0;
    cr::solve_profile(h, *opts, nrep, ms, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_apply_precond(cr_hybrid h, int32_t method, const double *r_d, double *z_d, cr_stream_t s) {
    cr::Range nvtx_range("cr_apply_precond");
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
    cr::Range nvtx_range("cr_recover");
    CR_API_BEGIN
    CR_REQUIRE(h && W_d && U_d && P_d, CR_ERR_INVALID_ARG, "null argument");
    cr::recover(h, W_d, U_d, P_d, diag_d, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_newton_update(int64_t nU, double *U_d, const double *dU_d, int64_t nP, double *P_d, const double *dP_d,
                           double lam, double *norms_h, cr_stream_t s) {
    cr::Range nvtx_range("cr_newton_update");
    CR_API_BEGIN
    CR_REQUIRE(nU >= 0 && nP >= 0 && U_d && dU_d && norms_h && (!dP_d || P_d), CR_ERR_INVALID_ARG, "bad arguments");
    cr::newton_update(nU, U_d, dU_d, nP, P_d, dP_d, lam, norms_h, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_coupled_rhs_norm(cr_mesh m, const cr_params *prm, const cr_data *data, double *norm_h, cr_stream_t s) {
    cr::Range nvtx_range("cr_coupled_rhs_norm");
    CR_API_BEGIN
    CR_REQUIRE(m && prm && data && norm_h, CR_ERR_INVALID_ARG, "null argument");
    cr_coupled_s c;
    cr::assemble_coupled(&c, m, *prm, *data, (cudaStream_t)s);
    *norm_h = cr::norm2(c.rhs.get(), c.n_rows, (cudaStream_t)s);
    CR_API_END
}

cr_status cr_hybrid_method_host(int32_t dim, int64_t nv, const double *coords_h, int64_t nc, const int32_t *cells_h,
                                const cr_params *prm, const double *fbar_h, const double *dirichlet_h,
                                const cr_solver_opts *opts, double *U_h, double *P_h, const int64_t *sizes_h,
                                cr_mesh_info_t *mesh_info, cr_solve_report *rep, cr_stream_t s) {
    cr::Range nvtx_range("cr_hybrid_method_host");
    CR_API_BEGIN
    CR_REQUIRE(coords_h && cells_h && prm && fbar_h && opts && U_h && P_h && sizes_h, CR_ERR_INVALID_ARG,
               "null argument");
    CR_REQUIRE((dim == 2 || dim == 3) && nv > 0 && nc > 0, CR_ERR_INVALID_ARG, "bad mesh sizes");
    if (rep) std::memset(rep, 0, sizeof(*rep));
    cudaStream_t st = (cudaStream_t)s;
    // host -> device (DMA straight from pinned buffers; the driver stages pageable ones)
    cr::DevBuf<double> coords, fbar, dir;
    cr::DevBuf<int32_t> cells;
    coords.alloc((size_t)nv * dim, st);
    cells.alloc((size_t)nc * (dim + 1), st);
    fbar.alloc((size_t)nc * dim, st);
    CR_CUDA(cudaMemcpyAsync(coords.get(), coords_h, (size_t)nv * dim * sizeof(double), cudaMemcpyHostToDevice, st));
    CR_CUDA(cudaMemcpyAsync(cells.get(), cells_h, (size_t)nc * (dim + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CR_CUDA(cudaMemcpyAsync(fbar.get(), fbar_h, (size_t)nc * dim * sizeof(double), cudaMemcpyHostToDevice, st));
    if (dirichlet_h) {
        dir.alloc((size_t)nc * (dim + 1) * dim, st);
        CR_CUDA(cudaMemcpyAsync(dir.get(), dirichlet_h, (size_t)nc * (dim + 1) * dim * sizeof(double),
                                cudaMemcpyHostToDevice, st));
    }
    std::unique_ptr<cr_mesh_s> m(new cr_mesh_s());
    cr::build_mesh(m.get(), dim, nv, coords.get(), nc, cells.get(), st);
    const int64_t nU = (int64_t)dim * m->nf_int;
    CR_REQUIRE(sizes_h[0] >= nU && sizes_h[1] >= nc, CR_ERR_INVALID_ARG, "U_h / P_h capacity too small");
    if (mesh_info) {
        mesh_info->dim = dim;
        mesh_info->nv = nv;
        mesh_info->nc = nc;
        mesh_info->nf = m->nf;
        mesh_info->nf_int = m->nf_int;
        mesh_info->n_unknowns = nU;
    }
    const cr_data data{fbar.get(), dirichlet_h ? dir.get() : nullptr, nullptr, nullptr};
    std::unique_ptr<cr_hybrid_s> h(new cr_hybrid_s());
    cr::hybridise(h.get(), m.get(), *prm, data, nullptr, st);
    cr::DevBuf<double> W, U, P;
    W.alloc(nU, st);
    W.zero(st);
    U.alloc(nU, st);
    P.alloc(nc, st);
    if (opts->method == CR_DC_FGMRES) cr::solve_dc(h.get(), *opts, W.get(), st, rep);
    else cr::solve(h.get(), *opts, W.get(), st, rep);
    cr::recover(h.get(), W.get(), U.get(), P.get(), nullptr, st);
    // device -> host
    CR_CUDA(cudaMemcpyAsync(U_h, U.get(), nU * sizeof(double), cudaMemcpyDeviceToHost, st));
    CR_CUDA(cudaMemcpyAsync(P_h, P.get(), nc * sizeof(double), cudaMemcpyDeviceToHost, st));
    CR_CUDA(cudaStreamSynchronize(st));
    CR_API_END
}

}  // extern "C"
