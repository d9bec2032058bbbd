// Internal declarations of libcr (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "coarse.cuh"
#include "cr.h"

namespace cr {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    cr_status code;
    Error(cr_status c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &m);

#define CR_CUDA(call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            throw ::cr::Error(e_ == cudaErrorMemoryAllocation ? CR_ERR_OOM : CR_ERR_CUDA,  \
                              std::string(#call) + ": " + cudaGetErrorString(e_));         \
        }                                                                                  \
    } while (0)

#define CR_CHECK_LAUNCH() do { ::cr::count_launches(1); CR_CUDA(cudaGetLastError()); } while (0)

#define CR_REQUIRE(cond, code, msg)                     \
    do {                                                \
        if (!(cond)) throw ::cr::Error((code), (msg));  \
    } while (0)

// ------------------------------------------------------------------ device buffer
// Stream-ordered: allocated with cudaMallocAsync on stream s and freed with cudaFreeAsync on
// the same stream, so a temporary released while kernels that use it are still queued is
// only recycled after them.  Handle destructors (cr_destroy_*) synchronise the device first
// and set g_sync_free, because the caller's stream may no longer exist at that point.
inline thread_local bool g_sync_free = false;
struct SyncFreeScope {
    SyncFreeScope() { cudaDeviceSynchronize(); g_sync_free = true; }
    ~SyncFreeScope() { g_sync_free = false; }
};

// the library's own stream-ordered memory pool on the current device (api.cu): created on first
// use with a release threshold of UINT64_MAX, so memory freed by one call is re-used by the next
// without remapping; the device's DEFAULT pool (and the host application's) is never touched.
cudaMemPool_t lib_pool();
// SMs of the current device (cached per device): grids are sized from it, never from a constant
int num_sms();
// kernels launched by the library on this process (cr_kernel_launches): direct launches are
// counted in CR_CHECK_LAUNCH, kernels replayed inside the solvers' CUDA graphs by the solver
void count_launches(int64_t n);
extern thread_local bool g_capturing;   // inside a solver graph capture: launches not counted

template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s_ = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), s_(o.s_) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s_ = o.s_; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count, cudaStream_t s) {
        release();
        n = count;
        s_ = s;
        if (count == 0) return;
        CR_CUDA(cudaMallocFromPoolAsync((void **)&p, count * sizeof(T) + 16, lib_pool(), s));
    }
    void zero(cudaStream_t s) { if (n) CR_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s)); }
    void fill_bytes(int v, cudaStream_t s) { if (n) CR_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), s)); }
    void release() {
        if (p) {
            if (g_sync_free) cudaFree(p);
            else cudaFreeAsync(p, s_);
        }
        p = nullptr;
        n = 0;
    }
    T *get() const { return p; }
};

// error word written by kernels (first error wins)
enum DevErr : int {
    DE_OK = 0, DE_RANGE = 1, DE_DEGENERATE = 2, DE_NONMANIFOLD = 3, DE_NOINTERIOR = 4,
    DE_SINGULAR = 5, DE_BZERO = 6
};

// grid sizing: streaming kernels use a fixed grid per device (deterministic partials), a
// multiple of the device's SM count (148 on B200)

// Grid of exactly one wave of resident blocks (occupancy of `kernel` at `threads` per block) for
// grid-stride kernels: a second, partial wave would leave SMs idle while it drains.  Cached per
// kernel; the grid only depends on the kernel and the GPU, so block partials stay deterministic.
template <class F>
inline int occ_grid(F kernel, int threads, int64_t work, int reserve = 0) {
    static thread_local std::vector<std::pair<const void *, int>> cache;
    const void *key = reinterpret_cast<const void *>(kernel);
    int nb = 0;
    for (auto &kv : cache)
        if (kv.first == key) nb = kv.second;
    if (nb == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, 0) != cudaSuccess || nb < 1) nb = 1;
        nb = nb > 16 ? 16 : nb;
        cache.emplace_back(key, nb);
    }
    int64_t b = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * (nb > reserve ? nb - reserve : 1);
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}
inline int grid_for(int64_t work, int threads, int max_blocks_per_sm = 8) {
    int64_t b = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms() * max_blocks_per_sm;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// NVTX range around an ABI call (domain-less push/pop; a no-op unless a profiler injects NVTX):
// nsys / ncu --nvtx show the stages of the path by name.
struct Range {
    explicit Range(const char *name);
    ~Range();
    Range(const Range &) = delete;
    Range &operator=(const Range &) = delete;
};

// CR_TRACE=1: host wall time of setup phases on stderr (synchronises the stream at each mark);
// every mark is also an NVTX marker.
struct Trace {
    bool on = false;
    double t0 = 0.0;
    cudaStream_t s = nullptr;
    explicit Trace(cudaStream_t st);
    void mark(const char *what);
};

}  // namespace cr

// ------------------------------------------------------------------ handles
struct cr_mesh_s {
    int dim = 0;
    int64_t nv = 0, nc = 0, nf = 0, nf_int = 0;
    cr::DevBuf<int32_t> faces, face_cells, cell_faces, face_dof, dof_face;
    cr::DevBuf<double> vol, xK, xs, a;
};

// sliced block-ELL of G
struct BlockEll {
    int d = 0, W = 0;            // block size, blocks per row (2d+1)
    int64_t nrows = 0;           // block rows = nf_int
    int64_t nslices = 0;         // ceil(nrows / 32)
    cr::DevBuf<int32_t> cols;    // [slice][slot][lane]
    cr::DevBuf<double> vals;     // [slice][slot*d*d + i*d + j][lane]
    int64_t nblocks = 0;         // true (unpadded) blocks
};

namespace cr { struct SolverWork; }

namespace cr {
// host partition plan (partition.cu)
struct PartPlan {
    int rank = 0, nranks = 1;
    int64_t row0 = 0, row1 = 0;
    std::vector<int64_t> ghosts;                  // ascending global block rows
    std::vector<int64_t> recv_counts, send_counts;  // per peer (block rows)
    std::vector<int32_t> send_rows;               // global block rows, by peer then ascending
};
void plan_partition(int dim, int64_t nf_int, const int32_t *cell_faces, const int32_t *face_cells,
                    const int32_t *face_dof, const int32_t *dof_face, int rank, int nranks, PartPlan &pl);
int64_t part_row0(int64_t nrows, int rank, int nranks);

// device-side partition of a hybrid system (empty when not partitioned)
struct Part {
    bool on = false;
    int rank = 0, nranks = 1;
    int64_t row0 = 0, row1 = 0, nloc = 0, nghost = 0, nglobal = 0;
    std::vector<int64_t> rcount, roff, scount, soff;   // per peer, block rows
    std::vector<int64_t> all_row0;                     // row0 of every rank, + nglobal
    int64_t nsend = 0;
    DevBuf<int32_t> send_rows;   // LOCAL row of each packed send entry
    DevBuf<int32_t> g2l;         // [nglobal] global block row -> local index (owned, then ghosts) or -1
    DevBuf<int32_t> l2g;         // [nloc + nghost]
    DevBuf<double> sendbuf;      // [nsend * D]
};

// collectives of the partitioned path (comm.cu)
struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() {}
    virtual bool capturable() const = 0;
    virtual void allreduce(double *d, int n, bool max, cudaStream_t s) = 0;
    // a sum over a second communicator (the coarse path on its own stream); has_side() == false:
    // none (the caller then keeps the coarse path on the main stream)
    virtual bool has_side() const { return false; }
    virtual void allreduce_side(double *d, int n, cudaStream_t s) { allreduce(d, n, false, s); }
    virtual void halo(const Part &P, const double *sendbuf, double *xghost, int D, cudaStream_t s) = 0;
    virtual void allgatherv(const double *local, double *full, const std::vector<int64_t> &counts,
                            const std::vector<int64_t> &displs, cudaStream_t s) = 0;
};
}  // namespace cr

// overlapping-patch additive Schwarz preconditioner (afw.cuh layout)
struct AfwPrec {
    int built = -1;              // mode it was built for (-1 = not built)
    int slots = 0, kmax = 0;     // patches per face (2D 2, 3D 3); largest patch
    int shared = 0;              // 1: one (component-averaged) block per patch (experiment)
    int64_t npatch = 0, nslices = 0, nfallback = 0;
    cr::DevBuf<int64_t> ioff, voff;
    cr::DevBuf<uint8_t> kl;
    cr::DevBuf<int32_t> ids;
    cr::DevBuf<int32_t> ids_so;  // ids with solve-order rows (cr_hybrid_s::so)
    cr::DevBuf<double> vals;
};
enum { AFW_SPD = 0, AFW_ABS = 1, AFW_GEN = 2 };

// sparse direct coarse solve (coarse.cu, "ND"): nested dissection of the coarse node grid into
// fronts (separator slabs 2 nodes thick: Z^t G Z couples nodes up to 2 apart), multifrontal
// elimination with explicit front inverses.  Per front f (unknowns I = its pivots, B = the
// ancestors' unknowns it couples to): Finv = F_II^{-1}, W = F_BI Finv (column-major, ld ldW).
struct NdFrontDev {
    int64_t ioff, boff;       // into nodes[]: I nodes, B nodes
    int64_t finv, w, wt, bi, u;   // into the pools (wt: W^t, nI x nB, ld nI)
    int64_t lb, inv, uoff;        // local B rhs; children's u per local unknown (CSR row); global unknowns
    int64_t map;              // into map[]: this front's B unknown -> parent local unknown
    int32_t nI, nB;           // unknowns
    int32_t kid_off, kid_cnt; // child fronts: kids[kid_off .. kid_off + kid_cnt)
    int32_t ldFi, ldW;        // leading dimensions of Finv (>= nI) and W (>= nB)
    // solve layouts (16-byte aligned rows, even leading dimensions, zero padding): Finv rows
    // (fs, ldFs), W rows = W^t columns (wts, ldWts: the forward B rows), W columns (ws, ldWs: the
    // backward pivot rows)
    int64_t fs, wts, ws;
    int32_t ldFs, ldWts, ldWs, pad_;
    int64_t yb;               // backward: this front's y_B gathered contiguously (ldWs entries, zero pad)
};
struct CoarseNd {
    bool on = false;
    int m = 0, maxdepth = 0;
    int64_t nfront = 0, bytes = 0;   // fronts; bytes one solve reads (Finv + 2 W)
    cr::DevBuf<NdFrontDev> fr;
    cr::DevBuf<int32_t> nodes, map;
    cr::DevBuf<double> finv, w, wt, bi, u;
    cr::DevBuf<double> fs, wts, ws;            // solve layouts (see NdFrontDev)
    cr::DevBuf<double> lb;                     // forward: local right-hand side on B
    cr::DevBuf<int64_t> invp;                  // per front local unknown: CSR offsets into invl
    cr::DevBuf<int32_t> invl, kids;            // children's u indices landing on it; child front lists
    cr::DevBuf<int32_t> uidx;                  // per front: global unknown of each local unknown
    cr::DevBuf<int2> la, lbr, lc;              // (front, local index) work lists by level
    std::vector<int> aoff, boff, coff;         // level offsets into la / lbr / lc
    std::vector<int> gb;                       // lanes per B row of each forward level
    cr::DevBuf<int2> lg;                       // backward: (front, b) entries of the y_B gathers by depth
    std::vector<int> goff;                     // depth offsets into lg
    cr::DevBuf<double> yb;                     // gathered y_B of every front
    cr::DevBuf<unsigned> bar;                  // grid barrier of the persistent solve kernel
    int grid = 0;
};

// two-level coarse correction (coarse.cu)
struct CoarseOp {
    int built = 0;               // H it was built for (0 = not built)
    double weight = 1.0;         // theta: relative weight of the coarse term in the additive preconditioner
    int absmode = 0;             // 1: Einv = |E|^{-1} (eigendecomposition; MINRES on the indefinite G)
    int requested = 0;           // H asked for when it was built
    cr::CoarseGrid g;
    int64_t nE = 0, nchunk = 0;
    cr::DevBuf<float> fx, fa, fxp, fap;
    cr::DevBuf<int32_t> perm;
    cr::DevBuf<int64_t> chunk_start, cell_chunk;
    cr::DevBuf<double> part, c, y, Einv;
    cr::DevBuf<double> gpart;    // block partials of the coarse GEMV (its own: it runs concurrently)
    CoarseNd nd;                 // sparse direct solve (default); Einv (dense inverse) when off
    // the solve order (cr_hybrid_s::so): sorted position -> solve-order row, per-row data by solve-order row
    cr::DevBuf<int32_t> perm_so;
    cr::DevBuf<float> fx_so, fa_so;
    cr::CoarseView view() const {
        return cr::CoarseView{g, fx.get(), fa.get(), perm.get(), fxp.get(), fap.get(), chunk_start.get(), cell_chunk.get(), nE};
    }
    cr::CoarseView view_so() const {
        return cr::CoarseView{g, fx_so.get(), fa_so.get(), perm_so.get(), fxp.get(), fap.get(), chunk_start.get(),
                              cell_chunk.get(), nE};
    }
};

// matrix-free factored G (mf.cuh layout)
struct MfOp {
    bool built = false;
    int64_t ncells = 0;          // padded to a multiple of 32
    cr::DevBuf<int32_t> ids;
    cr::DevBuf<int32_t> ids_so;  // ids in the solve order (cr_hybrid_s::so)
    cr::DevBuf<uint8_t> sg;
    cr::DevBuf<double> v;
    cr::DevBuf<uint8_t> nb;      // in-warp face partners (mf.cuh)
    cr::DevBuf<int32_t> slot;    // [nc] slot t of cell K (-1: not stored on this rank)
};

struct cr_hybrid_s {
    const cr_mesh_s *mesh = nullptr;
    cr_params prm{};
    int is_ns = 0;
    // owned copies of the problem data (recovery needs them again)
    cr::DevBuf<double> fbar, dir, uit, pit;
    bool has_dir = false, has_uit = false, has_pit = false;
    cr::DevBuf<double> rcell, gcell;   // explicit cell right-hand sides (dc.cu), empty unless set
    cr::DevBuf<double> uhat;           // recovery scratch: per-cell copies of U
    // shift
    cr::DevBuf<uint8_t> inM1;
    cr::DevBuf<double> lam, E;   // lam [nc], E [nc][d+1]
    // G, S, preconditioners
    BlockEll G;
    cr::DevBuf<double> S, dinv, absdinv, bdinv;   // bdinv [nrows][d][d] inverse diagonal blocks
    cr::DevBuf<uint8_t> rowlen;                   // true blocks per block row
    AfwPrec afw;
    MfOp mf;
    CoarseOp coarse;
    // Solve order: the face rows renumbered in the order the matrix-free cells visit them (a row's
    // position = the first (cell, local face) slot touching it), so that the gathers of the
    // iteration's kernels (p at a cell's faces, r at a patch's faces) read nearby rows.  Built for
    // the matrix-free patch-preconditioned PCG on one GPU; the solve permutes S, W in and W out,
    // every other entry point keeps the mesh's face order.
    struct {
        bool built = false;
        cr::DevBuf<int32_t> perm, iperm;   // solve-order row -> row, row -> solve-order row
    } so;
    cr::Part part;               // row partition (multi-GPU); part.on == false on one GPU
    cr_comm_s *comm = nullptr;   // borrowed
    cr::SolverWork *work = nullptr;
    ~cr_hybrid_s();
};

struct cr_coupled_s {
    int64_t n_rows = 0, nnz = 0;
    cr::DevBuf<int64_t> row_ptr;
    cr::DevBuf<int32_t> cols;
    cr::DevBuf<double> vals, rhs;
};

struct cr_comm_s {
    int rank = 0, nranks = 1;
    cr::Comm *impl = nullptr;   // null for a single rank
};

namespace cr {
// mesh.cu
void build_mesh(cr_mesh_s *m, int dim, int64_t nv, const double *coords, int64_t nc,
                const int32_t *cells, cudaStream_t s);
// hybrid.cu
void hybridise(cr_hybrid_s *h, const cr_mesh_s *m, const cr_params &prm, const cr_data &data, cr_comm_s *comm,
               cudaStream_t s);
void hybrid_update_rhs(cr_hybrid_s *h, cudaStream_t s);   // recompute S only (same G)
void transient_rhs(const cr_hybrid_s *h, const double *Uprev, double *R, double *g, cudaStream_t s);
void cell_face_values(const cr_mesh_s *m, const double *U, const double *bnd, double *out, cudaStream_t s);
// dc.cu
void solve_dc(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep);
void coupled_spmv(const cr_coupled_s *c, const double *x, double *y, cudaStream_t s);
// partition.cu
void setup_part(cr_hybrid_s *h, const cr_mesh_s *m, cr_comm_s *comm, cudaStream_t s);
void hybrid_export_csr(const cr_hybrid_s *h, int64_t *row_ptr, int32_t *cols, double *vals, double *S,
                       cudaStream_t s);
void assemble_coupled(cr_coupled_s *c, const cr_mesh_s *m, const cr_params &prm, const cr_data &data,
                      cudaStream_t s);
void spmv(const BlockEll &G, const double *x, double *y, cudaStream_t s);
// recover.cu
void recover(const cr_hybrid_s *h, const double *W, double *U, double *P, double *diag, cudaStream_t s);
void newton_update(int64_t nU, double *U, const double *dU, int64_t nP, double *P, const double *dP, double lam,
                   double *norms, cudaStream_t s);
// refine.cu: ||a||_2 of a device vector (fixed-order block partials: deterministic), host result
double norm2(const double *a, int64_t n, cudaStream_t s);
// solve.cu
void solve(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep);
void solve_profile(cr_hybrid_s *h, const cr_solver_opts &o, int nrep, double *ms, cudaStream_t s);
// one solve of G W = rhs (rhs NULL: S) with the fp64 solvers (solve.cu)
void solve_rhs(cr_hybrid_s *h, const cr_solver_opts &o, double *W, cudaStream_t s, cr_solve_report *rep,
               const double *rhs);
// refine.cu: r = S - G W with G W summed in double-double (the assembled G, or the matrix-free
// factors when `mf`); returns ||r||_2 and ||S||_2 (host)
void residual_dd(cr_hybrid_s *h, bool mf, const double *W, double *r, double *rnorm, double *snorm, cudaStream_t s);
void free_solver_work(SolverWork *w);
void apply_precond(cr_hybrid_s *h, int method, const double *r, double *z, cudaStream_t s);
void spmv_part(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s);
void spmv_mf(cr_hybrid_s *h, const double *x, double *y, cudaStream_t s);
// precond.cu
void build_afw(cr_hybrid_s *h, int mode, cudaStream_t s);
// mf.cu
void build_mf(cr_hybrid_s *h, cudaStream_t s);
// the solve order h->so from the matrix-free cell order, and mf.ids_so (mf.cu)
void build_so(cr_hybrid_s *h, cudaStream_t s);
// afw.ids_so from afw.ids (precond.cu)
void afw_so(cr_hybrid_s *h, cudaStream_t s);
// coarse.cu
// applyG(z, Y, colour, ncol, stride): Y_c = G z_c for the ncol vectors z_c = z + c stride, each a
// colour sum of coarse columns (colour < 0: any z; Y arrives zero on the rows G z can reach)
using ApplyG = std::function<void(const double *, double *, int, int, int64_t)>;
// applyGc(colour, Y, stride) (optional, single rank): Y_(k D + l) = G z_(k,l) for the D^2 columns of
// `colour` computed without materialising z (Y arrives zero)
using ApplyGColour = std::function<void(int, double *, int64_t)>;
void build_coarse(cr_hybrid_s *h, int H, const ApplyG &applyG, const ApplyGColour &applyGc,
                  cudaStream_t s, bool absmode = false);
void coarse_restrict_solve(cr_hybrid_s *h, const double *r, double *qout, double *partials, unsigned *ticket,
                           cudaStream_t s, bool side = false, bool so = false);
// the coarse space's solve-order copies (perm_so, fx_so, fa_so) once h->so is built
void coarse_so(cr_hybrid_s *h, cudaStream_t s);
// shared: copy problem data into hybrid-owned buffers
struct ProbView;
ProbView prob_view(const cr_hybrid_s *h);
void copy_problem_data(cr_hybrid_s *h, const cr_mesh_s *m, const cr_data &data, cudaStream_t s);
}  // namespace cr
