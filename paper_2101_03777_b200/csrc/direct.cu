// cr_sparse_direct_solve: sparse direct solve of a canonical CSR system on the GPU with cuSOLVER
// (dlopen'ed libcusolver.so.11 / libcusparse.so.12: plain library factorisations, like cuBLAS).
// It reproduces the paper's direct-solver comparison (Table 4): the hybrid system G is
// SPD -> sparse Cholesky; the coupled saddle matrix is symmetric indefinite ->
// sparse QR.  Used by bench.py's `direct_table4` and its tests only; the iterative path does not
// depend on it.
#include <dlfcn.h>

#include "internal.cuh"

namespace cr {
namespace {

struct SpSolver {
    void *hs = nullptr, *hp = nullptr, *handle = nullptr, *descr = nullptr;
    int (*Create)(void **) = nullptr;
    int (*SetStream)(void *, cudaStream_t) = nullptr;
    int (*Chol)(void *, int, int, void *, const double *, const int *, const int *, const double *, double, int,
                double *, int *) = nullptr;
    int (*Qr)(void *, int, int, void *, const double *, const int *, const int *, const double *, double, int,
              double *, int *) = nullptr;
    int (*CreateDescr)(void **) = nullptr;
    int (*SetType)(void *, int) = nullptr;
    int (*SetBase)(void *, int) = nullptr;
};

SpSolver &sp() {
    static thread_local SpSolver S = [] {
        SpSolver x;
        x.hp = dlopen("libcusparse.so.12", RTLD_NOW | RTLD_GLOBAL);
        x.hs = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!x.hs || !x.hp) return x;
        x.Create = (decltype(x.Create))dlsym(x.hs, "cusolverSpCreate");
        x.SetStream = (decltype(x.SetStream))dlsym(x.hs, "cusolverSpSetStream");
        x.Chol = (decltype(x.Chol))dlsym(x.hs, "cusolverSpDcsrlsvchol");
        x.Qr = (decltype(x.Qr))dlsym(x.hs, "cusolverSpDcsrlsvqr");
        x.CreateDescr = (decltype(x.CreateDescr))dlsym(x.hp, "cusparseCreateMatDescr");
        x.SetType = (decltype(x.SetType))dlsym(x.hp, "cusparseSetMatType");
        x.SetBase = (decltype(x.SetBase))dlsym(x.hp, "cusparseSetMatIndexBase");
        if (!(x.Create && x.SetStream && x.Chol && x.Qr && x.CreateDescr && x.SetType && x.SetBase)) return x;
        if (x.Create(&x.handle) != 0 || x.CreateDescr(&x.descr) != 0) {
            x.handle = nullptr;
            return x;
        }
        x.SetType(x.descr, 0);   // CUSPARSE_MATRIX_TYPE_GENERAL
        x.SetBase(x.descr, 0);   // CUSPARSE_INDEX_BASE_ZERO
        return x;
    }();
    return S;
}

__global__ void k_rowptr32(int64_t n, const int64_t *in, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)in[i];
}

}  // namespace
}  // namespace cr

extern "C" cr_status cr_sparse_direct_solve(int64_t n, int64_t nnz, const int64_t *row_ptr_d, const int32_t *cols_d,
                                            const double *vals_d, const double *b_d, double *x_d, int32_t method,
                                            int32_t reorder, cr_stream_t s, int32_t *singularity) {
    try {
        CR_REQUIRE(n > 0 && nnz > 0 && nnz < ((int64_t)1 << 31) && row_ptr_d && cols_d && vals_d && b_d && x_d,
                   CR_ERR_INVALID_ARG, "bad arguments");
        CR_REQUIRE(method == 0 || method == 1, CR_ERR_INVALID_ARG, "method: 0 Cholesky, 1 QR");
        CR_REQUIRE(reorder >= 0 && reorder <= 3, CR_ERR_INVALID_ARG, "reorder: 0 none, 1 symrcm, 2 symamd, 3 metis");
        cr::SpSolver &S = cr::sp();
        CR_REQUIRE(S.handle, CR_ERR_CUDA, "cuSOLVER sparse (libcusolver.so.11 / libcusparse.so.12) unavailable");
        cudaStream_t st = (cudaStream_t)s;
        cr::DevBuf<int32_t> rp;
        rp.alloc(n + 1, st);
        cr::k_rowptr32<<<cr::grid_for(n + 1, 256), 256, 0, st>>>(n, row_ptr_d, rp.get());
        CR_CHECK_LAUNCH();
        S.SetStream(S.handle, st);
        int sing = -1;
        const int rc = method == 0
                           ? S.Chol(S.handle, (int)n, (int)nnz, S.descr, vals_d, rp.get(), cols_d, b_d, 1e-14, reorder, x_d, &sing)
                           : S.Qr(S.handle, (int)n, (int)nnz, S.descr, vals_d, rp.get(), cols_d, b_d, 1e-14, reorder, x_d, &sing);
        CR_CUDA(cudaStreamSynchronize(st));
        if (singularity) *singularity = sing;
        CR_REQUIRE(rc == 0, CR_ERR_CUDA, "cusolverSp csrlsv failed");
        CR_REQUIRE(sing < 0, CR_ERR_SINGULAR_LOCAL, "matrix singular to the direct solver's tolerance");
        return CR_OK;
    } catch (const cr::Error &e) {
        cr::set_last_error(e.what());
        return e.code;
    } catch (const std::exception &e) {
        cr::set_last_error(e.what());
        return CR_ERR_INVALID_ARG;
    }
}
