// Communicators for the partitioned path.
//
// Three collectives are all the hybrid method needs across ranks:
//   allreduce  — the Krylov dot products (a handful of doubles per reduction),
//   halo       — ghost entries of the SpMV input vector from the peers that own them,
//   allgatherv — the solution W for the per-cell recovery (once per solve).
//
// NcclComm    one process per GPU; NCCL is loaded with dlopen (libnccl.so.2, the copy torch
//             already mapped when it is imported), so libcr itself loads on a CPU-only box.
//             Every call is enqueued on the caller's stream, so the solver's CUDA graphs
//             capture them.
// LoopComm    R ranks as R host threads of ONE process on one GPU (tests): the exchange goes
//             through device-to-device copies between the ranks' buffers and fixed-order host
//             sums, with host barriers between phases.  Nothing waits on the device for
//             another rank, and nothing is captured into graphs (capturable() == false).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.cuh"

namespace cr {

// ------------------------------------------------------------------ NCCL through dlopen
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, void *) = nullptr;
};

static NcclApi &nccl() {
    static NcclApi a = [] {
        NcclApi n;
        n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) return n;
        n.GetUniqueId = (decltype(n.GetUniqueId))dlsym(n.h, "ncclGetUniqueId");
        n.CommInitRank = (decltype(n.CommInitRank))dlsym(n.h, "ncclCommInitRank");
        n.CommDestroy = (decltype(n.CommDestroy))dlsym(n.h, "ncclCommDestroy");
        n.AllReduce = (decltype(n.AllReduce))dlsym(n.h, "ncclAllReduce");
        n.Send = (decltype(n.Send))dlsym(n.h, "ncclSend");
        n.Recv = (decltype(n.Recv))dlsym(n.h, "ncclRecv");
        n.GroupStart = (decltype(n.GroupStart))dlsym(n.h, "ncclGroupStart");
        n.GroupEnd = (decltype(n.GroupEnd))dlsym(n.h, "ncclGroupEnd");
        n.GetErrorString = (decltype(n.GetErrorString))dlsym(n.h, "ncclGetErrorString");
        n.CommSplit = (decltype(n.CommSplit))dlsym(n.h, "ncclCommSplit");
        return n;
    }();
    CR_REQUIRE(a.h && a.CommInitRank && a.AllReduce && a.Send && a.Recv, CR_ERR_NCCL,
               "libnccl.so.2 could not be loaded (import torch first, or put NCCL on the library path)");
    return a;
}

#define CR_NCCL(call)                                                                                     \
    do {                                                                                                  \
        ncclResult_t r_ = (call);                                                                         \
        if (r_ != ncclSuccess)                                                                            \
            throw ::cr::Error(CR_ERR_NCCL, std::string(#call) + ": " +                                    \
                                               (nccl().GetErrorString ? nccl().GetErrorString(r_) : "?")); \
    } while (0)

struct NcclComm : Comm {
    ncclComm_t c = nullptr;
    // a second communicator over the same ranks (ncclCommSplit) for the coarse path, which runs on
    // its own stream concurrently with the fine-level kernels: collectives of ONE communicator
    // must be issued in the same order on every rank, which two streams would not guarantee
    ncclComm_t side = nullptr;
    bool capturable() const override { return true; }
    bool has_side() const override { return side != nullptr; }
    void allreduce(double *d, int n, bool mx, cudaStream_t s) override {
        CR_NCCL(nccl().AllReduce(d, d, (size_t)n, ncclDouble, mx ? ncclMax : ncclSum, c, s));
    }
    void allreduce_side(double *d, int n, cudaStream_t s) override {
        CR_NCCL(nccl().AllReduce(d, d, (size_t)n, ncclDouble, ncclSum, side ? side : c, s));
    }
    void halo(const Part &P, const double *sendbuf, double *xghost, int D, cudaStream_t s) override {
        CR_NCCL(nccl().GroupStart());
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            if (P.scount[q]) CR_NCCL(nccl().Send(sendbuf + P.soff[q] * D, (size_t)(P.scount[q] * D), ncclDouble, q, c, s));
            if (P.rcount[q]) CR_NCCL(nccl().Recv(xghost + P.roff[q] * D, (size_t)(P.rcount[q] * D), ncclDouble, q, c, s));
        }
        CR_NCCL(nccl().GroupEnd());
    }
    void allgatherv(const double *local, double *full, const std::vector<int64_t> &cnt, const std::vector<int64_t> &dsp,
                    cudaStream_t s) override {
        CR_CUDA(cudaMemcpyAsync(full + dsp[rank], local, cnt[rank] * sizeof(double), cudaMemcpyDeviceToDevice, s));
        CR_NCCL(nccl().GroupStart());
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            if (cnt[rank]) CR_NCCL(nccl().Send(local, (size_t)cnt[rank], ncclDouble, q, c, s));
            if (cnt[q]) CR_NCCL(nccl().Recv(full + dsp[q], (size_t)cnt[q], ncclDouble, q, c, s));
        }
        CR_NCCL(nccl().GroupEnd());
    }
    ~NcclComm() override {
        if (side && nccl().CommDestroy) nccl().CommDestroy(side);
        if (c && nccl().CommDestroy) nccl().CommDestroy(c);
    }
};

// ------------------------------------------------------------------ in-process loopback
struct LoopGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<std::vector<double>> red;                 // per rank: its local reduction values
    std::vector<const double *> buf;                      // per rank: send buffer / local W
    std::vector<std::vector<int64_t>> soff, scount;       // per rank: its send table (rows)
    explicit LoopGroup(int n_) : n(n_), red(n_), buf(n_, nullptr), soff(n_), scount(n_) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == n) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LoopComm : Comm {
    LoopGroup *g = nullptr;
    bool capturable() const override { return false; }
    void allreduce(double *d, int n, bool mx, cudaStream_t s) override {
        std::vector<double> v(n);
        CR_CUDA(cudaMemcpyAsync(v.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        CR_CUDA(cudaStreamSynchronize(s));
        g->red[rank] = v;
        g->barrier();
        std::vector<double> acc = g->red[0];
        for (int q = 1; q < nranks; ++q)      // fixed rank order: identical on every rank
            for (int i = 0; i < n; ++i) acc[i] = mx ? fmax(acc[i], g->red[q][i]) : acc[i] + g->red[q][i];
        CR_CUDA(cudaMemcpyAsync(d, acc.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void halo(const Part &P, const double *sendbuf, double *xghost, int D, cudaStream_t s) override {
        CR_CUDA(cudaStreamSynchronize(s));
        g->buf[rank] = sendbuf;
        g->soff[rank] = P.soff;
        g->scount[rank] = P.scount;
        g->barrier();
        for (int q = 0; q < nranks; ++q) {
            if (q == rank || !P.rcount[q]) continue;
            CR_REQUIRE(g->scount[q][rank] == P.rcount[q], CR_ERR_INVALID_ARG, "halo plan mismatch between ranks");
            CR_CUDA(cudaMemcpyAsync(xghost + P.roff[q] * D, g->buf[q] + g->soff[q][rank] * D,
                                    P.rcount[q] * D * sizeof(double), cudaMemcpyDeviceToDevice, s));
        }
        CR_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
    void allgatherv(const double *local, double *full, const std::vector<int64_t> &cnt, const std::vector<int64_t> &dsp,
                    cudaStream_t s) override {
        CR_CUDA(cudaStreamSynchronize(s));
        g->buf[rank] = local;
        g->barrier();
        for (int q = 0; q < nranks; ++q)
            if (cnt[q])
                CR_CUDA(cudaMemcpyAsync(full + dsp[q], g->buf[q], cnt[q] * sizeof(double), cudaMemcpyDeviceToDevice, s));
        CR_CUDA(cudaStreamSynchronize(s));
        g->barrier();
    }
};

}  // namespace cr

struct cr_loopback_s {
    cr::LoopGroup g;
    explicit cr_loopback_s(int n) : g(n) {}
};

#define CR_TRY try {
#define CR_CATCH                                 \
    return CR_OK;                                \
    }                                            \
    catch (const cr::Error &e) {                 \
        cr::set_last_error(e.what());            \
        return e.code;                           \
    }                                            \
    catch (const std::exception &e) {           \
        cr::set_last_error(e.what());            \
        return CR_ERR_NCCL;                      \
    }

extern "C" {

cr_status cr_nccl_unique_id(void *out128) {
    CR_TRY
    CR_REQUIRE(out128, CR_ERR_INVALID_ARG, "null argument");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    {
        using cr::nccl;
        CR_NCCL(cr::nccl().GetUniqueId(&id));
    }
    memcpy(out128, &id, sizeof(id));
    CR_CATCH
}

cr_status cr_comm_init(const void *nccl_unique_id, int32_t rank, int32_t nranks, cr_comm *out) {
    CR_TRY
    CR_REQUIRE(out && nranks >= 1 && rank >= 0 && rank < nranks, CR_ERR_INVALID_ARG, "bad communicator arguments");
    *out = nullptr;
    cr_comm_s *c = new cr_comm_s();
    c->rank = rank;
    c->nranks = nranks;
    // with a unique id the communicator is NCCL-backed even for one rank (hybrids built with it
    // take the partitioned path: used to exercise the NCCL calls inside the solver graphs)
    if (nranks > 1 || nccl_unique_id) {
        CR_REQUIRE(nccl_unique_id, CR_ERR_INVALID_ARG, "nranks > 1 needs the NCCL unique id of rank 0");
        auto *nc = new cr::NcclComm();
        nc->rank = rank;
        nc->nranks = nranks;
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof(id));
        try {
            using cr::nccl;
            CR_NCCL(cr::nccl().CommInitRank(&nc->c, nranks, id, rank));
            // the coarse path's communicator (collective over all ranks; absent: no overlap)
            if (cr::nccl().CommSplit && cr::nccl().CommSplit(nc->c, 0, rank, &nc->side, nullptr) != ncclSuccess)
                nc->side = nullptr;
        } catch (...) {
            delete nc;
            delete c;
            throw;
        }
        c->impl = nc;
    }
    *out = c;
    CR_CATCH
}

cr_status cr_loopback_create(int32_t nranks, cr_loopback *out) {
    CR_TRY
    CR_REQUIRE(out && nranks >= 1, CR_ERR_INVALID_ARG, "bad arguments");
    *out = new cr_loopback_s(nranks);
    CR_CATCH
}

void cr_loopback_destroy(cr_loopback g) { delete g; }

cr_status cr_comm_init_loopback(cr_loopback g, int32_t rank, cr_comm *out) {
    CR_TRY
    CR_REQUIRE(g && out && rank >= 0 && rank < g->g.n, CR_ERR_INVALID_ARG, "bad arguments");
    cr_comm_s *c = new cr_comm_s();
    c->rank = rank;
    c->nranks = g->g.n;
    auto *lc = new cr::LoopComm();
    lc->rank = rank;
    lc->nranks = g->g.n;
    lc->g = &g->g;
    c->impl = lc;
    *out = c;
    CR_CATCH
}

void cr_comm_destroy(cr_comm c) {
    if (!c) return;
    delete c->impl;
    delete c;
}

}  // extern "C"
