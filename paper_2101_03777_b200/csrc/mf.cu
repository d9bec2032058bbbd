// Setup of the matrix-free factored operator (layout and algebra in mf.cuh).  One thread per
// cell recomputes the cell's elimination in double-double (the same LDL^t as the assembly,
// local.cuh), forms Shat_K^{-1} column by column, splits off the 1/(mu|K|) 1 1^t part for
// cells with all faces interior (transient), scales w by 1/sqrt(B_K), and rounds once.
#include <cub/cub.cuh>
#include <cmath>
#include <cstdlib>

#include "local.cuh"
#include "mf.cuh"

namespace cr {

// cells with at least one owned interior face (all cells when not partitioned)
template <int D>
__global__ void k_mf_flag(MeshView mv, int64_t nc, int64_t row0, int64_t row1, uint8_t *flag) {
    constexpr int NF = D + 1;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nc; K += (int64_t)gridDim.x * blockDim.x) {
        uint8_t f = 0;
#pragma unroll
        for (int l = 0; l < NF; ++l) {
            const int dof = mv.face_dof[mv.cell_faces[K * NF + l]];
            if (dof >= row0 && dof < row1) f = 1;
        }
        flag[K] = f;
    }
}

template <int D>
__global__ void __launch_bounds__(128) k_mf_build(MeshView mv, ProbView p, const int32_t *cells, int64_t ncell,
                                                  const int32_t *g2l, int32_t *ids, uint8_t *sg, double *v, int *err) {
    using LY = MfLayout<D>;
    constexpr int NF = LY::NF, NT = LY::NT, NE = LY::NE;
    const int64_t npad = ((ncell + 31) >> 5) << 5;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npad; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slice = t >> 5;
        const int lane = (int)(t & 31);
        int32_t *ip = ids + slice * (NF * 32) + lane;
        double *vp = v + slice * ((int64_t)NE * 32) + lane;
        if (t >= ncell) {   // padding lane of the last slice: no faces, zero operator
            for (int l = 0; l < NF; ++l) ip[l * 32] = -1;
            sg[t] = 0;
            for (int e = 0; e < NE; ++e) vp[e * 32] = 0.0;
            continue;
        }
        const int64_t K = cells[t];
        Cell<D> c;
        load_cell<D>(mv, K, c);
        StokesElim<D> e;
        stokes_eliminate<D>(c, p, e);
        if (e.status != DE_OK) { atomicCAS(err, DE_OK, e.status); continue; }
        unsigned mask = 0;
        for (int l = 0; l < NF; ++l) {
            const int dof = c.dof[l];
            ip[l * 32] = dof < 0 ? -1 : (g2l ? g2l[dof] : dof);
            if (c.C[l] < 0) mask |= 1u << l;
        }
        sg[t] = (uint8_t)mask;
        // Shat^{-1} (compact s x s) by solves with unit vectors, expanded to local faces
        dd Si[NF][NF];
        for (int a = 0; a < NF; ++a)
            for (int b = 0; b < NF; ++b) Si[a][b] = dd_of(0.0);
        for (int q = 0; q < c.s; ++q) {
            dd col[NF];
            for (int r = 0; r < c.s; ++r) col[r] = dd_of(r == q ? 1.0 : 0.0);
            ldl_solve<D>(e, c.s, col);
            for (int r = 0; r < c.s; ++r) Si[c.map[r]][c.map[q]] = col[r];
        }
        const bool split = (c.s == NF) && p.mu > 0.0 && !p.E;
        dd cb = dd_of(0.0);
        if (split) cb = dd_of(1.0) / (two_prod(p.mu, c.vol));   // 1/(alpha (d+1)), alpha = mu|K|/(d+1)
        vp[0] = dd_round(cb);
        for (int a = 0; a < NF; ++a)
            for (int b = 0; b <= a; ++b) vp[(1 + a * (a + 1) / 2 + b) * 32] = dd_round(Si[a][b] - cb);
        // u = w / sqrt(B) (K0: no pressure unknown, no projection)
        const bool k0 = (K == p.k0);
        dd sq = dd_of(0.0);
        if (!k0) {
            const double s0 = sqrt(e.B.hi);
            sq = dd_of(s0) + (e.B - two_prod(s0, s0)) / (2.0 * s0);   // one Newton step in dd
        }
        for (int i = 0; i < D; ++i)
            for (int l = 0; l < NF; ++l) vp[(1 + NT + i * NF + l) * 32] = 0.0;
        if (!k0)
            for (int i = 0; i < D; ++i)
                for (int q = 0; q < c.s; ++q) vp[(1 + NT + i * NF + c.map[q]) * 32] = dd_round(e.w[i][q] / sq);
    }
}

__global__ void k_mf_slot(const int32_t *list, int64_t n, int32_t *slot) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        slot[list[t]] = (int32_t)t;
}

// nb code of (slot t, local face l): the other cell of the face, if stored in the same 32-slot slice
template <int D>
__global__ void k_mf_partners(MeshView mv, const int32_t *list, int64_t ncell, int64_t npad, const int32_t *slot,
                              uint8_t *nb) {
    constexpr int NF = D + 1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < npad; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slice = t >> 5;
        const int lane = (int)(t & 31);
        for (int l = 0; l < NF; ++l) {
            uint8_t code = 0;
            if (t < ncell) {
                const int64_t K = list[t];
                const int64_t f = mv.cell_faces[K * NF + l];
                const int64_t c0 = mv.face_cells[2 * f], c1 = mv.face_cells[2 * f + 1];
                if (c1 >= 0 && mv.face_dof[f] >= 0) {
                    const int64_t L = (c0 == K) ? c1 : c0;
                    const int64_t tL = slot[L];
                    if (tL >= 0 && (tL >> 5) == slice) {
                        int lp = 0;
                        for (int q = 0; q < NF; ++q)
                            if (mv.cell_faces[L * NF + q] == (int32_t)f) lp = q;
                        code = (uint8_t)(0x80u | ((unsigned)lp << 5) | (unsigned)(tL & 31));
                    }
                }
            }
            nb[slice * (NF * 32) + l * 32 + lane] = code;
        }
    }
}

// Morton key of a cell centroid (21 bits per direction in 3D, 31 in 2D) inside the mesh bounding box
__device__ __forceinline__ uint64_t spread2(uint64_t v) {   // 32 -> 64 bits, one zero between bits
    v &= 0xffffffffull;
    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}
__device__ __forceinline__ uint64_t spread3(uint64_t v) {   // 21 -> 63 bits, two zeros between bits
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}
// lex = 0: Morton (Z-order) key; lex = 1: lexicographic key (last coordinate most significant: the
// order in which the face numbering sweeps the mesh); lex = 2: blocks of 2^-bb of the box in
// lexicographic order, Morton inside a block (compact warps for the in-warp face pairing, and a
// sweep whose working set of x / q is a slab of blocks: the two cells of a face are processed close
// in time)
template <int D>
__global__ void k_mf_morton(const double *xK, const int32_t *list, int64_t n, const double *lo, const double *hi,
                            uint64_t *key, int lex, int bb) {
    constexpr int QB = D == 2 ? 31 : 21;   // bits per coordinate
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t K = list[t];
        uint64_t k = 0, blk = 0, in = 0;
        for (int i = 0; i < D; ++i) {
            const double w = hi[i] - lo[i];
            const double u = w > 0 ? (xK[K * D + i] - lo[i]) / w : 0.0;
            const double scale = D == 2 ? 2147483647.0 : 2097151.0;
            const uint64_t q = (uint64_t)fmin(fmax(u * scale, 0.0), scale);
            if (lex == 1) k |= q << (i * QB);
            else if (lex == 0) k |= (D == 2 ? spread2(q) : spread3(q)) << i;
            else {
                blk |= (q >> (QB - bb)) << (i * bb);
                const uint64_t qi = q & ((1ull << (QB - bb)) - 1);
                in |= (D == 2 ? spread2(qi) : spread3(qi)) << i;
            }
        }
        key[t] = lex == 2 ? (blk << (D * (QB - bb))) | in : k;
    }
}

template <int D>
static void build_mf_t(cr_hybrid_s *h, cudaStream_t s) {
    using LY = MfLayout<D>;
    const cr_mesh_s *m = h->mesh;
    MfOp &M = h->mf;
    const int64_t nc = m->nc;
    const int T = 256;
    MeshView mv = mesh_view(m);
    ProbView p = prob_view(h);
    const int64_t row0 = h->part.on ? h->part.row0 : 0, row1 = h->part.on ? h->part.row1 : m->nf_int;
    DevBuf<uint8_t> flag;
    flag.alloc(nc, s);
    k_mf_flag<D><<<grid_for(nc, T), T, 0, s>>>(mv, nc, row0, row1, flag.get());
    CR_CHECK_LAUNCH();
    DevBuf<int32_t> list;
    list.alloc(nc, s);
    DevBuf<int64_t> nsel;
    nsel.alloc(1, s);
    size_t tb = 0;
    cub::CountingInputIterator<int32_t> it(0);
    CR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag.get(), list.get(), nsel.get(), (int64_t)nc, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, s);
    CR_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, flag.get(), list.get(), nsel.get(), (int64_t)nc, s));
    int64_t ncell = 0;
    CR_CUDA(cudaMemcpyAsync(&ncell, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    {
        // cells in Morton order of their centroids: a 32-cell warp covers a compact block (4 x 4
        // squares in 2D), so most of its faces are shared inside the warp (summed in registers)
        // instead of needing an atomic from each side
        DevBuf<double> lo, hi, comp;
        lo.alloc(D, s); hi.alloc(D, s); comp.alloc(nc, s);
        for (int i = 0; i < D; ++i) {
            CR_CUDA(cudaMemcpy2DAsync(comp.get(), sizeof(double), m->xK.get() + i, D * sizeof(double), sizeof(double), nc,
                                      cudaMemcpyDeviceToDevice, s));
            size_t tr = 0;
            CR_CUDA(cub::DeviceReduce::Min(nullptr, tr, comp.get(), lo.get() + i, (int)nc, s));
            DevBuf<uint8_t> rt;
            rt.alloc(tr, s);
            CR_CUDA(cub::DeviceReduce::Min(rt.get(), tr, comp.get(), lo.get() + i, (int)nc, s));
            CR_CUDA(cub::DeviceReduce::Max(rt.get(), tr, comp.get(), hi.get() + i, (int)nc, s));
        }
        DevBuf<uint64_t> key, key2;
        DevBuf<int32_t> list2;
        key.alloc(ncell, s); key2.alloc(ncell, s); list2.alloc(ncell, s);
        // CR_MF_ORDER: "lex" lexicographic, "morton" Morton; default: lexicographic blocks of ~4 mesh
        // cells per side (2^bb blocks per direction) with Morton inside (3D apply 0.958 vs 0.992 ms)
        static const char *eo = std::getenv("CR_MF_ORDER");
        const int lex = (eo && eo[0] == 'l') ? 1 : (eo && eo[0] == 'm') ? 0 : 2;   // default: blocks
        const double side = D == 2 ? std::sqrt((double)nc / 2.0) : std::cbrt((double)nc / 6.0);
        int bb = 1;
        while (bb < (D == 2 ? 30 : 20) && (double)(1 << (bb + 1)) <= side / 4.0) ++bb;
        static const char *ebb = std::getenv("CR_MF_BLOCK_BITS");
        if (ebb) bb = std::max(1, std::min(atoi(ebb), D == 2 ? 30 : 20));
        k_mf_morton<D><<<grid_for(ncell, T), T, 0, s>>>(m->xK.get(), list.get(), ncell, lo.get(), hi.get(), key.get(), lex,
                                                        bb);
        CR_CHECK_LAUNCH();
        size_t ts = 0;
        CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, ts, key.get(), key2.get(), list.get(), list2.get(), (int)ncell, 0,
                                                D == 2 ? 64 : 63, s));
        DevBuf<uint8_t> st;
        st.alloc(ts, s);
        CR_CUDA(cub::DeviceRadixSort::SortPairs(st.get(), ts, key.get(), key2.get(), list.get(), list2.get(), (int)ncell, 0,
                                                D == 2 ? 64 : 63, s));
        CR_CUDA(cudaMemcpyAsync(list.get(), list2.get(), ncell * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    }
    const int64_t nsl = (ncell + 31) / 32;
    M.ncells = nsl * 32;
    M.ids.alloc(nsl * 32 * LY::NF, s);
    M.sg.alloc(nsl * 32, s);
    M.v.alloc(nsl * 32 * LY::NE, s);
    DevBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    k_mf_build<D><<<grid_for(nsl * 32, 128, 16), 128, 0, s>>>(mv, p, list.get(), ncell,
                                                               h->part.on ? h->part.g2l.get() : nullptr, M.ids.get(),
                                                               M.sg.get(), M.v.get(), err.get());
    CR_CHECK_LAUNCH();
    // in-warp face partners
    DevBuf<int32_t> &slot = M.slot;   // kept: the dd residual (refine.cu) finds a cell's factors by it
    slot.alloc(nc, s);
    slot.fill_bytes(0xFF, s);
    k_mf_slot<<<grid_for(ncell, T), T, 0, s>>>(list.get(), ncell, slot.get());
    CR_CHECK_LAUNCH();
    M.nb.alloc(nsl * 32 * LY::NF, s);
    k_mf_partners<D><<<grid_for(nsl * 32, T), T, 0, s>>>(mv, list.get(), ncell, nsl * 32, slot.get(), M.nb.get());
    CR_CHECK_LAUNCH();
    int he = 0;
    CR_CUDA(cudaMemcpyAsync(&he, err.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    CR_REQUIRE(he == DE_OK, CR_ERR_SINGULAR_LOCAL, "local elimination failed while building the matrix-free operator");
    M.built = true;
}

// ------------------------------------------------------------------ solve order
// key of a row = the first stored (cell slot, local face) position touching it
template <int D>
__global__ void k_so_key(const int32_t *ids, int64_t npos, uint32_t *key) {
    constexpr int NF = D + 1;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npos; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = p / NF;
        const int l = (int)(p - t * NF);
        const int32_t id = ids[(t >> 5) * (NF * 32) + l * 32 + (t & 31)];
        if (id >= 0) atomicMin(key + id, (uint32_t)p);
    }
}
__global__ void k_so_inverse(const int32_t *perm, int64_t n, int32_t *iperm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        iperm[perm[i]] = (int32_t)i;
}
__global__ void k_so_map(const int32_t *in, int64_t n, const int32_t *iperm, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = in[i];
        out[i] = v >= 0 ? iperm[v] : -1;
    }
}
__global__ void k_iota_i32(int32_t *a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

template <int D>
static void build_so_t(cr_hybrid_s *h, cudaStream_t s) {
    constexpr int NF = D + 1;
    MfOp &M = h->mf;
    const int64_t nrows = h->G.nrows, npos = M.ncells * NF;
    CR_REQUIRE(npos < ((int64_t)1 << 32), CR_ERR_INVALID_ARG, "mesh too large for the solve order");
    const int T = 256;
    DevBuf<uint32_t> key, key2;
    DevBuf<int32_t> idx;
    key.alloc(nrows, s); key2.alloc(nrows, s); idx.alloc(nrows, s);
    key.fill_bytes(0xFF, s);
    k_so_key<D><<<grid_for(npos, T), T, 0, s>>>(M.ids.get(), npos, key.get());
    CR_CHECK_LAUNCH();
    k_iota_i32<<<grid_for(nrows, T), T, 0, s>>>(idx.get(), nrows);
    CR_CHECK_LAUNCH();
    h->so.perm.alloc(nrows, s);
    h->so.iperm.alloc(nrows, s);
    size_t tb = 0;
    CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), key2.get(), idx.get(), h->so.perm.get(), (int)nrows, 0,
                                            32, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, s);
    CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.get(), key2.get(), idx.get(), h->so.perm.get(), (int)nrows,
                                            0, 32, s));
    k_so_inverse<<<grid_for(nrows, T), T, 0, s>>>(h->so.perm.get(), nrows, h->so.iperm.get());
    CR_CHECK_LAUNCH();
    M.ids_so.alloc(M.ids.n, s);
    k_so_map<<<grid_for((int64_t)M.ids.n, T), T, 0, s>>>(M.ids.get(), (int64_t)M.ids.n, h->so.iperm.get(), M.ids_so.get());
    CR_CHECK_LAUNCH();
    h->so.built = true;
}

void build_so(cr_hybrid_s *h, cudaStream_t s) {
    if (h->so.built) return;
    CR_REQUIRE(h->mf.built && !h->part.on, CR_ERR_INVALID_ARG, "the solve order needs the matrix-free operator, one GPU");
    if (h->mesh->dim == 2) build_so_t<2>(h, s);
    else build_so_t<3>(h, s);
}

void build_mf(cr_hybrid_s *h, cudaStream_t s) {
    if (h->mf.built) return;
    CR_REQUIRE(!h->is_ns && h->prm.shift == CR_SHIFT_NONE && h->prm.mu > 0.0, CR_ERR_INVALID_ARG,
               "the matrix-free operator covers transient Stokes (mu > 0, no shift) only");
    if (h->mesh->dim == 2) build_mf_t<2>(h, s);
    else build_mf_t<3>(h, s);
}

}  // namespace cr
