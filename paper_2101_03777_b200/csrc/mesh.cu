// cr_build_mesh on the device (§2 item 1).
//
// K1 face_keys   : one key per (cell, local face) = the sorted vertex tuple of the face opposite
//                  local vertex l, packed in ceil(log2 nv) bits per vertex (one 64-bit key when
//                  d*bits <= 64, else an LSD two-pass sort: (v1,v2) then v0, both stable).
// K2 radix sort  : cub::DeviceRadixSort::SortPairs (stable) -> lexicographic face order; equal
//                  keys keep ascending (cell, l) order, so face_cells[f][0] < face_cells[f][1].
// K3 incidence   : run heads -> face ids (inclusive scan), faces, face_cells, cell_faces; a run
//                  of 3 equal tuples is a non-manifold input; interior faces -> face_dof (scan).
// K4 geometry    : |K|, x_K, a_{K,l} (from the SORTED tuple of face l, signed away from vertex l,
//                  no FMA contraction so the oracle's plain fp64 ops are reproduced), x_sigma.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace cr {

template <int D>
__device__ __forceinline__ void face_tuple(const int32_t *cells, int64_t c, int l, int32_t t[D]) {
    int k = 0;
#pragma unroll
    for (int v = 0; v < D + 1; ++v)
        if (v != l) t[k++] = cells[c * (D + 1) + v];
    // sort D <= 3 values
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j + 1 < D - i; ++j)
            if (t[j] > t[j + 1]) { int32_t x = t[j]; t[j] = t[j + 1]; t[j + 1] = x; }
}

__global__ void k_check_cells(const int32_t *cells, int64_t n, int64_t nv, int *err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = cells[i];
        if (v < 0 || v >= nv) atomicCAS(err, DE_OK, DE_RANGE);
    }
}

template <int D>
__global__ void k_face_keys(const int32_t *cells, int64_t nc, int bits, int pass_lo_only,
                            uint64_t *keys, uint32_t *vals) {
    int64_t n = nc * (D + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t c = i / (D + 1);
        int l = (int)(i - c * (D + 1));
        int32_t t[D];
        face_tuple<D>(cells, c, l, t);
        uint64_t k = 0;
        if (pass_lo_only) {      // two-pass: low part = last D-1 vertices
#pragma unroll
            for (int j = 1; j < D; ++j) k = (k << bits) | (uint64_t)t[j];
        } else {
#pragma unroll
            for (int j = 0; j < D; ++j) k = (k << bits) | (uint64_t)t[j];
        }
        keys[i] = k;
        vals[i] = (uint32_t)i;
    }
}

template <int D>
__global__ void k_first_vertex_keys(const int32_t *cells, int64_t n, const uint32_t *vals, uint64_t *keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = vals[i];
        int64_t c = v / (D + 1);
        int32_t t[D];
        face_tuple<D>(cells, c, (int)(v - c * (D + 1)), t);
        keys[i] = (uint64_t)t[0];
    }
}

template <int D>
__global__ void k_heads(const int32_t *cells, int64_t n, const uint32_t *vals, int32_t *head, int *err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = vals[i];
        int32_t t[D], u[D], w[D];
        face_tuple<D>(cells, v / (D + 1), v % (D + 1), t);
        int h = 1;
        if (i > 0) {
            uint32_t v1 = vals[i - 1];
            face_tuple<D>(cells, v1 / (D + 1), v1 % (D + 1), u);
            bool eq = true;
#pragma unroll
            for (int j = 0; j < D; ++j) eq = eq && (t[j] == u[j]);
            h = eq ? 0 : 1;
            if (eq && i > 1) {
                uint32_t v2 = vals[i - 2];
                face_tuple<D>(cells, v2 / (D + 1), v2 % (D + 1), w);
                bool eq2 = true;
#pragma unroll
                for (int j = 0; j < D; ++j) eq2 = eq2 && (t[j] == w[j]);
                if (eq2) atomicCAS(err, DE_OK, DE_NONMANIFOLD);
            }
        }
        head[i] = h;
    }
}

template <int D>
__global__ void k_incidence(const int32_t *cells, int64_t n, const uint32_t *vals, const int32_t *head,
                            const int32_t *fid_incl, int32_t *faces, int32_t *face_cells, int32_t *cell_faces) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = vals[i];
        int32_t c = (int32_t)(v / (D + 1));
        int l = v % (D + 1);
        int32_t f = fid_incl[i] - 1;
        cell_faces[v] = f;
        if (head[i]) {
            int32_t t[D];
            face_tuple<D>(cells, c, l, t);
#pragma unroll
            for (int j = 0; j < D; ++j) faces[(int64_t)f * D + j] = t[j];
            face_cells[2 * (int64_t)f] = c;
        } else {
            face_cells[2 * (int64_t)f + 1] = c;
        }
    }
}

__global__ void k_interior_flag(const int32_t *face_cells, int64_t nf, int32_t *flag) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x)
        flag[f] = face_cells[2 * f + 1] >= 0 ? 1 : 0;
}

__global__ void k_face_dof(const int32_t *flag, const int32_t *excl, int64_t nf, int32_t *face_dof, int32_t *dof_face) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        if (flag[f]) {
            face_dof[f] = excl[f];
            dof_face[excl[f]] = (int32_t)f;
        } else {
            face_dof[f] = -1;
        }
    }
}

// geometry: plain fp64 operations in the oracle's order, explicit _rn intrinsics (no FMA)
template <int D>
__global__ void k_cell_geometry(const double *coords, const int32_t *cells, int64_t nc, double *vol,
                                double *xK, double *a, int *err) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
        double X[D + 1][D];
#pragma unroll
        for (int v = 0; v < D + 1; ++v)
#pragma unroll
            for (int i = 0; i < D; ++i) X[v][i] = coords[(int64_t)cells[c * (D + 1) + v] * D + i];
        // |K|
        double det;
        double E[D][D];
#pragma unroll
        for (int v = 0; v < D; ++v)
#pragma unroll
            for (int i = 0; i < D; ++i) E[v][i] = __dsub_rn(X[v + 1][i], X[0][i]);
        if (D == 2) {
            det = E[0][0] * E[1][1] - E[0][1] * E[1][0];
        } else {
            det = E[0][0] * (E[1][1] * E[2][2] - E[1][2] * E[2][1]) -
                  E[0][1] * (E[1][0] * E[2][2] - E[1][2] * E[2][0]) +
                  E[0][2] * (E[1][0] * E[2][1] - E[1][1] * E[2][0]);
        }
        double vK = fabs(det) / (D == 2 ? 2.0 : 6.0);
        vol[c] = vK;
        double hmax = 0.0;
#pragma unroll
        for (int v = 0; v < D + 1; ++v)
#pragma unroll
            for (int w = 0; w < v; ++w) {
                double s = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) s += (X[v][i] - X[w][i]) * (X[v][i] - X[w][i]);
                hmax = fmax(hmax, sqrt(s));
            }
        double hd = D == 2 ? hmax * hmax : hmax * hmax * hmax;
        if (!(vK > 1e-14 * hd)) atomicCAS(err, DE_OK, DE_DEGENERATE);
        // x_K = (sum of vertices)/(d+1), summed in vertex order
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = X[0][i];
#pragma unroll
            for (int v = 1; v < D + 1; ++v) s = __dadd_rn(s, X[v][i]);
            xK[c * D + i] = __ddiv_rn(s, (double)(D + 1));
        }
        // a_{K,l}
#pragma unroll
        for (int l = 0; l < D + 1; ++l) {
            int32_t t[D];
            face_tuple<D>(cells, c, l, t);
            double P[D], Q[D], n[D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                P[i] = coords[(int64_t)t[0] * D + i];
                Q[i] = coords[(int64_t)t[1] * D + i];
            }
            if (D == 2) {
                double e0 = __dsub_rn(Q[0], P[0]), e1 = __dsub_rn(Q[1], P[1]);
                n[0] = e1;
                n[1] = -e0;
            } else {
                double R[D];
#pragma unroll
                for (int i = 0; i < D; ++i) R[i] = coords[(int64_t)t[D - 1] * D + i];
                double u0 = __dsub_rn(Q[0], P[0]), u1 = __dsub_rn(Q[1], P[1]), u2 = __dsub_rn(Q[2 % D], P[2 % D]);
                double w0 = __dsub_rn(R[0], P[0]), w1 = __dsub_rn(R[1], P[1]), w2 = __dsub_rn(R[2 % D], P[2 % D]);
                n[0] = __dmul_rn(0.5, __dsub_rn(__dmul_rn(u1, w2), __dmul_rn(u2, w1)));
                n[1] = __dmul_rn(0.5, __dsub_rn(__dmul_rn(u2, w0), __dmul_rn(u0, w2)));
                n[2 % D] = __dmul_rn(0.5, __dsub_rn(__dmul_rn(u0, w1), __dmul_rn(u1, w0)));
            }
            double dot = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) dot += n[i] * (P[i] - X[l][i]);
            double sg = dot < 0.0 ? -1.0 : 1.0;
#pragma unroll
            for (int i = 0; i < D; ++i) a[(c * (D + 1) + l) * D + i] = n[i] * sg;
        }
    }
}

template <int D>
__global__ void k_face_centroid(const double *coords, const int32_t *faces, int64_t nf, double *xs) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = coords[(int64_t)faces[f * D] * D + i];
#pragma unroll
            for (int v = 1; v < D; ++v) s = __dadd_rn(s, coords[(int64_t)faces[f * D + v] * D + i]);
            xs[f * D + i] = __ddiv_rn(s, (double)D);
        }
    }
}

static int read_err(int *err_d, cudaStream_t s) {
    int h = 0;
    CR_CUDA(cudaMemcpyAsync(&h, err_d, sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    return h;
}

template <int D>
static void build_mesh_t(cr_mesh_s *m, int64_t nv, const double *coords, int64_t nc, const int32_t *cells,
                         cudaStream_t s) {
    const int T = 256;
    const int64_t n = nc * (D + 1);
    DevBuf<int> err;
    err.alloc(1, s);
    err.zero(s);
    k_check_cells<<<grid_for(n, T), T, 0, s>>>(cells, n, nv, err.get());
    CR_CHECK_LAUNCH();
    CR_REQUIRE(read_err(err.get(), s) == DE_OK, CR_ERR_DEGENERATE_CELL, "cell references a vertex out of range");

    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < nv) ++bits;
    const bool two_pass = (int64_t)bits * D > 64;

    DevBuf<uint64_t> k0, k1;
    DevBuf<uint32_t> v0, v1;
    k0.alloc(n, s); k1.alloc(n, s); v0.alloc(n, s); v1.alloc(n, s);
    k_face_keys<D><<<grid_for(n, T), T, 0, s>>>(cells, nc, bits, two_pass ? 1 : 0, k0.get(), v0.get());
    CR_CHECK_LAUNCH();
    size_t tmp_bytes = 0;
    int end_bit = two_pass ? bits * (D - 1) : bits * D;
    CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0.get(), k1.get(), v0.get(), v1.get(), (int)n, 0,
                                            end_bit, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tmp_bytes, s);
    CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, k0.get(), k1.get(), v0.get(), v1.get(), (int)n, 0,
                                            end_bit, s));
    uint32_t *vals = v1.get();
    if (two_pass) {
        k_first_vertex_keys<D><<<grid_for(n, T), T, 0, s>>>(cells, n, v1.get(), k0.get());
        CR_CHECK_LAUNCH();
        size_t tb2 = 0;
        CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, k0.get(), k1.get(), v1.get(), v0.get(), (int)n, 0, bits, s));
        if (tb2 > tmp_bytes) { tmp.alloc(tb2, s); tmp_bytes = tb2; }
        CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb2, k0.get(), k1.get(), v1.get(), v0.get(), (int)n, 0, bits, s));
        vals = v0.get();
    }
    k1.release();
    DevBuf<int32_t> head, fid;
    head.alloc(n, s); fid.alloc(n, s);
    k_heads<D><<<grid_for(n, T), T, 0, s>>>(cells, n, vals, head.get(), err.get());
    CR_CHECK_LAUNCH();
    size_t tb3 = 0;
    CR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb3, head.get(), fid.get(), (int)n, s));
    if (tb3 > tmp_bytes) { tmp.alloc(tb3, s); tmp_bytes = tb3; }
    CR_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb3, head.get(), fid.get(), (int)n, s));
    int32_t nf32 = 0;
    CR_CUDA(cudaMemcpyAsync(&nf32, fid.get() + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CR_REQUIRE(read_err(err.get(), s) == DE_OK, CR_ERR_NONMANIFOLD, "non-manifold input: a face shared by more than two cells");
    const int64_t nf = nf32;
    m->nf = nf;
    m->faces.alloc(nf * D, s);
    m->face_cells.alloc(nf * 2, s);
    m->face_cells.fill_bytes(0xFF, s);   // -1
    m->cell_faces.alloc(n, s);
    k_incidence<D><<<grid_for(n, T), T, 0, s>>>(cells, n, vals, head.get(), fid.get(), m->faces.get(),
                                                 m->face_cells.get(), m->cell_faces.get());
    CR_CHECK_LAUNCH();
    // interior faces -> dof
    DevBuf<int32_t> flag, excl;
    flag.alloc(nf, s); excl.alloc(nf, s);
    k_interior_flag<<<grid_for(nf, T), T, 0, s>>>(m->face_cells.get(), nf, flag.get());
    CR_CHECK_LAUNCH();
    size_t tb4 = 0;
    CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb4, flag.get(), excl.get(), (int)nf, s));
    if (tb4 > tmp_bytes) { tmp.alloc(tb4, s); tmp_bytes = tb4; }
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb4, flag.get(), excl.get(), (int)nf, s));
    int32_t last_excl = 0, last_flag = 0;
    CR_CUDA(cudaMemcpyAsync(&last_excl, excl.get() + (nf - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&last_flag, flag.get() + (nf - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    m->nf_int = (int64_t)last_excl + last_flag;
    m->face_dof.alloc(nf, s);
    m->dof_face.alloc(m->nf_int > 0 ? m->nf_int : 1, s);
    k_face_dof<<<grid_for(nf, T), T, 0, s>>>(flag.get(), excl.get(), nf, m->face_dof.get(), m->dof_face.get());
    CR_CHECK_LAUNCH();
    // geometry
    m->vol.alloc(nc, s);
    m->xK.alloc(nc * D, s);
    m->a.alloc(nc * (D + 1) * D, s);
    m->xs.alloc(nf * D, s);
    k_cell_geometry<D><<<grid_for(nc, T), T, 0, s>>>(coords, cells, nc, m->vol.get(), m->xK.get(), m->a.get(), err.get());
    CR_CHECK_LAUNCH();
    k_face_centroid<D><<<grid_for(nf, T), T, 0, s>>>(coords, m->faces.get(), nf, m->xs.get());
    CR_CHECK_LAUNCH();
    CR_REQUIRE(read_err(err.get(), s) == DE_OK, CR_ERR_DEGENERATE_CELL, "degenerate cell (|K| <= 1e-14 h^d)");
}

void build_mesh(cr_mesh_s *m, int dim, int64_t nv, const double *coords, int64_t nc, const int32_t *cells,
                cudaStream_t s) {
    CR_REQUIRE(dim == 2 || dim == 3, CR_ERR_INVALID_ARG, "dim must be 2 or 3");
    CR_REQUIRE(nv > 0 && nc > 0 && coords && cells, CR_ERR_INVALID_ARG, "empty mesh or null pointer");
    CR_REQUIRE(nc * (dim + 1) < ((int64_t)1 << 31), CR_ERR_INVALID_ARG, "nc*(dim+1) must be < 2^31");
    CR_REQUIRE(nv < ((int64_t)1 << 31), CR_ERR_INVALID_ARG, "nv must be < 2^31");
    m->dim = dim;
    m->nv = nv;
    m->nc = nc;
    if (dim == 2) build_mesh_t<2>(m, nv, coords, nc, cells, s);
    else build_mesh_t<3>(m, nv, coords, nc, cells, s);
}

}  // namespace cr
