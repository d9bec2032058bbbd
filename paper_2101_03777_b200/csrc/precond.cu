// Setup of the overlapping-patch additive Schwarz preconditioner (layout and rationale in
// afw.cuh).  Everything runs on the device:
//
//   1. (key, dof*SLOTS+slot) pairs: 2D key = vertex of the face (edge), 3D key = edge (a,b)
//      of the face (triangle), for every interior face;
//   2. stable CUB radix sort by key -> patches = runs of equal keys, faces in ascending dof
//      order inside a patch (deterministic);
//   3. per 32-patch slice: k = largest patch, offsets by exclusive scans;
//   4. one thread per patch: B_p = R_p G R_p^t per component, read from the assembled G,
//      inverted in fp64 (Cholesky for SPD G, |B_p| by Jacobi eigen-decomposition for the
//      symmetric indefinite steady G, Gauss-Jordan for the nonsymmetric Navier-Stokes G).
#include <cub/cub.cuh>
#include <cstdlib>

#include "afw.cuh"
#include "internal.cuh"
#include "spmv.cuh"

namespace cr {

template <int D>
__global__ void k_patch_pairs(const int32_t *faces, const int32_t *dof_face, int64_t nrows, int bits,
                              uint64_t *keys, uint32_t *vals) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = dof_face[r];
        int32_t t[D];
#pragma unroll
        for (int j = 0; j < D; ++j) t[j] = faces[f * D + j];
        if constexpr (D == 2) {
            keys[2 * r] = (uint64_t)t[0];
            keys[2 * r + 1] = (uint64_t)t[1];
        } else {
            keys[3 * r] = ((uint64_t)t[0] << bits) | (uint64_t)t[1];
            keys[3 * r + 1] = ((uint64_t)t[0] << bits) | (uint64_t)t[2];
            keys[3 * r + 2] = ((uint64_t)t[1] << bits) | (uint64_t)t[2];
        }
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) vals[SLOTS * r + s] = (uint32_t)(SLOTS * r + s);
    }
}

// key of patch p (run p of the sorted pairs): its first face in the solve order
template <int SLOTS>
__global__ void k_patch_so_key(const int64_t *start, const uint32_t *sorted, int64_t npatch, const int32_t *iperm,
                               uint32_t *key, int32_t *idx) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npatch; p += (int64_t)gridDim.x * blockDim.x) {
        uint32_t k = 0xFFFFFFFFu;
        for (int64_t e = start[p]; e < start[p + 1]; ++e) k = min(k, (uint32_t)iperm[sorted[e] / SLOTS]);
        key[p] = k;
        idx[p] = (int32_t)p;
    }
}

__global__ void k_patch_heads(const uint64_t *keys, int64_t n, int32_t *head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_patch_starts(const int32_t *head, const int32_t *pid, int64_t n, int64_t *start) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (head[i]) start[pid[i] - 1] = i;
        if (i == n - 1) start[pid[i]] = n;
    }
}

// perm (may be null): patch p of the layout is run perm[p] of the sorted pairs
__global__ void k_slice_sizes(const int64_t *start, const int32_t *perm, int64_t npatch, int64_t nslices, int D, int sym,
                              uint8_t *kl, int64_t *isz, int64_t *vsz, int *kmax) {
    for (int64_t sl = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sl < nslices; sl += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        for (int64_t p = sl * 32; p < npatch && p < sl * 32 + 32; ++p) {
            const int64_t o = perm ? perm[p] : p;
            k = max(k, (int)(start[o + 1] - start[o]));
        }
        kl[sl] = (uint8_t)min(k, 255);
        isz[sl] = (int64_t)k * 32;
        const int64_t T = sym ? (int64_t)k * (k + 1) / 2 : (int64_t)k * k;
        vsz[sl] = (int64_t)D * T * 32;
        atomicMax(kmax, k);
    }
}

// G[(ra, i), (cb, i)] from the sliced block-ELL (0 when cb is not in row ra's stencil)
template <int D>
__device__ __forceinline__ double g_entry(const EllView<D> &G, const uint8_t *rowlen, int64_t ra, int64_t cb, int i) {
    constexpr int W = 2 * D + 1, B2 = D * D;
    const int64_t slice = ra >> 5;
    const int lane = (int)(ra & 31);
    const int n = rowlen[ra];
    for (int s = 0; s < n; ++s)
        if (G.cols[slice * (W * 32) + s * 32 + lane] == (int32_t)cb)
            return G.vals[slice * ((int64_t)W * B2 * 32) + (s * B2 + i * D + i) * 32 + lane];
    return 0.0;
}

// in-place inverse of the k x k block; returns false if the block is (numerically) singular
template <int KMAX>
__device__ bool inv_spd(double (&B)[KMAX][KMAX], int k) {
    double L[KMAX][KMAX];
    for (int a = 0; a < k; ++a) {
        for (int b = 0; b <= a; ++b) {
            double s = B[a][b];
            for (int c = 0; c < b; ++c) s -= L[a][c] * L[b][c];
            if (a == b) {
                if (!(s > 0.0)) return false;
                L[a][a] = sqrt(s);
            } else {
                L[a][b] = s / L[b][b];
            }
        }
    }
    // L^{-1} (lower), then B^{-1} = L^{-t} L^{-1}
    double Li[KMAX][KMAX];
    for (int a = 0; a < k; ++a) {
        for (int b = 0; b < a; ++b) Li[a][b] = 0.0;
        Li[a][a] = 1.0 / L[a][a];
        for (int b = a - 1; b >= 0; --b) {
            double s = 0.0;
            for (int c = b; c < a; ++c) s += L[a][c] * Li[c][b];
            Li[a][b] = -s / L[a][a];
        }
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b <= a; ++b) {
            double s = 0.0;
            for (int c = a; c < k; ++c) s += Li[c][a] * Li[c][b];
            B[a][b] = s;
            B[b][a] = s;
        }
    return true;
}

// |B|^{-1} = V |Lambda|^{-1} V^t by cyclic Jacobi rotations (symmetric B)
template <int KMAX>
__device__ bool inv_abs(double (&B)[KMAX][KMAX], int k) {
    double V[KMAX][KMAX];
    double nrm = 0.0;
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) {
            V[a][b] = (a == b) ? 1.0 : 0.0;
            nrm = fmax(nrm, fabs(B[a][b]));
        }
    if (!(nrm > 0.0)) return false;
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) off = fmax(off, fabs(B[a][b]));
        if (off <= 1e-17 * nrm) break;
        for (int a = 0; a < k; ++a)
            for (int b = a + 1; b < k; ++b) {
                if (B[a][b] == 0.0) continue;
                const double th = (B[b][b] - B[a][a]) / (2.0 * B[a][b]);
                const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int q = 0; q < k; ++q) {   // B <- B J
                    const double x = B[q][a], y = B[q][b];
                    B[q][a] = c * x - sn * y;
                    B[q][b] = sn * x + c * y;
                }
                for (int q = 0; q < k; ++q) {   // B <- J^t B
                    const double x = B[a][q], y = B[b][q];
                    B[a][q] = c * x - sn * y;
                    B[b][q] = sn * x + c * y;
                }
                for (int q = 0; q < k; ++q) {
                    const double x = V[q][a], y = V[q][b];
                    V[q][a] = c * x - sn * y;
                    V[q][b] = sn * x + c * y;
                }
            }
    }
    double il[KMAX];
    for (int a = 0; a < k; ++a) {
        const double l = fabs(B[a][a]);
        if (!(l > 1e-300)) return false;
        il[a] = 1.0 / l;
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b <= a; ++b) {
            double s = 0.0;
            for (int c = 0; c < k; ++c) s += V[a][c] * il[c] * V[b][c];
            B[a][b] = s;
            B[b][a] = s;
        }
    return true;
}

template <int KMAX>
__device__ bool inv_gen(double (&B)[KMAX][KMAX], int k) {
    double X[KMAX][KMAX];
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) X[a][b] = (a == b) ? 1.0 : 0.0;
    for (int c = 0; c < k; ++c) {
        int pv = c;
        for (int a = c + 1; a < k; ++a) if (fabs(B[a][c]) > fabs(B[pv][c])) pv = a;
        if (!(fabs(B[pv][c]) > 0.0)) return false;
        if (pv != c)
            for (int b = 0; b < k; ++b) {
                double t = B[c][b]; B[c][b] = B[pv][b]; B[pv][b] = t;
                t = X[c][b]; X[c][b] = X[pv][b]; X[pv][b] = t;
            }
        const double inv = 1.0 / B[c][c];
        for (int b = 0; b < k; ++b) { B[c][b] *= inv; X[c][b] *= inv; }
        for (int a = 0; a < k; ++a) {
            if (a == c) continue;
            const double f = B[a][c];
            if (f == 0.0) continue;
            for (int b = 0; b < k; ++b) { B[a][b] -= f * B[c][b]; X[a][b] -= f * X[c][b]; }
        }
    }
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < k; ++b) B[a][b] = X[a][b];
    return true;
}

template <int D, int KMAX, int MODE>
__global__ void __launch_bounds__(64) k_patch_setup(EllView<D> G, const uint8_t *rowlen, const int64_t *start,
                                                    const int32_t *perm, const uint32_t *sorted, int64_t npatch, AfwView A,
                                                    int32_t *ids, double *vals, unsigned long long *nfallback) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    constexpr bool SYM = MODE != AFW_GEN;
    const int64_t nsl = (npatch + 31) / 32;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nsl * 32; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slice = p >> 5;
        const int lane = (int)(p & 31);
        const int ks = A.kl[slice];
        const int64_t o = (p < npatch && perm) ? perm[p] : p;
        const int k = p < npatch ? (int)(start[o + 1] - start[o]) : 0;
        int32_t *ip = ids + A.ioff[slice] + lane;
        int64_t dof[KMAX];
        for (int j = 0; j < ks; ++j) {
            if (j < k) {
                const uint32_t v = sorted[start[o] + j];
                ip[j * 32] = (int32_t)v;
                dof[j] = v / SLOTS;
            } else {
                ip[j * 32] = -1;
            }
        }
        const int T = SYM ? ks * (ks + 1) / 2 : ks * ks;
        double *vp = vals + A.voff[slice] + lane;
        for (int i = 0; i < (A.shared ? 1 : D); ++i) {
            double B[KMAX][KMAX];
            for (int a = 0; a < k; ++a)
                for (int b = 0; b < k; ++b) {
                    if (A.shared) {   // the components' blocks averaged (SPD: a mean of SPD blocks)
                        double g = 0.0;
                        for (int c = 0; c < D; ++c) g += g_entry<D>(G, rowlen, dof[a], dof[b], c);
                        B[a][b] = g / D;
                    } else {
                        B[a][b] = g_entry<D>(G, rowlen, dof[a], dof[b], i);
                    }
                }
            bool ok;
            if (MODE == AFW_SPD) ok = inv_spd<KMAX>(B, k);
            else if (MODE == AFW_ABS) ok = inv_abs<KMAX>(B, k);
            else ok = inv_gen<KMAX>(B, k);
            if (!ok) {   // singular patch block: fall back to its (absolute) diagonal
                for (int a = 0; a < k; ++a)
                    for (int b = 0; b < k; ++b) {
                        const double g = g_entry<D>(G, rowlen, dof[a], dof[b], i);
                        B[a][b] = (a == b) ? 1.0 / (MODE == AFW_GEN ? g : fabs(g)) : 0.0;
                    }
                if (k > 0) atomicAdd(nfallback, 1ull);
            }
            double *vi = vp + (int64_t)i * T * 32;
            for (int a = 0; a < ks; ++a) {
                if (SYM) {
                    for (int b = 0; b <= a; ++b) vi[(a * (a + 1) / 2 + b) * 32] = (a < k && b < k) ? B[a][b] : 0.0;
                } else {
                    for (int b = 0; b < ks; ++b) vi[(a * ks + b) * 32] = (a < k && b < k) ? B[a][b] : 0.0;
                }
            }
        }
    }
}

template <int D>
static void build_afw_t(cr_hybrid_s *h, int mode, cudaStream_t s) {
    constexpr int SLOTS = D == 2 ? 2 : 3;
    const cr_mesh_s *m = h->mesh;
    const int64_t nrows = h->G.nrows, n = nrows * SLOTS;
    CR_REQUIRE(n < ((int64_t)1 << 31), CR_ERR_INVALID_ARG, "too many (face, patch) pairs for the patch preconditioner");
    const int T = 256;
    AfwPrec &P = h->afw;
    P.built = -1;
    P.slots = SLOTS;
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < m->nv) ++bits;
    DevBuf<uint64_t> k0, k1;
    DevBuf<uint32_t> v0, v1;
    k0.alloc(n, s); k1.alloc(n, s); v0.alloc(n, s); v1.alloc(n, s);
    k_patch_pairs<D><<<grid_for(nrows, T), T, 0, s>>>(m->faces.get(), m->dof_face.get() + (h->part.on ? h->part.row0 : 0),
                                                       nrows, bits, k0.get(), v0.get());
    CR_CHECK_LAUNCH();
    const int end_bit = D == 2 ? bits : 2 * bits;
    size_t tb = 0;
    CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.get(), k1.get(), v0.get(), v1.get(), (int)n, 0, end_bit, s));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb, s);
    CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, k0.get(), k1.get(), v0.get(), v1.get(), (int)n, 0, end_bit, s));
    DevBuf<int32_t> head, pid;
    head.alloc(n, s); pid.alloc(n, s);
    k_patch_heads<<<grid_for(n, T), T, 0, s>>>(k1.get(), n, head.get());
    CR_CHECK_LAUNCH();
    size_t tb2 = 0;
    CR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, head.get(), pid.get(), (int)n, s));
    if (tb2 > tb) { tmp.alloc(tb2, s); tb = tb2; }
    CR_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb2, head.get(), pid.get(), (int)n, s));
    int32_t np32 = 0;
    CR_CUDA(cudaMemcpyAsync(&np32, pid.get() + (n - 1), sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    const int64_t npatch = np32;
    DevBuf<int64_t> start;
    start.alloc(npatch + 1, s);
    k_patch_starts<<<grid_for(n, T), T, 0, s>>>(head.get(), pid.get(), n, start.get());
    CR_CHECK_LAUNCH();
    const int64_t nsl = (npatch + 31) / 32;
    P.npatch = npatch;
    P.nslices = nsl;
    P.kl.alloc(nsl, s);
    DevBuf<int64_t> isz, vsz;
    isz.alloc(nsl, s); vsz.alloc(nsl, s);
    P.ioff.alloc(nsl, s); P.voff.alloc(nsl, s);
    DevBuf<int> kmax;
    kmax.alloc(1, s);
    kmax.zero(s);
    // PCG (SPD mode): one block per patch, the mean of the D component blocks, serves all components
    // (configs[4]: 441 vs 439 iterations, 5.83 vs 6.44 ms each; the operator 7.8 -> 2.6 GB).
    // CR_AFW_SHARED=0 restores one block per component; MINRES's |block| keeps them.
    static const char *esh = std::getenv("CR_AFW_SHARED");
    P.shared = (!(esh && atoi(esh) == 0) && mode == AFW_SPD) ? 1 : 0;
    // with the solve order built: patches ordered by their first solve-order row, so a warp's 32
    // patches gather r from nearby rows (the layout's ids stay mesh rows; ids_so maps them)
    DevBuf<int32_t> perm;
    if (h->so.built) {
        DevBuf<uint32_t> pk, pk2;
        DevBuf<int32_t> pi;
        pk.alloc(npatch, s); pk2.alloc(npatch, s); pi.alloc(npatch, s); perm.alloc(npatch, s);
        k_patch_so_key<SLOTS><<<grid_for(npatch, T), T, 0, s>>>(start.get(), v1.get(), npatch, h->so.iperm.get(),
                                                               pk.get(), pi.get());
        CR_CHECK_LAUNCH();
        size_t ts = 0;
        CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, ts, pk.get(), pk2.get(), pi.get(), perm.get(), (int)npatch, 0, 32, s));
        if (ts > tb) { tmp.alloc(ts, s); tb = ts; }
        CR_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), ts, pk.get(), pk2.get(), pi.get(), perm.get(), (int)npatch, 0, 32, s));
    }
    k_slice_sizes<<<grid_for(nsl, T), T, 0, s>>>(start.get(), perm.get(), npatch, nsl, P.shared ? 1 : D, mode != AFW_GEN,
                                                 P.kl.get(), isz.get(), vsz.get(), kmax.get());
    CR_CHECK_LAUNCH();
    size_t tb3 = 0;
    CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb3, isz.get(), P.ioff.get(), (int)nsl, s));
    if (tb3 > tb) { tmp.alloc(tb3, s); tb = tb3; }
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb3, isz.get(), P.ioff.get(), (int)nsl, s));
    CR_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb3, vsz.get(), P.voff.get(), (int)nsl, s));
    int64_t last[4];
    int hk = 0;
    CR_CUDA(cudaMemcpyAsync(&last[0], P.ioff.get() + nsl - 1, 8, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&last[1], isz.get() + nsl - 1, 8, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&last[2], P.voff.get() + nsl - 1, 8, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&last[3], vsz.get() + nsl - 1, 8, cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaMemcpyAsync(&hk, kmax.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    P.kmax = hk;
    CR_REQUIRE(hk <= 16, CR_ERR_INVALID_ARG, "patch preconditioner: a patch has more than 16 faces");
    P.ids.alloc(last[0] + last[1], s);
    P.vals.alloc(last[2] + last[3], s);
    DevBuf<unsigned long long> nfb;
    nfb.alloc(1, s);
    nfb.zero(s);
    EllView<D> Gv{h->G.cols.get(), h->G.vals.get(), nrows};
    AfwView A{P.ioff.get(), P.voff.get(), P.kl.get(), P.ids.get(), P.vals.get(), npatch, nrows, P.shared};
    const int grid = grid_for(nsl * 32, 64, 16);
#define CR_SETUP(KM, MD) \
    k_patch_setup<D, KM, MD><<<grid, 64, 0, s>>>(Gv, h->rowlen.get(), start.get(), perm.get(), v1.get(), npatch, A, P.ids.get(), P.vals.get(), nfb.get())
    if (hk <= 8) {
        if (mode == AFW_SPD) CR_SETUP(8, AFW_SPD);
        else if (mode == AFW_ABS) CR_SETUP(8, AFW_ABS);
        else CR_SETUP(8, AFW_GEN);
    } else {
        if (mode == AFW_SPD) CR_SETUP(16, AFW_SPD);
        else if (mode == AFW_ABS) CR_SETUP(16, AFW_ABS);
        else CR_SETUP(16, AFW_GEN);
    }
#undef CR_SETUP
    CR_CHECK_LAUNCH();
    unsigned long long hf = 0;
    CR_CUDA(cudaMemcpyAsync(&hf, nfb.get(), sizeof(hf), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    P.nfallback = (int64_t)hf;
    P.ids_so.release();
    P.built = mode;
    if (h->so.built) afw_so(h, s);
}

__global__ void k_afw_ids_so(const int32_t *ids, int64_t n, int slots, const int32_t *iperm, int32_t *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = ids[i];
        out[i] = v >= 0 ? iperm[v / slots] * slots + v % slots : -1;
    }
}

void afw_so(cr_hybrid_s *h, cudaStream_t s) {
    AfwPrec &P = h->afw;
    if (P.built < 0 || P.ids_so.n == P.ids.n || !h->so.built) return;
    P.ids_so.alloc(P.ids.n, s);
    const int T = 256;
    k_afw_ids_so<<<grid_for((int64_t)P.ids.n, T), T, 0, s>>>(P.ids.get(), (int64_t)P.ids.n, P.slots, h->so.iperm.get(),
                                                            P.ids_so.get());
    CR_CHECK_LAUNCH();
}

void build_afw(cr_hybrid_s *h, int mode, cudaStream_t s) {
    if (h->afw.built == mode) return;
    if (h->G.d == 2) build_afw_t<2>(h, mode, s);
    else build_afw_t<3>(h, mode, s);
}

}  // namespace cr
