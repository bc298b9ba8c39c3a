// fl_boundary.cu -- set_boundary_flags' face matching on the GPU.
//
// The reference (mesh.hpp:251-304) sorts all (d+1)*NT face keys (sorted vertex
// tuples) and flags every key that occurs exactly once: a boundary face, whose
// centroid (sum of its vertices in kTriFaces / kTetFaces order from 0.0, then
// / d) goes to the classifier.  Here the node->element plan replaces the sort:
// a face is owned by its smallest vertex a, and every element containing the
// face is incident to a.  One warp per node a walks a's incidences, inserts the
// faces it owns (key = the other d-1 vertices, sorted) into a shared-memory hash
// with counts, then marks the faces counted once.  A scan over the marks lists
// the boundary faces in ascending (t, lf) order with their centroids; the
// classifier runs on the host (fl_boundary_faces_copy), and
// fl_mesh_set_boundary_flags scatters its values (interior faces get 0).
#include <cuda_runtime.h>

#include <cstdint>

#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

namespace {

constexpr int kBWarps = 4;
constexpr int kBHash = 256;  // owned faces per node (3-D Kuhn: ~24)

__device__ __forceinline__ void face_vertices(int D, const int32_t* v, int lf, int32_t f[3]) {
    // kTriFaces = {1,2},{2,0},{0,1}; kTetFaces = {1,3,2},{0,2,3},{0,3,1},{0,1,2} (mesh.hpp:29-30)
    if (D == 2) {
        f[0] = v[lf == 0 ? 1 : lf == 1 ? 2 : 0];
        f[1] = v[lf == 0 ? 2 : lf == 1 ? 0 : 1];
        f[2] = -1;
    } else {
        f[0] = v[lf == 0 ? 1 : 0];
        f[1] = v[lf == 0 ? 3 : lf == 1 ? 2 : lf == 2 ? 3 : 1];
        f[2] = v[lf == 0 ? 2 : lf == 1 ? 3 : lf == 2 ? 1 : 2];
    }
}

// key of face lf of element v owned by vertex a (a must be the face's minimum):
// the remaining d-1 vertices, sorted; 0 = not owned by a
template <int D>
__device__ __forceinline__ uint64_t owned_key(const int32_t* v, int lf, int32_t a) {
    int32_t f[3];
    face_vertices(D, v, lf, f);
    if (D == 2) {
        const int32_t o = f[0] == a ? f[1] : f[0];
        if (!(f[0] == a || f[1] == a) || o < a) return 0;
        return (uint64_t)(uint32_t)o + 1;
    }
    int32_t x, y;
    if (f[0] == a) {
        x = f[1];
        y = f[2];
    } else if (f[1] == a) {
        x = f[0];
        y = f[2];
    } else if (f[2] == a) {
        x = f[0];
        y = f[1];
    } else {
        return 0;
    }
    if (x < a || y < a) return 0;
    if (x > y) {
        const int32_t z = x;
        x = y;
        y = z;
    }
    return (((uint64_t)(uint32_t)x << 32) | (uint32_t)y) + 1;
}

template <int D>
__global__ void __launch_bounds__(kBWarps * 32)
k_boundary_mark(int32_t n_nodes, const int32_t* __restrict__ elems, const int32_t* __restrict__ inc_ptr,
                const uint32_t* __restrict__ inc, uint8_t* __restrict__ bmark,
                unsigned int* __restrict__ ticket, uint32_t* __restrict__ err) {
    constexpr int NV = D + 1;
    __shared__ unsigned long long keys[kBWarps][kBHash];
    __shared__ int cnt[kBWarps][kBHash];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    while (true) {
        int32_t a = 0;
        if (lane == 0) a = (int32_t)atomicAdd(ticket, 1u);
        a = __shfl_sync(0xffffffffu, a, 0);
        if (a >= n_nodes) break;
        for (int h = lane; h < kBHash; h += 32) {
            keys[w][h] = 0ull;
            cnt[w][h] = 0;
        }
        __syncwarp();
        const int32_t p0 = __ldg(inc_ptr + a), m = __ldg(inc_ptr + a + 1) - p0;
        // pass 1: insert the owned faces, counting multiplicities
        for (int base = 0; base < m; base += 32) {
            if (base + lane < m) {
                const uint32_t key = __ldg(inc + p0 + base + lane);
                const int32_t t = (int32_t)(key & 0x3FFFFFFFu);
                const int j = (int)(key >> 30);
                int32_t v[NV];
#pragma unroll
                for (int k = 0; k < NV; ++k) v[k] = __ldg(elems + (size_t)t * NV + k);
#pragma unroll
                for (int lf = 0; lf < NV; ++lf) {
                    if (lf == j) continue;
                    const uint64_t fk = owned_key<D>(v, lf, a);
                    if (!fk) continue;
                    uint32_t h = (uint32_t)((fk * 0x9E3779B97F4A7C15ull) >> 56) & (kBHash - 1);
                    bool done = false;
                    for (int probe = 0; probe < kBHash && !done; ++probe) {
                        const unsigned long long old = atomicCAS(&keys[w][h], 0ull, fk);
                        if (old == 0ull || old == fk) {
                            atomicAdd(&cnt[w][h], 1);
                            done = true;
                        } else {
                            h = (h + 1) & (kBHash - 1);
                        }
                    }
                    if (!done) atomicOr(err, DERR_OVERFLOW);
                }
            }
        }
        __syncwarp();
        // pass 2: faces counted once are boundary faces
        for (int base = 0; base < m; base += 32) {
            if (base + lane < m) {
                const uint32_t key = __ldg(inc + p0 + base + lane);
                const int32_t t = (int32_t)(key & 0x3FFFFFFFu);
                const int j = (int)(key >> 30);
                int32_t v[NV];
#pragma unroll
                for (int k = 0; k < NV; ++k) v[k] = __ldg(elems + (size_t)t * NV + k);
#pragma unroll
                for (int lf = 0; lf < NV; ++lf) {
                    if (lf == j) continue;
                    const uint64_t fk = owned_key<D>(v, lf, a);
                    if (!fk) continue;
                    uint32_t h = (uint32_t)((fk * 0x9E3779B97F4A7C15ull) >> 56) & (kBHash - 1);
                    for (int probe = 0; probe < kBHash; ++probe) {
                        if (keys[w][h] == fk) {
                            if (cnt[w][h] == 1) bmark[(size_t)t * NV + lf] = 1;
                            break;
                        }
                        if (keys[w][h] == 0ull) break;
                        h = (h + 1) & (kBHash - 1);
                    }
                }
            }
        }
        __syncwarp();
    }
}

// boundary face q = the q-th marked (t, lf); centroid as mesh.hpp:287-294
template <int D>
__global__ void k_boundary_emit(int64_t n_entries, const int32_t* __restrict__ elems,
                                const double* __restrict__ nodes, const uint8_t* __restrict__ bmark,
                                const int32_t* __restrict__ pos, int32_t* __restrict__ faces,
                                double* __restrict__ cent) {
    constexpr int NV = D + 1;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_entries;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (!bmark[e]) continue;
        const int32_t q = pos[e];
        const int32_t t = (int32_t)(e / NV);
        const int lf = (int)(e - (int64_t)t * NV);
        faces[2 * (size_t)q] = t;
        faces[2 * (size_t)q + 1] = lf;
        int32_t v[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) v[k] = __ldg(elems + (size_t)t * NV + k);
        int32_t f[3];
        face_vertices(D, v, lf, f);
        double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int x = 0; x < D; ++x) c[x] = __dadd_rn(c[x], __ldg(nodes + (size_t)f[k] * D + x));
#pragma unroll
        for (int x = 0; x < D; ++x) c[x] = __ddiv_rn(c[x], (double)D);
        cent[3 * (size_t)q] = c[0];
        cent[3 * (size_t)q + 1] = c[1];
        cent[3 * (size_t)q + 2] = D == 3 ? c[2] : 0.0;
    }
}

// flags[t*(d+1)+lf] = values[q] (or fill) for boundary face q, 0 elsewhere
__global__ void k_boundary_scatter(int64_t n_entries, const uint8_t* __restrict__ bmark,
                                   const int32_t* __restrict__ pos, const int8_t* __restrict__ values,
                                   int8_t fill, int8_t* __restrict__ flags, uint32_t* __restrict__ err) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_entries;
         e += (int64_t)gridDim.x * blockDim.x) {
        int8_t f = 0;
        if (bmark[e]) {
            f = values ? values[pos[e]] : fill;
            if (f < 0 || f > 3) atomicOr(err, DERR_FLAG);
        }
        flags[e] = f;
    }
}

}  // namespace

int launch_boundary_faces(fl_ctx* ctx, fl_mesh* mesh, int64_t* n_faces) {
    const cudaStream_t s = ctx->stream;
    const int nv = mesh->dim + 1;
    const int64_t ne = (int64_t)mesh->n_elems * nv;
    FL_TRY(mesh->bmark.ensure((size_t)std::max<int64_t>(ne, 1)));
    FL_TRY(mesh->bpos.ensure(sizeof(int32_t) * ((size_t)ne + 1)));
    FL_TRY(mesh->stats.ensure(sizeof(unsigned long long) * 4));
    uint8_t* bmark = mesh->bmark.as<uint8_t>();
    FL_CUDA(cudaMemsetAsync(bmark, 0, (size_t)std::max<int64_t>(ne, 1), s));
    uint32_t* words = reinterpret_cast<uint32_t*>(mesh->stats.as<unsigned long long>() + 2);
    FL_CUDA(cudaMemsetAsync(words, 0, sizeof(uint32_t) * 2, s));  // [0] ticket, [1] error
    if (mesh->n_nodes > 0 && ne > 0) {
        const int grid = ctx->sm_count * 8;
        if (mesh->dim == 2)
            k_boundary_mark<2><<<grid, kBWarps * 32, 0, s>>>(mesh->n_nodes, mesh->elems.as<int32_t>(),
                                                             mesh->inc_ptr.as<int32_t>(),
                                                             mesh->inc.as<uint32_t>(), bmark, words,
                                                             words + 1);
        else
            k_boundary_mark<3><<<grid, kBWarps * 32, 0, s>>>(mesh->n_nodes, mesh->elems.as<int32_t>(),
                                                             mesh->inc_ptr.as<int32_t>(),
                                                             mesh->inc.as<uint32_t>(), bmark, words,
                                                             words + 1);
        count_launch(ctx);
    }
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(ne)));
    const uint8_t* bm = bmark;
    FL_CUDA(launch_scan<int32_t>(
        ne, [bm] __device__(int64_t i) { return (int64_t)bm[i]; }, mesh->bpos.as<int32_t>(),
        ctx->scan_ws.p, s));
    count_launch(ctx);
    uint32_t* h = static_cast<uint32_t*>(ctx->pinned);
    FL_CUDA(cudaMemcpyAsync(h, mesh->bpos.as<int32_t>() + ne, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaMemcpyAsync(h + 1, words + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    if (h[1] & DERR_OVERFLOW) return set_error(FL_ERR_UNSUPPORTED, "a node owns more faces than the boundary kernel's table");
    const int64_t nb = (int32_t)h[0];
    FL_TRY(mesh->bfaces.ensure(sizeof(int32_t) * 2 * (size_t)std::max<int64_t>(nb, 1)));
    FL_TRY(mesh->bcent.ensure(sizeof(double) * 3 * (size_t)std::max<int64_t>(nb, 1)));
    if (nb > 0) {
        const int grid = (int)std::min<int64_t>(div_up(ne, 256), (int64_t)ctx->sm_count * 16);
        if (mesh->dim == 2)
            k_boundary_emit<2><<<grid, 256, 0, s>>>(ne, mesh->elems.as<int32_t>(), mesh->nodes.as<double>(),
                                                    bmark, mesh->bpos.as<int32_t>(),
                                                    mesh->bfaces.as<int32_t>(), mesh->bcent.as<double>());
        else
            k_boundary_emit<3><<<grid, 256, 0, s>>>(ne, mesh->elems.as<int32_t>(), mesh->nodes.as<double>(),
                                                    bmark, mesh->bpos.as<int32_t>(),
                                                    mesh->bfaces.as<int32_t>(), mesh->bcent.as<double>());
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    mesh->n_bfaces = nb;
    *n_faces = nb;
    return FL_OK;
}

int launch_boundary_scatter(fl_ctx* ctx, fl_mesh* mesh, const int8_t* values, int8_t fill) {
    const cudaStream_t s = ctx->stream;
    const int64_t ne = (int64_t)mesh->n_elems * (mesh->dim + 1);
    FL_TRY(mesh->flags.ensure((size_t)std::max<int64_t>(ne, 1)));
    uint32_t* words = reinterpret_cast<uint32_t*>(mesh->stats.as<unsigned long long>() + 2);
    FL_CUDA(cudaMemsetAsync(words + 1, 0, sizeof(uint32_t), s));
    if (ne > 0) {
        const int grid = (int)std::min<int64_t>(div_up(ne, 256), (int64_t)ctx->sm_count * 16);
        k_boundary_scatter<<<grid, 256, 0, s>>>(ne, mesh->bmark.as<uint8_t>(), mesh->bpos.as<int32_t>(),
                                                values, fill, mesh->flags.as<int8_t>(), words + 1);
        count_launch(ctx);
    }
    uint32_t* h = static_cast<uint32_t*>(ctx->pinned);
    FL_CUDA(cudaMemcpyAsync(h, words + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    if (h[0] & DERR_FLAG) return set_error(FL_E_INVALID_FLAG_VALUE, "classifier returned a flag outside {0,1,2,3}");
    mesh->has_flags = true;
    return FL_OK;
}

}  // namespace fl
