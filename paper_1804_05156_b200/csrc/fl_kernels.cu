// fl_kernels.cu -- device side of the B200 P1 assembly path (v1, general).
//
// Pipeline:
//   plan    k_inc_count -> scan -> k_inc_fill -> k_inc_sort -> k_plan_stats
//           node -> incidence lists sorted by (local index j, element t): the
//           order in which the reference's blockwise triplets reach a column
//           (assembly.hpp:286-298 + the stable counting sorts sparse.hpp:79-89).
//   mark    k_mark_boundary -> scan -> k_partition (partition_boundary, system.hpp:50-67)
//   column  k_columns<D>: one warp per output column c = one reference CSC column,
//           exact per-entry summation order (i, j, t), zero drop, fused load
//           vector, Neumann, Dirichlet lift, A(free,free) and b_f, with CSC
//           offsets from a decoupled look-back over column tiles.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

// ===========================================================================
// plan
// ===========================================================================
// Consecutive entries of element-ordered meshes repeat vertices (the tets of a
// Kuhn cube share 8 vertices over 24 entries): lanes holding the same node are
// grouped with match_any and the group leader issues one atomic for all of them.
// Block-contiguous: block b counts entries [b*256*it, (b+1)*256*it), blocks
// issued in element order, so the live counters stay in L2.  B200, it = 16 vs
// a grid-stride loop: C5 plan 5.30 -> 5.16 ms, C4 0.48 -> 0.46 ms (it = 1,
// one entry per thread: C5 +0.8 ms).
constexpr int kCountIters = 16;
__global__ void k_inc_count(int64_t n_entries, int32_t n_nodes, int32_t c_begin, int32_t n_cols, int it,
                            const int32_t* __restrict__ elems, int32_t* __restrict__ cnt,
                            uint32_t* __restrict__ err) {
    const unsigned lower = (1u << (threadIdx.x & 31)) - 1;
    const int64_t b0 = (int64_t)blockIdx.x * blockDim.x * it;
    for (int k = 0; k < it; ++k) {
        const int64_t e = b0 + (int64_t)k * blockDim.x + threadIdx.x;
        if (e - (threadIdx.x & 31) >= n_entries) break;  // warp-uniform
        int32_t key = -1;
        if (e < n_entries) {
            const int32_t v = __ldg(elems + e);
            if (v < 0 || v >= n_nodes) {
                atomicOr(err, DERR_INDEX);
            } else if ((uint32_t)(v - c_begin) < (uint32_t)n_cols) {
                key = v - c_begin;
            }
        }
        const unsigned g = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && (g & lower) == 0) atomicAdd(cnt + key, __popc(g));
    }
}

// U rounds of 32 consecutive entries per warp iteration: the rounds' atomics
// (which return the slot, so each costs an L2 round trip) are all in flight
// before the first dependent store
constexpr int kFillRounds = 4;
template <int U>
__global__ void k_inc_fill(int32_t n_elems, int nv, int32_t n_nodes, int32_t c_begin, int32_t n_cols,
                           const int32_t* __restrict__ elems, const int32_t* __restrict__ inc_ptr,
                           int32_t* __restrict__ cursor, uint32_t* __restrict__ inc,
                           uint8_t* __restrict__ emark) {
    (void)inc_ptr;
    const int64_t n_entries = (int64_t)n_elems * nv;
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t e0 = warp * 32 * U; e0 < n_entries; e0 += nwarps * 32 * U) {
        int32_t key[U];
        unsigned grp[U];
        int32_t pos[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * 32 + lane;
            key[u] = -1;
            if (e < n_entries) {
                const int32_t v = __ldg(elems + e);
                if (v >= 0 && v < n_nodes && (uint32_t)(v - c_begin) < (uint32_t)n_cols) key[u] = v - c_begin;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) grp[u] = __match_any_sync(0xffffffffu, key[u]);
        // cursor starts at inc_ptr (one random-access array instead of two); the
        // leader reserves the group's slots, members take base + rank
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pos[u] = 0;
            if (key[u] >= 0 && (grp[u] & lower) == 0) pos[u] = atomicAdd(cursor + key[u], __popc(grp[u]));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t p0 = __shfl_sync(0xffffffffu, pos[u], __ffs(grp[u]) - 1) + __popc(grp[u] & lower);
            if (key[u] >= 0) {
                const int64_t e = e0 + u * 32 + lane;
                const int32_t t = entry_elem(e, nv);
                const uint32_t j = (uint32_t)(e - (int64_t)t * nv);
                inc[p0] = (j << 30) | (uint32_t)t;
                if (emark) emark[t] = 1;
            }
        }
    }
}

// ---- bucketed plan (large meshes).  Random node ids turn k_inc_fill's 4-byte
// writes into sector-granular read-modify-writes over the whole incidence array.
// Instead: (1) count per node AND per bucket of 2^shift consecutive nodes;
// (2) partition the incidences by bucket into a staging array (block-local
// smem ranks, one global atomic per bucket per block: coalesced runs);
// (3) fill from the staging in bucket order, so the live destination range is
// one bucket's slice of the incidence array, resident in L2.
constexpr int kPlanBlock = 256, kPlanItems = 16, kMaxBuckets = 1024;

__global__ void __launch_bounds__(kPlanBlock)
k_inc_count_b(int64_t n_entries, int32_t n_nodes, int32_t c_begin, int32_t n_cols, int shift,
              const int32_t* __restrict__ elems, int32_t* __restrict__ cnt,
              int32_t* __restrict__ bcnt, uint32_t* __restrict__ err) {
    __shared__ int32_t hist[kMaxBuckets];
    const int nb = ((n_cols - 1) >> shift) + 1;
    for (int b = threadIdx.x; b < nb; b += kPlanBlock) hist[b] = 0;
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_entries;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = __ldg(elems + e);
        if (v < 0 || v >= n_nodes) {
            atomicOr(err, DERR_INDEX);
            continue;
        }
        const uint32_t lv = (uint32_t)(v - c_begin);
        if (lv < (uint32_t)n_cols) {
            atomicAdd(cnt + lv, 1);
            atomicAdd(&hist[lv >> shift], 1);
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kPlanBlock)
        if (hist[b]) atomicAdd(bcnt + b, hist[b]);
}

__global__ void __launch_bounds__(kPlanBlock)
k_bucket_scatter(int64_t n_entries, int nv, int32_t n_nodes, int32_t c_begin, int32_t n_cols,
                 int shift, const int32_t* __restrict__ elems, const int32_t* __restrict__ boff,
                 int32_t* __restrict__ bcur, int2* __restrict__ stage) {
    __shared__ int32_t hist[kMaxBuckets];
    __shared__ int32_t base[kMaxBuckets];
    const int nb = ((n_cols - 1) >> shift) + 1;
    constexpr int CH = kPlanBlock * kPlanItems;
    for (int64_t e0 = (int64_t)blockIdx.x * CH; e0 < n_entries; e0 += (int64_t)gridDim.x * CH) {
        for (int b = threadIdx.x; b < nb; b += kPlanBlock) hist[b] = 0;
        __syncthreads();
        int32_t lv[kPlanItems], rk[kPlanItems];
        uint32_t key[kPlanItems];
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k) {
            const int64_t e = e0 + k * kPlanBlock + threadIdx.x;
            lv[k] = -1;
            if (e < n_entries) {
                const int32_t v = __ldg(elems + e);
                const uint32_t l = (uint32_t)(v - c_begin);
                if (v >= 0 && v < n_nodes && l < (uint32_t)n_cols) {
                    lv[k] = (int32_t)l;
                    const int32_t t = entry_elem(e, nv);
                    key[k] = ((uint32_t)(e - (int64_t)t * nv) << 30) | (uint32_t)t;
                    rk[k] = atomicAdd(&hist[l >> shift], 1);
                }
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += kPlanBlock)
            if (hist[b]) base[b] = __ldg(boff + b) + atomicAdd(bcur + b, hist[b]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPlanItems; ++k)
            if (lv[k] >= 0) stage[base[lv[k] >> shift] + rk[k]] = make_int2(lv[k], (int32_t)key[k]);
        __syncthreads();
    }
}

__global__ void k_bucket_offsets(int nb, int shift, int32_t n_cols, const int32_t* __restrict__ inc_ptr,
                                 int32_t* __restrict__ boff) {
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        boff[b] = inc_ptr[min((int64_t)b << shift, (int64_t)n_cols)];
}

// total staged = inc_ptr[n_cols] (read on the device: no host sync in the plan)
__global__ void __launch_bounds__(kPlanBlock)
k_inc_fill_b(const int32_t* __restrict__ total, const int2* __restrict__ stage,
             const int32_t* __restrict__ inc_ptr, int32_t* __restrict__ cursor,
             uint32_t* __restrict__ inc, uint8_t* __restrict__ emark) {
    // four consecutive staged incidences per thread: their slot reservations are
    // in flight together before the dependent stores
    const int64_t n_staged = *total;
    for (int64_t q0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; q0 < n_staged;
         q0 += (int64_t)gridDim.x * blockDim.x * 4) {
        int2 sv[4];
        int32_t pos[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sv[u] = q0 + u < n_staged ? __ldg(stage + q0 + u) : make_int2(-1, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) pos[u] = sv[u].x >= 0 ? atomicAdd(cursor + sv[u].x, 1) : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (sv[u].x < 0) continue;
            inc[pos[u]] = (uint32_t)sv[u].y;
            if (emark) emark[(uint32_t)sv[u].y & 0x3FFFFFFFu] = 1;
        }
    }
}

// Sort each node's incidence keys ascending = (j, t) order.  Segments are
// short (2-D ~6, 3-D Kuhn 24): insertion sort per thread.
__global__ void k_inc_sort(int32_t n_nodes, const int32_t* __restrict__ inc_ptr,
                           uint32_t* __restrict__ inc, const int32_t* __restrict__ list) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_nodes) return;
    const int32_t c = list ? list[q] : q;
    const int32_t p0 = inc_ptr[c], p1 = inc_ptr[c + 1];
    for (int32_t a = p0 + 1; a < p1; ++a) {
        const uint32_t key = inc[a];
        int32_t b = a - 1;
        while (b >= p0 && inc[b] > key) {
            inc[b + 1] = inc[b];
            --b;
        }
        inc[b + 1] = key;
    }
}

// stats[0] += sum_c min(m_c * d + 1, N)  (nnz upper bound), stats[1] = max m_c
__global__ void k_plan_stats(int32_t n_cols, int32_t n_nodes, int dim,
                             const int32_t* __restrict__ inc_ptr,
                             unsigned long long* __restrict__ stats) {
    int64_t bound = 0;
    int32_t mx = 0;
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n_cols;
         c += gridDim.x * blockDim.x) {
        const int32_t m = inc_ptr[c + 1] - inc_ptr[c];
        const int64_t b = (int64_t)m * dim + 1;
        bound += b < n_nodes ? b : n_nodes;
        mx = m > mx ? m : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bound += __shfl_xor_sync(0xffffffffu, bound, o);
        const int32_t y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(stats, (unsigned long long)bound);
        atomicMax(stats + 1, (unsigned long long)mx);
    }
}

// ===========================================================================
// validation (make_mesh, mesh.hpp:148-187)
// ===========================================================================
template <int D>
__global__ void k_validate(int32_t n_elems, int32_t n_nodes, const double* __restrict__ nodes,
                           const int32_t* __restrict__ elems, const int8_t* __restrict__ flags,
                           uint32_t* __restrict__ err) {
    constexpr int NV = D + 1;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_elems;
         t += gridDim.x * blockDim.x) {
        int32_t v[NV];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            v[k] = elems[(size_t)t * NV + k];
            ok &= (v[k] >= 0 && v[k] < n_nodes);
            if (flags) {
                const int8_t f = flags[(size_t)t * NV + k];
                if (f < 0 || f > 3) atomicOr(err, DERR_FLAG);
            }
        }
        if (!ok) {
            atomicOr(err, DERR_INDEX);
            continue;
        }
        double m;
        if (D == 2) {
            const double* a = nodes + 2 * (size_t)v[0];
            const double* b = nodes + 2 * (size_t)v[1];
            const double* c = nodes + 2 * (size_t)v[2];
            // mesh.hpp:34-38
            const double e2x = a[0] - c[0], e2y = a[1] - c[1];
            const double e3x = b[0] - a[0], e3y = b[1] - a[1];
            m = 0.5 * (-e3x * e2y + e3y * e2x);
        } else {
            const double* p1 = nodes + 3 * (size_t)v[0];
            const double* p2 = nodes + 3 * (size_t)v[1];
            const double* p3 = nodes + 3 * (size_t)v[2];
            const double* p4 = nodes + 3 * (size_t)v[NV - 1];
            // mesh.hpp:42-51 (division by 6 keeps the sign: test the numerator)
            const double ax = p2[0] - p1[0], ay = p2[1] - p1[1], az = p2[2] - p1[2];
            const double bx = p3[0] - p1[0], by = p3[1] - p1[1], bz = p3[2] - p1[2];
            const double cx = p4[0] - p1[0], cy = p4[1] - p1[1], cz = p4[2] - p1[2];
            const double nx = ay * bz - az * by;
            const double ny = az * bx - ax * bz;
            const double nz = ax * by - ay * bx;
            m = (nx * cx + ny * cy + nz * cz) / 6.0;
        }
        if (!(m > 0.0)) atomicOr(err, DERR_MEASURE);
    }
}

// ===========================================================================
// boundary marking: partition_boundary (system.hpp:50-67) / boundary_faces
// (mesh.hpp:222-246).  is_dir[v] = 1 for every vertex of a flag-1 face.
// ===========================================================================
template <int D>
__global__ void k_mark_boundary(int32_t n_elems, int32_t n_nodes, const int32_t* __restrict__ elems,
                                const int8_t* __restrict__ flags, int8_t* __restrict__ is_dir,
                                int8_t* __restrict__ is_neu, uint32_t* __restrict__ counters) {
    constexpr int NV = D + 1;
    const int64_t n_entries = (int64_t)n_elems * NV;
    uint32_t dir_faces = 0, neu_faces = 0, err = 0;
    auto visit = [&](int64_t e, int8_t f) {
        if (f == 3) err |= DERR_ROBIN;
        if (f < 0 || f > 3) err |= DERR_FLAG;
        if (f != 1 && f != 2) return;
        const int32_t t = (int32_t)(e / NV);
        const int lf = (int)(e - (int64_t)t * NV);
        int8_t* mark = (f == 1) ? is_dir : is_neu;
        if (f == 1) ++dir_faces;
        else ++neu_faces;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            if (k == lf) continue;
            // a vertex id outside [0, N) is reported (index_out_of_range), never written
            const int32_t v = elems[(size_t)t * NV + k];
            if ((uint32_t)v < (uint32_t)n_nodes) mark[v] = 1;
            else err |= DERR_INDEX;
        }
    };
    // 16 flags per load: nearly all are 0 (interior faces)
    const int64_t n_vec = n_entries >> 4;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = tid; i < n_vec; i += stride) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(flags) + i);
        if ((v.x | v.y | v.z | v.w) == 0) continue;
        const int32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int8_t f = (int8_t)(w[b >> 2] >> (8 * (b & 3)));
            if (f != 0) visit(i * 16 + b, f);
        }
    }
    for (int64_t e = (n_vec << 4) + tid; e < n_entries; e += stride) {
        const int8_t f = flags[e];
        if (f != 0) visit(e, f);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dir_faces += __shfl_xor_sync(0xffffffffu, dir_faces, o);
        neu_faces += __shfl_xor_sync(0xffffffffu, neu_faces, o);
        err |= __shfl_xor_sync(0xffffffffu, err, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (dir_faces) atomicAdd(counters + CNT_DIR_FACES, dir_faces);
        if (neu_faces) atomicAdd(counters + CNT_NEU_FACES, neu_faces);
        if (err) atomicOr(counters + CNT_ERR, err);
    }
}

// free rank scan output -> lists (ascending, system.hpp:63-65) and row map
__global__ void k_partition(int32_t n_nodes, const int8_t* __restrict__ is_dir,
                            const int32_t* __restrict__ free_rank, int32_t* __restrict__ fidx,
                            int32_t* __restrict__ dir_nodes, int32_t* __restrict__ free_nodes,
                            uint32_t* __restrict__ counters) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_nodes;
         k += gridDim.x * blockDim.x) {
        const int32_t fr = free_rank[k];
        if (is_dir[k]) {
            fidx[k] = -1;
            dir_nodes[k - fr] = k;
        } else {
            fidx[k] = fr;
            free_nodes[fr] = k;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) counters[CNT_N_DIR] = n_nodes - free_rank[n_nodes];
}

// ===========================================================================
// FaceLists of partition_boundary: boundary_faces(mesh, 1) and (mesh, 2)
// (mesh.hpp:222-246): faces whose flag equals the value, face-major -- every
// local face 0 over t ascending, then local face 1, ... -- each with its
// vertices in kTriFaces / kTetFaces order (mesh.hpp:29-30), its element and
// its local face.  Ordered compaction: per-block counts per (value, lf), an
// exclusive scan over (lf, block), then each block writes its faces in order.
// ===========================================================================
constexpr int kFaceThreads = 256, kFaceItems = 16;  // elements per thread
constexpr int kFaceBlockElems = kFaceThreads * kFaceItems;

template <int D>
__device__ __forceinline__ uint32_t elem_flags(const int8_t* __restrict__ flags, int64_t t) {
    if constexpr (D == 3) return (uint32_t)__ldg(reinterpret_cast<const int32_t*>(flags) + t);
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) w |= (uint32_t)(uint8_t)__ldg(flags + t * 3 + k) << (8 * k);
    return w;
}

// per-thread counts of its kFaceItems elements, 16-bit fields: word 0 = Dirichlet
// lf 0..3, word 1 = Neumann lf 0..3
template <int D>
__device__ __forceinline__ void face_counts(const int8_t* __restrict__ flags, int32_t n_elems, int64_t t0,
                                            uint64_t& cd, uint64_t& cn) {
    cd = cn = 0;
    for (int k = 0; k < kFaceItems; ++k) {
        const int64_t t = t0 + k;
        if (t >= n_elems) break;
        const uint32_t w = elem_flags<D>(flags, t);
        if (!w) continue;
#pragma unroll
        for (int lf = 0; lf <= D; ++lf) {
            const int8_t f = (int8_t)(w >> (8 * lf));
            if (f == 1) cd += 1ull << (16 * lf);
            else if (f == 2) cn += 1ull << (16 * lf);
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kFaceThreads) k_face_count(int32_t n_elems, const int8_t* __restrict__ flags,
                                                            int32_t nblk, int32_t* __restrict__ bcnt) {
    __shared__ uint64_t s[2][kFaceThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t cd, cn;
    face_counts<D>(flags, n_elems, (int64_t)blockIdx.x * kFaceBlockElems + (int64_t)threadIdx.x * kFaceItems, cd, cn);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cd += __shfl_xor_sync(0xffffffffu, cd, o);
        cn += __shfl_xor_sync(0xffffffffu, cn, o);
    }
    if (lane == 0) {
        s[0][w] = cd;
        s[1][w] = cn;
    }
    __syncthreads();
    if (threadIdx.x <= 2 * D + 1) {  // (value, lf) = category
        const int v = threadIdx.x / (D + 1), lf = threadIdx.x % (D + 1);
        int32_t tot = 0;
        for (int i = 0; i < kFaceThreads / 32; ++i) tot += (int32_t)((s[v][i] >> (16 * lf)) & 0xFFFFu);
        // Dirichlet then Neumann; each lf-major over the blocks
        bcnt[(int64_t)(v * (D + 1) + lf) * nblk + blockIdx.x] = tot;
    }
}

template <int D>
__global__ void __launch_bounds__(kFaceThreads) k_face_emit(int32_t n_elems, const int32_t* __restrict__ elems,
                                                           const int8_t* __restrict__ flags, int32_t nblk,
                                                           const int32_t* __restrict__ boff,
                                                           int32_t* __restrict__ dfaces, int32_t* __restrict__ delem,
                                                           int32_t* __restrict__ dlocal, int32_t* __restrict__ nfaces,
                                                           int32_t* __restrict__ nelem, int32_t* __restrict__ nlocal) {
    constexpr int NV = D + 1;
    __shared__ uint64_t s[2][kFaceThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * kFaceBlockElems + (int64_t)threadIdx.x * kFaceItems;
    uint64_t cd, cn;
    face_counts<D>(flags, n_elems, t0, cd, cn);
    // block-wide exclusive scan of the packed counts (fields never carry: <= 4096)
    uint64_t id = cd, in = cn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t a = __shfl_up_sync(0xffffffffu, id, o), b = __shfl_up_sync(0xffffffffu, in, o);
        if (lane >= o) {
            id += a;
            in += b;
        }
    }
    if (lane == 31) {
        s[0][w] = id;
        s[1][w] = in;
    }
    __syncthreads();
    uint64_t pd = id - cd, pn = in - cn;  // exclusive within the warp
    for (int i = 0; i < w; ++i) {
        pd += s[0][i];
        pn += s[1][i];
    }
    if (!(cd | cn)) return;
    int32_t pos[2][NV];
#pragma unroll
    for (int lf = 0; lf < NV; ++lf) {
        pos[0][lf] = __ldg(boff + (int64_t)lf * nblk + blockIdx.x) + (int32_t)((pd >> (16 * lf)) & 0xFFFFu);
        pos[1][lf] = __ldg(boff + (int64_t)(NV + lf) * nblk + blockIdx.x) + (int32_t)((pn >> (16 * lf)) & 0xFFFFu);
    }
    for (int k = 0; k < kFaceItems; ++k) {
        const int64_t t = t0 + k;
        if (t >= n_elems) break;
        const uint32_t fw = elem_flags<D>(flags, t);
        if (!fw) continue;
#pragma unroll
        for (int lf = 0; lf < NV; ++lf) {
            const int8_t f = (int8_t)(fw >> (8 * lf));
            if (f != 1 && f != 2) continue;
            const int v = f - 1;
            const int32_t q = pos[v][lf]++;
            int32_t* faces = v ? nfaces : dfaces;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                // kTriFaces = {1,2},{2,0},{0,1}; kTetFaces = {1,3,2},{0,2,3},{0,3,1},{0,1,2}
                int lv;
                if constexpr (D == 2) lv = (lf + 1 + a) % 3;
                else lv = (lf == 0) ? (a == 0 ? 1 : a == 1 ? 3 : 2)
                          : (lf == 1) ? (a == 0 ? 0 : a == 1 ? 2 : 3)
                          : (lf == 2) ? (a == 0 ? 0 : a == 1 ? 3 : 1)
                                      : a;
                faces[(int64_t)q * D + a] = __ldg(elems + t * NV + lv);
            }
            (v ? nelem : delem)[q] = (int32_t)t;
            (v ? nlocal : dlocal)[q] = lf;
        }
    }
}

// ===========================================================================
// column kernel
// ===========================================================================
constexpr int kHS = 256;           // per-warp slot table (distinct rows of a column)
constexpr int kMaxSlots = 192;     // load factor 0.75
constexpr int kMaxNeu = 128;       // Neumann items per node
constexpr int kWarps = 4;          // columns per tile (one warp each)
constexpr int32_t kEmpty = -1;

struct WarpSmem {
    int32_t keys[kHS];
    double acc[kHS];
    double tacc[kHS];
    int32_t out_rows[kHS];
    double out_vals[kHS];
    int32_t ff_rows[kHS];
    double ff_vals[kHS];
    double stage[32];
    uint32_t neu_key[kMaxNeu];
    double neu_val[kMaxNeu];
    int32_t n_a, n_ff;
};

__device__ __forceinline__ uint32_t slot_hash(int32_t row) {
    return ((uint32_t)row * 2654435761u) >> 24;  // 8 bits
}

// -1: the column has more distinct rows than the table holds (DERR_OVERFLOW)
__device__ __forceinline__ int find_or_insert(WarpSmem& ws, int32_t row) {
    uint32_t h = slot_hash(row);
    for (int probe = 0; probe < kMaxSlots; ++probe) {
        const int32_t prev = atomicCAS(&ws.keys[h], kEmpty, row);
        if (prev == kEmpty) {
            ws.acc[h] = -0.0;   // -0.0 + x == x for every x: the fold starts at
            ws.tacc[h] = -0.0;  // the first value exactly as sparse.hpp:101
            return (int)h;
        }
        if (prev == row) return (int)h;
        h = (h + 1) & (kHS - 1);
    }
    return -1;
}

__device__ __forceinline__ int find_slot(const WarpSmem& ws, int32_t row) {
    uint32_t h = slot_hash(row);
    for (int probe = 0; probe < kHS; ++probe) {
        if (ws.keys[h] == row) return (int)h;
        h = (h + 1) & (kHS - 1);
    }
    return -1;
}

__device__ __forceinline__ double field_at_node(const FieldDesc& g, const double* nodes, int dim,
                                                int32_t k) {
    if (g.kind == FL_FIELD_SAMPLES) return __ldg(g.samples + k);
    if (g.kind == FL_FIELD_CONST) return g.value;
    const double x = nodes[(size_t)k * dim];
    const double y = nodes[(size_t)k * dim + 1];
    const double z = dim == 3 ? nodes[(size_t)k * dim + 2] : 0.0;
    return eval_point(g, x, y, z);
}

// Bitonic sort of up to kHS (row, val, tval) entries in warp smem, ascending row.
__device__ void smem_sort_rows(int32_t* rows, double* vals, int n, int lane) {
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int i = n + lane; i < p2; i += 32) rows[i] = INT_MAX;
    __syncwarp();
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < p2; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    if ((rows[i] > rows[ixj]) == up) {
                        const int32_t r = rows[i];
                        rows[i] = rows[ixj];
                        rows[ixj] = r;
                        const double v = vals[i];
                        vals[i] = vals[ixj];
                        vals[ixj] = v;
                    }
                }
            }
            __syncwarp();
        }
    }
}

template <int D>
struct Lane {
    int32_t t;
    int j;
    bool valid;
    int32_t R[D + 1];
    double s[D + 1];
    double l;
};

template <int D>
__device__ __forceinline__ void lane_compute(const ColParams& p, Lane<D>& L, int32_t p0, int32_t m,
                                             int k, const Recip& R3, const Recip& R6,
                                             ElemCol<D>& ec) {
    L.valid = k < m;
    if (!L.valid) return;
    const uint32_t key = __ldg(p.inc + p0 + k);
    L.t = (int32_t)(key & 0x3FFFFFFFu);
    L.j = (int)(key >> 30);
    if (p.srec) {  // hybrid pass: the element records are already computed
        const double* row = p.srec + ((size_t)L.t * (D + 1) + L.j) * (rec64<D>() ? 8 : 4);
#pragma unroll
        for (int i = 0; i <= D; ++i) L.s[i] = __ldg(row + i);
        L.l = !p.want_b ? 0.0 : rec64<D>() ? __ldg(row + 4) : __ldg(p.lrec + (size_t)L.t * 4 + L.j);
#pragma unroll
        for (int i = 0; i <= D; ++i) L.R[i] = __ldg(p.elems + (size_t)L.t * (D + 1) + i);
        if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE) ec.load(p.nodes, L.R);
        return;
    }
    if (D == 3) {
        const int4 q = __ldg(reinterpret_cast<const int4*>(p.elems) + L.t);
        L.R[0] = q.x;
        L.R[1] = q.y;
        L.R[2] = q.z;
        L.R[D] = q.w;
    } else {
#pragma unroll
        for (int i = 0; i <= D; ++i) L.R[i] = __ldg(p.elems + (size_t)L.t * (D + 1) + i);
    }
    ec.load(p.nodes, L.R);
    double meas;
    if constexpr (D == 2) meas = ec.stiffness_col(L.j, L.s);
    else meas = ec.stiffness_col(L.j, L.s, R6);
    if (meas == 0.0) atomicOr(p.err, DERR_DEGENERATE);
    if (p.want_a && p.coef.kind != FL_FIELD_NONE) {
        double a;
        if (p.coef.kind == FL_FIELD_CONST) a = p.coef.value;
        else if (p.coef.kind == FL_FIELD_SAMPLES) a = __ldg(p.coef.samples + L.t);
        else a = ec.coef_c5(R3);
#pragma unroll
        for (int i = 0; i <= D; ++i) L.s[i] = L.s[i] * a;
    }
    if (p.want_b) {
        if constexpr (D == 2) L.l = ec.load_col(L.j, L.t, p.f, R6);
        else L.l = ec.load_col(L.j, L.t, meas, p.f);
    } else {
        L.l = 0.0;
    }
}

// One warp assembles column c.  Results stay in ws (out_* lists) until the
// tile offsets are known.
template <int D>
__device__ void column_warp(const ColParams& p, int32_t c, WarpSmem& ws, int lane,
                            double& b_out, double& bmod_out, double& u0_out) {
    const unsigned FULL = 0xffffffffu;
    const int32_t p0 = p.inc_ptr[c - p.c_begin];
    const int32_t m = p.inc_ptr[c - p.c_begin + 1] - p0;
    const int nchunks = (m + 31) >> 5;
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);

    for (int h = lane; h < kHS; h += 32) ws.keys[h] = kEmpty;
    const int w = threadIdx.x >> 5;
    if (lane == 0) ws.n_a = ws.n_ff = 0;
    __syncwarp();


    Lane<D> L;
    ElemCol<D> ec;
    double b = 0.0;
    // ---- normal passes: order (i, k) == the reference's (i*(d+1)+j, t) per entry
    for (int i = 0; i <= D; ++i) {
        for (int ch = 0; ch < nchunks; ++ch) {
            if (i == 0 || nchunks > 1) {
                lane_compute<D>(p, L, p0 + ch * 32, m - ch * 32, lane, R3, R6, ec);
                if (i == 0 && p.want_b) {
                    // b[c] = 0.0 + contributions in (j, t) order (system.hpp:114-118)
                    const int cnt = min(32, m - ch * 32);
                    for (int q = 0; q < cnt; ++q) b = b + __shfl_sync(FULL, L.l, q);
                }
            }
            if (!p.want_a) continue;
            const int32_t key = L.valid ? L.R[i] : kEmpty;
            const unsigned g = __match_any_sync(FULL, key);
            ws.stage[lane] = L.s[i];
            __syncwarp();
            if (L.valid && lane == __ffs(g) - 1) {
                const int slot = find_or_insert(ws, key);
                if (slot >= 0) {
                    double a = ws.acc[slot];
                    for (unsigned mm = g; mm; mm &= mm - 1) a = a + ws.stage[__ffs(mm) - 1];
                    ws.acc[slot] = a;
                } else {
                    atomicOr(p.err, DERR_OVERFLOW);
                }
            }
            __syncwarp();
        }
        if (!p.want_a) break;
    }

    // ---- Neumann data (system.hpp:123-172), only at nodes on a flag-2 face
    double neu_add = 0.0;
    bool neu_active = false;
    if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE && p.is_neu[c]) {
        neu_active = true;
        __shared__ int s_nneu[kWarps];
        if (lane == 0) s_nneu[w] = 0;
        __syncwarp();
        for (int ch = 0; ch < nchunks; ++ch) {
            if (nchunks > 1 || !p.want_a)
                lane_compute<D>(p, L, p0 + ch * 32, m - ch * 32, lane, R3, R6, ec);
            if (L.valid) {
                for (int lf = 0; lf <= D; ++lf) {
                    if (lf == L.j) continue;
                    if (p.flags[(size_t)L.t * (D + 1) + lf] != 2) continue;
                    const int q = atomicAdd(&s_nneu[w], 1);
                    if (q < kMaxNeu) {
                        ws.neu_key[q] = ((uint32_t)lf << 30) | (uint32_t)L.t;
                        ws.neu_val[q] = ec.face_share(lf, p.g_neu, R3, L.t);
                    } else {
                        atomicOr(p.err, DERR_OVERFLOW);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            // face-major order (lf, t) (mesh.hpp:229-244), accumulate from 0.0
            const int n = min(s_nneu[w], kMaxNeu);
            double add = 0.0;
            uint32_t last = 0;
            bool first = true;
            for (int r = 0; r < n; ++r) {
                int best = -1;
                for (int q = 0; q < n; ++q) {
                    const uint32_t k2 = ws.neu_key[q];
                    if ((first || k2 > last) && (best < 0 || k2 < ws.neu_key[best])) best = q;
                }
                last = ws.neu_key[best];
                first = false;
                add = add + ws.neu_val[best];
            }
            neu_add = add;
        }
        neu_add = __shfl_sync(FULL, neu_add, 0);
    }
    if (neu_active) b = b + neu_add;

    // ---- transposed folds for the Dirichlet lift: A(c, r) in the order
    //      (i_c*(d+1)+j_r, t) of entry (row c, col r) = passes (j, i, k)
    if (p.want_a && p.need_lift) {
        for (int jb = 0; jb <= D; ++jb)
            for (int i = 0; i <= D; ++i)
                for (int ch = 0; ch < nchunks; ++ch) {
                    if (nchunks > 1) lane_compute<D>(p, L, p0 + ch * 32, m - ch * 32, lane, R3, R6, ec);
                    const bool act = L.valid && L.j == jb;
                    const int32_t key = act ? L.R[i] : kEmpty;
                    const unsigned g = __match_any_sync(FULL, key);
                    ws.stage[lane] = L.s[i];
                    __syncwarp();
                    if (act && lane == __ffs(g) - 1) {
                        const int slot = find_slot(ws, key);
                        if (slot >= 0) {
                            double a = ws.tacc[slot];
                            for (unsigned mm = g; mm; mm &= mm - 1) a = a + ws.stage[__ffs(mm) - 1];
                            ws.tacc[slot] = a;
                        }
                    }
                    __syncwarp();
                }
    }

    // ---- compact the slot table, sort by row, drop exact zeros (sparse.hpp:105)
    double y = 0.0;
    if (p.want_a) {
        __syncwarp();
        int n = 0;
        for (int base = 0; base < kHS; base += 32) {
            const int h = base + lane;
            const bool v = ws.keys[h] != kEmpty;
            const unsigned bal = __ballot_sync(FULL, v);
            if (v) {
                const int pos = n + __popc(bal & ((1u << lane) - 1));
                ws.out_rows[pos] = ws.keys[h];
                ws.out_vals[pos] = ws.acc[h];
            }
            n += __popc(bal);
        }
        __syncwarp();
        if (n <= 32) {
            int32_t r = lane < n ? ws.out_rows[lane] : INT_MAX;
            double v = lane < n ? ws.out_vals[lane] : 0.0;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    const int32_t ro = __shfl_xor_sync(FULL, r, jj);
                    const double vo = __shfl_xor_sync(FULL, v, jj);
                    const bool lower = (lane & jj) == 0;
                    const bool up = (lane & k) == 0;
                    const bool take = lower ? ((r > ro) == up) : ((r < ro) == up);
                    if (take) {
                        r = ro;
                        v = vo;
                    }
                }
            }
            __syncwarp();
            if (lane < n) {
                ws.out_rows[lane] = r;
                ws.out_vals[lane] = v;
            }
            __syncwarp();
        } else {
            smem_sort_rows(ws.out_rows, ws.out_vals, n, lane);
        }
        // drop zeros (A) and restrict to free rows/cols (A_ff); keep order
        const bool col_free = p.want_sys && p.fidx[c] >= 0;
        int na = 0, nf = 0;
        for (int base = 0; base < n; base += 32) {
            const int q = base + lane;
            const bool in = q < n;
            const int32_t r = in ? ws.out_rows[q] : 0;
            const double v = in ? ws.out_vals[q] : 0.0;
            const bool keep = in && v != 0.0;
            const int32_t fr = (keep && col_free) ? p.fidx[r] : -1;
            const bool keep_ff = fr >= 0;
            const unsigned ba = __ballot_sync(FULL, keep);
            const unsigned bf = __ballot_sync(FULL, keep_ff);
            __syncwarp();
            if (keep) {
                const int pos = na + __popc(ba & ((1u << lane) - 1));
                ws.out_rows[pos] = r;  // pos <= q: in-place forward compaction
                ws.out_vals[pos] = v;
            }
            if (keep_ff) {
                const int pos = nf + __popc(bf & ((1u << lane) - 1));
                ws.ff_rows[pos] = fr;
                ws.ff_vals[pos] = v;
            }
            na += __popc(ba);
            nf += __popc(bf);
            __syncwarp();
        }
        if (lane == 0) {
            ws.n_a = na;
            ws.n_ff = nf;
        }
        __syncwarp();
    }
    if (p.want_a && p.need_lift) {
        // y = (A u0)[c]: matvec (sparse.hpp:129-141) adds A(c, r) * u0[r] over
        // the stored entries of row c in ascending column r; A(c, r) is the
        // transposed fold above.  Walk the slot table in ascending row order.
        __syncwarp();
        if (lane == 0) {
            // gather (row, tval) from the table, then ascending-row walk
            double yy = 0.0;
            int32_t last = INT_MIN;
            while (true) {
                int32_t best = INT_MAX;
                int bh = -1;
                for (int h = 0; h < kHS; ++h) {
                    const int32_t r = ws.keys[h];
                    if (r != kEmpty && r > last && r < best) {
                        best = r;
                        bh = h;
                    }
                }
                if (bh < 0) break;
                last = best;
                const double a_cr = ws.tacc[bh];
                if (a_cr != 0.0 && p.is_dir[best]) {
                    const double u = field_at_node(p.g_dir, p.nodes, D, best);
                    if (u != 0.0) yy = yy + a_cr * u;
                }
            }
            y = yy;
        }
        y = __shfl_sync(FULL, y, 0);
    }

    b_out = b;
    double u0 = 0.0;
    if (p.want_sys && p.is_dir[c]) u0 = field_at_node(p.g_dir, p.nodes, D, c);
    u0_out = u0;
    bmod_out = p.need_lift ? b - y : b - 0.0;
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32) k_columns(ColParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem* wsm = reinterpret_cast<WarpSmem*>(smem_raw);
    __shared__ int64_t s_tile;
    __shared__ uint64_t s_off;
    __shared__ int s_na[kWarps], s_nf[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem& ws = wsm[w];

    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(p.ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= p.n_tiles) break;
        const int64_t q64 = tile * kWarps + w;
        const bool has = p.col_list ? q64 < p.n_list : q64 < p.n_cols;
        const int32_t lc = p.col_list ? (has ? p.col_list[q64] : 0) : (int32_t)q64;
        const int32_t c = p.c_begin + lc;
        double b = 0.0, bmod = 0.0, u0 = 0.0;
        if (has) {
            column_warp<D>(p, c, ws, lane, b, bmod, u0);
        } else if (lane == 0) {
            ws.n_a = ws.n_ff = 0;
        }
        __syncwarp();
        if (lane == 0) {
            s_na[w] = p.want_a && has ? ws.n_a : 0;
            s_nf[w] = p.want_a && has ? ws.n_ff : 0;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            uint64_t agg_a = 0, agg_f = 0;
            for (int q = 0; q < kWarps; ++q) {
                agg_a += (uint64_t)s_na[q];
                agg_f += (uint64_t)s_nf[q];
            }
            uint64_t e;
            if (p.col_list) {  // hybrid: any staging order will do (offsets are recorded)
                e = 0;
                if (threadIdx.x == 0) {
                    const unsigned long long oa = atomicAdd(p.ov_alloc, (unsigned long long)agg_a);
                    const unsigned long long of = atomicAdd(p.ov_alloc + 1, (unsigned long long)agg_f);
                    e = (of << 31) | oa;
                }
            } else {
                // packed [61:31] = A(free,free) count, [30:0] = A count
                e = warp_lookback(p.tile_status, tile, (agg_f << 31) | agg_a);
            }
            if (threadIdx.x == 0) s_off = e;
        }
        __syncthreads();
        if (has) {
            uint64_t off_a = s_off & 0x7FFFFFFFull, off_f = s_off >> 31;
            for (int q = 0; q < w; ++q) {
                off_a += (uint64_t)s_na[q];
                off_f += (uint64_t)s_nf[q];
            }
            if (p.want_a) {
                const int na = s_na[w], nf = s_nf[w];
                if ((int64_t)(off_a + na) > p.cap_a || (int64_t)(off_f + nf) > p.cap_ff) {
                    if (lane == 0) atomicOr(p.err, DERR_CAPACITY);
                } else {
                    for (int q = lane; q < na; q += 32) {
                        p.row_idx[off_a + q] = ws.out_rows[q];
                        p.values[off_a + q] = ws.out_vals[q];
                    }
                    if (lane == 0 && p.col_list) {  // hybrid: counts / offsets per listed column
                        p.ov_cnt[q64] = na;
                        p.ov_cnt[p.n_list + q64] = nf;
                        p.ov_off[q64] = (int32_t)off_a;
                        p.ov_off[p.n_list + q64] = (int32_t)off_f;
                    } else if (lane == 0) {
                        p.col_ptr[lc + 1] = (int32_t)(off_a + na);
                    }
                    if (p.want_sys) {
                        const int32_t fc = p.fidx[c] - free_base(p);
                        for (int q = lane; q < nf; q += 32) {
                            p.ff_row_idx[off_f + q] = ws.ff_rows[q];
                            p.ff_values[off_f + q] = ws.ff_vals[q];
                        }
                        if (lane == 0 && fc >= 0 && !p.col_list) p.ff_col_ptr[fc + 1] = (int32_t)(off_f + nf);
                    }
                }
            }
            if (lane == 0) {
                if (p.want_b) p.b[lc] = b;
                if (p.want_sys) {
                    p.u0[lc] = u0;
                    p.b_mod[lc] = bmod;
                    const int32_t fc = p.fidx[c];
                    if (fc >= 0) p.b_f[fc - free_base(p)] = bmod;
                }
            }
        }
        __syncthreads();
    }
}

size_t column_smem_bytes() { return sizeof(WarpSmem) * kWarps; }
int column_tile_width() { return kWarps; }

// ===========================================================================
// general submatrix (sparse.hpp:159-183)
// ===========================================================================
__global__ void k_sub_rowmap(int32_t n_rows, const int32_t* __restrict__ rows,
                             int32_t* __restrict__ row_map, int32_t bound_m,
                             uint32_t* __restrict__ err) {
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_rows; q += gridDim.x * blockDim.x) {
        const int32_t r = rows[q];
        if (r < 0 || r >= bound_m) {
            atomicOr(err, 1u);
            continue;
        }
        if (q > 0 && r <= rows[q - 1]) atomicOr(err, 2u);
        row_map[r] = q;
    }
}

__global__ void k_sub_count(int32_t n_cols, const int32_t* __restrict__ cols, int32_t bound_n,
                            const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                            const int32_t* __restrict__ row_map, int32_t* __restrict__ cnt,
                            uint32_t* __restrict__ err) {
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_cols; q += gridDim.x * blockDim.x) {
        const int32_t c = cols[q];
        if (c < 0 || c >= bound_n) {
            atomicOr(err, 4u);
            cnt[q] = 0;
            continue;
        }
        if (q > 0 && c <= cols[q - 1]) atomicOr(err, 8u);
        int32_t k = 0;
        for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) k += row_map[row_idx[e]] >= 0;
        cnt[q] = k;
    }
}

__global__ void k_sub_fill(int32_t n_cols, const int32_t* __restrict__ cols,
                           const int32_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                           const double* __restrict__ values, const int32_t* __restrict__ row_map,
                           const int32_t* __restrict__ out_ptr, int32_t* __restrict__ out_rows,
                           double* __restrict__ out_vals) {
    for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_cols; q += gridDim.x * blockDim.x) {
        const int32_t c = cols[q];
        int32_t w = out_ptr[q];
        for (int32_t e = col_ptr[c]; e < col_ptr[c + 1]; ++e) {
            const int32_t r = row_map[row_idx[e]];
            if (r < 0) continue;
            out_rows[w] = r;
            out_vals[w] = values[e];
            ++w;
        }
    }
}

// ===========================================================================
// division self-test (fl_selftest_div)
// ===========================================================================
__global__ void k_selftest_div(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ q_fast, double* __restrict__ q_ieee) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const Recip R = recip(b[i]);
        const double q1 = div_by(a[i], R);
        // the batched form (div_fast + the all-or-nothing IEEE fallback) must agree
        // bit for bit with div_by; a disagreement is reported as a finite sentinel
        bool ok = divisor_ok(R);
        double q2 = div_fast(a[i], R, ok);
        if (!ok) q2 = __ddiv_rn(a[i], b[i]);
        const bool same = __double_as_longlong(q1) == __double_as_longlong(q2);
        q_fast[i] = same ? q1 : __longlong_as_double(0x7fefdeadbeefcafell);  // finite sentinel
        q_ieee[i] = __ddiv_rn(a[i], b[i]);
    }
}

// ===========================================================================
// host launchers
// ===========================================================================
int launch_plan_kernels(fl_ctx* ctx, fl_mesh* mesh, uint32_t* d_err) {
    const cudaStream_t s = ctx->stream;
    mesh->inc_sorted = false;
    const int nv = mesh->dim + 1;
    const int64_t n_entries = (int64_t)mesh->n_elems * nv;
    const int32_t N = mesh->n_nodes;
    const int32_t c0 = mesh->col_begin, nc = mesh->col_end - mesh->col_begin;
    FL_TRY(mesh->inc_ptr.ensure(sizeof(int32_t) * ((size_t)nc + 1)));
    FL_TRY(mesh->cursor.ensure(sizeof(int32_t) * ((size_t)nc + 1)));
    FL_TRY(mesh->inc.ensure(sizeof(uint32_t) * (size_t)(n_entries > 0 ? n_entries : 1)));
    FL_TRY(mesh->stats.ensure(sizeof(unsigned long long) * 4));
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(nc)));
    int32_t* cnt = mesh->cursor.as<int32_t>();
    FL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)nc + 1), s));
    FL_CUDA(cudaMemsetAsync(mesh->stats.p, 0, sizeof(unsigned long long) * 4, s));
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(div_up(n_entries, 256), 1),
                                            (int64_t)ctx->sm_count * 16);
    uint8_t* emark = nullptr;
    if (nc < N) {  // sharded: mark the elements the owned columns touch
        FL_TRY(mesh->emark.ensure((size_t)std::max<int32_t>(mesh->n_elems, 1)));
        emark = mesh->emark.as<uint8_t>();
        FL_CUDA(cudaMemsetAsync(emark, 0, (size_t)mesh->n_elems, s));
    }
    // bucketed fill for large 2-D meshes (FL_PLAN=0|1 overrides).  Measured on
    // B200 (profiles/r01_launches_C3/C5): C3 (100M incidences, 6 per node) plan
    // 8.4 -> 4.9 ms; C5 (400M, 24 per node) 9.8 -> 11.9 ms, so 3-D keeps the
    // direct fill, whose 96-byte per-node segments already batch the writes.
    const char* env = std::getenv("FL_PLAN");
    const bool bucketed = nc > 0 && n_entries > 0 &&
                          (env ? env[0] == '1' : (mesh->dim == 2 && n_entries >= ((int64_t)1 << 26)));
    // as many buckets of 2^shift nodes as the block histograms hold: a bucket's
    // slice of the incidence array (~3 MB at C5) stays in L2 while it is filled
    int shift = 0;
    // (fewer buckets -- longer runs per bucket in the scatter -- measured slower on C3)
    while (nc > 0 && ((int64_t)(nc - 1) >> shift) + 1 > kMaxBuckets) ++shift;
    const int nb = nc > 0 ? ((nc - 1) >> shift) + 1 : 0;
    int32_t* bcnt = nullptr;
    if (bucketed) {
        FL_TRY(mesh->bcnt.ensure(sizeof(int32_t) * 3 * (kMaxBuckets + 1)));
        bcnt = mesh->bcnt.as<int32_t>();
        FL_CUDA(cudaMemsetAsync(bcnt, 0, sizeof(int32_t) * 3 * (kMaxBuckets + 1), s));
        k_inc_count_b<<<grid, kPlanBlock, 0, s>>>(n_entries, N, c0, nc, shift,
                                                  mesh->elems.as<int32_t>(), cnt, bcnt, d_err);
        count_launch(ctx);
    } else if (n_entries > 0) {
        // up to kCountIters per block, fewer on small meshes so the grid still fills the SMs
        const int it = (int)std::max<int64_t>(
            1, std::min<int64_t>(kCountIters, n_entries / (256 * (int64_t)ctx->sm_count * 8)));
        k_inc_count<<<(int)std::max<int64_t>(div_up(n_entries, 256 * (int64_t)it), 1), 256, 0, s>>>(
            n_entries, N, c0, nc, it, mesh->elems.as<int32_t>(), cnt, d_err);
        count_launch(ctx);
    }
    const int32_t* cnt_c = cnt;
    FL_CUDA(launch_scan<int32_t>(
        nc, [cnt_c] __device__(int64_t i) { return (int64_t)cnt_c[i]; },
        mesh->inc_ptr.as<int32_t>(), ctx->scan_ws.p, s));
    count_launch(ctx);
    // fill cursors start at the segment offsets
    FL_CUDA(cudaMemcpyAsync(cnt, mesh->inc_ptr.p, sizeof(int32_t) * ((size_t)nc + 1),
                            cudaMemcpyDeviceToDevice, s));
    if (bucketed) {
        // bucket offsets = inc_ptr at the bucket boundaries
        int32_t* boff = bcnt + (kMaxBuckets + 1);
        int32_t* bcur = bcnt + 2 * (kMaxBuckets + 1);
        const int32_t* ip = mesh->inc_ptr.as<int32_t>();
        const int sh = shift;
        const int32_t ncc = nc;
        k_bucket_offsets<<<1, kMaxBuckets, 0, s>>>(nb, sh, ncc, ip, boff);
        count_launch(ctx);
        FL_TRY(mesh->bstage.ensure(sizeof(int2) * (size_t)n_entries));
        int2* stage = mesh->bstage.as<int2>();
        const int64_t chunks = (n_entries + kPlanBlock * kPlanItems - 1) / (kPlanBlock * kPlanItems);
        // one chunk per block, blocks issued in element order: consecutive chunks
        // append to each bucket's run back to back (C3 plan 3.83 -> 3.70 ms vs a
        // grid-stride loop over sm_count * 8 blocks)
        const int g2 = (int)std::min<int64_t>(chunks, INT_MAX);
        k_bucket_scatter<<<g2, kPlanBlock, 0, s>>>(n_entries, nv, N, c0, nc, shift,
                                                   mesh->elems.as<int32_t>(), boff, bcur, stage);
        count_launch(ctx);
        // one pass per block in staging order, as for k_inc_fill below: the live
        // bucket slice stays in L2 (C3 plan 4.13 -> 3.83 ms vs a grid-stride loop)
        const int bgrid = (int)std::min<int64_t>(std::max<int64_t>(div_up(n_entries, kPlanBlock * 4), 1), INT_MAX);
        k_inc_fill_b<<<bgrid, kPlanBlock, 0, s>>>(ip + nc, stage, ip, cnt, mesh->inc.as<uint32_t>(),
                                                 emark);
        count_launch(ctx);
    } else if (n_entries > 0) {
        // one warp iteration per block: blocks are issued in element order, so
        // the live set of destination segments is one resident wave's worth and
        // stays in L2 until its sectors are complete (a grid-stride loop lets
        // warps drift apart and the partial sectors go back to DRAM).  B200:
        // C5 plan 7.36 -> 5.31 ms, C4 0.53 -> 0.48 ms.
        // (4 rounds per warp measured best with this launch: C5 plan 5.96 / 5.55 /
        // 5.33 / 5.88 ms at 1 / 2 / 4 / 8)
        const int fgrid = (int)std::min<int64_t>(std::max<int64_t>(div_up(n_entries, 256 * kFillRounds), 1),
                                                 INT_MAX);
        auto kf = k_inc_fill<kFillRounds>;
        kf<<<fgrid, 256, 0, s>>>(mesh->n_elems, nv, N, c0, nc, mesh->elems.as<int32_t>(),
                                 mesh->inc_ptr.as<int32_t>(), cnt, mesh->inc.as<uint32_t>(), emark);
        count_launch(ctx);
    }
    if (nc > 0) {
        k_plan_stats<<<std::min(div_up(nc, 256), ctx->sm_count * 8), 256, 0, s>>>(
            nc, N, mesh->dim, mesh->inc_ptr.as<int32_t>(), mesh->stats.as<unsigned long long>());
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// The general kernel needs each node's incidences in (j, t) order; the tiled
// kernel ranks them itself, so this pass only runs on the fallback path.
int launch_inc_sort(fl_ctx* ctx, fl_mesh* mesh) {
    const int32_t nc = mesh->col_end - mesh->col_begin;
    if (nc > 0) {
        k_inc_sort<<<div_up(nc, 128), 128, 0, ctx->stream>>>(nc, mesh->inc_ptr.as<int32_t>(),
                                                            mesh->inc.as<uint32_t>(), nullptr);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    mesh->inc_sorted = true;
    return FL_OK;
}

// {n_cols, n_free_cols, nnz, nnz_ff} of a result, on the device (no host sync)
__global__ void k_result_counts(int32_t n_cols, int32_t col_begin, int32_t n_rows, int want_a,
                                int want_sys, const int32_t* __restrict__ col_ptr,
                                const int32_t* __restrict__ free_rank,
                                const int32_t* __restrict__ ff_col_ptr, int64_t* __restrict__ out) {
    const int32_t nf = want_sys ? free_rank[col_begin + n_cols] - free_rank[col_begin] : 0;
    out[0] = n_cols;
    out[1] = nf;
    out[2] = want_a ? col_ptr[n_cols] : 0;
    out[3] = want_sys ? ff_col_ptr[nf] : 0;
    (void)n_rows;
}

int launch_result_counts(fl_ctx* ctx, fl_result* res, int64_t* dev_out) {
    const bool want_a = res->what & FL_OUT_STIFFNESS, want_sys = res->what & FL_OUT_SYSTEM;
    k_result_counts<<<1, 1, 0, ctx->stream>>>(
        res->n, res->col_begin, res->m, want_a, want_sys, res->arr[FL_A_COL_PTR].as<int32_t>(),
        want_sys ? res->fidx.as<int32_t>() + (size_t)res->m + 1 : nullptr,
        res->arr[FL_AFF_COL_PTR].as<int32_t>(), dev_out);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// ---------------------------------------------------------------------------
// hybrid column pass: register kernel for columns of <= L incidences, the
// general kernel for the rest (unstructured meshes), per-column placement
// ---------------------------------------------------------------------------
__global__ void k_list_big(int32_t n_cols, int32_t n_nodes, int dim, int lanes,
                           const int32_t* __restrict__ inc_ptr, int32_t* __restrict__ list,
                           int32_t* __restrict__ ovidx, unsigned long long* __restrict__ acc) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; base < n_cols; base += stride) {
        const int32_t lc = (int32_t)(base + lane);
        const int32_t m = lc < n_cols ? inc_ptr[lc + 1] - inc_ptr[lc] : 0;
        const bool big = m > lanes;
        const unsigned bal = __ballot_sync(0xffffffffu, big);  // one atomic per warp
        int64_t bnd = big ? ((int64_t)m * dim + 1 < n_nodes ? (int64_t)m * dim + 1 : (int64_t)n_nodes) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bnd += __shfl_xor_sync(0xffffffffu, bnd, o);
        int32_t q0 = 0;
        if (lane == 0 && bal) {
            q0 = (int32_t)atomicAdd(acc, (unsigned long long)__popc(bal));
            atomicAdd(acc + 1, (unsigned long long)bnd);
        }
        q0 = __shfl_sync(0xffffffffu, q0, 0);
        int32_t q = -1;
        if (big) {
            q = q0 + __popc(bal & ((1u << lane) - 1));
            list[q] = lc;
        }
        if (lc < n_cols) ovidx[lc] = q;
    }
}

// entries of each owned column: register-kernel tiles (in-tile inclusive
// counts) or the general kernel's listed columns
__global__ void k_hyb_counts(ColParams p, int tc, const int32_t* __restrict__ ovidx, int32_t* __restrict__ ca,
                             int32_t* __restrict__ cf) {
    for (int32_t lc = blockIdx.x * blockDim.x + threadIdx.x; lc < p.n_cols; lc += gridDim.x * blockDim.x) {
        const int32_t q = ovidx[lc];
        int32_t a, f = 0;
        if (q >= 0) {
            a = p.ov_cnt[q];
            f = p.want_sys ? p.ov_cnt[p.n_list + q] : 0;
        } else {
            const bool first = lc % tc == 0;
            a = p.colcnt_a[lc] - (first ? 0 : p.colcnt_a[lc - 1]);
            if (p.want_sys) f = p.colcnt_f[lc] - (first ? 0 : p.colcnt_f[lc - 1]);
        }
        ca[lc] = a;
        cf[lc] = f;
    }
}

// warp per column: copy its entries from the tile staging or the overflow
// staging to col_ptr / the A(free,free) position
__global__ void k_hyb_copy(ColParams p, int tc, const int32_t* __restrict__ ovidx,
                           const int32_t* __restrict__ pf, const int32_t* __restrict__ ov_row,
                           const double* __restrict__ ov_val, const int32_t* __restrict__ ovf_row,
                           const double* __restrict__ ovf_val) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int32_t fb = free_base(p);
    for (int64_t lc64 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; lc64 < p.n_cols; lc64 += nw) {
        const int32_t lc = (int32_t)lc64;
        const int32_t q = ovidx[lc];
        const int32_t da = p.col_ptr[lc], na = p.col_ptr[lc + 1] - da;
        const int32_t df = pf[lc], nf = pf[lc + 1] - df;
        if ((int64_t)da + na > p.cap_a || (int64_t)df + nf > p.cap_ff) {
            if (lane == 0) atomicOr(p.err, DERR_CAPACITY);
            continue;
        }
        const int32_t* ra;
        const double* va;
        const int32_t* rf;
        const double* vf;
        if (q >= 0) {
            ra = ov_row + p.ov_off[q];
            va = ov_val + p.ov_off[q];
            rf = ovf_row + p.ov_off[p.n_list + q];
            vf = ovf_val + p.ov_off[p.n_list + q];
        } else {
            const int64_t t = lc / tc;
            const bool first = lc % tc == 0;
            const int64_t sa = t * p.tile_cap + (first ? 0 : p.colcnt_a[lc - 1]);
            ra = p.st_a_row + sa;
            va = p.st_a_val + sa;
            const int64_t sf = t * p.tile_cap + (first || !p.want_sys ? 0 : p.colcnt_f[lc - 1]);
            rf = p.st_f_row + sf;
            vf = p.st_f_val + sf;
        }
        for (int k = lane; k < na; k += 32) {
            p.row_idx[da + k] = ra[k];
            p.values[da + k] = va[k];
        }
        if (p.want_sys) {
            for (int k = lane; k < nf; k += 32) {
                p.ff_row_idx[df + k] = rf[k];
                p.ff_values[df + k] = vf[k];
            }
            const int32_t fc = p.fidx[p.c_begin + lc];
            if (lane == 0 && fc >= 0) p.ff_col_ptr[fc - fb + 1] = df + nf;
        }
    }
}

int launch_hybrid(fl_ctx* ctx, int dim, ColParams& p, fl_mesh* mesh, fl_result* res, bool pre) {
    const cudaStream_t s = ctx->stream;
    const int lanes = columns3_lanes(dim, mesh->max_inc);
    const int32_t NC = p.n_cols;
    // 1. the columns above the register kernel's valence, and their output bound
    FL_TRY(res->hyb[0].ensure(sizeof(int32_t) * 2 * ((size_t)NC + 1)));  // list | ovidx
    FL_TRY(res->hyb[1].ensure(sizeof(unsigned long long) * 4));
    int32_t* list = res->hyb[0].as<int32_t>();
    int32_t* ovidx = list + NC + 1;
    unsigned long long* acc = res->hyb[1].as<unsigned long long>();
    FL_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 4, s));
    k_list_big<<<std::max(1, std::min(div_up(NC, 256), ctx->sm_count * 8)), 256, 0, s>>>(
        NC, p.n_nodes, dim, lanes, p.inc_ptr, list, ovidx, acc);
    count_launch(ctx);
    unsigned long long* h = static_cast<unsigned long long*>(ctx->pinned);
    FL_CUDA(cudaMemcpyAsync(h, acc, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    const int32_t n_list = (int32_t)h[0];
    const int64_t bound = std::max<int64_t>((int64_t)h[1], 1);
    // 2. the register kernel over every column (listed ones left empty)
    p.hybrid = true;
    FL_TRY(launch_columns3(ctx, dim, p, mesh->max_inc, res, pre, false));
    // 3. the general kernel over the listed columns into overflow staging
    ColParams q = p;
    q.hybrid = false;
    q.col_list = list;
    q.n_list = n_list;
    FL_TRY(res->hyb[2].ensure(sizeof(int32_t) * 4 * ((size_t)n_list + 1)));
    q.ov_cnt = res->hyb[2].as<int32_t>();
    q.ov_off = q.ov_cnt + 2 * ((size_t)n_list + 1);
    for (int k = 0; k < 4; ++k)
        FL_TRY(res->hyb[3 + k].ensure((k % 2 ? sizeof(double) : sizeof(int32_t)) * (size_t)bound));
    q.row_idx = res->hyb[3].as<int32_t>();
    q.values = res->hyb[4].as<double>();
    q.ff_row_idx = res->hyb[5].as<int32_t>();
    q.ff_values = res->hyb[6].as<double>();
    q.ov_alloc = acc + 2;
    q.cap_a = q.want_a ? bound : 0;
    q.cap_ff = q.want_sys ? bound : 0;
    if (n_list > 0) {
        k_inc_sort<<<div_up(n_list, 128), 128, 0, s>>>(n_list, p.inc_ptr, const_cast<uint32_t*>(p.inc), list);
        count_launch(ctx);
        const int tw = column_tile_width();
        q.n_tiles = (n_list + tw - 1) / tw;
        FL_TRY(res->tile_status.ensure(sizeof(uint64_t) * ((size_t)q.n_tiles + 1)));
        FL_CUDA(cudaMemsetAsync(res->tile_status.p, 0, sizeof(uint64_t) * ((size_t)q.n_tiles + 1), s));
        q.tile_status = res->tile_status.as<uint64_t>();
        FL_CUDA(cudaMemsetAsync(q.ticket, 0, sizeof(uint32_t), s));
        FL_TRY(launch_columns(ctx, dim, q));
    }
    // 4. per-column placement
    if (!p.want_a) return FL_OK;
    const int tc = dim == 2 ? 32 : 8;  // the register kernel's columns per tile (V3::WTC)
    FL_TRY(res->hyb[7].ensure(sizeof(int32_t) * 3 * ((size_t)NC + 1)));
    int32_t* ca = res->hyb[7].as<int32_t>();
    int32_t* cf = ca + NC + 1;
    int32_t* pf = cf + NC + 1;
    ColParams r = p;
    r.ov_cnt = q.ov_cnt;
    r.ov_off = q.ov_off;
    r.n_list = n_list;
    const int g = std::max(1, std::min(div_up(NC, 256), ctx->sm_count * 8));
    k_hyb_counts<<<g, 256, 0, s>>>(r, tc, ovidx, ca, cf);
    count_launch(ctx);
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(NC)));
    const int32_t* cac = ca;
    FL_CUDA(launch_scan<int32_t>(NC, [cac] __device__(int64_t i) { return (int64_t)cac[i]; }, p.col_ptr,
                                 ctx->scan_ws.p, s));
    const int32_t* cfc = cf;
    FL_CUDA(launch_scan<int32_t>(NC, [cfc] __device__(int64_t i) { return (int64_t)cfc[i]; }, pf,
                                 ctx->scan_ws.p, s));
    count_launch(ctx, 2);
    const int64_t warps = std::min<int64_t>(NC, (int64_t)ctx->sm_count * 64);
    k_hyb_copy<<<(int)std::max<int64_t>(1, (warps * 32 + 255) / 256), 256, 0, s>>>(
        r, tc, ovidx, pf, q.row_idx, q.values, q.ff_row_idx, q.ff_values);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// ---------------------------------------------------------------------------
// Neumann shares for the register kernel (apply_neumann, system.hpp:123-172):
// add[c] = 0.0 + the shares of the flag-2 faces containing node c in face-major
// (lf, t) order; the column kernel (id-space register kernel or the label-space
// one) then forms b[c] + add[c].  Warp per node on a flag-2 face.
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(kWarps * 32) k_neumann_add(ColParams p, double* __restrict__ add_out) {
    const unsigned FULL = 0xffffffffu;
    __shared__ uint32_t skey[kWarps][kMaxNeu];
    __shared__ double sval[kWarps][kMaxNeu];
    __shared__ int scnt[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const Recip R3 = recip(3.0);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t lc64 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; lc64 < p.n_cols; lc64 += nw) {
        const int32_t lc = (int32_t)lc64, c = p.c_begin + lc;
        if (!p.is_neu[c]) continue;  // warp-uniform
        if (lane == 0) scnt[w] = 0;
        __syncwarp();
        // the node's incidences: its id-space segment, or (label plan) the first
        // lcnt[l] of the lcap slots of its label l
        int64_t p0;
        int32_t m;
        if (p.lcnt) {
            const int32_t l = __ldg(p.lab + c);
            p0 = (int64_t)l * p.lcap;
            m = min(__ldg(p.lcnt + l), p.lcap);
        } else {
            p0 = p.inc_ptr[lc];
            m = p.inc_ptr[lc + 1] - (int32_t)p0;
        }
        for (int base = 0; base < m; base += 32) {
            if (base + lane < m) {
                const uint32_t key = __ldg(p.inc + p0 + base + lane);
                const int32_t t = (int32_t)(key & 0x3FFFFFFFu);
                const int j = (int)(key >> 30);
                int32_t R[D + 1];
#pragma unroll
                for (int i = 0; i <= D; ++i) R[i] = __ldg(p.elems + (size_t)t * (D + 1) + i);
                ElemCol<D> ec;
                ec.load(p.nodes, R);
                for (int lf = 0; lf <= D; ++lf) {
                    if (lf == j || p.flags[(size_t)t * (D + 1) + lf] != 2) continue;
                    const int q = atomicAdd(&scnt[w], 1);
                    if (q < kMaxNeu) {
                        skey[w][q] = ((uint32_t)lf << 30) | (uint32_t)t;
                        sval[w][q] = ec.face_share(lf, p.g_neu, R3, t);
                    } else {
                        atomicOr(p.err, DERR_OVERFLOW);
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) {  // face-major (lf, t) order (mesh.hpp:222-246), from 0.0
            const int n = min(scnt[w], kMaxNeu);
            double a = 0.0;
            uint32_t last = 0;
            bool first = true;
            for (int r = 0; r < n; ++r) {
                int best = -1;
                for (int q = 0; q < n; ++q) {
                    const uint32_t k2 = skey[w][q];
                    if ((first || k2 > last) && (best < 0 || k2 < skey[w][best])) best = q;
                }
                last = skey[w][best];
                first = false;
                a = a + sval[w][best];
            }
            add_out[lc] = a;
        }
        __syncwarp(FULL);
    }
}

int launch_neumann_add(fl_ctx* ctx, int dim, ColParams& p, fl_result* res) {
    FL_TRY(res->hyb[8].ensure(sizeof(double) * ((size_t)p.n_cols + 1)));
    double* add = res->hyb[8].as<double>();
    const int64_t warps = std::min<int64_t>(std::max<int32_t>(p.n_cols, 1), (int64_t)ctx->sm_count * 64);
    const int grid = (int)std::max<int64_t>(1, (warps + kWarps - 1) / kWarps);
    if (dim == 2) k_neumann_add<2><<<grid, kWarps * 32, 0, ctx->stream>>>(p, add);
    else k_neumann_add<3><<<grid, kWarps * 32, 0, ctx->stream>>>(p, add);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    p.nadd = add;
    return FL_OK;
}

int launch_validate(fl_ctx* ctx, fl_mesh* mesh, uint32_t* d_err) {
    if (mesh->n_elems == 0) return FL_OK;
    const int grid = std::min(div_up(mesh->n_elems, 256), ctx->sm_count * 16);
    const int8_t* fl = mesh->has_flags ? mesh->flags.as<int8_t>() : nullptr;
    if (mesh->dim == 2)
        k_validate<2><<<grid, 256, 0, ctx->stream>>>(mesh->n_elems, mesh->n_nodes,
                                                     mesh->nodes.as<double>(),
                                                     mesh->elems.as<int32_t>(), fl, d_err);
    else
        k_validate<3><<<grid, 256, 0, ctx->stream>>>(mesh->n_elems, mesh->n_nodes,
                                                     mesh->nodes.as<double>(),
                                                     mesh->elems.as<int32_t>(), fl, d_err);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

int launch_partition(fl_ctx* ctx, fl_mesh* mesh, fl_result* res) {
    const cudaStream_t s = ctx->stream;
    const int32_t N = mesh->n_nodes;
    const int64_t n_entries = (int64_t)mesh->n_elems * (mesh->dim + 1);
    uint32_t* counters = res->counters.as<uint32_t>();
    int8_t* is_dir = res->is_dir.as<int8_t>();
    int8_t* is_neu = res->is_neu.as<int8_t>();
    FL_CUDA(cudaMemsetAsync(is_dir, 0, (size_t)N + 1, s));
    FL_CUDA(cudaMemsetAsync(is_neu, 0, (size_t)N + 1, s));
    if (mesh->has_flags && n_entries > 0) {
        const int grid = (int)std::min<int64_t>(div_up(n_entries, 256), (int64_t)ctx->sm_count * 16);
        if (mesh->dim == 2)
            k_mark_boundary<2><<<grid, 256, 0, s>>>(mesh->n_elems, N, mesh->elems.as<int32_t>(),
                                                   mesh->flags.as<int8_t>(), is_dir, is_neu, counters);
        else
            k_mark_boundary<3><<<grid, 256, 0, s>>>(mesh->n_elems, N, mesh->elems.as<int32_t>(),
                                                   mesh->flags.as<int8_t>(), is_dir, is_neu, counters);
        count_launch(ctx);
    }
    // free_rank = exclusive scan of (1 - is_dir) into the FL_B_F slot's int32 twin
    int32_t* free_rank = res->fidx.as<int32_t>() + ((size_t)N + 1);
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(N)));
    const int8_t* isd = is_dir;
    FL_CUDA(launch_scan<int32_t>(
        N, [isd] __device__(int64_t i) { return (int64_t)(isd[i] ? 0 : 1); }, free_rank,
        ctx->scan_ws.p, s));
    count_launch(ctx);
    k_partition<<<std::max(1, std::min(div_up(N, 256), ctx->sm_count * 8)), 256, 0, s>>>(
        N, is_dir, free_rank, res->fidx.as<int32_t>(), res->arr[FL_DIR_NODES].as<int32_t>(),
        res->arr[FL_FREE_NODES].as<int32_t>(), counters);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// ---------------------------------------------------------------------------
// apply_dirichlet (system.hpp:182-201) for a caller-supplied A and b:
// u0 = g at Dirichlet nodes (0 elsewhere), b - matvec(A, u0) (sparse.hpp:129-141).
// ---------------------------------------------------------------------------
__global__ void k_dirichlet_u0(int32_t n, const int8_t* __restrict__ is_dir, FieldDesc g,
                               const double* __restrict__ nodes, int dim, double* __restrict__ u0) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        u0[k] = is_dir[k] ? field_at_node(g, nodes, dim, k) : 0.0;
}

__global__ void k_sub(int32_t n, const double* __restrict__ b, const double* __restrict__ y,
                      double* __restrict__ out) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        out[k] = b[k] - y[k];  // system.hpp:197-198
}

int launch_dirichlet_lift(fl_ctx* ctx, fl_mesh* mesh, fl_result* res, const FieldDesc& g,
                          const int32_t* col_ptr, const int32_t* row_idx, const double* values,
                          const double* b) {
    const int32_t N = mesh->n_nodes;
    const cudaStream_t s = ctx->stream;
    FL_TRY(res->arr[FL_U0].ensure(sizeof(double) * ((size_t)N + 1)));
    FL_TRY(res->arr[FL_B_MOD].ensure(sizeof(double) * ((size_t)N + 1)));
    FL_TRY(res->v4[2].ensure(sizeof(double) * ((size_t)N + 1)));
    double* u0 = res->arr[FL_U0].as<double>();
    double* au0 = res->v4[2].as<double>();
    const int grid = std::max(1, std::min(div_up(N, 256), ctx->sm_count * 8));
    if (N > 0) {
        k_dirichlet_u0<<<grid, 256, 0, s>>>(N, res->is_dir.as<int8_t>(), g, mesh->nodes.as<double>(), mesh->dim, u0);
        count_launch(ctx);
    }
    FL_TRY(matvec_device(ctx, N, N, col_ptr, row_idx, values, u0, au0));
    if (N > 0) {
        k_sub<<<grid, 256, 0, s>>>(N, b, au0, res->arr[FL_B_MOD].as<double>());
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// accumulate (sparse.hpp:186-198) from a one-column from_triplets result:
// out = 0.0 everywhere, then out[row] = the entry (the duplicate sum in original
// order; exactly-zero sums were dropped and stay 0.0, as 0.0 + ... gives there)
__global__ void k_scatter_column(int32_t nnz_unused, const int32_t* __restrict__ col_ptr,
                                 const int32_t* __restrict__ row_idx, const double* __restrict__ values,
                                 double* __restrict__ out) {
    (void)nnz_unused;
    const int32_t nnz = col_ptr[1];
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += gridDim.x * blockDim.x)
        out[row_idx[k]] = values[k];
}

int launch_scatter_column(fl_ctx* ctx, fl_result* col, int32_t size, double* out) {
    FL_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)size, ctx->stream));
    k_scatter_column<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(0, col->arr[FL_A_COL_PTR].as<int32_t>(),
                                                                 col->arr[FL_A_ROW_IDX].as<int32_t>(),
                                                                 col->arr[FL_A_VALUES].as<double>(), out);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

int launch_face_lists(fl_ctx* ctx, fl_mesh* mesh, fl_result* res) {
    const cudaStream_t s = ctx->stream;
    const int D = mesh->dim, NV = D + 1;
    const int32_t NT = mesh->n_elems;
    // capacity: at most one face per (t, lf)
    const size_t cap = (size_t)std::max<int64_t>((int64_t)NT * NV, 1);
    FL_TRY(res->arr[FL_DIR_FACES].ensure(sizeof(int32_t) * cap * D));
    FL_TRY(res->arr[FL_DIR_FACE_ELEM].ensure(sizeof(int32_t) * cap));
    FL_TRY(res->arr[FL_DIR_FACE_LOCAL].ensure(sizeof(int32_t) * cap));
    FL_TRY(res->arr[FL_NEU_FACES].ensure(sizeof(int32_t) * cap * D));
    FL_TRY(res->arr[FL_NEU_FACE_ELEM].ensure(sizeof(int32_t) * cap));
    FL_TRY(res->arr[FL_NEU_FACE_LOCAL].ensure(sizeof(int32_t) * cap));
    if (!mesh->has_flags || NT == 0) return FL_OK;  // no flags: empty lists
    const int32_t nblk = (int32_t)(((int64_t)NT + kFaceBlockElems - 1) / kFaceBlockElems);
    const int64_t ncat = (int64_t)NV * nblk;  // per value
    FL_TRY(res->v4[3].ensure(sizeof(int32_t) * (size_t)(4 * ncat + 2)));
    int32_t* bcnt = res->v4[3].as<int32_t>();
    int32_t* boff = bcnt + 2 * ncat;
    if (D == 2) k_face_count<2><<<nblk, kFaceThreads, 0, s>>>(NT, mesh->flags.as<int8_t>(), nblk, bcnt);
    else k_face_count<3><<<nblk, kFaceThreads, 0, s>>>(NT, mesh->flags.as<int8_t>(), nblk, bcnt);
    count_launch(ctx);
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(ncat)));
    for (int v = 0; v < 2; ++v) {
        const int32_t* src = bcnt + v * ncat;
        FL_CUDA(launch_scan<int32_t>(
            ncat, [src] __device__(int64_t i) { return (int64_t)src[i]; }, boff + v * ncat, ctx->scan_ws.p, s));
        count_launch(ctx);
    }
    // launch_scan writes out[n] = total past each region's end: the Neumann
    // region is scanned second, so the Dirichlet total it overwrote is not used
    auto emit = D == 2 ? k_face_emit<2> : k_face_emit<3>;
    emit<<<nblk, kFaceThreads, 0, s>>>(NT, mesh->elems.as<int32_t>(), mesh->flags.as<int8_t>(), nblk, boff,
                                       res->arr[FL_DIR_FACES].as<int32_t>(), res->arr[FL_DIR_FACE_ELEM].as<int32_t>(),
                                       res->arr[FL_DIR_FACE_LOCAL].as<int32_t>(), res->arr[FL_NEU_FACES].as<int32_t>(),
                                       res->arr[FL_NEU_FACE_ELEM].as<int32_t>(),
                                       res->arr[FL_NEU_FACE_LOCAL].as<int32_t>());
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

int launch_columns(fl_ctx* ctx, int dim, ColParams& p) {
    const size_t smem = column_smem_bytes();
    const int grid_max = ctx->sm_count * 4;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.n_tiles, grid_max));
    if (dim == 2) {
        FL_CUDA(cudaFuncSetAttribute(k_columns<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        k_columns<2><<<grid, kWarps * 32, smem, ctx->stream>>>(p);
    } else {
        FL_CUDA(cudaFuncSetAttribute(k_columns<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        k_columns<3><<<grid, kWarps * 32, smem, ctx->stream>>>(p);
    }
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

int launch_submatrix(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr,
                     const int32_t* row_idx, const double* values, int32_t n_rows,
                     const int32_t* rows, int32_t n_cols, const int32_t* cols, fl_result* res,
                     int32_t* row_map, int32_t* cnt, uint32_t* d_err, int64_t* nnz_out) {
    const cudaStream_t s = ctx->stream;
    FL_CUDA(cudaMemsetAsync(row_map, 0xFF, sizeof(int32_t) * ((size_t)m + 1), s));
    if (n_rows > 0) {
        k_sub_rowmap<<<std::max(1, std::min(div_up(n_rows, 256), ctx->sm_count * 8)), 256, 0, s>>>(
            n_rows, rows, row_map, m, d_err);
        count_launch(ctx);
    }
    if (n_cols > 0) {
        k_sub_count<<<std::max(1, std::min(div_up(n_cols, 256), ctx->sm_count * 8)), 256, 0, s>>>(
            n_cols, cols, n, col_ptr, row_idx, row_map, cnt, d_err);
        count_launch(ctx);
    }
    FL_TRY(res->arr[FL_A_COL_PTR].ensure(sizeof(int32_t) * ((size_t)n_cols + 1)));
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(n_cols)));
    const int32_t* cc = cnt;
    FL_CUDA(launch_scan<int32_t>(
        n_cols, [cc] __device__(int64_t i) { return (int64_t)cc[i]; },
        res->arr[FL_A_COL_PTR].as<int32_t>(), ctx->scan_ws.p, s));
    count_launch(ctx);
    // total -> host (needed to size the outputs)
    int32_t total = 0;
    FL_CUDA(cudaMemcpyAsync(ctx->pinned, res->arr[FL_A_COL_PTR].as<int32_t>() + n_cols,
                            sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    uint32_t herr = 0;
    FL_CUDA(cudaMemcpyAsync(static_cast<char*>(ctx->pinned) + 8, d_err, sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    total = *static_cast<int32_t*>(ctx->pinned);
    herr = *reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->pinned) + 8);
    if (herr & (1u | 4u)) return set_error(FL_E_INDEX_OUT_OF_RANGE, "submatrix: index out of range");
    if (herr & (2u | 8u))
        return set_error(FL_E_UNSORTED_INDEX_SET, "submatrix: index set is not strictly increasing");
    FL_TRY(res->arr[FL_A_ROW_IDX].ensure(sizeof(int32_t) * ((size_t)total + 1)));
    FL_TRY(res->arr[FL_A_VALUES].ensure(sizeof(double) * ((size_t)total + 1)));
    if (n_cols > 0) {
        k_sub_fill<<<std::max(1, std::min(div_up(n_cols, 256), ctx->sm_count * 8)), 256, 0, s>>>(
            n_cols, cols, col_ptr, row_idx, values, row_map, res->arr[FL_A_COL_PTR].as<int32_t>(),
            res->arr[FL_A_ROW_IDX].as<int32_t>(), res->arr[FL_A_VALUES].as<double>());
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    *nnz_out = total;
    return FL_OK;
}

int launch_selftest_div(fl_ctx* ctx, int64_t n, const double* a, const double* b, double* qf,
                        double* qi) {
    if (n <= 0) return FL_OK;
    k_selftest_div<<<(int)std::min<int64_t>(div_up(n, 256), ctx->sm_count * 16), 256, 0,
                     ctx->stream>>>(n, a, b, qf, qi);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

}  // namespace fl
