// fl_columns4.cu -- the label-space pipeline (v4), default fast path of fl_assemble.
//
// Why labels.  The reference's output is in node-id order, and config C5 (and
// C3) number their nodes randomly.  Indexing the plan, the coordinates and the
// partition by node id turns every access of the column pass into a random
// DRAM sector: the id-space v3 pass read 109 GB on C5 for 3.6 GB of compulsory
// traffic.  Here every node gets a LABEL -- its place in the Morton order of the
// nodes' coordinates (cells of ~8 nodes) -- and all intermediate work runs in
// label order:
//
//   plan     k4_bbox / k4_cell / scan / k4_cell_scatter   labels (lab: node -> label)
//            k4_fill      one pass over the elements: (j << 30 | t) keys into
//                         fixed-capacity label segments (the per-label count is
//                         the cursor: no count pass, no scan) and the elements
//                         rewritten with vertex labels (lel); large 2-D meshes
//                         go through buckets of labels (k4_bucket_scatter + k4_fill_b)
//            k4_stats     nnz bound and maximum valence
//   per call k4_xl        xl[label] = node coordinates + {node id, free rank}
//            k_columns4   one group of L lanes per column (label), K incidences
//                         per lane: element geometry computed in the kernel from
//                         xl (no element-record round trip through HBM), the
//                         reference's exact per-entry fold order, zero drop,
//                         load vector, Neumann shares, Dirichlet lift,
//                         A(free,free); entries staged at the column's node id
//            k4_place     CSC column pointers in node-id order (scan + look-back),
//                         staged runs streamed to their CSC positions, vectors
//
// A column range (multi-GPU shard) labels its own nodes first, so the plan and the
// column pass cover labels [0, n_owned) only.
//
// Labels never reach the output: rows are node ids, every fold runs in the
// reference's (i*(d+1)+j, t) order with the original element index t, so the
// result is bitwise the id-space pipeline's (and the reference's) whatever the
// labelling.  Citations: /root/reference/proj/include/femlite/<file>:<line>.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

constexpr unsigned kFull = 0xffffffffu;
__host__ __device__ constexpr int lg2c(int x) { return x <= 1 ? 0 : 1 + lg2c(x >> 1); }

// ===========================================================================
// plan
// ===========================================================================
constexpr int kP4Block = 256;

// misc buffer layout: u64 stats[4] (nnz bound, max valence, -, -), u32 spare,
// u32 error word (read back as the high half of the fifth u64)
struct P4Misc {
    unsigned long long stats[4];
    uint32_t spare;
    uint32_t err;
};

// ---- labels: nodes bucketed by the Morton cell of their coordinates (cells of ~8
// nodes along a Z-curve over the bounding box), whatever the element order (C3
// permutes its elements: a first-touch order of the element stream is random there).
__global__ void k4_bbox(int32_t n, int dim, const double* __restrict__ nodes, double* __restrict__ part) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        for (int d = 0; d < dim; ++d) {
            const double x = __ldg(nodes + (size_t)v * dim + d);
            lo[d] = fmin(lo[d], x);
            hi[d] = fmax(hi[d], x);
        }
    __shared__ double s[6][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fmin(lo[d], __shfl_xor_sync(kFull, lo[d], o));
            hi[d] = fmax(hi[d], __shfl_xor_sync(kFull, hi[d], o));
        }
        if (lane == 0) {
            s[d][w] = lo[d];
            s[3 + d][w] = hi[d];
        }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
        double r = s[threadIdx.x][0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
            r = threadIdx.x < 3 ? fmin(r, s[threadIdx.x][i]) : fmax(r, s[threadIdx.x][i]);
        part[blockIdx.x * 6 + threadIdx.x] = r;
    }
}

__device__ __forceinline__ uint32_t spread3(uint32_t x) {  // 10 bits -> every third bit
    x &= 0x3FFu;
    x = (x | (x << 16)) & 0x030000FFu;
    x = (x | (x << 8)) & 0x0300F00Fu;
    x = (x | (x << 4)) & 0x030C30C3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}
__device__ __forceinline__ uint32_t spread2(uint32_t x) {  // 15 bits -> every second bit
    x &= 0x7FFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// cell of every node (Morton code of its quantised coordinates) and per-cell counts
// A column range [c0, c1) (multi-GPU shard) puts the nodes outside it into a
// second run of cells: the owned nodes take labels [0, c1 - c0), still in Morton
// order, and every other node keeps a label for its xl record.
__global__ void k4_cell(int32_t n, int dim, int bits, int nparts, const double* __restrict__ nodes,
                        const double* __restrict__ part, int32_t c0, int32_t c1, int32_t* __restrict__ cell,
                        int32_t* __restrict__ ccnt) {
    __shared__ double box[6];
    if (threadIdx.x < 6) {
        double r = part[threadIdx.x];
        for (int b = 1; b < nparts; ++b) r = threadIdx.x < 3 ? fmin(r, part[b * 6 + threadIdx.x]) : fmax(r, part[b * 6 + threadIdx.x]);
        box[threadIdx.x] = r;
    }
    __syncthreads();
    const double side = (double)(1u << bits);
    double sc[3];
    for (int d = 0; d < 3; ++d) sc[d] = box[3 + d] > box[d] ? side / (box[3 + d] - box[d]) : 0.0;
    const uint32_t qmax = (1u << bits) - 1;
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        uint32_t q[3] = {0, 0, 0};
        for (int d = 0; d < dim; ++d) {
            const double x = __ldg(nodes + (size_t)v * dim + d);
            const double f = (x - box[d]) * sc[d];
            q[d] = f > 0.0 ? min((uint32_t)f, qmax) : 0u;  // NaN coordinates land in cell 0
        }
        uint32_t code = dim == 3 ? (spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2))
                                 : (spread2(q[0]) | (spread2(q[1]) << 1));
        if (v < c0 || v >= c1) code += 1u << (dim * bits);
        cell[v] = (int32_t)code;
        atomicAdd(ccnt + code, 1);
    }
}

// label = the node's place in its cell's run (cursor seeded with the cell offsets)
__global__ void k4_cell_scatter(int32_t n, const int32_t* __restrict__ cell, int32_t* __restrict__ cursor,
                                int32_t* __restrict__ lab) {
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        lab[v] = atomicAdd(cursor + __ldg(cell + v), 1);
}

// lel rows are 4 labels wide in both dimensions (a triangle's row is one aligned
// 16-byte load in the column kernel, not three 4-byte ones: the 2-D kernel is bound
// by L1 wavefronts)
__device__ __forceinline__ int64_t lel_index(int64_t e, int nv) {
    if (nv == 4) return e;
    const int32_t t = entry_elem(e, nv);
    return (int64_t)t * 4 + (e - (int64_t)t * nv);
}

// (j << 30 | t) keys into the label segments and the elements with vertex labels
// (lel), one pass: label l owns the `cap` slots linc[l * cap ..], its count
// cnt[l] (zeroed before) is the fill cursor -- no separate count pass, no scan.
// Slots beyond cap are dropped; the count keeps running, so a valence above cap
// shows in the statistics and in the column kernel (which then defers to the
// general kernel).  U rounds of 32 consecutive entries per warp, blocks issued in
// element order (the live segments stay in L2 until their sectors are complete).
template <int U>
__global__ void k4_fill(int64_t n_entries, int nv, int32_t n_nodes, int32_t c0, int32_t c1, int cap,
                        const int32_t* __restrict__ elems, const int32_t* __restrict__ lab,
                        int32_t* __restrict__ cnt, uint32_t* __restrict__ linc, int32_t* __restrict__ lel,
                        P4Misc* __restrict__ misc) {
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1;
    const bool sharded = c0 > 0 || c1 < n_nodes;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t err = 0;
    // persistent warps: the next iteration's vertex ids are loaded one iteration
    // ahead (the chain per iteration is then label gather -> atomic -> store)
    int32_t vnext[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t e = warp * 32 * U + u * 32 + lane;
        vnext[u] = e < n_entries ? __ldg(elems + e) : -1;
    }
    for (int64_t e0 = warp * 32 * U; e0 < n_entries; e0 += nwarps * 32 * U) {
        int32_t key[U], vtx[U];
        bool tch[U];
        unsigned grp[U];
        int32_t pos[U];
        int32_t vcur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            vcur[u] = vnext[u];
            const int64_t en = e0 + nwarps * 32 * U + u * 32 + lane;
            vnext[u] = en < n_entries ? __ldg(elems + en) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * 32 + lane;
            key[u] = -1;
            vtx[u] = -1;
            tch[u] = false;
            if (e < n_entries) {
                const int32_t v = vcur[u];
                // a shard skips the elements that touch none of its columns: no
                // label gather, no lel row (the column pass never reads it)
                bool touched = true;
                if (sharded && nv != 4) {  // (nv == 4: the element's four lanes vote below)
                    const int64_t t0 = (int64_t)entry_elem(e, nv) * nv;
                    touched = false;
                    for (int i = 0; i < nv; ++i) {
                        const int32_t w = __ldg(elems + t0 + i);
                        touched = touched || (w >= c0 && w < c1);
                    }
                }
                vtx[u] = v;
                tch[u] = touched;
            }
        }
        if (sharded && nv == 4) {
            // a tetrahedron's entries sit in four consecutive lanes (rounds start at
            // multiples of 32): touched = any of them owned
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool own = vtx[u] >= c0 && vtx[u] < c1;
                const unsigned b = __ballot_sync(kFull, own);
                tch[u] = ((b >> (lane & ~3)) & 0xFu) != 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + u * 32 + lane;
            if (e < n_entries) {
                const int32_t v = vtx[u];
                const bool touched = tch[u];
                if ((uint32_t)v >= (uint32_t)n_nodes) err = DERR_INDEX;
                if (touched) {
                    int32_t lb = -1;
                    if ((uint32_t)v < (uint32_t)n_nodes) lb = __ldg(lab + v);
                    lel[lel_index(e, nv)] = lb;
                    if (v >= c0 && v < c1) key[u] = lb;  // keys for this shard's columns only
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) grp[u] = __match_any_sync(kFull, key[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pos[u] = 0;
            if (key[u] >= 0 && (grp[u] & lower) == 0) pos[u] = atomicAdd(cnt + key[u], __popc(grp[u]));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t p0 = __shfl_sync(kFull, pos[u], __ffs(grp[u]) - 1) + __popc(grp[u] & lower);
            if (key[u] >= 0 && p0 < cap) {
                const int64_t e = e0 + u * 32 + lane;
                const int32_t t = entry_elem(e, nv);
                const uint32_t j = (uint32_t)(e - (int64_t)t * nv);
                linc[(int64_t)key[u] * cap + p0] = (j << 30) | (uint32_t)t;
            }
        }
    }
    if (__any_sync(kFull, err != 0) && lane == 0) atomicOr(&misc->err, DERR_INDEX);
}

// ---- bucketed fill (large 2-D meshes, element order not spatial: C3).  The
// direct fill scatters 4-byte keys over the whole incidence array there, each a
// sector read-modify-write.  Instead: (1) partition (label, key) pairs into
// buckets of 2^shift consecutive labels (block-local shared-memory ranks, one
// global reservation per bucket per block: coalesced runs), writing lel on the
// way; bucket b's staging area is its labels' capacity, (b << shift) * cap on;
// (2) fill from the staging in bucket order, so the live range of the
// incidence array is one bucket's slice, resident in L2.
constexpr int kB4Items = 16, kB4MaxBuckets = 1024;

__global__ void __launch_bounds__(kP4Block)
k4_bucket_scatter(int64_t n_entries, int nv, int32_t n_nodes, int32_t c0, int32_t c1, int shift, int cap,
                  const int32_t* __restrict__ elems, const int32_t* __restrict__ lab,
                  int32_t* __restrict__ bcur, int2* __restrict__ stage, int32_t* __restrict__ lel,
                  P4Misc* __restrict__ misc) {
    __shared__ int32_t hist[kB4MaxBuckets];
    __shared__ int32_t base[kB4MaxBuckets];
    const int nb = ((n_nodes - 1) >> shift) + 1;
    const bool sharded = c0 > 0 || c1 < n_nodes;
    constexpr int CH = kP4Block * kB4Items;
    const int64_t e0 = (int64_t)blockIdx.x * CH;
    for (int b = threadIdx.x; b < nb; b += kP4Block) hist[b] = 0;
    __syncthreads();
    int32_t lv[kB4Items], rk[kB4Items];
    uint32_t key[kB4Items];
    uint32_t err = 0;
#pragma unroll
    for (int k = 0; k < kB4Items; ++k) {
        const int64_t e = e0 + k * kP4Block + threadIdx.x;
        lv[k] = -1;
        if (e < n_entries) {
            const int32_t v = __ldg(elems + e);
            bool touched = true;  // a shard skips the elements touching none of its columns
            if (sharded) {
                const int64_t t0 = (int64_t)entry_elem(e, nv) * nv;
                touched = false;
                for (int i = 0; i < nv; ++i) {
                    const int32_t w = __ldg(elems + t0 + i);
                    touched = touched || (w >= c0 && w < c1);
                }
            }
            if ((uint32_t)v >= (uint32_t)n_nodes) err = DERR_INDEX;
            if (touched) {
                if ((uint32_t)v < (uint32_t)n_nodes) lv[k] = __ldg(lab + v);
                lel[lel_index(e, nv)] = lv[k];
            }
            if (v < c0 || v >= c1) lv[k] = -1;  // staged for this shard's columns only
            if (lv[k] >= 0) {
                const int32_t t = entry_elem(e, nv);
                key[k] = ((uint32_t)(e - (int64_t)t * nv) << 30) | (uint32_t)t;
                rk[k] = atomicAdd(&hist[lv[k] >> shift], 1);
            }
        }
    }
    if (err) atomicOr(&misc->err, DERR_INDEX);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += kP4Block)
        if (hist[b]) base[b] = atomicAdd(bcur + b, hist[b]);
    __syncthreads();
    const int32_t bucket_cap = cap << shift;
#pragma unroll
    for (int k = 0; k < kB4Items; ++k)
        if (lv[k] >= 0) {
            const int b = lv[k] >> shift;
            const int32_t q = base[b] + rk[k];
            if (q < bucket_cap) stage[(int64_t)b * bucket_cap + q] = make_int2(lv[k], (int32_t)key[k]);
            else atomicOr(&misc->err, DERR_V2_OVERFLOW);  // some label of the bucket exceeds cap
        }
}

// staged incidences in bucket order -> their label segments.  Block = (bucket,
// chunk of 4 * 256 staged entries); chunks past the bucket's count exit.
__global__ void __launch_bounds__(kP4Block)
k4_fill_b(int shift, int cap, int chunks_per_bucket, const int32_t* __restrict__ bcur,
          const int2* __restrict__ stage, int32_t* __restrict__ cnt, uint32_t* __restrict__ linc) {
    const int b = blockIdx.x / chunks_per_bucket, ch = blockIdx.x - b * chunks_per_bucket;
    const int32_t bucket_cap = cap << shift;
    const int32_t n_staged = min(__ldg(bcur + b), bucket_cap);
    const int32_t q0 = (ch * kP4Block + threadIdx.x) * 4;
    if (q0 >= n_staged) return;
    const int2* st = stage + (int64_t)b * bucket_cap;
    int2 sv[4];
    int32_t pos[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sv[u] = q0 + u < n_staged ? __ldg(st + q0 + u) : make_int2(-1, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) pos[u] = sv[u].x >= 0 ? atomicAdd(cnt + sv[u].x, 1) : 0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
        if (sv[u].x >= 0 && pos[u] < cap) linc[(int64_t)sv[u].x * cap + pos[u]] = (uint32_t)sv[u].y;
}

// stats[0] += sum_l min(m_l d + 1, N) (nnz upper bound), stats[1] = max m_l
__global__ void k4_stats(int32_t n, int32_t n_rows, int dim, const int32_t* __restrict__ lcnt,
                         P4Misc* __restrict__ misc) {
    int64_t bound = 0;
    int32_t mx = 0;
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int32_t m = lcnt[c];
        const int64_t b = (int64_t)m * dim + 1;
        bound += b < n_rows ? b : n_rows;
        mx = m > mx ? m : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bound += __shfl_xor_sync(kFull, bound, o);
        const int32_t y = __shfl_xor_sync(kFull, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&misc->stats[0], (unsigned long long)bound);
        atomicMax(&misc->stats[1], (unsigned long long)mx);
    }
}

// ===========================================================================
// per call: label-ordered nodes
// ===========================================================================
__global__ void k4_xl(int32_t n, int dim, const int32_t* __restrict__ lab, const double* __restrict__ nodes,
                      const int32_t* __restrict__ fidx, double4* __restrict__ xl) {
    // node order in, label order out: the coordinates, labels and free ranks are
    // read as streams and each record is one full 32-byte sector written at the
    // node's label (a gather by label read 3.5 GB of DRAM for 0.41 GB of nodes on C5)
    for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const int32_t l = __ldg(lab + v);
        const double* p = nodes + (size_t)v * dim;
        const double x = __ldg(p), y = __ldg(p + 1), z = dim == 3 ? __ldg(p + 2) : 0.0;
        const int32_t fr = fidx ? __ldg(fidx + v) : 0;
        xl[l] = make_double4(x, y, z, __hiloint2double(fr, v));
    }
}

// ===========================================================================
// column kernel
// ===========================================================================

template <int D, int L, int K>
struct V4 {
    static constexpr int NV = D + 1;
    static constexpr int GPW = 32 / L;                 // column groups per warp
    static constexpr int LK = L * K;                   // incidences a group takes (<= 32)
    static constexpr int HS = D == 2 ? 16 : 32;        // slot table entries per group
    static constexpr int MAXS = D == 2 ? 12 : 24;      // distinct rows accepted per column
    static constexpr int WTC = D == 2 ? 32 : 16;       // columns per warp tile
    static constexpr int ITERS = WTC / GPW;
    static constexpr int WARPS = D == 3 ? 2 : 4;       // warps per CTA (static smem <= 48 KB)
    static_assert(LK <= 32, "pass masks are 32-bit");
};

template <int D, int L, int K, bool LIFT>
struct V4Smem {  // one per column group
    using C = V4<D, L, K>;
    static constexpr int NV = D + 1;
    alignas(16) int32_t row[C::HS];    // slot -> row (node id, -1 empty)
    // occupied rows, compacted (-1 padded); during the incidence loop the same
    // words hold each lane's vertex node ids (lr[g * NV + i]) -- read back with a
    // run-time i instead of a register select chain
    union alignas(16) {
        int32_t crow[C::HS];
        int32_t lr[L * NV > C::HS ? L * NV : C::HS];
    };
    int32_t lfr[L * NV];               // ... and their free ranks
    int32_t cslot[C::HS];              // their slots (the sorted keys during the incidence loop)
    int32_t frk[C::HS];                // slot -> free rank of the row (-1: Dirichlet)
    uint32_t msk[C::HS][NV];           // slot -> pass-i mask over incidences
    // items and folds first; once every fold is done the same bytes hold the
    // column's ranked output (rows, free ranks, values, lift products)
    union {
        struct {
            double itm[NV][C::LK];     // item (i, incidence) = s_ij of the incidence's element
            double lb[C::LK];          // load shares in incidence order
            double ld[C::LK];          // s_jj in incidence order
        } in;
        struct {
            int32_t srow[C::MAXS];     // rows in ascending order
            int32_t sfrk[C::MAXS];
            double sval[C::MAXS];
            double stv[C::MAXS];       // lift: A(c, row), then A(c, row) u0[row]
        } out;
    } u;
    static_assert(sizeof(u.out) <= sizeof(u.in), "output must fit in the item space");
};

// The column groups of a warp access the same offsets of their own V4Smem at the
// same time: a struct size that is a multiple of 128 B maps them all onto the same
// banks (4-way conflicts in 3-D).  Pad so consecutive groups start 8 banks apart.
template <class S>
struct alignas(16) Padded {
    static constexpr size_t kPad = (sizeof(S) % 128 == 32) ? 0 : ((160 - sizeof(S) % 128) % 128);
    S s;
    char pad[kPad == 0 ? 16 : kPad];
};

// one staged entry: 16 bytes {row, free rank of the row or -1, value} (one run per
// column: the placement gathers 64-byte granules at random, so row and value
// share them)
// Entry k of local column lc lives in the column's first-level run (kStageFirst
// entries at lc * kStageFirst: 128 bytes, enough for most columns, read by the
// placement as a dense stream) or, beyond that, in its overflow run.
constexpr int kStageFirst = 8;
__device__ __forceinline__ double2* stage_slot(const ColParams& p, int64_t lc, int k) {
    double2* a = reinterpret_cast<double2*>(p.st_a_row);
    double2* b = reinterpret_cast<double2*>(p.st_a_val);
    return k < kStageFirst ? a + lc * kStageFirst + k : b + lc * (p.tile_cap - kStageFirst) + (k - kStageFirst);
}
__device__ __forceinline__ void stage_entry(const ColParams& p, int64_t lc, int k, int32_t row, int32_t frk,
                                            double v) {
    *stage_slot(p, lc, k) = make_double2(__hiloint2double(frk, row), v);
}

__device__ __forceinline__ double4 ld_xl(const double4* p) {
    double4 r;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
        : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ double node_field4(const FieldDesc& g, const double* nodes, int dim, int32_t k) {
    if (g.kind == FL_FIELD_SAMPLES) return __ldg(g.samples + k);
    if (g.kind == FL_FIELD_CONST) return g.value;
    const double x = nodes[(size_t)k * dim];
    const double y = nodes[(size_t)k * dim + 1];
    const double z = dim == 3 ? nodes[(size_t)k * dim + 2] : 0.0;
    return eval_point(g, x, y, z);
}

// Column j of an element: s_ij for i = 0..d and the measure -- ElemCol<D>::
// stiffness_col's operations (assembly.hpp:133-170, 283-292), with the d+1
// quotients' fast-path acceptance tested together (div_fast) instead of one
// branch per quotient.
__device__ __forceinline__ double geom_col(const ElemCol<3>& ec, int j, double s[4], const Recip& R6) {
    double n[4][3];
    ec.normals(n);
    const double vol = ec.volume(n[3], R6);
    const Recip R = recip(36.0 * vol);
    double nj[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) nj[c] = (j == 0) ? n[0][c] : (j == 1) ? n[1][c] : (j == 2) ? n[2][c] : n[3][c];
    double dot[4];
    bool ok = divisor_ok(R);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        dot[i] = n[i][0] * nj[0] + n[i][1] * nj[1] + n[i][2] * nj[2];
        s[i] = div_fast(dot[i], R, ok);
    }
    if (!ok)
#pragma unroll
        for (int i = 0; i < 4; ++i) s[i] = __ddiv_rn(dot[i], R.b);
    return vol;
}

__device__ __forceinline__ double geom_col(const ElemCol<2>& ec, int j, double s[3], const Recip&) {
    const double ex[3] = {ec.x[2] - ec.x[1], ec.x[0] - ec.x[2], ec.x[1] - ec.x[0]};
    const double ey[3] = {ec.y[2] - ec.y[1], ec.y[0] - ec.y[2], ec.y[1] - ec.y[0]};
    const double area = 0.5 * fabs(-ex[2] * ey[1] + ey[2] * ex[1]);
    const Recip R = recip(4.0 * area);
    const double njx = (j == 0) ? -ey[0] : (j == 1) ? -ey[1] : -ey[2];
    const double njy = (j == 0) ? ex[0] : (j == 1) ? ex[1] : ex[2];
    double dot[3];
    bool ok = divisor_ok(R);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        dot[i] = (-ey[i]) * njx + ex[i] * njy + 0.0 * 0.0;
        s[i] = div_fast(dot[i], R, ok);
    }
    if (!ok)
#pragma unroll
        for (int i = 0; i < 3; ++i) s[i] = __ddiv_rn(dot[i], R.b);
    return area;
}

// the load share of local vertex j (system.hpp:97-111 / 80-96); a constant f
// takes the short path with the same operations
__device__ __forceinline__ double load_share(const ElemCol<3>& ec, int j, int32_t t, double vol,
                                             const FieldDesc& f, const Recip&) {
    if (f.kind != FL_FIELD_CONST) return ec.load_col(j, t, vol, f);
    const double w = vol * 0.25 * f.value;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += w * ((q == j) ? kTet4A : kTet4B);
    return acc;
}
__device__ __forceinline__ double load_share(const ElemCol<2>& ec, int j, int32_t t, double,
                                             const FieldDesc& f, const Recip& R6) {
    return ec.load_col(j, t, f, R6);
}

// A group of L lanes owns one column (label l, node c); GPW = 32 / L columns per
// warp share every instruction.  Lane g takes incidences e = kk*L + g (kk < K) in
// (j, t) order after the sort.  Per column:
//   keys sorted (bitonic over L*K, distances >= L pair a lane's registers) and
//   kept in shared memory;
//   per incidence (one at a time per lane, so few registers live): the element's
//   vertex labels (lel), their xl records (coordinates, node ids, free ranks),
//   s_ij for i = 0..d and the load share (fl_geometry.cuh: the reference's
//   operations, FMA-free, exact division) staged in shared memory; each nonzero
//   off-diagonal item's row inserted into the group's slot table (CAS) with the
//   incidence's bit set in the slot's pass-i mask;
//   b = 0.0 + shares in incidence order (system.hpp:114-118), A(c,c) = fold of
//   s_jj in incidence order; each slot folds its items pass by pass, incidences
//   ascending = the reference's (i*(d+1)+j, t) order (assembly.hpp:283-298
//   after the stable passes sparse.hpp:79-89); exact zeros dropped
//   (sparse.hpp:105); rows ranked by node id; A(free,free) keeps rows with a
//   free rank.
template <int D, int L, int K, bool LIFT, int MINB>
__global__ void __launch_bounds__(V4<D, L, K>::WARPS * 32, MINB) k_columns4(ColParams p) {
    using C = V4<D, L, K>;
    constexpr int NV = D + 1;
    constexpr int LK = C::LK;
    __shared__ Padded<V4Smem<D, L, K, LIFT>> sm_all[C::WARPS * C::GPW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / L, g = lane % L;
    const unsigned gmask = (L == 32) ? kFull : (((1u << L) - 1) << (gi * L));
    const unsigned lower = (1u << lane) - 1;
    V4Smem<D, L, K, LIFT>& sm = sm_all[warp * C::GPW + gi].s;
    static_assert(sizeof(Padded<V4Smem<D, L, K, LIFT>>) % 128 == 32 ||
                      sizeof(Padded<V4Smem<D, L, K, LIFT>>) % 128 == 48,
                  "group stride must be 8 (+-) banks off a multiple of 32");
    const Recip R3 = p.r3;
    const Recip R6 = p.r6;

    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(p.ticket, 1u);
        tile = __shfl_sync(kFull, tile, 0);
        if (tile >= p.n_tiles) break;
        bool bad = false;
        const int32_t lc0 = (int32_t)(tile * C::WTC);
        const int ncol_t = (int)min((int64_t)C::WTC, (int64_t)p.n_cols - lc0);
        // label l's keys are the first lcnt[l] of the lcap slots at inc[l * lcap]
        const int32_t mcl = lane < ncol_t ? __ldg(p.lcnt + lc0 + lane) : 0;
        auto col_range = [&](int q, int64_t& p0, int32_t& m) {
            m = __shfl_sync(kFull, mcl, q & 31);
            if (q >= ncol_t) m = 0;
            p0 = (int64_t)(lc0 + q) * p.lcap;
        };
        int64_t p0n;
        int32_t mn;
        col_range(gi, p0n, mn);
        uint32_t key_next[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
            key_next[kk] = (kk * L + g < mn && mn <= LK) ? __ldg(p.inc + p0n + kk * L + g) : 0xFFFFFFFFu;
#pragma unroll 1
        for (int it = 0; it < C::ITERS; ++it) {
            const int q = it * C::GPW + gi;
            const int32_t l = lc0 + q;  // label = column of this group
            const bool act = q < ncol_t;
            // the column's own node: id and free rank from its xl record
            double4 xc = make_double4(0.0, 0.0, 0.0, 0.0);
            if (act && g == 0) xc = ld_xl(p.xl + l);
            int32_t m = mn;
            uint32_t key[K];
#pragma unroll
            for (int kk = 0; kk < K; ++kk) key[kk] = key_next[kk];
            if (it + 1 < C::ITERS) {
                col_range(q + C::GPW, p0n, mn);
#pragma unroll
                for (int kk = 0; kk < K; ++kk)
                    key_next[kk] = (kk * L + g < mn && mn <= LK) ? __ldg(p.inc + p0n + kk * L + g) : 0xFFFFFFFFu;
            }
            if (m > LK) {  // too many incidences for this kernel: the general kernel reruns
                bad = true;
                m = 0;
#pragma unroll
                for (int kk = 0; kk < K; ++kk) key[kk] = 0xFFFFFFFFu;
            }
            const int32_t c = __shfl_sync(kFull, __double2loint(xc.w), gi * L);       // node id
            const int32_t fc_c = __shfl_sync(kFull, __double2hiint(xc.w), gi * L);    // free rank
            // ---- 1. keys ascending inside the group: incidence e = kk*L + g
#pragma unroll
            for (int k = 2; k <= LK; k <<= 1) {
#pragma unroll
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    if (jj >= L) {
#pragma unroll
                        for (int kk = 0; kk < K; ++kk) {
                            const int pk = kk ^ (jj / L);
                            if (pk > kk) {
                                const bool up = ((kk * L + g) & k) == 0;
                                const uint32_t a = key[kk], b2 = key[pk];
                                key[kk] = up ? min(a, b2) : max(a, b2);
                                key[pk] = up ? max(a, b2) : min(a, b2);
                            }
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < K; ++kk) {
                            const uint32_t o = __shfl_xor_sync(kFull, key[kk], jj, L);
                            const bool up = ((kk * L + g) & k) == 0;
                            const bool lo = (g & jj) == 0;
                            key[kk] = (lo == up) ? min(key[kk], o) : max(key[kk], o);
                        }
                    }
                }
            }
            if (p.want_a) {
                for (int h = g; h < C::HS; h += L) {
                    sm.row[h] = -1;
#pragma unroll
                    for (int i = 0; i < NV; ++i) sm.msk[h][i] = 0u;
                }
            }
            // the sorted keys wait in cslot (free until the slots are compacted):
            // one shared load per incidence instead of a register select chain
            static_assert(C::HS >= LK, "cslot holds the sorted keys during the incidence loop");
#pragma unroll
            for (int kk = 0; kk < K; ++kk) sm.cslot[kk * L + g] = (int32_t)key[kk];
            __syncwarp();
            // ---- 2. per incidence: geometry of column j of element t from the
            //      label-ordered nodes, staged; its off-diagonal items' rows inserted
            // the element's vertex labels one incidence ahead: incidence kk+1's
            // load is in flight while incidence kk is processed
            auto key_at = [&](int kk) -> uint32_t { return (uint32_t)sm.cslot[kk * L + g]; };
            auto lel_of = [&](int kk) {
                int4 v = make_int4(0, 0, 0, 0);
                if (kk * L + g < m) {
                    const int32_t tt = (int32_t)(key_at(kk) & 0x3FFFFFFFu);
                    v = __ldg(reinterpret_cast<const int4*>(p.lel) + tt);  // (2-D: .w unused)
                }
                return v;
            };
            int4 lel_next = lel_of(0);
#pragma unroll 1
            for (int kk = 0; kk < K; ++kk) {
                const int e = kk * L + g;
                const int4 lel_cur = lel_next;
                if (kk + 1 < K) lel_next = lel_of(kk + 1);
                if (e >= m) {
                    if (e < LK) {
#pragma unroll
                        for (int i = 0; i < NV; ++i) sm.u.in.itm[i][e] = 0.0;
                        sm.u.in.lb[e] = 0.0;
                        sm.u.in.ld[e] = 0.0;
                    }
                    continue;
                }
                const uint32_t ky = key_at(kk);
                const int32_t t_ = (int32_t)(ky & 0x3FFFFFFFu);
                const int j_ = (int)(ky >> 30);
                int32_t lv[NV];
                lv[0] = lel_cur.x;
                lv[1] = lel_cur.y;
                lv[2] = lel_cur.z;
                if constexpr (D == 3) lv[3] = lel_cur.w;
                bool okv = true;
#pragma unroll
                for (int i = 0; i < NV; ++i) okv = okv && lv[i] >= 0;
                if (!okv) {  // an out-of-range vertex id (the plan left it unlabelled)
                    atomicOr(p.err, DERR_INDEX);
#pragma unroll
                    for (int i = 0; i < NV; ++i) lv[i] = 0;
                }
                ElemCol<D> ec;
                int32_t R[NV], FR[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const double4 X = ld_xl(p.xl + lv[i]);
                    ec.x[i] = X.x;
                    ec.y[i] = X.y;
                    if constexpr (D == 3) ec.z[i] = X.z;
                    R[i] = __double2loint(X.w);
                    FR[i] = __double2hiint(X.w);
                }
                double s[NV];
                const double meas = geom_col(ec, j_, s, R6);
                if (meas == 0.0) atomicOr(p.err, DERR_DEGENERATE);
                if (p.want_a && p.coef.kind != FL_FIELD_NONE) {
                    double a;
                    if (p.coef.kind == FL_FIELD_CONST) a = p.coef.value;
                    else if (p.coef.kind == FL_FIELD_SAMPLES) a = __ldg(p.coef.samples + t_);
                    else a = ec.coef_c5(R3);
#pragma unroll
                    for (int i = 0; i < NV; ++i) s[i] = s[i] * a;
                }
                const double lsh = p.want_b ? load_share(ec, j_, t_, meas, p.f, R6) : 0.0;
                double sjj = 0.0;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    sm.u.in.itm[i][e] = s[i];
                    if (i == j_) sjj = s[i];
                }
                sm.u.in.lb[e] = lsh;
                sm.u.in.ld[e] = sjj;
                if (!p.want_a) continue;
                // exact-zero items are skipped: x + (+-0) == x for x != 0, a zero
                // prefix only changes the sign of a zero the next nonzero item
                // absorbs, and an all-zero entry is dropped anyway (sparse.hpp:105)
                // lanes walk their own nonzero items (a static loop over i ran each
                // pass with a third of the lanes on Kuhn meshes: most items are 0)
                uint32_t todo = 0;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    sm.lr[g * NV + i] = R[i];
                    sm.lfr[g * NV + i] = FR[i];
                    todo |= (i != j_ && s[i] != 0.0) ? (1u << i) : 0u;
                }
#pragma unroll 1
                for (; todo; todo &= todo - 1) {
                    const int i = __ffs(todo) - 1;
                    const int32_t r = sm.lr[g * NV + i], fr = sm.lfr[g * NV + i];
                    uint32_t h = ((uint32_t)r * 2654435761u) >> (32 - lg2c(C::HS));
                    int slot = -1;
#pragma unroll 1
                    for (int probe = 0; probe < C::HS; ++probe) {
                        const int32_t old = atomicCAS(&sm.row[h], -1, r);
                        if (old == -1 || old == r) {
                            slot = (int)h;
                            break;
                        }
                        h = (h + 1) & (C::HS - 1);
                    }
                    if (slot >= 0) {
                        sm.frk[slot] = fr;
                        atomicOr(&sm.msk[slot][i], 1u << e);
                    } else {
                        bad = true;
                    }
                }
            }
            __syncwarp();
            // ---- 3. b and the diagonal: sequential folds in incidence order (lanes 0 / 1)
            double fold = g == 0 ? 0.0 : -0.0;
            if (g < 2) {
                const double* src = g == 0 ? sm.u.in.lb : sm.u.in.ld;
                const double2* src2 = reinterpret_cast<const double2*>(src);
                const int np = m >> 1;
#pragma unroll 2
                for (int qq = 0; qq < np; ++qq) {
                    const double2 v = src2[qq];
                    fold = fold + v.x;
                    fold = fold + v.y;
                }
                if (m & 1) fold = fold + src[m - 1];
            }
            double b = __shfl_sync(kFull, fold, 0, L);
            const double dg = __shfl_sync(kFull, fold, 1, L);
            // apply_neumann (system.hpp:123-172): b + the node's accumulated face shares
            if (p.nadd && act && p.is_neu[c]) b = b + p.nadd[c - p.c_begin];
            double ylift = 0.0;
            uint64_t meta = 0;  // count of A << 40 | count of A(free, free) << 48
            // the column's staged run sits at its NODE ID (the placement then reads the
            // staging as a stream; the scattered writes cost this kernel nothing)
            const int64_t cbase = c - p.c_begin;
            if (p.want_a) {
                // ---- 4. the diagonal slot, the folds, rows ranked, zero drop
                for (int h = g; h < C::HS; h += L) sm.crow[h] = -1;  // (held the lanes' rows until here)
                if (g == 0 && act && m > 0) {
                    uint32_t h = ((uint32_t)c * 2654435761u) >> (32 - lg2c(C::HS));
#pragma unroll 1
                    for (int probe = 0; probe < C::HS; ++probe) {
                        if (sm.row[h] == -1) {
                            sm.row[h] = c;
                            sm.frk[h] = fc_c;
                            break;
                        }
                        h = (h + 1) & (C::HS - 1);
                    }
                }
                __syncwarp();
                int nocc = 0;
#pragma unroll
                for (int base = 0; base < C::HS; base += L) {
                    const int32_t r = sm.row[base + g];
                    const unsigned bal = __ballot_sync(kFull, r >= 0) & gmask;
                    if (r >= 0) {
                        sm.crow[nocc + __popc(bal & lower)] = r;
                        sm.cslot[nocc + __popc(bal & lower)] = base + g;
                    }
                    nocc += __popc(bal);
                }
                __syncwarp();
                const int n4 = (nocc + 3) >> 2;
                uint32_t jm[NV];  // lift: incidences (bit e) whose own j == jj
#pragma unroll
                for (int jj = 0; jj < NV; ++jj) jm[jj] = 0u;
                if constexpr (LIFT) {
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) {
                        const int e = kk * L + g;
                        const int je = e < m ? (int)(key[kk] >> 30) : -1;
#pragma unroll
                        for (int jj = 0; jj < NV; ++jj)
                            jm[jj] |= ((__ballot_sync(kFull, je == jj) & gmask) >> (gi * L)) << (kk * L);
                    }
                }
                // one lane per occupied slot (the compacted list): every fold into
                // registers first, then the ranked output over the item space
                constexpr int NI = C::HS / L;
                double accv[NI], taccv[NI];
                int32_t rowv[NI], frkv[NI];
#pragma unroll
                for (int ii = 0; ii < NI; ++ii) {
                    const int k = g + ii * L;
                    rowv[ii] = -1;
                    frkv[ii] = -1;
                    accv[ii] = dg;
                    taccv[ii] = dg;  // A(c, r): the transposed entry (lift only)
                    if (k < nocc) {
                        const int h = sm.cslot[k];
                        const int32_t r = sm.crow[k];
                        rowv[ii] = r;
                        frkv[ii] = sm.frk[h];
                        if (r != c) {
                            double acc = -0.0;  // -0.0 + x == x: the fold starts at its first value
#pragma unroll
                            for (int i = 0; i < NV; ++i)
                                for (uint32_t mm = sm.msk[h][i]; mm; mm &= mm - 1)
                                    acc = acc + sm.u.in.itm[i][__ffs(mm) - 1];
                            accv[ii] = acc;
                            if constexpr (LIFT) {
                                // A(c, r) folds the same items in (i_c*(d+1)+j_r, t) order:
                                // the incidence's own j first (incidences are sorted by j:
                                // contiguous ranges jm[jj]), then the pass, then incidences
                                double tacc = -0.0;
#pragma unroll
                                for (int jj = 0; jj < NV; ++jj)
#pragma unroll
                                    for (int i = 0; i < NV; ++i)
                                        for (uint32_t mm = sm.msk[h][i] & jm[jj]; mm; mm &= mm - 1)
                                            tacc = tacc + sm.u.in.itm[i][__ffs(mm) - 1];
                                taccv[ii] = tacc;
                            }
                        }
                    }
                }
                if constexpr (!LIFT) {
                    // ranked output straight from registers: bit rk of `kept` = the row
                    // of rank rk survives the zero drop (sparse.hpp:105); its place in
                    // the column is the number of kept rows ranked below it
                    const bool col_free = fc_c >= 0 && p.want_sys;
                    int rkv[NI];
                    uint32_t kept = 0, keptf = 0;
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii) {
                        rkv[ii] = -1;
                        const int32_t r = rowv[ii];
                        if (r < 0) continue;
                        int rk = 0;  // rows below r; unused entries (-1) compare as huge
                        const int4* r4 = reinterpret_cast<const int4*>(sm.crow);
                        for (int qq = 0; qq < n4; ++qq) {
                            const int4 v = r4[qq];
                            rk += ((uint32_t)v.x < (uint32_t)r) + ((uint32_t)v.y < (uint32_t)r) +
                                  ((uint32_t)v.z < (uint32_t)r) + ((uint32_t)v.w < (uint32_t)r);
                        }
                        rkv[ii] = rk;
                        if (rk < C::MAXS && accv[ii] != 0.0) {
                            kept |= 1u << rk;
                            if (col_free && frkv[ii] >= 0) keptf |= 1u << rk;
                        }
                    }
#pragma unroll
                    for (int o = 1; o < L; o <<= 1) {
                        kept |= __shfl_xor_sync(kFull, kept, o, L);
                        keptf |= __shfl_xor_sync(kFull, keptf, o, L);
                    }
                    if (nocc > C::MAXS) {
                        bad = true;
                        kept = keptf = 0;
                    }
                    const int na = __popc(kept), nf = __popc(keptf);
                    meta = ((uint64_t)na << 40) | ((uint64_t)nf << 48);
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii) {
                        const int rk = rkv[ii];
                        if (rk < 0 || !((kept >> rk) & 1u)) continue;
                        stage_entry(p, cbase, __popc(kept & ((1u << rk) - 1)), rowv[ii], p.want_sys ? frkv[ii] : -1,
                                    accv[ii]);
                    }
                } else {
                __syncwarp();
#pragma unroll
                for (int ii = 0; ii < NI; ++ii) {
                    const int32_t r = rowv[ii];
                    if (r < 0) continue;
                    int rk = 0;  // rows below r; unused entries (-1) compare as huge
                    const int4* r4 = reinterpret_cast<const int4*>(sm.crow);
                    for (int qq = 0; qq < n4; ++qq) {
                        const int4 v = r4[qq];
                        rk += ((uint32_t)v.x < (uint32_t)r) + ((uint32_t)v.y < (uint32_t)r) +
                              ((uint32_t)v.z < (uint32_t)r) + ((uint32_t)v.w < (uint32_t)r);
                    }
                    if (rk < C::MAXS) {
                        sm.u.out.srow[rk] = r;
                        sm.u.out.sfrk[rk] = frkv[ii];
                        sm.u.out.sval[rk] = accv[ii];
                        if constexpr (LIFT) sm.u.out.stv[rk] = taccv[ii];
                    }
                }
                if (nocc > C::MAXS) {
                    bad = true;
                    nocc = 0;
                }
                const int nslot = nocc;
                __syncwarp();
                if constexpr (LIFT) {
                    // y = (A u0)[c] = 0.0 + A(c, r) u0[r] over the stored entries of row c,
                    // r ascending (matvec, sparse.hpp:129-141); u0 = g at Dirichlet nodes
                    uint32_t umask = 0;
                    for (int base = 0; base < C::MAXS; base += L) {
                        const int qq = base + g;
                        bool use = false;
                        if (qq < nslot) {
                            const double a = sm.u.out.stv[qq];
                            const int32_t r = sm.u.out.srow[qq];
                            if (a != 0.0 && sm.u.out.sfrk[qq] < 0) {
                                const double u = node_field4(p.g_dir, p.nodes, D, r);
                                use = u != 0.0;
                                sm.u.out.stv[qq] = a * u;
                            }
                        }
                        umask |= ((__ballot_sync(kFull, use) & gmask) >> (gi * L)) << base;
                    }
                    __syncwarp();
                    if (g == 0) {
                        double yy = 0.0;
                        for (uint32_t mm = umask; mm; mm &= mm - 1) yy = yy + sm.u.out.stv[__ffs(mm) - 1];
                        ylift = yy;
                    }
                    __syncwarp();
                }
                const bool col_free = fc_c >= 0;
                // compaction in chunks of L entries into ONE staged run per column:
                // {row, free rank of the row or -1} + value; A(free, free) is the
                // subset with a free rank in a free column (placed by k4_place)
                constexpr int NCH = (C::MAXS + L - 1) / L;
                int na = 0, nf = 0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int qq = ch * L + g;
                    const bool in = qq < nslot;
                    const double v = in ? sm.u.out.sval[qq] : 0.0;
                    const bool keep = in && v != 0.0;  // sparse.hpp:105
                    const bool keepf = keep && col_free && p.want_sys && sm.u.out.sfrk[qq] >= 0;
                    na += __popc(__ballot_sync(kFull, keep) & gmask);
                    nf += __popc(__ballot_sync(kFull, keepf) & gmask);
                }
                int wa = 0;  // entries of this column staged so far
                meta = ((uint64_t)na << 40) | ((uint64_t)nf << 48);
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int qq = ch * L + g;
                    const bool in = qq < nslot;
                    const double v = in ? sm.u.out.sval[qq] : 0.0;
                    const int32_t r = in ? sm.u.out.srow[qq] : 0;
                    const int32_t fr = (in && p.want_sys) ? sm.u.out.sfrk[qq] : -1;
                    const bool keep = in && v != 0.0;
                    const unsigned ba = __ballot_sync(kFull, keep) & gmask;
                    if (keep) {
                        stage_entry(p, cbase, wa + __popc(ba & lower), r, fr, v);
                    }
                    wa += __popc(ba);
                }
                }  // LIFT
            }
            // ---- per-column record, by NODE ID (the placement then streams it):
            //      {b, u0, b - A u0, staging meta}
            if (act && g == 0) {
                double u0 = 0.0, bmod = b;
                if (p.want_sys) {
                    u0 = fc_c < 0 ? node_field4(p.g_dir, p.nodes, D, c) : 0.0;
                    bmod = LIFT ? b - ylift : b - 0.0;  // system.hpp:197-198
                }
                p.vst[c - p.c_begin] = make_double4(b, u0, bmod, __longlong_as_double((long long)meta));
            }
            __syncwarp();
        }
        if (__any_sync(kFull, bad) && lane == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
    }
}

// ===========================================================================
// placement: label-ordered staging -> node-id-ordered CSC and vectors, one pass
// ===========================================================================
// Tile = kPlaceItems sub-tiles of 256 consecutive node ids (one per thread and
// sub-tile), tiles taken in order from a ticket.  Each node's record vst[v]
// (written by k_columns4 at the node id) holds its vectors and, packed in .w, the
// counts of its A and A(free, free) entries; its staged run sits at the node id
// too (stage_slot).  The column pointers are an exclusive scan over node ids
// (block scans + ONE decoupled look-back per tile on (nnz_A, nnz_Aff) packed in
// 64 bits: with 256-node tiles a third of the kernel's stalls were blocks waiting
// for their predecessor); a warp's 32 consecutive columns are one contiguous
// destination run, copied with every store instruction writing 32 consecutive entries.
constexpr int kPlaceThreads = 256, kPlaceItems = 4, kPlaceRounds = 4;

__global__ void __launch_bounds__(kPlaceThreads) k4_place(ColParams p, uint64_t* __restrict__ status,
                                                          unsigned int* __restrict__ ticket) {
    __shared__ int64_t warp_sums[kPlaceThreads / 32];
    __shared__ int64_t s_tile, s_excl;
    const int lane = threadIdx.x & 31;
    const int32_t N = p.n_cols;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    // free ranks relative to the shard: free nodes below c_begin come first
    const int32_t fb = p.want_sys ? free_base(p) : 0;
    int32_t frv[kPlaceItems], cav[kPlaceItems], cfv[kPlaceItems];
#pragma unroll
    for (int k = 0; k < kPlaceItems; ++k) {
        const int32_t v = (int32_t)(tile * kPlaceThreads * kPlaceItems) + k * kPlaceThreads + threadIdx.x;
        const bool in = v < N;  // column c_begin + v
        int32_t fr = (in && p.want_sys) ? __ldg(p.fidx + p.c_begin + v) : -1;
        if (fr >= 0) fr -= fb;
        double4 vs = make_double4(0.0, 0.0, 0.0, 0.0);
        if (in) vs = ld_xl(p.vst + v);  // the record of node v, in node order
        const uint64_t meta = (uint64_t)__double_as_longlong(vs.w);
        frv[k] = fr;
        cav[k] = in ? (int32_t)((meta >> 40) & 0xFF) : 0;
        cfv[k] = fr >= 0 ? (int32_t)((meta >> 48) & 0xFF) : 0;
        if (in) {
            if (p.want_b) p.b[v] = vs.x;
            if (p.want_sys) {
                p.u0[v] = vs.y;
                p.b_mod[v] = vs.z;
                if (fr >= 0) p.b_f[fr] = vs.z;
            }
        }
    }
    if (!p.want_a) return;
    // exclusive prefix over node ids of (A count, A(free, free) count)
    int64_t exv[kPlaceItems], run = 0;
#pragma unroll
    for (int k = 0; k < kPlaceItems; ++k) {
        int64_t total;
        exv[k] = run + block_exclusive_sum<kPlaceThreads>((int64_t)cav[k] | ((int64_t)cfv[k] << 32), warp_sums, total);
        run += total;
    }
    if (threadIdx.x < 32) {
        const uint64_t e = warp_lookback(status, tile, (uint64_t)run);
        if (threadIdx.x == 0) s_excl = (int64_t)e;
    }
    __syncthreads();
    const int64_t tile_excl = s_excl;
#pragma unroll 1
    for (int k = 0; k < kPlaceItems; ++k) {
        const int32_t v = (int32_t)(tile * kPlaceThreads * kPlaceItems) + k * kPlaceThreads + threadIdx.x;
        const bool in = v < N;
        const int32_t fr = frv[k], ca = cav[k], cf = cfv[k];
        const int64_t excl = exv[k] + tile_excl;
        const int32_t pa = (int32_t)(excl & 0xFFFFFFFF), pf = (int32_t)(excl >> 32);
        if (in) {
            p.col_ptr[v] = pa;
            if (fr >= 0) p.ff_col_ptr[fr] = pf;
            if (v == N - 1) {
                p.col_ptr[N] = pa + ca;
                if (p.want_sys)  // free_rank[c_begin + N] - free_rank[c_begin] free columns
                    p.ff_col_ptr[__ldg(p.fidx + (int64_t)p.n_nodes + 1 + p.c_begin + N) - fb] = pf + cf;
            }
            if ((int64_t)pa + ca > p.cap_a || (p.want_sys && (int64_t)pf + cf > p.cap_ff))
                atomicOr(p.err, DERR_CAPACITY);
        }
        // the warp's 32 columns are one contiguous run of A: every store writes 32
        // consecutive entries; A(free, free) takes the entries with a free row in a
        // free column, at the column's pointer + their rank among them
        int32_t pre = ca;  // inclusive prefix over the warp's lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(kFull, pre, o);
            if (lane >= o) pre += y;
        }
        const int32_t total_w = __shfl_sync(kFull, pre, 31);
        if (total_w == 0) continue;
        const int32_t ex = pre - ca;
        const int32_t d0 = __shfl_sync(kFull, pa, 0);
        if ((int64_t)d0 + total_w > p.cap_a) continue;  // flagged above
        const int cfree_l = fr >= 0 ? 1 : 0;
        int carry_k = -1, carry = 0;
        // kPlaceRounds rounds of 32 entries per iteration: all their loads are issued
        // before any is stored (the copy is bound by bytes in flight; C5 placement
        // 1.54 / 1.46 / 1.38 ms at 1 / 2 / 4 rounds)
        for (int32_t q0 = 0; q0 < total_w; q0 += 32 * kPlaceRounds) {
            int kkv[kPlaceRounds];
            int32_t ekv[kPlaceRounds], pfkv[kPlaceRounds];
            int cfv2[kPlaceRounds];
            double2 rec[kPlaceRounds];
#pragma unroll
            for (int r = 0; r < kPlaceRounds; ++r) {
                const int32_t qq = q0 + 32 * r + lane;
                // largest kk with ex[kk] <= qq (lanes with len 0 share prefixes: the search
                // lands on the last of them, whose run holds qq)
                int kk = 0;
#pragma unroll
                for (int stp = 16; stp > 0; stp >>= 1) {
                    const int32_t ek = __shfl_sync(kFull, ex, kk + stp);
                    if (ek <= qq) kk += stp;
                }
                kkv[r] = kk;
                ekv[r] = __shfl_sync(kFull, ex, kk);
                const int64_t sk = __shfl_sync(kFull, v, kk);  // the column whose staged run holds qq
                pfkv[r] = __shfl_sync(kFull, pf, kk);
                cfv2[r] = __shfl_sync(kFull, cfree_l, kk);
                rec[r] = make_double2(0.0, 0.0);
                if (qq < total_w) rec[r] = __ldcs(stage_slot(p, sk, qq - ekv[r]));  // {row | free rank << 32, value}
            }
#pragma unroll
            for (int r = 0; r < kPlaceRounds; ++r) {
                const int32_t qr = q0 + 32 * r;
                if (qr >= total_w) break;  // warp-uniform
                const int32_t qq = qr + lane;
                const int kk = kkv[r];
                const int32_t ek = ekv[r];
                int2 rf = make_int2(0, -1);
                double val = 0.0;
                if (qq < total_w) {
                    rf = make_int2(__double2loint(rec[r].x), __double2hiint(rec[r].x));
                    val = rec[r].y;
                    p.row_idx[d0 + qq] = rf.x;
                    p.values[d0 + qq] = val;
                }
                const bool isf = qq < total_w && p.want_sys && cfv2[r] && rf.y >= 0;
                const unsigned bal = __ballot_sync(kFull, isf);
                const int start = ek > qr ? (int)(ek - qr) : 0;  // column kk's first lane in this round
                const unsigned below = (1u << lane) - 1, before = (1u << start) - 1;
                const int rank = __popc(bal & below & ~before) + (kk == carry_k ? carry : 0);
                if (isf) {
                    p.ff_row_idx[pfkv[r] + rank] = rf.y;
                    p.ff_values[pfkv[r] + rank] = val;
                }
                // the column holding lane 31 may continue into the next round
                const int k31 = __shfl_sync(kFull, kk, 31), st31 = __shfl_sync(kFull, start, 31);
                carry = (k31 == carry_k ? carry : 0) + __popc(bal & ~((1u << st31) - 1));
                carry_k = k31;
            }
        }
    }
}

// ===========================================================================
// host side
// ===========================================================================
int v4_lanes(int dim) { return dim == 2 ? 16 : 32; }  // incidences per column the kernel takes

// the divisor halves of x / 3 and x / 6 (fl::recip: device instructions), once per context
__global__ void k4_recip_consts(double* out) {
    const Recip a = recip(3.0), b = recip(6.0);
    out[0] = a.b;
    out[1] = a.r;
    out[2] = b.b;
    out[3] = b.r;
}
int v4_init_consts(fl_ctx* ctx) {
    double* d = nullptr;
    FL_CUDA(cudaMalloc(&d, sizeof(double) * 4));
    k4_recip_consts<<<1, 1, 0, ctx->stream>>>(d);
    FL_CUDA(cudaMemcpyAsync(ctx->recip_consts, d, sizeof(double) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    FL_CUDA(cudaStreamSynchronize(ctx->stream));
    FL_CUDA(cudaFree(d));
    return FL_OK;
}

// slots per label segment for a mesh of maximum valence max_inc: the column
// kernel variant's incidences per column (2-D: 8 lanes x 1 or 2; 3-D: 8 x 4)
int v4_cap(int dim, int max_inc) { return dim == 2 ? (max_inc <= 8 ? 8 : 16) : 32; }

// keys + relabelled elements for capacity `cap`, then the statistics
static int v4_fill(fl_ctx* ctx, fl_mesh* mesh, int cap) {
    const cudaStream_t s = ctx->stream;
    auto& lp = mesh->lp;
    const int nv = mesh->dim + 1;
    const int32_t N = mesh->n_nodes;
    const int32_t c0 = mesh->col_begin, c1 = mesh->col_end;
    const int64_t n_entries = (int64_t)mesh->n_elems * nv;
    P4Misc* misc = lp.misc.as<P4Misc>();
    int32_t* cnt = lp.lptr.as<int32_t>();  // per-label counts = fill cursors
    FL_TRY(lp.linc.ensure(sizeof(uint32_t) * (size_t)std::max<int64_t>((int64_t)N * cap, 1)));
    FL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)N + 1), s));
    FL_CUDA(cudaMemsetAsync(misc, 0, sizeof(P4Misc), s));
    // bucketed fill for large 2-D meshes (FL_PLAN=0|1 overrides; the element order
    // of a 3-D mesh is left spatial by every generator here, C5 included)
    const char* penv = std::getenv("FL_PLAN");
    const bool bucketed = n_entries > 0 &&
                          (penv ? penv[0] == '1' : (mesh->dim == 2 && n_entries >= ((int64_t)1 << 26)));
    if (bucketed) {
        int shift = 0;
        while (((int64_t)(N - 1) >> shift) + 1 > kB4MaxBuckets) ++shift;
        const int nb = ((N - 1) >> shift) + 1;
        const int64_t bucket_cap = (int64_t)cap << shift;
        FL_TRY(lp.stage.ensure(sizeof(int2) * (size_t)(bucket_cap * nb) + sizeof(int32_t) * (kB4MaxBuckets + 1)));
        int2* stg = lp.stage.as<int2>();
        int32_t* bcur = reinterpret_cast<int32_t*>(stg + bucket_cap * nb);
        FL_CUDA(cudaMemsetAsync(bcur, 0, sizeof(int32_t) * (size_t)(nb + 1), s));
        const int64_t chunks = (n_entries + kP4Block * kB4Items - 1) / (kP4Block * kB4Items);
        k4_bucket_scatter<<<(int)chunks, kP4Block, 0, s>>>(n_entries, nv, N, c0, c1, shift, cap,
                                                           mesh->elems.as<int32_t>(), lp.lab.as<int32_t>(), bcur,
                                                           stg, lp.lel.as<int32_t>(), misc);
        count_launch(ctx);
        const int cpb = (int)((bucket_cap + kP4Block * 4 - 1) / (kP4Block * 4));
        k4_fill_b<<<nb * cpb, kP4Block, 0, s>>>(shift, cap, cpb, bcur, stg, cnt, lp.linc.as<uint32_t>());
        count_launch(ctx);
    } else if (n_entries > 0) {  // the direct fill (one key per store)
        constexpr int U = 4;
        int per_sm = 1;  // persistent: one resident wave of blocks, warps stride over the entries
        FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_fill<U>, 256, 0));
        const int fgrid = (int)std::min<int64_t>(std::max<int64_t>(div_up(n_entries, 256 * U), 1),
                                                 (int64_t)ctx->sm_count * std::max(per_sm, 1));
        k4_fill<U><<<fgrid, 256, 0, s>>>(n_entries, nv, N, c0, c1, cap, mesh->elems.as<int32_t>(),
                                         lp.lab.as<int32_t>(), cnt, lp.linc.as<uint32_t>(), lp.lel.as<int32_t>(),
                                         misc);
        count_launch(ctx);
    }
    if (c1 > c0) {  // statistics over the owned labels [0, c1 - c0)
        k4_stats<<<std::min(div_up(c1 - c0, 256), ctx->sm_count * 8), 256, 0, s>>>(c1 - c0, N, mesh->dim, cnt, misc);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    lp.cap = cap;
    return FL_OK;
}

int v4_plan(fl_ctx* ctx, fl_mesh* mesh, bool sync) {
    const cudaStream_t s = ctx->stream;
    auto& lp = mesh->lp;
    const int nv = mesh->dim + 1;
    const int32_t N = mesh->n_nodes;
    // owned columns (a multi-GPU shard); the whole mesh otherwise
    const int32_t c0 = mesh->col_begin, c1 = mesh->col_end;
    const bool sharded = c0 != 0 || c1 != N;
    const int64_t n_entries = (int64_t)mesh->n_elems * nv;
    FL_TRY(lp.lab.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.lptr.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.lel.ensure(sizeof(int32_t) * 4 * (size_t)std::max<int32_t>(mesh->n_elems, 1)));
    FL_TRY(lp.misc.ensure(sizeof(P4Misc)));
    P4Misc* misc = lp.misc.as<P4Misc>();
    int32_t* lab = lp.lab.as<int32_t>();
    if (N > 0) {
        // Morton cells of ~cn nodes (FL_CELL_NODES, default 8: C5 column pass 18.2 / 17.8
        // / 17.7 ms at 64 / 8 / 1, plan +0.6 ms at 1): 2^(dim*bits) cells
        const int dim = mesh->dim;
        const char* cenv = std::getenv("FL_CELL_NODES");
        const int64_t cn = cenv ? std::max(1, std::atoi(cenv)) : 8;
        int bits = 1;
        while (bits < (dim == 3 ? 10 : 15) && ((int64_t)1 << (dim * (bits + 1))) * cn <= (int64_t)N) ++bits;
        const int64_t ncell = ((int64_t)1 << (dim * bits)) * (sharded ? 2 : 1);
        const int nparts = std::min(div_up(N, 256), ctx->sm_count * 4);
        FL_TRY(lp.cells.ensure(sizeof(int32_t) * ((size_t)N + 2 * (size_t)ncell + 2) + sizeof(double) * (6 * (size_t)nparts + 1)));
        int32_t* cellv = lp.cells.as<int32_t>();
        int32_t* ccnt = cellv + N;
        int32_t* coff = ccnt + ncell + 1;
        double* part = reinterpret_cast<double*>(coff + ncell + 1 + ((N + 2 * ncell + 2) & 1));
        FL_CUDA(cudaMemsetAsync(ccnt, 0, sizeof(int32_t) * (size_t)(ncell + 1), s));
        k4_bbox<<<nparts, 256, 0, s>>>(N, dim, mesh->nodes.as<double>(), part);
        count_launch(ctx);
        k4_cell<<<std::min(div_up(N, 256), ctx->sm_count * 8), 256, 0, s>>>(N, dim, bits, nparts, mesh->nodes.as<double>(),
                                                                          part, c0, c1, cellv, ccnt);
        count_launch(ctx);
        FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(ncell)));
        const int32_t* cc = ccnt;
        FL_CUDA(launch_scan<int32_t>(ncell, [cc] __device__(int64_t i) { return (int64_t)cc[i]; }, coff,
                                     ctx->scan_ws.p, s));
        count_launch(ctx);
        k4_cell_scatter<<<std::min(div_up(N, 256), ctx->sm_count * 8), 256, 0, s>>>(N, cellv, coff, lab);
        count_launch(ctx);
    }
    // Segment capacity: a re-plan keeps the last known valence class (a topology
    // that outgrows it is flagged by the column kernel and rerun on the general
    // kernel, fl_result_sizes); the first plan fills at the largest class and,
    // should the mesh fit a smaller one, once more at that.
    const int lanes = v4_lanes(mesh->dim);
    FL_TRY(v4_fill(ctx, mesh, sync ? lanes : v4_cap(mesh->dim, lp.max_inc)));
    lp.planned = true;
    lp.ever = true;
    if (!sync) {
        lp.stale = true;
        return FL_OK;
    }
    FL_CUDA(cudaMemcpyAsync(ctx->pinned, misc, sizeof(P4Misc), cudaMemcpyDeviceToHost, s));
    FL_CUDA(cudaStreamSynchronize(s));
    const P4Misc* h = static_cast<const P4Misc*>(ctx->pinned);
    lp.stale = false;
    if (h->err & DERR_INDEX) {
        lp.planned = false;
        return set_error(FL_E_INDEX_OUT_OF_RANGE, "element vertex index out of range");
    }
    lp.nnz_bound = (int64_t)h->stats[0];
    lp.max_inc = (int32_t)h->stats[1];
    lp.ok = lp.max_inc <= lanes && !(h->err & DERR_V2_OVERFLOW);
    if (lp.ok && v4_cap(mesh->dim, lp.max_inc) < lanes) FL_TRY(v4_fill(ctx, mesh, v4_cap(mesh->dim, lp.max_inc)));
    return FL_OK;
}

template <int D, int L, int K, bool LIFT, int MINB>
static int launch4(fl_ctx* ctx, ColParams& p) {
    using C = V4<D, L, K>;
    auto kern = k_columns4<D, L, K, LIFT, MINB>;
    int per_sm = 1;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::WARPS * 32, 0));
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((p.n_tiles + C::WARPS - 1) / C::WARPS, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    kern<<<(int)grid, C::WARPS * 32, 0, ctx->stream>>>(p);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

// Resident CTAs per SM the kernel is compiled for (its register cap).  2-D: 8 CTAs
// of 4 warps at 64 registers (C3 column pass 6.42 / 5.74 / 5.08 / 5.43 ms at
// 5 / 6 / 8 / 10 CTAs: occupancy pays until the spills take over).  3-D: 10 CTAs
// of 2 warps at 96 registers, the shared-memory limit (128 registers, 8 CTAs,
// measured the same).
template <int D, int L, int K>
static int launch4_sel(fl_ctx* ctx, ColParams& p) {
    constexpr int MINB = D == 3 ? 10 : 8;
    return p.need_lift ? launch4<D, L, K, true, MINB>(ctx, p) : launch4<D, L, K, false, MINB>(ctx, p);
}

// The column pass of fl_assemble on the label plan (the whole mesh or a column range).  p carries the outputs, the
// fields and the partition; the plan pointers are replaced here by the label plan's.
int v4_columns(fl_ctx* ctx, fl_mesh* mesh, ColParams& p, fl_result* res) {
    const cudaStream_t s = ctx->stream;
    auto& lp = mesh->lp;
    const int dim = mesh->dim;
    const int32_t N = mesh->n_nodes;
    const int wtc = dim == 2 ? V4<2, 8, 1>::WTC : V4<3, 8, 4>::WTC;
    const int maxs = dim == 2 ? V4<2, 8, 1>::MAXS : V4<3, 8, 4>::MAXS;
    FL_TRY(res->v4[0].ensure(sizeof(double4) * ((size_t)N + 1)));  // xl
    FL_TRY(res->v4[1].ensure(sizeof(double4) * ((size_t)N + 1)));  // vst
    double4* xl = res->v4[0].as<double4>();
    p.xl = xl;
    p.vst = res->v4[1].as<double4>();
    p.lel = lp.lel.as<int32_t>();
    p.inc_ptr = nullptr;
    p.r3 = Recip{ctx->recip_consts[0], ctx->recip_consts[1]};
    p.r6 = Recip{ctx->recip_consts[2], ctx->recip_consts[3]};
    p.lab = lp.lab.as<int32_t>();
    p.lcnt = lp.lptr.as<int32_t>();
    p.lcap = lp.cap;
    p.inc = lp.linc.as<uint32_t>();
    p.keys_sorted = false;
    if (N > 0) {
        k4_xl<<<std::min(div_up(N, 256), ctx->sm_count * 16), 256, 0, s>>>(
            N, dim, lp.lab.as<int32_t>(), p.nodes, p.want_sys ? p.fidx : nullptr, xl);
        count_launch(ctx);
    }
    // one staged run per column of 16-byte entries {row, free rank, value}
    // (A(free, free) rides along), maxs slots at the column's node id
    p.n_tiles = (p.n_cols + wtc - 1) / wtc;
    p.tile_cap = maxs;  // slots per column: kStageFirst in stage[0], the rest in stage[1]
    FL_TRY(res->stage[0].ensure(sizeof(double2) * ((size_t)p.n_cols + 1) * kStageFirst));
    FL_TRY(res->stage[1].ensure(sizeof(double2) * ((size_t)p.n_cols + 1) * (size_t)(maxs - kStageFirst)));
    p.st_a_row = res->stage[0].as<int32_t>();
    p.st_a_val = res->stage[1].as<double>();
    FL_CUDA(cudaMemsetAsync(p.ticket, 0, sizeof(uint32_t), s));
    // Neumann data: per-node face shares first (k_neumann_add on the label plan)
    p.nadd = nullptr;
    if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE) FL_TRY(launch_neumann_add(ctx, dim, p, res));
    if (ctx->profile) {
        FL_CUDA(cudaEventRecord(ctx->ev[5], s));
        FL_CUDA(cudaEventRecord(ctx->ev[6], s));
        ctx->kernel_timed = true;
    }
    // 8 lanes per column, 4 columns per warp: 2-D 1 or 2 incidences per lane
    // (valence <= 8 / 16), 3-D 4 (valence <= 32)
    if (dim == 2) {
        if (lp.cap <= 8) FL_TRY((launch4_sel<2, 8, 1>(ctx, p)));
        else FL_TRY((launch4_sel<2, 8, 2>(ctx, p)));
    } else {
        // FL_V4_SHAPE=16x2: 16 lanes x 2 incidences, 2 columns per warp (experiment)
        const char* sh = std::getenv("FL_V4_SHAPE");
        if (sh && sh[0] == '1') FL_TRY((launch4_sel<3, 16, 2>(ctx, p)));
        else FL_TRY((launch4_sel<3, 8, 4>(ctx, p)));
    }
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[7], s));
    // placement: column pointers in node-id order, the copy and the vectors, one pass
    if (p.n_cols > 0) {
        const int64_t ptiles = ((int64_t)p.n_cols + kPlaceThreads * kPlaceItems - 1) / (kPlaceThreads * kPlaceItems);
        FL_TRY(res->v4[2].ensure(sizeof(uint64_t) * (size_t)(ptiles + 2)));
        uint64_t* status = res->v4[2].as<uint64_t>();
        FL_CUDA(cudaMemsetAsync(status, 0, sizeof(uint64_t) * (size_t)(ptiles + 2), s));
        unsigned int* ticket = reinterpret_cast<unsigned int*>(status + ptiles + 1);
        k4_place<<<(int)ptiles, kPlaceThreads, 0, s>>>(p, status, ticket);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    res->v4_used = true;
    return FL_OK;
}

}  // namespace fl
