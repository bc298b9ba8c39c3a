// fl_columns4.cu -- the label-space pipeline (v4), default fast path of fl_assemble.
//
// Why labels.  The reference's output is in node-id order, and config C5 (and
// C3) number their nodes randomly.  Indexing the plan, the coordinates and the
// partition by node id turns every access of the column pass into a random
// DRAM sector: the id-space v3 pass read 109 GB on C5 for 3.6 GB of compulsory
// traffic.  Here every node gets a LABEL, the order in which the element
// stream first touches it (computed inside the count pass, no sort), and all
// intermediate work runs in label order:
//
//   plan     k4_count     per-node incidence counts + first-touch labels
//            k4_untouched labels for nodes no element references
//            scan         label segments lptr = exclusive scan of counts by label
//            k4_fill      (j << 30 | t) keys into the label segments; the
//                         elements rewritten with vertex labels (lel)
//   per call k4_xl        xl[label] = node coordinates + {node id, free rank}
//            k_columns4   one group of L lanes per column (label), K incidences
//                         per lane: element geometry computed in the kernel from
//                         xl (no element-record round trip through HBM), the
//                         reference's exact per-entry fold order, zero drop,
//                         load vector, Dirichlet lift, A(free,free); entries
//                         staged per tile of labels
//            scans + k4_place  CSC column pointers in node-id order, staged
//                         runs copied to their node-id positions, vectors
//
// Labels never reach the output: rows are node ids, every fold runs in the
// reference's (i*(d+1)+j, t) order with the original element index t, so the
// result is bitwise the id-space pipeline's (and the reference's) whatever the
// labelling.  Citations: /root/reference/proj/include/femlite/<file>:<line>.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

constexpr unsigned kFull = 0xffffffffu;

// ===========================================================================
// plan
// ===========================================================================
constexpr int kP4Block = 256, kP4Iters = 16;

// misc buffer layout: u64 stats[4] (nnz bound, max valence, -, -), u32 label
// counter, u32 error word
struct P4Misc {
    unsigned long long stats[4];
    uint32_t lctr;
    uint32_t err;
};

// Counts per node and first-touch labels.  Block b covers entries
// [b*256*16, (b+1)*256*16) (blocks issued in element order).  Lanes holding
// the same node are grouped with match_any; the group leader adds the group's
// count, and the one whose add returns 0 is the node's first toucher.  Labels
// are handed out per block (one atomic), warp-major then iteration then lane.
__global__ void __launch_bounds__(kP4Block)
k4_count(int64_t n_entries, int32_t n_nodes, const int32_t* __restrict__ elems,
         int32_t* __restrict__ cnt, int32_t* __restrict__ lab, int32_t* __restrict__ ilab,
         P4Misc* __restrict__ misc) {
    __shared__ int32_t wsum[kP4Block / 32];
    __shared__ int32_t s_base;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lower = (1u << lane) - 1;
    const int64_t b0 = (int64_t)blockIdx.x * kP4Block * kP4Iters;
    int32_t fv[kP4Iters];
    unsigned bal[kP4Iters];
    int wtot = 0;
    uint32_t err = 0;
#pragma unroll
    for (int k = 0; k < kP4Iters; ++k) {
        const int64_t e = b0 + (int64_t)k * kP4Block + threadIdx.x;
        int32_t key = -1;
        if (e < n_entries) {
            const int32_t v = __ldg(elems + e);
            if ((uint32_t)v >= (uint32_t)n_nodes) err = DERR_INDEX;
            else key = v;
        }
        const unsigned g = __match_any_sync(kFull, key);
        bool first = false;
        if (key >= 0 && (g & lower) == 0) first = atomicAdd(cnt + key, __popc(g)) == 0;
        fv[k] = key;
        bal[k] = __ballot_sync(kFull, first);
        wtot += __popc(bal[k]);
    }
    if (__any_sync(kFull, err != 0) && lane == 0) atomicOr(&misc->err, DERR_INDEX);
    if (lane == 0) wsum[w] = wtot;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t s = 0;
#pragma unroll
        for (int i = 0; i < kP4Block / 32; ++i) {
            const int32_t x = wsum[i];
            wsum[i] = s;
            s += x;
        }
        s_base = s ? (int32_t)atomicAdd(&misc->lctr, (uint32_t)s) : 0;
    }
    __syncthreads();
    int32_t base = s_base + wsum[w];
#pragma unroll
    for (int k = 0; k < kP4Iters; ++k) {
        if ((bal[k] >> lane) & 1u) {
            const int32_t lb = base + __popc(bal[k] & lower);
            lab[fv[k]] = lb;
            ilab[lb] = fv[k];
        }
        base += __popc(bal[k]);
    }
}

// nodes no element references (their columns are empty) take the last labels
__global__ void __launch_bounds__(kP4Block)
k4_untouched(int32_t n_nodes, const int32_t* __restrict__ cnt, int32_t* __restrict__ lab,
             int32_t* __restrict__ ilab, P4Misc* __restrict__ misc) {
    __shared__ int32_t wsum[kP4Block / 32];
    __shared__ int32_t s_base;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lower = (1u << lane) - 1;
    const int32_t v = blockIdx.x * kP4Block + threadIdx.x;
    const bool un = v < n_nodes && __ldg(cnt + v) == 0;
    const unsigned b = __ballot_sync(kFull, un);
    if (lane == 0) wsum[w] = __popc(b);
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t s = 0;
        for (int i = 0; i < kP4Block / 32; ++i) {
            const int32_t x = wsum[i];
            wsum[i] = s;
            s += x;
        }
        s_base = s ? (int32_t)atomicAdd(&misc->lctr, (uint32_t)s) : 0;
    }
    __syncthreads();
    if (un) {
        const int32_t lb = s_base + wsum[w] + __popc(b & lower);
        lab[v] = lb;
        ilab[lb] = v;
    }
}

// (j << 30 | t) keys into the label segments (cursor seeded with lptr) and the
// elements with vertex labels.  U rounds of 32 consecutive entries per warp,
// one warp iteration per block, blocks issued in element order (as k_inc_fill:
// the live destination segments stay in L2 until their sectors are complete).
template <int U>
__global__ void k4_fill(int64_t n_entries, int nv, int32_t n_nodes, const int32_t* __restrict__ elems,
                        const int32_t* __restrict__ lab, int32_t* __restrict__ cursor,
                        uint32_t* __restrict__ linc, int32_t* __restrict__ lel) {
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
                if ((uint32_t)v < (uint32_t)n_nodes) key[u] = __ldg(lab + v);
                lel[e] = key[u];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) grp[u] = __match_any_sync(kFull, key[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            pos[u] = 0;
            if (key[u] >= 0 && (grp[u] & lower) == 0) pos[u] = atomicAdd(cursor + key[u], __popc(grp[u]));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t p0 = __shfl_sync(kFull, pos[u], __ffs(grp[u]) - 1) + __popc(grp[u] & lower);
            if (key[u] >= 0) {
                const int64_t e = e0 + u * 32 + lane;
                const int32_t t = (int32_t)(e / nv);
                const uint32_t j = (uint32_t)(e - (int64_t)t * nv);
                linc[p0] = (j << 30) | (uint32_t)t;
            }
        }
    }
}

// stats[0] += sum_l min(m_l d + 1, N) (nnz upper bound), stats[1] = max m_l
__global__ void k4_stats(int32_t n, int dim, const int32_t* __restrict__ lptr, P4Misc* __restrict__ misc) {
    int64_t bound = 0;
    int32_t mx = 0;
    for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
        const int32_t m = lptr[c + 1] - lptr[c];
        const int64_t b = (int64_t)m * dim + 1;
        bound += b < n ? b : n;
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
__global__ void k4_xl(int32_t n, int dim, const int32_t* __restrict__ ilab, const double* __restrict__ nodes,
                      const int32_t* __restrict__ fidx, double4* __restrict__ xl) {
    for (int32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
        const int32_t v = __ldg(ilab + l);
        const double* p = nodes + (size_t)v * dim;
        const double x = __ldg(p), y = __ldg(p + 1), z = dim == 3 ? __ldg(p + 2) : 0.0;
        const int32_t fr = fidx ? __ldg(fidx + v) : 0;
        xl[l] = make_double4(x, y, z, __hiloint2double(fr, v));
    }
}

// ===========================================================================
// column kernel
// ===========================================================================
__host__ __device__ constexpr int lg2c(int x) { return x <= 1 ? 0 : 1 + lg2c(x >> 1); }

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
    alignas(16) int32_t row[C::HS];    // slot -> row (node id, -1 empty)
    alignas(16) int32_t crow[C::HS];   // occupied rows, compacted (-1 padded)
    int32_t cslot[C::HS];              // their slots
    int32_t frk[C::HS];                // slot -> free rank of the row (-1: Dirichlet)
    uint32_t msk[C::HS][D + 1];        // slot -> pass-i mask over incidences
    int32_t srow[C::HS];               // rows in ascending order
    int32_t sfrk[C::HS];
    double sval[C::HS];
    double stv[LIFT ? C::HS : 1];      // lift: A(c, row), then A(c, row) u0[row]
    alignas(16) double lb[C::LK];      // load shares in incidence order
    alignas(16) double ld[C::LK];      // s_jj in incidence order
    double itm[D + 1][C::LK];          // item (i, incidence) = s_ij of the incidence's element
    uint32_t skey[C::LK];              // sorted incidence keys
};

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
template <int D, int L, int K, bool LIFT>
__global__ void __launch_bounds__(V4<D, L, K>::WARPS * 32, D == 3 ? 8 : 4) k_columns4(ColParams p) {
    using C = V4<D, L, K>;
    constexpr int NV = D + 1;
    constexpr int LK = C::LK;
    __shared__ V4Smem<D, L, K, LIFT> sm_all[C::WARPS * C::GPW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / L, g = lane % L;
    const unsigned gmask = (L == 32) ? kFull : (((1u << L) - 1) << (gi * L));
    const unsigned lower = (1u << lane) - 1;
    V4Smem<D, L, K, LIFT>& sm = sm_all[warp * C::GPW + gi];
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);

    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(p.ticket, 1u);
        tile = __shfl_sync(kFull, tile, 0);
        if (tile >= p.n_tiles) break;
        const int64_t sbase = tile * p.tile_cap;
        int run_a = 0, run_f = 0;  // warp-uniform: entries staged so far in this tile
        bool bad = false;
        const int32_t lc0 = (int32_t)(tile * C::WTC);
        const int ncol_t = (int)min((int64_t)C::WTC, (int64_t)p.n_cols - lc0);
        const int32_t ipl = lane <= ncol_t ? __ldg(p.inc_ptr + lc0 + lane) : 0;
        const int32_t ipe = __ldg(p.inc_ptr + lc0 + ncol_t);
        auto col_range = [&](int q, int32_t& p0, int32_t& m) {
            const int32_t a = __shfl_sync(kFull, ipl, q & 31);
            const int32_t b = __shfl_sync(kFull, ipl, (q + 1) & 31);
            p0 = a;
            m = q < ncol_t ? ((q + 1 >= ncol_t) ? ipe : b) - a : 0;
        };
        int32_t p0n, mn;
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
#pragma unroll
            for (int kk = 0; kk < K; ++kk) sm.skey[kk * L + g] = key[kk];
            if (p.want_a) {
                for (int h = g; h < C::HS; h += L) {
                    sm.row[h] = -1;
                    sm.crow[h] = -1;
#pragma unroll
                    for (int i = 0; i < NV; ++i) sm.msk[h][i] = 0u;
                }
            }
            __syncwarp();
            // ---- 2. per incidence: geometry of column j of element t from the
            //      label-ordered nodes, staged; its off-diagonal items' rows inserted
#pragma unroll 1
            for (int kk = 0; kk < K; ++kk) {
                const int e = kk * L + g;
                if (e >= m) {
                    if (e < LK) {
#pragma unroll
                        for (int i = 0; i < NV; ++i) sm.itm[i][e] = 0.0;
                        sm.lb[e] = 0.0;
                        sm.ld[e] = 0.0;
                    }
                    continue;
                }
                const uint32_t ky = sm.skey[e];
                const int32_t t_ = (int32_t)(ky & 0x3FFFFFFFu);
                const int j_ = (int)(ky >> 30);
                int32_t lv[NV];
                if constexpr (D == 3) {
                    const int4 ev = __ldg(reinterpret_cast<const int4*>(p.lel) + t_);
                    lv[0] = ev.x;
                    lv[1] = ev.y;
                    lv[2] = ev.z;
                    lv[3] = ev.w;
                } else {
#pragma unroll
                    for (int i = 0; i < NV; ++i) lv[i] = __ldg(p.lel + (size_t)t_ * NV + i);
                }
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
                    sm.itm[i][e] = s[i];
                    if (i == j_) sjj = s[i];
                }
                sm.lb[e] = lsh;
                sm.ld[e] = sjj;
                if (!p.want_a) continue;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    // exact-zero items are skipped: x + (+-0) == x for x != 0, a zero
                    // prefix only changes the sign of a zero the next nonzero item
                    // absorbs, and an all-zero entry is dropped anyway (sparse.hpp:105)
                    if (i == j_ || s[i] == 0.0) continue;
                    const int32_t r = R[i];
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
                        sm.frk[slot] = FR[i];
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
                const double* src = g == 0 ? sm.lb : sm.ld;
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
            const double b = __shfl_sync(kFull, fold, 0, L);
            const double dg = __shfl_sync(kFull, fold, 1, L);
            double ylift = 0.0;
            if (p.want_a) {
                // ---- 4. the diagonal slot, the folds, rows ranked, zero drop
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
                        const int je = e < m ? (int)(sm.skey[e] >> 30) : -1;
#pragma unroll
                        for (int jj = 0; jj < NV; ++jj)
                            jm[jj] |= ((__ballot_sync(kFull, je == jj) & gmask) >> (gi * L)) << (kk * L);
                    }
                }
                // one lane per occupied slot (the compacted list)
#pragma unroll 1
                for (int k = g; k < nocc; k += L) {
                    const int h = sm.cslot[k];
                    const int32_t r = sm.crow[k];
                    {
                        double acc = dg;
                        double tacc = dg;  // A(c, r): the transposed entry (lift only)
                        if (r != c) {
                            acc = -0.0;  // -0.0 + x == x: the fold starts at its first value
#pragma unroll
                            for (int i = 0; i < NV; ++i)
                                for (uint32_t mm = sm.msk[h][i]; mm; mm &= mm - 1)
                                    acc = acc + sm.itm[i][__ffs(mm) - 1];
                            if constexpr (LIFT) {
                                // A(c, r) folds the same items in (i_c*(d+1)+j_r, t) order:
                                // the incidence's own j first (incidences are sorted by j:
                                // contiguous ranges jm[jj]), then the pass, then incidences
                                tacc = -0.0;
#pragma unroll
                                for (int jj = 0; jj < NV; ++jj)
#pragma unroll
                                    for (int i = 0; i < NV; ++i)
                                        for (uint32_t mm = sm.msk[h][i] & jm[jj]; mm; mm &= mm - 1)
                                            tacc = tacc + sm.itm[i][__ffs(mm) - 1];
                            }
                        }
                        int rk = 0;  // rows below r; unused entries (-1) compare as huge
                        const int4* r4 = reinterpret_cast<const int4*>(sm.crow);
                        for (int qq = 0; qq < n4; ++qq) {
                            const int4 v = r4[qq];
                            rk += ((uint32_t)v.x < (uint32_t)r) + ((uint32_t)v.y < (uint32_t)r) +
                                  ((uint32_t)v.z < (uint32_t)r) + ((uint32_t)v.w < (uint32_t)r);
                        }
                        if (rk < C::MAXS) {
                            sm.srow[rk] = r;
                            sm.sfrk[rk] = sm.frk[h];
                            sm.sval[rk] = acc;
                            if constexpr (LIFT) sm.stv[rk] = tacc;
                        }
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
                            const double a = sm.stv[qq];
                            const int32_t r = sm.srow[qq];
                            if (a != 0.0 && sm.sfrk[qq] < 0) {
                                const double u = node_field4(p.g_dir, p.nodes, D, r);
                                use = u != 0.0;
                                sm.stv[qq] = a * u;
                            }
                        }
                        umask |= ((__ballot_sync(kFull, use) & gmask) >> (gi * L)) << base;
                    }
                    __syncwarp();
                    if (g == 0) {
                        double yy = 0.0;
                        for (uint32_t mm = umask; mm; mm &= mm - 1) yy = yy + sm.stv[__ffs(mm) - 1];
                        ylift = yy;
                    }
                    __syncwarp();
                }
                const bool col_free = fc_c >= 0;
                // compaction in chunks of L entries: counts per group first (the
                // groups of a warp stage their columns one after another)
                constexpr int NCH = (C::MAXS + L - 1) / L;
                int na = 0, nf = 0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int qq = ch * L + g;
                    const bool in = qq < nslot;
                    const double v = in ? sm.sval[qq] : 0.0;
                    const bool keep = in && v != 0.0;  // sparse.hpp:105
                    const bool keepf = keep && col_free && p.want_sys && sm.sfrk[qq] >= 0;
                    na += __popc(__ballot_sync(kFull, keep) & gmask);
                    nf += __popc(__ballot_sync(kFull, keepf) & gmask);
                }
                int pa = na, pf = nf;  // inclusive prefix over the groups (column order)
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    const int ya = __shfl_up_sync(kFull, pa, o);
                    const int yf = __shfl_up_sync(kFull, pf, o);
                    if (lane >= o) {
                        pa += ya;
                        pf += yf;
                    }
                }
                const int tot_a = __shfl_sync(kFull, pa, 31), tot_f = __shfl_sync(kFull, pf, 31);
                int wa = run_a + pa - na, wf = run_f + pf - nf;  // this column's first slot
                if (act && g == 0) {
                    p.colcnt_a[l] = wa + na;
                    if (p.want_sys) p.colcnt_f[l] = wf + nf;
                }
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int qq = ch * L + g;
                    const bool in = qq < nslot;
                    const double v = in ? sm.sval[qq] : 0.0;
                    const int32_t r = in ? sm.srow[qq] : 0;
                    const int32_t fr = in ? sm.sfrk[qq] : -1;
                    const bool keep = in && v != 0.0;
                    const bool keepf = keep && col_free && p.want_sys && fr >= 0;
                    const unsigned ba = __ballot_sync(kFull, keep) & gmask;
                    const unsigned bf = __ballot_sync(kFull, keepf) & gmask;
                    if (keep) {
                        const int64_t o = sbase + wa + __popc(ba & lower);
                        p.st_a_row[o] = r;
                        p.st_a_val[o] = v;
                    }
                    if (keepf) {
                        const int64_t o = sbase + wf + __popc(bf & lower);
                        p.st_f_row[o] = fr;
                        p.st_f_val[o] = v;
                    }
                    wa += __popc(ba);
                    wf += __popc(bf);
                }
                run_a += tot_a;
                run_f += tot_f;
            }
            // ---- per-column vectors, by label: {b, u0, b - A u0}
            if (act && g == 0) {
                double u0 = 0.0, bmod = b;
                if (p.want_sys) {
                    u0 = fc_c < 0 ? node_field4(p.g_dir, p.nodes, D, c) : 0.0;
                    bmod = LIFT ? b - ylift : b - 0.0;  // system.hpp:197-198
                }
                p.vst[l] = make_double4(b, u0, bmod, 0.0);
            }
            __syncwarp();
        }
        if (__any_sync(kFull, bad) && lane == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
    }
}

// ===========================================================================
// placement: label-ordered staging -> node-id-ordered CSC and vectors
// ===========================================================================
// entries of label l: tile l / wtc, in-tile inclusive count colcnt[l]
__device__ __forceinline__ int32_t col_count(const int32_t* colcnt, int32_t l, int wtc) {
    return colcnt[l] - ((l % wtc) ? colcnt[l - 1] : 0);
}

// Warp per 32 consecutive nodes.  Their destination runs are contiguous in the
// CSC arrays, so lanes copy entry q of the warp's run (found by a binary search
// over the 32 column prefixes): every store instruction writes 32 consecutive
// entries; the loads gather a few staged runs.
__global__ void __launch_bounds__(256) k4_place(ColParams p, int wtc, const int32_t* __restrict__ lab,
                                                const int32_t* __restrict__ ffscan) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int32_t N = p.n_cols;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w * 32 < N; w += nwarps) {
        const int32_t v = (int32_t)(w * 32) + lane;
        const bool in = v < N;
        const int32_t l = in ? __ldg(lab + v) : 0;
        const int32_t fr = (in && p.want_sys) ? __ldg(p.fidx + v) : -1;
        // vectors
        if (in) {
            const double4 vs = p.vst[l];
            if (p.want_b) p.b[v] = vs.x;
            if (p.want_sys) {
                p.u0[v] = vs.y;
                p.b_mod[v] = vs.z;
                if (fr >= 0) {
                    p.b_f[fr] = vs.z;
                    p.ff_col_ptr[fr] = __ldg(ffscan + v);
                }
            }
        }
        // A(free, free) col_ptr[n_free] = its nnz (free_rank[N] = n_free, k_partition's scan)
        if (w == 0 && lane == 0 && p.want_sys && p.want_a)
            p.ff_col_ptr[__ldg(p.fidx + 2 * (int64_t)N + 1)] = __ldg(ffscan + N);
        if (!p.want_a) continue;
#pragma unroll
        for (int f = 0; f < 2; ++f) {  // 0: A, 1: A(free, free)
            if (f == 1 && !p.want_sys) break;
            const int32_t* colcnt = f ? p.colcnt_f : p.colcnt_a;
            const int32_t* srow = f ? p.st_f_row : p.st_a_row;
            const double* sval = f ? p.st_f_val : p.st_a_val;
            int32_t* drow = f ? p.ff_row_idx : p.row_idx;
            double* dval = f ? p.ff_values : p.values;
            const int64_t cap = f ? p.cap_ff : p.cap_a;
            const bool has = in && (f == 0 || fr >= 0);
            const int32_t len = has ? col_count(colcnt, l, wtc) : 0;
            const int64_t src = has ? (int64_t)(l / wtc) * p.tile_cap + colcnt[l] - len : 0;
            int32_t pre = len;  // inclusive prefix over lanes
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(kFull, pre, o);
                if (lane >= o) pre += y;
            }
            const int32_t total = __shfl_sync(kFull, pre, 31);
            if (total == 0) continue;
            const int32_t excl = pre - len;
            // first destination: col_ptr of the warp's first column (f = 0), or of its
            // first free column (f = 1)
            int32_t d0;
            if (f == 0) {
                d0 = p.col_ptr[w * 32];
            } else {
                const unsigned fb = __ballot_sync(kFull, has);
                const int first = __ffs(fb) - 1;
                d0 = __shfl_sync(kFull, in ? __ldg(ffscan + v) : 0, first);
            }
            if ((int64_t)d0 + total > cap) {
                if (lane == 0) atomicOr(p.err, DERR_CAPACITY);
                continue;
            }
            for (int32_t q0 = 0; q0 < total; q0 += 32) {
                const int32_t qq = q0 + lane;
                // largest k with excl[k] <= qq (columns with len 0 share prefixes:
                // the search lands on the last of them, whose run holds qq)
                int k = 0;
#pragma unroll
                for (int stp = 16; stp > 0; stp >>= 1) {
                    const int32_t ek = __shfl_sync(kFull, excl, k + stp);
                    if (ek <= qq) k += stp;
                }
                const int32_t ek = __shfl_sync(kFull, excl, k);
                const int64_t sk = __shfl_sync(kFull, src, k);
                if (qq < total) {
                    const int64_t s = sk + (qq - ek);
                    drow[d0 + qq] = __ldcs(srow + s);
                    dval[d0 + qq] = __ldcs(sval + s);
                }
            }
        }
    }
}

// ===========================================================================
// host side
// ===========================================================================
int v4_lanes(int dim) { return dim == 2 ? 16 : 32; }  // incidences per column the kernel takes

int v4_plan(fl_ctx* ctx, fl_mesh* mesh, bool sync) {
    const cudaStream_t s = ctx->stream;
    auto& lp = mesh->lp;
    const int nv = mesh->dim + 1;
    const int32_t N = mesh->n_nodes;
    const int64_t n_entries = (int64_t)mesh->n_elems * nv;
    FL_TRY(lp.lab.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.ilab.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.lptr.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.lcnt.ensure(sizeof(int32_t) * ((size_t)N + 1)));
    FL_TRY(lp.linc.ensure(sizeof(uint32_t) * (size_t)std::max<int64_t>(n_entries, 1)));
    FL_TRY(lp.lel.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(n_entries, 4)));
    FL_TRY(lp.misc.ensure(sizeof(P4Misc)));
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(N)));
    P4Misc* misc = lp.misc.as<P4Misc>();
    int32_t* cnt = lp.lcnt.as<int32_t>();
    int32_t* lab = lp.lab.as<int32_t>();
    int32_t* ilab = lp.ilab.as<int32_t>();
    FL_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)N + 1), s));
    FL_CUDA(cudaMemsetAsync(misc, 0, sizeof(P4Misc), s));
    if (n_entries > 0) {
        const int64_t blocks = (n_entries + kP4Block * kP4Iters - 1) / (kP4Block * kP4Iters);
        k4_count<<<(int)blocks, kP4Block, 0, s>>>(n_entries, N, mesh->elems.as<int32_t>(), cnt, lab, ilab,
                                                  misc);
        count_launch(ctx);
    }
    if (N > 0) {
        k4_untouched<<<div_up(N, kP4Block), kP4Block, 0, s>>>(N, cnt, lab, ilab, misc);
        count_launch(ctx);
    }
    const int32_t* cc = cnt;
    const int32_t* il = ilab;
    FL_CUDA(launch_scan<int32_t>(
        N, [cc, il] __device__(int64_t i) { return (int64_t)cc[il[i]]; }, lp.lptr.as<int32_t>(),
        ctx->scan_ws.p, s));
    count_launch(ctx);
    // fill cursors start at the segment offsets
    FL_CUDA(cudaMemcpyAsync(cnt, lp.lptr.p, sizeof(int32_t) * ((size_t)N + 1), cudaMemcpyDeviceToDevice, s));
    if (n_entries > 0) {
        constexpr int U = 4;
        const int fgrid = (int)std::min<int64_t>(std::max<int64_t>(div_up(n_entries, 256 * U), 1), INT_MAX);
        k4_fill<U><<<fgrid, 256, 0, s>>>(n_entries, nv, N, mesh->elems.as<int32_t>(), lab, cnt,
                                         lp.linc.as<uint32_t>(), lp.lel.as<int32_t>());
        count_launch(ctx);
    }
    if (N > 0) {
        k4_stats<<<std::min(div_up(N, 256), ctx->sm_count * 8), 256, 0, s>>>(N, mesh->dim, lp.lptr.as<int32_t>(),
                                                                            misc);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
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
    lp.ok = lp.max_inc <= v4_lanes(mesh->dim);
    return FL_OK;
}

template <int D, int L, int K, bool LIFT>
static int launch4(fl_ctx* ctx, ColParams& p) {
    using C = V4<D, L, K>;
    int per_sm = 1;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_columns4<D, L, K, LIFT>, C::WARPS * 32, 0));
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((p.n_tiles + C::WARPS - 1) / C::WARPS, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    k_columns4<D, L, K, LIFT><<<(int)grid, C::WARPS * 32, 0, ctx->stream>>>(p);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

template <int D, int L, int K>
static int launch4_sel(fl_ctx* ctx, ColParams& p) {
    return p.need_lift ? launch4<D, L, K, true>(ctx, p) : launch4<D, L, K, false>(ctx, p);
}

// The column pass of fl_assemble on the label plan (whole mesh, no Neumann data:
// fl_api.cu routes those to the id-space kernels).  p carries the outputs, the
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
    FL_TRY(res->v4[2].ensure(sizeof(int32_t) * ((size_t)N + 2)));  // A_ff column scan by node id
    double4* xl = res->v4[0].as<double4>();
    p.xl = xl;
    p.vst = res->v4[1].as<double4>();
    p.lel = lp.lel.as<int32_t>();
    p.inc_ptr = lp.lptr.as<int32_t>();
    p.inc = lp.linc.as<uint32_t>();
    p.keys_sorted = false;
    if (N > 0) {
        k4_xl<<<std::min(div_up(N, 256), ctx->sm_count * 16), 256, 0, s>>>(
            N, dim, lp.ilab.as<int32_t>(), p.nodes, p.want_sys ? p.fidx : nullptr, xl);
        count_launch(ctx);
    }
    FL_TRY(prepare_staging(ctx, p, res, wtc, (int64_t)wtc * maxs));
    FL_CUDA(cudaMemsetAsync(p.ticket, 0, sizeof(uint32_t), s));
    if (ctx->profile) {
        FL_CUDA(cudaEventRecord(ctx->ev[5], s));
        FL_CUDA(cudaEventRecord(ctx->ev[6], s));
        ctx->kernel_timed = true;
    }
    // 8 lanes per column, 4 columns per warp: 2-D 1 or 2 incidences per lane
    // (valence <= 8 / 16), 3-D 4 (valence <= 32)
    const int kmax = lp.max_inc;
    if (dim == 2) {
        if (kmax <= 8) FL_TRY((launch4_sel<2, 8, 1>(ctx, p)));
        else FL_TRY((launch4_sel<2, 8, 2>(ctx, p)));
    } else {
        FL_TRY((launch4_sel<3, 8, 4>(ctx, p)));
    }
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[7], s));
    // placement: column pointers in node-id order, then the copy
    const int32_t* labp = lp.lab.as<int32_t>();
    int32_t* ffscan = res->v4[2].as<int32_t>();
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(N)));
    if (p.want_a) {
        const int32_t* ca = p.colcnt_a;
        const int w = wtc;
        FL_CUDA(launch_scan<int32_t>(
            N, [ca, labp, w] __device__(int64_t v) { return (int64_t)col_count(ca, labp[v], w); }, p.col_ptr,
            ctx->scan_ws.p, s));
        count_launch(ctx);
        if (p.want_sys) {
            const int32_t* cf = p.colcnt_f;
            const int32_t* fx = p.fidx;
            FL_CUDA(launch_scan<int32_t>(
                N,
                [cf, labp, fx, w] __device__(int64_t v) {
                    return (int64_t)(fx[v] >= 0 ? col_count(cf, labp[v], w) : 0);
                },
                ffscan, ctx->scan_ws.p, s));
            count_launch(ctx);
        }
    }
    if (N > 0) {
        const int64_t warps = std::min<int64_t>(((int64_t)N + 31) / 32, (int64_t)ctx->sm_count * 64);
        k4_place<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(p, wtc, labp, ffscan);
        count_launch(ctx);
    }
    FL_CUDA(cudaGetLastError());
    res->v4_used = true;
    return FL_OK;
}

}  // namespace fl
