// fl_columns2.cu -- the tiled column kernel (v2), the fast path of fl_assemble.
//
// One CTA assembles a tile of TC consecutive output columns (= reference CSC
// columns) in four phases:
//   1. incidence keys of the tile -> smem (unsorted, straight from the plan);
//   2. lane-per-incidence: rank of the key inside its column (the (j, t) order of
//      assembly.hpp:486-498 after sparse.hpp:79-89's stable passes), element
//      geometry for column j (fl_geometry.cuh), s_ij (i = 0..d) and the load
//      share, written to smem at the ranked position;
//   3. thread-per-column: b = 0 + sum of load shares in (j, t) order
//      (system.hpp:114-118); every entry (r, c) folded sequentially in the
//      reference order (i, j, t) (sweep i outer, ranked incidences inner);
//      optional transposed folds for the Dirichlet lift; zero drop
//      (sparse.hpp:105); A(free, free) rows; b, u0, b_mod, b_f;
//   4. CTA offsets by decoupled look-back, coalesced copy of the tile's entries.
// Columns that do not fit (too many incidences per tile / distinct rows per
// column) raise DERR_V2_OVERFLOW and the host reruns the mesh on the general
// warp-per-column kernel (fl_kernels.cu k_columns).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

template <int D>
struct Tile;
template <>
struct Tile<2> {
    static constexpr int TC = 64;      // columns per tile
    static constexpr int CAP = 768;    // incidences per tile
    static constexpr int HS = 16;      // slot table per column (distinct rows)
    static constexpr int MAXS = 12;    // max distinct rows accepted (load 0.75)
    static constexpr int THREADS = 128;
};
template <>
struct Tile<3> {
    static constexpr int TC = 32;
    static constexpr int CAP = 1024;
    static constexpr int HS = 32;
    static constexpr int MAXS = 24;
    static constexpr int THREADS = 128;
};

template <int D>
struct TileSmem {
    using T = Tile<D>;
    static constexpr int NV = D + 1;
    // phase 1/2 buffers (reused for the output lists after the fold)
    union {
        struct {
            double S[T::CAP][NV];  // s_ij for i = 0..D, ranked incidence order
            double Lb[T::CAP];     // load share
            int32_t R[T::CAP][NV]; // element vertices (rows)
            uint32_t ks[T::CAP];   // ranked keys (j << 30 | t)
        } in;
        struct {
            int32_t a_row[T::MAXS][T::TC];
            double a_val[T::MAXS][T::TC];
            int32_t f_row[T::MAXS][T::TC];
            double f_val[T::MAXS][T::TC];
        } out;
    } u;
    uint32_t key[T::CAP];          // unsorted keys
    int32_t ptr[T::TC + 1];
    int32_t tab_row[T::HS][T::TC];
    double tab_acc[T::HS][T::TC];
    double tab_tacc[T::HS][T::TC];
    int32_t na[T::TC + 1], nf[T::TC + 1];
    int64_t off_a, off_f;
    int32_t total_a, total_f;
    int32_t bad;
};

template <int D>
size_t tile_smem_bytes() { return sizeof(TileSmem<D>); }

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

template <int D>
__device__ __forceinline__ int tab_find_or_insert(TileSmem<D>& sm, int col, int32_t row, int& n) {
    constexpr int HS = Tile<D>::HS;
    uint32_t h = ((uint32_t)row * 2654435761u) >> (32 - ilog2(HS));
    while (true) {
        const int32_t k = sm.tab_row[h][col];
        if (k == row) return (int)h;
        if (k == -1) {
            if (n >= Tile<D>::MAXS) return -1;  // table at its load limit: overflow
            sm.tab_row[h][col] = row;
            sm.tab_acc[h][col] = -0.0;  // -0.0 + x == x: the fold starts at its first value
            sm.tab_tacc[h][col] = -0.0;
            ++n;
            return (int)h;
        }
        h = (h + 1) & (HS - 1);
    }
}

template <int D>
__device__ __forceinline__ int tab_find(const TileSmem<D>& sm, int col, int32_t row) {
    constexpr int HS = Tile<D>::HS;
    uint32_t h = ((uint32_t)row * 2654435761u) >> (32 - ilog2(HS));
    while (sm.tab_row[h][col] != row) h = (h + 1) & (HS - 1);
    return (int)h;
}

__device__ __forceinline__ double node_field(const FieldDesc& g, const double* nodes, int dim,
                                             int32_t k) {
    if (g.kind == FL_FIELD_SAMPLES) return __ldg(g.samples + k);
    if (g.kind == FL_FIELD_CONST) return g.value;
    const double x = nodes[(size_t)k * dim];
    const double y = nodes[(size_t)k * dim + 1];
    const double z = dim == 3 ? nodes[(size_t)k * dim + 2] : 0.0;
    return eval_point(g, x, y, z);
}

template <int D>
__global__ void __launch_bounds__(Tile<D>::THREADS) k_columns2(ColParams p) {
    using T = Tile<D>;
    constexpr int NV = D + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem<D>& sm = *reinterpret_cast<TileSmem<D>*>(smem_raw);
    __shared__ int64_t s_tile;
    const int tid = threadIdx.x;
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);

    while (true) {
        if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= p.n_tiles) break;
        const int32_t c0 = (int32_t)(tile * T::TC);
        const int ncols = min(T::TC, p.n_nodes - c0);

        // ---- phase 1: keys of the tile
        const int32_t base = __ldg(p.inc_ptr + c0);
        if (tid <= T::TC) {
            const int cc = min(tid, ncols);
            sm.ptr[tid] = __ldg(p.inc_ptr + c0 + cc) - base;
        }
        if (tid == 0) sm.bad = 0;
        __syncthreads();
        const int M = sm.ptr[ncols];
        if (M > T::CAP) {
            if (tid == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
            // keep the look-back chain alive
            if (tid == 0) lookback(p.tile_status, tile, 0);
            __syncthreads();
            continue;
        }
        for (int q = tid; q < M; q += T::THREADS) sm.key[q] = __ldg(p.inc + base + q);
        __syncthreads();

        // ---- phase 2: rank + geometry, lane per incidence
        for (int q = tid; q < M; q += T::THREADS) {
            const uint32_t key = sm.key[q];
            int lo = 0, hi = ncols;  // column: ptr[col] <= q < ptr[col+1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (sm.ptr[mid] <= q) lo = mid;
                else hi = mid;
            }
            const int pb = sm.ptr[lo], pe = sm.ptr[lo + 1];
            int rank = 0;
            for (int r = pb; r < pe; ++r) rank += sm.key[r] < key;
            const int pos = pb + rank;
            const int32_t t = (int32_t)(key & 0x3FFFFFFFu);
            const int j = (int)(key >> 30);
            int32_t V[NV];
            if constexpr (D == 3) {
                const int4 e = __ldg(reinterpret_cast<const int4*>(p.elems) + t);
                V[0] = e.x;
                V[1] = e.y;
                V[2] = e.z;
                V[3] = e.w;
            } else {
#pragma unroll
                for (int i = 0; i < NV; ++i) V[i] = __ldg(p.elems + (size_t)t * NV + i);
            }
            ElemCol<D> ec;
            ec.load(p.nodes, V);
            double s[NV];
            double meas;
            if constexpr (D == 2) meas = ec.stiffness_col(j, s);
            else meas = ec.stiffness_col(j, s, R6);
            if (meas == 0.0) atomicOr(p.err, DERR_DEGENERATE);
            if (p.want_a && p.coef.kind != FL_FIELD_NONE) {
                double a;
                if (p.coef.kind == FL_FIELD_CONST) a = p.coef.value;
                else if (p.coef.kind == FL_FIELD_SAMPLES) a = __ldg(p.coef.samples + t);
                else a = ec.coef_c5(R3);
#pragma unroll
                for (int i = 0; i < NV; ++i) s[i] = s[i] * a;
            }
            double l = 0.0;
            if (p.want_b) {
                if constexpr (D == 2) l = ec.load_col(j, t, p.f, R6);
                else l = ec.load_col(j, t, meas, p.f);
            }
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                sm.u.in.S[pos][i] = s[i];
                sm.u.in.R[pos][i] = V[i];
            }
            sm.u.in.Lb[pos] = l;
            sm.u.in.ks[pos] = key;
        }
        __syncthreads();

        // ---- phase 3: thread per column, exact sequential folds
        const int col = tid;
        const bool mine = col < ncols;
        const int32_t c = c0 + col;
        double b = 0.0, y = 0.0;
        int nslots = 0;
        if (mine) {
            const int pb = sm.ptr[col], pe = sm.ptr[col + 1];
            if (p.want_b)
                for (int k = pb; k < pe; ++k) b = b + sm.u.in.Lb[k];
            if (p.want_a) {
#pragma unroll
                for (int h = 0; h < T::HS; ++h) sm.tab_row[h][col] = -1;
                for (int i = 0; i < NV; ++i)
                    for (int k = pb; k < pe; ++k) {
                        const int32_t r = sm.u.in.R[k][i];
                        const int h = tab_find_or_insert<D>(sm, col, r, nslots);
                        if (h < 0) {
                            nslots = T::MAXS + 1;
                            break;
                        }
                        sm.tab_acc[h][col] = sm.tab_acc[h][col] + sm.u.in.S[k][i];
                    }
                if (nslots > T::MAXS) sm.bad = 1;
                if (p.need_lift && nslots <= T::MAXS) {
                    // entry (c, r) in its own order (i_c*(d+1)+j_r, t): sweep j (= local
                    // index of c, the ranked order's major key), then i, then t
                    int k0 = pb;
                    while (k0 < pe) {
                        const uint32_t jb = sm.u.in.ks[k0] >> 30;
                        int k1 = k0;
                        while (k1 < pe && (sm.u.in.ks[k1] >> 30) == jb) ++k1;
                        for (int i = 0; i < NV; ++i)
                            for (int k = k0; k < k1; ++k) {
                                const int h = tab_find<D>(sm, col, sm.u.in.R[k][i]);
                                sm.tab_tacc[h][col] = sm.tab_tacc[h][col] + sm.u.in.S[k][i];
                            }
                        k0 = k1;
                    }
                }
            }
            // Neumann data (system.hpp:123-172) at nodes on flag-2 faces: face-major
            // (lf, t) order, accumulated from 0.0, then b += add
            if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE && p.is_neu[c]) {
                double add = 0.0;
                for (int lf = 0; lf < NV; ++lf) {
                    int32_t last = -1;
                    while (true) {  // next element t > last with a flag-2 face lf containing c
                        int32_t best = INT_MAX;
                        int kb = -1;
                        for (int k = pb; k < pe; ++k) {
                            const uint32_t key = sm.u.in.ks[k];
                            const int32_t t = (int32_t)(key & 0x3FFFFFFFu);
                            const int j = (int)(key >> 30);
                            if (j == lf || t <= last || t >= best) continue;
                            if (p.flags[(size_t)t * NV + lf] != 2) continue;
                            best = t;
                            kb = k;
                        }
                        if (kb < 0) break;
                        last = best;
                        int32_t V[NV];
#pragma unroll
                        for (int i = 0; i < NV; ++i) V[i] = sm.u.in.R[kb][i];
                        ElemCol<D> ec;
                        ec.load(p.nodes, V);
                        add = add + ec.face_share(lf, p.g_neu, R3, best);
                    }
                }
                b = b + add;
            }
        }
        __syncthreads();  // all folds done: the input buffers become the output lists
        if (tid == 0) sm.total_a = sm.total_f = 0;
        if (mine && p.want_a) {
            // extract slots, insertion-sort by row into the output lists
            int n = 0;
            if (nslots <= T::MAXS) {
                for (int h = 0; h < T::HS; ++h) {
                    const int32_t r = sm.tab_row[h][col];
                    if (r < 0) continue;
                    const double v = sm.tab_acc[h][col];
                    const double tv = sm.tab_tacc[h][col];
                    int q = n++;
                    while (q > 0 && sm.u.out.a_row[q - 1][col] > r) {
                        sm.u.out.a_row[q][col] = sm.u.out.a_row[q - 1][col];
                        sm.u.out.a_val[q][col] = sm.u.out.a_val[q - 1][col];
                        sm.u.out.f_val[q][col] = sm.u.out.f_val[q - 1][col];
                        --q;
                    }
                    sm.u.out.a_row[q][col] = r;
                    sm.u.out.a_val[q][col] = v;
                    sm.u.out.f_val[q][col] = tv;  // transposed value (lift), parked
                }
            }
            // Dirichlet lift: (A u0)[c] = sum over stored A(c, r) in ascending r
            if (p.need_lift) {
                for (int q = 0; q < n; ++q) {
                    const int32_t r = sm.u.out.a_row[q][col];
                    const double a_cr = sm.u.out.f_val[q][col];
                    if (a_cr != 0.0 && p.is_dir[r]) {
                        const double u = node_field(p.g_dir, p.nodes, D, r);
                        if (u != 0.0) y = y + a_cr * u;
                    }
                }
            }
            // zero drop (sparse.hpp:105); A(free, free) keeps free rows of free columns
            const bool col_free = p.want_sys && p.fidx[c] >= 0;
            int na = 0, nf = 0;
            for (int q = 0; q < n; ++q) {
                const int32_t r = sm.u.out.a_row[q][col];
                const double v = sm.u.out.a_val[q][col];
                if (v == 0.0) continue;
                sm.u.out.a_row[na][col] = r;
                sm.u.out.a_val[na][col] = v;
                ++na;
                if (col_free) {
                    const int32_t fr = p.fidx[r];
                    if (fr >= 0) {
                        sm.u.out.f_row[nf][col] = fr;
                        sm.u.out.f_val[nf][col] = v;
                        ++nf;
                    }
                }
            }
            sm.na[col] = na;
            sm.nf[col] = nf;
        } else if (tid < T::TC) {
            sm.na[tid] = sm.nf[tid] = 0;
        }
        __syncthreads();
        // ---- phase 4: tile prefix, look-back, coalesced writes
        if (tid == 0) {
            int32_t ra = 0, rf = 0;
            for (int q = 0; q < T::TC; ++q) {
                const int32_t a = sm.na[q], f = sm.nf[q];
                sm.na[q] = ra;
                sm.nf[q] = rf;
                ra += a;
                rf += f;
            }
            sm.na[T::TC] = ra;
            sm.nf[T::TC] = rf;
            if (sm.bad) atomicOr(p.err, DERR_V2_OVERFLOW);
            const uint64_t ex = lookback(p.tile_status, tile, ((uint64_t)rf << 31) | (uint64_t)ra);
            sm.off_a = (int64_t)(ex & 0x7FFFFFFFull);
            sm.off_f = (int64_t)(ex >> 31);
        }
        __syncthreads();
        const int64_t off_a = sm.off_a, off_f = sm.off_f;
        const int ta = sm.na[T::TC], tf = sm.nf[T::TC];
        if (p.want_a) {
            if (off_a + ta > p.cap_a || off_f + tf > p.cap_ff) {
                if (tid == 0) atomicOr(p.err, DERR_CAPACITY);
            } else {
                for (int e = tid; e < ta; e += T::THREADS) {
                    int lo = 0, hi = T::TC;  // column of entry e
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (sm.na[mid] <= e) lo = mid;
                        else hi = mid;
                    }
                    while (lo + 1 < T::TC && sm.na[lo + 1] <= e) ++lo;
                    const int q = e - sm.na[lo];
                    p.row_idx[off_a + e] = sm.u.out.a_row[q][lo];
                    p.values[off_a + e] = sm.u.out.a_val[q][lo];
                }
                if (p.want_sys)
                    for (int e = tid; e < tf; e += T::THREADS) {
                        int lo = 0, hi = T::TC;
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (sm.nf[mid] <= e) lo = mid;
                            else hi = mid;
                        }
                        while (lo + 1 < T::TC && sm.nf[lo + 1] <= e) ++lo;
                        const int q = e - sm.nf[lo];
                        p.ff_row_idx[off_f + e] = sm.u.out.f_row[q][lo];
                        p.ff_values[off_f + e] = sm.u.out.f_val[q][lo];
                    }
                if (mine) {
                    p.col_ptr[c + 1] = (int32_t)(off_a + sm.na[col + 1]);
                }
            }
        }
        if (mine) {
            if (p.want_b) p.b[c] = b;
            if (p.want_sys) {
                const bool dir = p.is_dir[c];
                const double u0 = dir ? node_field(p.g_dir, p.nodes, D, c) : 0.0;
                const double bmod = p.need_lift ? b - y : b - 0.0;
                p.u0[c] = u0;
                p.b_mod[c] = bmod;
                const int32_t fc = p.fidx[c];
                if (fc >= 0) {
                    p.b_f[fc] = bmod;
                    if (p.want_a) p.ff_col_ptr[fc + 1] = (int32_t)(off_f + sm.nf[col + 1]);
                }
            }
        }
        __syncthreads();
    }
}

int launch_columns2(fl_ctx* ctx, int dim, ColParams& p) {
    if (dim == 2) {
        const size_t smem = sizeof(TileSmem<2>);
        p.n_tiles = (p.n_nodes + Tile<2>::TC - 1) / Tile<2>::TC;
        FL_CUDA(cudaFuncSetAttribute(k_columns2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_columns2<2>, Tile<2>::THREADS, smem);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.n_tiles, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
        k_columns2<2><<<grid, Tile<2>::THREADS, smem, ctx->stream>>>(p);
    } else {
        const size_t smem = sizeof(TileSmem<3>);
        p.n_tiles = (p.n_nodes + Tile<3>::TC - 1) / Tile<3>::TC;
        FL_CUDA(cudaFuncSetAttribute(k_columns2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_columns2<3>, Tile<3>::THREADS, smem);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(p.n_tiles, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
        k_columns2<3><<<grid, Tile<3>::THREADS, smem, ctx->stream>>>(p);
    }
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

int64_t columns2_tiles(int dim, int32_t n_nodes) {
    const int tc = dim == 2 ? Tile<2>::TC : Tile<3>::TC;
    return (n_nodes + tc - 1) / tc;
}

}  // namespace fl
