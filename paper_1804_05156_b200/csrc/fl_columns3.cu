// fl_columns3.cu -- the register-centric column kernel (v3), fast path of fl_assemble.
//
// A group of L lanes (L = 8 in 2-D, 32 in 3-D; a warp holds 32/L groups) owns
// one output column c = one reference CSC column.  No block barriers: every warp
// is independent, so the SM hides latency with occupancy.
//   1. lane g < m loads incidence key g of c (j << 30 | t, unsorted from the
//      plan) and the group bitonic-sorts the keys: lane g then holds the g-th
//      incidence in (j, t) order -- the order in which the reference's
//      blockwise triplets reach column c (assembly.hpp:286-298 after the stable
//      passes sparse.hpp:79-89);
//   2. each lane reads its incidence's row of the element record (k_elem_records,
//      s_ij for i = 0..d, the load share, the vertices; FMA-free, exact
//      division) -- or, with FL_KERNEL=3, computes them itself (fl_geometry.cuh);
//   3. b = 0.0 + shares in lane order (system.hpp:114-118) and the diagonal
//      A(c,c) = fold of s_jj in lane order (its items are exactly those): the
//      shares are staged in smem and group lanes 0 / 1 run the two folds;
//   4. off-diagonal items (i != j) are staged at itm[i][lane]; every lane inserts
//      its rows into the group's small smem hash (CAS: equal rows meet on one
//      slot) and sets its lane bit in the slot's pass-i mask (atomicOr); the
//      slot's lane then folds its items pass by pass, lanes ascending = the
//      reference's (i*(d+1)+j, t) order;
//   5. slots ranked by row, exact zeros dropped (sparse.hpp:105), A(free,free)
//      rows kept, all written to the tile staging (k_stage_copy places them).
// Limits (fallback to the general kernel through DERR_V2_OVERFLOW): m > L, or
// more distinct rows than the group table holds.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

// 2-D records are stored straight from registers as whole 32-byte sectors; 3-D
// ones go through shared memory for coalesced stores (each measured faster on
// its dimension: C3 records 2.99 -> 2.92 ms direct, C4 0.55 -> 0.62 ms direct)
template <int D>
__host__ __device__ constexpr bool rec_direct() { return D == 2; }

__host__ __device__ constexpr int lg2(int x) { return x <= 1 ? 0 : 1 + lg2(x >> 1); }

// K incidences per lane: K = 2 (3-D) takes columns of up to 64 incidences
template <int D, int L, int K = 1>
struct V3 {
    static constexpr int NV = D + 1;
    static constexpr int GPW = 32 / L;                 // column groups per warp
    static constexpr int HS = D == 2 ? 16 : L * K;          // slot table entries per group
    static constexpr int MAXS = D == 2 ? 12 : (3 * L * K) / 4;  // distinct rows accepted per column
    static constexpr int WTC = D == 2 ? 32 : 8;        // columns per warp tile
    static constexpr int ITERS = WTC / GPW;            // group iterations per warp tile
    static constexpr int WARPS = 4;                    // warps per CTA
};

template <int D, int L, int K = 1>
struct V3Smem {  // one per group
    using C = V3<D, L, K>;
    alignas(16) int32_t row[C::HS];   // slot -> row (-1 empty)
    alignas(16) int32_t crow[C::HS];  // occupied rows, compacted (-1 padded)
    uint4 msk[C::HS][K];              // slot -> lane mask of its items, word [kk].(pass)
    int32_t srow[C::HS];              // rows in ascending order
    double sval[C::HS];
    double stv[C::HS];                // lift: A(c, row) in row order, then A(c,row) u0[row]
    alignas(16) double lb[L * K];     // load shares in incidence order
    alignas(16) double ld[L * K];     // s_jj in incidence order
    double itm[D + 1][L * K];         // item (i, incidence) = s_i of the incidence's element
};

__device__ __forceinline__ unsigned& mword(uint4& w, int i) { return reinterpret_cast<unsigned*>(&w)[i]; }

__device__ __forceinline__ double node_field3(const FieldDesc& g, const double* nodes, int dim,
                                              int32_t k) {
    if (g.kind == FL_FIELD_SAMPLES) return __ldg(g.samples + k);
    if (g.kind == FL_FIELD_CONST) return g.value;
    const double x = nodes[(size_t)k * dim];
    const double y = nodes[(size_t)k * dim + 1];
    const double z = dim == 3 ? nodes[(size_t)k * dim + 2] : 0.0;
    return eval_point(g, x, y, z);
}

// Element-first records: one thread per element computes the whole local
// matrix (stiffness_all: the same operations as stiffness_col, s_ij == s_ji)
// times the coefficient, and the load shares of its D+1 vertices, once --
// instead of once per incident column.
constexpr int kElemThreads = 128;

template <int D>
__global__ void __launch_bounds__(kElemThreads, D == 3 ? 8 : 6) k_elem_records(ColParams p) {
    constexpr int NV = D + 1;
    // per element: D == 3: the full local matrix, row-major (8 int4) + 4 load
    // shares (2 int4); D == 2: rows {s_0j, s_1j, s_2j, load_j} (6 int4)
    constexpr int WS = rec64<D>() ? 4 * NV : 8, WL = rec64<D>() ? 0 : 2;
    constexpr int W = WS + WL + 1;  // +1: no bank conflicts
    __shared__ int4 stage[rec_direct<D>() ? 1 : kElemThreads * W];
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);
    for (int64_t t0 = (int64_t)blockIdx.x * kElemThreads; t0 < p.n_elems;
         t0 += (int64_t)gridDim.x * kElemThreads) {
        const int64_t t = t0 + threadIdx.x;
        if (t < p.n_elems && (!p.emark || p.emark[t])) {
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
            // vertex ids outside [0, N): reported, never dereferenced
            bool okv = true;
#pragma unroll
            for (int i = 0; i < NV; ++i) okv = okv && (uint32_t)V[i] < (uint32_t)p.n_nodes;
            if (!okv) {
                atomicOr(p.err, DERR_INDEX);
#pragma unroll
                for (int i = 0; i < NV; ++i) V[i] = 0;
            }
            ElemCol<D> ec;
            ec.load(p.nodes, V);
            double S[NV][NV];
            double meas;
            if constexpr (D == 2) meas = ec.stiffness_all(S);
            else meas = ec.stiffness_all(S, R6);
            if (meas == 0.0) atomicOr(p.err, DERR_DEGENERATE);
            if (p.want_a && p.coef.kind != FL_FIELD_NONE) {
                double a;
                if (p.coef.kind == FL_FIELD_CONST) a = p.coef.value;
                else if (p.coef.kind == FL_FIELD_SAMPLES) a = __ldg(p.coef.samples + t);
                else a = ec.coef_c5(R3);
#pragma unroll
                for (int j = 0; j < NV; ++j)
#pragma unroll
                    for (int i = 0; i < NV; ++i) S[j][i] = S[j][i] * a;
            }
            double Lj[NV];
            if constexpr (D == 2) {
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    Lj[j] = p.want_b ? ec.load_col(j, (int32_t)t, p.f, R6) : 0.0;
            } else {
                if (p.want_b) ec.load_all((int32_t)t, meas, p.f, Lj);
                else Lj[0] = Lj[1] = Lj[2] = Lj[3] = 0.0;
            }
            // records: row j of the local matrix (= column j, s_ij == s_ji) is one
            // 32-byte line the column kernel reads with a single 256-bit load
            if constexpr (rec_direct<D>()) {
            // whole 32-byte sectors straight from registers (256-bit stores)
            auto st32 = [](double* a, double x0, double x1, double x2, double x3) {
                asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(a), "d"(x0), "d"(x1), "d"(x2),
                             "d"(x3)
                             : "memory");
            };
            if constexpr (rec64<D>()) {
                double* rec = p.srec + (size_t)t * NV * 8;
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    st32(rec + 8 * j, S[j][0], S[j][1], S[j][2], D == 3 ? S[j][3] : Lj[j]);
                    st32(rec + 8 * j + 4, Lj[j], __hiloint2double(V[1], V[0]),
                         __hiloint2double(D == 3 ? V[D] : 0, V[2]), 0.0);
                }
            } else {
                double* rec = p.srec + (size_t)t * NV * 4;
#pragma unroll
                for (int j = 0; j < NV; ++j) st32(rec + 4 * j, S[j][0], S[j][1], S[j][2], D == 3 ? S[j][3] : Lj[j]);
                if constexpr (D == 3) st32(p.lrec + (size_t)t * 4, Lj[0], Lj[1], Lj[2], Lj[3]);
            }
            } else {
            int4* st = stage + threadIdx.x * W;
            if constexpr (rec64<D>()) {
                const int4 ids = make_int4(V[0], V[1], V[2], D == 3 ? V[D] : 0);
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    double2 w0 = make_double2(S[j][0], S[j][1]);
                    double2 w1 = make_double2(S[j][2], D == 3 ? S[j][3] : Lj[j]);
                    st[4 * j] = *reinterpret_cast<int4*>(&w0);
                    st[4 * j + 1] = *reinterpret_cast<int4*>(&w1);
                    st[4 * j + 2] = make_int4(__double2loint(Lj[j]), __double2hiint(Lj[j]), ids.x, ids.y);
                    st[4 * j + 3] = make_int4(ids.z, ids.w, 0, 0);
                }
            } else {
#pragma unroll
                for (int j = 0; j < NV; ++j) {
                    double2 w0 = make_double2(S[j][0], S[j][1]);
                    double2 w1 = make_double2(S[j][2], D == 3 ? S[j][3] : Lj[j]);
                    st[2 * j] = *reinterpret_cast<int4*>(&w0);
                    st[2 * j + 1] = *reinterpret_cast<int4*>(&w1);
                }
            }
            if constexpr (D == 3 && WL > 0) {
                double2 l01 = make_double2(Lj[0], Lj[1]), l23 = make_double2(Lj[2], Lj[3]);
                st[WS] = *reinterpret_cast<int4*>(&l01);
                st[WS + 1] = *reinterpret_cast<int4*>(&l23);
            }
            }
        }
        if constexpr (rec_direct<D>()) continue;  // no staging: nothing to synchronise
        __syncthreads();
        // coalesced write-out of the block's contiguous records
        const int64_t n = min((int64_t)kElemThreads, p.n_elems - t0);
        int4* out = reinterpret_cast<int4*>(p.srec) + t0 * WS;
        for (int q = threadIdx.x; q < n * WS; q += kElemThreads) out[q] = stage[(q / WS) * W + q % WS];
        if constexpr (WL > 0) {
            int4* outl = reinterpret_cast<int4*>(p.lrec) + t0 * WL;
            for (int q = threadIdx.x; q < n * WL; q += kElemThreads)
                outl[q] = stage[(q / WL) * W + WS + q % WL];
        }
        __syncthreads();
    }
}

template <int D, int L, bool PRE, bool LIFT, int K>
__global__ void __launch_bounds__(V3<D, L>::WARPS * 32, PRE ? (K == 1 ? 10 : (L == 16 ? 8 : 6)) : 5) k_columns3(ColParams p) {
    using C = V3<D, L, K>;
    constexpr int NV = D + 1;
    constexpr int LK = L * K;  // incidences a group takes
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ V3Smem<D, L, K> sm_all[C::WARPS * C::GPW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gi = lane / L, g = lane % L;  // group in warp, lane in group
    const unsigned gmask = (L == 32) ? FULL : (((1u << L) - 1) << (gi * L));
    const unsigned lower = (1u << lane) - 1;
    V3Smem<D, L, K>& sm = sm_all[warp * C::GPW + gi];
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);

    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(p.ticket, 1u);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= p.n_tiles) break;
        const int64_t sbase = tile * p.tile_cap;
        int run_a = 0, run_f = 0;  // warp-uniform: entries staged so far in this tile
        bool bad = false;
        // the tile's column bounds: one inc_ptr load per lane (WTC <= 32), then
        // shuffles; the next column's keys are prefetched one iteration ahead
        const int32_t lc0 = (int32_t)(tile * C::WTC);
        const int ncol_t = (int)min((int64_t)C::WTC, (int64_t)p.n_cols - lc0);
        const int32_t ipl = lane <= ncol_t ? __ldg(p.inc_ptr + lc0 + lane) : 0;
        const int32_t ipe = __ldg(p.inc_ptr + lc0 + ncol_t);
        auto col_range = [&](int q, int32_t& p0, int32_t& m) {
            const int32_t a = __shfl_sync(FULL, ipl, q & 31);
            const int32_t b = __shfl_sync(FULL, ipl, (q + 1) & 31);
            p0 = a;
            m = q < ncol_t ? ((q + 1 >= ncol_t) ? ipe : b) - a : 0;
        };
        int32_t p0n, mn;
        col_range(gi, p0n, mn);
        uint32_t key_next[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
            key_next[kk] = (kk * L + g < mn && mn <= LK) ? __ldg(p.inc + p0n + kk * L + g) : 0xFFFFFFFFu;
        for (int it = 0; it < C::ITERS; ++it) {
            const int q = it * C::GPW + gi;
            const int32_t lc = lc0 + q;  // owned column
            const bool act = q < ncol_t;
            const int32_t c = p.c_begin + lc;  // global node
            // the column's partition data, loaded early (used after the folds)
            const int32_t fc_c = (act && p.want_sys) ? __ldg(p.fidx + c) : -1;
            const bool dir_c = act && p.want_sys && __ldg(p.is_dir + c);
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
            if (m > LK) {  // hybrid: the general kernel takes the column afterwards
                if (!p.hybrid) bad = true;
                m = 0;
#pragma unroll
                for (int kk = 0; kk < K; ++kk) key[kk] = 0xFFFFFFFFu;
            }
            // ---- 1. keys, sorted ascending inside the group: incidence e = kk*L + g
            //      (bitonic over L*K; distances >= L pair registers of one lane);
            //      a cached plan's segments were sorted once (k_inc_sort)
            if (!p.keys_sorted)
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
                            const uint32_t o = __shfl_xor_sync(FULL, key[kk], jj, L);
                            const bool up = ((kk * L + g) & k) == 0;
                            const bool lo = (g & jj) == 0;
                            key[kk] = (lo == up) ? min(key[kk], o) : max(key[kk], o);
                        }
                    }
                }
            }
            bool valid[K];
            int32_t t[K];
            int j[K];
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                valid[kk] = kk * L + g < m;
                t[kk] = (int32_t)(key[kk] & 0x3FFFFFFFu);
                j[kk] = valid[kk] ? (int)(key[kk] >> 30) : 0;
            }
            // ---- 2. geometry of column j of element t
            int32_t RR[K][NV];
            double ss[K][NV];
            double ll[K], sjjk[K];
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
            int32_t* R = RR[kk];
            double* s = ss[kk];
            double l = 0.0, sjj = 0.0;
            const int32_t t_ = t[kk];
            const int j_ = j[kk];
            const bool valid_ = valid[kk];
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                R[i] = -1;
                s[i] = 0.0;
            }
            if (valid_ && PRE && rec64<D>()) {
                // the incidence's 64-byte record: two 256-bit loads of one block
                const double* row = p.srec + ((size_t)t_ * NV + j_) * 8;
                double q0, q1, q2, q3;
                uint32_t w[8];
                asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                    : "=d"(q0), "=d"(q1), "=d"(q2), "=d"(q3) : "l"(row));
                asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                      "=r"(w[7])
                    : "l"(row + 4));
                s[0] = q0;
                s[1] = q1;
                s[2] = q2;
                if constexpr (D == 3) s[3] = q3;
                l = __hiloint2double((int)w[1], (int)w[0]);
#pragma unroll
                for (int i = 0; i < NV; ++i) R[i] = (int32_t)w[2 + i];
            } else if (valid_ && PRE) {
                // row j of the element's local matrix: one 256-bit load; the load
                // share (3-D) and the vertex ids from their own arrays
                const double* row = p.srec + ((size_t)t_ * NV + j_) * 4;
                double q0, q1, q2, q3;
                asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                    : "=d"(q0), "=d"(q1), "=d"(q2), "=d"(q3) : "l"(row));
                s[0] = q0;
                s[1] = q1;
                s[2] = q2;
                if constexpr (D == 3) {
                    s[3] = q3;
                    l = __ldg(p.lrec + (size_t)t_ * 4 + j_);
                    const int4 e = __ldg(reinterpret_cast<const int4*>(p.elems) + t_);
                    R[0] = e.x;
                    R[1] = e.y;
                    R[2] = e.z;
                    R[3] = e.w;
                } else {
                    l = q3;
#pragma unroll
                    for (int i = 0; i < NV; ++i) R[i] = __ldg(p.elems + (size_t)t_ * NV + i);
                }
            } else if (valid_) {
                if constexpr (D == 3) {
                    const int4 e = __ldg(reinterpret_cast<const int4*>(p.elems) + t_);
                    R[0] = e.x;
                    R[1] = e.y;
                    R[2] = e.z;
                    R[3] = e.w;
                } else {
#pragma unroll
                    for (int i = 0; i < NV; ++i) R[i] = __ldg(p.elems + (size_t)t_ * NV + i);
                }
                {
                    ElemCol<D> ec;
                    ec.load(p.nodes, R);
                    double meas;
                    if constexpr (D == 2) meas = ec.stiffness_col(j_, s);
                    else meas = ec.stiffness_col(j_, s, R6);
                    if (meas == 0.0) atomicOr(p.err, DERR_DEGENERATE);
                    if (p.want_a && p.coef.kind != FL_FIELD_NONE) {
                        double a;
                        if (p.coef.kind == FL_FIELD_CONST) a = p.coef.value;
                        else if (p.coef.kind == FL_FIELD_SAMPLES) a = __ldg(p.coef.samples + t_);
                        else a = ec.coef_c5(R3);
#pragma unroll
                        for (int i = 0; i < NV; ++i) s[i] = s[i] * a;
                    }
                    if (p.want_b) {
                        if constexpr (D == 2) l = ec.load_col(j_, t_, p.f, R6);
                        else l = ec.load_col(j_, t_, meas, p.f);
                    }
                }
            }
            if (valid_) {
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    if (i == j_) sjj = s[i];
            }
            ll[kk] = l;
            sjjk[kk] = sjj;
            }

            // ---- 3. b and the diagonal: sequential folds in lane order (lanes 0 / 1)
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                sm.lb[kk * L + g] = ll[kk];
                sm.ld[kk * L + g] = sjjk[kk];
            }
            __syncwarp();
            double fold = g == 0 ? 0.0 : -0.0;
            if (g < 2) {
                const double* src = g == 0 ? sm.lb : sm.ld;
                const double2* src2 = reinterpret_cast<const double2*>(src);
                const int np = m >> 1;
#pragma unroll 2
                for (int q = 0; q < np; ++q) {
                    const double2 v = src2[q];
                    fold = fold + v.x;
                    fold = fold + v.y;
                }
                if (m & 1) fold = fold + src[m - 1];
            }
            double b = __shfl_sync(FULL, fold, 0, L);
            const double dg = __shfl_sync(FULL, fold, 1, L);
            if (p.nadd && act && p.is_neu[c]) b = b + p.nadd[lc];  // apply_neumann: b + add
            double ylift = 0.0;  // (A u0)[c], lift path (group lane 0)
            // ---- 4. off-diagonal items.  Item (i, lane) sits at itm[i][lane]; its
            //      row's slot (CAS insert) gets the lane's bit in msk[slot][i].
            //      Slot h then folds its items pass by pass, lanes ascending: the
            //      reference's (i*(d+1)+j, t) order.
            if (p.want_a) {
                for (int h = g; h < C::HS; h += L) {
                    sm.row[h] = -1;
                    sm.crow[h] = -1;
#pragma unroll
                    for (int kk = 0; kk < K; ++kk) sm.msk[h][kk] = make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int kk = 0; kk < K; ++kk)
#pragma unroll
                    for (int i = 0; i < NV; ++i) sm.itm[i][kk * L + g] = ss[kk][i];
                __syncwarp();
#pragma unroll
                for (int i = 0; i < NV; ++i)
#pragma unroll
                for (int kk = 0; kk < K; ++kk) {
                    // exact-zero items are skipped: x + (+-0) == x for x != 0, a zero
                    // prefix only changes the sign of a zero that the next nonzero item
                    // absorbs, and an entry whose items are all zero is dropped anyway
                    // (sparse.hpp:105) -- so its row never needs a slot
                    if (!valid[kk] || i == j[kk] || ss[kk][i] == 0.0) continue;
                    // every lane inserts its own row (equal rows meet on one slot: the
                    // CAS returns the row) and sets its bit in the slot's pass-i mask;
                    // the bit position is the lane, so atomic order does not matter
                    const int32_t r = RR[kk][i];
                    uint32_t h = ((uint32_t)r * 2654435761u) >> (32 - lg2(C::HS));
                    int slot = -1;
                    for (int probe = 0; probe < C::HS; ++probe) {
                        const int32_t old = atomicCAS(&sm.row[h], -1, r);
                        if (old == -1 || old == r) {
                            slot = (int)h;
                            break;
                        }
                        h = (h + 1) & (C::HS - 1);
                    }
                    if (slot >= 0) atomicOr(&mword(sm.msk[slot][kk], i), 1u << g);
                    else bad = true;
                }
                __syncwarp();
                // ---- 5. the diagonal slot, the folds, rows ranked, zero drop
                if (g == 0 && act && m > 0) {
                    uint32_t h = ((uint32_t)c * 2654435761u) >> (32 - lg2(C::HS));
                    for (int probe = 0; probe < C::HS; ++probe) {
                        if (sm.row[h] == -1) {
                            sm.row[h] = c;
                            break;
                        }
                        h = (h + 1) & (C::HS - 1);
                    }
                }
                __syncwarp();
                // occupied slots, compacted (rank candidates)
                int nocc = 0;
#pragma unroll
                for (int base = 0; base < C::HS; base += L) {
                    const int32_t r = sm.row[base + g];
                    const unsigned bal = __ballot_sync(FULL, r >= 0) & gmask;
                    if (r >= 0) sm.crow[nocc + __popc(bal & lower)] = r;
                    nocc += __popc(bal);
                }
                __syncwarp();
                const int n4 = (nocc + 3) >> 2;
                unsigned jm[NV][K];  // lift: lanes (group-relative) whose incidence has j == jj
#pragma unroll
                for (int jj = 0; jj < NV; ++jj)
#pragma unroll
                    for (int kk = 0; kk < K; ++kk)
                        jm[jj][kk] = LIFT ? (__ballot_sync(FULL, valid[kk] && j[kk] == jj) & gmask) >> (gi * L) : 0u;
#pragma unroll
                for (int base = 0; base < C::HS; base += L) {
                    const int h = base + g;
                    const int32_t r = sm.row[h];
                    if (r >= 0) {
                        double acc = dg;
                        double tacc = dg;  // A(c, r): the transposed entry (lift only)
                        if (r != c) {
                            acc = -0.0;  // -0.0 + x == x: the fold starts at its first value
                            // bit b of the concatenated pass masks = item itm[b / L][b % L]:
                            // ascending bits walk (i, lane) in the reference's order
                            const uint4 mk4 = sm.msk[h][0];
                            if constexpr (D == 3) {  // pass by pass, incidences ascending
#pragma unroll
                                for (int i = 0; i < NV; ++i)
#pragma unroll
                                    for (int kk = 0; kk < K; ++kk)
                                        for (unsigned mm = mword(sm.msk[h][kk], i); mm; mm &= mm - 1)
                                            acc = acc + sm.itm[i][kk * L + __ffs(mm) - 1];
                            } else {  // the passes' L-bit masks concatenated: bit b = itm[b / L][b % L]
                                const double* flat = &sm.itm[0][0];
                                if constexpr (3 * L <= 32) {  // L = 8: one 32-bit word
                                    const uint32_t w0 = mk4.x | (mk4.y << L) | (mk4.z << (2 * L));
                                    for (uint32_t w = w0; w; w &= w - 1) acc = acc + flat[__ffs(w) - 1];
                                } else {
                                    const uint64_t w0 = (uint64_t)mk4.x | ((uint64_t)mk4.y << L) |
                                                        ((uint64_t)mk4.z << (2 * L));
                                    for (uint64_t w = w0; w; w &= w - 1) acc = acc + flat[__ffsll(w) - 1];
                                }
                            }
                            if constexpr (LIFT) {
                                // A(c, r) folds the same items in (i_c*(d+1)+j_r, t) order: the
                                // lane's own j (lanes are sorted by j: contiguous ranges jm[jj])
                                // first, then the pass, then lanes ascending
                                tacc = -0.0;
#pragma unroll
                                for (int jj = 0; jj < NV; ++jj)
#pragma unroll
                                    for (int i = 0; i < NV; ++i)
#pragma unroll
                                        for (int kk = 0; kk < K; ++kk)
                                            for (unsigned mm = mword(sm.msk[h][kk], i) & jm[jj][kk]; mm;
                                                 mm &= mm - 1)
                                                tacc = tacc + sm.itm[i][kk * L + __ffs(mm) - 1];
                            }
                        }
                        int rk = 0;  // rows below r; unused entries (-1) compare as huge
                        const int4* r4 = reinterpret_cast<const int4*>(sm.crow);
                        for (int q = 0; q < n4; ++q) {
                            const int4 v = r4[q];
                            rk += ((uint32_t)v.x < (uint32_t)r) + ((uint32_t)v.y < (uint32_t)r) +
                                  ((uint32_t)v.z < (uint32_t)r) + ((uint32_t)v.w < (uint32_t)r);
                        }
                        if (rk < C::MAXS) {
                            sm.srow[rk] = r;
                            sm.sval[rk] = acc;
                            sm.stv[rk] = tacc;
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
                    // y = (A u0)[c] = 0.0 + A(c, r) * u0[r] over the stored entries of row c,
                    // r ascending (matvec, sparse.hpp:129-141); u0 = g at Dirichlet nodes
                    uint32_t umask = 0;  // rows whose product enters the sum
                    for (int base = 0; base < C::MAXS; base += L) {
                        const int q = base + g;
                        bool use = false;
                        if (q < nslot) {
                            const double a = sm.stv[q];
                            const int32_t r = sm.srow[q];
                            if (a != 0.0 && p.is_dir[r]) {
                                const double u = node_field3(p.g_dir, p.nodes, D, r);
                                use = u != 0.0;
                                sm.stv[q] = a * u;
                            }
                        }
                        umask |= ((__ballot_sync(FULL, use) & gmask) >> (gi * L)) << base;
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
                int na = 0, nf = 0;
                // compaction in chunks of L entries; pass 1: counts per group (one
                // group per warp: the column starts at the warp's running count)
                constexpr int NCH = (C::MAXS + L - 1) / L;
                int32_t frc[NCH];  // free ranks of the chunk rows (pass 1 -> pass 2)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) frc[ch] = -1;
                if (L < 32)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int q = ch * L + g;
                    const bool in = q < nslot;
                    const double v = in ? sm.sval[q] : 0.0;
                    const int32_t r = in ? sm.srow[q] : 0;
                    const bool keep = in && v != 0.0;  // sparse.hpp:105
                    frc[ch] = (keep && col_free) ? __ldg(p.fidx + r) : -1;
                    const bool keepf = frc[ch] >= 0;
                    na += __popc(__ballot_sync(FULL, keep) & gmask);
                    nf += __popc(__ballot_sync(FULL, keepf) & gmask);
                }
                // exclusive prefix over the groups of the warp (column order)
                int pa = na, pf = nf;
#pragma unroll
                for (int o = L; o < 32; o <<= 1) {
                    const int ya = __shfl_up_sync(FULL, pa, o);
                    const int yf = __shfl_up_sync(FULL, pf, o);
                    if (lane >= o) {
                        pa += ya;
                        pf += yf;
                    }
                }
                int tot_a = __shfl_sync(FULL, pa, 31), tot_f = __shfl_sync(FULL, pf, 31);
                int wa = run_a + pa - na, wf = run_f + pf - nf;  // this column's first slot
                if (L < 32 && act && g == 0) {
                    p.colcnt_a[lc] = wa + na;
                    if (p.want_sys) p.colcnt_f[lc] = wf + nf;
                }
                // pass 2: write
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int q = ch * L + g;
                    const bool in = q < nslot;
                    const double v = in ? sm.sval[q] : 0.0;
                    const int32_t r = in ? sm.srow[q] : 0;
                    const bool keep = in && v != 0.0;
                    const int32_t fr = L < 32 ? frc[ch] : ((keep && col_free) ? __ldg(p.fidx + r) : -1);
                    const bool keepf = fr >= 0;
                    const unsigned ba = __ballot_sync(FULL, keep) & gmask;
                    const unsigned bf = __ballot_sync(FULL, keepf) & gmask;
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
                if (L == 32) {
                    tot_a = wa - run_a;
                    tot_f = wf - run_f;
                    if (act && g == 0) {
                        p.colcnt_a[lc] = wa;
                        if (p.want_sys) p.colcnt_f[lc] = wf;
                    }
                }
                run_a += tot_a;
                run_f += tot_f;
                __syncwarp();
            }
            // ---- per-column vectors
            if (act && g == 0) {
                if (p.want_b) p.b[lc] = b;
                if (p.want_sys) {
                    const double u0 = dir_c ? node_field3(p.g_dir, p.nodes, D, c) : 0.0;
                    const double bmod = LIFT ? b - ylift : b - 0.0;  // system.hpp:197-198
                    p.u0[lc] = u0;
                    p.b_mod[lc] = bmod;
                    const int32_t fc = fc_c;
                    if (fc >= 0) p.b_f[fc - free_base(p)] = bmod;
                }
            }
        }
        if (lane == 0) {
            p.tile_tot[tile] = run_a;
            p.tile_tot[p.n_tiles + 1 + tile] = run_f;
        }
        if (__any_sync(FULL, bad) && lane == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
    }
}

// element-first records into the result's erec buffers (p.srec / p.lrec)
int launch_elem_records(fl_ctx* ctx, int dim, ColParams& p, fl_result* res) {
    const size_t ne = (size_t)std::max<int32_t>(p.n_elems, 1);
    const bool r64 = dim == 2 ? rec64<2>() : rec64<3>();
    FL_TRY(res->erec[0].ensure(sizeof(double) * (r64 ? 8 : 4) * (dim + 1) * ne));
    if (!r64) FL_TRY(res->erec[1].ensure(sizeof(double) * 4 * ne));
    p.srec = res->erec[0].as<double>();
    p.lrec = r64 ? nullptr : res->erec[1].as<double>();
    if (p.n_elems > 0) {
        const int g = std::min(div_up(p.n_elems, kElemThreads), ctx->sm_count * 16);
        if (dim == 3) k_elem_records<3><<<g, kElemThreads, 0, ctx->stream>>>(p);
        else k_elem_records<2><<<g, kElemThreads, 0, ctx->stream>>>(p);
        count_launch(ctx);
        FL_CUDA(cudaGetLastError());
    }
    return FL_OK;
}

template <int D, int L, bool PRE, bool LIFT, int K>
static int launch3(fl_ctx* ctx, ColParams& p, fl_result* res, bool finish) {
    using C = V3<D, L, K>;
    FL_TRY(prepare_staging(ctx, p, res, C::WTC, (int64_t)C::WTC * C::MAXS));
    if (ctx->profile) {
        FL_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
        ctx->kernel_timed = true;
    }
    if constexpr (PRE) FL_TRY(launch_elem_records(ctx, D, p, res));
    int per_sm = 1;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_columns3<D, L, PRE, LIFT, K>,
                                                          C::WARPS * 32, 0));
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((p.n_tiles + C::WARPS - 1) / C::WARPS,
                             (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[6], ctx->stream));
    k_columns3<D, L, PRE, LIFT, K><<<(int)grid, C::WARPS * 32, 0, ctx->stream>>>(p);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    if (ctx->profile) FL_CUDA(cudaEventRecord(ctx->ev[7], ctx->stream));
    return finish ? finish_staging(ctx, p, C::WTC) : FL_OK;
}

// kmax: the plan's largest node valence; the lift (nonzero Dirichlet data) is a template branch.
// pre: element-first records (default) or per-incidence geometry in the kernel.
// incidences per column the register kernel takes (3-D: two per lane above 32)
int columns3_lanes(int dim, int kmax) { return dim == 2 ? (kmax <= 8 ? 8 : 16) : (kmax <= 32 ? 32 : 64); }

template <int D, int L, int K>
static int launch3_sel(fl_ctx* ctx, ColParams& p, fl_result* res, bool pre, bool finish) {
    if constexpr (K == 1) {
        if (!pre) return launch3<D, L, false, false, 1>(ctx, p, res, finish);  // no lift (routed to v2)
    }
    return p.need_lift ? launch3<D, L, true, true, K>(ctx, p, res, finish)
                       : launch3<D, L, true, false, K>(ctx, p, res, finish);
}

int launch_columns3(fl_ctx* ctx, int dim, ColParams& p, int kmax, fl_result* res, bool pre, bool finish) {
    if (dim == 2) {
        if (kmax <= 8) return launch3_sel<2, 8, 1>(ctx, p, res, pre, finish);
        return launch3_sel<2, 16, 1>(ctx, p, res, pre, finish);
    }
    if (kmax > 32 && pre) return launch3_sel<3, 32, 2>(ctx, p, res, pre, finish);
    return launch3_sel<3, 32, 1>(ctx, p, res, pre, finish);
}

}  // namespace fl
