// fl_columns2.cu -- the tiled column kernel (v2), the fast path of fl_assemble.
//
// One CTA assembles a tile of TC consecutive output columns (= reference CSC
// columns; the pattern is symmetric, so also CSR rows) in four phases:
//   1. the tile's incidence keys (j << 30 | t) -> smem, unsorted from the plan;
//   2. lane per incidence: rank of the key inside its column = the (j, t) order in
//      which the reference's blockwise triplets reach that column
//      (assembly.hpp:286-298 + the stable passes sparse.hpp:79-89); element
//      geometry for column j (fl_geometry.cuh) -> s_ij (i = 0..d) and the load
//      share, stored at [rank][i][column] (column-interleaved: conflict-free);
//   3. P threads per column; thread u owns the distinct rows whose hash selects u
//      and sweeps the column's items in the reference order (i outer, ranked
//      incidence inner) folding only its own rows, so every entry (r, c) is the
//      sequential sum of sparse.hpp:98-104 in (i*(d+1)+j, t) order.  Thread 0 of
//      the column also folds b (0.0 + shares in (j, t) order, system.hpp:114-118)
//      and the Neumann data; optional transposed folds give A(c, r) for the
//      Dirichlet lift (matvec sparse.hpp:129-141);
//   4. merge the P slot lists, sort rows, drop exact zeros (sparse.hpp:105),
//      A(free, free) rows, CTA offsets by a warp-wide decoupled look-back,
//      coalesced copy of the tile's entries; b, u0, b_mod, b_f per column.
// A column with more than KMAX incidences or more distinct rows than the slot
// tables hold raises DERR_V2_OVERFLOW; the host then reruns the mesh on the
// general warp-per-column kernel (fl_kernels.cu k_columns).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"
#include "fl_kernels.cuh"
#include "fl_scan.cuh"

namespace fl {

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// Tile shape: TC columns per CTA of THREADS threads; per-column slot table of
// HSU entries holding at most MAXS distinct rows (load factor 0.75).
template <int D, int TC_, int THREADS_>
struct Tile {
    static constexpr int TC = TC_;
    static constexpr int THREADS = THREADS_;
    static constexpr int HSU = D == 2 ? 16 : 32;
    static constexpr int MAXU = D == 2 ? 12 : 24;
    static constexpr int MAXS = MAXU;
};

template <class T_, int D, int KMAX, bool LIFT>
struct Layout {
    using T = T_;
    static constexpr int NV = D + 1;
    static constexpr int TC = T::TC;
    static constexpr int P = 1;                   // fold threads per column
    static constexpr int SROW = NV * TC + 1;      // padded stride of one rank row
    static constexpr int LROW = TC + 1;
    // byte offsets of the dynamic smem carve-up
    static constexpr size_t S_OFF = 0;                                          // double [KMAX][SROW]
    static constexpr size_t R_OFF = S_OFF + sizeof(double) * KMAX * SROW;       // int32 [KMAX][SROW]
    static constexpr size_t L_OFF = (R_OFF + sizeof(int32_t) * KMAX * SROW + 7) & ~size_t(7);
    static constexpr size_t KS_OFF = L_OFF + sizeof(double) * KMAX * LROW;      // uint32 [KMAX][LROW]
    static constexpr size_t IN_END = KS_OFF + sizeof(uint32_t) * KMAX * LROW;
    // output lists alias the phase-2 buffers after the folds
    static constexpr size_t M_ROW = 0;                                          // int32 [MAXS][TC]
    static constexpr size_t M_VAL = M_ROW + sizeof(int32_t) * T::MAXS * TC;     // double
    static constexpr size_t M_TV = M_VAL + sizeof(double) * T::MAXS * TC;       // double
    static constexpr size_t F_ROW = M_TV + sizeof(double) * T::MAXS * TC;       // int32
    static constexpr size_t F_VAL = F_ROW + sizeof(int32_t) * T::MAXS * TC;     // double
    static constexpr size_t OUT_END = F_VAL + sizeof(double) * T::MAXS * TC;
    static constexpr size_t UNION_END = IN_END > OUT_END ? IN_END : OUT_END;
    static constexpr size_t KEY_OFF = (UNION_END + 15) & ~size_t(15);           // uint32 [TC*KMAX]
    static constexpr size_t TR_OFF = KEY_OFF + sizeof(uint32_t) * TC * KMAX;    // int32 [HSU][TC]
    static constexpr size_t TA_OFF = TR_OFF + sizeof(int32_t) * T::HSU * TC;    // double
    static constexpr size_t TT_OFF = TA_OFF + sizeof(double) * T::HSU * TC;     // double (LIFT)
    static constexpr size_t TAB_END = TT_OFF + (LIFT ? sizeof(double) * T::HSU * TC : 0);
    static constexpr size_t TF_OFF = TAB_END;                                    // int32 [HSU][TC]
    static constexpr size_t PTR_OFF = TF_OFF + sizeof(int32_t) * T::HSU * TC;   // int32 [TC+1]
    static constexpr size_t NA_OFF = PTR_OFF + sizeof(int32_t) * (TC + 1);      // int32 [TC+1]
    static constexpr size_t NF_OFF = NA_OFF + sizeof(int32_t) * (TC + 1);       // int32 [TC+1]
    // parallel fold (LIFT == false): per-item slot ids and ranks, per (pass, slot)
    // counts and offsets, per-column item lists, per-slot results
    static constexpr size_t SL_OFF = NF_OFF + sizeof(int32_t) * (TC + 1);       // u8 [KMAX][NV*TC]
    static constexpr size_t RK_OFF = SL_OFF + (size_t)KMAX * NV * TC;           // u8 [KMAX][NV*TC]
    static constexpr size_t CN_OFF = RK_OFF + (size_t)KMAX * NV * TC;           // u8 [NV][HSU][TC]
    static constexpr size_t PO_OFF = CN_OFF + (size_t)NV * T::HSU * TC;         // u8 [NV][HSU][TC]
    static constexpr size_t LS_OFF = PO_OFF + (size_t)NV * T::HSU * TC;         // u8 [KMAX*NV][TC]
    static constexpr size_t TK_OFF = LS_OFF + (size_t)KMAX * NV * TC;           // u8 [HSU][TC] rank
    static constexpr size_t TN_OFF = TK_OFF + (size_t)T::HSU * TC;              // u8 [HSU][TC] count
    static constexpr size_t DG_OFF = (TN_OFF + (size_t)T::HSU * TC + 7) & ~size_t(7);  // double [TC]
    static constexpr size_t NS_OFF = DG_OFF + sizeof(double) * TC;              // int32 [TC] slots
    static constexpr size_t MISC_OFF = (NS_OFF + sizeof(int32_t) * TC + 15) & ~size_t(15);
    static constexpr size_t BYTES = MISC_OFF + 64;
};

__device__ __forceinline__ double node_field(const FieldDesc& g, const double* nodes, int dim,
                                             int32_t k) {
    if (g.kind == FL_FIELD_SAMPLES) return __ldg(g.samples + k);
    if (g.kind == FL_FIELD_CONST) return g.value;
    const double x = nodes[(size_t)k * dim];
    const double y = nodes[(size_t)k * dim + 1];
    const double z = dim == 3 ? nodes[(size_t)k * dim + 2] : 0.0;
    return eval_point(g, x, y, z);
}

template <int D, int TCX, int THR, int KMAX, bool LIFT>
__global__ void __launch_bounds__(THR) k_columns2(ColParams p) {
    using T = Tile<D, TCX, THR>;
    using LY = Layout<T, D, KMAX, LIFT>;
    constexpr int NV = D + 1;
    constexpr int TC = T::TC;
    constexpr int P = LY::P;
    constexpr int LOGP = ilog2(P);
    constexpr int LOGH = ilog2(T::HSU);
    extern __shared__ __align__(16) unsigned char smem[];
    double* S = reinterpret_cast<double*>(smem + LY::S_OFF);
    int32_t* R = reinterpret_cast<int32_t*>(smem + LY::R_OFF);
    double* Lb = reinterpret_cast<double*>(smem + LY::L_OFF);
    uint32_t* KS = reinterpret_cast<uint32_t*>(smem + LY::KS_OFF);
    int32_t* o_row = reinterpret_cast<int32_t*>(smem + LY::M_ROW);
    double* o_val = reinterpret_cast<double*>(smem + LY::M_VAL);
    double* o_tv = reinterpret_cast<double*>(smem + LY::M_TV);
    int32_t* f_row = reinterpret_cast<int32_t*>(smem + LY::F_ROW);
    double* f_val = reinterpret_cast<double*>(smem + LY::F_VAL);
    uint32_t* key = reinterpret_cast<uint32_t*>(smem + LY::KEY_OFF);
    int32_t* tab_row = reinterpret_cast<int32_t*>(smem + LY::TR_OFF);
    double* tab_acc = reinterpret_cast<double*>(smem + LY::TA_OFF);
    double* tab_tacc = reinterpret_cast<double*>(smem + LY::TT_OFF);
    int32_t* tab_fidx = reinterpret_cast<int32_t*>(smem + LY::TF_OFF);
    int32_t* ptr = reinterpret_cast<int32_t*>(smem + LY::PTR_OFF);
    int32_t* na = reinterpret_cast<int32_t*>(smem + LY::NA_OFF);
    int32_t* nf = reinterpret_cast<int32_t*>(smem + LY::NF_OFF);
    int64_t* misc = reinterpret_cast<int64_t*>(smem + LY::MISC_OFF);  // tile, off_a, off_f, bad

    const int tid = threadIdx.x;
    const Recip R3 = recip(3.0);
    const Recip R6 = recip(6.0);
    // phase-3 identity: column `col`, owner slot `u`
    const int col = tid >> LOGP;
    const int u = tid & (P - 1);
    long long ph_t = 0, ph_acc[6] = {0, 0, 0, 0, 0, 0};
#define FL_MARK(k)                                              \
    if (p.phase_cycles && tid == 0) {                           \
        const long long now_ = clock64();                       \
        ph_acc[k] += now_ - ph_t;                               \
        ph_t = now_;                                            \
    }

    while (true) {
        if (tid == 0) misc[0] = atomicAdd(p.ticket, 1u);
        __syncthreads();
        const int64_t tile = misc[0];
        if (tile >= p.n_tiles) {
            if (p.phase_cycles && tid == 0)
                for (int q = 0; q < 6; ++q) atomicAdd(p.phase_cycles + q, (unsigned long long)ph_acc[q]);
            break;
        }
        if (p.phase_cycles && tid == 0) ph_t = clock64();
        const int32_t lc0 = (int32_t)(tile * TC);  // first owned column of the tile
        const int32_t c0 = p.c_begin + lc0;         // ... as a global node
        const int ncols = min(TC, p.n_cols - lc0);

        // ---- phase 1: the tile's incidence keys
        const int32_t base = __ldg(p.inc_ptr + lc0);
        for (int q = tid; q <= TC; q += T::THREADS) ptr[q] = __ldg(p.inc_ptr + lc0 + min(q, ncols)) - base;
        if (tid == 0) misc[3] = 0;
        __syncthreads();
        const int M = ptr[ncols];
        bool too_big = false;
        if (tid < ncols) too_big = ptr[tid + 1] - ptr[tid] > KMAX;
        if (__syncthreads_or(too_big)) {
            if (tid == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
            if (tid == 0) p.tile_tot[tile] = p.tile_tot[p.n_tiles + 1 + tile] = 0;
            __syncthreads();
            continue;
        }
        for (int q = tid; q < M; q += T::THREADS) key[q] = __ldg(p.inc + base + q);
        __syncthreads();

        FL_MARK(0)
        // ---- phase 2: rank + geometry, lane per incidence
        for (int q = tid; q < M; q += T::THREADS) {
            const uint32_t kq = key[q];
            int lo = 0, hi = ncols;  // column of q: ptr[lo] <= q < ptr[lo + 1]
#pragma unroll 1
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (ptr[mid] <= q) lo = mid;
                else hi = mid;
            }
            const int pb = ptr[lo], pe = ptr[lo + 1];
            int rank = 0;
            for (int r = pb; r < pe; ++r) rank += key[r] < kq;
            const int32_t t = (int32_t)(kq & 0x3FFFFFFFu);
            const int j = (int)(kq >> 30);
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
                S[rank * LY::SROW + i * TC + lo] = s[i];
                R[rank * LY::SROW + i * TC + lo] = V[i];
            }
            Lb[rank * LY::LROW + lo] = l;
            KS[rank * LY::LROW + lo] = kq;
        }
        __syncthreads();

        FL_MARK(1)
        // ---- phase 3: folds
        const bool mine = col < ncols;
        const int32_t c = c0 + col;
        const int m = mine ? ptr[col + 1] - ptr[col] : 0;
        double b = 0.0, y = 0.0;
        int nown = 0;
        if constexpr (LIFT) {
            // general path (Dirichlet lift): one thread per column, hashed slots
            if (mine && p.want_a) {
                const int32_t* __restrict__ Rc = R + col;
                const double* __restrict__ Sc = S + col;
                int32_t* __restrict__ trow = tab_row + col;
                double* __restrict__ tacc = tab_acc + col;
#pragma unroll
                for (int h = 0; h < T::HSU; ++h) trow[h * TC] = -1;
                bool over = false;
                for (int i = 0; i < NV; ++i) {
                    for (int k = 0; k < m; ++k) {
                        const int32_t r = Rc[k * LY::SROW + i * TC];
                        const double sv = Sc[k * LY::SROW + i * TC];
                        uint32_t h = ((uint32_t)r * 2654435761u) >> (32 - LOGH);
                        int slot = -1;
                        while (true) {
                            const int32_t kk = trow[h * TC];
                            if (kk == r) {
                                slot = (int)h;
                                break;
                            }
                            if (kk == -1) {
                                if (nown >= T::MAXU) break;
                                trow[h * TC] = r;
                                tacc[h * TC] = -0.0;  // -0.0 + x == x: the fold starts at its first value
                                tab_tacc[h * TC + col] = -0.0;
                                ++nown;
                                slot = (int)h;
                                break;
                            }
                            h = (h + 1) & (T::HSU - 1);
                        }
                        if (slot < 0) {
                            over = true;
                            continue;
                        }
                        tacc[slot * TC] = tacc[slot * TC] + sv;
                    }
                }
                if (over) misc[3] = 1;
                if (!over) {
                    // entry (c, r) in its own order (i_c*(d+1)+j_r, t): j-buckets of the
                    // ranked incidences (j = local index of c) outer, then i, then t
                    int k0 = 0;
                    while (k0 < m) {
                        const uint32_t jb = KS[k0 * LY::LROW + col] >> 30;
                        int k1 = k0;
                        while (k1 < m && (KS[k1 * LY::LROW + col] >> 30) == jb) ++k1;
                        for (int i = 0; i < NV; ++i)
                            for (int k = k0; k < k1; ++k) {
                                const int32_t r = R[k * LY::SROW + i * TC + col];
                                uint32_t h = ((uint32_t)r * 2654435761u) >> (32 - LOGH);
                                while (tab_row[h * TC + col] != r) h = (h + 1) & (T::HSU - 1);
                                double& a = tab_tacc[h * TC + col];
                                a = a + S[k * LY::SROW + i * TC + col];
                            }
                        k0 = k1;
                    }
                }
            }
        }
        if (mine && u == 0) {
            // b = 0.0 + load shares in (j, t) order; the diagonal entry (c, c) is the
            // fold of s_{j_k j_k} in the same (j, t) order (its items all have i = j)
            double dg = -0.0;
            for (int k = 0; k < m; ++k) {
                if (p.want_b) b = b + Lb[k * LY::LROW + col];
                if (!LIFT && p.want_a) {
                    const int jk = (int)(KS[k * LY::LROW + col] >> 30);
                    dg = dg + S[k * LY::SROW + jk * TC + col];
                }
            }
            if (!LIFT && p.want_a) reinterpret_cast<double*>(smem + LY::DG_OFF)[col] = dg;
            // Neumann data (system.hpp:123-172) at nodes on flag-2 faces: face-major
            // (lf, t) order, accumulated from 0.0, then b += add
            if (p.want_b && p.has_neumann && p.g_neu.kind != FL_FIELD_NONE && p.is_neu[c]) {
                double add = 0.0;
                for (int lf = 0; lf < NV; ++lf) {
                    int32_t last = -1;
                    while (true) {
                        int32_t best = INT_MAX;
                        int kb = -1;
                        for (int k = 0; k < m; ++k) {
                            const uint32_t kq = KS[k * LY::LROW + col];
                            const int32_t t = (int32_t)(kq & 0x3FFFFFFFu);
                            if ((int)(kq >> 30) == lf || t <= last || t >= best) continue;
                            if (p.flags[(size_t)t * NV + lf] != 2) continue;
                            best = t;
                            kb = k;
                        }
                        if (kb < 0) break;
                        last = best;
                        int32_t V[NV];
#pragma unroll
                        for (int i = 0; i < NV; ++i) V[i] = R[kb * LY::SROW + i * TC + col];
                        ElemCol<D> ec;
                        ec.load(p.nodes, V);
                        add = add + ec.face_share(lf, p.g_neu, R3, best);
                    }
                }
                b = b + add;
            }
        }
        if constexpr (LIFT) {
            __syncthreads();  // folds done: the phase-2 buffers become the output lists
            if (p.want_sys && p.want_a)
                for (int e = tid; e < T::HSU * TC; e += T::THREADS) {
                    const int32_t r = tab_row[e];
                    if (r >= 0 && (e % TC) < ncols) tab_fidx[e] = __ldg(p.fidx + r);
                }
            __syncthreads();
            FL_MARK(2)
            if (p.want_a) {
                if (mine && nown <= T::MAXS) {
                    // extract the slots with an insertion sort by row
                    int n = 0;
                    for (int h = 0; h < T::HSU; ++h) {
                        const int32_t r = tab_row[h * TC + col];
                        if (r < 0) continue;
                        const double v = tab_acc[h * TC + col];
                        const double tv = tab_tacc[h * TC + col];
                        const int32_t fx = p.want_sys ? tab_fidx[h * TC + col] : -1;
                        int q = n++;
                        while (q > 0) {
                            const int32_t rp = o_row[(q - 1) * TC + col];
                            if (rp < r) break;
                            o_row[q * TC + col] = rp;
                            o_val[q * TC + col] = o_val[(q - 1) * TC + col];
                            f_row[q * TC + col] = f_row[(q - 1) * TC + col];
                            o_tv[q * TC + col] = o_tv[(q - 1) * TC + col];
                            --q;
                        }
                        o_row[q * TC + col] = r;
                        o_val[q * TC + col] = v;
                        f_row[q * TC + col] = fx;  // free rank of the row (-1: Dirichlet)
                        o_tv[q * TC + col] = tv;
                    }
                }
                if (mine) {
                    const int n = nown <= T::MAXS ? nown : 0;
                    // Dirichlet lift: (A u0)[c] = sum over stored A(c, r), ascending r
                    for (int q = 0; q < n; ++q) {
                        const int32_t r = o_row[q * TC + col];
                        const double a_cr = o_tv[q * TC + col];
                        if (a_cr != 0.0 && f_row[q * TC + col] < 0) {
                            const double uu = node_field(p.g_dir, p.nodes, D, r);
                            if (uu != 0.0) y = y + a_cr * uu;
                        }
                    }
                    const bool col_free = p.want_sys && p.fidx[c] >= 0;
                    int ka = 0, kf = 0;
                    for (int q = 0; q < n; ++q) {
                        const int32_t r = o_row[q * TC + col];
                        const double v = o_val[q * TC + col];
                        const int32_t fr = f_row[q * TC + col];
                        if (v == 0.0) continue;  // sparse.hpp:105
                        o_row[ka * TC + col] = r;
                        o_val[ka * TC + col] = v;
                        ++ka;
                        if (col_free && fr >= 0) {
                            f_row[kf * TC + col] = fr;
                            f_val[kf * TC + col] = v;
                            ++kf;
                        }
                    }
                    na[col] = ka;
                    nf[col] = kf;
                }
            }
        } else if (p.want_a) {
            // parallel path: every thread works on every step
            uint8_t* SLb = smem + LY::SL_OFF;  // slot of item (k, i, col)
            uint8_t* RKb = smem + LY::RK_OFF;  // rank of the item inside its (pass, slot)
            uint8_t* CNb = smem + LY::CN_OFF;  // items per (pass, slot)
            uint8_t* POb = smem + LY::PO_OFF;  // list offset of (pass, slot)
            uint8_t* LSb = smem + LY::LS_OFF;  // per-column item list, codes k*NV + i
            uint8_t* TKb = smem + LY::TK_OFF;  // sorted position of a slot's row
            uint8_t* TNb = smem + LY::TN_OFF;  // items of a slot
            const double* DG = reinterpret_cast<const double*>(smem + LY::DG_OFF);
            int32_t* NS = reinterpret_cast<int32_t*>(smem + LY::NS_OFF);
            constexpr int IS = NV * TC;  // item-row stride of SL/RK
            constexpr int HT = T::HSU * TC;
            constexpr int G = T::HSU;     // lanes per column group (16 or 32)
            constexpr int GPW = 32 / G;   // column groups per warp
            constexpr int NW = T::THREADS / 32;
            const int lane = tid & 31, wid = tid >> 5, gl = lane % G, gi = lane / G;
            for (int e = tid; e < HT; e += T::THREADS) tab_row[e] = -1;
            __syncthreads();
            // F1: slot of every item -- shared hash insert, CAS only for new rows
            bool over = false;
            for (int pos = tid; pos < KMAX * TC; pos += T::THREADS) {
                const int k = pos / TC, cc = pos - k * TC;
                if (cc >= ncols || k >= ptr[cc + 1] - ptr[cc]) continue;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int32_t r = R[k * LY::SROW + i * TC + cc];
                    uint32_t h = ((uint32_t)r * 2654435761u) >> (32 - LOGH);
                    int probes = 0;
                    while (true) {
                        const int32_t v = tab_row[h * TC + cc];
                        if (v == r) break;
                        if (v == -1) {
                            const int32_t old = atomicCAS(&tab_row[h * TC + cc], -1, r);
                            if (old == -1 || old == r) break;
                        }
                        h = (h + 1) & (T::HSU - 1);
                        if (++probes > T::HSU) {
                            over = true;
                            break;
                        }
                    }
                    SLb[k * IS + i * TC + cc] = (uint8_t)h;
                }
            }
            if (over) misc[3] = 1;
            __syncthreads();
            // F2: per (pass, column): stable rank of each item among its slot's items
            for (int task = tid; task < IS; task += T::THREADS) {
                const int i = task / TC, cc = task - i * TC;
                if (cc >= ncols) continue;
                uint8_t* cn = CNb + i * HT + cc;
#pragma unroll
                for (int h = 0; h < T::HSU; ++h) cn[h * TC] = 0;
                const int m2 = ptr[cc + 1] - ptr[cc];
                for (int k = 0; k < m2; ++k) {
                    const int s = SLb[k * IS + i * TC + cc];
                    const uint8_t x = cn[s * TC];
                    RKb[k * IS + i * TC + cc] = x;
                    cn[s * TC] = x + 1;
                }
            }
            __syncthreads();
            // F3: per column (G lanes = G table entries): item counts, list offsets,
            // sorted position of each row
            for (int cc = wid * GPW + gi; cc < TC; cc += NW * GPW) {
                const bool act = cc < ncols;
                const int32_t r = act ? tab_row[gl * TC + cc] : -1;
                const bool valid = r >= 0;
                int ni[NV], nh = 0;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    ni[i] = valid ? CNb[i * HT + gl * TC + cc] : 0;
                    nh += ni[i];
                }
                int incl = nh;
#pragma unroll
                for (int o = 1; o < G; o <<= 1) {
                    const int yv = __shfl_up_sync(0xffffffffu, incl, o, G);
                    if (gl >= o) incl += yv;
                }
                int run = incl - nh;
                int rank = 0;
#pragma unroll 8
                for (int q = 0; q < G; ++q) {
                    const int32_t rq = __shfl_sync(0xffffffffu, r, q, G);
                    rank += (rq >= 0) & (rq < r);
                }
                const unsigned bv = __ballot_sync(0xffffffffu, valid);
                const int nvalid = __popc(G == 32 ? bv : (bv >> (gi * G)) & ((1u << G) - 1));
                if (valid) {
#pragma unroll
                    for (int i = 0; i < NV; ++i) {
                        POb[i * HT + gl * TC + cc] = (uint8_t)run;
                        run += ni[i];
                    }
                    TKb[gl * TC + cc] = (uint8_t)rank;
                    TNb[gl * TC + cc] = (uint8_t)nh;
                }
                if (gl == 0 && act) {
                    NS[cc] = nvalid;
                    if (nvalid > T::MAXS) misc[3] = 1;
                }
            }
            __syncthreads();
            // F4: item codes into each column's list, ordered by (slot, pass, k)
            for (int task = tid; task < IS; task += T::THREADS) {
                const int i = task / TC, cc = task - i * TC;
                if (cc >= ncols) continue;
                const int m2 = ptr[cc + 1] - ptr[cc];
                for (int k = 0; k < m2; ++k) {
                    const int s = SLb[k * IS + i * TC + cc];
                    const int pos = POb[i * HT + s * TC + cc] + RKb[k * IS + i * TC + cc];
                    LSb[pos * TC + cc] = (uint8_t)(k * NV + i);
                }
            }
            __syncthreads();
            // F5: each off-diagonal entry = sequential fold of its list, i.e. in the
            // reference order (i*(d+1)+j, t); the diagonal comes from the column thread
            for (int e = tid; e < HT; e += T::THREADS) {
                const int h = e / TC, cc = e - h * TC;
                const int32_t r = tab_row[e];
                if (r < 0 || cc >= ncols) continue;
                double acc;
                if (r == c0 + cc) {
                    acc = DG[cc];
                } else {
                    const int base = POb[h * TC + cc];
                    const int n = TNb[e];
                    acc = -0.0;
                    for (int q = 0; q < n; ++q) {
                        const int code = LSb[(base + q) * TC + cc];
                        const int kk = code / NV, ii = code - kk * NV;
                        acc = acc + S[kk * LY::SROW + ii * TC + cc];
                    }
                }
                tab_acc[e] = acc;
                if (p.want_sys) tab_fidx[e] = __ldg(p.fidx + r);
            }
            __syncthreads();  // S is dead: the output lists may overwrite it
            FL_MARK(2)
            // F6: rows in ascending order, exact zeros dropped, A(free, free) rows
            for (int cc = wid * GPW + gi; cc < TC; cc += NW * GPW) {
                const bool act = cc < ncols;
                const int32_t r = act ? tab_row[gl * TC + cc] : -1;
                if (r >= 0) {
                    const int q = TKb[gl * TC + cc];
                    o_row[q * TC + cc] = r;
                    o_val[q * TC + cc] = tab_acc[gl * TC + cc];
                    f_row[q * TC + cc] = p.want_sys ? tab_fidx[gl * TC + cc] : -1;
                }
                __syncwarp();
                const int n = act ? NS[cc] : 0;
                const bool in = gl < n && n <= T::MAXS;
                const int32_t rr = in ? o_row[gl * TC + cc] : 0;
                const double vv = in ? o_val[gl * TC + cc] : 0.0;
                const int32_t ff = in ? f_row[gl * TC + cc] : -1;
                const bool col_free = act && p.want_sys && __ldg(p.fidx + c0 + cc) >= 0;
                const bool keep = in && vv != 0.0;  // sparse.hpp:105
                const bool keep_f = keep && col_free && ff >= 0;
                const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1) << (gi * G));
                const unsigned ba = __ballot_sync(0xffffffffu, keep) & gmask;
                const unsigned bf = __ballot_sync(0xffffffffu, keep_f) & gmask;
                const unsigned lower = (1u << lane) - 1;
                __syncwarp();
                if (keep) {
                    const int pa = __popc(ba & lower);
                    o_row[pa * TC + cc] = rr;
                    o_val[pa * TC + cc] = vv;
                }
                if (keep_f) {
                    const int pf = __popc(bf & lower);
                    f_row[pf * TC + cc] = ff;
                    f_val[pf * TC + cc] = vv;
                }
                if (gl == 0 && act) {
                    na[cc] = __popc(ba);
                    nf[cc] = __popc(bf);
                }
                __syncwarp();
            }
        }
        for (int q = tid; q < TC; q += T::THREADS)
            if (q >= ncols || !p.want_a) na[q] = nf[q] = 0;
        __syncthreads();

        FL_MARK(3)
        // ---- phase 4b: in-tile prefix, staged writes (offsets resolved later by
        //      a scan over tile totals and k_stage_copy: no waiting on other tiles)
        if (tid < 32) {
            constexpr int PER = (TC + 31) / 32;  // columns per lane
            int va[PER], vf[PER], sa = 0, sf = 0;
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int q = tid * PER + e;
                va[e] = q < TC ? na[q] : 0;
                vf[e] = q < TC ? nf[q] : 0;
                sa += va[e];
                sf += vf[e];
            }
            int ia = sa, iff = sf;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ya = __shfl_up_sync(0xffffffffu, ia, o);
                const int yf = __shfl_up_sync(0xffffffffu, iff, o);
                if (tid >= o) {
                    ia += ya;
                    iff += yf;
                }
            }
            const int ta = __shfl_sync(0xffffffffu, ia, 31);
            const int tf = __shfl_sync(0xffffffffu, iff, 31);
            int ea = ia - sa, ef = iff - sf;
            __syncwarp();
#pragma unroll
            for (int e = 0; e < PER; ++e) {
                const int q = tid * PER + e;
                if (q < TC) {
                    na[q] = ea;
                    nf[q] = ef;
                }
                ea += va[e];
                ef += vf[e];
            }
            if (tid == 0) {
                na[TC] = ta;
                nf[TC] = tf;
                p.tile_tot[tile] = ta;
                p.tile_tot[p.n_tiles + 1 + tile] = tf;
                if (misc[3]) atomicOr(p.err, DERR_V2_OVERFLOW);
            }
        }
        __syncthreads();
        FL_MARK(4)
        if (p.want_a) {
            const int64_t sbase = tile * p.tile_cap;
            // a warp per column: each column's entries are one contiguous run
            constexpr int NW = T::THREADS / 32;
            const int lane = tid & 31, wid = tid >> 5;
            for (int cc = wid; cc < ncols; cc += NW) {
                const int b0 = na[cc], n = na[cc + 1] - b0;
                for (int q = lane; q < n; q += 32) {
                    p.st_a_row[sbase + b0 + q] = o_row[q * TC + cc];
                    p.st_a_val[sbase + b0 + q] = o_val[q * TC + cc];
                }
                if (p.want_sys) {
                    const int f0 = nf[cc], nn = nf[cc + 1] - f0;
                    for (int q = lane; q < nn; q += 32) {
                        p.st_f_row[sbase + f0 + q] = f_row[q * TC + cc];
                        p.st_f_val[sbase + f0 + q] = f_val[q * TC + cc];
                    }
                }
            }
            if (mine && u == 0) {
                p.colcnt_a[lc0 + col] = na[col + 1];
                if (p.want_sys) p.colcnt_f[lc0 + col] = nf[col + 1];
            }
        }
        if (mine && u == 0) {
            const int32_t lc = lc0 + col;
            if (p.want_b) p.b[lc] = b;
            if (p.want_sys) {
                const double u0 = p.is_dir[c] ? node_field(p.g_dir, p.nodes, D, c) : 0.0;
                const double bmod = LIFT ? b - y : b - 0.0;
                p.u0[lc] = u0;
                p.b_mod[lc] = bmod;
                const int32_t fc = p.fidx[c];
                if (fc >= 0) p.b_f[fc - free_base(p)] = bmod;
            }
        }
        __syncthreads();
        FL_MARK(5)
    }
}

// Places the staged tiles: tile t's A entries go to [tile_off_a[t], +tot), and
// col_ptr[c+1] = tile_off + the in-tile inclusive count (same for A(free,free),
// whose columns are the free columns in ascending order).
__global__ void k_stage_copy(ColParams p, int tc) {
    // a warp places kGroup consecutive tiles: their destinations are one
    // contiguous run, so every store instruction writes 32 consecutive entries
    constexpr int kGroup = 4;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t ngroups = (p.n_tiles + kGroup - 1) / kGroup;
    for (int64_t gidx = warp; gidx < ngroups; gidx += nwarps) {
        const int64_t t0 = gidx * kGroup;
        const int nt = (int)min((int64_t)kGroup, p.n_tiles - t0);
#pragma unroll
        for (int f = 0; f < 2; ++f) {  // 0: A, 1: A(free, free)
            if (f == 1 && !p.want_sys) break;
            const int32_t* off = p.tile_off + (f ? p.n_tiles + 1 : 0);
            const int32_t* tot = p.tile_tot + (f ? p.n_tiles + 1 : 0);
            const int32_t* srow = f ? p.st_f_row : p.st_a_row;
            const double* sval = f ? p.st_f_val : p.st_a_val;
            int32_t* drow = f ? p.ff_row_idx : p.row_idx;
            double* dval = f ? p.ff_values : p.values;
            const int64_t cap = f ? p.cap_ff : p.cap_a;
            const int32_t my_off = lane < nt ? off[t0 + lane] : 0;
            const int32_t my_tot = lane < nt ? tot[t0 + lane] : 0;
            const int32_t base = __shfl_sync(0xffffffffu, my_off, 0);
            const int32_t end = __shfl_sync(0xffffffffu, my_off + my_tot, nt - 1);
            if ((int64_t)end > cap) {
                if (lane == 0) atomicOr(p.err, DERR_CAPACITY);
                continue;
            }
            int32_t rel[kGroup];
#pragma unroll
            for (int k = 0; k < kGroup; ++k) rel[k] = __shfl_sync(0xffffffffu, my_off, k) - base;
            // eight strides per round, all loads issued before the stores (B200, C5
            // placement: 1.51 / 1.35 / 1.12 / 1.49 ms at 1 / 4 / 8 / 16 strides)
            constexpr int R = 8;
            const int32_t n = end - base;
            for (int32_t q0 = 0; q0 < n; q0 += 32 * R) {
                int32_t rw[R];
                double vv[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t q = q0 + r * 32 + lane;
                    if (q < n) {
                        int k = 0;
#pragma unroll
                        for (int kk = 1; kk < kGroup; ++kk)
                            if (kk < nt && q >= rel[kk]) k = kk;
                        const int64_t src = (t0 + k) * p.tile_cap + (q - rel[k]);
                        rw[r] = __ldcs(srow + src);
                        vv[r] = __ldcs(sval + src);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t q = q0 + r * 32 + lane;
                    if (q < n) {
                        drow[base + q] = rw[r];
                        dval[base + q] = vv[r];
                    }
                }
            }
        }
        // col_ptr (and A(free,free) col_ptr): in-tile inclusive counts + tile offsets
        const int32_t fb = free_base(p);
        for (int q = lane; q < nt * tc; q += 32) {
            const int k = q / tc;
            const int32_t c = (int32_t)((t0 + k) * tc + (q - k * tc));
            if (c >= p.n_cols) continue;
            p.col_ptr[c + 1] = p.tile_off[t0 + k] + p.colcnt_a[c];
            if (p.want_sys) {
                const int32_t fc = p.fidx[p.c_begin + c];
                if (fc >= 0) p.ff_col_ptr[fc - fb + 1] = p.tile_off[p.n_tiles + 1 + t0 + k] + p.colcnt_f[c];
            }
        }
    }
}

template <int D, int TCX, int THR, int KMAX, bool LIFT>
static int launch_variant(fl_ctx* ctx, ColParams& p, fl_result* res) {
    using T = Tile<D, TCX, THR>;
    using LY = Layout<T, D, KMAX, LIFT>;
    const size_t smem = LY::BYTES;
    auto kern = k_columns2<D, TCX, THR, KMAX, LIFT>;
    const cudaStream_t s = ctx->stream;
    FL_TRY(prepare_staging(ctx, p, res, TCX, (int64_t)TCX * T::MAXS));
    FL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THR, smem));
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>(p.n_tiles, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    kern<<<(int)grid, THR, smem, s>>>(p);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return finish_staging(ctx, p, TCX);
}

// staging buffers for a tiled launch with `tc` columns and `cap` entries per tile
int prepare_staging(fl_ctx* ctx, ColParams& p, fl_result* res, int tc, int64_t cap) {
    (void)ctx;
    p.n_tiles = (p.n_cols + tc - 1) / tc;
    p.tile_cap = cap;
    const size_t nst = (size_t)p.n_tiles * (size_t)p.tile_cap;
    FL_TRY(res->stage[0].ensure(sizeof(int32_t) * nst));
    FL_TRY(res->stage[1].ensure(sizeof(double) * nst));
    if (p.want_sys) {
        FL_TRY(res->stage[2].ensure(sizeof(int32_t) * nst));
        FL_TRY(res->stage[3].ensure(sizeof(double) * nst));
    }
    FL_TRY(res->tile_tot.ensure(sizeof(int32_t) * 2 * ((size_t)p.n_tiles + 1)));
    FL_TRY(res->tile_off.ensure(sizeof(int32_t) * 2 * ((size_t)p.n_tiles + 1)));
    FL_TRY(res->colcnt.ensure(sizeof(int32_t) * 2 * ((size_t)p.n_cols + 1)));
    p.st_a_row = res->stage[0].as<int32_t>();
    p.st_a_val = res->stage[1].as<double>();
    p.st_f_row = res->stage[2].as<int32_t>();
    p.st_f_val = res->stage[3].as<double>();
    p.tile_tot = res->tile_tot.as<int32_t>();
    p.tile_off = res->tile_off.as<int32_t>();
    p.colcnt_a = res->colcnt.as<int32_t>();
    p.colcnt_f = res->colcnt.as<int32_t>() + p.n_cols + 1;
    return FL_OK;
}

// tile offsets (exclusive scans of the tile totals) and the placement copy
int finish_staging(fl_ctx* ctx, ColParams& p, int tc) {
    const cudaStream_t s = ctx->stream;
    if (!p.want_a) return FL_OK;
    FL_TRY(ctx->scan_ws.ensure(scan_ws_bytes(p.n_tiles)));
    const int32_t* ta = p.tile_tot;
    FL_CUDA(launch_scan<int32_t>(
        p.n_tiles, [ta] __device__(int64_t i) { return (int64_t)ta[i]; }, p.tile_off,
        ctx->scan_ws.p, s));
    count_launch(ctx);
    if (p.want_sys) {
        const int32_t* tf = p.tile_tot + p.n_tiles + 1;
        FL_CUDA(launch_scan<int32_t>(
            p.n_tiles, [tf] __device__(int64_t i) { return (int64_t)tf[i]; },
            p.tile_off + p.n_tiles + 1, ctx->scan_ws.p, s));
        count_launch(ctx);
    }
    const int64_t warps = std::min<int64_t>((p.n_tiles + 3) / 4, (int64_t)ctx->sm_count * 64);
    k_stage_copy<<<(int)((warps * 32 + 255) / 256), 256, 0, s>>>(p, tc);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

template <int D, int TCX, int THR>
static int launch_shape(fl_ctx* ctx, ColParams& p, int kmax, fl_result* res) {
    constexpr int K_SMALL = D == 2 ? 8 : 24, K_LARGE = D == 2 ? 16 : 32;
    if (kmax <= K_SMALL)
        return p.need_lift ? launch_variant<D, TCX, THR, K_SMALL, true>(ctx, p, res)
                           : launch_variant<D, TCX, THR, K_SMALL, false>(ctx, p, res);
    return p.need_lift ? launch_variant<D, TCX, THR, K_LARGE, true>(ctx, p, res)
                       : launch_variant<D, TCX, THR, K_LARGE, false>(ctx, p, res);
}

// kmax: the plan's largest node valence (incidences per node).  FL_TILE=<TC>x<THREADS>
// selects an alternative tile shape (tuning experiments).
int launch_columns2(fl_ctx* ctx, int dim, ColParams& p, int kmax, fl_result* res) {
    const char* env = std::getenv("FL_TILE");
    const std::string shape = env ? env : "";
    if (dim == 2) {
        if (shape == "32x64") return launch_shape<2, 32, 64>(ctx, p, kmax, res);
        if (shape == "16x64") return launch_shape<2, 16, 64>(ctx, p, kmax, res);
        if (shape == "32x128") return launch_shape<2, 32, 128>(ctx, p, kmax, res);
        if (shape == "128x128") return launch_shape<2, 128, 128>(ctx, p, kmax, res);
        return launch_shape<2, 64, 128>(ctx, p, kmax, res);
    }
    if (shape == "8x64") return launch_shape<3, 8, 64>(ctx, p, kmax, res);
    if (shape == "8x32") return launch_shape<3, 8, 32>(ctx, p, kmax, res);
    if (shape == "16x64") return launch_shape<3, 16, 64>(ctx, p, kmax, res);
    if (shape == "16x128") return launch_shape<3, 16, 128>(ctx, p, kmax, res);
    if (shape == "32x64") return launch_shape<3, 32, 64>(ctx, p, kmax, res);
    return launch_shape<3, 32, 128>(ctx, p, kmax, res);
}

}  // namespace fl
