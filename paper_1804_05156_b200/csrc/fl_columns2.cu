// fl_columns2.cu -- the tiled column kernel (v2), the fast path of fl_assemble.
//
// One CTA assembles a tile of TC consecutive output columns (= reference CSC
// columns; the pattern is symmetric, so also CSR rows) in four phases:
//   1. the tile's incidence keys (j << 30 | t) -> smem, unsorted from the plan;
//   2. lane per incidence: rank of the key inside its column = the (j, t) order in
//      which the reference's blockwise triplets reach that column
//      (assembly.hpp:486-498 + the stable passes sparse.hpp:79-89); element
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
    static constexpr size_t MISC_OFF = (NF_OFF + sizeof(int32_t) * (TC + 1) + 15) & ~size_t(15);
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
        const int32_t c0 = (int32_t)(tile * TC);
        const int ncols = min(TC, p.n_nodes - c0);

        // ---- phase 1: the tile's incidence keys
        const int32_t base = __ldg(p.inc_ptr + c0);
        for (int q = tid; q <= TC; q += T::THREADS) ptr[q] = __ldg(p.inc_ptr + c0 + min(q, ncols)) - base;
        if (tid == 0) misc[3] = 0;
        __syncthreads();
        const int M = ptr[ncols];
        bool too_big = false;
        if (tid < ncols) too_big = ptr[tid + 1] - ptr[tid] > KMAX;
        if (__syncthreads_or(too_big)) {
            if (tid == 0) atomicOr(p.err, DERR_V2_OVERFLOW);
            if (tid < 32) warp_lookback(p.tile_status, tile, 0);  // keep the chain alive
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
        // ---- phase 3: folds, P threads per column
        const bool mine = col < ncols;
        const int32_t c = c0 + col;
        const int m = mine ? ptr[col + 1] - ptr[col] : 0;
        double b = 0.0, y = 0.0;
        int nown = 0;
        if (mine && p.want_a) {
            const int32_t* __restrict__ Rc = R + col;
            const double* __restrict__ Sc = S + col;
            int32_t* __restrict__ trow = tab_row + col;
            double* __restrict__ tacc = tab_acc + col;
#pragma unroll
            for (int h = 0; h < T::HSU; ++h) trow[h * TC] = -1;
            bool over = false;
            for (int i = 0; i < NV; ++i) {
                // software pipeline: the next item's row/value are loaded before
                // the current accumulator update
                int32_t r_nx = m > 0 ? Rc[i * TC] : 0;
                double s_nx = m > 0 ? Sc[i * TC] : 0.0;
                for (int k = 0; k < m; ++k) {
                    const int32_t r = r_nx;
                    const double sv = s_nx;
                    if (k + 1 < m) {
                        r_nx = Rc[(k + 1) * LY::SROW + i * TC];
                        s_nx = Sc[(k + 1) * LY::SROW + i * TC];
                    }
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
                            if (LIFT) tab_tacc[h * TC + col] = -0.0;
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
            if (LIFT && !over) {
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
        if (mine && u == 0) {
            if (p.want_b)
                for (int k = 0; k < m; ++k) b = b + Lb[k * LY::LROW + col];
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
        __syncthreads();  // folds done: the phase-2 buffers become the output lists
        // free ranks of every slot row, gathered by all threads at once (the
        // zero-drop loop below would otherwise wait on one gather per entry)
        if (p.want_sys && p.want_a)
            for (int e = tid; e < T::HSU * TC; e += T::THREADS) {
                const int32_t r = tab_row[e];
                if (r >= 0 && (e % TC) < ncols) tab_fidx[e] = __ldg(p.fidx + r);
            }
        __syncthreads();
        FL_MARK(2)

        // ---- phase 4a: slots -> rows in ascending order, drop exact zeros
        if (p.want_a) {
            if (mine && nown <= T::MAXS) {
                // extract the slots with an insertion sort by row
                int n = 0;
                for (int h = 0; h < T::HSU; ++h) {
                    const int32_t r = tab_row[h * TC + col];
                    if (r < 0) continue;
                    const double v = tab_acc[h * TC + col];
                    const double tv = LIFT ? tab_tacc[h * TC + col] : 0.0;
                    const int32_t fx = p.want_sys ? tab_fidx[h * TC + col] : -1;
                    int q = n++;
                    while (q > 0) {
                        const int32_t rp = o_row[(q - 1) * TC + col];
                        if (rp < r) break;
                        o_row[q * TC + col] = rp;
                        o_val[q * TC + col] = o_val[(q - 1) * TC + col];
                        f_row[q * TC + col] = f_row[(q - 1) * TC + col];
                        if (LIFT) o_tv[q * TC + col] = o_tv[(q - 1) * TC + col];
                        --q;
                    }
                    o_row[q * TC + col] = r;
                    o_val[q * TC + col] = v;
                    f_row[q * TC + col] = fx;  // free rank of the row (-1: Dirichlet)
                    if (LIFT) o_tv[q * TC + col] = tv;
                }
            }
            if (mine) {
                const int n = nown <= T::MAXS ? nown : 0;
                // Dirichlet lift: (A u0)[c] = sum over stored A(c, r), ascending r
                if (LIFT)
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
                    if (col_free) {
                        if (fr >= 0) {
                            f_row[kf * TC + col] = fr;
                            f_val[kf * TC + col] = v;
                            ++kf;
                        }
                    }
                }
                na[col] = ka;
                nf[col] = kf;
            }
        }
        for (int q = tid; q < TC; q += T::THREADS)
            if (q >= ncols || !p.want_a) na[q] = nf[q] = 0;
        __syncthreads();

        FL_MARK(3)
        // ---- phase 4b: tile prefix, look-back, coalesced writes
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
            }
            const uint64_t ex =
                warp_lookback(p.tile_status, tile, ((uint64_t)tf << 31) | (uint64_t)ta);
            if (tid == 0) {
                misc[1] = (int64_t)(ex & 0x7FFFFFFFull);
                misc[2] = (int64_t)(ex >> 31);
                if (misc[3]) atomicOr(p.err, DERR_V2_OVERFLOW);
            }
        }
        __syncthreads();
        FL_MARK(4)
        const int64_t off_a = misc[1], off_f = misc[2];
        const int ta = na[TC], tf = nf[TC];
        if (p.want_a) {
            if (off_a + ta > p.cap_a || (p.want_sys && off_f + tf > p.cap_ff)) {
                if (tid == 0) atomicOr(p.err, DERR_CAPACITY);
            } else {
                // a warp per column: each column's entries are one contiguous run
                constexpr int NW = T::THREADS / 32;
                const int lane = tid & 31, wid = tid >> 5;
                for (int cc = wid; cc < ncols; cc += NW) {
                    const int b0 = na[cc], n = na[cc + 1] - b0;
                    for (int q = lane; q < n; q += 32) {
                        p.row_idx[off_a + b0 + q] = o_row[q * TC + cc];
                        p.values[off_a + b0 + q] = o_val[q * TC + cc];
                    }
                    if (p.want_sys) {
                        const int f0 = nf[cc], nn = nf[cc + 1] - f0;
                        for (int q = lane; q < nn; q += 32) {
                            p.ff_row_idx[off_f + f0 + q] = f_row[q * TC + cc];
                            p.ff_values[off_f + f0 + q] = f_val[q * TC + cc];
                        }
                    }
                }
                if (mine && u == 0) p.col_ptr[c + 1] = (int32_t)(off_a + na[col + 1]);
            }
        }
        if (mine && u == 0) {
            if (p.want_b) p.b[c] = b;
            if (p.want_sys) {
                const double u0 = p.is_dir[c] ? node_field(p.g_dir, p.nodes, D, c) : 0.0;
                const double bmod = LIFT ? b - y : b - 0.0;
                p.u0[c] = u0;
                p.b_mod[c] = bmod;
                const int32_t fc = p.fidx[c];
                if (fc >= 0) {
                    p.b_f[fc] = bmod;
                    if (p.want_a) p.ff_col_ptr[fc + 1] = (int32_t)(off_f + nf[col + 1]);
                }
            }
        }
        __syncthreads();
        FL_MARK(5)
    }
}


template <int D, int TCX, int THR, int KMAX, bool LIFT>
static int launch_variant(fl_ctx* ctx, ColParams& p) {
    using T = Tile<D, TCX, THR>;
    using LY = Layout<T, D, KMAX, LIFT>;
    const size_t smem = LY::BYTES;
    auto kern = k_columns2<D, TCX, THR, KMAX, LIFT>;
    FL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    FL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THR, smem));
    p.n_tiles = (p.n_nodes + TCX - 1) / TCX;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>(p.n_tiles, (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    kern<<<(int)grid, THR, smem, ctx->stream>>>(p);
    count_launch(ctx);
    FL_CUDA(cudaGetLastError());
    return FL_OK;
}

template <int D, int TCX, int THR>
static int launch_shape(fl_ctx* ctx, ColParams& p, int kmax) {
    constexpr int K_SMALL = D == 2 ? 8 : 24, K_LARGE = D == 2 ? 16 : 32;
    if (kmax <= K_SMALL)
        return p.need_lift ? launch_variant<D, TCX, THR, K_SMALL, true>(ctx, p)
                           : launch_variant<D, TCX, THR, K_SMALL, false>(ctx, p);
    return p.need_lift ? launch_variant<D, TCX, THR, K_LARGE, true>(ctx, p)
                       : launch_variant<D, TCX, THR, K_LARGE, false>(ctx, p);
}

// kmax: the plan's largest node valence (incidences per node).  FL_TILE=<TC>x<THREADS>
// selects an alternative tile shape (tuning experiments).
int launch_columns2(fl_ctx* ctx, int dim, ColParams& p, int kmax) {
    const char* env = std::getenv("FL_TILE");
    const std::string shape = env ? env : "";
    if (dim == 2) {
        if (shape == "32x64") return launch_shape<2, 32, 64>(ctx, p, kmax);
        if (shape == "32x128") return launch_shape<2, 32, 128>(ctx, p, kmax);
        if (shape == "128x128") return launch_shape<2, 128, 128>(ctx, p, kmax);
        return launch_shape<2, 64, 128>(ctx, p, kmax);
    }
    if (shape == "16x64") return launch_shape<3, 16, 64>(ctx, p, kmax);
    if (shape == "16x128") return launch_shape<3, 16, 128>(ctx, p, kmax);
    if (shape == "32x64") return launch_shape<3, 32, 64>(ctx, p, kmax);
    return launch_shape<3, 32, 128>(ctx, p, kmax);
}

}  // namespace fl
