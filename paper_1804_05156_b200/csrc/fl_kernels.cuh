// fl_kernels.cuh -- kernel parameter blocks and host launchers.
#pragma once

#include <cstdint>

#include "fl_geometry.cuh"
#include "fl_internal.cuh"

namespace fl {

// Element records.  2-D: 64 bytes per (element, local vertex j) -- {s_0j, s_1j,
// s_2j, load_j} then {load_j, ids v0|v1, ids v2|0, 0} -- so a column reads one
// aligned 64-byte block per incidence (C3 column pass 6.8 -> 5.6 ms).  3-D: the
// 32-byte row {s_0j..s_3j}, the load shares and the element's vertex ids stay
// separate: the 64-byte form cost more in the record writes than it saved in the
// column reads on C4 / C5 (measured).
template <int D>
__host__ __device__ constexpr bool rec64() { return D == 2; }

struct ColParams {
    int32_t n_nodes, n_elems;
    // owned columns [c_begin, c_begin + n_cols).  Column-indexed inputs (is_dir,
    // fidx, node fields) use the global column c; the plan (inc_ptr) and the
    // column outputs (col_ptr, b, u0, b_mod, colcnt_*) use lc = c - c_begin, and
    // A(free, free) columns / b_f use fidx[c] - *f_begin (free nodes below c_begin).
    int32_t c_begin, n_cols;
    const int32_t* f_begin;  // device scalar, nullptr = 0
    int64_t n_tiles;
    const double* nodes;
    const int32_t* elems;
    const int8_t* flags;
    const int32_t* inc_ptr;
    const uint32_t* inc;
    FieldDesc f, coef, g_dir, g_neu;
    bool want_a, want_b, want_sys, need_lift, has_neumann;
    const int8_t* is_dir;
    const int8_t* is_neu;
    const int32_t* fidx;
    int32_t* col_ptr;
    int32_t* row_idx;
    double* values;
    double* b;
    double* u0;
    double* b_mod;
    int32_t* ff_col_ptr;
    int32_t* ff_row_idx;
    double* ff_values;
    double* b_f;
    uint64_t* tile_status;
    unsigned int* ticket;
    uint32_t* err;
    int64_t cap_a, cap_ff;
    unsigned long long* phase_cycles;  // diagnostics: per-phase SM cycles (nullptr = off)
    // tiled kernel staging (no in-kernel look-back): tile t writes its compacted
    // entries at [t * tile_cap, ...) and its totals; k_stage_copy places them
    int64_t tile_cap;
    int32_t* st_a_row;
    double* st_a_val;
    int32_t* st_f_row;
    double* st_f_val;
    int32_t* tile_tot;   // [2][n_tiles + 1]: A totals, then A(free,free) totals
    int32_t* tile_off;   // [2][n_tiles + 1]: exclusive scans of tile_tot
    int32_t* colcnt_a;   // [N] in-tile inclusive count after column c
    int32_t* colcnt_f;   // [N] same for A(free, free) (indexed by column c)
    // element-first records (k_elem_records): srec row (t, j) at 4(t(d+1) + j) =
    // {s_0j, s_1j, s_2j, s_3j} (3-D) / {s_0j, s_1j, s_2j, load_j} (2-D); lrec
    // [t][j] = load share (3-D)
    double* srec;
    double* lrec;
    const uint8_t* emark;  // sharded: records only for elements touching owned columns
    // hybrid pass (columns above the fast kernels' valence): the register kernel
    // leaves them empty (hybrid); the general kernel then runs on col_list only,
    // writing its entries to overflow staging and per-listed-column counts /
    // offsets into ov_cnt / ov_off ([2][n_list]: A, A(free,free))
    bool hybrid;
    const int32_t* col_list;
    int32_t n_list;
    int32_t* ov_cnt;
    int32_t* ov_off;
    unsigned long long* ov_alloc;  // [2] running A / A(free,free) overflow-staging tops
    const double* nadd;  // Neumann shares per owned column (k_neumann_add), nullptr = none
    bool keys_sorted;    // the plan's segments are already in (j, t) order: no in-kernel sort
    // label-space pipeline (v4, fl_columns4.cu): columns are labels; inc holds the
    // label plan's keys; lel = elements with vertex labels (4 per row); xl[label] =
    // the node's coordinates and {node id, free rank or -1} in .w; vst[node] =
    // {b, u0, b - A u0, entry counts}; staging there: st_a_row = the columns' first
    // kStageFirst 16-byte entries at the node id, st_a_val = their overflow runs,
    // tile_cap = entries per column
    const int32_t* lel;
    Recip r3, r6;         // recip(3.0), recip(6.0) computed once per context (kernel parameters
                          // are constant-bank operands: no registers held across the column loop)
    const int32_t* lab;   // node id -> label
    const int32_t* lcnt;  // incidences per label; label l's keys at inc[l * lcap ..]
    int32_t lcap;
    const double4* xl;
    double4* vst;
};

__device__ __forceinline__ int32_t free_base(const ColParams& p) {
    return p.f_begin ? __ldg(p.f_begin) : 0;
}

int launch_plan_kernels(fl_ctx* ctx, fl_mesh* mesh, uint32_t* d_err);
int launch_validate(fl_ctx* ctx, fl_mesh* mesh, uint32_t* d_err);
int launch_partition(fl_ctx* ctx, fl_mesh* mesh, fl_result* res);
int launch_columns(fl_ctx* ctx, int dim, ColParams& p);
int launch_submatrix(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr,
                     const int32_t* row_idx, const double* values, int32_t n_rows,
                     const int32_t* rows, int32_t n_cols, const int32_t* cols, fl_result* res,
                     int32_t* row_map, int32_t* cnt, uint32_t* d_err, int64_t* nnz_out);
int launch_selftest_div(fl_ctx* ctx, int64_t n, const double* a, const double* b, double* qf,
                        double* qi);
int launch_columns2(fl_ctx* ctx, int dim, ColParams& p, int kmax, fl_result* res);
int launch_columns3(fl_ctx* ctx, int dim, ColParams& p, int kmax, fl_result* res, bool pre,
                    bool finish = true);
int columns3_lanes(int dim, int kmax);
int launch_elem_records(fl_ctx* ctx, int dim, ColParams& p, fl_result* res);

int launch_neumann_add(fl_ctx* ctx, int dim, ColParams& p, fl_result* res);
int launch_hybrid(fl_ctx* ctx, int dim, ColParams& p, fl_mesh* mesh, fl_result* res, bool pre);
int prepare_staging(fl_ctx* ctx, ColParams& p, fl_result* res, int tc, int64_t cap);
int finish_staging(fl_ctx* ctx, ColParams& p, int tc);
int launch_inc_sort(fl_ctx* ctx, fl_mesh* mesh);
int launch_result_counts(fl_ctx* ctx, fl_result* res, int64_t* dev_out);
int launch_boundary_faces(fl_ctx* ctx, fl_mesh* mesh, int64_t* n_faces);
int launch_boundary_scatter(fl_ctx* ctx, fl_mesh* mesh, const int8_t* values, int8_t fill);
int cg_solve_device(fl_ctx* ctx, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                    const double* values, const double* b, double rel_tol, int64_t max_iter,
                    int precond, double* x_out, int64_t* iterations, double* relres, int32_t* converged);
int scatter_free(fl_ctx* ctx, int32_t nf, const int32_t* free_nodes, const double* x, double* u);
int solve_neumann_device(fl_ctx* ctx, int dim, int32_t n, int32_t nt, const double* nodes,
                         const int32_t* elems, const int32_t* col_ptr, const int32_t* row_idx,
                         const double* values, const double* b, int32_t pin, double rel_tol,
                         int64_t max_iter, int precond, double* u, int64_t* iterations, double* relres,
                         int32_t* converged);
int launch_from_triplets(fl_ctx* ctx, int32_t m, int32_t n, int64_t nz, const int32_t* ii,
                         const int32_t* jj, const double* ss, fl_result* res);
int matvec_device(fl_ctx* ctx, int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                  const double* values, const double* x, double* y);
size_t column_smem_bytes();
// v4 (fl_columns4.cu)
int v4_lanes(int dim);
int v4_init_consts(fl_ctx* ctx);
int v4_cap(int dim, int max_inc);
int v4_plan(fl_ctx* ctx, fl_mesh* mesh, bool sync);
int v4_columns(fl_ctx* ctx, fl_mesh* mesh, ColParams& p, fl_result* res);
// FaceLists of partition_boundary (mesh.hpp:222-246) into res->faces
int launch_face_lists(fl_ctx* ctx, fl_mesh* mesh, fl_result* res);
// apply_dirichlet for a caller-supplied A and b (after launch_partition)
int launch_dirichlet_lift(fl_ctx* ctx, fl_mesh* mesh, fl_result* res, const FieldDesc& g,
                          const int32_t* col_ptr, const int32_t* row_idx, const double* values,
                          const double* b);
int launch_scatter_column(fl_ctx* ctx, fl_result* col, int32_t size, double* out);
// fl_result::what bit of an fl_apply_dirichlet result (u0 and b - A u0 held)
constexpr uint32_t kWhatLift = 1u << 8;
int column_tile_width();

}  // namespace fl
