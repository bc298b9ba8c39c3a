/* femlite_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the femlite reference's P1 assembly hot path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER.  Nothing in paper_1804_05156_b200/ links or calls this.  Every
 * function cites the reference lines it restates (paths relative to
 * /root/reference/proj/include/femlite/).  It is pinned against the compiled
 * reference (oracle/_ref) and the golden fixtures in tests/golden/.
 *
 * Status codes mirror the reference: 0 ok, 1 + femlite::ErrorCode ordinal
 * (error.hpp:10-26) on a reference error.  All output arrays are malloc'd and
 * released with fo_free().
 */
#ifndef FEMLITE_ORACLE_H
#define FEMLITE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FO_OK = 0 };
/* field kinds shared with the product ABI (include/femlite_b200.h) */
enum {
    FO_FIELD_NONE = 0,    /* absent std::function: zero / no-op                 */
    FO_FIELD_CONST = 1,   /* f(x) = value                                       */
    FO_FIELD_SINSIN = 2,  /* sin(pi x) sin(pi y), glibc sin                      */
    FO_FIELD_X = 3,       /* x                                                  */
    FO_FIELD_XYZ = 4,     /* x + y + z                                          */
    FO_FIELD_SAMPLES = 6  /* caller-provided samples at the rule's points        */
};

typedef struct {
    int32_t m, n, nnz;
    int32_t* col_ptr; /* n + 1 */
    int32_t* row_idx; /* nnz   */
    double* values;   /* nnz   */
} fo_csc;

void fo_free(void* p);
void fo_csc_free(fo_csc* a);

/* mesh.hpp:410-419 (unit_square 349-370, unit_cube 372-409, lshape 411-444) */
int fo_generate_mesh(int shape, int n, int32_t* dim, int32_t* n_nodes, int32_t* n_elems,
                     double** nodes, int32_t** elems);
/* mesh.hpp:174-187 + 187-208 (make_mesh validation) */
int fo_validate_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, const int8_t* flags);
/* mesh.hpp:251-304 with the classifiers of presets.hpp:36-45 (+ L-shape, see .c) */
int fo_set_boundary_flags(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int classifier, int8_t* flags_out);

/* sparse.hpp:61-115 */
int fo_from_triplets(int32_t m, int32_t n, int64_t count, const int32_t* ii, const int32_t* jj,
                     const double* ss, fo_csc* out);
/* sparse.hpp:186-198 */
int fo_accumulate(int64_t count, const int32_t* idx, const double* vals, int32_t size,
                  double* out);
/* sparse.hpp:129-141 */
int fo_matvec(const fo_csc* a, const double* x, double* y);
/* sparse.hpp:159-183 */
int fo_submatrix(const fo_csc* a, int32_t n_rows, const int32_t* rows, int32_t n_cols,
                 const int32_t* cols, fo_csc* out);

/* assembly.hpp:175-189 local_stiffness_normals (out: (d+1)^2 row-major) */
int fo_local_stiffness_normals(int dim, const double* verts, double* out, double* measure);
/* assembly.hpp:261-300; coef (nullable) = per-element coefficient multiplied
 * after the reference division. */
int fo_assemble_blockwise(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, const double* coef, fo_csc* out);
/* Same values as fo_assemble_blockwise restricted to the (strictly increasing)
 * column set `cols`, computed by scanning all elements once: the reference's
 * (i*(d+1)+j, t) summation order per entry, zero drop.  out->n = ncols,
 * out->m = n_nodes.  Used for full-size spot checks. */
int fo_assemble_columns(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                        const int32_t* elems, const double* coef, int32_t ncols,
                        const int32_t* cols, fo_csc* out);

/* system.hpp:71-119.  f_samples (kind SAMPLES): per element, f at the rule's
 * points: 2-D edge midpoints (t*3+i, face i), 3-D tet4 points (t*4+q). */
int fo_assemble_load(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, int f_kind, double f_value, const double* f_samples,
                     double* b_out);
/* Host-side sampling of a built-in field at the load rule's points, with the
 * reference's point formulas (system.hpp:86-90, 104-107). */
int fo_sample_load_points(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int f_kind, double f_value, double* samples);

/* system.hpp:50-67 */
int fo_partition_boundary(int dim, int32_t n_nodes, int32_t n_elems, const int32_t* elems,
                          const int8_t* flags, int32_t* n_dir, int32_t** dir_nodes,
                          int32_t* n_free, int32_t** free_nodes, int32_t* n_dir_faces,
                          int32_t* n_neu_faces);
/* boundary_faces (mesh.hpp:222-246), arrays malloc'ed (fo_free) */
int fo_boundary_faces(int dim, int32_t n_elems, const int32_t* elems, const int8_t* flags, int value,
                      int32_t* n_faces, int32_t** faces, int32_t** parent, int32_t** local);
/* system.hpp:182-201 (g of kind NONE is rejected like calling an empty
 * std::function; SAMPLES = g at every node, used only at Dirichlet nodes) */
int fo_apply_dirichlet(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                       const int32_t* elems, const int8_t* flags, const fo_csc* a,
                       const double* b, int g_kind, double g_value, const double* g_samples,
                       double* u0_out, double* b_out);
/* system.hpp:123-172 (g kinds NONE/CONST/X/XYZ/SINSIN) */
int fo_apply_neumann(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, const int8_t* flags, int g_kind, double g_value,
                     double* b_inout);

/* Config-5 coefficient a(x) = 1 + 0.5 sin(2 pi x1) at element barycentres
 * (SURVEY.md §8 a11), glibc sin. */
int fo_coefficient_c5(int dim, int32_t n_elems, const double* nodes, const int32_t* elems,
                      double* coef_out);

/* Text writers: the bytes of write_matrix_market
 * (matrix_market.hpp:15-24) and write_mesh (mesh_io.hpp:125-142), "%.17g" for
 * every double (detail::format_real, mesh_io.hpp:56-60) and decimal integers,
 * into a malloc'd buffer (*text, *len bytes; free with fo_free). */
int fo_write_matrix_market(const fo_csc* a, char** text, int64_t* len);
int fo_write_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                  const int32_t* elems, const int8_t* flags, char** text, int64_t* len);

#ifdef __cplusplus
}
#endif
#endif
