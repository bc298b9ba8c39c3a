/* femlite_oracle.c -- TEST INFRASTRUCTURE ONLY (see femlite_oracle.h).
 *
 * Plain-C restatement of the femlite reference hot path.  Built FMA-free
 * (-ffp-contract=off, no -march; oracle/Makefile) so every expression rounds
 * exactly as the reference's g++ -O3 x86-64 build does.  Expressions keep the
 * reference's evaluation order; citations are to
 * /root/reference/proj/include/femlite/<file>:<line>.
 */
#include "femlite_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* error.hpp:10-26 ordinals, returned as 1 + ordinal */
enum {
    E_INDEX_OUT_OF_RANGE = 1 + 0,
    E_SHAPE_MISMATCH = 1 + 1,
    E_NON_POSITIVE_VOLUME = 1 + 2,
    E_INVALID_FLAG_VALUE = 1 + 3,
    E_DEGENERATE = 1 + 4,
    E_INVALID_PARAMETER = 1 + 5,
    E_UNSORTED_INDEX_SET = 1 + 9,
    E_NO_DIRICHLET = 1 + 13,
    E_UNSUPPORTED_BOUNDARY = 1 + 14,
    E_NOMEM = 100
};

/* mesh.hpp:29-30 */
static const int kTriFaces[3][2] = {{1, 2}, {2, 0}, {0, 1}};
static const int kTetFaces[4][3] = {{1, 3, 2}, {0, 2, 3}, {0, 3, 1}, {0, 1, 2}};
/* quadrature.hpp:62-73 (tet4) */
static const double kTet4A = 0.58541019662496845;
static const double kTet4B = 0.13819660112501051;

void fo_free(void* p) { free(p); }
void fo_csc_free(fo_csc* a) {
    if (!a) return;
    free(a->col_ptr);
    free(a->row_idx);
    free(a->values);
    a->col_ptr = NULL;
    a->row_idx = NULL;
    a->values = NULL;
}

static void* xmalloc(size_t n) { return malloc(n ? n : 1); }
static void* xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s ? s : 1); }

/* ---- fields --------------------------------------------------------------- */
static double eval_field(int kind, double value, const double x[3]) {
    switch (kind) {
    case FO_FIELD_CONST: return value;
    case FO_FIELD_SINSIN: return sin(M_PI * x[0]) * sin(M_PI * x[1]);
    case FO_FIELD_X: return x[0];
    case FO_FIELD_XYZ: return x[0] + x[1] + x[2];
    default: return 0.0;
    }
}

/* ---- mesh.hpp ---------------------------------------------------------------- */
/* mesh.hpp:34-38 */
static double signed_area(const double* v1, const double* v2, const double* v3) {
    const double e2x = v1[0] - v3[0], e2y = v1[1] - v3[1];
    const double e3x = v2[0] - v1[0], e3y = v2[1] - v1[1];
    return 0.5 * (-e3x * e2y + e3y * e2x);
}
/* mesh.hpp:42-51 */
static double signed_volume(const double* v1, const double* v2, const double* v3,
                            const double* v4) {
    const double ax = v2[0] - v1[0], ay = v2[1] - v1[1], az = v2[2] - v1[2];
    const double bx = v3[0] - v1[0], by = v3[1] - v1[1], bz = v3[2] - v1[2];
    const double cx = v4[0] - v1[0], cy = v4[1] - v1[1], cz = v4[2] - v1[2];
    const double nx = ay * bz - az * by;
    const double ny = az * bx - ax * bz;
    const double nz = ax * by - ay * bx;
    return (nx * cx + ny * cy + nz * cz) / 6.0;
}

static double elem_signed_measure(int dim, const double* nodes, const int32_t* v) {
    if (dim == 2)
        return signed_area(nodes + 2 * (size_t)v[0], nodes + 2 * (size_t)v[1],
                           nodes + 2 * (size_t)v[2]);
    return signed_volume(nodes + 3 * (size_t)v[0], nodes + 3 * (size_t)v[1],
                         nodes + 3 * (size_t)v[2], nodes + 3 * (size_t)v[3]);
}

int fo_validate_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, const int8_t* flags) {
    if (dim != 2 && dim != 3) return E_INVALID_PARAMETER;
    if (n_nodes < 0 || n_elems < 0) return E_SHAPE_MISMATCH;
    const int nv = dim + 1;
    for (size_t k = 0; k < (size_t)n_elems * nv; ++k)
        if (elems[k] < 0 || elems[k] >= n_nodes) return E_INDEX_OUT_OF_RANGE;
    if (flags)
        for (size_t k = 0; k < (size_t)n_elems * nv; ++k)
            if (flags[k] < 0 || flags[k] > 3) return E_INVALID_FLAG_VALUE;
    for (int32_t t = 0; t < n_elems; ++t) {
        const double m = elem_signed_measure(dim, nodes, elems + (size_t)t * nv);
        if (!(m > 0.0)) return E_NON_POSITIVE_VOLUME;
    }
    return FO_OK;
}

/* mesh.hpp:310-331 */
static int gen_unit_square(int n, double** nodes_out, int32_t** elems_out, int32_t* nn,
                           int32_t* ne) {
    const double h = 1.0 / n;
    const size_t N = (size_t)(n + 1) * (n + 1), NT = (size_t)2 * n * n;
    double* nodes = xmalloc(sizeof(double) * N * 2);
    int32_t* elems = xmalloc(sizeof(int32_t) * NT * 3);
    if (!nodes || !elems) return E_NOMEM;
    size_t p = 0;
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
            nodes[p++] = i * h;
            nodes[p++] = j * h;
        }
    p = 0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int32_t v00 = j * (n + 1) + i, v10 = j * (n + 1) + i + 1;
            const int32_t v01 = (j + 1) * (n + 1) + i, v11 = (j + 1) * (n + 1) + i + 1;
            elems[p++] = v00; elems[p++] = v10; elems[p++] = v11;
            elems[p++] = v00; elems[p++] = v11; elems[p++] = v01;
        }
    *nodes_out = nodes;
    *elems_out = elems;
    *nn = (int32_t)N;
    *ne = (int32_t)NT;
    return FO_OK;
}

/* mesh.hpp:333-370 (Kuhn split) */
static int gen_unit_cube(int n, double** nodes_out, int32_t** elems_out, int32_t* nn,
                         int32_t* ne) {
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                    {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const int odd[6] = {0, 1, 1, 0, 0, 1};
    const double h = 1.0 / n;
    const size_t N = (size_t)(n + 1) * (n + 1) * (n + 1), NT = (size_t)6 * n * n * n;
    double* nodes = xmalloc(sizeof(double) * N * 3);
    int32_t* elems = xmalloc(sizeof(int32_t) * NT * 4);
    if (!nodes || !elems) return E_NOMEM;
    size_t p = 0;
    for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) {
                nodes[p++] = i * h;
                nodes[p++] = j * h;
                nodes[p++] = k * h;
            }
    p = 0;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                for (int q = 0; q < 6; ++q) {
                    int c[3] = {i, j, k};
                    int32_t tet[4];
                    tet[0] = (c[2] * (n + 1) + c[1]) * (n + 1) + c[0];
                    for (int s = 0; s < 3; ++s) {
                        ++c[perms[q][s]];
                        tet[s + 1] = (c[2] * (n + 1) + c[1]) * (n + 1) + c[0];
                    }
                    if (odd[q]) {
                        const int32_t tmp = tet[2];
                        tet[2] = tet[3];
                        tet[3] = tmp;
                    }
                    for (int s = 0; s < 4; ++s) elems[p++] = tet[s];
                }
    *nodes_out = nodes;
    *elems_out = elems;
    *nn = (int32_t)N;
    *ne = (int32_t)NT;
    return FO_OK;
}

/* mesh.hpp:372-405 */
static int gen_lshape(int n, double** nodes_out, int32_t** elems_out, int32_t* nn,
                      int32_t* ne) {
    const double h = 1.0 / n;
    const int m = 2 * n;
#define CELL_KEPT(i, j) (!((i) >= n && (j) < n))
    int32_t* remap = xmalloc(sizeof(int32_t) * (size_t)(m + 1) * (m + 1));
    double* nodes = xmalloc(sizeof(double) * (size_t)(m + 1) * (m + 1) * 2);
    int32_t* elems = xmalloc(sizeof(int32_t) * (size_t)n * n * 18);
    if (!remap || !nodes || !elems) return E_NOMEM;
    int32_t next = 0;
    size_t p = 0;
    for (int j = 0; j <= m; ++j)
        for (int i = 0; i <= m; ++i) {
            const int used = (i > 0 && j > 0 && CELL_KEPT(i - 1, j - 1)) ||
                             (i < m && j > 0 && CELL_KEPT(i, j - 1)) ||
                             (i > 0 && j < m && CELL_KEPT(i - 1, j)) ||
                             (i < m && j < m && CELL_KEPT(i, j));
            remap[(size_t)j * (m + 1) + i] = -1;
            if (!used) continue;
            remap[(size_t)j * (m + 1) + i] = next++;
            nodes[p++] = -1.0 + i * h;
            nodes[p++] = -1.0 + j * h;
        }
    size_t q = 0;
    for (int j = 0; j < m; ++j)
        for (int i = 0; i < m; ++i) {
            if (!CELL_KEPT(i, j)) continue;
            const int32_t v00 = remap[(size_t)j * (m + 1) + i];
            const int32_t v10 = remap[(size_t)j * (m + 1) + i + 1];
            const int32_t v01 = remap[(size_t)(j + 1) * (m + 1) + i];
            const int32_t v11 = remap[(size_t)(j + 1) * (m + 1) + i + 1];
            elems[q++] = v00; elems[q++] = v10; elems[q++] = v11;
            elems[q++] = v00; elems[q++] = v11; elems[q++] = v01;
        }
#undef CELL_KEPT
    free(remap);
    *nodes_out = nodes;
    *elems_out = elems;
    *nn = next;
    *ne = (int32_t)(q / 3);
    return FO_OK;
}

int fo_generate_mesh(int shape, int n, int32_t* dim, int32_t* n_nodes, int32_t* n_elems,
                     double** nodes, int32_t** elems) {
    if (n < 1) return E_INVALID_PARAMETER;
    switch (shape) {
    case 0: *dim = 2; return gen_unit_square(n, nodes, elems, n_nodes, n_elems);
    case 1: *dim = 3; return gen_unit_cube(n, nodes, elems, n_nodes, n_elems);
    case 2: *dim = 2; return gen_lshape(n, nodes, elems, n_nodes, n_elems);
    }
    return E_INVALID_PARAMETER;
}

/* classifiers: presets.hpp:36-45 (0 dirichlet, 1 pure neumann, 2 mixed) plus the
 * config/test ones defined identically in oracle/ref_shim.cpp. */
static int classify(int kind, const double p[3]) {
    const double tol = 1e-10;
    switch (kind) {
    case 0: return 1;
    case 1: return 2;
    case 2: return fabs(p[1]) < tol ? 2 : 1;
    case 3: {
        const int reentrant = (fabs(p[0]) < tol && p[1] < 0.0) || (fabs(p[1]) < tol && p[0] > 0.0);
        return reentrant ? 2 : 1;
    }
    case 4: return 0;
    case 5: return fabs(p[1]) < tol ? 2 : 0;
    case 6: return fabs(p[2]) < tol ? 2 : 0;
    case 7: return 3;
    }
    return -1;
}

typedef struct {
    int32_t key[3];
    int32_t t;
    int32_t lf;
} face_entry;

static int cmp_face(const void* a, const void* b) {
    const face_entry* x = a;
    const face_entry* y = b;
    for (int k = 0; k < 3; ++k) {
        if (x->key[k] < y->key[k]) return -1;
        if (x->key[k] > y->key[k]) return 1;
    }
    return 0;
}

static void sort3(int32_t* k) {
    int32_t t;
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
    if (k[1] > k[2]) { t = k[1]; k[1] = k[2]; k[2] = t; }
    if (k[0] > k[1]) { t = k[0]; k[0] = k[1]; k[1] = t; }
}

/* mesh.hpp:251-304 */
int fo_set_boundary_flags(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int classifier, int8_t* flags_out) {
    (void)n_nodes;
    const int d = dim, nv = dim + 1;
    const size_t ne = (size_t)n_elems * nv;
    face_entry* e = xmalloc(sizeof(face_entry) * ne);
    if (!e) return E_NOMEM;
    size_t p = 0;
    for (int32_t t = 0; t < n_elems; ++t) {
        const int32_t* v = elems + (size_t)t * nv;
        for (int lf = 0; lf < nv; ++lf) {
            face_entry* x = &e[p++];
            x->t = t;
            x->lf = lf;
            if (d == 2) {
                x->key[0] = v[kTriFaces[lf][0]];
                x->key[1] = v[kTriFaces[lf][1]];
                x->key[2] = 0;
                if (x->key[0] > x->key[1]) {
                    const int32_t tmp = x->key[0];
                    x->key[0] = x->key[1];
                    x->key[1] = tmp;
                }
            } else {
                x->key[0] = v[kTetFaces[lf][0]];
                x->key[1] = v[kTetFaces[lf][1]];
                x->key[2] = v[kTetFaces[lf][2]];
                sort3(x->key);
            }
        }
    }
    qsort(e, ne, sizeof(face_entry), cmp_face);
    memset(flags_out, 0, ne);
    int rc = FO_OK;
    for (size_t i = 0; i < ne;) {
        size_t j = i + 1;
        while (j < ne && cmp_face(&e[j], &e[i]) == 0) ++j;
        if (j - i == 1) {
            const int32_t* v = elems + (size_t)e[i].t * nv;
            double c[3] = {0.0, 0.0, 0.0};
            for (int k = 0; k < d; ++k) {
                const int32_t vi = (d == 2) ? v[kTriFaces[e[i].lf][k]] : v[kTetFaces[e[i].lf][k]];
                for (int q = 0; q < d; ++q) c[q] += nodes[(size_t)vi * d + q];
            }
            for (int q = 0; q < d; ++q) c[q] /= d;
            const int flag = classify(classifier, c);
            if (flag < 0 || flag > 3) { rc = E_INVALID_FLAG_VALUE; break; }
            flags_out[(size_t)e[i].t * nv + e[i].lf] = (int8_t)flag;
        }
        i = j;
    }
    free(e);
    return rc;
}

/* ---- sparse.hpp ------------------------------------------------------------- */
/* sparse.hpp:61-115: two stable counting passes (row key, then column key),
 * duplicate groups summed in original order starting from the first value,
 * exact-zero sums dropped. */
int fo_from_triplets(int32_t m, int32_t n, int64_t count, const int32_t* ii, const int32_t* jj,
                     const double* ss, fo_csc* out) {
    if (m < 0 || n < 0) return E_SHAPE_MISMATCH;
    const size_t nz = (size_t)count;
    for (size_t k = 0; k < nz; ++k)
        if (ii[k] < 0 || ii[k] >= m || jj[k] < 0 || jj[k] >= n) return E_INDEX_OUT_OF_RANGE;
    uint32_t* perm = xmalloc(sizeof(uint32_t) * nz);
    uint32_t* tmp = xmalloc(sizeof(uint32_t) * nz);
    size_t* cnt = xmalloc(sizeof(size_t) * ((size_t)(m > n ? m : n) + 2));
    if (!perm || !tmp || !cnt) return E_NOMEM;
    for (size_t k = 0; k < nz; ++k) perm[k] = (uint32_t)k;
    for (int pass = 0; pass < 2 && nz > 0; ++pass) {
        const int32_t* key = pass == 0 ? ii : jj;
        const size_t bins = (size_t)(pass == 0 ? m : n);
        uint32_t* src = pass == 0 ? perm : tmp;
        uint32_t* dst = pass == 0 ? tmp : perm;
        memset(cnt, 0, sizeof(size_t) * (bins + 1));
        for (size_t k = 0; k < nz; ++k) ++cnt[(size_t)key[src[k]] + 1];
        for (size_t b = 1; b <= bins; ++b) cnt[b] += cnt[b - 1];
        for (size_t k = 0; k < nz; ++k) dst[cnt[(size_t)key[src[k]]]++] = src[k];
    }
    out->m = m;
    out->n = n;
    out->col_ptr = xcalloc((size_t)n + 1, sizeof(int32_t));
    out->row_idx = xmalloc(sizeof(int32_t) * nz);
    out->values = xmalloc(sizeof(double) * nz);
    if (!out->col_ptr || !out->row_idx || !out->values) return E_NOMEM;
    size_t k = 0, w = 0;
    while (k < nz) {
        const int32_t row = ii[perm[k]], col = jj[perm[k]];
        double sum = ss[perm[k]];
        size_t k2 = k + 1;
        while (k2 < nz && ii[perm[k2]] == row && jj[perm[k2]] == col) sum += ss[perm[k2++]];
        if (sum != 0.0) {
            out->row_idx[w] = row;
            out->values[w] = sum;
            ++w;
            ++out->col_ptr[(size_t)col + 1];
        }
        k = k2;
    }
    for (int32_t c = 0; c < n; ++c) out->col_ptr[c + 1] += out->col_ptr[c];
    out->nnz = (int32_t)w;
    free(perm);
    free(tmp);
    free(cnt);
    return FO_OK;
}

/* sparse.hpp:186-198 */
int fo_accumulate(int64_t count, const int32_t* idx, const double* vals, int32_t size,
                  double* out) {
    for (int32_t k = 0; k < size; ++k) out[k] = 0.0;
    for (int64_t k = 0; k < count; ++k) {
        if (idx[k] < 0 || idx[k] >= size) return E_INDEX_OUT_OF_RANGE;
        out[idx[k]] += vals[k];
    }
    return FO_OK;
}

/* sparse.hpp:129-141 */
int fo_matvec(const fo_csc* a, const double* x, double* y) {
    for (int32_t r = 0; r < a->m; ++r) y[r] = 0.0;
    for (int32_t c = 0; c < a->n; ++c) {
        const double xc = x[c];
        for (int32_t k = a->col_ptr[c]; k < a->col_ptr[c + 1]; ++k)
            y[a->row_idx[k]] += a->values[k] * xc;
    }
    return FO_OK;
}

/* sparse.hpp:145-154 */
static int check_index_set(int32_t len, const int32_t* set, int32_t bound) {
    for (int32_t p = 0; p < len; ++p) {
        if (set[p] < 0 || set[p] >= bound) return E_INDEX_OUT_OF_RANGE;
        if (p > 0 && set[p] <= set[p - 1]) return E_UNSORTED_INDEX_SET;
    }
    return FO_OK;
}

/* sparse.hpp:159-183 */
int fo_submatrix(const fo_csc* a, int32_t n_rows, const int32_t* rows, int32_t n_cols,
                 const int32_t* cols, fo_csc* out) {
    int rc = check_index_set(n_rows, rows, a->m);
    if (rc) return rc;
    rc = check_index_set(n_cols, cols, a->n);
    if (rc) return rc;
    int32_t* row_map = xmalloc(sizeof(int32_t) * (size_t)a->m);
    for (int32_t r = 0; r < a->m; ++r) row_map[r] = -1;
    for (int32_t p = 0; p < n_rows; ++p) row_map[rows[p]] = p;
    size_t cap = 0;
    for (int32_t q = 0; q < n_cols; ++q) cap += (size_t)(a->col_ptr[cols[q] + 1] - a->col_ptr[cols[q]]);
    out->m = n_rows;
    out->n = n_cols;
    out->col_ptr = xcalloc((size_t)n_cols + 1, sizeof(int32_t));
    out->row_idx = xmalloc(sizeof(int32_t) * cap);
    out->values = xmalloc(sizeof(double) * cap);
    size_t w = 0;
    for (int32_t q = 0; q < n_cols; ++q) {
        const int32_t c = cols[q];
        for (int32_t k = a->col_ptr[c]; k < a->col_ptr[c + 1]; ++k) {
            const int32_t r = row_map[a->row_idx[k]];
            if (r < 0) continue;
            out->row_idx[w] = r;
            out->values[w] = a->values[k];
            ++w;
        }
        out->col_ptr[q + 1] = (int32_t)w;
    }
    out->nnz = (int32_t)w;
    free(row_map);
    return FO_OK;
}

/* ---- assembly.hpp ------------------------------------------------------------ */
static void cross3(const double u[3], const double v[3], double out[3]) {
    /* assembly.hpp:76-80 */
    out[0] = u[1] * v[2] - u[2] * v[1];
    out[1] = u[2] * v[0] - u[0] * v[2];
    out[2] = u[0] * v[1] - u[1] * v[0];
}

/* assembly.hpp:133-170; returns the unsigned measure, 0 if degenerate */
static double scaled_normals(int dim, const double* vertices, double normals[4][3]) {
    if (dim == 2) {
        const double* v[3] = {&vertices[0], &vertices[2], &vertices[4]};
        double e[3][2];
        for (int i = 0; i < 3; ++i) {
            const int a = kTriFaces[i][1], b = kTriFaces[i][0];
            e[i][0] = v[a][0] - v[b][0];
            e[i][1] = v[a][1] - v[b][1];
        }
        const double area = 0.5 * fabs(-e[2][0] * e[1][1] + e[2][1] * e[1][0]);
        for (int i = 0; i < 3; ++i) {
            normals[i][0] = -e[i][1];
            normals[i][1] = e[i][0];
            normals[i][2] = 0.0;
        }
        return area;
    }
    const double* v[4] = {&vertices[0], &vertices[3], &vertices[6], &vertices[9]};
    double v12[4][3], v13[4][3];
    for (int i = 0; i < 4; ++i) {
        const int f0 = kTetFaces[i][0], f1 = kTetFaces[i][1], f2 = kTetFaces[i][2];
        for (int c = 0; c < 3; ++c) {
            v12[i][c] = v[f1][c] - v[f0][c];
            v13[i][c] = v[f2][c] - v[f0][c];
        }
        cross3(v12[i], v13[i], normals[i]);
    }
    double v14[3];
    for (int c = 0; c < 3; ++c) v14[c] = v[3][c] - v[0][c];
    double cr[3];
    cross3(v12[3], v13[3], cr);
    return fabs(cr[0] * v14[0] + cr[1] * v14[1] + cr[2] * v14[2]) / 6.0;
}

/* assembly.hpp:204-211 */
static void gather_vertices(int dim, const double* nodes, const int32_t* v, double* out) {
    for (int k = 0; k <= dim; ++k)
        for (int c = 0; c < dim; ++c) out[k * dim + c] = nodes[(size_t)v[k] * dim + c];
}

/* assembly.hpp:291-292: one blockwise triplet value */
static double local_entry(const double normals[4][3], double factor, double measure, int i, int j) {
    const double* ni = normals[i];
    const double* nj = normals[j];
    return (ni[0] * nj[0] + ni[1] * nj[1] + ni[2] * nj[2]) / (factor * measure);
}

int fo_local_stiffness_normals(int dim, const double* verts, double* out, double* measure) {
    double normals[4][3];
    const double m = scaled_normals(dim, verts, normals);
    if (m == 0.0) return E_DEGENERATE;
    const double factor = (dim == 2) ? 4.0 : 36.0; /* assembly.hpp:182 */
    for (int i = 0; i <= dim; ++i)
        for (int j = 0; j <= dim; ++j) out[i * (dim + 1) + j] = local_entry(normals, factor, m, i, j);
    *measure = m;
    return FO_OK;
}

/* assembly.hpp:261-300 */
int fo_assemble_blockwise(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, const double* coef, fo_csc* out) {
    const int d = dim, nv = dim + 1;
    const size_t count = (size_t)n_elems;
    double* normals = xmalloc(sizeof(double) * (size_t)nv * count * 3);
    double* measure = xmalloc(sizeof(double) * count);
    const size_t ntrip = count * nv * nv;
    int32_t* ti = xmalloc(sizeof(int32_t) * ntrip);
    int32_t* tj = xmalloc(sizeof(int32_t) * ntrip);
    double* ts = xmalloc(sizeof(double) * ntrip);
    if (!normals || !measure || !ti || !tj || !ts) return E_NOMEM;
    double verts[12], local[4][3];
    for (size_t t = 0; t < count; ++t) {
        gather_vertices(d, nodes, elems + t * nv, verts);
        measure[t] = scaled_normals(d, verts, local);
        if (measure[t] == 0.0) return E_DEGENERATE;
        for (int i = 0; i < nv; ++i)
            for (int c = 0; c < 3; ++c) normals[((size_t)i * count + t) * 3 + c] = local[i][c];
    }
    const double factor = (d == 2) ? 4.0 : 36.0;
    size_t p = 0;
    for (int i = 0; i < nv; ++i)
        for (int j = 0; j < nv; ++j)
            for (size_t t = 0; t < count; ++t) {
                const double* ni = normals + ((size_t)i * count + t) * 3;
                const double* nj = normals + ((size_t)j * count + t) * 3;
                double s = (ni[0] * nj[0] + ni[1] * nj[1] + ni[2] * nj[2]) / (factor * measure[t]);
                if (coef) s = s * coef[t];
                ti[p] = elems[t * nv + i];
                tj[p] = elems[t * nv + j];
                ts[p] = s;
                ++p;
            }
    free(normals);
    free(measure);
    const int rc = fo_from_triplets(n_nodes, n_nodes, (int64_t)ntrip, ti, tj, ts, out);
    free(ti);
    free(tj);
    free(ts);
    return rc;
}

typedef struct {
    int32_t sel, row, key;
    int32_t t;
    double s;
} col_item;

static int cmp_item(const void* a, const void* b) {
    const col_item* x = a;
    const col_item* y = b;
    if (x->sel != y->sel) return x->sel < y->sel ? -1 : 1;
    if (x->row != y->row) return x->row < y->row ? -1 : 1;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    return 0;
}

int fo_assemble_columns(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                        const int32_t* elems, const double* coef, int32_t ncols,
                        const int32_t* cols, fo_csc* out) {
    const int d = dim, nv = dim + 1;
    int32_t* sel = xmalloc(sizeof(int32_t) * (size_t)n_nodes);
    if (!sel) return E_NOMEM;
    for (int32_t k = 0; k < n_nodes; ++k) sel[k] = -1;
    for (int32_t q = 0; q < ncols; ++q) sel[cols[q]] = q;
    size_t cap = 1024, n_items = 0;
    col_item* items = xmalloc(sizeof(col_item) * cap);
    double verts[12], normals[4][3];
    const double factor = (d == 2) ? 4.0 : 36.0;
    for (int32_t t = 0; t < n_elems; ++t) {
        const int32_t* v = elems + (size_t)t * nv;
        int any = 0;
        for (int j = 0; j < nv; ++j) any |= sel[v[j]] >= 0;
        if (!any) continue;
        gather_vertices(d, nodes, v, verts);
        const double m = scaled_normals(d, verts, normals);
        for (int j = 0; j < nv; ++j) {
            if (sel[v[j]] < 0) continue;
            for (int i = 0; i < nv; ++i) {
                if (n_items == cap) {
                    cap *= 2;
                    items = realloc(items, sizeof(col_item) * cap);
                }
                double s = local_entry(normals, factor, m, i, j);
                if (coef) s = s * coef[t];
                col_item it = {sel[v[j]], v[i], i * nv + j, t, s};
                items[n_items++] = it;
            }
        }
    }
    qsort(items, n_items, sizeof(col_item), cmp_item);
    out->m = n_nodes;
    out->n = ncols;
    out->col_ptr = xcalloc((size_t)ncols + 1, sizeof(int32_t));
    out->row_idx = xmalloc(sizeof(int32_t) * n_items);
    out->values = xmalloc(sizeof(double) * n_items);
    size_t k = 0, w = 0;
    while (k < n_items) {
        double sum = items[k].s;
        size_t k2 = k + 1;
        while (k2 < n_items && items[k2].sel == items[k].sel && items[k2].row == items[k].row)
            sum += items[k2++].s;
        if (sum != 0.0) {
            out->row_idx[w] = items[k].row;
            out->values[w] = sum;
            ++w;
            ++out->col_ptr[items[k].sel + 1];
        }
        k = k2;
    }
    for (int32_t q = 0; q < ncols; ++q) out->col_ptr[q + 1] += out->col_ptr[q];
    out->nnz = (int32_t)w;
    free(items);
    free(sel);
    return FO_OK;
}

/* ---- system.hpp --------------------------------------------------------------- */
int fo_sample_load_points(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                          const int32_t* elems, int f_kind, double f_value, double* samples) {
    (void)n_nodes;
    const int nv = dim + 1;
    double verts[12];
    for (int32_t t = 0; t < n_elems; ++t) {
        gather_vertices(dim, nodes, elems + (size_t)t * nv, verts);
        if (dim == 2) {
            for (int i = 0; i < 3; ++i) { /* system.hpp:86-90 */
                const int a = kTriFaces[i][0], b = kTriFaces[i][1];
                const double mid[3] = {(verts[2 * a] + verts[2 * b]) / 2.0,
                                       (verts[2 * a + 1] + verts[2 * b + 1]) / 2.0, 0.0};
                samples[(size_t)t * 3 + i] = eval_field(f_kind, f_value, mid);
            }
        } else {
            for (int q = 0; q < 4; ++q) { /* system.hpp:103-107 */
                double x[3] = {0.0, 0.0, 0.0};
                for (int k = 0; k < 4; ++k) {
                    const double lam = (k == q) ? kTet4A : kTet4B;
                    for (int c = 0; c < 3; ++c) x[c] += lam * verts[k * 3 + c];
                }
                samples[(size_t)t * 4 + q] = eval_field(f_kind, f_value, x);
            }
        }
    }
    return FO_OK;
}

/* system.hpp:71-119 */
int fo_assemble_load(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, int f_kind, double f_value, const double* f_samples,
                     double* b_out) {
    const int nv = dim + 1;
    if (f_kind == FO_FIELD_NONE) {
        for (int32_t k = 0; k < n_nodes; ++k) b_out[k] = 0.0;
        return FO_OK;
    }
    const size_t nt = (size_t)n_elems;
    double* contrib = xcalloc((size_t)nv * nt, sizeof(double));
    int32_t* idx = xmalloc(sizeof(int32_t) * (size_t)nv * nt);
    if (!contrib || !idx) return E_NOMEM;
    double verts[12];
    for (size_t t = 0; t < nt; ++t) {
        gather_vertices(dim, nodes, elems + t * nv, verts);
        if (dim == 2) {
            const double area = fabs(signed_area(&verts[0], &verts[2], &verts[4]));
            double fmid[3];
            for (int i = 0; i < 3; ++i) {
                if (f_kind == FO_FIELD_SAMPLES) {
                    fmid[i] = f_samples[t * 3 + i];
                } else {
                    const int a = kTriFaces[i][0], b = kTriFaces[i][1];
                    const double mid[3] = {(verts[2 * a] + verts[2 * b]) / 2.0,
                                           (verts[2 * a + 1] + verts[2 * b + 1]) / 2.0, 0.0};
                    fmid[i] = eval_field(f_kind, f_value, mid);
                }
            }
            for (int i = 0; i < 3; ++i)
                contrib[(size_t)i * nt + t] = area * (fmid[(i + 1) % 3] + fmid[(i + 2) % 3]) / 6.0;
        } else {
            const double volume = fabs(signed_volume(&verts[0], &verts[3], &verts[6], &verts[9]));
            for (int q = 0; q < 4; ++q) {
                double fx;
                if (f_kind == FO_FIELD_SAMPLES) {
                    fx = f_samples[t * 4 + q];
                } else {
                    double x[3] = {0.0, 0.0, 0.0};
                    for (int k = 0; k < 4; ++k) {
                        const double lam = (k == q) ? kTet4A : kTet4B;
                        for (int c = 0; c < 3; ++c) x[c] += lam * verts[k * 3 + c];
                    }
                    fx = eval_field(f_kind, f_value, x);
                }
                const double w = volume * 0.25 * fx;
                for (int i = 0; i < 4; ++i) {
                    const double lam = (i == q) ? kTet4A : kTet4B;
                    contrib[(size_t)i * nt + t] += w * lam;
                }
            }
        }
    }
    for (int i = 0; i < nv; ++i)
        for (size_t t = 0; t < nt; ++t) idx[(size_t)i * nt + t] = elems[t * nv + i];
    const int rc = fo_accumulate((int64_t)nv * (int64_t)nt, idx, contrib, n_nodes, b_out);
    free(contrib);
    free(idx);
    return rc;
}

/* system.hpp:50-67 with boundary_faces mesh.hpp:222-246 */
int fo_partition_boundary(int dim, int32_t n_nodes, int32_t n_elems, const int32_t* elems,
                          const int8_t* flags, int32_t* n_dir, int32_t** dir_nodes,
                          int32_t* n_free, int32_t** free_nodes, int32_t* n_dir_faces,
                          int32_t* n_neu_faces) {
    const int d = dim, nv = dim + 1;
    for (size_t k = 0; k < (size_t)n_elems * nv; ++k)
        if (flags && flags[k] == 3) return E_UNSUPPORTED_BOUNDARY;
    uint8_t* is_dir = xcalloc((size_t)n_nodes, 1);
    int32_t nd = 0, nn = 0;
    for (int lf = 0; lf <= d; ++lf)
        for (int32_t t = 0; t < n_elems; ++t) {
            const int8_t f = flags ? flags[(size_t)t * nv + lf] : 0;
            if (f == 2) ++nn;
            if (f != 1) continue;
            ++nd;
            const int32_t* v = elems + (size_t)t * nv;
            for (int k = 0; k < d; ++k)
                is_dir[d == 2 ? v[kTriFaces[lf][k]] : v[kTetFaces[lf][k]]] = 1;
        }
    int32_t cd = 0;
    for (int32_t k = 0; k < n_nodes; ++k) cd += is_dir[k];
    *dir_nodes = xmalloc(sizeof(int32_t) * (size_t)cd);
    *free_nodes = xmalloc(sizeof(int32_t) * (size_t)(n_nodes - cd));
    int32_t a = 0, b = 0;
    for (int32_t k = 0; k < n_nodes; ++k) {
        if (is_dir[k]) (*dir_nodes)[a++] = k;
        else (*free_nodes)[b++] = k;
    }
    *n_dir = a;
    *n_free = b;
    *n_dir_faces = nd;
    *n_neu_faces = nn;
    free(is_dir);
    return FO_OK;
}

/* boundary_faces (mesh.hpp:222-246): faces with flag == value, face-major
 * (all local faces 0 over t, then 1, ...), vertices in kTriFaces / kTetFaces
 * order, with the parent element and the local face. */
int fo_boundary_faces(int dim, int32_t n_elems, const int32_t* elems, const int8_t* flags, int value,
                      int32_t* n_faces, int32_t** faces, int32_t** parent, int32_t** local) {
    const int d = dim, nv = dim + 1;
    if (value < 1 || value > 3) return E_INVALID_FLAG_VALUE;
    int32_t n = 0;
    for (size_t k = 0; flags && k < (size_t)n_elems * nv; ++k) n += flags[k] == value;
    *faces = xmalloc(sizeof(int32_t) * (size_t)(n ? n * d : 1));
    *parent = xmalloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    *local = xmalloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int32_t q = 0;
    for (int lf = 0; lf <= d && flags; ++lf)
        for (int32_t t = 0; t < n_elems; ++t) {
            if (flags[(size_t)t * nv + lf] != value) continue;
            const int32_t* v = elems + (size_t)t * nv;
            for (int k = 0; k < d; ++k) (*faces)[(size_t)q * d + k] = d == 2 ? v[kTriFaces[lf][k]] : v[kTetFaces[lf][k]];
            (*parent)[q] = t;
            (*local)[q] = lf;
            ++q;
        }
    *n_faces = n;
    return FO_OK;
}

/* system.hpp:182-201 */
int fo_apply_dirichlet(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                       const int32_t* elems, const int8_t* flags, const fo_csc* a,
                       const double* b, int g_kind, double g_value, const double* g_samples,
                       double* u0_out, double* b_out) {
    int32_t nd, nf, ndf, nnf, *dn, *fn;
    int rc = fo_partition_boundary(dim, n_nodes, n_elems, elems, flags, &nd, &dn, &nf, &fn,
                                   &ndf, &nnf);
    if (rc) return rc;
    if (ndf == 0) { free(dn); free(fn); return E_NO_DIRICHLET; }
    if (a->m != n_nodes || a->n != n_nodes) { free(dn); free(fn); return E_SHAPE_MISMATCH; }
    if (g_kind == FO_FIELD_NONE) { free(dn); free(fn); return 100; } /* empty std::function */
    for (int32_t k = 0; k < n_nodes; ++k) u0_out[k] = 0.0;
    for (int32_t p = 0; p < nd; ++p) {
        const int32_t k = dn[p];
        double x[3] = {0.0, 0.0, 0.0};
        for (int c = 0; c < dim; ++c) x[c] = nodes[(size_t)k * dim + c];
        u0_out[k] = g_kind == FO_FIELD_SAMPLES ? g_samples[k] : eval_field(g_kind, g_value, x);
    }
    double* au0 = xmalloc(sizeof(double) * (size_t)n_nodes);
    fo_matvec(a, u0_out, au0);
    for (int32_t k = 0; k < n_nodes; ++k) b_out[k] = b[k] - au0[k];
    free(au0);
    free(dn);
    free(fn);
    return FO_OK;
}

/* system.hpp:123-172 */
int fo_apply_neumann(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                     const int32_t* elems, const int8_t* flags, int g_kind, double g_value,
                     double* b_inout) {
    const int d = dim, nv = dim + 1;
    if (g_kind == FO_FIELD_NONE) return FO_OK;
    size_t nf = 0;
    for (size_t k = 0; k < (size_t)n_elems * nv; ++k) nf += flags[k] == 2;
    if (nf == 0) return FO_OK;
    int32_t* idx = xmalloc(sizeof(int32_t) * nf * d);
    double* vals = xmalloc(sizeof(double) * nf * d);
    size_t p = 0;
    for (int lf = 0; lf <= d; ++lf)
        for (int32_t t = 0; t < n_elems; ++t) {
            if (flags[(size_t)t * nv + lf] != 2) continue;
            const int32_t* v = elems + (size_t)t * nv;
            int32_t fv[3];
            for (int k = 0; k < d; ++k) fv[k] = d == 2 ? v[kTriFaces[lf][k]] : v[kTetFaces[lf][k]];
            if (d == 2) {
                const double* p0 = nodes + (size_t)fv[0] * 2;
                const double* p1 = nodes + (size_t)fv[1] * 2;
                const double ex = p1[0] - p0[0], ey = p1[1] - p0[1];
                const double length = sqrt(ex * ex + ey * ey);
                const double mid[3] = {(p0[0] + p1[0]) / 2.0, (p0[1] + p1[1]) / 2.0, 0.0};
                const double share = length * eval_field(g_kind, g_value, mid) / 2.0;
                for (int k = 0; k < 2; ++k) { idx[p] = fv[k]; vals[p] = share; ++p; }
            } else {
                const double* p0 = nodes + (size_t)fv[0] * 3;
                const double* p1 = nodes + (size_t)fv[1] * 3;
                const double* p2 = nodes + (size_t)fv[2] * 3;
                double u[3], w[3], cr[3];
                for (int c = 0; c < 3; ++c) { u[c] = p1[c] - p0[c]; w[c] = p2[c] - p0[c]; }
                cross3(u, w, cr);
                const double area = 0.5 * sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
                const double bc[3] = {(p0[0] + p1[0] + p2[0]) / 3.0, (p0[1] + p1[1] + p2[1]) / 3.0,
                                      (p0[2] + p1[2] + p2[2]) / 3.0};
                const double share = area * eval_field(g_kind, g_value, bc) / 3.0;
                for (int k = 0; k < 3; ++k) { idx[p] = fv[k]; vals[p] = share; ++p; }
            }
        }
    double* add = xmalloc(sizeof(double) * (size_t)n_nodes);
    fo_accumulate((int64_t)p, idx, vals, n_nodes, add);
    for (int32_t k = 0; k < n_nodes; ++k) b_inout[k] += add[k];
    free(add);
    free(idx);
    free(vals);
    return FO_OK;
}

/* a_t = 1 + 0.5 sin(2 pi xbar_t), xbar_t = (((x0+x1)+x2)+x3)/4 */
int fo_coefficient_c5(int dim, int32_t n_elems, const double* nodes, const int32_t* elems,
                      double* coef_out) {
    const int nv = dim + 1;
    for (int32_t t = 0; t < n_elems; ++t) {
        const int32_t* v = elems + (size_t)t * nv;
        double xs = 0.0;
        for (int k = 0; k < nv; ++k) xs = (k == 0) ? nodes[(size_t)v[0] * dim] : xs + nodes[(size_t)v[k] * dim];
        const double xbar = xs / (double)nv;
        coef_out[t] = 1.0 + 0.5 * sin((2.0 * M_PI) * xbar);
    }
    return FO_OK;
}

/* ---- text writers ------------------------------------ */
typedef struct {
    char* p;
    int64_t n, cap;
} fo_buf;

static void buf_put(fo_buf* b, const char* s, int64_t k) {
    if (b->n + k + 1 > b->cap) {
        b->cap = (b->n + k + 1) * 2;
        b->p = (char*)realloc(b->p, (size_t)b->cap);
    }
    memcpy(b->p + b->n, s, (size_t)k);
    b->n += k;
}

/* matrix_market.hpp:15-24: header, "m n nnz", then "row+1 col+1 %.17g" per
 * entry, columns ascending */
int fo_write_matrix_market(const fo_csc* a, char** text, int64_t* len) {
    fo_buf b = {NULL, 0, 0};
    char tmp[96];
    int k = snprintf(tmp, sizeof tmp, "%%%%MatrixMarket matrix coordinate real general\n");
    buf_put(&b, tmp, k);
    k = snprintf(tmp, sizeof tmp, "%d %d %d\n", a->m, a->n, a->col_ptr[a->n]);
    buf_put(&b, tmp, k);
    for (int32_t c = 0; c < a->n; ++c)
        for (int32_t q = a->col_ptr[c]; q < a->col_ptr[c + 1]; ++q) {
            char v[32];
            snprintf(v, sizeof v, "%.17g", a->values[q]);
            k = snprintf(tmp, sizeof tmp, "%d %d %s\n", a->row_idx[q] + 1, c + 1, v);
            buf_put(&b, tmp, k);
        }
    *text = b.p;
    *len = b.n;
    return FO_OK;
}

/* mesh_io.hpp:125-142: "d N NT", node coordinates ("%.17g", single spaces),
 * one-based element vertices, flags as int */
int fo_write_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                  const int32_t* elems, const int8_t* flags, char** text, int64_t* len) {
    fo_buf b = {NULL, 0, 0};
    char tmp[128];
    const int nv = dim + 1;
    int k = snprintf(tmp, sizeof tmp, "%d %d %d\n", dim, n_nodes, n_elems);
    buf_put(&b, tmp, k);
    for (int32_t q = 0; q < n_nodes; ++q) {
        for (int c = 0; c < dim; ++c) {
            k = snprintf(tmp, sizeof tmp, "%s%.17g", c ? " " : "", nodes[(size_t)q * dim + c]);
            buf_put(&b, tmp, k);
        }
        buf_put(&b, "\n", 1);
    }
    for (int32_t t = 0; t < n_elems; ++t) {
        for (int c = 0; c < nv; ++c) {
            k = snprintf(tmp, sizeof tmp, "%s%d", c ? " " : "", elems[(size_t)t * nv + c] + 1);
            buf_put(&b, tmp, k);
        }
        buf_put(&b, "\n", 1);
    }
    for (int32_t t = 0; t < n_elems; ++t) {
        for (int c = 0; c < nv; ++c) {
            k = snprintf(tmp, sizeof tmp, "%s%d", c ? " " : "", flags ? (int)flags[(size_t)t * nv + c] : 0);
            buf_put(&b, tmp, k);
        }
        buf_put(&b, "\n", 1);
    }
    *text = b.p;
    *len = b.n;
    return FO_OK;
}
