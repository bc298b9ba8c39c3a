// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" face over the UNMODIFIED femlite reference headers
// (compiled from where they lie under /root/reference/proj/include by
// oracle/Makefile; no reference source is copied into this repository).
// It lets tests/ and bench.py --impl reference drive the reference's own
// hot-path functions through ctypes:
//
//   generate_mesh        mesh.hpp:410     set_boundary_flags  mesh.hpp:251
//   assemble_blockwise   assembly.hpp:261 assemble(strategy)  assembly.hpp:302
//   assemble_load        system.hpp:71    partition_boundary  system.hpp:50
//   apply_neumann        system.hpp:123   apply_dirichlet     system.hpp:182
//   submatrix            sparse.hpp:159   from_triplets       sparse.hpp:61
//   accumulate           sparse.hpp:186   local_stiffness_*   assembly.hpp:88,175
//
// The config-5 variable coefficient does not exist in the reference
// (SPEC.md:386).  ref_assemble_blockwise_coef restates the blockwise loop
// (assembly.hpp:261-300) around the reference's own detail::scaled_normals /
// detail::gather_vertices / from_triplets with s_ij multiplied by the element
// coefficient after the reference division; with a == 1 it
// is bit-identical to assemble_blockwise (checked in tests).
//
// Errors: every entry point returns 0 on success, 1 + femlite::ErrorCode on a
// femlite::Error, 100 on any other exception; ref_last_error() has the text.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <sstream>
#include <atomic>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "femlite/femlite.hpp"

using namespace femlite;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 100;
    }
}

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

Mesh mesh_from(int dim, int n_nodes, int n_elems, const double* nodes, const int32_t* elems,
               const int8_t* flags) {
    std::vector<double> nv(nodes, nodes + std::size_t(n_nodes) * dim);
    std::vector<index_t> ev(elems, elems + std::size_t(n_elems) * (dim + 1));
    std::vector<std::int8_t> fv;
    if (flags) fv.assign(flags, flags + std::size_t(n_elems) * (dim + 1));
    return make_mesh(dim, std::move(nv), std::move(ev), std::move(fv));
}

// Scalar fields the tests and configs need (kind, value) or a C callback.
typedef double (*ref_field_cb)(const double* xyz, void* user);

ScalarField make_field(int kind, double value, ref_field_cb cb, void* user) {
    using std::numbers::pi;
    switch (kind) {
    case 0: return nullptr;                                          // absent
    case 1: return [value](const Point&) { return value; };           // constant
    case 2: return [](const Point& x) { return std::sin(pi * x[0]) * std::sin(pi * x[1]); };
    case 3: return [](const Point& x) { return x[0]; };
    case 4: return [](const Point& x) { return x[0] + x[1] + x[2]; };
    case 5:
        return [cb, user](const Point& x) {
            double p[3] = {x[0], x[1], x[2]};
            return cb(p, user);
        };
    }
    throw Error(ErrorCode::invalid_parameter, "unknown field kind");
}

std::function<int(const Point&)> make_classifier(int kind) {
    constexpr double tol = 1e-10;
    switch (kind) {
    case 0: return [](const Point&) { return 1; };                   // all Dirichlet
    case 1: return [](const Point&) { return 2; };                   // pure Neumann
    case 2: return [tol](const Point& p) { return std::abs(p[1]) < tol ? 2 : 1; }; // mixed
    case 3:                                                          // L-shape re-entrant
        return [tol](const Point& p) {
            const bool reentrant = (std::abs(p[0]) < tol && p[1] < 0.0) ||
                                   (std::abs(p[1]) < tol && p[0] > 0.0);
            return reentrant ? 2 : 1;
        };
    case 4: return [](const Point&) { return 0; };                   // unflagged
    case 5: return [tol](const Point& p) { return std::abs(p[1]) < tol ? 2 : 0; };
    case 6: return [tol](const Point& p) { return std::abs(p[2]) < tol ? 2 : 0; };
    case 7: return [](const Point&) { return 3; };                   // Robin
    }
    throw Error(ErrorCode::invalid_parameter, "unknown classifier");
}

void export_csc(const CscMatrix& a, int32_t* nnz, int32_t** col_ptr, int32_t** row_idx,
                double** values) {
    *nnz = a.nnz();
    *col_ptr = dup(a.col_ptr);
    *row_idx = dup(a.row_idx);
    *values = dup(a.values);
}

CscMatrix import_csc(int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                     const double* values) {
    CscMatrix a;
    a.m = m;
    a.n = n;
    a.col_ptr.assign(col_ptr, col_ptr + n + 1);
    const int32_t nnz = col_ptr[n];
    a.row_idx.assign(row_idx, row_idx + nnz);
    a.values.assign(values, values + nnz);
    return a;
}

// assembly.hpp:261-300 loop structure with an element coefficient (a11).
CscMatrix blockwise_with_coefficient(const Mesh& mesh, const double* coef) {
    const int d = mesh.dim();
    const index_t n = mesh.num_nodes();
    const index_t nt = mesh.num_elems();
    const std::size_t count = static_cast<std::size_t>(nt);
    std::vector<double> normals(std::size_t(d + 1) * count * 3);
    std::vector<double> measure(count);
    double verts[12];
    double local[4][3];
    for (index_t t = 0; t < nt; ++t) {
        detail::gather_vertices(mesh, t, verts);
        measure[std::size_t(t)] = detail::scaled_normals(
            d, std::span<const double>(verts, std::size_t(d + 1) * d), local);
        for (int i = 0; i <= d; ++i)
            for (int c = 0; c < 3; ++c) normals[(std::size_t(i) * count + t) * 3 + c] = local[i][c];
    }
    const double factor = (d == 2) ? 4.0 : 36.0;
    Triplets trip(n, n);
    trip.reserve(std::size_t(nt) * (d + 1) * (d + 1));
    for (int i = 0; i <= d; ++i)
        for (int j = 0; j <= d; ++j)
            for (std::size_t t = 0; t < count; ++t) {
                const double* ni = normals.data() + (std::size_t(i) * count + t) * 3;
                const double* nj = normals.data() + (std::size_t(j) * count + t) * 3;
                const double s =
                    (ni[0] * nj[0] + ni[1] * nj[1] + ni[2] * nj[2]) / (factor * measure[t]);
                const index_t* v = mesh.elem(static_cast<index_t>(t));
                trip.push(v[i], v[j], s * coef[t]);
            }
    return from_triplets(trip);
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// ---- meshes ---------------------------------------------------------------
int ref_generate_mesh(int shape, int n, int32_t* dim, int32_t* n_nodes, int32_t* n_elems,
                      double** nodes, int32_t** elems) {
    return guarded([&] {
        const Mesh m = generate_mesh(static_cast<MeshShape>(shape), n);
        *dim = m.dim();
        *n_nodes = m.num_nodes();
        *n_elems = m.num_elems();
        *nodes = dup(m.nodes());
        *elems = dup(m.elems());
    });
}

int ref_set_boundary_flags(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                           const int32_t* elems, int classifier, int8_t* flags_out) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, nullptr);
        const Mesh f = set_boundary_flags(m, make_classifier(classifier));
        std::memcpy(flags_out, f.bd_flags().data(), f.bd_flags().size());
    });
}

int ref_validate_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                      const int32_t* elems, const int8_t* flags) {
    return guarded([&] { (void)mesh_from(dim, n_nodes, n_elems, nodes, elems, flags); });
}

// ---- assembly -------------------------------------------------------------
int ref_assemble(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                 const int32_t* elems, int strategy, int symmetric_fill, int32_t* nnz,
                 int32_t** col_ptr, int32_t** row_idx, double** values) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, nullptr);
        const CscMatrix a = (strategy == 2 && symmetric_fill)
                                ? assemble_blockwise(m, true)
                                : assemble(m, static_cast<AssemblyStrategy>(strategy));
        export_csc(a, nnz, col_ptr, row_idx, values);
    });
}

int ref_assemble_blockwise_coef(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                                const int32_t* elems, const double* coef, int32_t* nnz,
                                int32_t** col_ptr, int32_t** row_idx, double** values) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, nullptr);
        export_csc(blockwise_with_coefficient(m, coef), nnz, col_ptr, row_idx, values);
    });
}

int ref_local_stiffness(int dim, const double* verts, int which, double* out16,
                        double* measure) {
    return guarded([&] {
        std::span<const double> v(verts, std::size_t(dim + 1) * dim);
        const LocalStiffness s =
            which == 0 ? local_stiffness_reference(dim, v) : local_stiffness_normals(dim, v);
        for (int i = 0; i < 16; ++i) out16[i] = s.a[std::size_t(i)];
        *measure = s.measure;
    });
}

int ref_assemble_load(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                      const int32_t* elems, int f_kind, double f_value, ref_field_cb cb,
                      void* user, double* b_out) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, nullptr);
        const std::vector<double> b = assemble_load(m, make_field(f_kind, f_value, cb, user));
        std::memcpy(b_out, b.data(), sizeof(double) * b.size());
    });
}

int ref_apply_neumann(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                      const int32_t* elems, const int8_t* flags, int g_kind, double g_value,
                      ref_field_cb cb, void* user, double* b_inout) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        std::vector<double> b(b_inout, b_inout + n_nodes);
        b = apply_neumann(std::move(b), m, make_field(g_kind, g_value, cb, user));
        std::memcpy(b_inout, b.data(), sizeof(double) * b.size());
    });
}

int ref_partition_boundary(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                           const int32_t* elems, const int8_t* flags, int32_t* n_dir,
                           int32_t** dir_nodes, int32_t* n_free, int32_t** free_nodes,
                           int32_t* n_dir_faces, int32_t* n_neu_faces) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const BoundaryPartition p = partition_boundary(m);
        *n_dir = static_cast<int32_t>(p.dirichlet_nodes.size());
        *n_free = static_cast<int32_t>(p.free_nodes.size());
        *dir_nodes = dup(p.dirichlet_nodes);
        *free_nodes = dup(p.free_nodes);
        *n_dir_faces = static_cast<int32_t>(p.dirichlet_faces.size());
        *n_neu_faces = static_cast<int32_t>(p.neumann_faces.size());
    });
}

int ref_boundary_faces(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                       const int32_t* elems, const int8_t* flags, int value, int32_t* n_faces,
                       int32_t** faces, int32_t** parent, int32_t** local) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const FaceList f = boundary_faces(m, value);
        *n_faces = static_cast<int32_t>(f.size());
        *faces = dup(f.faces);
        *parent = dup(f.parent_elem);
        std::vector<int32_t> lf(f.local_face.begin(), f.local_face.end());
        *local = dup(lf);
    });
}

int ref_apply_dirichlet(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                        const int32_t* elems, const int8_t* flags, const int32_t* col_ptr,
                        const int32_t* row_idx, const double* values, const double* b,
                        int g_kind, double g_value, ref_field_cb cb, void* user, double* u0_out,
                        double* b_out) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const CscMatrix a = import_csc(n_nodes, n_nodes, col_ptr, row_idx, values);
        const DirichletSystem s = apply_dirichlet(a, std::span<const double>(b, n_nodes), m,
                                                  make_field(g_kind, g_value, cb, user));
        std::memcpy(u0_out, s.u0.data(), sizeof(double) * s.u0.size());
        std::memcpy(b_out, s.b.data(), sizeof(double) * s.b.size());
    });
}

int ref_submatrix(int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                  const double* values, int32_t n_rows, const int32_t* rows, int32_t n_cols,
                  const int32_t* cols, int32_t* nnz, int32_t** out_col_ptr,
                  int32_t** out_row_idx, double** out_values) {
    return guarded([&] {
        const CscMatrix a = import_csc(m, n, col_ptr, row_idx, values);
        const CscMatrix s = submatrix(a, std::span<const index_t>(rows, std::size_t(n_rows)),
                                      std::span<const index_t>(cols, std::size_t(n_cols)));
        export_csc(s, nnz, out_col_ptr, out_row_idx, out_values);
    });
}

int ref_from_triplets(int32_t m, int32_t n, int64_t count, const int32_t* ii, const int32_t* jj,
                      const double* ss, int32_t* nnz, int32_t** col_ptr, int32_t** row_idx,
                      double** values) {
    return guarded([&] {
        Triplets t(m, n);
        t.i.assign(ii, ii + count);
        t.j.assign(jj, jj + count);
        t.s.assign(ss, ss + count);
        export_csc(from_triplets(t), nnz, col_ptr, row_idx, values);
    });
}

int ref_accumulate(int64_t count, const int32_t* idx, const double* vals, int32_t size,
                   double* out) {
    return guarded([&] {
        const std::vector<double> r =
            accumulate(std::span<const index_t>(idx, std::size_t(count)),
                       std::span<const double>(vals, std::size_t(count)), size);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

// ---- the reference's own CPU path, timed in-process --------------------------
// One "step" of the hot path exactly as solve_poisson runs it before the solve
// (solver.hpp:226-242): partition_boundary, assemble_blockwise (or the a11
// coefficient loop), assemble_load, apply_neumann, apply_dirichlet, submatrix,
// b_f gather.  Returns wall seconds per step for `reps` steps (steady_clock,
// as bench.hpp:88-97) and the assembled sizes for a consistency check.
int ref_time_system(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                    const int32_t* elems, const int8_t* flags, int f_kind, double f_value,
                    const double* coef, int reps, double* seconds_out, int64_t* nnz_out,
                    int64_t* nnz_ff_out) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const ScalarField f = make_field(f_kind, f_value, nullptr, nullptr);
        const ScalarField zero = [](const Point&) { return 0.0; };
        for (int r = 0; r < reps; ++r) {
            const auto t0 = std::chrono::steady_clock::now();
            const BoundaryPartition part = partition_boundary(m);
            const CscMatrix a = coef ? blockwise_with_coefficient(m, coef) : assemble_blockwise(m);
            std::vector<double> b = assemble_load(m, f);
            b = apply_neumann(std::move(b), m, nullptr);
            DirichletSystem sys = apply_dirichlet(a, b, m, zero);
            const std::vector<index_t>& fr = sys.partition.free_nodes;
            const CscMatrix a_ff = submatrix(a, fr, fr);
            std::vector<double> b_f(fr.size());
            for (std::size_t k = 0; k < fr.size(); ++k) b_f[k] = sys.b[std::size_t(fr[k])];
            seconds_out[r] =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            nnz_out[0] = a.nnz();
            nnz_ff_out[0] = a_ff.nnz();
            (void)part;
        }
    });
}

// The same pipeline on `threads` host threads at once, each on its own copy of
// the pipeline's outputs over the shared (read-only) mesh: the reference is
// single-threaded by construction, so "all host threads" is throughput --
// threads x NT elements per wall-clock step.  seconds_out[r] = wall time of
// round r (all threads started together, timed until the last one finishes).
int ref_time_system_mt(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                       const int32_t* elems, const int8_t* flags, int f_kind, double f_value,
                       const double* coef, int reps, int threads, double* seconds_out) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const ScalarField f = make_field(f_kind, f_value, nullptr, nullptr);
        const ScalarField zero = [](const Point&) { return 0.0; };
        std::atomic<int> failed{0};
        auto work = [&]() {
            try {
                const BoundaryPartition part = partition_boundary(m);
                const CscMatrix a = coef ? blockwise_with_coefficient(m, coef) : assemble_blockwise(m);
                std::vector<double> b = assemble_load(m, f);
                b = apply_neumann(std::move(b), m, nullptr);
                DirichletSystem sys = apply_dirichlet(a, b, m, zero);
                const std::vector<index_t>& fr = sys.partition.free_nodes;
                const CscMatrix a_ff = submatrix(a, fr, fr);
                std::vector<double> b_f(fr.size());
                for (std::size_t k = 0; k < fr.size(); ++k) b_f[k] = sys.b[std::size_t(fr[k])];
                (void)part;
                (void)a_ff;
            } catch (...) {
                failed = 1;
            }
        };
        for (int r = 0; r < reps; ++r) {
            std::vector<std::thread> pool;
            const auto t0 = std::chrono::steady_clock::now();
            for (int k = 0; k < threads; ++k) pool.emplace_back(work);
            for (auto& t : pool) t.join();
            seconds_out[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        if (failed) throw std::runtime_error("a worker thread failed");
    });
}

// sparse.hpp:129-141
int ref_matvec(int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
               const double* values, const double* x, double* y_out) {
    return guarded([&] {
        const CscMatrix a = import_csc(m, n, col_ptr, row_idx, values);
        const std::vector<double> y = matvec(a, std::span<const double>(x, std::size_t(n)));
        std::memcpy(y_out, y.data(), sizeof(double) * y.size());
    });
}

// solver.hpp:63-136; precond 0 none, 1 jacobi, 2 auto
int ref_cg_solve(int32_t n, const int32_t* col_ptr, const int32_t* row_idx, const double* values,
                 const double* b, double rel_tol, int64_t max_iter, int precond, double* x_out,
                 int64_t* iterations, double* relres, int32_t* converged) {
    return guarded([&] {
        const CscMatrix a = import_csc(n, n, col_ptr, row_idx, values);
        SolveOptions o;
        o.rel_tol = rel_tol;
        o.max_iter = static_cast<index_t>(max_iter);
        o.preconditioner = precond == 0 ? Preconditioner::none
                         : precond == 1 ? Preconditioner::jacobi : Preconditioner::auto_select;
        const CgResult r = cg_solve(a, std::span<const double>(b, std::size_t(n)), o);
        std::memcpy(x_out, r.x.data(), sizeof(double) * r.x.size());
        *iterations = r.iterations;
        *relres = r.relres;
        *converged = r.converged ? 1 : 0;
    });
}

// solver.hpp:223-247 (Dirichlet meshes): u, iterations, relres; wall seconds
int ref_solve_poisson(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                      const int32_t* elems, const int8_t* flags, int f_kind, double f_value,
                      int g_kind, double g_value, double rel_tol, double* u_out,
                      int64_t* iterations, double* relres, double* seconds) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        PoissonProblem pb;
        pb.f = make_field(f_kind, f_value, nullptr, nullptr);
        pb.g_dirichlet = make_field(g_kind, g_value, nullptr, nullptr);
        SolveOptions o;
        o.rel_tol = rel_tol;
        const auto t0 = std::chrono::steady_clock::now();
        const Solution sol = solve_poisson(m, pb, o);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(u_out, sol.u.data(), sizeof(double) * sol.u.size());
        *iterations = sol.iterations;
        *relres = sol.final_relres;
    });
}

// ---- text writers (matrix_market.hpp:15-24, mesh_io.hpp:125-142) -----------
static void export_text(const std::string& t, char** text, int64_t* len) {
    *len = static_cast<int64_t>(t.size());
    *text = static_cast<char*>(std::malloc(t.size() + 1));
    std::memcpy(*text, t.data(), t.size());
}

int ref_write_matrix_market(int32_t m, int32_t n, const int32_t* col_ptr, const int32_t* row_idx,
                            const double* values, char** text, int64_t* len, double* seconds) {
    return guarded([&] {
        const CscMatrix a = import_csc(m, n, col_ptr, row_idx, values);
        const auto t0 = std::chrono::steady_clock::now();
        std::ostringstream os;
        write_matrix_market(a, os);
        const std::string t = os.str();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        export_text(t, text, len);
    });
}

int ref_write_mesh(int dim, int32_t n_nodes, int32_t n_elems, const double* nodes,
                   const int32_t* elems, const int8_t* flags, char** text, int64_t* len,
                   double* seconds) {
    return guarded([&] {
        const Mesh m = mesh_from(dim, n_nodes, n_elems, nodes, elems, flags);
        const auto t0 = std::chrono::steady_clock::now();
        std::ostringstream os;
        write_mesh(m, os);
        const std::string t = os.str();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        export_text(t, text, len);
    });
}

} // extern "C"
