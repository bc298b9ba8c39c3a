// femlite_b200_adapter.hpp -- the femlite-side binding of the B200 C-ABI.
//
// Header-only C++20 over include/femlite_b200.h with the reference's own types
// and signatures (paths relative to femlite's proj/include/femlite/):
//
//   femlite_b200::assemble_blockwise(mesh)           assembly.hpp:261  assemble_blockwise
//   femlite_b200::assemble(mesh, strategy)           assembly.hpp:302  assemble
//   femlite_b200::assemble_load(mesh, f)             system.hpp:71     assemble_load
//   femlite_b200::partition_boundary(mesh)           system.hpp:50     partition_boundary
//   femlite_b200::apply_neumann(b, mesh, g)          system.hpp:123    apply_neumann
//   femlite_b200::poisson_system(mesh, problem)      solver.hpp:226-242 (pre-solve path:
//                                                    partition, A, b, Neumann, Dirichlet lift,
//                                                    A(free, free), b_f -- one fused pass)
//   femlite_b200::submatrix(a, rows, cols)           sparse.hpp:159    submatrix
//   femlite_b200::apply_dirichlet(a, b, mesh, g)     system.hpp:182    apply_dirichlet (any A, b)
//   femlite_b200::from_triplets(t)                   sparse.hpp:61     from_triplets
//   femlite_b200::accumulate(idx, vals, size)        sparse.hpp:186    accumulate
//   femlite_b200::matvec / cg_solve / solve_poisson  sparse.hpp:129, solver.hpp:63, :223
//   femlite_b200::write_matrix_market(a, out)        matrix_market.hpp:15 write_matrix_market
//   femlite_b200::write_mesh(mesh, out)              mesh_io.hpp:125      write_mesh
//
// Include it after the femlite headers.  Errors are rethrown as
// femlite::Error with the reference's ErrorCode (the ABI status is
// 1 + ordinal).  Host callables (ScalarField) are evaluated on the host at the
// reference's quadrature / face points (fl_host_points) and passed as samples,
// so results are bitwise the reference's.  INTEGRATION.md shows the one-line
// hook in femlite's assemble() dispatcher.
#pragma once

#include <cstdint>
#include <memory>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "femlite/error.hpp"
#include "femlite/mesh.hpp"
#include "femlite/solver.hpp"
#include "femlite/sparse.hpp"
#include "femlite/system.hpp"
#include "femlite_b200.h"

namespace femlite_b200 {

inline void check(int rc, const char* what) {
    if (rc == FL_OK) return;
    const std::string msg = std::string(what) + ": " + fl_last_error();
    if (rc >= 1 && rc <= 1 + static_cast<int>(femlite::ErrorCode::unsupported_boundary_type))
        throw femlite::Error(static_cast<femlite::ErrorCode>(rc - 1), msg);
    throw std::runtime_error(msg);
}

/// One device + stream; the default context (device 0) is created on first use.
class Context {
public:
    explicit Context(int device = 0) { check(fl_create(device, &ctx_), "fl_create"); }
    ~Context() { fl_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    fl_ctx* get() const { return ctx_; }
    static Context& default_context() {
        static Context ctx(0);
        return ctx;
    }

private:
    fl_ctx* ctx_ = nullptr;
};

namespace detail {

struct MeshHandle {
    fl_mesh* m = nullptr;
    MeshHandle(Context& ctx, const femlite::Mesh& mesh) {
        const auto& fl = mesh.bd_flags();
        check(fl_mesh_create(ctx.get(), mesh.dim(), mesh.num_nodes(), mesh.num_elems(),
                             mesh.nodes().data(), mesh.elems().data(),
                             fl.empty() ? nullptr : fl.data(), FL_MEM_HOST, &m),
              "fl_mesh_create");
    }
    ~MeshHandle() { fl_mesh_destroy(m); }
    MeshHandle(const MeshHandle&) = delete;
    MeshHandle& operator=(const MeshHandle&) = delete;
};

struct ResultHandle {
    fl_result* r = nullptr;
    explicit ResultHandle(Context& ctx) { check(fl_result_create(ctx.get(), &r), "fl_result_create"); }
    ~ResultHandle() { fl_result_destroy(r); }
    ResultHandle(const ResultHandle&) = delete;
    ResultHandle& operator=(const ResultHandle&) = delete;

    fl_sizes sizes() const {
        fl_sizes z{};
        check(fl_result_sizes(r, &z), "fl_result_sizes");
        return z;
    }
    template <class T>
    std::vector<T> array(int which, int64_t count) const {
        std::vector<T> out(static_cast<std::size_t>(count));
        check(fl_result_copy(r, which, out.empty() ? nullptr : out.data(),
                             static_cast<int64_t>(out.size() * sizeof(T)), FL_MEM_HOST),
              "fl_result_copy");
        return out;
    }
    femlite::CscMatrix matrix(int m) const {
        const fl_sizes z = sizes();
        femlite::CscMatrix a;
        a.m = m;
        a.n = z.n;
        a.col_ptr = array<femlite::index_t>(FL_A_COL_PTR, z.n + 1);
        a.row_idx = array<femlite::index_t>(FL_A_ROW_IDX, z.nnz);
        a.values = array<double>(FL_A_VALUES, z.nnz);
        return a;
    }
    femlite::CscMatrix matrix_ff() const {
        const fl_sizes z = sizes();
        femlite::CscMatrix a;
        a.m = z.n_free;
        a.n = z.n_free_cols;
        a.col_ptr = array<femlite::index_t>(FL_AFF_COL_PTR, z.n_free_cols + 1);
        a.row_idx = array<femlite::index_t>(FL_AFF_ROW_IDX, z.nnz_ff);
        a.values = array<double>(FL_AFF_VALUES, z.nnz_ff);
        return a;
    }
};

/// f sampled at the reference's points of `rule` (0: load, 3: Neumann faces)
inline std::vector<double> sample(const femlite::Mesh& mesh, const femlite::ScalarField& f,
                                  int rule) {
    const std::size_t np = static_cast<std::size_t>(mesh.num_elems()) * (mesh.dim() + 1);
    std::vector<double> xyz(np * 3), out(np);
    check(fl_host_points(mesh.dim(), mesh.num_nodes(), mesh.num_elems(), mesh.nodes().data(),
                         mesh.elems().data(), rule, xyz.data()),
          "fl_host_points");
    for (std::size_t k = 0; k < np; ++k)
        out[k] = f(femlite::Point{xyz[3 * k], xyz[3 * k + 1], xyz[3 * k + 2]});
    return out;
}

inline std::vector<double> sample_nodes(const femlite::Mesh& mesh, const femlite::ScalarField& g) {
    std::vector<double> out(static_cast<std::size_t>(mesh.num_nodes()));
    for (femlite::index_t k = 0; k < mesh.num_nodes(); ++k) out[k] = g(mesh.node_point(k));
    return out;
}

inline fl_field none() { return fl_field{FL_FIELD_NONE, FL_MEM_HOST, 0.0, nullptr, 0}; }
inline fl_field samples(const std::vector<double>& v) {
    return fl_field{FL_FIELD_SAMPLES, FL_MEM_HOST, 0.0, v.data(), static_cast<int64_t>(v.size())};
}

/// boundary_faces(mesh, 1 | 2) (mesh.hpp:222-246) as the GPU produced them
inline femlite::FaceList face_list_of(const femlite::Mesh& mesh, const ResultHandle& r, bool dirichlet) {
    const fl_sizes z = r.sizes();
    const int64_t n = dirichlet ? z.n_dir_faces : z.n_neu_faces;
    femlite::FaceList f;
    f.dim = mesh.dim();
    f.faces = r.array<femlite::index_t>(dirichlet ? FL_DIR_FACES : FL_NEU_FACES, n * mesh.dim());
    f.parent_elem = r.array<femlite::index_t>(dirichlet ? FL_DIR_FACE_ELEM : FL_NEU_FACE_ELEM, n);
    const std::vector<int32_t> lf = r.array<int32_t>(dirichlet ? FL_DIR_FACE_LOCAL : FL_NEU_FACE_LOCAL, n);
    f.local_face.assign(lf.begin(), lf.end());
    return f;
}

inline femlite::BoundaryPartition partition_of(const femlite::Mesh& mesh, const ResultHandle& r) {
    const fl_sizes z = r.sizes();
    femlite::BoundaryPartition p;
    p.dirichlet_nodes = r.array<femlite::index_t>(FL_DIR_NODES, z.n_dir);
    p.free_nodes = r.array<femlite::index_t>(FL_FREE_NODES, z.n_free);
    p.dirichlet_faces = face_list_of(mesh, r, true);
    p.neumann_faces = face_list_of(mesh, r, false);
    return p;
}

}  // namespace detail

/// assembly.hpp:261 on the GPU (symmetric_fill only changes the reference's
/// triplet multiset and is rejected, as the GPU path has no triplets).
inline femlite::CscMatrix assemble_blockwise(const femlite::Mesh& mesh, bool symmetric_fill = false,
                                             Context& ctx = Context::default_context()) {
    if (symmetric_fill)
        throw femlite::Error(femlite::ErrorCode::invalid_parameter,
                             "symmetric_fill is a CPU triplet-order option");
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    const fl_field n = detail::none();
    check(fl_assemble(ctx.get(), m.m, &n, &n, &n, &n, FL_OUT_STIFFNESS, r.r), "fl_assemble");
    return r.matrix(mesh.num_nodes());
}

/// assembly.hpp:302: blockwise runs on the GPU; the reference's CPU oracles
/// (dense_oracle, triplet_loop) are its own cross-checks and stay on the CPU.
inline femlite::CscMatrix assemble(const femlite::Mesh& mesh, femlite::AssemblyStrategy strategy,
                                   Context& ctx = Context::default_context()) {
    if (strategy != femlite::AssemblyStrategy::blockwise)
        throw femlite::Error(femlite::ErrorCode::invalid_parameter,
                             "only the blockwise strategy runs on the B200 path");
    return assemble_blockwise(mesh, false, ctx);
}

/// system.hpp:71
inline std::vector<double> assemble_load(const femlite::Mesh& mesh, const femlite::ScalarField& f,
                                         Context& ctx = Context::default_context()) {
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    std::vector<double> fs;
    fl_field ff = detail::none();
    if (f) {
        fs = detail::sample(mesh, f, 0);
        ff = detail::samples(fs);
    }
    const fl_field n = detail::none();
    check(fl_assemble(ctx.get(), m.m, &ff, &n, &n, &n, FL_OUT_LOAD, r.r), "fl_assemble");
    return r.array<double>(FL_B, r.sizes().n);
}

/// system.hpp:50
inline femlite::BoundaryPartition partition_boundary(const femlite::Mesh& mesh,
                                                     Context& ctx = Context::default_context()) {
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    const fl_field n = detail::none();
    check(fl_assemble(ctx.get(), m.m, &n, &n, &n, &n, FL_OUT_PARTITION, r.r), "fl_assemble");
    return detail::partition_of(mesh, r);
}

/// system.hpp:123: the Neumann face shares accumulated on the GPU, then added
/// to b entry by entry (b[k] += add[k], system.hpp:170)
inline std::vector<double> apply_neumann(std::vector<double> b, const femlite::Mesh& mesh,
                                         const femlite::ScalarField& g,
                                         Context& ctx = Context::default_context()) {
    if (static_cast<femlite::index_t>(b.size()) != mesh.num_nodes())
        throw femlite::Error(femlite::ErrorCode::shape_mismatch, "apply_neumann: vector length");
    if (!g) return b;
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    const std::vector<double> gs = detail::sample(mesh, g, 3);
    const fl_field gn = detail::samples(gs), n = detail::none();
    check(fl_assemble(ctx.get(), m.m, &n, &n, &n, &gn, FL_OUT_LOAD, r.r), "fl_assemble");
    const std::vector<double> add = r.array<double>(FL_B, r.sizes().n);
    for (std::size_t k = 0; k < b.size(); ++k) b[k] += add[k];
    return b;
}

/// Everything solve_poisson builds before its solve (solver.hpp:226-242).
struct PoissonSystem {
    femlite::CscMatrix a;
    std::vector<double> b;
    femlite::DirichletSystem dirichlet;  // u0, b - A u0, partition
    femlite::CscMatrix a_ff;
    std::vector<double> b_f;
};

inline PoissonSystem poisson_system(const femlite::Mesh& mesh, const femlite::PoissonProblem& pb,
                                    Context& ctx = Context::default_context()) {
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    std::vector<double> fs, gd, gn;
    fl_field ff = detail::none(), fd = detail::none(), fn = detail::none();
    const fl_field n = detail::none();
    if (pb.f) ff = detail::samples(fs = detail::sample(mesh, pb.f, 0));
    if (pb.g_dirichlet) fd = detail::samples(gd = detail::sample_nodes(mesh, pb.g_dirichlet));
    if (pb.g_neumann) fn = detail::samples(gn = detail::sample(mesh, pb.g_neumann, 3));
    check(fl_assemble(ctx.get(), m.m, &ff, &n, &fd, &fn, FL_OUT_SYSTEM, r.r), "fl_assemble");
    const fl_sizes z = r.sizes();
    PoissonSystem s;
    s.a = r.matrix(mesh.num_nodes());
    s.b = r.array<double>(FL_B, z.n);
    s.dirichlet.u0 = r.array<double>(FL_U0, z.n);
    s.dirichlet.b = r.array<double>(FL_B_MOD, z.n);
    s.dirichlet.partition = detail::partition_of(mesh, r);
    s.a_ff = r.matrix_ff();
    s.b_f = r.array<double>(FL_B_F, z.n_free_cols);
    return s;
}

/// sparse.hpp:129-141, bitwise
inline std::vector<double> matvec(const femlite::CscMatrix& a, std::span<const double> x,
                                  Context& ctx = Context::default_context()) {
    if (static_cast<femlite::index_t>(x.size()) != a.n)
        throw femlite::Error(femlite::ErrorCode::shape_mismatch, "matvec: vector length mismatch");
    std::vector<double> y(static_cast<std::size_t>(a.m));
    check(fl_matvec(ctx.get(), a.m, a.n, a.col_ptr.data(), a.row_idx.data(), a.values.data(), x.data(),
                    y.data(), FL_MEM_HOST),
          "fl_matvec");
    return y;
}

/// solver.hpp:63-136 on the GPU (dot products are tree reductions: iterates
/// agree with the reference to rounding)
inline femlite::CgResult cg_solve(const femlite::CscMatrix& a, std::span<const double> b,
                                  const femlite::SolveOptions& opts = {},
                                  Context& ctx = Context::default_context()) {
    if (a.m != a.n) throw femlite::Error(femlite::ErrorCode::shape_mismatch, "cg_solve: matrix not square");
    if (static_cast<femlite::index_t>(b.size()) != a.n)
        throw femlite::Error(femlite::ErrorCode::shape_mismatch, "cg_solve: vector length mismatch");
    fl_cg_options o{opts.rel_tol, opts.max_iter,
                    opts.preconditioner == femlite::Preconditioner::none     ? 0
                    : opts.preconditioner == femlite::Preconditioner::jacobi ? 1
                                                                            : 2,
                    0};
    femlite::CgResult r;
    r.x.resize(b.size());
    int64_t it = 0;
    int32_t conv = 1;
    check(fl_cg_solve(ctx.get(), a.n, a.col_ptr.data(), a.row_idx.data(), a.values.data(), b.data(),
                      FL_MEM_HOST, &o, r.x.data(), &it, &r.relres, &conv),
          "fl_cg_solve");
    r.iterations = static_cast<femlite::index_t>(it);
    r.converged = conv != 0;
    return r;
}

/// solver.hpp:223-276 device-resident: with Dirichlet faces the free-node
/// system (lift, A(free, free), b_f) and CG; without them the pure-Neumann path
/// (compatibility, pinned node opts.pin_node, zero-average shift).  Throws
/// max_iter_exceeded like solve_reduced.  SolveMethod::dense_direct is the
/// reference's small-system CPU check (a dense factorisation guarded by
/// kDenseGuardLimit): rejected here with invalid_parameter.
inline femlite::Solution solve_poisson(const femlite::Mesh& mesh, const femlite::PoissonProblem& pb,
                                       const femlite::SolveOptions& opts = {},
                                       Context& ctx = Context::default_context()) {
    if (opts.method == femlite::SolveMethod::dense_direct)
        throw femlite::Error(femlite::ErrorCode::invalid_parameter,
                             "dense_direct is the reference's CPU check; the B200 path solves with CG");
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    std::vector<double> fs, gd, gn;
    fl_field ff = detail::none(), fd = detail::none(), fn = detail::none();
    const fl_field n = detail::none();
    if (pb.f) ff = detail::samples(fs = detail::sample(mesh, pb.f, 0));
    if (pb.g_neumann) fn = detail::samples(gn = detail::sample(mesh, pb.g_neumann, 3));
    // partition_boundary first (solver.hpp:226): Robin flags, Dirichlet or not
    detail::ResultHandle part(ctx);
    check(fl_assemble(ctx.get(), m.m, &n, &n, &n, &n, FL_OUT_PARTITION, part.r), "fl_assemble");
    const bool dirichlet = part.sizes().n_dir_faces > 0;
    fl_cg_options o{opts.rel_tol, opts.max_iter,
                    opts.preconditioner == femlite::Preconditioner::none     ? 0
                    : opts.preconditioner == femlite::Preconditioner::jacobi ? 1
                                                                            : 2,
                    0};
    femlite::Solution sol;
    sol.u.resize(static_cast<std::size_t>(mesh.num_nodes()));
    int64_t it = 0;
    if (dirichlet) {
        if (pb.g_dirichlet) fd = detail::samples(gd = detail::sample_nodes(mesh, pb.g_dirichlet));
        check(fl_assemble(ctx.get(), m.m, &ff, &n, &fd, &fn, FL_OUT_SYSTEM, r.r), "fl_assemble");
        check(fl_solve_system(ctx.get(), r.r, &o, sol.u.data(), FL_MEM_HOST, &it, &sol.final_relres),
              "fl_solve_system");
        sol.partition = detail::partition_of(mesh, r);
    } else {
        const femlite::index_t pin = opts.pin_node.value_or(0);
        if (pin < 0 || pin >= mesh.num_nodes())
            throw femlite::Error(femlite::ErrorCode::index_out_of_range, "pin_node out of range");
        check(fl_assemble(ctx.get(), m.m, &ff, &n, &n, &fn, FL_OUT_STIFFNESS | FL_OUT_LOAD | FL_OUT_PARTITION, r.r),
              "fl_assemble");
        check(fl_solve_neumann(ctx.get(), m.m, r.r, pin, &o, sol.u.data(), FL_MEM_HOST, &it, &sol.final_relres),
              "fl_solve_neumann");
        sol.partition = detail::partition_of(mesh, r);
    }
    sol.iterations = static_cast<femlite::index_t>(it);
    return sol;
}

/// system.hpp:182-201 for any caller-supplied A and b: the partition, u0 = g at
/// the Dirichlet nodes, b - A u0 (matvec's column order, sparse.hpp:129-141), on
/// the GPU, bitwise.  g is sampled at every node on the host.
inline femlite::DirichletSystem apply_dirichlet(const femlite::CscMatrix& a, std::span<const double> b,
                                                const femlite::Mesh& mesh, const femlite::ScalarField& g,
                                                Context& ctx = Context::default_context()) {
    detail::MeshHandle m(ctx, mesh);
    detail::ResultHandle r(ctx);
    std::vector<double> gs;
    fl_field gd = detail::none();
    if (g) gd = detail::samples(gs = detail::sample_nodes(mesh, g));
    check(fl_apply_dirichlet(ctx.get(), m.m, a.m, a.n, a.col_ptr.data(), a.row_idx.data(), a.values.data(),
                             static_cast<int64_t>(b.size()), b.data(), FL_MEM_HOST, &gd, r.r),
          "fl_apply_dirichlet");
    const fl_sizes z = r.sizes();
    femlite::DirichletSystem s;
    s.u0 = r.array<double>(FL_U0, z.n);
    s.b = r.array<double>(FL_B_MOD, z.n);
    s.partition = detail::partition_of(mesh, r);
    return s;
}

/// sparse.hpp:61-115 on the GPU (stable by (column, row), duplicates summed in
/// their original order, exact-zero sums dropped), bitwise
inline femlite::CscMatrix from_triplets(const femlite::Triplets& t, Context& ctx = Context::default_context()) {
    if (t.i.size() != t.s.size() || t.j.size() != t.s.size())
        throw femlite::Error(femlite::ErrorCode::shape_mismatch, "triplet arrays differ in length");
    detail::ResultHandle r(ctx);
    check(fl_from_triplets(ctx.get(), t.m, t.n, static_cast<int64_t>(t.size()), t.i.data(), t.j.data(),
                           t.s.data(), FL_MEM_HOST, r.r),
          "fl_from_triplets");
    return r.matrix(t.m);
}

/// sparse.hpp:186-198 on the GPU, bitwise
inline std::vector<double> accumulate(std::span<const femlite::index_t> idx, std::span<const double> vals,
                                      femlite::index_t size, Context& ctx = Context::default_context()) {
    if (idx.size() != vals.size())
        throw femlite::Error(femlite::ErrorCode::shape_mismatch, "accumulate: index/value lengths differ");
    std::vector<double> out(static_cast<std::size_t>(size > 0 ? size : 0));
    check(fl_accumulate(ctx.get(), static_cast<int64_t>(idx.size()), idx.data(), vals.data(), size,
                        out.empty() ? nullptr : out.data(), FL_MEM_HOST),
          "fl_accumulate");
    return out;
}

/// sparse.hpp:159 (strictly increasing index sets, validated on the GPU)
inline femlite::CscMatrix submatrix(const femlite::CscMatrix& a,
                                    std::span<const femlite::index_t> rows,
                                    std::span<const femlite::index_t> cols,
                                    Context& ctx = Context::default_context()) {
    detail::ResultHandle r(ctx);
    check(fl_submatrix(ctx.get(), a.m, a.n, a.col_ptr.data(), a.row_idx.data(), a.values.data(),
                       static_cast<int32_t>(rows.size()), rows.data(),
                       static_cast<int32_t>(cols.size()), cols.data(), FL_MEM_HOST, r.r),
          "fl_submatrix");
    return r.matrix(static_cast<femlite::index_t>(rows.size()));
}

namespace detail {
struct TextHandle {
    fl_text* t = nullptr;
    explicit TextHandle(Context& ctx) { check(fl_text_create(ctx.get(), &t), "fl_text_create"); }
    ~TextHandle() { fl_text_destroy(t); }
    TextHandle(const TextHandle&) = delete;
    TextHandle& operator=(const TextHandle&) = delete;
    void write_to(std::ostream& out) const {
        int64_t n = 0;
        check(fl_text_size(t, &n), "fl_text_size");
        std::string s(static_cast<std::size_t>(n), '\0');
        check(fl_text_copy(t, s.data(), n, FL_MEM_HOST), "fl_text_copy");
        out.write(s.data(), static_cast<std::streamsize>(n));
    }
};
}  // namespace detail

/// matrix_market.hpp:15-24: the same bytes, formatted on the GPU (exact %.17g)
inline void write_matrix_market(const femlite::CscMatrix& a, std::ostream& out,
                                Context& ctx = Context::default_context()) {
    detail::TextHandle t(ctx);
    check(fl_write_matrix_market(ctx.get(), a.m, a.n, a.col_ptr.data(), a.row_idx.data(),
                                 a.values.data(), FL_MEM_HOST, t.t),
          "fl_write_matrix_market");
    t.write_to(out);
}

/// mesh_io.hpp:125-142: the same bytes, formatted on the GPU
inline void write_mesh(const femlite::Mesh& mesh, std::ostream& out,
                       Context& ctx = Context::default_context()) {
    detail::MeshHandle m(ctx, mesh);
    detail::TextHandle t(ctx);
    check(fl_write_mesh(ctx.get(), m.m, t.t), "fl_write_mesh");
    t.write_to(out);
}

}  // namespace femlite_b200
