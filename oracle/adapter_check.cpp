// adapter_check.cpp -- TEST INFRASTRUCTURE: the femlite reference (its own
// headers, unmodified) against the B200 path called through the C++ adapter
// (include/femlite_b200_adapter.hpp -> the C-ABI -> libfemlite_b200.so).
// Built by oracle/Makefile into _ref/adapter_check where /root/reference
// exists; tests/test_gpu_adapter.py runs the binary on the GPU box.
// Exit 0 = every comparison bitwise equal (CscMatrix::operator==, memcmp).
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <numbers>
#include <sstream>
#include <vector>

#include "femlite/assembly.hpp"
#include "femlite/matrix_market.hpp"
#include "femlite/mesh_io.hpp"
#include "femlite/mesh.hpp"
#include "femlite/solver.hpp"
#include "femlite/sparse.hpp"
#include "femlite/system.hpp"
#include "femlite_b200_adapter.hpp"

namespace {

int failures = 0, checks = 0;

void expect(bool ok, const char* what, const char* mesh) {
    ++checks;
    if (!ok) {
        ++failures;
        std::printf("FAIL %s on %s\n", what, mesh);
    }
}

bool same(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() &&
           (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
}

femlite::Mesh jitter(const femlite::Mesh& m, double amp, unsigned seed) {
    // deterministic interior jitter (boundary nodes stay put): LCG, no <random>
    std::vector<double> nodes = m.nodes();
    std::vector<char> on(static_cast<std::size_t>(m.num_nodes()), 0);
    const int nv = m.dim() + 1;
    for (femlite::index_t t = 0; t < m.num_elems(); ++t)
        for (int f = 0; f < nv; ++f)
            if (m.flag(t, f) != 0)
                for (int k = 0; k < nv; ++k)
                    if (k != f) on[m.elem(t)[k]] = 1;
    unsigned s = seed;
    for (std::size_t k = 0; k < on.size(); ++k)
        for (int c = 0; c < m.dim(); ++c) {
            s = s * 1664525u + 1013904223u;
            if (!on[k]) nodes[k * m.dim() + c] += amp * ((s >> 8) * (1.0 / 16777216.0) - 0.5);
        }
    return femlite::make_mesh(m.dim(), nodes, m.elems(), m.bd_flags());
}

// FaceList (mesh.hpp:101-109) element by element
bool same_faces(const femlite::FaceList& a, const femlite::FaceList& b) {
    return a.dim == b.dim && a.faces == b.faces && a.parent_elem == b.parent_elem && a.local_face == b.local_face;
}

void run(const char* name, const femlite::Mesh& mesh) {
    using namespace femlite;
    const double pi = std::numbers::pi;
    const ScalarField f = [pi](const Point& p) { return std::sin(pi * p[0]) * std::sin(pi * p[1]); };
    const ScalarField g = [](const Point& p) { return 1.0 + p[0] - 0.5 * p[1] + p[2]; };
    const ScalarField gn = [](const Point& p) { return 0.25 + p[1]; };

    expect(assemble_blockwise(mesh) == femlite_b200::assemble_blockwise(mesh), "assemble_blockwise", name);
    expect(femlite::assemble(mesh, AssemblyStrategy::blockwise) ==
               femlite_b200::assemble(mesh, AssemblyStrategy::blockwise),
           "assemble(blockwise)", name);
    const std::vector<double> b = assemble_load(mesh, f);
    expect(same(b, femlite_b200::assemble_load(mesh, f)), "assemble_load", name);
    const BoundaryPartition p = partition_boundary(mesh);
    const BoundaryPartition q = femlite_b200::partition_boundary(mesh);
    expect(p.dirichlet_nodes == q.dirichlet_nodes && p.free_nodes == q.free_nodes, "partition_boundary nodes",
           name);
    expect(same_faces(p.dirichlet_faces, q.dirichlet_faces), "partition_boundary dirichlet_faces", name);
    expect(same_faces(p.neumann_faces, q.neumann_faces), "partition_boundary neumann_faces", name);
    expect(same(apply_neumann(b, mesh, gn), femlite_b200::apply_neumann(b, mesh, gn)), "apply_neumann",
           name);
    if (p.dirichlet_faces.size() > 0) {
        // solve_poisson's pre-solve path (solver.hpp:226-242) vs the fused GPU pass
        const CscMatrix a = assemble_blockwise(mesh);
        const std::vector<double> bn = apply_neumann(b, mesh, gn);
        const DirichletSystem ds = apply_dirichlet(a, bn, mesh, g);
        const CscMatrix aff = submatrix(a, p.free_nodes, p.free_nodes);
        std::vector<double> bf;
        for (index_t k : p.free_nodes) bf.push_back(ds.b[static_cast<std::size_t>(k)]);
        const PoissonProblem pb{f, g, gn};
        const femlite_b200::PoissonSystem s = femlite_b200::poisson_system(mesh, pb);
        expect(s.a == a, "poisson_system A", name);
        expect(same(s.b, bn), "poisson_system b (load + Neumann)", name);
        expect(same(s.dirichlet.u0, ds.u0), "poisson_system u0", name);
        expect(same(s.dirichlet.b, ds.b), "poisson_system b - A u0", name);
        expect(s.a_ff == aff, "poisson_system A(free, free)", name);
        expect(same(s.b_f, bf), "poisson_system b_f", name);
        // the solve after the path (tolerance: CG dot products differ in order)
        expect(same(matvec(a, bn), femlite_b200::matvec(a, bn)), "matvec", name);
        SolveOptions so;
        const Solution ref_sol = femlite::solve_poisson(mesh, pb, so);
        const Solution gpu_sol = femlite_b200::solve_poisson(mesh, pb, so);
        double worst = 0.0, scale = 1.0;
        for (std::size_t k = 0; k < ref_sol.u.size(); ++k) {
            worst = std::max(worst, std::abs(ref_sol.u[k] - gpu_sol.u[k]));
            scale = std::max(scale, std::abs(ref_sol.u[k]));
        }
        expect(worst <= 1e-7 * scale, "solve_poisson u (1e-7 relative)", name);
        expect(std::abs(ref_sol.iterations - gpu_sol.iterations) <= 2, "solve_poisson iterations", name);
        // apply_dirichlet with an A and b that are not the assembled ones (system.hpp:182-201)
        CscMatrix a2 = a;
        for (double& v : a2.values) v = 2.0 * v;
        std::vector<double> b2(bn.size());
        for (std::size_t k = 0; k < b2.size(); ++k) b2[k] = 0.5 * bn[k] - 1.0 / double(k + 3);
        const DirichletSystem d2 = apply_dirichlet(a2, b2, mesh, g);
        const DirichletSystem q2 = femlite_b200::apply_dirichlet(a2, b2, mesh, g);
        expect(same(d2.u0, q2.u0) && same(d2.b, q2.b), "apply_dirichlet(2A, b')", name);
        expect(same_faces(d2.partition.dirichlet_faces, q2.partition.dirichlet_faces) &&
                   d2.partition.free_nodes == q2.partition.free_nodes,
               "apply_dirichlet partition", name);
        // ... and with A from from_triplets of a scrambled COO (duplicates, cancellations)
        Triplets t(a.m, a.n);
        for (index_t c = 0; c < a.n; ++c)
            for (index_t k = a.col_ptr[c]; k < a.col_ptr[c + 1]; ++k) {
                const index_t r = a.row_idx[k];
                t.push(r, c, a.values[k] * 0.75);
                t.push((r * 7 + c) % a.m, (c * 3 + 1) % a.n, 1.0 / double(k + 1));
                t.push((r * 7 + c) % a.m, (c * 3 + 1) % a.n, -1.0 / double(k + 1));
            }
        const CscMatrix at = from_triplets(t);
        expect(at == femlite_b200::from_triplets(t), "from_triplets", name);
        const DirichletSystem r3 = apply_dirichlet(at, b2, mesh, g);
        const DirichletSystem q3 = femlite_b200::apply_dirichlet(at, b2, mesh, g);
        expect(same(r3.u0, q3.u0) && same(r3.b, q3.b), "apply_dirichlet(from_triplets A, b')", name);
        // accumulate (sparse.hpp:186-198)
        std::vector<index_t> idx;
        std::vector<double> vals;
        for (std::size_t k = 0; k < t.size(); ++k) {
            idx.push_back(t.i[k]);
            vals.push_back(t.s[k]);
        }
        expect(same(accumulate(idx, vals, a.m), femlite_b200::accumulate(idx, vals, a.m)), "accumulate", name);
        // dense_direct is rejected explicitly
        SolveOptions dd;
        dd.method = SolveMethod::dense_direct;
        try {
            femlite_b200::solve_poisson(mesh, pb, dd);
            expect(false, "dense_direct rejected", name);
        } catch (const Error& e) {
            expect(e.code() == ErrorCode::invalid_parameter, "dense_direct rejected", name);
        }
        // general submatrix
        std::vector<index_t> rows, cols;
        for (index_t k = 0; k < a.m; k += 2) rows.push_back(k);
        for (index_t k = 1; k < a.n; k += 3) cols.push_back(k);
        expect(submatrix(a, rows, cols) == femlite_b200::submatrix(a, rows, cols), "submatrix", name);
        // text writers (matrix_market.hpp:15-24, mesh_io.hpp:125-142): the same bytes
        std::ostringstream r1, g1, r2, g2;
        write_matrix_market(a, r1);
        femlite_b200::write_matrix_market(a, g1);
        expect(r1.str() == g1.str(), "write_matrix_market", name);
        write_mesh(mesh, r2);
        femlite_b200::write_mesh(mesh, g2);
        expect(r2.str() == g2.str(), "write_mesh", name);
    }
}

}  // namespace

int main() {
    using namespace femlite;
    auto dirichlet = [](const Point&) { return 1; };
    auto mixed = [](const Point& p) { return p[0] < 1e-10 ? 2 : 1; };
    auto lshape = [](const Point& p) {
        return ((std::abs(p[0]) < 1e-10 && p[1] < 0) || (std::abs(p[1]) < 1e-10 && p[0] > 0)) ? 2 : 1;
    };
    const Mesh sq = set_boundary_flags(generate_mesh(MeshShape::unit_square, 12), mixed);
    run("unit_square:12 mixed", sq);
    run("unit_square:12 mixed jittered", jitter(sq, 0.02, 7));
    const Mesh ls = set_boundary_flags(generate_mesh(MeshShape::lshape, 8), lshape);
    run("lshape:8 jittered", jitter(ls, 0.03, 11));
    const Mesh cu = set_boundary_flags(generate_mesh(MeshShape::unit_cube, 4), dirichlet);
    run("unit_cube:4", cu);
    run("unit_cube:4 jittered", jitter(cu, 0.04, 13));
    run("unit_cube:3 mixed", set_boundary_flags(generate_mesh(MeshShape::unit_cube, 3), mixed));
    // pure-Neumann solve_poisson (solver.hpp:253-276): no Dirichlet face
    {
        const Mesh pn = set_boundary_flags(generate_mesh(MeshShape::unit_square, 10), [](const Point&) { return 2; });
        const double pi = std::numbers::pi;
        const PoissonProblem pb{[pi](const Point& p) { return std::cos(pi * p[0]) * std::cos(pi * p[1]); }, {},
                                [](const Point& p) { return p[0] - 0.5; }};
        for (int pin : {0, 7}) {
            SolveOptions so;
            so.pin_node = pin;
            const Solution rs = femlite::solve_poisson(pn, pb, so);
            const Solution gs = femlite_b200::solve_poisson(pn, pb, so);
            double worst = 0.0, scale = 1.0;
            for (std::size_t k = 0; k < rs.u.size(); ++k) {
                worst = std::max(worst, std::abs(rs.u[k] - gs.u[k]));
                scale = std::max(scale, std::abs(rs.u[k]));
            }
            expect(worst <= 1e-7 * scale, "solve_poisson pure-Neumann u (1e-7 relative)", "unit_square:10 neumann");
            expect(same_faces(rs.partition.neumann_faces, gs.partition.neumann_faces),
                   "solve_poisson pure-Neumann partition", "unit_square:10 neumann");
        }
    }
    // errors surface as femlite::Error with the reference's code
    try {
        const Mesh robin = set_boundary_flags(generate_mesh(MeshShape::unit_square, 2),
                                              [](const Point&) { return 3; });
        femlite_b200::partition_boundary(robin);
        expect(false, "Robin flags rejected", "unit_square:2 robin");
    } catch (const Error& e) {
        expect(e.code() == ErrorCode::unsupported_boundary_type, "Robin error code", "unit_square:2 robin");
    }
    std::printf("adapter_check: %d checks, %d failures\n", checks, failures);
    return failures == 0 ? 0 : 1;
}
