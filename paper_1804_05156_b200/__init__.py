"""B200-native P1 finite element assembly (drop-in for femlite's hot path).

Public API mirrors femlite (/root/reference/proj/include/femlite/):

    Mesh, make_mesh, generate_mesh, MeshShape, set_boundary_flags      mesh.hpp
    CscMatrix, submatrix                                                sparse.hpp
    assemble_blockwise, assemble, AssemblyStrategy                      assembly.hpp
    assemble_load, partition_boundary, apply_neumann,
    BoundaryPartition, DirichletSystem                                  system.hpp
    assemble_system / poisson_system  (solve_poisson's pre-solve path,  solver.hpp:226-242)
    matvec, cg_solve, solve_poisson (§8(f) row 2)                       sparse.hpp, solver.hpp
    boundary.set_boundary_flags (GPU face matching, §8(f) row 1)        mesh.hpp:251-304
    write_matrix_market, write_mesh, format_real (§8(f) row 4)        matrix_market.hpp, mesh_io.hpp
    ErrorCode, Error                                                    error.hpp

All compute runs in libfemlite_b200.so (hand-written sm_100a kernels behind
the C-ABI of include/femlite_b200.h); importing does not touch the GPU.
"""
from .api import (AssemblyResult, AssemblyStrategy, BoundaryPartition, CgResult, CscMatrix, FaceList,
                  DirichletSystem, PoissonSystem, Solution, assemble, assemble_blockwise,
                  accumulate, apply_dirichlet, assemble_load, assemble_system, apply_neumann, cg_solve,
                  from_triplets, matvec,
                  partition_boundary,
                  poisson_system, run, solve_poisson, submatrix)
from .context import Context
from .text import (Text, format_real, format_reals, write_matrix_market, write_mesh,
                   write_result_matrix_market)
from .errors import Error, ErrorCode
from .mesh import (Mesh, MeshShape, boundary_face_mask, classifier_dirichlet, classifier_lshape,
                   classifier_mixed, classifier_neumann, flag_generated, generate_mesh, make_mesh,
                   set_boundary_flags)

__all__ = [
    "AssemblyResult", "AssemblyStrategy", "BoundaryPartition", "CgResult", "Context", "CscMatrix", "FaceList",
    "DirichletSystem", "Error", "ErrorCode", "Mesh", "MeshShape", "PoissonSystem", "assemble",
    "accumulate", "apply_dirichlet", "assemble_blockwise", "assemble_load", "assemble_system",
    "apply_neumann",
    "boundary_face_mask", "classifier_dirichlet", "classifier_lshape", "classifier_mixed",
    "classifier_neumann", "flag_generated", "generate_mesh", "make_mesh", "partition_boundary",
    "poisson_system", "run", "set_boundary_flags", "submatrix", "cg_solve", "matvec", "solve_poisson",
    "Solution", "from_triplets", "Text", "format_real", "format_reals", "write_matrix_market",
    "write_mesh", "write_result_matrix_market",
]
