"""B200-native P1 finite element assembly (drop-in for femlite's hot path).

Public API mirrors femlite (/root/reference/proj/include/femlite/):

    Mesh, make_mesh, generate_mesh, MeshShape, set_boundary_flags      mesh.hpp
    CscMatrix, submatrix                                                sparse.hpp
    assemble_blockwise, assemble, AssemblyStrategy                      assembly.hpp
    assemble_load, partition_boundary, apply_neumann,
    BoundaryPartition, DirichletSystem                                  system.hpp
    assemble_system / poisson_system  (solve_poisson's pre-solve path,  solver.hpp:226-242)
    ErrorCode, Error                                                    error.hpp

All compute runs in libfemlite_b200.so (hand-written sm_100a kernels behind
the C-ABI of include/femlite_b200.h); importing does not touch the GPU.
"""
from .api import (AssemblyResult, AssemblyStrategy, BoundaryPartition, CscMatrix, DirichletSystem,
                  PoissonSystem, assemble, assemble_blockwise, assemble_load, assemble_system,
                  apply_neumann, partition_boundary, poisson_system, run, submatrix)
from .context import Context
from .errors import Error, ErrorCode
from .mesh import (Mesh, MeshShape, boundary_face_mask, classifier_dirichlet, classifier_lshape,
                   classifier_mixed, classifier_neumann, flag_generated, generate_mesh, make_mesh,
                   set_boundary_flags)

__all__ = [
    "AssemblyResult", "AssemblyStrategy", "BoundaryPartition", "Context", "CscMatrix",
    "DirichletSystem", "Error", "ErrorCode", "Mesh", "MeshShape", "PoissonSystem", "assemble",
    "assemble_blockwise", "assemble_load", "assemble_system", "apply_neumann",
    "boundary_face_mask", "classifier_dirichlet", "classifier_lshape", "classifier_mixed",
    "classifier_neumann", "flag_generated", "generate_mesh", "make_mesh", "partition_boundary",
    "poisson_system", "run", "set_boundary_flags", "submatrix",
]
