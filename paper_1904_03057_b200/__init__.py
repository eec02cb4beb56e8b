"""B200-native tensor B-spline heat / elliptic solve path.

Drop-in for the solve path of the reference package ``bspde``
(arxiv/paper_1904_03057): grid/degree setup, exact separable mass and
stiffness Gram factors, the matrix-free operator apply, Jacobi-PCG and RHS
assembly -- with the apply, the CG iteration and the RHS running as
hand-written sm_100a CUDA kernels (``csrc/bspde_b200.cu``) behind a C ABI
(``include/bspde_b200.h``).  Adds implicit-Euler heat stepping and z-slab
multi-GPU sharding.  There is no CPU fallback.
"""

from .boundary import FACE_NAMES, DirichletPenalty, Neumann, Robin, realize_bc
from .domain import BoxDomain, Grid, MaskDomain, active_nodes, interior_nodes, node_classes
from .errors import (ConditioningWarning, ConfigurationError, DegreeError, DeterminismError,
                     DivergenceError, EmptyDomainError, FormatError, OutOfDomainError, IndefiniteOperatorError, NativeLibraryError,
                     ResourceError, ValidationError)
from .gram import GramFactor, basis_extension, edge_width, gram_factor, min_axis_length
from .heat import HeatProblem, HeatSolver, heat_solve
from .io import (export_vtk, read_field, read_mask, read_tensor, write_field, write_mask,
                 write_tensor)
from .problem import ProblemSpec, Solution, assemble_system, coarse_initialize, solve_problem
from .operator import B200Operator, OpStats, assembled_rhs, make_operator
from .solver import SolveConfig, SolveReport, pcg, pcg_device
from .system import SystemData, build_system, heat_system, mass_system
from .transform import direct_transform, sample_solution, transform_field

__all__ = [
    "BoxDomain", "Grid", "MaskDomain", "active_nodes", "interior_nodes", "node_classes", "FACE_NAMES", "Robin", "Neumann", "DirichletPenalty", "realize_bc",
    "basis_extension", "edge_width", "gram_factor", "min_axis_length",
    "GramFactor", "SystemData", "build_system", "heat_system", "mass_system",
    "B200Operator", "OpStats", "make_operator", "assembled_rhs",
    "SolveConfig", "SolveReport", "pcg", "pcg_device",
    "HeatProblem", "HeatSolver", "heat_solve",
    "direct_transform", "transform_field", "sample_solution",
    "ProblemSpec", "Solution", "assemble_system", "coarse_initialize", "solve_problem",
    "read_tensor", "write_tensor", "read_field", "write_field", "read_mask", "write_mask",
    "export_vtk", "FormatError", "EmptyDomainError", "OutOfDomainError",
    "ConditioningWarning", "ConfigurationError", "DegreeError", "DeterminismError",
    "DivergenceError", "IndefiniteOperatorError", "NativeLibraryError", "ResourceError",
    "ValidationError",
]

__version__ = "0.1.0"
