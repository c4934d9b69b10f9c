"""B200-native batched-Phi MGRIT-FAS for the 2D magnetoquasistatic model.

The reference (arxiv 1912.03106, package `pintmg`) advances every C-interval
of an MGRIT level one implicit-Euler step at a time; here the F-offset of all
owned intervals is one batched fp64 solve on the GPU (libpintgpu, sm_100a),
behind the reference's own problem / solver API:

    from paper_1912_03106_b200 import (GpuFemProblem, TimeHierarchy,
        build_uniform_grid, CycleSpec, StoppingCriterion, mgrit_solve, configs)

    spec = configs.config1()
    problem = GpuFemProblem(spec)
    grid = build_uniform_grid(0.0, 0.02, spec["n_steps"])
    run, sol = mgrit_solve(problem, TimeHierarchy.build(grid, [16]),
                           CycleSpec(kind="V", gamma=1),
                           StoppingCriterion(tolerance=1e-7))

See DESIGN.md for the data layout, kernels and rooflines.
"""

from . import configs
from .dropin import (GpuOperatorProblem, OperatorLevel, ReferenceProblemAdapter,
                     reference_1d_levels)
from .errors import InnerSolveError, NewtonConvergenceError, PintGpuError, TransportError
from .excitation import Excitation
from .mgrit import (CycleSpec, MgritSolver, SolverRun, StoppingCriterion,
                    StorageReport, mgrit_solve, qoi_change, sequential_solve,
                    storage_estimate)
from .problem import GpuFemProblem, GpuSurrogateProblem, StepDiagnostics, make_problem
from .runtime import Decomposition, DistTransport, NullTransport
from .spatial import SpatialHierarchy2D, assign_spatial_levels
from .state import BlockState, SpaceTimeVector
from .time_hierarchy import (CFSplitting, TimeGrid, TimeHierarchy,
                             build_uniform_grid, plan_coarsening)

__version__ = "0.1.0"

__all__ = [
    "BlockState", "CFSplitting", "CycleSpec", "Decomposition", "DistTransport",
    "Excitation", "GpuFemProblem", "GpuOperatorProblem", "GpuSurrogateProblem", "InnerSolveError", "make_problem",
    "MgritSolver", "NewtonConvergenceError",
    "NullTransport", "OperatorLevel", "PintGpuError", "ReferenceProblemAdapter", "SolverRun", "SpaceTimeVector",
    "SpatialHierarchy2D", "StepDiagnostics", "StoppingCriterion", "StorageReport",
    "TimeGrid", "TimeHierarchy", "TransportError", "assign_spatial_levels",
    "build_uniform_grid", "configs", "mgrit_solve", "plan_coarsening",
    "qoi_change", "reference_1d_levels", "sequential_solve", "storage_estimate",
]
