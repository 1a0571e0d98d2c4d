"""B200-native per-timestep quasi-Newton / L-BFGS hyperelastic solver
(arXiv 1604.07378), drop-in for the hot path of the reference package `qnsim`.

The public names mirror `qnsim.__all__` (pkg/src/qnsim/__init__.py:15-34).
Compute runs in `libqnsim_b200.so` (hand-written sm_100a CUDA + host C++)
through the C-ABI in include/qnsim_b200.h; there is no CPU fallback.
"""

from paper_1604_07378_b200.linalg import (
    Factorization,
    FactorizationError,
    RotVarSVD,
    factorize_spd,
    solve_prefactored,
    svd_rv,
    svd_rv_batch,
)
from paper_1604_07378_b200.mesh import (SpringNetwork, TetMesh, bar_mesh, grid_bar, load_obj_springs, load_tet_mesh,
                                        lumped_masses, tet_diff_operators)
from paper_1604_07378_b200.materials import (
    FitInterval,
    HermiteFn,
    LogFn,
    MaterialError,
    MaterialModel,
    PolyFn,
    ZeroFn,
    estimate_stiffness,
    make_builtin,
    vl_energy_batch,
    vl_stress_batch,
)
from paper_1604_07378_b200.dynamics import (
    DynamicsError,
    SimState,
    SimSystem,
    VLGroup,
    build_batch_system,
    build_system,
    gradient,
    inertia_target,
    objective,
)
from paper_1604_07378_b200.solvers import (
    ConvergenceRecord,
    ResidentRun,
    SolverConfig,
    SolverError,
    StagnationError,
    relative_error,
    direction_newton,
    newton_reference,
    simulate_frame,
)

__all__ = [
    "Factorization", "FactorizationError", "RotVarSVD", "factorize_spd", "solve_prefactored", "svd_rv",
    "svd_rv_batch", "SpringNetwork", "load_obj_springs", "TetMesh", "bar_mesh", "grid_bar", "load_tet_mesh", "lumped_masses", "tet_diff_operators",
    "FitInterval", "HermiteFn", "LogFn", "MaterialError", "MaterialModel", "PolyFn", "ZeroFn",
    "estimate_stiffness", "make_builtin", "vl_energy_batch", "vl_stress_batch", "DynamicsError", "SimState",
    "SimSystem", "VLGroup", "build_batch_system", "build_system", "gradient", "inertia_target", "objective",
    "ConvergenceRecord", "ResidentRun", "SolverConfig", "SolverError", "StagnationError", "relative_error",
    "simulate_frame", "direction_newton", "newton_reference",
]
