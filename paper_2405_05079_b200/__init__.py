"""B200-native PoVar / RiPoBA hot path (arXiv 2405.05079), drop-in for stratba's solver API.

Public names follow the reference package (pkg/src/stratba/__init__.py:3-68)
for the part of the API this path covers.
"""

from .types import (BOTH, JOINT, POSE_ONLY, STAGE1, STAGE2, VARPRO, BaProblem, ConvergenceTrace,
                    NumericFailureError, PoseConfig, ProjectionDegenerateError, ProjectiveState,
                    SolverConfig, StepReport, TraceRecord, solver_label)
from .solver import (DeviceProblem, SchurSystem, assemble_system, back_substitute, lm_minimize,
                     pcg_schur_solve,
                     power_schur_solve, random_init, riemannian_step, solve_landmarks,
                     solve_reduced, spectral_check, total_cost)
from .riemann import lift_stage1_to_stage2, retract

__version__ = "0.1.0"
