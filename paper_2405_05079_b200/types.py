"""Host-side data types of the PoVar hot path, mirroring the reference API.

The drop-in keeps the reference package's public types so that callers of
``stratba.lm_minimize`` can switch without code changes.  Each type here states
the reference definition it mirrors; field names, defaults, validation and
error classes follow the reference exactly.

* ``BaProblem`` / ``ProjectiveState``  -> pkg/src/stratba/bal_io.py:53-112
* ``PoseConfig``                       -> pkg/src/stratba/objective.py:39-47
* ``SolverConfig`` / ``StepReport``    -> pkg/src/stratba/solvers.py:60-105
* ``TraceRecord`` / ``ConvergenceTrace`` -> pkg/src/stratba/evaluation.py:33-59
* error classes                        -> solvers.py:56-57, objective.py:60-61
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import NamedTuple

import numpy as np

STAGE1 = 1
STAGE2 = 2

VARPRO = "varpro"
JOINT = "joint"

POSE_ONLY = "pose_only"
BOTH = "both"

# objective.py:33 -- |z| at or below this makes a stage-2 projection degenerate.
Z_EPSILON = 1e-12
# normal_eq.py:34-36 -- Jacobi damping clamp and landmark pseudo-inverse cutoff.
DAMPING_CLAMP = (1e-6, 1e6)
V_PINV_TOL = 1e-10
# objective.py:284-292 -- relative singular-value cutoff of the landmark re-solve.
RESOLVE_SVD_TOL = 1e-10
# riemannian.py:26 -- unit-norm tolerance of the tangent basis.
UNIT_TOL = 1e-9


class NumericFailureError(RuntimeError):
    """A stage could not start: the initial cost is not finite (solvers.py:56-57)."""


class ProjectionDegenerateError(ValueError):
    """Perspective division with |z| <= Z_EPSILON (objective.py:60-61)."""


def _readonly(a, dtype=np.float64) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=dtype)
    out.setflags(write=False)
    return out


@dataclass(frozen=True)
class BaProblem:
    """Immutable observation graph (bal_io.py:53-92)."""

    num_cameras: int
    num_landmarks: int
    num_observations: int
    camera_indices: np.ndarray  # (n_obs,) int64
    landmark_indices: np.ndarray  # (n_obs,) int64
    measurements: np.ndarray  # (n_obs, 2) float64
    metric_cameras: np.ndarray | None = None
    metric_points: np.ndarray | None = None

    def __post_init__(self):
        object.__setattr__(self, "camera_indices", _readonly(self.camera_indices, np.int64))
        object.__setattr__(self, "landmark_indices", _readonly(self.landmark_indices, np.int64))
        object.__setattr__(self, "measurements", _readonly(self.measurements))
        if self.metric_cameras is not None:
            object.__setattr__(self, "metric_cameras", _readonly(self.metric_cameras))
        if self.metric_points is not None:
            object.__setattr__(self, "metric_points", _readonly(self.metric_points))
        n = self.num_observations
        if len(self.camera_indices) != n or len(self.landmark_indices) != n:
            raise ValueError("observation count does not match index arrays")
        if self.measurements.shape != (n, 2):
            raise ValueError("measurement array must be (num_observations, 2)")
        if n:
            ci, li = self.camera_indices, self.landmark_indices
            if ci.min() < 0 or ci.max() >= self.num_cameras:
                raise ValueError("camera index out of range")
            if li.min() < 0 or li.max() >= self.num_landmarks:
                raise ValueError("landmark index out of range")


@dataclass(frozen=True)
class ProjectiveState:
    """Cameras (n_p, 3, 4) and homogeneous landmarks (n_l, 4) (bal_io.py:95-112)."""

    cameras: np.ndarray
    landmarks: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "cameras", _readonly(self.cameras))
        object.__setattr__(self, "landmarks", _readonly(self.landmarks))
        if self.cameras.ndim != 3 or self.cameras.shape[1:] != (3, 4):
            raise ValueError("cameras must be (n, 3, 4)")
        if self.landmarks.ndim != 2 or self.landmarks.shape[1] != 4:
            raise ValueError("landmarks must be (n, 4)")


@dataclass(frozen=True)
class PoseConfig:
    """pOSE blend weight eta in [0, 1] (objective.py:39-47)."""

    eta: float = 0.1

    def __post_init__(self):
        if not 0.0 <= self.eta <= 1.0:
            raise ValueError(f"eta must lie in [0, 1], got {self.eta}")


@dataclass(frozen=True)
class SolverConfig:
    """Outer-loop and inner-solver settings (solvers.py:60-93); paper defaults."""

    max_outer_iterations: int = 50
    function_tolerance: float = 1e-6
    initial_lambda: float = 1e-4
    max_power_order: int = 20
    power_threshold: float = 0.01
    max_inner_iterations: int = 500
    inner_solver: str = "power"  # power | pcg | direct
    mode: str = VARPRO  # varpro | joint
    pcg_tolerance: float = 1e-6
    lambda_increase: float = 4.0
    lambda_decrease: float = 0.5
    lambda_min: float = 1e-12
    lambda_max: float = 1e8
    pose: PoseConfig = field(default_factory=PoseConfig)

    def __post_init__(self):
        if self.inner_solver not in ("power", "pcg", "direct"):
            raise ValueError(f"unknown inner solver {self.inner_solver!r}")
        if self.mode not in (VARPRO, JOINT):
            raise ValueError(f"unknown mode {self.mode!r}")
        positive = ("max_outer_iterations", "function_tolerance", "initial_lambda",
                    "max_inner_iterations", "pcg_tolerance", "lambda_increase",
                    "lambda_decrease", "lambda_min", "lambda_max")
        for name in positive:
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.max_power_order < 0 or self.power_threshold < 0:
            raise ValueError("power series settings must be non-negative")


@dataclass
class StepReport:
    """One inner solve (solvers.py:96-105)."""

    pose_update: np.ndarray
    landmark_update: np.ndarray
    inner_iterations_used: int
    power_order_used: int
    truncation_estimate: float
    flag: str | None = None


class TraceRecord(NamedTuple):
    """(iteration, cost, cumulative seconds) (evaluation.py:33-36)."""

    iteration: int
    cost: float
    elapsed_seconds: float


@dataclass
class ConvergenceTrace:
    """Per-iteration records of one run (evaluation.py:39-59)."""

    solver_id: str
    problem_id: str
    stage: str
    records: list
    initial_cost: float

    def __post_init__(self):
        if not self.records:
            raise ValueError("a trace needs at least one record")
        if self.records[0].cost != self.initial_cost:
            raise ValueError("first record must carry the initial cost")
        t = [r.elapsed_seconds for r in self.records]
        if any(b < a for a, b in zip(t, t[1:])):
            raise ValueError("elapsed seconds must be non-decreasing")

    def best_cost(self) -> float:
        return min(r.cost for r in self.records)

    def final_cost(self) -> float:
        return self.records[-1].cost


def solver_label(stage: int, config: SolverConfig) -> str:
    """Trace solver names (solvers.py:298-308)."""
    if stage == STAGE1:
        names = {(VARPRO, "power"): "povar", (JOINT, "power"): "poba",
                 (VARPRO, "pcg"): "iterative", (VARPRO, "direct"): "direct"}
        return names.get((config.mode, config.inner_solver),
                         f"{config.mode}-{config.inner_solver}")
    return {"power": "ripoba", "pcg": "ripcg"}.get(config.inner_solver,
                                                  f"riemannian-{config.inner_solver}")


def is_finite(x: float) -> bool:
    return math.isfinite(x)
