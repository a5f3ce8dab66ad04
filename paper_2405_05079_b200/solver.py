"""Drop-in solver API of the PoVar hot path, running on the B200 through libpovar.so.

Mirrors the reference entry points on this path (pkg/src/stratba):

* ``lm_minimize``        -> solvers.py:318-393  (PoVar / PoBA stage 1, RiPoBA stage 2)
* ``power_schur_solve``  -> solvers.py:126-150  (on a device ``SchurSystem``)
* ``pcg_schur_solve``    -> solvers.py:153-187  (block-Jacobi PCG, "iterative" / "ripcg")
* ``solve_reduced``      -> solvers.py:251-260  (inner-solver dispatch: power | pcg)
* ``riemannian_step``    -> riemannian.py:125-138
* ``assemble_system``    -> normal_eq.py:62-89 + riemannian.py:67-85 + normal_eq.py:156-198
* ``total_cost``         -> objective.py:194-211
* ``solve_landmarks``    -> objective.py:251-298
* ``random_init``        -> bal_io.py:281-297

The LM state machine (accept/reject, damping schedule, convergence test,
trace records) stays in Python exactly as in the reference; every numeric
step runs in hand-written sm_100a kernels.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
import time
import weakref

import numpy as np

from . import _lib
from .types import (BOTH, JOINT, POSE_ONLY, STAGE1, STAGE2, VARPRO, BaProblem,
                    ConvergenceTrace, NumericFailureError, PoseConfig, ProjectiveState,
                    UNIT_TOL, SolverConfig, StepReport, TraceRecord, solver_label)


class DeviceProblem:
    """Device-resident observation graph + state of one landmark shard.

    ``lm_range=(begin, end)`` restricts the context to landmarks
    ``begin <= j < end`` (one rank of a sharded run); with ``world > 1`` every
    method is collective over the NCCL world given by ``nccl_id``.
    """

    def __init__(self, problem: BaProblem, eta: float = 0.1, *, device: int | None = None,
                 rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 lm_range: tuple[int, int] | None = None):
        lib = _lib.load()
        PoseConfig(eta)  # validation (objective.py:45-47)
        if device is None:
            device = _default_device()
        self.problem = problem
        self.eta = float(eta)
        self.device = int(device)
        self.rank, self.world = int(rank), int(world)
        b, e = lm_range if lm_range is not None else (0, problem.num_landmarks)
        self.lm_range = (int(b), int(e))
        ci = np.ascontiguousarray(problem.camera_indices, dtype=np.int64)
        li = np.ascontiguousarray(problem.landmark_indices, dtype=np.int64)
        m = np.ascontiguousarray(problem.measurements, dtype=np.float64)
        ctx = ctypes.c_void_p()
        rc = lib.pv_create(ctypes.byref(ctx), self.device, self.rank, self.world,
                           nccl_id, problem.num_cameras, problem.num_landmarks,
                           problem.num_observations, _lib.i64ptr(ci), _lib.i64ptr(li),
                           _lib.dptr(m), self.lm_range[0], self.lm_range[1], self.eta)
        _lib.check(rc, None)
        self._ctx = ctx
        self._lib = lib
        self._finalizer = weakref.finalize(self, lib.pv_destroy, ctx)
        info = self.info()
        self.n_p = int(info["n_p"])
        self.n_l_local = int(info["n_l_local"])
        self.n_o_local = int(info["n_o_local"])
        self._state_template = None

    # -- plumbing -----------------------------------------------------------
    def _call(self, name, *args):
        _lib.check(getattr(self._lib, name)(self._ctx, *args), self._ctx)

    def close(self):
        self._finalizer()

    def info(self) -> dict:
        out = np.zeros(_lib.PV_INFO_COUNT, dtype=np.int64)
        self._call("pv_info", _lib.i64ptr(out))
        return {k: int(out[i]) for i, k in enumerate(_lib.INFO_FIELDS)}

    def set_option(self, key: int, value: int) -> None:
        """Tuning knob of the term kernels (include/povar.h PV_OPT_*); results unchanged."""
        self._call("pv_set_option", int(key), int(value))

    @property
    def stream_handle(self) -> int:
        return int(self._lib.pv_stream(self._ctx) or 0)

    # -- state ----------------------------------------------------------------
    def set_state(self, state: ProjectiveState) -> None:
        cams = np.ascontiguousarray(state.cameras, dtype=np.float64)
        lms = np.ascontiguousarray(state.landmarks, dtype=np.float64)
        if cams.shape != (self.n_p, 3, 4) or lms.shape != (self.problem.num_landmarks, 4):
            raise ValueError("state does not match the problem")
        self._call("pv_set_state", _lib.dptr(cams), _lib.dptr(lms))
        self._state_template = lms

    def prepare_result(self) -> None:
        """Allocate the arrays the next :meth:`get_state` returns and touch their pages on a
        background thread.  ``lm_minimize`` calls this before its iterations: the first-touch
        page faults of a fresh 143 MB result (vlarge) then overlap the device work instead of
        sitting inside the download (13 -> ~6 ms, tools/time_state_io.py)."""
        import threading
        if self.n_l_local != self.problem.num_landmarks:
            return  # sharded contexts merge into a copy of the uploaded state
        cams = np.empty((self.n_p, 3, 4))
        lms = np.empty((self.problem.num_landmarks, 4))

        def touch():
            for a in (cams, lms):
                a.reshape(-1)[::512] = 0.0  # one write per 4 KB page

        th = threading.Thread(target=touch, daemon=True)
        th.start()
        self._result = (cams, lms, th)

    def get_state(self, trial: bool = False, out: ProjectiveState | None = None
                  ) -> ProjectiveState:
        """Download the (trial) state.  Landmarks this shard does not own (unobserved or
        other ranks') keep the values of the last uploaded state."""
        pre = self.__dict__.pop("_result", None)
        if pre is not None:
            cams, lms, th = pre
            th.join()
        else:
            cams = np.empty((self.n_p, 3, 4))
            if self.n_l_local == self.problem.num_landmarks:
                lms = np.empty((self.problem.num_landmarks, 4))
            else:
                lms = np.array(self._state_template, copy=True)
        self._call("pv_get_trial" if trial else "pv_get_state", _lib.dptr(cams), _lib.dptr(lms))
        return ProjectiveState(cams, lms)

    # -- numeric steps ----------------------------------------------------------
    def cost(self, stage: int, trial: bool = False) -> float:
        f = ctypes.c_double()
        self._call("pv_cost", int(stage), _lib.PV_TRIAL if trial else _lib.PV_CURRENT,
                   ctypes.byref(f))
        return f.value

    def linearize(self, stage: int) -> None:
        self._call("pv_linearize", int(stage))

    def damp(self, lam: float, both: bool) -> int:
        n = ctypes.c_int64()
        self._call("pv_damp", float(lam), int(bool(both)), ctypes.byref(n))
        return n.value

    def power_solve(self, max_order: int, threshold: float) -> tuple[int, float]:
        order, trunc = ctypes.c_int(), ctypes.c_double()
        self._call("pv_power_solve", int(max_order), float(threshold), ctypes.byref(order),
                   ctypes.byref(trunc))
        return order.value, trunc.value

    def pcg_solve(self, max_iterations: int, tolerance: float) -> tuple[int, float, str | None]:
        its, rel_res, flag = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        self._call("pv_pcg_solve", int(max_iterations), float(tolerance), ctypes.byref(its),
                   ctypes.byref(rel_res), ctypes.byref(flag))
        return its.value, rel_res.value, ("breakdown" if flag.value else None)

    def inner_solve(self, config: SolverConfig) -> tuple[int, int, float, str | None]:
        """solve_reduced (solvers.py:251-260) on the device system:
        (inner_iterations_used, power_order_used, truncation_estimate, flag)."""
        if config.inner_solver == "power":
            order, trunc = self.power_solve(config.max_power_order, config.power_threshold)
            return order, order, trunc, None
        if config.inner_solver == "pcg":
            its, rel_res, flag = self.pcg_solve(config.max_inner_iterations, config.pcg_tolerance)
            return its, 0, rel_res, flag
        raise NotImplementedError(
            f"inner_solver={config.inner_solver!r}: the GPU path runs 'power' and 'pcg'")

    def trial(self, stage: int) -> bool:
        ok = ctypes.c_int()
        self._call("pv_trial", int(stage), ctypes.byref(ok))
        return bool(ok.value)

    def accept(self, stage: int, resolve: bool) -> tuple[float, int]:
        f, n = ctypes.c_double(math.nan), ctypes.c_int64()
        self._call("pv_accept", int(stage), int(bool(resolve)), ctypes.byref(f), ctypes.byref(n))
        return f.value, n.value

    def resolve_current(self) -> int:
        n = ctypes.c_int64()
        self._call("pv_resolve_current", ctypes.byref(n))
        return n.value

    def back_substitute(self, dx: np.ndarray) -> None:
        """Device back-substitution of a given pose update on the damped system
        (normal_eq.py:239-250); the result becomes the device step (``step``, ``trial``)."""
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        self._call("pv_back_substitute", _lib.dptr(dx))

    def step(self, stage: int) -> tuple[np.ndarray, np.ndarray]:
        d = 12 if stage == STAGE1 else 11
        dx = np.zeros(self.n_p * d)
        dl = np.zeros(self.problem.num_landmarks * 3)
        self._call("pv_get_step", _lib.dptr(dx), _lib.dptr(dl))
        return dx, dl

    def schur_apply(self, stage: int, v: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        self._call("pv_schur_apply", int(stage), _lib.dptr(v), _lib.dptr(out))
        return out

    def bench_terms(self, stage: int, n_terms: int) -> dict:
        ms = (ctypes.c_float * 4)()
        self._call("pv_bench_terms", int(stage), int(n_terms), ms)
        # per term: landmark reduces and camera passes summed over every block launch
        # (events around each launch group), the block count, the whole term (no events)
        return {"lm_reduce_ms": ms[0], "cam_ms": ms[1], "blocks": int(ms[2]), "term_ms": ms[3]}

    def debug(self, which: int) -> np.ndarray:
        sizes = {_lib.PV_DBG_U: (self.n_p, 144), _lib.PV_DBG_ULIN: (self.n_p, 144),
                 _lib.PV_DBG_UINV: (self.n_p, 144), _lib.PV_DBG_BP: (self.n_p, 12),
                 _lib.PV_DBG_RHS: (self.n_p, 12), _lib.PV_DBG_X: (self.n_p, 12),
                 _lib.PV_DBG_V: (self.n_l_local, 6), _lib.PV_DBG_VPINV: (self.n_l_local, 6),
                 _lib.PV_DBG_BL: (self.n_l_local, 3), _lib.PV_DBG_DL: (self.n_l_local, 3),
                 _lib.PV_DBG_DEGEN: (self.n_l_local,), _lib.PV_DBG_W: (self.n_o_local, 36),
                 _lib.PV_DBG_SDIAG: (self.n_p, 144), _lib.PV_DBG_MINV: (self.n_p, 144)}
        out = np.zeros(sizes[which])
        self._call("pv_debug_get", int(which), _lib.dptr(out))
        return out


def _check_unit(state: ProjectiveState) -> None:
    """The tangent bases need unit vectors (riemannian.py:46-48, UNIT_TOL = riemannian.py:26).

    The device derives the Householder bases from the state itself, so this is the
    reference's check on the same vectors: every camera 12-vector, then every landmark.
    """
    for v in (state.cameras.reshape(len(state.cameras), 12), state.landmarks):
        if len(v) and np.abs(np.linalg.norm(v, axis=-1) - 1.0).max() > UNIT_TOL:
            raise ValueError("tangent basis requires unit vectors; retract first")


def _householder_bases(v: np.ndarray) -> np.ndarray:
    """The deterministic Householder complement bases (riemannian.py:37-56), (..., n, n-1)."""
    n = v.shape[-1]
    sigma = np.where(v[..., 0] >= 0, 1.0, -1.0)
    u = np.array(v, dtype=np.float64, copy=True)
    u[..., 0] += sigma
    u /= np.linalg.norm(u, axis=-1, keepdims=True)
    basis = -2.0 * u[..., :, None] * u[..., None, 1:]
    idx = np.arange(n - 1)
    basis[..., idx + 1, idx] += 1.0
    return basis


def _check_bases(state: ProjectiveState, bases) -> None:
    """Bases passed to ``riemannian_step`` must be the state's own Householder bases: the
    device applies those implicitly (h vectors, never stored) and cannot take others."""
    cams = state.cameras.reshape(len(state.cameras), 12)
    for given, v, name in ((bases.camera_bases, cams, "camera"),
                           (bases.landmark_bases, state.landmarks, "landmark")):
        given = np.asarray(given, dtype=np.float64)
        want = _householder_bases(v)
        if given.shape != want.shape or not np.allclose(given, want, rtol=0.0, atol=1e-12):
            raise ValueError(f"{name} bases differ from the Householder bases of the state "
                             "(riemannian.py:37-56), the only bases the device path applies")


def _default_device() -> int:
    import os
    return int(os.environ.get("LOCAL_RANK", "0")) if "LOCAL_RANK" in os.environ else 0


# one cached context per live problem object (BaProblem is immutable)
_CONTEXTS: dict = {}


def device_problem(problem: BaProblem, eta: float = 0.1) -> DeviceProblem:
    key = (id(problem), float(eta))
    hit = _CONTEXTS.get(key)
    if hit is not None and hit[0]() is problem:
        return hit[1]
    dp = DeviceProblem(problem, eta)
    _CONTEXTS[key] = (weakref.ref(problem, lambda _r, k=key: _CONTEXTS.pop(k, None)), dp)
    return dp


# ---------------------------------------------------------------------------
# reference-shaped API


def total_cost(state: ProjectiveState, problem: BaProblem, stage: int,
               config: PoseConfig | None = None, *, dp: DeviceProblem | None = None) -> float:
    """objective.py:194-211 on the device (+inf for a degenerate stage-2 state)."""
    if stage not in (STAGE1, STAGE2):
        raise ValueError(f"unknown stage {stage!r}")
    dp = dp or device_problem(problem, (config or PoseConfig()).eta)
    dp.set_state(state)
    return dp.cost(stage)


def solve_landmarks(state: ProjectiveState, problem: BaProblem,
                    config: PoseConfig | None = None, *, dp: DeviceProblem | None = None
                    ) -> np.ndarray:
    """Closed-form stage-1 landmarks (objective.py:251-298) on the device."""
    if problem.num_observations == 0:
        return np.array(state.landmarks, copy=True)
    dp = dp or device_problem(problem, (config or PoseConfig()).eta)
    dp.set_state(state)
    n_bad = dp.resolve_current()
    if n_bad:
        import logging
        logging.getLogger(__name__).warning(
            "left %d landmarks unchanged: rank-deficient closed-form systems", n_bad)
    return np.array(dp.get_state().landmarks)


def random_init(problem: BaProblem, seed: int, config: PoseConfig | None = None
                ) -> ProjectiveState:
    """Philox N(0,1) cameras + closed-form landmarks (bal_io.py:281-297)."""
    rng = np.random.Generator(np.random.Philox(int(seed) & 0xFFFFFFFFFFFFFFFF))
    cams = rng.standard_normal((problem.num_cameras, 3, 4))
    zero = np.zeros((problem.num_landmarks, 4))
    zero[:, 3] = 1.0
    lms = solve_landmarks(ProjectiveState(cams, zero), problem, config)
    return ProjectiveState(cams, lms)


class SchurSystem:
    """Handle on a damped block system living on the device (normal_eq.py:109-142)."""

    def __init__(self, dp: DeviceProblem, stage: int, lam: float, damping_mode: str):
        self.dp, self.stage, self.lam, self.damping_mode = dp, stage, lam, damping_mode
        self.n_degenerate = 0

    @property
    def n_cameras(self) -> int:
        return self.dp.n_p

    @property
    def pose_width(self) -> int:
        return 12 if self.stage == STAGE1 else 11

    @property
    def pose_dim(self) -> int:
        return self.n_cameras * self.pose_width


def assemble_system(problem: BaProblem, state: ProjectiveState, stage: int, lam: float,
                    damping_mode: str = POSE_ONLY, config: PoseConfig | None = None, *,
                    dp: DeviceProblem | None = None) -> SchurSystem:
    """Linearize + assemble on the device (normal_eq.py:62-89,156-198; riemannian.py:67-85)."""
    if lam < 0:
        raise ValueError("damping must be non-negative")
    if damping_mode not in (POSE_ONLY, BOTH):
        raise ValueError(f"unknown damping mode {damping_mode!r}")
    dp = dp or device_problem(problem, (config or PoseConfig()).eta)
    dp.set_state(state)
    dp.linearize(stage)
    sysm = SchurSystem(dp, stage, lam, damping_mode)
    sysm.n_degenerate = dp.damp(lam, damping_mode == BOTH)
    return sysm


def power_schur_solve(system: SchurSystem, config: SolverConfig) -> StepReport:
    """solvers.py:126-150 on a device system; returns host update vectors."""
    order, trunc = system.dp.power_solve(config.max_power_order, config.power_threshold)
    dx, dl = system.dp.step(system.stage)
    return StepReport(dx, dl, order, order, trunc)


def back_substitute(system: SchurSystem, pose_update: np.ndarray) -> np.ndarray:
    """normal_eq.py:239-250 on a device system: -V^+(b_l + W^T dx_p), zero for degenerate
    landmark blocks; (n_landmarks * 3,) like the reference."""
    pose_update = np.asarray(pose_update, dtype=np.float64).ravel()
    if pose_update.size != system.pose_dim:
        raise ValueError("pose update does not match the system")
    system.dp.back_substitute(pose_update)
    return system.dp.step(system.stage)[1]


def pcg_schur_solve(system: SchurSystem, config: SolverConfig) -> StepReport:
    """solvers.py:153-187 on a device system (block-Jacobi PCG, exact diagonal blocks)."""
    its, rel_res, flag = system.dp.pcg_solve(config.max_inner_iterations, config.pcg_tolerance)
    dx, dl = system.dp.step(system.stage)
    return StepReport(dx, dl, its, 0, rel_res, flag)


def spectral_check(system: SchurSystem, max_iterations: int = 50000, tol: float = 1e-14
                   ) -> float:
    """Largest eigenvalue of U^-1 W V^+ W^T by power iteration (solvers.py:263-295).

    Same algorithm as the reference: the symmetrized similar operator
    U^-1/2 W V^+ W^T U^-1/2, started from the normalized ones vector, stopped when
    the Rayleigh quotient moves by <= tol * max(1, |mu|).  Each application runs the
    coupling round trip W V^+ W^T on the device (the power-series term kernels,
    ``pv_schur_apply``); the per-camera U^-1/2 blocks (eigh of the damped U blocks,
    12x12 or 11x11) are applied on the host.  A property check for small systems.
    """
    dp, d, n = system.dp, system.pose_width, system.n_cameras
    U = dp.debug(_lib.PV_DBG_U).reshape(n, 12, 12)[:, :d, :d]
    w, q = np.linalg.eigh(U)
    if (w <= 0).any():
        raise ValueError("pose blocks must be positive-definite")
    uih = np.einsum("nij,nj,nkj->nik", q, 1.0 / np.sqrt(w), q)

    def half(v):
        return np.einsum("nij,nj->ni", uih, v.reshape(n, d)).ravel()

    dim = system.pose_dim
    v = np.full(dim, 1.0 / math.sqrt(dim))
    mu = 0.0
    for _ in range(max_iterations):
        av = half(dp.schur_apply(system.stage, half(v)))
        nrm = np.linalg.norm(av)
        if nrm == 0:
            return 0.0
        mu_new = float(v @ av)
        v = av / nrm
        if abs(mu_new - mu) <= tol * max(1.0, abs(mu_new)):
            return mu_new
        mu = mu_new
    return mu


_INNER_SOLVERS = {"power": power_schur_solve, "pcg": pcg_schur_solve}


def solve_reduced(system: SchurSystem, config: SolverConfig) -> StepReport:
    """Inner-solver dispatch (solvers.py:251-260).  ``direct`` (a sparse LU of the
    materialised reduced matrix) is not part of the GPU path."""
    fn = _INNER_SOLVERS.get(config.inner_solver)
    if fn is None:
        raise NotImplementedError(
            f"inner_solver={config.inner_solver!r}: the GPU path runs 'power' and 'pcg'")
    return fn(system, config)


def riemannian_step(problem: BaProblem, state: ProjectiveState, config: SolverConfig,
                    lam: float | None = None, bases=None, *, dp: DeviceProblem | None = None
                    ) -> StepReport:
    """riemannian.py:125-138: tangent-space reduced solve (11 per camera, 3 per landmark).

    The device derives the Householder bases (riemannian.py:37-56) from ``state``; as in
    the reference, a state off the unit spheres raises ``ValueError`` when no bases are
    given, and given ``bases`` must be those of ``state`` (checked on the host).
    """
    if lam is None:
        lam = config.initial_lambda
    if bases is None:
        _check_unit(state)
    else:
        _check_bases(state, bases)
    system = assemble_system(problem, state, STAGE2, lam, BOTH, config.pose, dp=dp)
    return solve_reduced(system, config)


def lm_minimize(problem: BaProblem, state: ProjectiveState, stage: int, config: SolverConfig,
                trace_sink=None, *, solver_id: str | None = None, problem_id: str = "",
                dp: DeviceProblem | None = None, decisions: list | None = None
                ) -> tuple[ProjectiveState, ConvergenceTrace]:
    """Levenberg-Marquardt outer loop (solvers.py:318-393) over device steps.

    Same accept rule (strict decrease), damping schedule, convergence test and
    trace records as the reference.  A rejected step leaves the state
    unchanged, so the linearization is reused (results-identical, SURVEY
    App. A.6).  ``decisions`` (optional list) receives one dict per iteration
    (lam, f_trial, accepted, power order) for parity checks.
    """
    if stage not in (STAGE1, STAGE2):
        raise ValueError(f"unknown stage {stage!r}")
    if config.inner_solver not in _INNER_SOLVERS:
        raise NotImplementedError(
            f"inner_solver={config.inner_solver!r}: the GPU path runs 'power' and 'pcg'")
    pose = config.pose
    dp = dp or device_problem(problem, pose.eta)
    dp.set_state(state)
    f = dp.cost(stage)
    if not math.isfinite(f):
        raise NumericFailureError(f"stage {stage} starting cost is not finite")
    dp.prepare_result()  # the result arrays' pages are touched while the device iterates
    label = solver_id if solver_id is not None else solver_label(stage, config)
    stage_name = "stage1" if stage == STAGE1 else "stage2"
    varpro = config.mode == VARPRO
    both = stage == STAGE2 or not varpro
    t0 = time.perf_counter()
    records = [TraceRecord(0, f, 0.0)]
    if trace_sink is not None:
        trace_sink(records[0])
    lam = config.initial_lambda
    linearized = False
    for it in range(1, config.max_outer_iterations + 1):
        if stage == STAGE2 and it == 1:
            # state_tangent_bases of the start (solvers.py:358-359): later states are
            # retracted trials, unit by construction
            _check_unit(state)
        if not linearized:
            dp.linearize(stage)  # FloatingPointError on a degenerate stage-2 point
            linearized = True
        dp.damp(lam, both)
        its, order, _trunc, _flag = dp.inner_solve(config)
        ok = dp.trial(stage)
        f_trial = dp.cost(stage, trial=True) if ok else math.inf
        converged = False
        accepted = f_trial < f
        if accepted:
            if stage == STAGE1 and varpro:
                f_trial, _ = dp.accept(stage, resolve=True)
            else:
                dp.accept(stage, resolve=False)
            linearized = False
            converged = abs(f - f_trial) / (f if f > 0 else 1.0) <= config.function_tolerance
            f = f_trial
            lam = max(config.lambda_min, lam * config.lambda_decrease)
        else:
            if math.isfinite(f_trial):
                converged = abs(f - f_trial) / (f if f > 0 else 1.0) <= config.function_tolerance
            lam = min(config.lambda_max, lam * config.lambda_increase)
        if decisions is not None:
            decisions.append(dict(iteration=it, f_trial=f_trial, accepted=accepted, order=order,
                                  inner_iterations=its, lam_next=lam))
        rec = TraceRecord(it, f, time.perf_counter() - t0)
        records.append(rec)
        if trace_sink is not None:
            trace_sink(rec)
        if converged:
            break
    final = dp.get_state()
    return final, ConvergenceTrace(label, problem_id, stage_name, records, records[0].cost)
