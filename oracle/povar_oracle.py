"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's PoVar / RiPoBA hot path
(``/root/reference/pkg/src/stratba``), organised around a landmark-CSR
observation order instead of the reference's per-track-length block groups.
It is the checker for the CUDA path: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm may
import it.  The product path (``paper_2405_05079_b200``) never imports it.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference package in
the build container and stores its outputs as fixtures under ``tests/golden``;
``tests/test_oracle.py`` checks this module against them.  Numerics are
NumPy 2.3 / OpenBLAS (eigh, svd, inv), the same libraries the reference
calls.

Every function cites the reference code it restates (file:line relative to
``pkg/src/stratba``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

Z_EPS = 1e-12  # objective.py:33
CLAMP_LO, CLAMP_HI = 1e-6, 1e6  # normal_eq.py:34
PINV_TOL = 1e-10  # normal_eq.py:36
SVD_TOL = 1e-10  # objective.py:284-292


# ---------------------------------------------------------------------------
# observation graph in landmark-CSR order


@dataclass
class Graph:
    """Landmark-major, camera-ascending observation order (objective.py:237-248).

    ``perm`` maps CSR position -> original observation index; ``lm`` is the
    landmark of each CSR row; ``offsets[j]:offsets[j+1]`` are the rows of
    landmark ``j`` (empty for unobserved landmarks).  ``cam_perm`` sorts the
    CSR rows by camera (stable) for per-camera segment sums.
    """

    n_cameras: int
    n_landmarks: int
    perm: np.ndarray
    cam: np.ndarray
    lm: np.ndarray
    meas: np.ndarray
    offsets: np.ndarray
    cam_perm: np.ndarray
    cam_offsets: np.ndarray
    orig_cam: np.ndarray
    orig_lm: np.ndarray
    orig_meas: np.ndarray

    @property
    def n_obs(self) -> int:
        return len(self.cam)


def make_graph(n_cameras, n_landmarks, cam_idx, lm_idx, meas) -> Graph:
    cam_idx = np.asarray(cam_idx, dtype=np.int64)
    lm_idx = np.asarray(lm_idx, dtype=np.int64)
    meas = np.asarray(meas, dtype=np.float64).reshape(-1, 2)
    perm = np.lexsort((cam_idx, lm_idx))
    cam, lm = cam_idx[perm], lm_idx[perm]
    counts = np.bincount(lm, minlength=n_landmarks)
    offsets = np.zeros(n_landmarks + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    cam_perm = np.argsort(cam, kind="stable")
    ccounts = np.bincount(cam, minlength=n_cameras)
    cam_offsets = np.zeros(n_cameras + 1, dtype=np.int64)
    np.cumsum(ccounts, out=cam_offsets[1:])
    return Graph(n_cameras, n_landmarks, perm, cam, lm, meas[perm], offsets, cam_perm,
                 cam_offsets, cam_idx, lm_idx, meas)


def graph_of(problem) -> Graph:
    return make_graph(problem.num_cameras, problem.num_landmarks, problem.camera_indices,
                      problem.landmark_indices, problem.measurements)


def _seg_sum_lm(g: Graph, rows: np.ndarray) -> np.ndarray:
    """Per-landmark sums over contiguous CSR segments (zeros for empty ones)."""
    out = np.zeros((g.n_landmarks,) + rows.shape[1:])
    if g.n_obs == 0:
        return out
    counts = np.diff(g.offsets)
    nz = counts > 0
    out[nz] = np.add.reduceat(rows, g.offsets[:-1][nz], axis=0)
    return out


def _seg_sum_cam(g: Graph, rows: np.ndarray) -> np.ndarray:
    out = np.zeros((g.n_cameras,) + rows.shape[1:])
    if g.n_obs == 0:
        return out
    counts = np.diff(g.cam_offsets)
    nz = counts > 0
    out[nz] = np.add.reduceat(rows[g.cam_perm], g.cam_offsets[:-1][nz], axis=0)
    return out


# ---------------------------------------------------------------------------
# residual rows and Jacobians


def pose_rows(P: np.ndarray, X: np.ndarray, m: np.ndarray, eta: float):
    """Stage-1 pOSE rows: r (n,4), J_p (n,4,12), J_l (n,4,3).

    objective.py:68-82 (residual) and :85-110 (Jacobians); camera vec index is
    4*row + col (row-major 3x4).
    """
    a, b = math.sqrt(1.0 - eta), math.sqrt(eta)
    u = np.einsum("nij,nj->ni", P, X)
    r = np.empty((len(P), 4))
    r[:, 0:2] = a * (u[:, 0:2] - u[:, 2:3] * m)
    r[:, 2:4] = b * (u[:, 0:2] - m)
    jp = np.zeros((len(P), 4, 12))
    jp[:, 0, 0:4] = a * X
    jp[:, 1, 4:8] = a * X
    jp[:, 0, 8:12] = -a * m[:, 0:1] * X
    jp[:, 1, 8:12] = -a * m[:, 1:2] * X
    jp[:, 2, 0:4] = b * X
    jp[:, 3, 4:8] = b * X
    p0, p1, p2 = P[:, 0, :3], P[:, 1, :3], P[:, 2, :3]
    jl = np.stack([a * (p0 - m[:, 0:1] * p2), a * (p1 - m[:, 1:2] * p2), b * p0, b * p1], axis=1)
    return r, jp, jl


def proj_rows(P: np.ndarray, X: np.ndarray, m: np.ndarray):
    """Stage-2 reprojection rows: r (n,2), J_p (n,2,12), J_l (n,2,4), valid (n,).

    objective.py:117-125 (residual) and :128-146 (Jacobians).
    """
    u = np.einsum("nij,nj->ni", P, X)
    valid = np.abs(u[:, 2]) > Z_EPS
    z = np.where(valid, u[:, 2], 1.0)
    iz = 1.0 / z
    r = u[:, 0:2] / z[:, None] - m
    d = np.zeros((len(P), 2, 3))
    d[:, 0, 0] = iz
    d[:, 1, 1] = iz
    d[:, 0, 2] = -u[:, 0] * iz ** 2
    d[:, 1, 2] = -u[:, 1] * iz ** 2
    jl = np.einsum("nrc,ncj->nrj", d, P)
    jp = (d[:, :, :, None] * X[:, None, None, :]).reshape(len(P), 2, 12)
    return r, jp, jl, valid


def total_cost(g: Graph, cams: np.ndarray, lms: np.ndarray, stage: int, eta: float = 0.1
               ) -> float:
    """Sum of squared residuals in original observation order (objective.py:194-211)."""
    P = cams[g.orig_cam]
    X = lms[g.orig_lm]
    if stage == 1:
        r = pose_rows(P, X, g.orig_meas, eta)[0]
    else:
        r, _, _, valid = proj_rows(P, X, g.orig_meas)
        if not valid.all():
            return math.inf
    return float(np.sum(r * r))


# ---------------------------------------------------------------------------
# closed-form landmark re-solve


def resolve_landmarks(g: Graph, cams: np.ndarray, lms: np.ndarray, eta: float = 0.1
                      ) -> tuple[np.ndarray, int]:
    """Per-landmark min-norm least squares via SVD (objective.py:251-298).

    Returns the new (n_l, 4) landmarks and the count of rank-deficient
    (unchanged) observed landmarks.
    """
    out = np.array(lms, copy=True)
    if g.n_obs == 0:
        return out, 0
    P = cams[g.cam]
    e3 = np.zeros((g.n_obs, 4))
    e3[:, 3] = 1.0
    c_rows, _, a_rows = pose_rows(P, e3, g.meas, eta)
    counts = np.diff(g.offsets)
    n_bad = 0
    for k in np.unique(counts[counts > 0]):
        sel = np.nonzero(counts == k)[0]
        idx = g.offsets[sel][:, None] + np.arange(k)[None, :]
        A = a_rows[idx].reshape(len(sel), 4 * k, 3)
        c = c_rows[idx].reshape(len(sel), 4 * k)
        U, s, Vt = np.linalg.svd(A, full_matrices=False)
        keep = s > SVD_TOL * s[:, :1]
        s_inv = np.where(keep, 1.0 / np.where(keep, s, 1.0), 0.0)
        coef = np.einsum("gki,gk->gi", U, c) * s_inv
        v = -np.einsum("gij,gi->gj", Vt, coef)
        full = keep.all(axis=1) & (s[:, 0] > 0)
        n_bad += int((~full).sum())
        tgt = sel[full]
        out[tgt, :3] = v[full]
        out[tgt, 3] = 1.0
    return out, n_bad


# ---------------------------------------------------------------------------
# tangent bases (stage 2)


def householder_basis(v: np.ndarray) -> np.ndarray:
    """Trailing n-1 columns of the Householder reflector of unit v (riemannian.py:37-56)."""
    v = np.asarray(v, dtype=float)
    if np.abs(np.linalg.norm(v, axis=-1) - 1.0).max(initial=0.0) > 1e-9:
        raise ValueError("tangent basis requires unit vectors; retract first")
    n = v.shape[-1]
    sgn = np.where(v[..., 0] >= 0, 1.0, -1.0)
    h = v.copy()
    h[..., 0] += sgn
    h /= np.linalg.norm(h, axis=-1, keepdims=True)
    B = -2.0 * h[..., :, None] * h[..., None, 1:]
    i = np.arange(n - 1)
    B[..., i + 1, i] += 1.0
    return B


# ---------------------------------------------------------------------------
# linearization and the damped block system


@dataclass
class Linearization:
    """Per-CSR-row Jacobian bands and residuals (projected in stage 2)."""

    jp: np.ndarray  # (n, rows, d_p)
    jl: np.ndarray  # (n, rows, d_l)
    r: np.ndarray  # (n, rows)
    cam_bases: np.ndarray | None = None  # (n_p, 12, 11) stage 2
    lm_bases: np.ndarray | None = None  # (n_l, 4, 3) stage 2


def linearize(g: Graph, cams: np.ndarray, lms: np.ndarray, stage: int, eta: float = 0.1
              ) -> Linearization:
    """build_stage1_blocks / build_stage2_blocks + project_blocks in CSR order.

    normal_eq.py:62-89 and riemannian.py:59-85.  Stage 2 raises
    FloatingPointError on any |z| <= 1e-12 (normal_eq.py:86-87).
    """
    P = cams[g.cam]
    X = lms[g.lm]
    if stage == 1:
        r, jp, jl = pose_rows(P, X, g.meas, eta)
        return Linearization(jp, jl, r)
    r, jp, jl, valid = proj_rows(P, X, g.meas)
    if not valid.all():
        raise FloatingPointError("degenerate projection while linearizing stage 2")
    cb = householder_basis(cams.reshape(-1, 12))
    lb = householder_basis(lms)
    jp = np.einsum("nri,nij->nrj", jp, cb[g.cam])
    jl = np.einsum("nri,nij->nrj", jl, lb[g.lm])
    return Linearization(jp, jl, r, cb, lb)


@dataclass
class BlockSystem:
    """Damped U, V, V+, W (per CSR row), b_p, b_l (normal_eq.py:109-142)."""

    g: Graph
    U: np.ndarray
    V: np.ndarray
    V_pinv: np.ndarray
    degenerate: np.ndarray
    W: np.ndarray  # (n_obs, d_p, d_l) in CSR order
    b_p: np.ndarray
    b_l: np.ndarray
    lam: float
    both: bool
    U_raw: np.ndarray = field(default=None)
    V_raw: np.ndarray = field(default=None)

    @property
    def d_p(self) -> int:
        return self.U.shape[1]


def jacobi_damp(blocks: np.ndarray, lam: float) -> np.ndarray:
    """D += lam * clip(sqrt(diag), 1e-6, 1e6)^2 on every block (normal_eq.py:182-192)."""
    out = blocks.copy()
    d = np.einsum("nii->ni", blocks)
    np.einsum("nii->ni", out)[...] += lam * np.clip(np.sqrt(d), CLAMP_LO, CLAMP_HI) ** 2
    return out


def pinv_psd(V: np.ndarray, rel_tol: float = PINV_TOL):
    """eigh pseudo-inverse, dropping w <= rel_tol*max(trace,0) (normal_eq.py:145-153)."""
    w, Q = np.linalg.eigh(V)
    tol = rel_tol * np.maximum(np.trace(V, axis1=1, axis2=2), 0.0)
    keep = w > tol[:, None]
    wi = np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)
    return np.einsum("nij,nj,nkj->nik", Q, wi, Q), ~keep.all(axis=1)


def assemble(g: Graph, lin: Linearization, lam: float, both: bool) -> BlockSystem:
    """U = sum Jp^T Jp, V = sum Jl^T Jl, W = Jp^T Jl, b = J^T r; damping; V+.

    normal_eq.py:156-198.
    """
    if lam < 0:
        raise ValueError("damping must be non-negative")
    U_raw = _seg_sum_cam(g, np.einsum("nri,nrj->nij", lin.jp, lin.jp))
    b_p = _seg_sum_cam(g, np.einsum("nri,nr->ni", lin.jp, lin.r))
    V_raw = _seg_sum_lm(g, np.einsum("nri,nrj->nij", lin.jl, lin.jl))
    b_l = _seg_sum_lm(g, np.einsum("nri,nr->ni", lin.jl, lin.r))
    W = np.einsum("nri,nrj->nij", lin.jp, lin.jl)
    U = jacobi_damp(U_raw, lam)
    V = jacobi_damp(V_raw, lam) if both else V_raw
    Vp, degen = pinv_psd(V)
    return BlockSystem(g, U, V, Vp, degen, W, b_p, b_l, lam, both, U_raw, V_raw)


# ---------------------------------------------------------------------------
# reduced system operators and the power series


def w_transpose_apply(s: BlockSystem, v: np.ndarray) -> np.ndarray:
    """Per-landmark sum_i W_ij^T v_i (normal_eq.py:205-211 before V+)."""
    vb = v.reshape(s.g.n_cameras, -1)
    return _seg_sum_lm(s.g, np.einsum("nij,ni->nj", s.W, vb[s.g.cam]))


def w_apply(s: BlockSystem, t: np.ndarray) -> np.ndarray:
    """Per-camera sum_j W_ij t_j (normal_eq.py:214-218)."""
    return _seg_sum_cam(s.g, np.einsum("nij,nj->ni", s.W, t[s.g.lm]))


def coupling(s: BlockSystem, v: np.ndarray) -> np.ndarray:
    """S'.v = W V+ W^T v, flattened (solvers.py:117-123)."""
    t = np.einsum("nij,nj->ni", s.V_pinv, w_transpose_apply(s, v))
    return w_apply(s, t).ravel()


def schur_rhs(s: BlockSystem) -> np.ndarray:
    """-(b_p - W V+ b_l) (normal_eq.py:221-226)."""
    t = np.einsum("nij,nj->ni", s.V_pinv, s.b_l)
    return -(s.b_p - w_apply(s, t)).ravel()


def apply_schur(s: BlockSystem, x: np.ndarray) -> np.ndarray:
    """(U - W V+ W^T) x (normal_eq.py:229-236)."""
    xb = x.reshape(s.g.n_cameras, -1)
    return (np.einsum("nij,nj->ni", s.U, xb).ravel() - coupling(s, x))


def back_substitute(s: BlockSystem, x: np.ndarray) -> np.ndarray:
    """-V+(b_l + W^T x), degenerate landmarks zeroed (normal_eq.py:239-250)."""
    upd = -np.einsum("nij,nj->ni", s.V_pinv, s.b_l + w_transpose_apply(s, x))
    upd[s.degenerate] = 0.0
    return upd.ravel()


@dataclass
class PowerResult:
    pose_update: np.ndarray
    landmark_update: np.ndarray
    order_used: int
    truncation: float
    rhs: np.ndarray
    terms: list


def power_solve(s: BlockSystem, max_order: int, threshold: float,
                keep_terms: bool = False) -> PowerResult:
    """Truncated power series x = sum_i (U^-1 S')^i U^-1 rhs (solvers.py:126-150)."""
    rhs = schur_rhs(s)
    Ui = np.linalg.inv(s.U)
    n = s.g.n_cameras

    def uapply(v):
        return np.einsum("nij,nj->ni", Ui, v.reshape(n, -1)).ravel()

    t = uapply(rhs)
    x = t.copy()
    terms = [t.copy()] if keep_terms else []
    order = 0
    trunc = 1.0 if np.linalg.norm(x) > 0 else 0.0
    for i in range(1, max_order + 1):
        t = uapply(coupling(s, t))
        x += t
        if keep_terms:
            terms.append(t.copy())
        xn = np.linalg.norm(x)
        ratio = np.linalg.norm(t) / xn if xn > 0 else 0.0
        trunc = ratio
        if ratio <= threshold:
            order = i - 1
            break
        order = i
    return PowerResult(x, back_substitute(s, x), order, trunc, rhs, terms)


def schur_diag_blocks(s: BlockSystem) -> np.ndarray:
    """Exact block diagonal U_i - sum_j W_ij V+_j W_ij^T (normal_eq.py:253-260)."""
    contrib = np.einsum("nij,njk,nlk->nil", s.W, s.V_pinv[s.g.lm], s.W)
    return s.U - _seg_sum_cam(s.g, contrib)


@dataclass
class PcgResult:
    pose_update: np.ndarray
    landmark_update: np.ndarray
    iterations: int
    rel: float
    flag: str | None
    rhs: np.ndarray


def pcg_solve(s: BlockSystem, max_iterations: int, tolerance: float) -> PcgResult:
    """Block-Jacobi preconditioned CG on the reduced system (solvers.py:153-187)."""
    rhs = schur_rhs(s)
    rhs_norm = np.linalg.norm(rhs)
    if rhs_norm == 0:
        zero = np.zeros_like(rhs)
        return PcgResult(zero, back_substitute(s, zero), 0, 0.0, None, rhs)
    diag = schur_diag_blocks(s)
    try:
        m_inv = np.linalg.inv(diag)
    except np.linalg.LinAlgError:
        m_inv = pinv_psd(diag, 1e-12)[0]
    n = s.g.n_cameras

    def mapply(v):
        return np.einsum("nij,nj->ni", m_inv, v.reshape(n, -1)).ravel()

    x = np.zeros_like(rhs)
    r = rhs.copy()
    z = mapply(r)
    p = z.copy()
    rz = float(r @ z)
    flag, iterations, rel = None, 0, 1.0
    for it in range(1, max_iterations + 1):
        iterations = it
        sp = apply_schur(s, p)
        curvature = float(p @ sp)
        if curvature <= 0:
            flag = "breakdown"
            break
        alpha = rz / curvature
        x += alpha * p
        r -= alpha * sp
        rel = np.linalg.norm(r) / rhs_norm
        if rel <= tolerance:
            break
        z = mapply(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return PcgResult(x, back_substitute(s, x), iterations, rel, flag, rhs)


def tangent_trial(cams, lms, cam_bases, lm_bases, dx, dl):
    """Back-project, add, normalize; None on a zero norm (riemannian.py:110-122)."""
    n_p = len(cam_bases)
    c = cams.reshape(n_p, 12) + np.einsum("nij,nj->ni", cam_bases, dx.reshape(n_p, 11))
    x = lms + np.einsum("nij,nj->ni", lm_bases, dl.reshape(-1, 3))
    cn = np.linalg.norm(c, axis=1)
    xn = np.linalg.norm(x, axis=1)
    if (cn == 0).any() or (xn == 0).any():
        return None
    return (c / cn[:, None]).reshape(n_p, 3, 4), x / xn[:, None]


def retract(cams, lms):
    """Unit-normalize cameras (as 12-vectors) and landmarks (riemannian.py:88-98)."""
    c = cams.reshape(-1, 12)
    cn = np.linalg.norm(c, axis=1)
    xn = np.linalg.norm(lms, axis=1)
    if (cn == 0).any() or (xn == 0).any():
        raise ValueError("cannot retract a zero-norm parameter vector")
    return (c / cn[:, None]).reshape(cams.shape), lms / xn[:, None]


# ---------------------------------------------------------------------------
# one step and the LM outer loop


@dataclass
class StepResult:
    system: BlockSystem
    power: PowerResult
    trial_cams: np.ndarray | None
    trial_lms: np.ndarray | None
    f_trial: float
    lin: Linearization


def lm_step(g: Graph, cams, lms, stage: int, lam: float, eta: float, max_order: int,
            threshold: float, both: bool, inner: str = "power", max_inner: int = 500,
            pcg_tol: float = 1e-6) -> StepResult:
    """Linearize, assemble, inner-solve and form the trial (solvers.py:349-367)."""
    lin = linearize(g, cams, lms, stage, eta)
    sys_ = assemble(g, lin, lam, both or stage == 2)
    if inner == "power":
        pw = power_solve(sys_, max_order, threshold)
    elif inner == "pcg":
        pw = pcg_solve(sys_, max_inner, pcg_tol)
    else:
        raise ValueError(f"unknown inner solver {inner!r}")
    if stage == 1:
        tc = cams + pw.pose_update.reshape(cams.shape)
        tl = np.array(lms, copy=True)
        tl[:, :3] += pw.landmark_update.reshape(-1, 3)
    else:
        res = tangent_trial(cams, lms, lin.cam_bases, lin.lm_bases, pw.pose_update,
                            pw.landmark_update)
        tc, tl = (None, None) if res is None else res
    f_trial = math.inf if tc is None else total_cost(g, tc, tl, stage, eta)
    return StepResult(sys_, pw, tc, tl, f_trial, lin)


@dataclass
class LmLog:
    costs: list
    decisions: str  # 'A' accepted / 'R' rejected, per iteration
    lambdas: list  # damping used at each iteration
    orders: list
    f_trials: list
    cams: np.ndarray
    lms: np.ndarray
    states: list = field(default_factory=list)  # (cams, lms, lam) before each iteration


def lm_minimize(g: Graph, cams, lms, stage: int, *, max_iterations=50, ftol=1e-6,
                lam0=1e-4, max_order=20, threshold=0.01, eta=0.1, varpro=True,
                lam_inc=4.0, lam_dec=0.5, lam_min=1e-12, lam_max=1e8,
                keep_states=False, inner="power", max_inner=500, pcg_tol=1e-6) -> LmLog:
    """Levenberg-Marquardt outer loop (solvers.py:318-393)."""
    cams = np.array(cams, dtype=float)
    lms = np.array(lms, dtype=float)
    f = total_cost(g, cams, lms, stage, eta)
    if not math.isfinite(f):
        raise RuntimeError(f"stage {stage} starting cost is not finite")
    log = LmLog([f], "", [], [], [], cams, lms)
    lam = lam0
    both = (not varpro) or stage == 2
    for _ in range(max_iterations):
        if keep_states:
            log.states.append((cams.copy(), lms.copy(), lam))
        st = lm_step(g, cams, lms, stage, lam, eta, max_order, threshold, both, inner,
                     max_inner, pcg_tol)
        log.lambdas.append(lam)
        log.orders.append(st.power.order_used if inner == "power" else st.power.iterations)
        log.f_trials.append(st.f_trial)
        f_trial = st.f_trial
        converged = False
        if f_trial < f:
            tc, tl = st.trial_cams, st.trial_lms
            if stage == 1 and varpro:
                tl = resolve_landmarks(g, tc, tl, eta)[0]
                f_trial = total_cost(g, tc, tl, stage, eta)
            cams, lms = tc, tl
            converged = abs(f - f_trial) / (f if f > 0 else 1.0) <= ftol
            f = f_trial
            lam = max(lam_min, lam * lam_dec)
            log.decisions += "A"
        else:
            if math.isfinite(f_trial):
                converged = abs(f - f_trial) / (f if f > 0 else 1.0) <= ftol
            lam = min(lam_max, lam * lam_inc)
            log.decisions += "R"
        log.costs.append(f)
        if converged:
            break
    log.cams, log.lms = cams, lms
    return log


def spectral_check(s: BlockSystem, max_iterations: int = 50000, tol: float = 1e-14) -> float:
    """Largest eigenvalue of U^-1 W V+ W^T by power iteration on the symmetrized operator
    U^-1/2 W V+ W^T U^-1/2, starting from the normalized ones vector; stops when the
    Rayleigh quotient changes by <= tol * max(1, |mu|) (solvers.py:263-295)."""
    w, q = np.linalg.eigh(s.U)
    if (w <= 0).any():
        raise ValueError("pose blocks must be positive-definite")
    uih = np.einsum("nij,nj,nkj->nik", q, 1.0 / np.sqrt(w), q)
    n = s.g.n_cameras

    def half(v):
        return np.einsum("nij,nj->ni", uih, v.reshape(n, -1)).ravel()

    dim = n * s.d_p
    v = np.full(dim, 1.0 / math.sqrt(dim))
    mu = 0.0
    for _ in range(max_iterations):
        av = half(coupling(s, half(v)))
        nrm = np.linalg.norm(av)
        if nrm == 0:
            return 0.0
        mu_new = float(v @ av)
        v = av / nrm
        if abs(mu_new - mu) <= tol * max(1.0, abs(mu_new)):
            return mu_new
        mu = mu_new
    return mu


def dense_reduced_matrix(s: BlockSystem) -> np.ndarray:
    """Materialized U - W V+ W^T for small problems (normal_eq.py:263-283 analogue)."""
    n, d = s.g.n_cameras, s.d_p
    S = np.zeros((n * d, n * d))
    for i in range(n):
        S[i * d:(i + 1) * d, i * d:(i + 1) * d] = s.U[i]
    for j in range(s.g.n_landmarks):
        lo, hi = s.g.offsets[j], s.g.offsets[j + 1]
        for a in range(lo, hi):
            for b in range(lo, hi):
                ca, cb = s.g.cam[a], s.g.cam[b]
                S[ca * d:(ca + 1) * d, cb * d:(cb + 1) * d] -= s.W[a] @ s.V_pinv[j] @ s.W[b].T
    return S
