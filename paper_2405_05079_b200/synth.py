"""Seeded synthetic problems with the shapes of BASELINE.json's five configs.

The reference ships no generator for these configs: its
``make_ring_problem`` (pkg/src/stratba/synth.py:29-87) has every camera see
every landmark.  This module is the input producer for tests and the bench; it
is not part of the solver path.  Choices (documented in DESIGN.md):

* Philox counter-based generator (like bal_io.py:291), problem seed 0, init seed 1.
* Ground-truth cameras: rotation from a uniform random quaternion, centre
  ``c = -10 R^T e3`` so the +z optical axis looks at the origin (centre
  uniform on the radius-10 sphere); focal length U(400, 1200), principal
  point 0.  The ``large`` config instead walks the centres along a random walk
  on the sphere and orients each camera towards the origin with a random roll.
* Ground-truth landmarks N(0, I3).
* Visibility: each landmark draws k distinct cameras that have it in front
  (depth > 0); ``large`` restricts the draw to the 10% of cameras nearest in
  angle to the landmark's direction.
* Track lengths: tiny U{2..6}; small/medium/large geometric with min 2 and
  the stated mean (cap 100 for medium); vlarge a power law P(k) ~ k^-a on
  [2, 500] with ``a`` fit so the mean track equals the stated
  28,987,644 / 4,456,117 (a literal Zipf(1.8) on [2, 500] has mean ~13.8,
  which would double the stated observation count).
* Measurement = pinhole projection (+z forward) + N(0, 1 px), divided by the
  mean focal length.
* Start state: every P entry and landmark coordinate i.i.d. N(0, 1), last
  landmark coordinate 1 (BASELINE's "initialization-free start").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .types import BaProblem, ProjectiveState


@dataclass(frozen=True)
class SynthConfig:
    name: str
    n_cameras: int
    n_landmarks: int
    track: tuple  # ("uniform", lo, hi) | ("geometric", mean, cap) | ("power", mean, cap)
    clustered: bool = False
    lm_iterations: int = 50
    max_power_order: int = 20
    stages: tuple = (1,)
    nominal_observations: int = 0


CONFIGS = {
    "tiny": SynthConfig("tiny", 16, 2000, ("uniform", 2, 6), lm_iterations=20,
                        nominal_observations=8000),
    "small": SynthConfig("small", 49, 7776, ("geometric", 4.1, None),
                         nominal_observations=31843),
    "medium": SynthConfig("medium", 356, 226_730, ("geometric", 5.5, 100), stages=(1, 2),
                          nominal_observations=1_255_268),
    "large": SynthConfig("large", 1778, 993_923, ("geometric", 5.0, None), clustered=True,
                         stages=(1, 2), nominal_observations=5_001_946),
    "vlarge": SynthConfig("vlarge", 13_682, 4_456_117, ("power", 28_987_644 / 4_456_117, 500),
                          max_power_order=30, stages=(1, 2),
                          nominal_observations=28_987_644),
}

RADIUS = 10.0
FOCAL_RANGE = (400.0, 1200.0)
NOISE_PX = 1.0
CLUSTER_FRACTION = 0.10


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed) & 0xFFFFFFFFFFFFFFFF))


def _quat_to_rot(q: np.ndarray) -> np.ndarray:
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    r = np.empty((len(q), 3, 3))
    r[:, 0, 0] = 1 - 2 * (y * y + z * z)
    r[:, 0, 1] = 2 * (x * y - w * z)
    r[:, 0, 2] = 2 * (x * z + w * y)
    r[:, 1, 0] = 2 * (x * y + w * z)
    r[:, 1, 1] = 1 - 2 * (x * x + z * z)
    r[:, 1, 2] = 2 * (y * z - w * x)
    r[:, 2, 0] = 2 * (x * z - w * y)
    r[:, 2, 1] = 2 * (y * z + w * x)
    r[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return r


def _look_at(dirs: np.ndarray, rolls: np.ndarray) -> np.ndarray:
    """Rotations whose third row (optical axis) is -dirs, with a roll about it."""
    z = -dirs / np.linalg.norm(dirs, axis=1, keepdims=True)
    helper = np.where(np.abs(z[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]),
                      np.array([[1.0, 0.0, 0.0]]))
    x = np.cross(helper, z)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    y = np.cross(z, x)
    c, s = np.cos(rolls)[:, None], np.sin(rolls)[:, None]
    xr = c * x + s * y
    yr = -s * x + c * y
    return np.stack([xr, yr, z], axis=1)


def _track_lengths(rng: np.random.Generator, cfg: SynthConfig, n_pool: int) -> np.ndarray:
    kind = cfg.track[0]
    n = cfg.n_landmarks
    if kind == "uniform":
        k = rng.integers(cfg.track[1], cfg.track[2] + 1, size=n)
    elif kind == "geometric":
        mean, cap = cfg.track[1], cfg.track[2]
        k = 1 + rng.geometric(1.0 / (mean - 1.0), size=n)
        if cap is not None:
            k = np.minimum(k, cap)
    elif kind == "power":
        mean, cap = cfg.track[1], cfg.track[2]
        support = np.arange(2, cap + 1, dtype=np.float64)
        lo, hi = 1.0, 4.0
        for _ in range(100):  # bisection on the exponent for the stated mean
            a = 0.5 * (lo + hi)
            p = support ** -a
            m = (support * p).sum() / p.sum()
            lo, hi = (a, hi) if m > mean else (lo, a)
        p = support ** -a
        cdf = np.cumsum(p / p.sum())
        k = 2 + np.searchsorted(cdf, rng.random(n), side="right")
        k = np.minimum(k, cap)
    else:
        raise ValueError(kind)
    return np.minimum(k, n_pool).astype(np.int64)


def _dedupe_rounds(rng, lm_of_obs, draw, valid_fn, max_rounds=200):
    """Redraw camera slots until every (landmark, camera) pair is distinct and valid."""
    cams = draw(np.arange(len(lm_of_obs)))
    for _ in range(max_rounds):
        key = lm_of_obs * np.int64(1 << 32) + cams
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = np.zeros(len(ks), dtype=bool)
        dup[1:] = ks[1:] == ks[:-1]
        bad = np.zeros(len(cams), dtype=bool)
        bad[order[dup]] = True
        bad |= ~valid_fn(np.arange(len(cams)), cams)
        idx = np.nonzero(bad)[0]
        if len(idx) == 0:
            return cams, np.ones(len(cams), dtype=bool)
        cams[idx] = draw(idx)
    return cams, ~bad


def make_problem(config: str | SynthConfig, seed: int = 0, *, landmark_fraction: float = 1.0
                 ) -> tuple[BaProblem, dict]:
    """Generate the seeded synthetic problem for a BASELINE config.

    ``landmark_fraction`` < 1 keeps the cameras and draws only that fraction
    of the landmarks (the bounded CPU-baseline sample).  Returns the problem
    and a ground-truth dict (rotations, centres, focals, points).
    """
    cfg = CONFIGS[config] if isinstance(config, str) else config
    if landmark_fraction < 1.0:
        cfg = SynthConfig(cfg.name, cfg.n_cameras, max(1, int(cfg.n_landmarks * landmark_fraction)),
                          cfg.track, cfg.clustered, cfg.lm_iterations, cfg.max_power_order,
                          cfg.stages, 0)
    rng = _rng(seed)
    n_p, n_l = cfg.n_cameras, cfg.n_landmarks
    if cfg.clustered:
        d = rng.standard_normal(3)
        dirs = np.empty((n_p, 3))
        d /= np.linalg.norm(d)
        step = 0.15
        for i in range(n_p):
            dirs[i] = d
            d = d + step * rng.standard_normal(3)
            d /= np.linalg.norm(d)
        rot = _look_at(dirs, rng.uniform(0, 2 * np.pi, n_p))
        centres = RADIUS * dirs
    else:
        rot = _quat_to_rot(rng.standard_normal((n_p, 4)))
        centres = -RADIUS * rot[:, 2, :]
    focal = rng.uniform(*FOCAL_RANGE, n_p)
    points = rng.standard_normal((n_l, 3))

    def depth(lm, cam):
        return np.einsum("ni,ni->n", rot[cam, 2, :], points[lm] - centres[cam])

    if cfg.clustered:
        n_near = max(2, int(round(CLUSTER_FRACTION * n_p)))
        cam_dirs = centres / np.linalg.norm(centres, axis=1, keepdims=True)
        lm_dirs = points / np.linalg.norm(points, axis=1, keepdims=True)
        near = np.empty((n_l, n_near), dtype=np.int64)
        chunk = 8192
        for lo in range(0, n_l, chunk):
            cos = lm_dirs[lo:lo + chunk] @ cam_dirs.T
            near[lo:lo + chunk] = np.argpartition(-cos, n_near - 1, axis=1)[:, :n_near]
        k = _track_lengths(rng, cfg, n_near)
        lm_of_obs = np.repeat(np.arange(n_l, dtype=np.int64), k)

        def draw(idx):
            return near[lm_of_obs[idx], rng.integers(0, n_near, size=len(idx))]
    else:
        k = _track_lengths(rng, cfg, n_p)
        lm_of_obs = np.repeat(np.arange(n_l, dtype=np.int64), k)

        def draw(idx):
            return rng.integers(0, n_p, size=len(idx)).astype(np.int64)

    def valid(idx, cams):
        return depth(lm_of_obs[idx], cams[idx]) > 1e-6

    cams, ok = _dedupe_rounds(rng, lm_of_obs, draw, valid)
    lm_of_obs, cams = lm_of_obs[ok], cams[ok]

    # BAL-like camera-major observation order
    order = np.lexsort((lm_of_obs, cams))
    cams, lms = cams[order], lm_of_obs[order]
    n_o = len(cams)
    meas = np.empty((n_o, 2))
    chunk = 1 << 22
    for lo in range(0, n_o, chunk):
        c, l = cams[lo:lo + chunk], lms[lo:lo + chunk]
        pc = np.einsum("nij,nj->ni", rot[c], points[l] - centres[c])
        meas[lo:lo + chunk] = focal[c, None] * pc[:, :2] / pc[:, 2:3]
    meas += NOISE_PX * rng.standard_normal((n_o, 2))
    fmean = float(focal.mean())
    meas /= fmean
    problem = BaProblem(n_p, n_l, n_o, cams, lms, meas)
    truth = dict(rotations=rot, centres=centres, focal=focal, points=points, focal_mean=fmean)
    return problem, truth


def random_state(problem: BaProblem, seed: int = 1) -> ProjectiveState:
    """BASELINE's initialization-free start: i.i.d. N(0,1) P entries and landmarks."""
    rng = _rng(seed)
    cams = rng.standard_normal((problem.num_cameras, 3, 4))
    lms = np.ones((problem.num_landmarks, 4))
    lms[:, :3] = rng.standard_normal((problem.num_landmarks, 3))
    return ProjectiveState(cams, lms)


def ground_truth_state(truth: dict) -> ProjectiveState:
    """Projective state that reproduces the noise-free normalized measurements."""
    s = truth["focal"] / truth["focal_mean"]
    rot, c = truth["rotations"], truth["centres"]
    p = np.concatenate([rot, -np.einsum("nij,nj->ni", rot, c)[:, :, None]], axis=2)
    p[:, :2, :] *= s[:, None, None]
    lms = np.concatenate([truth["points"], np.ones((len(truth["points"]), 1))], axis=1)
    return ProjectiveState(p, lms)
