"""Known-answer cases restated from the reference test-suite (pkg/tests), shared by the
CPU oracle tests and the GPU parity tests.  Each builder returns plain arrays so
both sides consume identical inputs."""

from __future__ import annotations

import math

import numpy as np

from paper_2405_05079_b200.types import BaProblem, ProjectiveState


def problem(n_cams, n_lms, cam_idx, lm_idx, meas):
    return BaProblem(n_cams, n_lms, len(cam_idx), np.asarray(cam_idx, dtype=np.int64),
                     np.asarray(lm_idx, dtype=np.int64), np.asarray(meas, dtype=float))


def random_graph(n_cameras, n_landmarks, seed, k=None, shuffle=True):
    """Every landmark sees >= 2 distinct cameras (conftest.py:27-46 style)."""
    rng = np.random.default_rng(seed)
    ci, li = [], []
    for j in range(n_landmarks):
        kk = k or int(rng.integers(2, n_cameras + 1))
        kk = min(kk, n_cameras)
        for c in sorted(rng.choice(n_cameras, size=kk, replace=False)):
            ci.append(c)
            li.append(j)
    ci, li = np.array(ci), np.array(li)
    if shuffle:
        p = rng.permutation(len(ci))
        ci, li = ci[p], li[p]
    return problem(n_cameras, n_landmarks, ci, li, 2.0 * rng.standard_normal((len(ci), 2)))


def random_state(prob, seed, unit=False):
    rng = np.random.default_rng(seed)
    cams = rng.standard_normal((prob.num_cameras, 3, 4))
    lms = np.concatenate([rng.standard_normal((prob.num_landmarks, 3)),
                          np.ones((prob.num_landmarks, 1))], axis=1)
    if unit:
        cams = (cams.reshape(-1, 12) / np.linalg.norm(cams.reshape(-1, 12), axis=1)[:, None]
                ).reshape(cams.shape)
        lms = lms / np.linalg.norm(lms, axis=1)[:, None]
    return ProjectiveState(cams, lms)


def hand_residual_case():
    """test_objective.py:33-40: r = (0, 0, sqrt(.1) .75, sqrt(.1) 1.5)."""
    cam = np.array([[[1.0, 0, 0, 0], [0, 1, 0, 0], [0, 0, 1, 0]]])
    st = ProjectiveState(cam, np.array([[1.0, 2.0, 4.0, 1.0]]))
    pr = problem(1, 1, [0], [0], [[0.25, 0.5]])
    return pr, st, 0.1 * (0.75 ** 2 + 1.5 ** 2)


def pythagoras_case():
    """test_objective.py:223-240: stage-2 residual (3, 4) -> cost 25."""
    cam = np.concatenate([np.eye(3), np.zeros((3, 1))], axis=1)[None]
    st = ProjectiveState(cam, np.array([[3.0, 4.0, 1.0, 0.0]]))
    return problem(1, 1, [0], [0], [[0.0, 0.0]]), st, 25.0


def degenerate_depth_case():
    """test_objective.py:257-266: |z| = 0 -> stage-2 cost +inf."""
    cam = np.zeros((1, 3, 4))
    cam[0, 0, 0] = 1.0
    st = ProjectiveState(cam, np.array([[1.0, 0.0, 0.0, 0.0]]))
    return problem(1, 1, [0], [0], [[0.0, 0.0]]), st, math.inf


def recovery_case(seed):
    """test_objective.py:273-291: noise-free landmark recovered by the closed form."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 6))
    truth = np.append(rng.standard_normal(3), 1.0)
    cams = rng.standard_normal((n, 3, 4))
    for c in cams:
        c[2] /= c[2] @ truth
    meas = np.einsum("nij,j->ni", cams[:, :2, :], truth)
    pr = problem(n, 1, np.arange(n), np.zeros(n, dtype=int), meas)
    return pr, ProjectiveState(cams, np.array([[0.0, 0, 0, 1]])), truth, float(rng.uniform(0, 1))


def zero_rhs_case(seed=0):
    """test_objective.py:294-305: zero offsets -> landmark at the origin."""
    rng = np.random.default_rng(seed)
    cams = rng.standard_normal((3, 3, 4))
    cams[:, :, 3] = 0.0
    pr = problem(3, 1, np.arange(3), np.zeros(3, dtype=int), np.zeros((3, 2)))
    return pr, ProjectiveState(cams, np.array([[5.0, 5, 5, 1]])), np.array([0.0, 0, 0, 1])


def degenerate_landmark_case():
    """test_objective.py:323-336: zero cameras -> rank-0 system, landmark unchanged."""
    pr = problem(2, 1, np.arange(2), np.zeros(2, dtype=int), np.ones((2, 2)))
    x = np.array([[7.0, 8.0, 9.0, 1.0]])
    return pr, ProjectiveState(np.zeros((2, 3, 4)), x), x[0]


def uncoupled_case(seed=0):
    """test_solvers.py:25-41 analogue: W = 0 (camera 3x3 blocks zero) -> series order 0,
    truncation 0, update -U^-1 b_p."""
    rng = np.random.default_rng(seed)
    pr = random_graph(3, 8, seed)
    cams = rng.standard_normal((3, 3, 4))
    cams[:, :, :3] = 0.0
    lms = np.concatenate([rng.standard_normal((8, 3)), np.ones((8, 1))], axis=1)
    return pr, ProjectiveState(cams, lms)


def affine_consistent_case(seed=0):
    """test_solvers.py:238-262: exact zero of the stage-1 cost -> LM stops at iteration 1.

    Small-integer cameras and landmarks keep every product exact in fp64, so the
    zero residual is exact under any summation order (CPU or GPU FMAs)."""
    rng = np.random.default_rng(seed)
    base = random_graph(3, 6, seed, shuffle=False)
    cams = rng.integers(-3, 4, size=(3, 3, 4)).astype(float)
    cams[:, 2, :] = 0.0
    cams[:, 2, 3] = 1.0
    lms = np.concatenate([rng.integers(-3, 4, size=(6, 3)).astype(float), np.ones((6, 1))],
                         axis=1)
    meas = np.einsum("nij,nj->ni", cams[base.camera_indices][:, :2, :],
                     lms[base.landmark_indices])
    pr = problem(3, 6, base.camera_indices, base.landmark_indices, meas)
    return pr, ProjectiveState(cams, lms)


def long_track_case(seed=3):
    """Tracks longer than one warp (k > 32), an unobserved landmark and an unobserved
    camera, in a shuffled observation order."""
    rng = np.random.default_rng(seed)
    n_c, n_l = 48, 40
    ci, li = [], []
    for j in range(n_l):
        if j == 7:
            continue  # unobserved landmark
        k = 45 if j % 5 == 0 else int(rng.integers(2, 9))
        for c in sorted(rng.choice(n_c - 1, size=k, replace=False)):  # camera 47 unused
            ci.append(c)
            li.append(j)
    ci, li = np.array(ci), np.array(li)
    p = rng.permutation(len(ci))
    meas = 0.3 * rng.standard_normal((len(ci), 2))
    pr = problem(n_c, n_l, ci[p], li[p], meas[p])
    return pr, random_state(pr, seed + 1)
