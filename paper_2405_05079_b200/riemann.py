"""Stage bridge: retraction onto the unit spheres (riemannian.py:88-107).

A one-off O(n_p + n_l) state conversion between the two stages (not part of
the per-iteration hot path, which retracts on the device inside the trial
kernels).
"""

from __future__ import annotations

import numpy as np

from .types import ProjectiveState


def retract(state: ProjectiveState) -> ProjectiveState:
    """Normalize every camera 12-vector and landmark 4-vector (riemannian.py:88-98)."""
    cams = state.cameras.reshape(-1, 12)
    cn = np.linalg.norm(cams, axis=1)
    ln = np.linalg.norm(state.landmarks, axis=1)
    if (cn == 0).any() or (ln == 0).any():
        raise ValueError("cannot retract a zero-norm parameter vector")
    return ProjectiveState((cams / cn[:, None]).reshape(state.cameras.shape),
                           state.landmarks / ln[:, None])


def lift_stage1_to_stage2(state: ProjectiveState) -> ProjectiveState:
    """Stage-1 state (landmark w = 1) to stage-2 form (riemannian.py:101-107)."""
    return retract(state)
