"""GPU: spectral_check (solvers.py:263-295) with the coupling round trip on the device,
against the real reference's values on the mini systems (tests/golden/spectral.npz)."""

import numpy as np
import pytest

from _pvutil import golden, problem_from
from test_oracle_spectral import check_spectral

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pv():
    import paper_2405_05079_b200 as pv
    return pv


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("tag,stage,lam,mode,cams,lms", [
    ("s1v_", 1, 1e-4, "pose_only", "cams", "lms"),
    ("s1j_", 1, 0.3, "both", "cams", "lms"),
    ("s2_", 2, 1e-3, "both", "cams2", "lms2")])
def test_spectral_check_matches_reference(pv, seed, tag, stage, lam, mode, cams, lms):
    z = golden(f"mini_{seed}.npz")
    sp = golden("spectral.npz")
    pr = problem_from(z)
    sysm = pv.assemble_system(pr, pv.ProjectiveState(z[cams], z[lms]), stage, lam, mode)
    mu = pv.spectral_check(sysm, max_iterations=3000)
    check_spectral(mu, float(sp[f"m{seed}_{tag}mu3000"]), float(sp[f"m{seed}_{tag}dense"]))


def test_spectral_check_uncoupled(pv):
    """W = 0 (test_solvers.py:207-209): the power iterate is exactly zero."""
    import _kat
    pr, st = _kat.uncoupled_case()
    sysm = pv.assemble_system(pr, st, 1, 1e-4, "pose_only")
    assert pv.spectral_check(sysm) == 0.0
