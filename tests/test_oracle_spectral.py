"""CPU: the oracle's spectral_check (solvers.py:263-295) against the real reference's values
on the mini systems (tests/golden/spectral.npz, made by tests/golden/make_golden.py).

The power iterate approaches the top eigenvalue of U^-1 W V+ W^T from below; two correct
implementations that differ in the last bits of S'.v stop within rounding of each other
(3000-iteration cap, the reference's acceptance-test setting), and both satisfy the
reference suite's property against the dense eigenvalue (test_solvers.py:219-226).
"""

import pytest

from _pvutil import golden
from oracle import povar_oracle as O


def systems(seed):
    z = golden(f"mini_{seed}.npz")
    g = O.make_graph(int(z["n_cameras"]), int(z["n_landmarks"]), z["cam_idx"], z["lm_idx"],
                     z["meas"])
    lin1 = O.linearize(g, z["cams"], z["lms"], 1)
    lin2 = O.linearize(g, z["cams2"], z["lms2"], 2)
    return {"s1v_": O.assemble(g, lin1, 1e-4, False),
            "s1j_": O.assemble(g, lin1, 0.3, True),
            "s2_": O.assemble(g, lin2, 1e-3, True)}


def check_spectral(mu, ref, dense):
    """Shared with the GPU test: the reference's property (test_solvers.py:219-226) and
    agreement with the reference's own iterate."""
    assert 0.0 <= mu < 1.0
    assert mu <= dense * (1 + 1e-12) + 1e-12
    assert dense - mu <= 1e-3 * max(1.0, dense)
    assert abs(mu - ref) <= 1e-6 * max(1.0, abs(ref))


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("tag", ["s1v_", "s1j_", "s2_"])
def test_spectral_check_matches_reference(seed, tag):
    sp = golden("spectral.npz")
    mu = O.spectral_check(systems(seed)[tag], max_iterations=3000)
    check_spectral(mu, float(sp[f"m{seed}_{tag}mu3000"]), float(sp[f"m{seed}_{tag}dense"]))


def test_spectral_check_zero_coupling():
    import numpy as np
    s = systems(0)["s1v_"]
    s.W = np.zeros_like(s.W)
    assert O.spectral_check(s) == 0.0
