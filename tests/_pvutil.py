"""Test helpers (imported by test modules as ``_pvutil``)."""

from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def golden(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def problem_from(z):
    from paper_2405_05079_b200.types import BaProblem
    return BaProblem(int(z["n_cameras"]), int(z["n_landmarks"]), len(z["cam_idx"]),
                     z["cam_idx"].astype(np.int64), z["lm_idx"].astype(np.int64), z["meas"])


REF_INSTALL = ROOT / "baseline" / "_ref"


def reference_stratba():
    """The UNMODIFIED reference package installed under baseline/_ref (git-ignored; it
    travels to the GPU box with the working tree).  Used only as the caller whose plug
    point is switched to the device path, never as the thing measured."""
    import importlib
    import sys
    if not (REF_INSTALL / "stratba" / "__init__.py").exists():
        import pytest
        pytest.skip("reference not installed under baseline/_ref (DESIGN.md section 7)")
    if str(REF_INSTALL) not in sys.path:
        sys.path.insert(0, str(REF_INSTALL))
    mod = importlib.import_module("stratba")
    for sub in ("solvers", "pipeline", "bal_io", "evaluation", "riemannian", "objective"):
        importlib.import_module("stratba." + sub)
    return mod


# achieved parity errors of the GPU tests: every check() is recorded and, when
# PV_PARITY_REPORT names a file, written there at the end of the session (conftest.py)
REPORT = []


def check(label, err, tol):
    """Assert ``err <= tol`` and record the achieved error next to its tolerance."""
    import os
    test = os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    REPORT.append({"test": test, "quantity": label, "error": float(err), "tol": float(tol)})
    assert err <= tol, f"{label}: {err:.3e} > {tol:.0e}"
