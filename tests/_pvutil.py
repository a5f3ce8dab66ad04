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
