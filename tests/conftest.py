"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and call the CUDA path
through the C-ABI; everything else runs on CPU (oracle vs golden vectors,
host logic, library symbol checks, gloo multi-process tests)."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for _p in (str(ROOT), str(ROOT / "tests")):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpovar.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


from _pvutil import golden  # noqa: E402


@pytest.fixture(params=[0, 1, 2], ids=lambda s: f"mini{s}")
def mini(request):
    return golden(f"mini_{request.param}.npz")


def pytest_sessionfinish(session, exitstatus):
    import json

    import _pvutil
    path = os.environ.get("PV_PARITY_REPORT")
    if path and _pvutil.REPORT:
        Path(path).parent.mkdir(parents=True, exist_ok=True)
        Path(path).write_text(json.dumps(_pvutil.REPORT, indent=1))
