"""BAL input path (bal_io.py:115-297) over the native parser in libpovar.so.

* ``parse_bal``            -> bal_io.py:155-203 (pv_bal_header / pv_bal_parse,
                              multi-threaded, same grammar and BalParseError messages)
* ``load_bal``             -> bal_io.py:229-241 (gzip / bzip2 sniffing on the host)
* ``prune_underobserved``  -> bal_io.py:244-278 (distinct-camera counts in
                              pv_bal_prune_masks, O(n_obs) without a sort)
* ``write_bal``            -> bal_io.py:206-226

The native library is required (there is no Python fallback); the BAL entry
points are host-only and run without a GPU.
"""

from __future__ import annotations

import bz2
import ctypes
import gzip
import logging
from pathlib import Path
from typing import IO

import numpy as np

from . import _lib
from .types import BaProblem

logger = logging.getLogger(__name__)

CAMERA_FIELDS = 9
POINT_FIELDS = 3
_ERR_CAP = 4096


class BalParseError(ValueError):
    """Malformed BAL input; carries the 1-based line number of the offending token."""

    def __init__(self, line: int, message: str):
        self.line = line
        super().__init__(f"line {line}: {message}")


def _raise_parse(line: ctypes.c_int64, buf) -> None:
    raise BalParseError(int(line.value), buf.value.decode("utf-8", "replace"))


def parse_bytes(text: bytes, n_threads: int = 0) -> BaProblem:
    """Parse decompressed BAL text (bytes) into a :class:`BaProblem`."""
    lib = _lib.load()
    n_cam, n_pt, n_obs = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    line = ctypes.c_int64()
    err = ctypes.create_string_buffer(_ERR_CAP)
    rc = lib.pv_bal_header(text, len(text), ctypes.byref(n_cam), ctypes.byref(n_pt),
                           ctypes.byref(n_obs), ctypes.byref(line), err, _ERR_CAP)
    if rc != 0:
        _raise_parse(line, err)
    nc, npt, no = n_cam.value, n_pt.value, n_obs.value
    cam_idx = np.empty(no, dtype=np.int64)
    pt_idx = np.empty(no, dtype=np.int64)
    meas = np.empty((no, 2), dtype=np.float64)
    cams = np.empty((nc, CAMERA_FIELDS), dtype=np.float64)
    pts = np.empty((npt, POINT_FIELDS), dtype=np.float64)
    rc = lib.pv_bal_parse(text, len(text), int(n_threads), _lib.i64ptr(cam_idx),
                          _lib.i64ptr(pt_idx), _lib.dptr(meas), _lib.dptr(cams), _lib.dptr(pts),
                          ctypes.byref(line), err, _ERR_CAP)
    if rc != 0:
        _raise_parse(line, err)
    return BaProblem(nc, npt, no, cam_idx, pt_idx, meas, cams, pts)


def parse_bal(stream: IO[str]) -> BaProblem:
    """Parse a BAL-format text stream (bal_io.py:155-203)."""
    data = stream.read()
    if isinstance(data, str):
        data = data.encode("utf-8")
    return parse_bytes(data)


def load_bal(path: str | Path) -> BaProblem:
    """Read a BAL file, transparently decompressing gzip or bzip2 input (bal_io.py:229-241)."""
    path = Path(path)
    with open(path, "rb") as fh:
        magic = fh.read(3)
    if magic[:2] == b"\x1f\x8b":
        opener = gzip.open
    elif magic == b"BZh":
        opener = bz2.open
    else:
        opener = open
    with opener(path, "rb") as fh:
        return parse_bytes(fh.read())


def write_bal(problem: BaProblem, stream: IO[str]) -> None:
    """Serialize losslessly (17 significant digits; bal_io.py:206-226)."""
    stream.write(f"{problem.num_cameras} {problem.num_landmarks} {problem.num_observations}\n")
    for c, l, m in zip(problem.camera_indices, problem.landmark_indices, problem.measurements):
        stream.write(f"{c} {l} {m[0]:.17g} {m[1]:.17g}\n")
    cams = problem.metric_cameras
    if cams is None:
        cams = np.zeros((problem.num_cameras, CAMERA_FIELDS))
    for row in cams:
        for v in row:
            stream.write(f"{v:.17g}\n")
    pts = problem.metric_points
    if pts is None:
        pts = np.zeros((problem.num_landmarks, POINT_FIELDS))
    for row in pts:
        for v in row:
            stream.write(f"{v:.17g}\n")


def prune_underobserved(problem: BaProblem, min_cameras: int = 2) -> BaProblem:
    """Drop landmarks seen by fewer than ``min_cameras`` distinct cameras, then cameras
    left without observations; reindex densely (bal_io.py:244-278)."""
    lib = _lib.load()
    ci = np.ascontiguousarray(problem.camera_indices, dtype=np.int64)
    li = np.ascontiguousarray(problem.landmark_indices, dtype=np.int64)
    keep_lm = np.empty(problem.num_landmarks, dtype=np.uint8)
    cam_seen = np.empty(problem.num_cameras, dtype=np.uint8)
    kept = ctypes.c_int64()
    u8 = ctypes.POINTER(ctypes.c_uint8)
    rc = lib.pv_bal_prune_masks(problem.num_cameras, problem.num_landmarks,
                                problem.num_observations, _lib.i64ptr(ci), _lib.i64ptr(li),
                                int(min_cameras), keep_lm.ctypes.data_as(u8),
                                cam_seen.ctypes.data_as(u8), ctypes.byref(kept))
    if rc != 0:
        raise ValueError("observation indices out of range")
    keep_lm = keep_lm.astype(bool)
    cam_seen = cam_seen.astype(bool)
    if keep_lm.all() and cam_seen.all():
        return problem
    obs_keep = keep_lm[li]
    lm_map = np.cumsum(keep_lm) - 1
    cam_map = np.cumsum(cam_seen) - 1
    logger.info("pruned %d under-observed landmarks and %d empty cameras",
                int((~keep_lm).sum()), int((~cam_seen).sum()))
    return BaProblem(
        num_cameras=int(cam_seen.sum()),
        num_landmarks=int(keep_lm.sum()),
        num_observations=int(kept.value),
        camera_indices=cam_map[ci[obs_keep]],
        landmark_indices=lm_map[li[obs_keep]],
        measurements=problem.measurements[obs_keep],
        metric_cameras=None if problem.metric_cameras is None
        else problem.metric_cameras[cam_seen],
        metric_points=None if problem.metric_points is None else problem.metric_points[keep_lm],
    )
