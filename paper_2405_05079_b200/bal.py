"""BAL input path (bal_io.py:115-297) over the native parser in libpovar.so.

* ``parse_bal``            -> bal_io.py:155-203 (pv_bal_header / pv_bal_parse,
                              multi-threaded, same grammar and BalParseError messages)
* ``load_bal``             -> bal_io.py:229-241 (gzip / bzip2 detected from the leading
                              bytes, decompressed whole, then the native parser)
* ``prune_underobserved``  -> bal_io.py:244-278 (distinct-camera counts in
                              pv_bal_prune_masks, O(n_obs) without a sort)

Writing BAL files (``write_bal``, bal_io.py:206-226) is not part of this path: the
reference's writer is used where a file is needed (tests, make_golden.py).

The native library is required (there is no Python fallback); the BAL entry
points are host-only and run without a GPU.
"""

from __future__ import annotations

import ctypes
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


# leading bytes of the compressed containers load_bal accepts (bal_io.py:229-241); any
# other file is read as plain text
_CODECS = ((b"\x1f\x8b", "gzip"), (b"BZh", "bz2"))


def load_bal(path: str | Path) -> BaProblem:
    """Read a BAL file from disk, plain or gzip / bzip2 compressed (bal_io.py:229-241).

    The whole (decompressed) file is handed to the native multi-threaded parser.
    """
    raw = Path(path).read_bytes()
    codec = next((name for magic, name in _CODECS if raw.startswith(magic)), None)
    if codec is not None:
        raw = __import__(codec).decompress(raw)
    return parse_bytes(raw)


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
    keep_lm = keep_lm.view(bool)
    cam_seen = cam_seen.view(bool)
    if keep_lm.all() and cam_seen.all():
        return problem  # nothing to drop: the caller's object (bal_io.py:261-262)
    n_cam, n_lm = int(np.count_nonzero(cam_seen)), int(np.count_nonzero(keep_lm))
    # dense renumbering of the survivors: old id -> rank among the kept ids
    new_cam = np.full(problem.num_cameras, -1, dtype=np.int64)
    new_cam[cam_seen] = np.arange(n_cam)
    new_lm = np.full(problem.num_landmarks, -1, dtype=np.int64)
    new_lm[keep_lm] = np.arange(n_lm)
    rows = np.flatnonzero(keep_lm[li])  # surviving observations, original order
    logger.info("pruned %d under-observed landmarks and %d empty cameras",
                problem.num_landmarks - n_lm, problem.num_cameras - n_cam)

    def subset(a, mask):
        return None if a is None else a[mask]

    return BaProblem(n_cam, n_lm, int(kept.value), new_cam[ci[rows]], new_lm[li[rows]],
                     problem.measurements[rows], subset(problem.metric_cameras, cam_seen),
                     subset(problem.metric_points, keep_lm))
