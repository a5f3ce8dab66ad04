"""ctypes binding of libpovar.so (include/povar.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``).  There
is no CPU fallback: if the shared library or a CUDA device is missing, every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .types import NumericFailureError

# PV_LIB_PATH: an alternative build of the same library (tuning experiments, tools/)
LIB_PATH = os.environ.get("PV_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libpovar.so")

PV_OK, PV_EINVAL, PV_ECUDA, PV_ENCCL, PV_ENONFINITE, PV_EDEGENERATE, PV_ESINGULAR = range(7)
PV_CURRENT, PV_TRIAL = 0, 1
(PV_DBG_U, PV_DBG_UINV, PV_DBG_BP, PV_DBG_V, PV_DBG_VPINV, PV_DBG_BL, PV_DBG_DEGEN, PV_DBG_W,
 PV_DBG_RHS, PV_DBG_X, PV_DBG_DL, PV_DBG_ULIN, PV_DBG_SDIAG, PV_DBG_MINV) = range(14)
INFO_FIELDS = ("n_p", "n_l_local", "n_o_local", "tasks", "chunks", "launches", "rank", "world",
               "device_bytes", "n_l_global", "resolve_fallbacks", "blocks", "persist_l2",
               "warps_per_cam", "solve_rhs_us", "solve_terms_us", "solve_backsub_us",
               "solve_terms_launched", "xm_bytes", "pipe_warps")
PV_INFO_COUNT = 24
(PV_OPT_STAGE_CAP, PV_OPT_POL_STREAM, PV_OPT_POL_T, PV_OPT_POL_S, PV_OPT_DISCARD_S,
 PV_OPT_BLOCK_BYTES, PV_OPT_FORCE_COLLECTIVE, _PV_OPT_RESERVED7, PV_OPT_CAM_PIPE,
 PV_OPT_RESOLVE_SLOTS, PV_OPT_SPLIT_LAST, PV_OPT_RHS_REUSE, PV_OPT_COST_CS,
 PV_OPT_BENCH_SPLIT, PV_OPT_XM, PV_OPT_GRAPH, PV_OPT_BALANCE, PV_OPT_BAL_ITEM,
 PV_OPT_BAL_ROUND, PV_OPT_BAL_LAST, PV_OPT_BAL_RFIX, PV_OPT_BAL_ROBS8, PV_OPT_SERIES,
 PV_OPT_KSLOT) = range(24)

# (name, restype, argtypes) of every exported symbol declared in include/povar.h
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = [
    ("pv_nccl_unique_id", ctypes.c_int, [ctypes.c_char_p]),
    ("pv_loopback_id", ctypes.c_int, [ctypes.c_int, ctypes.c_char_p]),
    ("pv_create", ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                 _I64, _I64, _D, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_double]),
    ("pv_destroy", None, [_P]),
    ("pv_last_error", ctypes.c_char_p, [_P]),
    ("pv_info", ctypes.c_int, [_P, _I64]),
    ("pv_stream", _P, [_P]),
    ("pv_set_option", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int64]),
    ("pv_set_state", ctypes.c_int, [_P, _D, _D]),
    ("pv_get_state", ctypes.c_int, [_P, _D, _D]),
    ("pv_get_trial", ctypes.c_int, [_P, _D, _D]),
    ("pv_cost", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _D]),
    ("pv_linearize", ctypes.c_int, [_P, ctypes.c_int]),
    ("pv_damp", ctypes.c_int, [_P, ctypes.c_double, ctypes.c_int, _I64]),
    ("pv_power_solve", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_int), _D]),
    ("pv_pcg_solve", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double,
                                    ctypes.POINTER(ctypes.c_int), _D,
                                    ctypes.POINTER(ctypes.c_int)]),
    ("pv_trial", ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("pv_accept", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, _D, _I64]),
    ("pv_resolve_current", ctypes.c_int, [_P, _I64]),
    ("pv_back_substitute", ctypes.c_int, [_P, _D]),
    ("pv_get_step", ctypes.c_int, [_P, _D, _D]),
    ("pv_schur_apply", ctypes.c_int, [_P, ctypes.c_int, _D, _D]),
    ("pv_bench_terms", ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_float)]),
    ("pv_debug_get", ctypes.c_int, [_P, ctypes.c_int, _D]),
    # include/povar_bal.h (host-only BAL input path)
    ("pv_bal_header", ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, _I64, _I64, _I64, _I64,
                                     ctypes.c_char_p, ctypes.c_size_t]),
    ("pv_bal_parse", ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, _I64, _I64,
                                    _D, _D, _D, _I64, ctypes.c_char_p, ctypes.c_size_t]),
    ("pv_bal_prune_masks", ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I64,
                                          _I64, ctypes.c_int64,
                                          ctypes.POINTER(ctypes.c_uint8),
                                          ctypes.POINTER(ctypes.c_uint8), _I64]),
]

_lib = None


class PovarLibraryError(RuntimeError):
    """libpovar.so is missing or failed to load (no CPU fallback exists)."""


def _preload_nccl() -> None:
    """Make libnccl.so.2 resolve to PyTorch's bundled NCCL (2.28) before libpovar.so loads.

    libpovar.so and libtorch_cuda.so both need ``libnccl.so.2``; the dynamic loader binds
    that name to whichever copy is loaded first.  PyTorch needs symbols only 2.28 has, so
    the system 2.27 must not win when libpovar.so happens to load before ``import torch``.
    The bundled library is an ABI superset of the 2.27 header libpovar.so is built with.
    """
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for base in (spec.submodule_search_locations or []) if spec else []:
        path = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(path):
            ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
            return


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    _preload_nccl()
    if not os.path.exists(LIB_PATH):
        raise PovarLibraryError(
            f"{LIB_PATH} not found: build it with `make` (or __graft_entry__.build()); "
            "the PoVar path has no CPU fallback")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the host
        raise PovarLibraryError(f"cannot load {LIB_PATH}: {e}") from e
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error(ctx) -> str:
    msg = load().pv_last_error(ctx)
    return msg.decode() if msg else ""


def check(rc: int, ctx=None) -> None:
    if rc == PV_OK:
        return
    msg = last_error(ctx)
    if rc == PV_EINVAL:
        raise ValueError(msg)
    if rc == PV_ENONFINITE:
        raise NumericFailureError(msg)
    if rc == PV_EDEGENERATE:
        raise FloatingPointError(msg)
    if rc == PV_ESINGULAR:
        import numpy as np
        raise np.linalg.LinAlgError(msg)
    kind = "NCCL" if rc == PV_ENCCL else "CUDA"
    raise RuntimeError(f"libpovar {kind} error ({rc}): {msg}")


def dptr(a):
    return a.ctypes.data_as(_D)


def i64ptr(a):
    return a.ctypes.data_as(_I64)
