"""ctypes binding of include/oximap_b200.h.

This is the only module that touches the shared library.  It fails loudly
(NativeLibraryError) when the library is missing: there is no CPU fallback
anywhere on the product path.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

from .errors import (
    ArgumentError,
    DataError,
    IllConditionedPriorError,
    NativeLibraryError,
    NumericalError,
    SingularOperatorError,
)

import os

# OXM_LIB_PATH overrides the in-tree library (tools/em_variants.py builds
# tuning variants); the default is the in-tree build.
LIB_PATH = pathlib.Path(os.environ.get("OXM_LIB_PATH") or pathlib.Path(__file__).resolve().parent / "_lib" / "liboximap_b200.so")
HEADER_PATH = pathlib.Path(__file__).resolve().parent.parent / "include" / "oximap_b200.h"

OXM_OK = 0
OXM_ERR_ARGUMENT = -1
OXM_ERR_DATA = -2
OXM_ERR_NUMERICAL = -3
OXM_ERR_SINGULAR = -4
OXM_ERR_ILL_CONDITIONED = -5
OXM_ERR_CUDA = -10
OXM_ERR_WORKSPACE = -11

FLAG_NONFINITE = 1
FLAG_NEGATIVE_LL = 2
MAX_BANDS = 64

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f64 = ctypes.c_double


class Operators(ctypes.Structure):
    """Mirror of ``oxm_operators``."""

    _fields_ = [
        ("n_bands", ctypes.c_int32),
        ("max_iters", ctypes.c_int32),
        ("epsilon", _f64),
        ("rel_tol", _f64),
        ("fallback_below", _f64),
        ("solve", _vp),
        ("fit_mat", _vp),
        ("xi", _vp),
        ("sens", _vp),
        ("gain", _vp),
    ]


# name -> (restype, argtypes)
_SIGNATURES = {
    "oxm_abi_version": (_i32, []),
    "oxm_status_string": (ctypes.c_char_p, [_i32]),
    "oxm_last_error": (ctypes.c_char_p, []),
    "oxm_ctx_create": (_i32, [_i32, ctypes.POINTER(Operators), ctypes.POINTER(_vp)]),
    "oxm_ctx_destroy": (_i32, [_vp]),
    "oxm_ctx_set_em_lead": (_i32, [_vp, _f64, _f64, _f64]),
    "oxm_ctx_set_em_first_guard": (_i32, [_vp, _f64, _i32]),
    "oxm_ctx_set_em_debug_log": (_i32, [_vp, _vp, _vp]),
    "oxm_haar_layout": (_i32, [_i64, _i64, _i32, _vp, _vp]),
    "oxm_haar_forward_f32": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp]),
    "oxm_haar_forward_f64": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp]),
    "oxm_haar_inverse_f32": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "oxm_haar_inverse_f64": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "oxm_unmix_f32": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp]),
    "oxm_unmix_f64": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp]),
    "oxm_em_lowpass": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "oxm_expectation_step": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "oxm_fit_f32": (_i32, [_vp, _vp, _i64, _f64, _vp, _vp, _vp, _vp]),
    "oxm_fit_f64": (_i32, [_vp, _vp, _i64, _f64, _vp, _vp, _vp, _vp]),
    "oxm_expected_spectrum_f64": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "oxm_hybrid_workspace_bytes": (ctypes.c_size_t, [_vp, _i64, _i64, _i64, _i32]),
    "oxm_hybrid_em_counters": (_i32, [_vp, _vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "oxm_hybrid_maps_f32": (
        _i32,
        [_vp, _vp, _i64, _i64, _i64, _i32, _f64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "oxm_hybrid_frame_f64": (
        _i32,
        [_vp, _vp, _i64, _i64, _i64, _i32, _f64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "oxm_hybrid_maps_f32_split": (
        _i32,
        [_vp, _vp, _i64, _i64, _i64, _i32, _f64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32],
    ),
    "oxm_hybrid_maps_u16": (
        _i32,
        [_vp, _vp, _i32, _f64, _i64, _i64, _i64, _i32, _f64, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    ),
    "oxm_synth_frames_f32": (_i32, [_vp, _vp, _i64, _i64, _i64, _f64, _f64, ctypes.c_uint64, ctypes.c_uint64, _vp, _vp]),
    "oxm_synth_pulse_frames_f32": (
        _i32,
        [_vp, _vp, _i64, _i64, _i64, _f64, _f64, ctypes.c_uint64, ctypes.c_uint64, _f64, _f64, _f64, _vp, _vp],
    ),
    "oxm_patch_mean_f32": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp]),
    "oxm_pack_hwc3_f32": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "oxm_probe_fp64_fma": (_i32, [_i32, _i32, _vp, _vp, _vp]),
    "oxm_probe_mufu_lg2": (_i32, [_i32, _i32, _vp, _vp, _vp]),
    "oxm_selftest_math": (_i32, [_vp, _i64, _i32, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """The loaded library (declared signatures).  Raises NativeLibraryError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1706_07263_b200._build` "
                    "(or __graft_entry__.build()); there is no CPU fallback"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_names() -> list[str]:
    return list(_SIGNATURES)


def check(status: int, what: str) -> None:
    """Map an oxm status code onto the reference exception classes."""
    if status == OXM_OK:
        return
    lib = load()
    text = lib.oxm_status_string(status).decode()
    if status == OXM_ERR_ARGUMENT:
        raise ArgumentError(f"{what}: {text}")
    if status == OXM_ERR_DATA:
        raise DataError(f"{what}: {text}")
    if status == OXM_ERR_SINGULAR:
        raise SingularOperatorError(f"{what}: {text}")
    if status == OXM_ERR_ILL_CONDITIONED:
        raise IllConditionedPriorError(f"{what}: {text}")
    if status == OXM_ERR_NUMERICAL:
        raise NumericalError(f"{what}: {text}")
    detail = lib.oxm_last_error().decode()
    raise NativeLibraryError(f"{what}: {text} {detail}".strip())
