"""ctypes binding of libnrm_b200.so (include/nrm_b200.h).

The library is the product: there is no fallback. Importing this module on a
machine without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libnrm_b200.so"
if os.environ.get("NRM_B200_VARIANT"):  # development: tools/variants.py builds
    LIB_PATH = Path(__file__).resolve().parents[1] / "_variants" / os.environ["NRM_B200_VARIANT"] / "libnrm_b200.so"

NRM_OK, NRM_EINVAL, NRM_ENOSUPPORT, NRM_EDEGENERATE, NRM_ECUDA, NRM_ENOMEM, NRM_ESTATE = range(7)


class NrmError(RuntimeError):
    """CUDA / state failure inside libnrm_b200 (NRM_ECUDA, NRM_ENOMEM, NRM_ESTATE)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[nrm {code}] {msg}")
        self.code = code


class NoSupport(LookupError):
    """The reference returns std::nullopt (no node above the weight cutoff)."""


class BlendStats(C.Structure):
    """BlendStats (mosaic.hpp:184-189)."""

    _fields_ = [
        ("footprint_pixels", C.c_int64),
        ("blended_pixels", C.c_int64),
        ("skipped_no_support", C.c_int64),
        ("skipped_out_of_frame", C.c_int64),
    ]

    def as_tuple(self):
        return (self.footprint_pixels, self.blended_pixels, self.skipped_no_support,
                self.skipped_out_of_frame)

    def __repr__(self) -> str:
        return ("BlendStats(footprint_pixels=%d, blended_pixels=%d, skipped_no_support=%d, "
                "skipped_out_of_frame=%d)" % self.as_tuple())

    def __eq__(self, other) -> bool:
        return isinstance(other, BlendStats) and self.as_tuple() == other.as_tuple()


class Grid(C.Structure):
    _fields_ = [("x0", C.c_double), ("y0", C.c_double), ("width", C.c_int), ("height", C.c_int)]


class DetectorConfig(C.Structure):
    """nrm_detector_config = DetectorConfig (features.hpp:30-36)."""
    _fields_ = [("max_features", C.c_int), ("quality_level", C.c_double), ("nms_radius", C.c_int),
                ("ratio_test", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_U8 = C.POINTER(C.c_uint8)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)
_I = C.POINTER(C.c_int)

# (name, restype, argtypes) for every symbol declared in include/nrm_b200.h
SIGNATURES = [
    ("nrm_abi_version", C.c_int, []),
    ("nrm_last_error", C.c_char_p, []),
    ("nrm_ctx_create", C.c_int, [C.c_int, C.POINTER(_P)]),
    ("nrm_ctx_destroy", C.c_int, [_P]),
    ("nrm_ctx_set_stream", C.c_int, [_P, _P]),
    ("nrm_ctx_stream", _P, [_P]),
    ("nrm_ctx_synchronize", C.c_int, [_P]),
    ("nrm_ctx_launch_count", C.c_int, [_P, _I64]),
    ("nrm_canvas_create", C.c_int, [_P, C.POINTER(_P)]),
    ("nrm_canvas_destroy", C.c_int, [_P]),
    ("nrm_canvas_reserve", C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double]),
    ("nrm_canvas_ensure_contains", C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double]),
    ("nrm_canvas_info", C.c_int, [_P, _I64, _I64, _I, _I]),
    ("nrm_canvas_set_band", C.c_int, [_P, C.c_int, C.c_int]),
    ("nrm_canvas_download", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("nrm_canvas_upload", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("nrm_canvas_deform", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("nrm_canvas_deform_device", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("nrm_canvas_pack_rows_device", C.c_int, [_P, _P, C.c_int, _P]),
    ("nrm_canvas_unpack_rows_device", C.c_int, [_P, _P, C.c_int, _P]),
    ("nrm_canvas_occupied_count", C.c_int, [_P, _I64]),
    ("nrm_blend_frame", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, C.c_double,
                                  _P, C.c_int, C.POINTER(BlendStats)]),
    ("nrm_blend_frame_device", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int,
                                         C.c_double, _P, C.c_int, _P]),
    ("nrm_blend_frame_weighted", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, C.c_double, _P,
                                           C.c_int, _P, _P]),
    ("nrm_blend_frame_weighted_device", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, C.c_int, C.c_double,
                                                  _P, C.c_int, _P, _P]),
    ("nrm_render", C.c_int, [_P, C.c_int, _P, _I, _I, _D]),
    ("nrm_render_device", C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    ("nrm_canvas_occupied_bbox", C.c_int, [_P, _I, _I, _I, _I]),
    ("nrm_pixel_warp", C.c_int, [_P, _P, C.c_int, _P, _P, C.c_int, C.c_double, _P, _P]),
    ("nrm_node_field", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int, C.c_double, _P, _P]),
    ("nrm_node_field_device", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int, C.c_double, _P, _P]),
    ("nrm_node_field_band_device", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int, C.c_double, _P, _P, C.c_int, C.c_int]),
    ("nrm_save_png", C.c_int, [C.c_char_p, _P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]),
    ("nrm_variance_field", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int, C.c_double, _P]),
    ("nrm_variance_field_device", C.c_int, [_P, C.POINTER(Grid), _P, _P, C.c_int, C.c_double, _P]),
    ("nrm_invert_frame_boundary", C.c_int, [_P, C.c_int, C.c_int, _P, _P, C.c_int, C.c_double,
                                            C.c_double, _P, C.c_int, _I]),
    ("nrm_emdq_field", C.c_int, [_P, C.POINTER(Grid), _P, _P, _P, C.c_int, _P, C.c_int, C.c_double,
                                 C.c_int, C.c_double, _P, _P]),
    ("nrm_emdq_field_device", C.c_int, [_P, C.POINTER(Grid), _P, _P, _P, C.c_int, _P, C.c_int,
                                        C.c_double, C.c_int, C.c_double, _P, _P]),
    ("nrm_emdq_points", C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P, C.c_int, _P, C.c_int, C.c_double, C.c_int,
                                  C.c_double, _P, _P, _P, _P]),
    ("nrm_emdq_points_device", C.c_int, [_P, _P, _P, C.c_int, _P, _P, _P, C.c_int, _P, C.c_int, C.c_double,
                                         C.c_int, C.c_double, _P, _P, _P, _P]),
    ("nrm_blend_frames_device", C.c_int, [_P, C.c_int, _P, C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_double, _P,
                                          _P, _P]),
    ("nrm_detect_features", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(DetectorConfig), _P, _P, _I]),
    ("nrm_detect_features_gray", C.c_int, [_P, _P, C.c_int, C.c_int, C.POINTER(DetectorConfig), _P, _P, _I]),
    ("nrm_detect_features_device", C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, C.POINTER(DetectorConfig), _P,
                                             _P, _P]),
    ("nrm_match_features", C.c_int, [_P, _P, _P, C.c_int, _P, _P, C.c_int, C.c_double, _P, _I]),
    ("nrm_match_features_device", C.c_int, [_P, _P, _P, C.c_int, _P, _P, C.c_int, C.c_double, _P, _P]),
    ("nrm_selftest_libm", C.c_int, [_P, _P, _P, C.c_int, _P, _P]),
    ("nrm_selftest_peak", C.c_int, [_P, C.c_int, _D]),
    ("nrm_ctx_exceptions", C.c_int, [_P, _I64, _I64]),
    ("nrm_ctx_set_exception_capacity", C.c_int, [_P, C.c_int64]),
    ("nrm_ctx_spilled_launches", C.c_int, [_P, _I64]),
    ("nrm_ctx_profile", C.c_int, [_P, C.c_int]),
    ("nrm_ctx_profile_read", C.c_int, [_P, C.c_char_p, C.c_int, _P, _P, C.c_int, _I]),
    ("nrm_plan_ensure_contains", C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double,
                                           C.c_double, C.c_double, _I64, _I64, _I, _I]),
    ("nrm_plan_footprint", C.c_int, [_P, C.c_int, C.c_int64, C.c_int64, _I64, _I64]),
    ("nrm_band_owns_row", C.c_int, [C.c_int64, C.c_int, C.c_int]),
]

_lib: C.CDLL | None = None


def load() -> C.CDLL:
    """Loads libnrm_b200.so (raising if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2103_07414_b200.build` "
                          "(the CUDA library is required; there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == NRM_OK:
        return
    msg = load().nrm_last_error().decode(errors="replace")
    if rc == NRM_EINVAL:
        raise ValueError(msg)
    if rc == NRM_ENOSUPPORT:
        raise NoSupport(msg)
    if rc == NRM_EDEGENERATE:
        raise ValueError(msg)
    raise NrmError(rc, msg)
