"""ctypes binding of the C ABI in include/undertext_b200.h.

This is the one place Python touches the native library.  There is no
fallback: if ``lib/libundertext_b200.so`` is missing or fails to load, every
compute entry point raises ``RuntimeError`` (run ``__graft_entry__.build()`` or
``python -m paper_1612_06457_b200.build``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import DataError, NumericError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libundertext_b200.so"
if os.environ.get("UT_LIB_PATH"):  # dev: a kernel-variant build (tools/build_variant.py)
    LIB_PATH = Path(os.environ["UT_LIB_PATH"]).resolve()

UT_OK, UT_EDATA, UT_ENUMERIC, UT_ECUDA = 0, 1, 2, 3
UT_U8, UT_U16, UT_F16, UT_F32, UT_F64 = 0, 1, 2, 3, 4
UT_REGION_PATH_DFMA, UT_REGION_PATH_DMMA, UT_REGION_PATH_IMMA = 0, 1, 2
INFO_OK, INFO_ASYM_A, INFO_ASYM_M, INFO_NOT_PD, INFO_NO_CONVERGE = 0, 1, 2, 3, 4

# every symbol include/undertext_b200.h declares (checked by the CPU tests)
EXPORTS = (
    "ut_version", "ut_build_hash", "ut_last_error", "ut_moment_len", "ut_gather", "ut_class_moments_ws",
    "ut_class_moments", "ut_standardize", "ut_cube_class_moments", "ut_cva_solve", "ut_gen_eig_sym", "ut_region_moments_ws",
    "ut_region_moments", "ut_region_last_path", "ut_region_flag_offset", "ut_pca_solve", "ut_project_ws", "ut_project_minmax",
    "ut_stretch", "ut_plane_minmax_ws", "ut_plane_minmax", "ut_linear_to_codes",
    "ut_plane_select_ws", "ut_plane_select", "ut_normalize_ws", "ut_normalize_stack",
    "ut_synth_cube", "ut_class_of", "ut_encode_ws", "ut_encode_bound", "ut_encode_png",
    "ut_encode_tiff", "ut_compose_rgb", "ut_decode_strips", "ut_decode_streams", "ut_unpredict", "ut_untile", "ut_png_unfilter",
    "ut_comm_available", "ut_comm_unique_id", "ut_comm_init", "ut_comm_destroy",
    "ut_allreduce_f64", "ut_allreduce_f32", "ut_allgather_f64",
)
UT_OP_SUM, UT_OP_MIN, UT_OP_MAX = 0, 1, 2


class Cube(C.Structure):
    _fields_ = [("data", C.c_void_p), ("dtype", C.c_int32), ("bands", C.c_int32),
                ("rows", C.c_int64), ("cols", C.c_int64), ("band_stride", C.c_int64),
                ("row_stride", C.c_int64), ("row0", C.c_int64)]


class CvaOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("within", "between", "class_means", "counts",
                                           "grand_mean", "evals", "evecs", "aux", "info")]


class PcaOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("mean", "std", "corr", "evals", "evecs", "info")]


_lock = threading.Lock()
_lib = None

P = C.c_void_p
I32, I64, SZ, F64 = C.c_int32, C.c_int64, C.c_size_t, C.c_double

_SIGS = {
    "ut_version": (I32, []),
    "ut_build_hash": (C.c_char_p, []),
    "ut_last_error": (C.c_char_p, []),
    "ut_moment_len": (I64, [I32]),
    "ut_gather": (I32, [C.POINTER(Cube), P, I64, P, I64, P, P]),
    "ut_class_moments_ws": (SZ, [I64, I32, I32]),
    "ut_class_moments": (I32, [P, I64, P, I64, I32, I32, P, P, P, SZ, P]),
    "ut_standardize": (I32, [P, I64, I32, I64, P, I64, P, P, P]),
    "ut_cube_class_moments": (I32, [C.POINTER(Cube), P, P, I64, I32, P, P, P, P, SZ, P]),
    "ut_cva_solve": (I32, [P, I32, I32, I32, F64, I32, C.POINTER(CvaOut), P]),
    "ut_gen_eig_sym": (I32, [P, P, I32, F64, P, P, P, P, P]),
    "ut_region_moments_ws": (SZ, [I32]),
    "ut_region_moments": (I32, [C.POINTER(Cube), I64, I64, I64, I64, P, P, SZ, P]),
    "ut_region_last_path": (I32, []),
    "ut_region_flag_offset": (I64, []),
    "ut_pca_solve": (I32, [P, I32, I32, C.POINTER(PcaOut), P]),
    "ut_project_ws": (SZ, []),
    "ut_project_minmax": (I32, [C.POINTER(Cube), P, I32, P, I32, P, P, I32, P, P, P, P, SZ, P]),
    "ut_stretch": (I32, [P, P, I32, I32, I64, I32, P, P]),
    "ut_plane_minmax_ws": (SZ, []),
    "ut_plane_minmax": (I32, [P, I32, I64, P, P, P, SZ, P]),
    "ut_linear_to_codes": (I32, [P, I32, I64, P, I32, P, P]),
    "ut_plane_select_ws": (SZ, []),
    "ut_plane_select": (I32, [P, I32, I64, P, P, P, SZ, P]),
    "ut_normalize_ws": (SZ, []),
    "ut_normalize_stack": (I32, [C.POINTER(Cube), I32, P, P, P, P, SZ, P]),
    "ut_synth_cube": (I32, [C.POINTER(Cube), I64, P, P, I32, P, I32, C.c_uint64, P]),
    "ut_class_of": (I32, [P, I32, P, I64, P, P]),
    "ut_compose_rgb": (I32, [P, P, P, I32, I64, P, P]),
    "ut_decode_strips": (I32, [P, P, P, I64, I32, P, P, P, P, P]),
    "ut_decode_streams": (I32, [P, P, P, I64, I32, P, P, P, I64, P, P]),
    "ut_unpredict": (I32, [P, I32, I64, I64, I32, I32, I32, P]),
    "ut_untile": (I32, [P, P, I64, I64, I64, I64, I64, I64, P]),
    "ut_png_unfilter": (I32, [P, P, I64, P, P, P]),
    "ut_encode_ws": (SZ, [I64, I64, I32, I32, I32, I64]),
    "ut_encode_bound": (I64, [I64, I64, I32, I32, I32, I64]),
    "ut_encode_png": (I32, [P, I64, I64, I32, I32, P, I64, P, P, SZ, P]),
    "ut_encode_tiff": (I32, [P, I64, I64, I32, I32, I32, I64, P, I64, P, P, P, SZ, P]),
    "ut_comm_available": (I32, []),
    "ut_comm_unique_id": (I32, [P]),
    "ut_comm_init": (I32, [P, I32, I32, I32, C.POINTER(P)]),
    "ut_comm_destroy": (I32, [P]),
    "ut_allreduce_f64": (I32, [P, P, I64, I32, P]),
    "ut_allreduce_f32": (I32, [P, P, I64, I32, P]),
    "ut_allgather_f64": (I32, [P, P, P, I64, P]),
}


def lib():
    """Load (once) and return the native library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"B200 library not built: {LIB_PATH} is missing "
                    "(run __graft_entry__.build()); there is no CPU fallback")
            _check_stamp()
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def _check_stamp() -> None:
    """Refuse a library not built from the sources beside it (build provenance)."""
    if os.environ.get("UT_LIB_PATH"):
        return  # dev variant builds carry their own flags
    from . import build

    if not (build.CSRC.is_dir() and any(build.CSRC.glob("*.cu"))):
        return  # installed without sources: nothing to compare against
    want, got = build.source_hash(), build.library_hash(LIB_PATH)
    if got != want:
        raise RuntimeError(
            f"B200 library {LIB_PATH} was built from other sources (stamp {got}, "
            f"sources {want}); rebuild it with __graft_entry__.build()")


def check(rc: int, what: str) -> None:
    """Map a C-ABI status onto the reference's exception contract."""
    if rc == UT_OK:
        return
    msg = lib().ut_last_error().decode(errors="replace") or what
    if rc == UT_EDATA:
        raise DataError(msg)
    if rc == UT_ENUMERIC:
        raise NumericError(msg)
    raise RuntimeError(msg)
