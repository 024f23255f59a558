"""ctypes binding of libkvf.so (include/kvf.h).

Mirrors the C structs field for field.  Loading fails loudly: there is no CPU
fallback for any hot-path call — a missing or stale library is an error.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkvf.so")

KVF_OK, KVF_EINVAL, KVF_ECUDA, KVF_EUNSUPPORTED, KVF_EDECODE = range(5)
KVF_BF16, KVF_F16, KVF_F32, KVF_I8 = range(4)
KVF_PACK_AUTO, KVF_PACK_TWO_PASS, KVF_PACK_SINGLE_READ = range(3)
KVF_MAX_UNITS = 128
ABI_VERSION = 1


class kvf_plan(C.Structure):
    _fields_ = [
        ("T", C.c_int32), ("H", C.c_int32), ("D", C.c_int32),
        ("a_h", C.c_int32), ("b_h", C.c_int32), ("a_d", C.c_int32), ("b_d", C.c_int32),
        ("F", C.c_int32),
        ("tiles_per_frame", C.c_int32), ("grid_rows", C.c_int32), ("grid_cols", C.c_int32),
        ("frame_h", C.c_int32), ("frame_w", C.c_int32), ("frame_count", C.c_int32),
        ("group_size", C.c_int32),
    ]


class kvf_surface(C.Structure):
    _fields_ = [
        ("base", C.c_void_p),
        ("frame_stride", C.c_int64),
        ("plane_stride", C.c_int64),
        ("row_pitch", C.c_int64),
    ]


class kvf_paged(C.Structure):
    _fields_ = [
        ("layer", C.c_void_p * 3),
        ("block_table", C.c_void_p),
        ("block_size", C.c_int32),
        ("dtype", C.c_int32),
        ("block_stride", C.c_int64),
        ("slot_stride", C.c_int64),
        ("head_stride", C.c_int64),
        ("token_base", C.c_int32),
        ("reserved_", C.c_int32),
    ]


class kvf_restore_unit(C.Structure):
    _fields_ = [
        ("frames", kvf_surface),
        ("plan", kvf_plan),
        ("scales", C.c_void_p),
        ("dst", kvf_paged),
        ("first_frame", C.c_int32),
        ("n_frames", C.c_int32),
    ]


class kvf_pack_unit(C.Structure):
    _fields_ = [
        ("src", kvf_paged),
        ("plan", kvf_plan),
        ("absmax", C.c_void_p),
        ("scales", C.c_void_p),
        ("frames", kvf_surface),
    ]


class kvf_kvfc_info(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int32),
        ("height", C.c_int32),
        ("width", C.c_int32),
        ("bitmap_len", C.c_int32),
    ]


class kvf_rc_stream(C.Structure):
    _fields_ = [
        ("payload", C.c_void_p),
        ("len", C.c_int64),
        ("symbols", C.c_void_p),
        ("n_symbols", C.c_int64),
    ]


class kvf_feed_seg(C.Structure):
    _fields_ = [
        ("src", C.c_void_p),
        ("dst", C.c_void_p),
        ("len", C.c_int64),
    ]


class kvf_recon_plane(C.Structure):
    _fields_ = [
        ("symbols", C.c_void_p),
        ("modes", C.c_void_p),
        ("out", C.c_void_p),
        ("out_pitch", C.c_int64),
    ]


class kvf_resid_plane(C.Structure):
    _fields_ = [
        ("cur", C.c_void_p),
        ("prev", C.c_void_p),
        ("pitch", C.c_int64),
        ("symbols", C.c_void_p),
        ("modes", C.c_void_p),
        ("height", C.c_int32),
        ("width", C.c_int32),
    ]


class kvf_piece(C.Structure):
    _fields_ = [
        ("src", C.c_void_p),
        ("dst_off", C.c_int64),
        ("len", C.c_int64),
        ("pack_bits", C.c_int32),
        ("reserved_", C.c_int32),
    ]


class kvf_recon_chain(C.Structure):
    _fields_ = [
        ("first", C.c_int32),
        ("count", C.c_int32),
        ("height", C.c_int32),
        ("width", C.c_int32),
    ]


# symbol -> (restype, argtypes)
_VP = C.c_void_p
_SIGNATURES = {
    "kvf_abi_version": (C.c_int32, []),
    "kvf_last_error": (C.c_char_p, []),
    "kvf_plan_init": (C.c_int, [C.POINTER(kvf_plan)]),
    "kvf_plan_frame_bytes": (C.c_int64, [C.POINTER(kvf_plan)]),
    "kvf_restore": (C.c_int, [C.POINTER(kvf_surface), C.c_int32, C.c_int32,
                              C.POINTER(kvf_plan), _VP, C.POINTER(kvf_paged), _VP]),
    "kvf_restore_batch": (C.c_int, [C.POINTER(kvf_restore_unit), C.c_int32, _VP]),
    "kvf_pack_absmax": (C.c_int, [C.POINTER(kvf_paged), C.POINTER(kvf_plan), _VP, _VP]),
    "kvf_pack_frames": (C.c_int, [C.POINTER(kvf_paged), C.POINTER(kvf_plan), _VP, _VP,
                                  C.POINTER(kvf_surface), _VP]),
    "kvf_pack_batch": (C.c_int, [C.POINTER(kvf_pack_unit), C.c_int32, _VP]),
    "kvf_pack_frames_batch": (C.c_int, [C.POINTER(kvf_pack_unit), C.c_int32, _VP]),
    "kvf_pack_batch_ex": (C.c_int, [C.POINTER(kvf_pack_unit), C.c_int32, C.c_int32, C.c_int64,
                                    _VP]),
    "kvf_pack_scratch_words": (C.c_int64, [C.POINTER(kvf_plan)]),
    "kvf_quantize": (C.c_int, [_VP, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                               _VP, _VP, _VP, _VP]),
    "kvf_dequantize": (C.c_int, [_VP, _VP, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                 _VP, C.c_int32, _VP]),
    "kvf_ar1_scan": (C.c_int, [_VP, C.c_int64, C.c_int64, C.c_int64, C.c_float, _VP]),
    "kvf_kvfc_scan": (C.c_int, [_VP, C.c_int64, C.POINTER(kvf_kvfc_info), _VP, _VP, _VP, _VP,
                                C.c_int32, C.POINTER(C.c_int32)]),
    "kvf_kvfc_scan_batch": (C.c_int, [_VP, _VP, C.c_int32, _VP, _VP, _VP, _VP, _VP, _VP,
                                      C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kvf_restore_batch_heads": (C.c_int, [C.POINTER(kvf_restore_unit), C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_int64, C.c_int32, _VP]),
    "kvf_rc_decode": (C.c_int, [_VP, C.c_int32, _VP]),
    "kvf_rc_decode_fed": (C.c_int, [_VP, C.c_int32, _VP, _VP, C.c_int32, C.c_int32, C.c_int64,
                                    _VP, C.c_int32, _VP]),
    "kvf_kvfc_reconstruct": (C.c_int, [_VP, _VP, C.c_int32, _VP]),
    "kvf_kvfc_residuals": (C.c_int, [_VP, C.c_int32, C.c_int32, _VP]),
    "kvf_rc_encode": (C.c_int, [_VP, C.c_int32, _VP, _VP]),
    "kvf_gather": (C.c_int, [_VP, C.c_int32, _VP, _VP]),
}

_lib = None


class KvfError(RuntimeError):
    """A libkvf call failed (status, message)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"libkvf status {status}: {message}")
        self.status = status
        self.message = message


def load() -> C.CDLL:
    """Load libkvf.so once; raise if it is missing or its ABI does not match."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2602_09725_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.kvf_abi_version() != ABI_VERSION:
        raise RuntimeError("libkvf ABI version mismatch; rebuild the library")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == KVF_OK:
        return
    msg = load().kvf_last_error().decode(errors="replace")
    if status == KVF_EINVAL:
        raise ValueError(msg)
    raise KvfError(status, msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def declared_symbols(header: str | None = None) -> list[str]:
    """Function names declared in include/kvf.h (used by the export test)."""
    import re

    header = header or os.path.join(os.path.dirname(HERE), "include", "kvf.h")
    text = open(header).read()
    return sorted(set(re.findall(r"^[a-z_0-9 \*]+?\b(kvf_[a-z_0-9]+)\(", text, re.M)))
