"""ctypes binding of include/polar_b200.h and include/polar_b200_sim.h.

Loads the in-tree ``libpolar_b200.so`` (built by ``_build.py``).  There is no
fallback: a missing library raises ImportError at first use.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

PL_OK, PL_ERR_CONFIG, PL_ERR_PARSE, PL_ERR_CUDA, PL_ERR_ARG, PL_ERR_IO = 0, 1, 2, 3, 4, 5
PL_CHANNEL_HOST, PL_CHANNEL_DEVICE = 0, 1

# every symbol the two public headers declare
EXPORTS = (
    "pl_create", "pl_last_error", "pl_destroy", "pl_llr_stride", "pl_payload_stride",
    "pl_codeword_stride", "pl_decode", "pl_decode_host", "pl_last_launches", "pl_crc_parse",
    "pl_crc_compute", "pl_tree_build", "pl_construct_frozen_bhat", "pl_construct_frozen_ga",
    "pl_channel_generate", "pl_channel_generate_device", "pl_profile", "pl_last_kernel_ms",
    "pl_kernel_selftest", "pl_channel_generate_frames", "pl_precision", "pl_sim_point",
    "pl_format_csv_row", "pl_frozen_file_load", "pl_frozen_file_save", "pl_puncture_file_load",
    "pl_decode_packed", "pl_decode_host_packed", "pl_frame_latency", "pl_set_host_chunk", "pl_set_llr_layout",
    "pl_list_paths",
)


class pl_crc(C.Structure):
    _fields_ = [("width", C.c_int32), ("reflect", C.c_int32), ("poly", C.c_uint64),
                ("init", C.c_uint64), ("xorout", C.c_uint64)]


class pl_code(C.Structure):
    _fields_ = [("n", C.c_int32), ("k", C.c_int32), ("frozen", C.POINTER(C.c_uint8)),
                ("crc", pl_crc), ("channel_use", C.POINTER(C.c_uint8))]


class pl_pruning(C.Structure):
    _fields_ = [("rate_zero", C.c_int32), ("rate_one", C.c_int32), ("repetition", C.c_int32),
                ("single_parity", C.c_int32), ("rep_max", C.c_int32), ("spc_max", C.c_int32)]


class pl_sim_config(C.Structure):
    _fields_ = [("ebn0_db", C.c_double), ("seed", C.c_uint64), ("frame0", C.c_uint64),
                ("max_frames", C.c_uint64), ("max_fe", C.c_uint64), ("quant_scale", C.c_float),
                ("channel", C.c_int32), ("host_threads", C.c_int32), ("pad", C.c_int32),
                ("chunk_frames", C.c_int64)]


class pl_point_stats(C.Structure):
    _fields_ = [("ebn0_db", C.c_double), ("frames", C.c_uint64), ("bit_errors", C.c_uint64),
                ("frame_errors", C.c_uint64), ("esc_sum", C.c_uint64), ("ber", C.c_double),
                ("fer", C.c_double), ("ti_mbps", C.c_double), ("lat_avg_us", C.c_double),
                ("lat_worst_us", C.c_double), ("esc_mean", C.c_double)]


class pl_decoder(C.Structure):
    _fields_ = [("kind", C.c_int32), ("l", C.c_int32), ("precision", C.c_int32),
                ("pruning", pl_pruning)]


_LIB = None


def lib_path() -> str:
    # PLB_LIB: an alternative in-tree build of the same library (tuning runs)
    return os.environ.get("PLB_LIB") or _build.LIB


def lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"native library {path} is missing: run __graft_entry__.build()")
    L = C.CDLL(path)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    L.pl_create.argtypes = [vp, i32, vp, i32, vp]
    L.pl_create.restype = C.c_int
    L.pl_last_error.argtypes = [vp]
    L.pl_last_error.restype = C.c_char_p
    L.pl_destroy.argtypes = [vp]
    for f in ("pl_llr_stride", "pl_payload_stride", "pl_codeword_stride", "pl_last_launches"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = i64
    L.pl_decode.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.pl_decode_host.argtypes = [vp, vp, vp, i64, vp, vp, vp, vp, vp]
    L.pl_decode_packed.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp]
    L.pl_decode_host_packed.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp, vp, vp]
    L.pl_crc_parse.argtypes = [C.c_char_p, vp]
    L.pl_crc_compute.argtypes = [vp, vp, i64, vp]
    L.pl_tree_build.argtypes = [vp, i32, vp, vp, i32]
    L.pl_tree_build.restype = i32
    L.pl_construct_frozen_bhat.argtypes = [i32, i32, C.c_double, vp]
    L.pl_construct_frozen_ga.argtypes = [i32, i32, C.c_double, C.c_double, vp]
    L.pl_channel_generate.argtypes = [vp, C.c_double, u64, u64, i64, i32, C.c_float, vp, vp, i32]
    L.pl_channel_generate_device.argtypes = [vp, C.c_double, u64, u64, i64, i32, C.c_float, vp, vp, vp]
    L.pl_profile.argtypes = [vp, i32]
    L.pl_last_kernel_ms.argtypes = [vp, vp, vp, vp, i32]
    L.pl_last_kernel_ms.restype = i32
    L.pl_kernel_selftest.argtypes = [i32, vp]
    L.pl_channel_generate_frames.argtypes = [vp, C.c_double, u64, vp, i64, i32, C.c_float, vp, i64,
                                             vp, i64, i32]
    L.pl_precision.argtypes = [vp]
    L.pl_precision.restype = i32
    L.pl_sim_point.argtypes = [vp, vp, vp, vp]
    L.pl_format_csv_row.argtypes = [vp, C.c_char_p, i32]
    L.pl_format_csv_row.restype = i32
    L.pl_frozen_file_load.argtypes = [C.c_char_p, vp, vp, vp, i32]
    L.pl_frozen_file_save.argtypes = [C.c_char_p, i32, i32, vp]
    L.pl_puncture_file_load.argtypes = [C.c_char_p, vp, vp, i32]
    L.pl_frame_latency.argtypes = [vp, vp]
    L.pl_set_host_chunk.argtypes = [vp, i64]
    L.pl_set_llr_layout.argtypes = [vp, C.c_int32]
    L.pl_list_paths.argtypes = [vp, vp, vp]
    _LIB = L
    return L


def last_error(h) -> str:
    msg = lib().pl_last_error(h)
    return msg.decode() if msg else ""
