"""ctypes signatures of ``libcoe_cuda.so`` (``include/coe_cuda.h``)."""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_float, c_int, c_int32, c_int64, c_uint64, c_void_p


class MlpConfig(ctypes.Structure):
    _fields_ = [
        ("d", c_int32), ("h", c_int32), ("T", c_int32),
        ("x", c_void_p), ("act0", c_void_p), ("act1", c_void_p), ("act_rows", c_int64),
        ("h_scratch", c_void_p), ("h_rows", c_int64),
        ("slab", c_void_p), ("num_slots", c_int32), ("slot_stride_bytes", c_int64), ("act_ld", c_int32),
        ("x_rows", c_int64),
    ]


class MlpGroup(ctypes.Structure):
    _fields_ = [("rows", c_int32), ("slot", c_int32), ("batch", c_int32), ("h_row", c_int32),
                ("tile_start", c_int32), ("pad", c_int32 * 3)]


def declare(lib: ctypes.CDLL) -> None:
    lib.coe_cuda_last_error.argtypes = []
    lib.coe_cuda_last_error.restype = c_char_p
    lib.coe_group_sort_scratch_bytes.argtypes = [c_int64]
    lib.coe_group_sort_scratch_bytes.restype = c_int64
    lib.coe_group_sort.argtypes = [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.coe_group_sort.restype = c_int
    lib.coe_run_compact_scratch_bytes.argtypes = [c_int64, c_int, c_int]
    lib.coe_run_compact_scratch_bytes.restype = c_int64
    lib.coe_run_compact.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int,
                                    c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.coe_run_compact.restype = c_int
    lib.coe_mlp_create.argtypes = [POINTER(MlpConfig), POINTER(c_void_p)]
    lib.coe_mlp_create.restype = c_int
    lib.coe_mlp_destroy.argtypes = [c_void_p]
    lib.coe_mlp_destroy.restype = None
    lib.coe_mlp_max_groups.argtypes = []
    lib.coe_mlp_max_groups.restype = c_int
    lib.coe_grouped_mlp.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                    c_int, c_int, c_void_p]
    lib.coe_grouped_mlp.restype = c_int
    lib.coe_fill_uniform_bf16.argtypes = [c_void_p, c_int64, c_uint64, c_float, c_void_p]
    lib.coe_fill_uniform_bf16.restype = c_int
    lib.coe_fill_uniform_bf16_at.argtypes = [c_void_p, c_int64, c_int64, c_uint64, c_float, c_void_p]
    lib.coe_fill_uniform_bf16_at.restype = c_int


def check(lib: ctypes.CDLL, code: int, what: str = "") -> None:
    if code != 0:
        raise RuntimeError(f"{what}: {lib.coe_cuda_last_error().decode()} (code {code})")
