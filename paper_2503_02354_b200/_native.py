"""ctypes bindings to the in-tree native libraries.

* ``libcoe_planner.so`` -- host planner (``include/coe_planner.h``), plain C++.
* ``libcoe_cuda.so``    -- sm_100a kernels + runtime (``include/coe_cuda.h``).

Both are built in-tree by ``build.py`` (``__graft_entry__.build``).  There is
no fallback: a missing library raises ``ImportError`` with the build command.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
PLANNER_LIB = os.path.join(_HERE, "libcoe_planner.so")
CUDA_LIB = os.path.join(_HERE, "libcoe_cuda.so")

COE_OK = 0
COE_ERR_CONFIG = 2
COE_ERR_STARVATION = 3
COE_ERR_RUNTIME = 4
COE_ERR_VALUE = 5
COE_ERR_CUDA = 6

EVENT_NAMES = ("arrival", "assign", "evict", "load", "load_done", "batch_start", "batch_done",
               "follow_up", "complete")
OP_LOAD, OP_BATCH = 0, 1
TIER_NAMES = ("device", "host", "ssd", "peer")  # "peer": the (f3) NVLink tier extension
TIER_HOST, TIER_SSD, TIER_PEER = 1, 2, 3


class PlanConfig(ctypes.Structure):
    _fields_ = [
        ("num_experts", c_int32),
        ("expert_bytes", POINTER(c_int64)),
        ("usage_prob", POINTER(c_double)),
        ("expert_arch", POINTER(c_int32)),
        ("upstream_offsets", POINTER(c_int32)),
        ("upstream_index", POINTER(c_int32)),
        ("desc_order", POINTER(c_int32)),
        ("num_arches", c_int32),
        ("perf_valid", POINTER(c_uint8)),
        ("perf_max_batch", POINTER(c_int32)),
        ("perf_k", POINTER(c_double)),
        ("perf_b", POINTER(c_double)),
        ("cost_valid", POINTER(c_uint8)),
        ("cost_k", POINTER(c_double)),
        ("cost_b", POINTER(c_double)),
        ("cost_n_sat", POINTER(c_int64)),
        ("cost_gamma", POINTER(c_double)),
        ("cost_base_bytes", POINTER(c_int64)),
        ("cost_per_item_bytes", POINTER(c_int64)),
        ("numa", c_int32),
        ("host_bw", c_double),
        ("host_overhead", c_double),
        ("ssd_bw", c_double),
        ("ssd_overhead", c_double),
        ("host_mode", c_int32),
        ("host_cache_budget", c_double),
        ("num_executors", c_int32),
        ("exec_proc", POINTER(c_int32)),
        ("exec_expert_budget", POINTER(c_double)),
        ("exec_inference_budget", POINTER(c_double)),
        ("exec_k_scale", POINTER(c_double)),
        ("assign_makespan", c_int32),
        ("arrange", c_int32),
        ("evict", c_int32),
        ("num_requests", c_int32),
        ("request_id", POINTER(c_int64)),
        ("arrival_s", POINTER(c_double)),
        ("chain_offsets", POINTER(c_int32)),
        ("chain_experts", POINTER(c_int32)),
        ("record_trace", c_int32),
        ("record_ops", c_int32),
        ("peer_enabled", c_int32),
        ("peer_bw", c_double),
        ("peer_overhead", c_double),
    ]


class PlanMetrics(ctypes.Structure):
    _fields_ = [
        ("completed", c_int64),
        ("follow_ups", c_int64),
        ("makespan_s", c_double),
        ("evictions", c_int64),
        ("stale_predictions", c_int64),
        ("sched_wall_s", c_double),
        ("sched_calls", c_int64),
    ]


class Op(ctypes.Structure):
    _fields_ = [
        ("executor", c_int32),
        ("kind", c_int32),
        ("expert", c_int32),
        ("count", c_int32),
        ("offset", c_int64),
        ("time_s", c_double),
        ("tier", c_int32),
        ("seq", c_int32),
    ]


class Admission(ctypes.Structure):
    _fields_ = [("executor", c_int32), ("run_rank", c_int32), ("request", c_int32), ("stage", c_int32)]


_planner = None
_cuda = None


def _missing(path: str) -> ImportError:
    return ImportError(
        f"native library {os.path.basename(path)} not built at {path}; run `python build.py` "
        f"(or __graft_entry__.build()) first -- there is no Python fallback")


def planner_lib() -> ctypes.CDLL:
    global _planner
    if _planner is None:
        if not os.path.exists(PLANNER_LIB):
            raise _missing(PLANNER_LIB)
        lib = ctypes.CDLL(PLANNER_LIB)
        lib.coe_plan_create.argtypes = [POINTER(PlanConfig), POINTER(c_void_p)]
        lib.coe_plan_create.restype = c_int
        lib.coe_plan_run.argtypes = [c_void_p]
        lib.coe_plan_run.restype = c_int
        lib.coe_plan_destroy.argtypes = [c_void_p]
        lib.coe_plan_destroy.restype = None
        lib.coe_plan_last_error.argtypes = []
        lib.coe_plan_last_error.restype = c_char_p
        lib.coe_plan_metrics_get.argtypes = [c_void_p, POINTER(PlanMetrics)]
        lib.coe_plan_executor_stats.argtypes = [c_void_p, POINTER(c_double), POINTER(c_int64)]
        lib.coe_plan_trace_len.argtypes = [c_void_p]
        lib.coe_plan_trace_len.restype = c_int64
        lib.coe_plan_trace.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
        lib.coe_plan_initial_residency.argtypes = [c_void_p, c_void_p, c_void_p]
        lib.coe_plan_num_ops.argtypes = [c_void_p]
        lib.coe_plan_num_ops.restype = c_int64
        lib.coe_plan_ops.argtypes = [c_void_p]
        lib.coe_plan_ops.restype = POINTER(Op)
        lib.coe_plan_num_op_args.argtypes = [c_void_p]
        lib.coe_plan_num_op_args.restype = c_int64
        lib.coe_plan_op_args.argtypes = [c_void_p]
        lib.coe_plan_op_args.restype = POINTER(c_int32)
        lib.coe_plan_num_admissions.argtypes = [c_void_p]
        lib.coe_plan_num_admissions.restype = c_int64
        lib.coe_plan_admissions.argtypes = [c_void_p]
        lib.coe_plan_admissions.restype = POINTER(Admission)
        _planner = lib
    return _planner


def cuda_lib() -> ctypes.CDLL:
    """The sm_100a kernel library; raises if it was not built."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB):
            raise _missing(CUDA_LIB)
        _cuda = ctypes.CDLL(CUDA_LIB)
        from . import _cuda_sigs

        _cuda_sigs.declare(_cuda)
    return _cuda
