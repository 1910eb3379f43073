"""Host-side driver of the B200 serving runtime (``libcoe_cuda.so``).

``B200Runtime`` owns one executor's GPU state: the fixed-budget HBM expert
cache (slots), the pinned host expert store, activation buffers and the
compute / copy streams.  ``step(plan)`` hands the native planner's op log
(``engine.Plan``) to ``coe_runtime_step`` zero-copy; everything after that is
stream-ordered GPU work (K1 group sort, K2 compaction, K3 grouped MLP waves,
K4 swap-ins).  There is no CPU fallback: constructing a runtime without the
CUDA library or a GPU raises.

Reference seams: the *device* seam of ``CostModel``
(costmodel.py:39-92) gains physical ``execute`` / ``swap_in`` behaviour here,
while the numeric returns of the cost model keep driving decisions.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from ._cuda_sigs import check as _check

DEFAULT_WEIGHT_SEED = 0xC0E5E4E
DEFAULT_INPUT_SEED = 0x1A7E5
POOL_UNIT = 2 << 20  # allocation unit of the pooled expert slab (runtime.cu kPoolUnit)


class StepInput(ctypes.Structure):
    _fields_ = [
        ("executor", ctypes.c_int32),
        ("num_admissions", ctypes.c_int64), ("admissions", ctypes.c_void_p),
        ("num_ops", ctypes.c_int64), ("ops", ctypes.c_void_p),
        ("num_op_args", ctypes.c_int64), ("op_args", ctypes.c_void_p),
        ("num_initial", ctypes.c_int32), ("initial", ctypes.c_void_p),
        ("host_inputs", ctypes.c_void_p), ("host_outputs", ctypes.c_void_p),
        ("num_executors", ctypes.c_int32), ("initial_offsets", ctypes.c_void_p), ("initial_all", ctypes.c_void_p),
    ]


class StepStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("admissions", "batches", "waves", "launches", "h2d_input_bytes",
                                               "d2h_output_bytes", "loads", "load_bytes",
                                               "restores", "restore_bytes", "max_wave_rows")] + \
               [("max_wave_groups", ctypes.c_int32), ("rank_bits", ctypes.c_int32), ("ring_peak", ctypes.c_int32),
                ("landing_rows", ctypes.c_int32), ("peer_loads", ctypes.c_int64), ("peer_bytes", ctypes.c_int64),
                ("peer_tier_loads", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class StepTiming(ctypes.Structure):
    _fields_ = [(n, ctypes.c_float) for n in ("total_ms", "copy_busy_ms", "compute_busy_ms", "overlap_ms", "mlp_ms",
                                               "group_ms", "k3_busy_ms")] + \
               [("k3_launches", ctypes.c_int32), ("k3_flops", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {name: float(getattr(self, name)) for name, _ in self._fields_}


class PeerBuffers(ctypes.Structure):
    _fields_ = [("p0", ctypes.c_void_p), ("p1", ctypes.c_void_p), ("flags", ctypes.c_void_p)]


IPC_HANDLE_BYTES = 3 * 64  # P0, P1, flags (cudaIpcMemHandle_t each)


class RuntimeConfig(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("h", ctypes.c_int32), ("T", ctypes.c_int32),
                ("num_experts", ctypes.c_int32), ("num_slots", ctypes.c_int32), ("max_requests", ctypes.c_int32),
                ("max_wave_rows", ctypes.c_int64), ("max_admissions", ctypes.c_int64),
                ("max_batches", ctypes.c_int64), ("weight_seed", ctypes.c_uint64), ("profile", ctypes.c_int32),
                ("reserve_sms", ctypes.c_int32), ("swapped_stream", ctypes.c_int32), ("store_path", ctypes.c_char_p),
                ("wave_rows_cap", ctypes.c_int64), ("urgent_rows_cap", ctypes.c_int64),
                ("num_shapes", ctypes.c_int32), ("shape_d", ctypes.c_void_p), ("shape_h", ctypes.c_void_p),
                ("shape_slots", ctypes.c_void_p), ("expert_shape", ctypes.c_void_p), ("store_mask", ctypes.c_void_p),
                ("ring_slots", ctypes.c_int32), ("landing_slots", ctypes.c_int32), ("out_slots", ctypes.c_int32),
                ("device_io", ctypes.c_int32), ("expert_pool_bytes", ctypes.c_int64)]


_declared = False


def _lib():
    global _declared
    lib = _native.cuda_lib()
    if not _declared:
        P, V, I32, I64 = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.coe_runtime_create.argtypes = [P(RuntimeConfig), P(V)]
        lib.coe_runtime_destroy.argtypes = [V]
        lib.coe_runtime_destroy.restype = None
        lib.coe_runtime_init_experts.argtypes = [V]
        lib.coe_runtime_fill_inputs.argtypes = [V, ctypes.c_uint64, I32]
        lib.coe_runtime_upload_inputs.argtypes = [V, V, I32]
        lib.coe_runtime_step.argtypes = [V, P(StepInput), P(StepStats)]
        lib.coe_runtime_download_outputs.argtypes = [V, V, I32, V]
        lib.coe_runtime_synchronize.argtypes = [V]
        lib.coe_runtime_download_requests.argtypes = [V, V, V, I32, V]
        lib.coe_runtime_check.argtypes = [V, P(I32), P(I32)]
        lib.coe_runtime_members.argtypes = [V, V, V, V]
        lib.coe_runtime_timing.argtypes = [V, P(StepTiming)]
        lib.coe_runtime_buffer.argtypes = [V, ctypes.c_int]
        lib.coe_runtime_buffer.restype = V
        lib.coe_runtime_slot_of.argtypes = [V, I32]
        lib.coe_runtime_bench_mlp.argtypes = [V, I32, I32, I32, P(ctypes.c_float), P(ctypes.c_float)]
        lib.coe_runtime_bench_mlp.restype = ctypes.c_int
        lib.coe_comm_unique_id.argtypes = [ctypes.c_char_p, V]
        lib.coe_comm_unique_id.restype = ctypes.c_int
        lib.coe_comm_create.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, V, P(V)]
        lib.coe_comm_create.restype = ctypes.c_int
        lib.coe_comm_destroy.argtypes = [V]
        lib.coe_comm_destroy.restype = None
        lib.coe_local_hub_create.argtypes = [ctypes.c_int]
        lib.coe_local_hub_create.restype = V
        lib.coe_local_hub_destroy.argtypes = [V]
        lib.coe_local_hub_destroy.restype = None
        lib.coe_local_hub_reset.argtypes = [V]
        lib.coe_local_hub_reset.restype = None
        lib.coe_comm_create_local.argtypes = [V, ctypes.c_int, P(V)]
        lib.coe_comm_create_local.restype = ctypes.c_int
        lib.coe_runtime_set_knobs.argtypes = [V, I64, I64, I32]
        lib.coe_runtime_set_knobs.restype = ctypes.c_int
        lib.coe_runtime_attach_comm.argtypes = [V, V]
        lib.coe_runtime_attach_comm.restype = ctypes.c_int
        lib.coe_runtime_counts.argtypes = [V, P(I32), P(I32)]
        lib.coe_runtime_counts.restype = ctypes.c_int
        lib.coe_runtime_intervals.argtypes = [V, V, V, V]
        lib.coe_runtime_intervals.restype = ctypes.c_int
        lib.coe_runtime_join.argtypes = [V]
        lib.coe_runtime_join.restype = ctypes.c_int
        lib.coe_runtime_output_order.argtypes = [V, V, I32]
        lib.coe_runtime_output_order.restype = I32
        lib.coe_runtime_io_intervals.argtypes = [V, V, P(I32), P(I32)]
        lib.coe_runtime_io_intervals.restype = ctypes.c_int
        lib.coe_runtime_wave_phases.argtypes = [V, V, V]
        lib.coe_runtime_wave_phases.restype = ctypes.c_int
        lib.coe_runtime_read_buffer.argtypes = [V, ctypes.c_int, V, I64]
        lib.coe_runtime_read_buffer.restype = ctypes.c_int
        lib.coe_runtime_stream.argtypes = [V, ctypes.c_int]
        lib.coe_runtime_stream.restype = V
        lib.coe_runtime_peer_buffers.argtypes = [V, P(PeerBuffers)]
        lib.coe_runtime_peer_buffers.restype = ctypes.c_int
        lib.coe_runtime_ipc_export.argtypes = [V, V]
        lib.coe_runtime_ipc_export.restype = ctypes.c_int
        lib.coe_runtime_ipc_open.argtypes = [V, V, P(PeerBuffers)]
        lib.coe_runtime_ipc_open.restype = ctypes.c_int
        lib.coe_runtime_attach_peers.argtypes = [V, I32, I32, V, V]
        lib.coe_runtime_attach_peers.restype = ctypes.c_int
        lib.coe_runtime_attach_local_experts.argtypes = [V, V, I32]
        lib.coe_runtime_attach_local_experts.restype = ctypes.c_int
        lib.coe_runtime_ipc_export_experts.argtypes = [V, V, P(I32)]
        lib.coe_runtime_ipc_export_experts.restype = ctypes.c_int
        lib.coe_runtime_ipc_open_experts.argtypes = [V, I32, V, I32]
        lib.coe_runtime_ipc_open_experts.restype = ctypes.c_int
        lib.coe_runtime_residency_codes.argtypes = [V, V]
        lib.coe_runtime_residency_codes.restype = ctypes.c_int
        lib.coe_runtime_set_peer_residency.argtypes = [V, I32, V]
        lib.coe_runtime_set_peer_residency.restype = ctypes.c_int
        lib.coe_runtime_plan_rows.argtypes = [P(StepInput), I32, ctypes.c_int, ctypes.c_int, P(I32), P(I32)]
        lib.coe_runtime_plan_rows.restype = ctypes.c_int
        lib.coe_expert_seed.argtypes = [ctypes.c_uint64, I32, I32]
        lib.coe_expert_seed.restype = ctypes.c_uint64
        for name in ("coe_runtime_create", "coe_runtime_init_experts", "coe_runtime_fill_inputs",
                     "coe_runtime_upload_inputs", "coe_runtime_step", "coe_runtime_download_outputs",
                     "coe_runtime_download_requests",
                     "coe_runtime_synchronize", "coe_runtime_check", "coe_runtime_members", "coe_runtime_timing",
                     "coe_runtime_slot_of"):
            getattr(lib, name).restype = ctypes.c_int
        _declared = True
    return lib


def expert_seed(weight_seed: int, expert: int, matrix: int) -> int:
    return int(_lib().coe_expert_seed(weight_seed, expert, matrix))


@dataclass(frozen=True)
class RuntimeShape:
    d: int
    h: int
    T: int

    @property
    def expert_bytes(self) -> int:
        return 2 * self.d * self.h * 2


def shape_of(workload):
    """The workload's expert shape: one ``RuntimeShape`` when every arch shares it, else the
    ``{arch: (d, h, T)}`` map (heterogeneous experts; ``B200Runtime.for_plan`` accepts both)."""
    shapes = set(workload.shapes.values())
    if len(shapes) == 1:
        d, h, T = shapes.pop()
        return RuntimeShape(d, h, T)
    return dict(workload.shapes)


class B200Runtime:
    """One executor's GPU serving state (see module docstring)."""

    def __init__(self, shape, num_experts: int, num_slots, max_requests: int,
                 max_admissions: int, max_wave_rows: int | None = None, weight_seed: int = DEFAULT_WEIGHT_SEED,
                 profile: bool = False, init_experts: bool = True, reserve_sms: int = 0,
                 store_path: str | None = None, wave_rows_cap: int | None = None,
                 urgent_rows_cap: int | None = 8192, expert_shape=None, store_mask=None,
                 ring_slots: int | None = None, landing_slots: int = 0, out_slots: int = 0,
                 device_io: bool = True, expert_pool_bytes: int = 0):
        """``shape``: one ``RuntimeShape`` or a list (heterogeneous experts, ``expert_shape``
        maps each expert to its index); ``num_slots``: HBM slots (per shape for a list).
        ``ring_slots`` / ``landing_slots``: activation rows (``plan_rows``; default: one ring
        slot per request); ``device_io``: allocate the device-resident X / Y buffers."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("B200Runtime needs a CUDA device (no CPU fallback)")
        torch.cuda.init()
        self.lib = _lib()
        shapes = list(shape) if isinstance(shape, (list, tuple)) else [shape]
        slots = list(num_slots) if isinstance(num_slots, (list, tuple)) else [num_slots]
        if len({s.T for s in shapes}) != 1 or len(slots) != len(shapes):
            raise ValueError("one T for all shapes and one slot count per shape")
        self.shapes = shapes
        self.shape = shapes[0]
        self.act_ld = max(s.d for s in shapes)
        self.num_experts = num_experts
        self.num_slots = sum(slots)
        self.max_requests = max_requests
        self.weight_seed = weight_seed
        T = shapes[0].T
        rows = max_wave_rows or max(128, min(int(os.environ.get("COE_MAX_WAVE_ROWS", 32768)), max_admissions * T))
        self._keep = {
            "d": np.array([s.d for s in shapes], np.int32), "h": np.array([s.h for s in shapes], np.int32),
            "slots": np.array(slots, np.int32),
            "es": np.ascontiguousarray(expert_shape if expert_shape is not None else np.zeros(num_experts), np.int32),
            "mask": None if store_mask is None else np.ascontiguousarray(store_mask, np.uint8),
        }
        k = self._keep
        cfg = RuntimeConfig(shapes[0].d, shapes[0].h, T, num_experts, slots[0], max_requests, rows, max_admissions,
                            max_admissions, weight_seed, 1 if profile else 0,
                            int(os.environ.get("COE_RESERVE_SMS", reserve_sms)), 0,
                            store_path.encode() if store_path else None,
                            int(os.environ.get("COE_WAVE_ROWS", wave_rows_cap or 0)),
                            int(os.environ.get("COE_URGENT_ROWS", urgent_rows_cap or 0)),
                            len(shapes), k["d"].ctypes.data, k["h"].ctypes.data, k["slots"].ctypes.data,
                            k["es"].ctypes.data, None if k["mask"] is None else k["mask"].ctypes.data,
                            int(ring_slots if ring_slots is not None else max_requests), int(landing_slots),
                            int(out_slots), 1 if device_io else 0, int(expert_pool_bytes))
        self.expert_pool_bytes = int(expert_pool_bytes)
        self.ring_slots = cfg.ring_slots
        self.landing_slots = cfg.landing_slots
        self.device_io = device_io
        self.max_wave_rows = rows
        self.out_slots = out_slots or max(64, 2 * rows // T)

        self.profile = profile
        self.handle = ctypes.c_void_p()
        _check(self.lib, self.lib.coe_runtime_create(ctypes.byref(cfg), ctypes.byref(self.handle)), "runtime create")
        if init_experts:
            _check(self.lib, self.lib.coe_runtime_init_experts(self.handle), "init experts")

    def memory(self) -> dict:
        """Device bytes by role: expert slots (the budget), activations (ring + landing rows,
        the H scratch of the three wave streams, the e2e output staging ring) and the
        device-resident request inputs / outputs X, Y (device_io only)."""
        row = self.shapes[0].T * self.act_ld * 2
        act = {"ring": self.ring_slots * row, "landing": self.landing_slots * row,
               "h_scratch": 3 * self.max_wave_rows * max(s.h for s in self.shapes) * 2,
               "out_staging": self.out_slots * row}
        slots = self.expert_pool_bytes or sum(n * s.expert_bytes
                                              for n, s in zip(self._keep["slots"].tolist(), self.shapes))
        return {"expert_slots": int(slots), "activations": act, "activations_total": int(sum(act.values())),
                "device_io_xy": (2 * self.max_requests * row) if self.device_io else 0,
                "ring_slots": self.ring_slots, "landing_rows": self.landing_slots}

    @classmethod
    def for_plan(cls, plan, shape, executor: int = 0, **kw) -> "B200Runtime":
        """Size a runtime for a resolved plan.

        Slots per shape = min(experts of that shape this executor touches, expert budget //
        shape bytes): the planner's byte accounting (ModelPool, expert_pool.py:27-59) bounds
        how many can be resident at once.  ``shape``: a RuntimeShape (every expert that
        shape -- the committed configs, or a smaller physical stand-in), or the workload's
        ``{arch: (d, h, T)}`` map (per-expert shapes; heterogeneous configs)."""
        resolved = plan.resolved
        proc, budget, _inf, _k = resolved.executors[executor]
        if proc != "gpu":
            raise ValueError("B200Runtime serves gpu executors only")
        registry = resolved.config.registry
        ids = resolved.expert_ids
        touched = np.zeros(len(ids), np.uint8)
        stored = np.zeros(len(ids), np.uint8)  # the host tier: every expert a LOAD moves or evicts
        op_args = plan.op_args()
        for op in plan.ops():
            if op["executor"] == executor:
                touched[int(op["expert"])] = 1
                if op["kind"] == _native.OP_LOAD:
                    stored[int(op["expert"])] = 1
                    o = int(op["offset"])
                    stored[op_args[o:o + int(op["count"])]] = 1
        # (an initially resident expert the plan never evicts is generated on the device the
        # first time it runs; it never crosses PCIe, so it needs no host copy)
        adm = sum(len(c) for c in resolved.chains)
        # activation rows: the ring's peak for this executor's op log, e2e included (stage-0
        # inputs occupy slots too); with several executors also the NCCL transport's needs
        ring, landing = plan_rows(plan, executor, e2e=True)
        if len(resolved.executors) > 1:
            ring = max(ring, plan_rows(plan, executor, e2e=True, nccl=True)[0])
        kw.setdefault("ring_slots", max(1, ring))
        kw.setdefault("landing_slots", landing)
        if isinstance(shape, RuntimeShape):
            # one physical shape for every expert (the config's own, or a small stand-in for a
            # heterogeneous registry): as many slots as this executor holds at once in the
            # planner's byte accounting (never more than budget // bytes for a uniform registry)
            # (physically resident experts are always a subset of the plan's pool at that moment:
            # initial residents not yet evicted, or loaded / restored -- so its peak bounds them)
            slots = max(1, int(_peak_residency(plan, executor, np.zeros(len(ids), np.int32), 1, lazy=False)[0]))
            if not kw.get("store_path"):  # a shared store must hold every expert at fixed offsets
                kw.setdefault("store_mask", stored)
            return cls(shape, len(ids), slots, len(resolved.request_ids), adm, **kw)
        arch_shapes = shape
        width = {e: arch_shapes[registry.experts[eid].arch][0] for e, eid in enumerate(ids)}
        for r, chain in enumerate(resolved.chains):
            # activations are [T][max d] rows and an expert of width d reads the first d columns,
            # so a chain must keep one width (coe_runtime_config.num_shapes)
            if len({width[e] for e in chain}) > 1:
                raise ValueError(f"request {resolved.request_ids[r]}: its chain changes the expert width "
                                 f"({[width[e] for e in chain]}); every stage of a chain must share d")
        shapes = sorted({RuntimeShape(*arch_shapes[registry.experts[e].arch]) for e in ids},
                        key=lambda s: (s.d, s.h))
        index = {s: i for i, s in enumerate(shapes)}
        expert_shape = np.array([index[RuntimeShape(*arch_shapes[registry.experts[e].arch])] for e in ids], np.int32)
        # slots per shape = that shape's peak concurrent residency in this executor's op log
        # (initial placement, then each LOAD's victims out and its expert in): exactly what the
        # planner's byte-budgeted pool (expert_pool.py:27-59) holds at once, shape by shape
        # An initially resident expert only takes HBM once materialised: the runtime restores it
        # at its first batch (an expert this executor never runs needs no slot)
        peak = _peak_residency(plan, executor, expert_shape, len(shapes), lazy=False)
        if not kw.get("store_path"):
            kw.setdefault("store_mask", stored)
        if kw.pop("pooled", True):
            # one slab for every shape, addressed in 2 MB units: the planner's byte budget
            # (capped by what this executor ever holds at once), unit rounding per resident
            # expert, and three largest experts of slack against fragmentation (best fit, size
            # classes at opposite ends; tools/pool_sim.py)
            counts = [int((expert_shape == i).sum()) for i in range(len(shapes))]
            held = sum(int(p) * s.expert_bytes for p, s in zip(peak, shapes))
            largest = max(s.expert_bytes for s, p in zip(shapes, peak) if p > 0)
            kw.setdefault("expert_pool_bytes",
                          int(min(budget, held)) + 3 * largest + int(peak.sum()) * POOL_UNIT)
            return cls(shapes, len(ids), counts, len(resolved.request_ids), adm, expert_shape=expert_shape, **kw)
        slots = [max(1, int(p)) for p in peak]  # per-shape slabs of each shape's peak residency
        return cls(shapes, len(ids), slots, len(resolved.request_ids), adm, expert_shape=expert_shape, **kw)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.coe_runtime_destroy(self.handle)
            self.handle = None
        if getattr(self, "comm", None):
            self.lib.coe_comm_destroy(self.comm)
            self.comm = None

    def attach_local(self, hub: "LocalHub", rank: int) -> None:
        """Join an in-process hop transport (several executors sharing one GPU)."""
        self.comm = ctypes.c_void_p()
        _check(self.lib, self.lib.coe_comm_create_local(hub.handle, rank, ctypes.byref(self.comm)), "local comm")
        _check(self.lib, self.lib.coe_runtime_attach_comm(self.handle, self.comm), "attach comm")

    def attach_comm(self, rank: int, world: int) -> None:
        """Create the NCCL hop communicator (one executor per rank) and attach it.

        The 128-byte unique id travels over the default torch.distributed group."""
        import torch.distributed as dist

        path = nccl_library().encode()
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            _check(self.lib, self.lib.coe_comm_unique_id(path, uid), "nccl unique id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (ctypes.c_char * 128).from_buffer_copy(box[0])
        self.comm = ctypes.c_void_p()
        _check(self.lib, self.lib.coe_comm_create(path, rank, world, uid, ctypes.byref(self.comm)), "nccl comm")
        _check(self.lib, self.lib.coe_runtime_attach_comm(self.handle, self.comm), "attach comm")

    def peer_buffers(self) -> PeerBuffers:
        pb = PeerBuffers()
        _check(self.lib, self.lib.coe_runtime_peer_buffers(self.handle, ctypes.byref(pb)), "peer buffers")
        return pb

    def _attach_peers(self, rank: int, peers: list, hub: "LocalHub | None" = None) -> None:
        arr = (PeerBuffers * len(peers))(*peers)
        self._peer_hub = hub  # keep the hub alive as long as the runtime uses it
        _check(self.lib, self.lib.coe_runtime_attach_peers(self.handle, rank, len(peers), arr,
                                                           hub.handle if hub is not None else None), "attach peers")

    def attach_peers_ipc(self, rank: int, world: int) -> None:
        """Fused hops across processes (one executor per rank, normally one GPU each): every
        rank exports its P0 / P1 / flag buffers as CUDA IPC handles, the handles travel over
        the default torch.distributed group, and each rank maps every peer's buffers."""
        import torch.distributed as dist

        mine = (ctypes.c_char * IPC_HANDLE_BYTES)()
        _check(self.lib, self.lib.coe_runtime_ipc_export(self.handle, mine), "ipc export")
        gathered = [None] * world
        dist.all_gather_object(gathered, bytes(mine))
        peers = []
        for r in range(world):
            if r == rank:
                peers.append(self.peer_buffers())
                continue
            h = (ctypes.c_char * IPC_HANDLE_BYTES).from_buffer_copy(gathered[r])
            pb = PeerBuffers()
            _check(self.lib, self.lib.coe_runtime_ipc_open(self.handle, h, ctypes.byref(pb)), "ipc open")
            peers.append(pb)
        self._attach_peers(rank, peers)
        # (f3) expert memory too: peer-tier loads copy straight from the source rank's HBM
        exp = (ctypes.c_char * (64 * 16))()
        count = ctypes.c_int32()
        _check(self.lib, self.lib.coe_runtime_ipc_export_experts(self.handle, exp, ctypes.byref(count)), "ipc experts")
        gathered = [None] * world
        dist.all_gather_object(gathered, bytes(exp)[:64 * count.value])
        for r in range(world):
            if r != rank:
                blob = gathered[r]
                buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
                _check(self.lib, self.lib.coe_runtime_ipc_open_experts(self.handle, r, buf, len(blob) // 64),
                       "ipc open experts")
        self._ipc = (rank, world)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data --------------------------------------------------------------
    def fill_inputs(self, num_requests: int, seed: int = DEFAULT_INPUT_SEED) -> None:
        _check(self.lib, self.lib.coe_runtime_fill_inputs(self.handle, seed, num_requests), "fill inputs")

    def upload_inputs(self, host_ptr: int, num_requests: int) -> None:
        _check(self.lib, self.lib.coe_runtime_upload_inputs(self.handle, host_ptr, num_requests), "upload")

    def download_outputs(self, last_stage: np.ndarray, host_ptr: int) -> None:
        last = np.ascontiguousarray(last_stage, dtype=np.int32)
        _check(self.lib, self.lib.coe_runtime_download_outputs(self.handle, last.ctypes.data, len(last), host_ptr),
               "download")

    def download_requests(self, requests, stages) -> np.ndarray:
        """Final activations of selected requests: float32 [n, T, act_ld] (synchronous)."""
        req = np.ascontiguousarray(requests, dtype=np.int32)
        st = np.ascontiguousarray(stages, dtype=np.int32)
        if req.shape != st.shape:
            raise ValueError("one stage per request")
        T = self.shapes[0].T
        out = np.zeros((max(1, len(req)), T, self.act_ld), np.uint16)
        _check(self.lib, self.lib.coe_runtime_download_requests(self.handle, req.ctypes.data, st.ctypes.data,
                                                                len(req), out.ctypes.data), "download requests")
        return (out[:len(req)].astype(np.uint32) << 16).view(np.float32)

    def buffer(self, which: int) -> int:
        return int(self.lib.coe_runtime_buffer(self.handle, which) or 0)

    def read_buffer(self, which: int, host_ptr: int, nbytes: int) -> None:
        _check(self.lib, self.lib.coe_runtime_read_buffer(self.handle, which, host_ptr, nbytes), "read buffer")

    def stream_handle(self, which: int = 0) -> int:
        return int(self.lib.coe_runtime_stream(self.handle, which) or 0)

    # -- execution ---------------------------------------------------------
    def step(self, plan, executor: int = 0, host_inputs: int | None = None, host_outputs: int | None = None) -> dict:
        """Execute ``plan``'s op log for ``executor``.  With pinned host buffers the step is
        end to end: inputs (row r = request r) stream in just in time, final outputs stream
        out per wave in completion order (``output_order()`` names each row's request)."""
        lib = plan.lib
        h = plan.handle
        residency = plan.initial_residency()
        init = np.ascontiguousarray(residency[executor], dtype=np.int32)
        off = np.cumsum([0] + [len(r) for r in residency]).astype(np.int32)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(r, np.int32) for r in residency] + [np.zeros(1, np.int32)]))
        self._init_keep = (init, off, flat)
        inp = StepInput(
            executor,
            lib.coe_plan_num_admissions(h), ctypes.cast(lib.coe_plan_admissions(h), ctypes.c_void_p),
            lib.coe_plan_num_ops(h), ctypes.cast(lib.coe_plan_ops(h), ctypes.c_void_p),
            lib.coe_plan_num_op_args(h), ctypes.cast(lib.coe_plan_op_args(h), ctypes.c_void_p),
            len(init), init.ctypes.data if len(init) else None, host_inputs, host_outputs,
            len(residency), off.ctypes.data, flat.ctypes.data,
        )
        stats = StepStats()
        _check(self.lib, self.lib.coe_runtime_step(self.handle, ctypes.byref(inp), ctypes.byref(stats)), "step")
        if getattr(self, "_ipc", None) and _has_peer_loads(plan):
            self._exchange_residency()
        out = stats.as_dict()
        if host_outputs is not None:  # the completion order is fixed at issue time
            out["output_order"] = self.output_order()
        return out

    def _exchange_residency(self) -> None:
        """(f3, one executor per process) after every step of a plan with peer-tier loads: each
        rank's end-of-step residency (slab / offset codes) goes to every other rank, which
        copies peer-tier loads of the next step straight from that HBM (CUDA IPC mapping)."""
        import torch.distributed as dist

        rank, world = self._ipc
        n = self.num_experts
        codes = np.zeros(n, np.int64)
        _check(self.lib, self.lib.coe_runtime_residency_codes(self.handle, codes.ctypes.data), "residency")
        gathered = [None] * world
        dist.all_gather_object(gathered, codes)
        for r in range(world):
            if r != rank:
                c = np.ascontiguousarray(gathered[r], np.int64)
                _check(self.lib, self.lib.coe_runtime_set_peer_residency(self.handle, r, c.ctypes.data), "peer residency")

    def join(self) -> None:
        """Order the compute stream after the last e2e step's output downloads."""
        _check(self.lib, self.lib.coe_runtime_join(self.handle), "join")

    def synchronize(self) -> None:
        _check(self.lib, self.lib.coe_runtime_synchronize(self.handle), "synchronize")

    def check(self) -> tuple:
        runs, viol = ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib, self.lib.coe_runtime_check(self.handle, ctypes.byref(runs), ctypes.byref(viol)), "check")
        return runs.value, viol.value

    def members(self, num_admissions: int, num_batches: int):
        req = np.zeros(max(1, num_admissions), np.int32)
        stage = np.zeros(max(1, num_admissions), np.int32)
        boff = np.zeros(max(1, num_batches), np.int32)
        _check(self.lib, self.lib.coe_runtime_members(self.handle, req.ctypes.data, stage.ctypes.data,
                                                      boff.ctypes.data), "members")
        return req[:num_admissions], stage[:num_admissions], boff[:num_batches]

    def set_knobs(self, wave_rows_cap: int = 0, urgent_rows_cap: int = 0, reserve_sms: int = -1) -> None:
        _check(self.lib, self.lib.coe_runtime_set_knobs(self.handle, wave_rows_cap, urgent_rows_cap, reserve_sms),
               "set knobs")

    def intervals(self) -> dict:
        nc, nw = ctypes.c_int32(), ctypes.c_int32()
        self.lib.coe_runtime_counts(self.handle, ctypes.byref(nc), ctypes.byref(nw))
        cp = np.zeros(2 * max(1, nc.value), np.float32)
        wv = np.zeros(2 * max(1, nw.value), np.float32)
        info = np.zeros(3 * max(1, nw.value), np.int32)
        _check(self.lib, self.lib.coe_runtime_intervals(self.handle, cp.ctypes.data, wv.ctypes.data,
                                                        info.ctypes.data), "intervals")
        return {"copies": cp[:2 * nc.value].reshape(-1, 2).tolist(), "waves": wv[:2 * nw.value].reshape(-1, 2).tolist(),
                "wave_info": info[:3 * nw.value].reshape(-1, 3).tolist()}

    def wave_phases(self) -> dict:
        """Per wave: [up start, up end, down start, down end] (ms since step start) and FLOPs."""
        nc, nw = ctypes.c_int32(), ctypes.c_int32()
        self.lib.coe_runtime_counts(self.handle, ctypes.byref(nc), ctypes.byref(nw))
        iv = np.zeros(4 * max(1, nw.value), np.float32)
        fl = np.zeros(max(1, nw.value), np.float64)
        _check(self.lib, self.lib.coe_runtime_wave_phases(self.handle, iv.ctypes.data, fl.ctypes.data), "wave_phases")
        return {"phases": iv[:4 * nw.value].reshape(-1, 4).tolist(), "flops": fl[:nw.value].tolist()}

    def per_shape_k3(self) -> dict:
        """Profile mode, after a step: per expert shape, the algorithmic FLOPs of its waves and
        the GPU time they used.  K3 launches of different waves overlap (two main streams and
        the release stream), so each instant of K3 activity is shared equally among the
        launches running then (``k3_ms``; these sum to the K3 busy time of the step) ->
        achieved TFLOP/s per shape.  ``launch_ms``: the plain sum of launch durations."""
        ph = self.wave_phases()
        nw = len(ph["flops"])
        idx = np.zeros(max(1, nw), np.int32)
        self.lib.coe_runtime_wave_shapes.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        _check(self.lib, self.lib.coe_runtime_wave_shapes(self.handle, idx.ctypes.data), "wave shapes")
        keys, iv = [], []
        for i in range(nw):
            s = self.shapes[int(idx[i])]
            keys.append(f"{s.d}x{s.h}x{s.T}")
            u0, u1, d0, d1 = ph["phases"][i]
            iv += [(u0, u1, i), (d0, d1, i)]
        share = np.zeros(max(1, nw))
        edges = sorted({t for a, b, _ in iv for t in (a, b)})
        for t0, t1 in zip(edges[:-1], edges[1:]):
            active = [i for a, b, i in iv if a <= t0 and b >= t1 and b > a]
            for i in active:
                share[i] += (t1 - t0) / len(active)
        out = {}
        for i in range(nw):
            u0, u1, d0, d1 = ph["phases"][i]
            e = out.setdefault(keys[i], {"waves": 0, "flops": 0.0, "k3_ms": 0.0, "launch_ms": 0.0})
            e["waves"] += 1
            e["flops"] += ph["flops"][i]
            e["k3_ms"] += float(share[i])
            e["launch_ms"] += (u1 - u0) + (d1 - d0)
        for e in out.values():
            e["tflops"] = e["flops"] / (e["k3_ms"] / 1e3) / 1e12 if e["k3_ms"] > 0 else None
        return out

    def output_order(self) -> np.ndarray:
        """After an e2e step: the request id of each host_outputs row (completion order)."""
        n = self.lib.coe_runtime_output_order(self.handle, None, 0)
        out = np.zeros(max(1, n), np.int32)
        self.lib.coe_runtime_output_order(self.handle, out.ctypes.data, n)
        return out[:n]

    def io_intervals(self) -> dict:
        """e2e steps (profile mode): input-upload and output-download [start, end] ms."""
        ni, no = ctypes.c_int32(), ctypes.c_int32()
        _check(self.lib, self.lib.coe_runtime_io_intervals(self.handle, None, ctypes.byref(ni), ctypes.byref(no)), "io")
        iv = np.zeros(2 * (ni.value + no.value) + 1, np.float32)
        _check(self.lib, self.lib.coe_runtime_io_intervals(self.handle, iv.ctypes.data, ctypes.byref(ni),
                                                           ctypes.byref(no)), "io")
        pairs = iv[:2 * (ni.value + no.value)].reshape(-1, 2)
        return {"inputs": pairs[:ni.value].tolist(), "outputs": pairs[ni.value:].tolist()}

    def bench_mlp(self, groups: int, requests_per_group: int, iters: int = 10) -> tuple:
        up, down = ctypes.c_float(), ctypes.c_float()
        _check(self.lib, self.lib.coe_runtime_bench_mlp(self.handle, groups, requests_per_group, iters,
                                                        ctypes.byref(up), ctypes.byref(down)), "bench_mlp")
        return up.value, down.value

    def timing(self) -> dict:
        t = StepTiming()
        _check(self.lib, self.lib.coe_runtime_timing(self.handle, ctypes.byref(t)), "timing")
        return t.as_dict()


class LocalHub:
    """In-process hop transport for several runtimes on one device (coe_local_hub)."""

    def __init__(self, world: int):
        self.lib = _lib()
        self.handle = self.lib.coe_local_hub_create(world)

    def reset(self) -> None:
        self.lib.coe_local_hub_reset(self.handle)

    def __del__(self):
        try:
            self.lib.coe_local_hub_destroy(self.handle)
        except Exception:
            pass


def attach_peers_local(runtimes: list) -> "LocalHub":
    """Fused hops between runtimes of ONE process (several executors on one GPU): each stores
    straight into the others' buffers; readiness is handed over through a LocalHub (pass it
    to step_executors, which resets it between steps).  Also enables the (f3) peer-GPU
    swap-in tier between them (coe_runtime_attach_local_experts)."""
    hub = LocalHub(len(runtimes))
    peers = [rt.peer_buffers() for rt in runtimes]
    handles = (ctypes.c_void_p * len(runtimes))(*[rt.handle.value for rt in runtimes])
    for x, rt in enumerate(runtimes):
        rt._attach_peers(x, peers, hub)
        _check(rt.lib, rt.lib.coe_runtime_attach_local_experts(rt.handle, handles, len(runtimes)), "attach experts")
    return hub


def step_executors(plan, runtimes: list, hub: "LocalHub | None" = None) -> list:
    """Step every executor's runtime concurrently (one host thread each), then synchronise."""
    import threading

    results = [None] * len(runtimes)
    errors = []

    def work(x):
        try:
            results[x] = runtimes[x].step(plan, x)
        except Exception as exc:  # surfaced after join
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(x,)) for x in range(len(runtimes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for rt in runtimes:
        rt.synchronize()
    if hub is not None:
        hub.reset()
    if errors:
        raise errors[0]
    return results


def nccl_library() -> str:
    """Path of the NCCL torch loads (pip nvidia-nccl), dlopen'ed by libcoe_cuda."""
    try:
        import nvidia.nccl

        path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(path):
            return path
    except Exception:
        pass
    return "libnccl.so.2"


def _has_peer_loads(plan) -> bool:
    ops = plan.ops()
    return bool(len(ops)) and bool(((ops["kind"] == _native.OP_LOAD) & (ops["tier"] == _native.TIER_PEER)).any())


def _peak_residency(plan, executor: int, expert_shape: np.ndarray, num_shapes: int, lazy: bool = True) -> np.ndarray:
    """Per shape, the most experts this executor's op log holds in HBM at once (initial
    placement, then each LOAD's victims out and its expert in).  lazy: an initially resident
    expert only counts once materialised (the runtime restores it at its first batch); else
    from the start, if this executor ever touches it -- a bound on what is physically
    resident whatever earlier steps left behind (the runtime frees untouched residents at
    step start)."""
    cur = np.zeros(num_shapes, np.int64)
    pending = {int(e) for e in plan.initial_residency()[executor]}
    live = set()
    if not lazy:  # initial residents count from the start -- those this executor ever touches
        ops = plan.ops()
        touched = {int(op["expert"]) for op in ops if op["executor"] == executor}
        # (f3) and those other executors copy from it (kept all step, materialised at step start)
        args = plan.op_args()
        victims = {int(v) for op in ops if op["executor"] == executor and op["kind"] == _native.OP_LOAD
                   for v in args[int(op["offset"]):int(op["offset"]) + int(op["count"])]}
        touched |= {int(op["expert"]) for op in ops
                    if op["executor"] != executor and op["kind"] == _native.OP_LOAD
                    and op["tier"] == _native.TIER_PEER and int(op["seq"]) == executor} - victims
        for e in pending & touched:
            live.add(e)
            cur[expert_shape[e]] += 1
        pending = set()
    peak = cur.copy()
    args = plan.op_args()
    for op in plan.ops():
        if op["executor"] != executor:
            continue
        e = int(op["expert"])
        if op["kind"] == _native.OP_LOAD:
            o = int(op["offset"])
            for v in args[o:o + int(op["count"])]:
                v = int(v)
                pending.discard(v)
                if v in live:
                    live.discard(v)
                    cur[expert_shape[v]] -= 1
            pending.discard(e)
        elif e not in pending:
            continue
        else:
            pending.discard(e)
        if e not in live:
            live.add(e)
            k = expert_shape[e]
            cur[k] += 1
            peak[k] = max(peak[k], cur[k])
    return peak


def _step_input(plan, executor: int) -> StepInput:
    lib, h = plan.lib, plan.handle
    return StepInput(executor,
                     lib.coe_plan_num_admissions(h), ctypes.cast(lib.coe_plan_admissions(h), ctypes.c_void_p),
                     lib.coe_plan_num_ops(h), ctypes.cast(lib.coe_plan_ops(h), ctypes.c_void_p),
                     lib.coe_plan_num_op_args(h), ctypes.cast(lib.coe_plan_op_args(h), ctypes.c_void_p),
                     0, None, None, None, 0, None, None)


def plan_rows(plan, executor: int = 0, e2e: bool = True, nccl: bool = False) -> tuple:
    """(ring slots, landing rows) one step of ``plan`` needs on ``executor``: the activation
    ring's peak occupancy and the hop-in landing rows (act_rows.h; the runtime's own pass,
    host only).  ``e2e``: stage-0 inputs stream into ring slots too."""
    lib = _lib()
    ring, landing = ctypes.c_int32(), ctypes.c_int32()
    inp = _step_input(plan, executor)
    _check(lib, lib.coe_runtime_plan_rows(ctypes.byref(inp), len(plan.resolved.request_ids), 1 if e2e else 0,
                                          1 if nccl else 0, ctypes.byref(ring), ctypes.byref(landing)), "plan rows")
    return ring.value, landing.value


def hops_from_plan(plan) -> list:
    """Cross-executor hops (index, src, dst, request, stage) in global order (coe_plan_hops)."""
    lib, h = plan.lib, plan.handle
    lib.coe_plan_hops.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 5
    lib.coe_plan_hops.restype = ctypes.c_int64
    n = lib.coe_plan_hops(h, 0, None, None, None, None, None)
    idx = np.zeros(max(1, n), np.int64)
    cols = [np.zeros(max(1, n), np.int32) for _ in range(4)]
    lib.coe_plan_hops(h, n, idx.ctypes.data, *(c.ctypes.data for c in cols))
    return [(int(idx[i]), int(cols[0][i]), int(cols[1][i]), int(cols[2][i]), int(cols[3][i])) for i in range(n)]


def io_rows(plan, executor: int = 0) -> tuple:
    """e2e host buffer rows for one executor: (stage-0 requests it uploads, final outputs it
    returns).  host_inputs row i is the i-th smallest such request; outputs come back in
    completion order (``B200Runtime.output_order``)."""
    chains = plan.resolved.chains
    n_in = n_out = 0
    for _e, members in batches_from_plan(plan, executor):
        for r, s in members:
            n_in += s == 0
            n_out += s == len(chains[r]) - 1
    return n_in, n_out


def batches_from_plan(plan, executor: int = 0) -> list:
    """(expert, [(request, stage), ...]) per planned batch of ``executor``, in op order."""
    ops = plan.ops()
    args = plan.op_args()
    out = []
    for op in ops:
        if op["executor"] != executor or op["kind"] != _native.OP_BATCH:
            continue
        o, n = int(op["offset"]), int(op["count"])
        pairs = args[o:o + 2 * n].reshape(n, 2)
        out.append((int(op["expert"]), [(int(r), int(s)) for r, s in pairs]))
    return out


def last_stages(plan) -> np.ndarray:
    return np.array([len(c) - 1 for c in plan.resolved.chains], dtype=np.int32)


def env_flag(name: str, default: str = "0") -> bool:
    return os.environ.get(name, default) not in ("0", "", "false", "False")
