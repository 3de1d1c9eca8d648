"""Thin ctypes binding of libfsw (include/fsw.h).  Argument marshalling only: every step of
the swap-in-and-execute path runs in libfsw's C++ runtime and sm_100a kernels.

There is no CPU fallback: if libfsw.so is missing or no CUDA device is present, the calls
raise ``FswError``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSW_LIB selects another build of the library in this directory (libfsw_trace.so: the device-timeline
# stamps compiled in, tools/timeline.py); default libfsw.so
LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ.get("FSW_LIB", "libfsw.so")))

OK, EINVAL, ENOTFOUND, ENOMEM, EBUSY, ESTATE, ECUDA, ETIMEOUT, ETOPO = range(9)
STATUS_NAMES = ["OK", "EINVAL", "ENOTFOUND", "ENOMEM", "EBUSY", "ESTATE", "ECUDA", "ETIMEOUT", "ETOPO"]
NO_OVERLAP, DMA_BASELINE, HOST_WC, HOST_ONLY, NO_PEER_SWAP, DEBUG_POISON, TRACE = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20, 0x40
FAULT_NONE, FAULT_DROP_PIECE, FAULT_DROP_GROUP = 0, 1, 2
ORDER_EXEC, ORDER_REVERSE, ORDER_RANDOM = 0, 1, 2
SWAP_RESIDENT, SWAP_HOST, SWAP_PEER, SWAP_STRIPED = 0, 1, 2, 3
ENGINE_AUTO, ENGINE_SM, ENGINE_DMA, ENGINE_SMZ, ENGINE_DMAZ, ENGINE_DMAZT = 0, 1, 2, 3, 4, 5
REG_LINK_CODE = 0x2
EVICT_KEEP_PREFIX = 0x1

u32, u64, i32, dbl, vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p


class FswError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("n_gpus", u32), ("gpu_ids", ctypes.POINTER(i32)), ("pool_bytes_per_gpu", u64),
                ("workspace_bytes_per_gpu", u64), ("copy_ctas", u32), ("copy_threads", u32),
                ("chunk_bytes", u64), ("stripe_min_bytes", u64), ("flags", u32), ("engine", u32),
                ("dma_min_bytes", u64), ("dma_group_bytes", u64), ("dma_streams", u32),
                ("pcie_neighbor", ctypes.POINTER(i32)), ("dmaz_min_bytes", u64)]


class Tensor(ctypes.Structure):
    _fields_ = [("offset", u64), ("bytes", u64), ("dtype", u32), ("rank", u32), ("shape", u32 * 4)]


class Slot(ctypes.Structure):
    _fields_ = [("dtype", u32), ("rank", u32), ("shape", u32 * 4)]


class Layer(ctypes.Structure):
    _fields_ = [("op", u32), ("first_ref", u32), ("n_refs", u32), ("in0", i32), ("in1", i32), ("out", i32),
                ("attr", i32 * 8)]


class ModelDesc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("weights", vp), ("weight_bytes", u64),
                ("tensors", ctypes.POINTER(Tensor)), ("n_tensors", u32),
                ("refs", ctypes.POINTER(u32)), ("n_refs", u32),
                ("slots", ctypes.POINTER(Slot)), ("n_slots", u32),
                ("layers", ctypes.POINTER(Layer)), ("n_layers", u32),
                ("input_slot", i32), ("output_slot", i32), ("flags", u32)]


class ModelInfo(ctypes.Structure):
    _fields_ = [("store_bytes", u64), ("algorithmic_bytes", u64), ("n_layers", u32), ("n_tensors", u32),
                ("n_gemm_layers", u32), ("input_bytes", u64), ("output_bytes", u64), ("output_dtype", u32),
                ("coded_bytes", u64), ("numa_node", i32)]


class StoreTensor(ctypes.Structure):
    _fields_ = [("offset", u64), ("bytes", u64), ("layout", u32), ("rows", u32), ("cols", u32),
                ("rows_pad", u32), ("cols_pad", u32), ("owner_layer", u32)]


class InvokeStats(ctypes.Structure):
    _fields_ = [("total_ms", dbl), ("device_ms", dbl), ("swap_ms", dbl), ("swap_span_ms", dbl),
                ("compute_tail_ms", dbl), ("bytes_swapped", u64), ("link_gbps", dbl), ("gpu", i32),
                ("swap_kind", u32), ("n_sources", u32), ("n_kernels", u32), ("engine", u32), ("n_copies", u32),
                ("wire_bytes", u64), ("host_setup_ms", dbl), ("host_wait_ms", dbl)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class CodedPiece(ctypes.Structure):
    _fields_ = [("off", u64), ("coff", u64), ("bytes", u32), ("cbytes", u32), ("layer", u32), ("pad", u32),
                ("hdr", ctypes.c_uint32 * 16)]


class InvokeOpts(ctypes.Structure):
    _fields_ = [("gpu", i32), ("n_stripe_src", u32), ("chunk_bytes", u64), ("order", u32), ("order_seed", u32),
                ("copy_ctas", u32), ("flags", u32), ("engine", u32), ("dma_group_bytes", u64), ("dma_streams", u32),
                ("stripe_src", ctypes.POINTER(i32)), ("peer_src", u32)]


class PoolStats(ctypes.Structure):
    _fields_ = [("capacity", u64), ("used", u64), ("largest_free", u64), ("n_resident", u32), ("n_extents", u32),
                ("n_evictions", u64), ("bytes_swapped_total", u64), ("n_invokes_cold", u64),
                ("n_invokes_warm", u64), ("prefix_bytes_cached", u64), ("n_evictions_heavy", u64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Decision(ctypes.Structure):
    _fields_ = [("gpu", i32), ("kind", u32), ("src", i32)]


class SchedConfig(ctypes.Structure):
    _fields_ = [("alpha0", dbl), ("scalar", dbl), ("threshold", dbl), ("period_ms", dbl), ("max_inflight", u32)]


class RequestStats(ctypes.Structure):
    _fields_ = [("queue_ms", dbl), ("total_ms", dbl), ("device_ms", dbl), ("met_deadline", i32), ("gpu", i32),
                ("swap_kind", u32), ("status", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class FunctionStats(ctypes.Structure):
    _fields_ = [("n", u64), ("m", u64), ("rrc", dbl), ("rrc_normalized", dbl), ("avg_latency_ms", dbl), ("high", u32),
                ("queued", u32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SchedStats(ctypes.Structure):
    _fields_ = [("alpha", dbl), ("n_functions", u32), ("n_high", u32), ("active_functions", u32),
                ("slo_compliant_functions", u32), ("completed", u64), ("met_deadline", u64), ("n_resident", u64),
                ("n_host_swaps", u64), ("n_peer_swaps", u64), ("n_striped_swaps", u64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["fsw_init", "fsw_shutdown", "fsw_last_error", "fsw_version", "fsw_register_model",
           "fsw_unregister_model", "fsw_model_info_get", "fsw_store_tensor_get", "fsw_invoke", "fsw_invoke_ex",
           "fsw_evict", "fsw_pool_stats_get", "fsw_n_gpus", "fsw_debug_read_resident", "fsw_debug_read_store",
           "fsw_debug_read_slot", "fsw_arena_create", "fsw_arena_destroy", "fsw_arena_alloc", "fsw_arena_free",
           "fsw_arena_stats", "fsw_debug_dma_plan", "fsw_policy_rrc", "fsw_policy_partition", "fsw_policy_alpha",
           "fsw_policy_schedule", "fsw_policy_eviction_order", "fsw_model_set_heavy", "fsw_model_is_heavy",
           "fsw_sched_create", "fsw_sched_destroy", "fsw_function_register", "fsw_submit", "fsw_wait",
           "fsw_function_stats_get", "fsw_sched_stats_get", "fsw_evict_ex", "fsw_model_set_cache_prefix",
           "fsw_debug_read_coded", "fsw_debug_coded_pieces", "fsw_debug_coded_code", "fsw_debug_dmaz_plan", "fsw_policy_stripe_deal",
           "fsw_debug_set_fault", "fsw_debug_litmus", "fsw_policy_heavy", "fsw_model_set_slo",
           "fsw_set_heavy_policy", "fsw_debug_trace_read", "fsw_debug_mega_stamps"]

_lib = None


def lib():
    """Load libfsw.so (fails loudly when it is missing — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FswError(ECUDA, f"{LIB_PATH} not built; run `python -m paper_2306_03622_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.fsw_last_error.restype = ctypes.c_char_p
        L.fsw_version.restype = ctypes.c_char_p
        L.fsw_init.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(vp)]
        L.fsw_shutdown.argtypes = [vp]
        L.fsw_shutdown.restype = None
        L.fsw_register_model.argtypes = [vp, ctypes.POINTER(ModelDesc), ctypes.POINTER(u32)]
        L.fsw_unregister_model.argtypes = [vp, u32]
        L.fsw_model_info_get.argtypes = [vp, u32, ctypes.POINTER(ModelInfo)]
        L.fsw_store_tensor_get.argtypes = [vp, u32, u32, ctypes.POINTER(StoreTensor)]
        L.fsw_invoke.argtypes = [vp, u32, vp, u64, vp, u64, ctypes.POINTER(InvokeStats)]
        L.fsw_invoke_ex.argtypes = [vp, u32, ctypes.POINTER(InvokeOpts), vp, u64, vp, u64, ctypes.POINTER(InvokeStats)]
        L.fsw_evict.argtypes = [vp, u32, i32]
        L.fsw_evict_ex.argtypes = [vp, u32, i32, u32]
        L.fsw_model_set_cache_prefix.argtypes = [vp, u32, u64, ctypes.POINTER(u64)]
        L.fsw_pool_stats_get.argtypes = [vp, i32, ctypes.POINTER(PoolStats)]
        L.fsw_n_gpus.argtypes = [vp, ctypes.POINTER(u32)]
        L.fsw_debug_read_resident.argtypes = [vp, u32, i32, vp, u64]
        L.fsw_debug_read_store.argtypes = [vp, u32, vp, u64]
        L.fsw_debug_read_slot.argtypes = [vp, u32, i32, i32, vp, u64]
        L.fsw_debug_read_coded.argtypes = [vp, u32, vp, u64]
        L.fsw_debug_coded_pieces.argtypes = [vp, u32, vp, u32, ctypes.POINTER(u32)]
        L.fsw_debug_coded_code.argtypes = [vp, u32, vp]
        L.fsw_debug_dmaz_plan.argtypes = [vp, u32, u64, u32, vp, vp, u32, ctypes.POINTER(u32), vp]
        L.fsw_debug_set_fault.argtypes = [vp, u32, u32]
        L.fsw_debug_trace_read.argtypes = [vp, u32, i32, vp, u32, vp]
        L.fsw_debug_mega_stamps.argtypes = [vp, u32, i32, vp, vp, u64, ctypes.POINTER(u32), ctypes.POINTER(u32)]
        L.fsw_policy_heavy.argtypes = [dbl, dbl, dbl, dbl, dbl, ctypes.POINTER(i32)]
        L.fsw_model_set_slo.argtypes = [vp, u32, dbl]
        L.fsw_set_heavy_policy.argtypes = [vp, dbl, dbl]
        L.fsw_debug_litmus.argtypes = [vp, u32, i32, u32, u32, u32, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.fsw_arena_create.argtypes = [u64, u64]
        L.fsw_arena_create.restype = vp
        L.fsw_arena_destroy.argtypes = [vp]
        L.fsw_arena_destroy.restype = None
        L.fsw_arena_alloc.argtypes = [vp, u64, ctypes.POINTER(u64)]
        L.fsw_arena_free.argtypes = [vp, u64]
        L.fsw_arena_stats.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u32)]
        L.fsw_arena_stats.restype = None
        L.fsw_debug_dma_plan.argtypes = [vp, u32, u64, u32, vp, vp, u32, ctypes.POINTER(u32), vp]
        L.fsw_policy_rrc.argtypes = [u64, u64, dbl, ctypes.POINTER(dbl)]
        L.fsw_policy_partition.argtypes = [vp, u32, dbl, vp]
        L.fsw_policy_alpha.argtypes = [dbl, dbl, dbl, dbl, dbl, ctypes.POINTER(dbl)]
        L.fsw_policy_schedule.argtypes = [u32, vp, vp, vp, vp, vp, ctypes.POINTER(Decision)]
        L.fsw_policy_eviction_order.argtypes = [u32, vp, vp, vp, vp, vp, ctypes.POINTER(u32)]
        L.fsw_policy_stripe_deal.argtypes = [u32, vp, u32, vp, vp]
        L.fsw_model_set_heavy.argtypes = [vp, u32, i32]
        L.fsw_model_is_heavy.argtypes = [vp, u32, ctypes.POINTER(i32)]
        L.fsw_sched_create.argtypes = [vp, ctypes.POINTER(SchedConfig), ctypes.POINTER(vp)]
        L.fsw_sched_destroy.argtypes = [vp]
        L.fsw_sched_destroy.restype = None
        L.fsw_function_register.argtypes = [vp, u32, dbl, dbl, ctypes.POINTER(u32)]
        L.fsw_submit.argtypes = [vp, u32, vp, u64, vp, u64, ctypes.POINTER(u64)]
        L.fsw_wait.argtypes = [vp, u64, ctypes.POINTER(RequestStats)]
        L.fsw_function_stats_get.argtypes = [vp, u32, ctypes.POINTER(FunctionStats)]
        L.fsw_sched_stats_get.argtypes = [vp, ctypes.POINTER(SchedStats)]
        for name in EXPORTS:
            f = getattr(L, name)
            if f.restype is ctypes.c_int:  # default
                f.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OK:
        raise FswError(rc, lib().fsw_last_error().decode(errors="replace"))


class Arena:
    """Host-only extent allocator of the weight pool (usable without a GPU)."""

    def __init__(self, capacity: int, align: int = 64 << 10):
        self.h = lib().fsw_arena_create(capacity, align)
        if not self.h:
            raise FswError(EINVAL, "bad arena parameters")

    def alloc(self, nbytes: int) -> int:
        off = u64()
        _check(lib().fsw_arena_alloc(self.h, nbytes, ctypes.byref(off)))
        return off.value

    def free(self, off: int):
        _check(lib().fsw_arena_free(self.h, off))

    def stats(self):
        u, lf, n = u64(), u64(), u32()
        lib().fsw_arena_stats(self.h, ctypes.byref(u), ctypes.byref(lf), ctypes.byref(n))
        return {"used": u.value, "largest_free": lf.value, "n_allocated": n.value}

    def __del__(self):
        if getattr(self, "h", None):
            lib().fsw_arena_destroy(self.h)
            self.h = None


@dataclass
class Result:
    output: np.ndarray
    stats: dict


class Runtime:
    """One libfsw context (one per process): pool, host stores, per-GPU executors."""

    def __init__(self, n_gpus: int = 0, gpu_ids: Optional[Sequence[int]] = None, pool_bytes: int = 0,
                 workspace_bytes: int = 0, copy_ctas: int = 0, copy_threads: int = 0, chunk_bytes: int = 0,
                 flags: int = 0, engine: int = ENGINE_AUTO, dma_min_bytes: int = 0, dma_group_bytes: int = 0,
                 dma_streams: int = 0, stripe_min_bytes: int = 0, dmaz_min_bytes: int = 0):
        cfg = Config()
        cfg.n_gpus = n_gpus or (len(gpu_ids) if gpu_ids else 0)
        self._ids = (i32 * len(gpu_ids))(*gpu_ids) if gpu_ids else None
        cfg.gpu_ids = self._ids
        cfg.pool_bytes_per_gpu = pool_bytes
        cfg.workspace_bytes_per_gpu = workspace_bytes
        cfg.copy_ctas, cfg.copy_threads, cfg.chunk_bytes, cfg.flags = copy_ctas, copy_threads, chunk_bytes, flags
        cfg.engine, cfg.dma_min_bytes, cfg.dma_group_bytes, cfg.dma_streams = engine, dma_min_bytes, dma_group_bytes, dma_streams
        cfg.stripe_min_bytes = stripe_min_bytes
        cfg.dmaz_min_bytes = dmaz_min_bytes
        h = vp()
        _check(lib().fsw_init(ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        self._models = {}

    def close(self):
        if getattr(self, "h", None):
            lib().fsw_shutdown(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def n_gpus(self) -> int:
        n = u32()
        _check(lib().fsw_n_gpus(self.h, ctypes.byref(n)))
        return n.value

    # ---- registration -------------------------------------------------------------------
    def register(self, name: str, weights: np.ndarray, tensors, refs, slots, layers, input_slot: int,
                 output_slot: int, flags: int = 0) -> int:
        """tensors: [(offset, bytes, dtype, shape)], slots: [(dtype, shape)],
        layers: [(op, first_ref, n_refs, in0, in1, out, attr[8])], refs: [tensor index]."""
        T = (Tensor * max(1, len(tensors)))()
        for i, (off, nb, dt, shp) in enumerate(tensors):
            T[i].offset, T[i].bytes, T[i].dtype, T[i].rank = off, nb, dt, len(shp)
            for j, d in enumerate(shp):
                T[i].shape[j] = d
        S = (Slot * len(slots))()
        for i, (dt, shp) in enumerate(slots):
            S[i].dtype, S[i].rank = dt, len(shp)
            for j, d in enumerate(shp):
                S[i].shape[j] = d
        Ls = (Layer * len(layers))()
        for i, (op, fr, nr, a, b, o, attr) in enumerate(layers):
            Ls[i].op, Ls[i].first_ref, Ls[i].n_refs, Ls[i].in0, Ls[i].in1, Ls[i].out = op, fr, nr, a, b, o
            for j in range(8):
                Ls[i].attr[j] = attr[j]
        R = (u32 * max(1, len(refs)))(*refs)
        w = np.ascontiguousarray(weights).view(np.uint8)
        d = ModelDesc(name.encode(), w.ctypes.data, w.nbytes, T, len(tensors), R, len(refs), S, len(slots), Ls,
                      len(layers), input_slot, output_slot, flags)
        mid = u32()
        _check(lib().fsw_register_model(self.h, ctypes.byref(d), ctypes.byref(mid)))
        info = self.model_info(mid.value)
        self._models[mid.value] = info
        return mid.value

    def register_spec(self, spec, weights: np.ndarray, link_code: bool = False) -> int:
        """Register a synth.ModelSpec-shaped description (duck-typed); link_code builds the
        exponent-coded store the SMZ / DMAZ engines move (FSW_REG_LINK_CODE)."""
        spec.assign_offsets()
        tensors = [(t.offset, t.nbytes, t.dtype, t.shape) for t in spec.tensors]
        slots = [(s.dtype, s.shape) for s in spec.slots]
        refs, layers = [], []
        for l in spec.layers:
            layers.append((int(l.op), len(refs), len(l.refs), l.in0, l.in1, l.out, list(l.attr)))
            refs += list(l.refs)
        return self.register(spec.name, weights, tensors, refs, slots, layers, spec.input_slot, spec.output_slot,
                             REG_LINK_CODE if link_code else 0)

    def unregister(self, mid: int):
        _check(lib().fsw_unregister_model(self.h, mid))
        self._models.pop(mid, None)

    def model_info(self, mid: int) -> dict:
        i = ModelInfo()
        _check(lib().fsw_model_info_get(self.h, mid, ctypes.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def store_tensor(self, mid: int, t: int) -> dict:
        s = StoreTensor()
        _check(lib().fsw_store_tensor_get(self.h, mid, t, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    # ---- invoke -------------------------------------------------------------------------
    def invoke(self, mid: int, inp: np.ndarray, out: Optional[np.ndarray] = None, gpu: int = -1,
               chunk_bytes: int = 0, order: int = ORDER_EXEC, order_seed: int = 0, copy_ctas: int = 0,
               flags: int = 0, engine: int = 0, dma_group_bytes: int = 0, dma_streams: int = 0,
               stripe: Optional[Sequence[int]] = None, peer_src: int = -1) -> Result:
        info = self._models.get(mid) or self.model_info(mid)
        inp = np.ascontiguousarray(inp)
        if out is None:
            out = np.empty(info["output_bytes"] // 4, dtype=np.float32 if info["output_dtype"] == 1 else np.int32) \
                if info["output_dtype"] != 0 else np.empty(info["output_bytes"] // 2, dtype=np.uint16)
        st = InvokeStats()
        src = (i32 * len(stripe))(*stripe) if stripe else None
        opts = InvokeOpts(gpu, len(stripe) if stripe else 0, chunk_bytes, order, order_seed, copy_ctas, flags, engine,
                          dma_group_bytes, dma_streams, src, peer_src + 1)
        _check(lib().fsw_invoke_ex(self.h, mid, ctypes.byref(opts), inp.ctypes.data, inp.nbytes, out.ctypes.data,
                                   out.nbytes, ctypes.byref(st)))
        return Result(out, st.as_dict())

    def invoke_plain(self, mid: int, inp: np.ndarray, out: np.ndarray) -> dict:
        """fsw_invoke (scheduler's choice of GPU), the call a user makes."""
        st = InvokeStats()
        _check(lib().fsw_invoke(self.h, mid, inp.ctypes.data, inp.nbytes, out.ctypes.data, out.nbytes,
                                ctypes.byref(st)))
        return st.as_dict()

    def set_heavy(self, mid: int, heavy: int):
        _check(lib().fsw_model_set_heavy(self.h, mid, heavy))

    def is_heavy(self, mid: int) -> bool:
        h = i32()
        _check(lib().fsw_model_is_heavy(self.h, mid, ctypes.byref(h)))
        return bool(h.value)

    def set_slo(self, mid: int, deadline_ms: float):
        _check(lib().fsw_model_set_slo(self.h, mid, deadline_ms))

    def set_heavy_policy(self, theta: float = 0.05, queue_budget_ms: float = 0.0):
        _check(lib().fsw_set_heavy_policy(self.h, theta, queue_budget_ms))

    def evict(self, mid: int, gpu: int = -1, keep_prefix: bool = False):
        _check(lib().fsw_evict_ex(self.h, mid, gpu, EVICT_KEEP_PREFIX if keep_prefix else 0))

    def set_cache_prefix(self, mid: int, nbytes: int) -> int:
        """Partial-parameter caching: returns the prefix bytes actually kept (a layer boundary)."""
        a = u64()
        _check(lib().fsw_model_set_cache_prefix(self.h, mid, nbytes, ctypes.byref(a)))
        return a.value

    def pool_stats(self, gpu: int = 0) -> dict:
        p = PoolStats()
        _check(lib().fsw_pool_stats_get(self.h, gpu, ctypes.byref(p)))
        return p.as_dict()

    # ---- debug --------------------------------------------------------------------------
    def dma_plan(self, mid: int, group_bytes: int, streams: int):
        """DMA engine copy plan: (groups [n][2] = [lo, hi), stream [n], layer targets [n_layers][4])."""
        n = u32()
        lib().fsw_debug_dma_plan(self.h, mid, group_bytes, streams, None, None, 0, ctypes.byref(n), None)
        lohi = np.zeros((max(1, n.value), 2), np.uint64)
        st = np.zeros(max(1, n.value), np.uint32)
        tg = np.zeros((self.model_info(mid)["n_layers"], 4), np.uint32)
        _check(lib().fsw_debug_dma_plan(self.h, mid, group_bytes, streams, lohi.ctypes.data, st.ctypes.data,
                                        n.value, ctypes.byref(n), tg.ctypes.data))
        return lohi[:n.value], st[:n.value], tg

    def read_resident(self, mid: int, gpu: int = 0) -> np.ndarray:
        n = self.model_info(mid)["store_bytes"]
        buf = np.empty(n, dtype=np.uint8)
        _check(lib().fsw_debug_read_resident(self.h, mid, gpu, buf.ctypes.data, n))
        return buf

    def read_store(self, mid: int) -> np.ndarray:
        n = self.model_info(mid)["store_bytes"]
        buf = np.empty(n, dtype=np.uint8)
        _check(lib().fsw_debug_read_store(self.h, mid, buf.ctypes.data, n))
        return buf

    def read_coded(self, mid: int) -> np.ndarray:
        n = self.model_info(mid)["coded_bytes"]
        buf = np.empty(n, dtype=np.uint8)
        _check(lib().fsw_debug_read_coded(self.h, mid, buf.ctypes.data, n))
        return buf

    def coded_code(self, mid: int) -> np.ndarray:
        """The model's 16 canonical code lengths of entropy-coded pieces (all 0: none; include/fsw.h)."""
        out = np.zeros(16, np.uint8)
        _check(lib().fsw_debug_coded_code(self.h, mid, out.ctypes.data))
        return out

    def coded_pieces(self, mid: int) -> np.ndarray:
        """Piece table of the link-coded store: structured array (off, coff, bytes, cbytes, layer, hdr[16])."""
        n = u32()
        lib().fsw_debug_coded_pieces(self.h, mid, None, 0, ctypes.byref(n))
        arr = (CodedPiece * max(1, n.value))()
        _check(lib().fsw_debug_coded_pieces(self.h, mid, arr, n.value, ctypes.byref(n)))
        dt = np.dtype([("off", "<u8"), ("coff", "<u8"), ("bytes", "<u4"), ("cbytes", "<u4"), ("layer", "<u4"),
                       ("pad", "<u4"), ("hdr", "<u4", (16,))])
        return np.frombuffer(bytes(arr), dtype=dt)[:n.value].copy()

    def dmaz_plan(self, mid: int, group_bytes: int, streams: int = 1):
        """DMAZ copy plan: (groups [n][2] coded [lo, hi), stream [n], piece_group [n_pieces])."""
        n = u32()
        lib().fsw_debug_dmaz_plan(self.h, mid, group_bytes, streams, None, None, 0, ctypes.byref(n), None)
        lohi = np.zeros((max(1, n.value), 2), np.uint64)
        st = np.zeros(max(1, n.value), np.uint32)
        pg = np.zeros(max(1, len(self.coded_pieces(mid))), np.uint32)
        _check(lib().fsw_debug_dmaz_plan(self.h, mid, group_bytes, streams, lohi.ctypes.data, st.ctypes.data,
                                         n.value, ctypes.byref(n), pg.ctypes.data))
        return lohi[:n.value], st[:n.value], pg

    def set_fault(self, kind: int, index: int = 0):
        """Fault injection (negative controls): FAULT_DROP_PIECE / FAULT_DROP_GROUP / FAULT_NONE."""
        _check(lib().fsw_debug_set_fault(self.h, kind, index))

    def litmus(self, mid: int, engine: int, ctas: int, iters: int, gpu: int = 0):
        """Readiness litmus (fsw_debug_litmus): (bad 16-byte words, bytes checked) over `iters` runs."""
        bad, chk = u64(), u64()
        _check(lib().fsw_debug_litmus(self.h, mid, gpu, engine, ctas, iters, ctypes.byref(bad), ctypes.byref(chk)))
        return bad.value, chk.value

    def trace(self, mid: int, gpu: int = 0):
        """Device timeline of the last invoke (FSW_TRACE): ([n_layers][16] ns: entry, wait done, exit, first /
        last piece released, GEMM predecessor wait / MMA done / epilogue start / epilogue phases; 0 = none), [first piece claimed,
        last released, graph end] ns)."""
        n = self.model_info(mid)["n_layers"]
        out = np.zeros((n, 16), np.uint64)
        ti = np.zeros(3, np.uint64)
        _check(lib().fsw_debug_trace_read(self.h, mid, gpu, out.ctypes.data, n, ti.ctypes.data))
        return out, ti

    def mega_stamps(self, mid: int, gpu: int = 0):
        """Persistent-kernel phase stamps (FSW_MEGA_STAMPS=1): ([n_ops][ctas][8] ns, [n_ops][4] op info)."""
        n, c = u32(), u32()
        lib().fsw_debug_mega_stamps(self.h, mid, gpu, None, None, 0, ctypes.byref(n), ctypes.byref(c))
        out = np.zeros((n.value, c.value, 8), np.uint64)
        ops = np.zeros((n.value, 4), np.uint32)
        _check(lib().fsw_debug_mega_stamps(self.h, mid, gpu, out.ctypes.data, ops.ctypes.data, out.size,
                                           ctypes.byref(n), ctypes.byref(c)))
        return out, ops

    def read_slot(self, mid: int, slot: int, nbytes: int, gpu: int = 0) -> np.ndarray:
        buf = np.empty(nbytes, dtype=np.uint8)
        _check(lib().fsw_debug_read_slot(self.h, mid, gpu, slot, buf.ctypes.data, nbytes))
        return buf


# ---- node policies (pure host functions; include/fsw.h "Node policies") ----------------------
def policy_rrc(n: int, m: int, p: float) -> float:
    out = dbl()
    _check(lib().fsw_policy_rrc(n, m, p, ctypes.byref(out)))
    return out.value


def policy_partition(rrcs, alpha: float) -> np.ndarray:
    r = np.ascontiguousarray(rrcs, dtype=np.float64)
    high = np.zeros(len(r), np.uint8)
    _check(lib().fsw_policy_partition(r.ctypes.data, len(r), alpha, high.ctypes.data))
    return high


def policy_alpha(alpha, last_ratio, new_ratio, scalar=2.0, threshold=0.04) -> float:
    out = dbl()
    _check(lib().fsw_policy_alpha(alpha, last_ratio, new_ratio, scalar, threshold, ctypes.byref(out)))
    return out.value


def policy_schedule(available, hosts, neighbor=None, loading=None, link=None):
    """Algorithm 1: returns (gpu, kind, src) or None when no GPU is available (EBUSY)."""
    n = len(available)
    av = np.ascontiguousarray(available, np.uint8)
    ho = np.ascontiguousarray(hosts, np.uint8)
    nb = np.ascontiguousarray(neighbor, np.int32) if neighbor is not None else None
    ld = np.ascontiguousarray(loading, np.uint8) if loading is not None else None
    lk = np.ascontiguousarray(link, np.float32).reshape(-1) if link is not None else None
    d = Decision()
    rc = lib().fsw_policy_schedule(n, av.ctypes.data, ho.ctypes.data, nb.ctypes.data if nb is not None else None,
                                   ld.ctypes.data if ld is not None else None, lk.ctypes.data if lk is not None else None,
                                   ctypes.byref(d))
    if rc == EBUSY:
        return None
    _check(rc)
    return d.gpu, d.kind, d.src


def policy_heavy(swap_ms: float, resident_ms: float, deadline_ms: float = 0.0, queue_budget_ms: float = 0.0,
                 theta: float = 0.05) -> bool:
    h = i32()
    _check(lib().fsw_policy_heavy(swap_ms, resident_ms, deadline_ms, queue_budget_ms, theta, ctypes.byref(h)))
    return bool(h.value)


def policy_eviction_order(heavy, copies, last_use, in_use):
    n = len(heavy)
    h = np.ascontiguousarray(heavy, np.uint8)
    c = np.ascontiguousarray(copies, np.uint32)
    lu = np.ascontiguousarray(last_use, np.uint64)
    iu = np.ascontiguousarray(in_use, np.uint8)
    order = np.zeros(max(1, n), np.uint32)
    k = u32()
    _check(lib().fsw_policy_eviction_order(n, h.ctypes.data, c.ctypes.data, lu.ctypes.data, iu.ctypes.data,
                                           order.ctypes.data, ctypes.byref(k)))
    return list(order[:k.value])


def policy_stripe_deal(unit_node, src_node):
    """Striped swap: the source of every unit (node-local first, round-robin; fsw_policy_stripe_deal)."""
    un = np.ascontiguousarray(unit_node, np.int32)
    sn = np.ascontiguousarray(src_node, np.int32)
    out = np.zeros(max(1, len(un)), np.uint32)
    _check(lib().fsw_policy_stripe_deal(len(un), un.ctypes.data, len(sn), sn.ctypes.data, out.ctypes.data))
    return out[:len(un)]


class Scheduler:
    """Request scheduler over a Runtime (fsw_sched_*): functions, RRC queues, Algorithm 1 placement."""

    def __init__(self, rt: "Runtime", alpha0=0.0, scalar=0.0, threshold=0.0, period_ms=0.0, max_inflight=0):
        self.rt = rt
        cfg = SchedConfig(alpha0, scalar, threshold, period_ms, max_inflight)
        h = vp()
        _check(lib().fsw_sched_create(rt.h, ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        self._keep = {}

    def register_function(self, model_id: int, deadline_ms: float, p: float = 0.98) -> int:
        fid = u32()
        _check(lib().fsw_function_register(self.h, model_id, deadline_ms, p, ctypes.byref(fid)))
        return fid.value

    def submit(self, fid: int, inp: np.ndarray, out: np.ndarray) -> int:
        t = u64()
        _check(lib().fsw_submit(self.h, fid, inp.ctypes.data, inp.nbytes, out.ctypes.data, out.nbytes, ctypes.byref(t)))
        self._keep[t.value] = (inp, out)
        return t.value

    def wait(self, ticket: int) -> dict:
        st = RequestStats()
        rc = lib().fsw_wait(self.h, ticket, ctypes.byref(st))
        self._keep.pop(ticket, None)
        d = st.as_dict()
        d["rc"] = rc
        return d

    def function_stats(self, fid: int) -> dict:
        s = FunctionStats()
        _check(lib().fsw_function_stats_get(self.h, fid, ctypes.byref(s)))
        return s.as_dict()

    def stats(self) -> dict:
        s = SchedStats()
        _check(lib().fsw_sched_stats_get(self.h, ctypes.byref(s)))
        return s.as_dict()

    def close(self):
        if getattr(self, "h", None):
            lib().fsw_sched_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
