"""oracle — plain CPU forward pass (float64).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  The product path
(``paper_2306_03622_b200``) never imports, links or executes anything here.

See ``oracle.c`` for what is computed and the paper passages it follows.
Parity status of each function is listed in DESIGN.md §"Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


class _Tensor(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_uint64), ("bytes", ctypes.c_uint64), ("dtype", ctypes.c_uint32),
                ("rank", ctypes.c_uint32), ("shape", ctypes.c_uint32 * 4)]


class _Slot(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_uint32), ("rank", ctypes.c_uint32), ("shape", ctypes.c_uint32 * 4)]


class _Layer(ctypes.Structure):
    _fields_ = [("op", ctypes.c_uint32), ("first_ref", ctypes.c_uint32), ("n_refs", ctypes.c_uint32),
                ("in0", ctypes.c_int32), ("in1", ctypes.c_int32), ("out", ctypes.c_int32),
                ("attr", ctypes.c_int32 * 8)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_run.restype = ctypes.c_int
        _lib.oracle_load_input.restype = ctypes.c_int
        _lib.or_gelu_erf.restype = ctypes.c_double
        _lib.or_gelu_erf.argtypes = [ctypes.c_double]
        _lib.or_gelu_tanh.restype = ctypes.c_double
        _lib.or_gelu_tanh.argtypes = [ctypes.c_double]
    return _lib


def gelu_erf(x: float) -> float:
    return lib().or_gelu_erf(x)


def gelu_tanh(x: float) -> float:
    return lib().or_gelu_tanh(x)


def _marshal(spec):
    spec.assign_offsets()
    T = (_Tensor * len(spec.tensors))()
    for i, t in enumerate(spec.tensors):
        T[i].offset, T[i].bytes, T[i].dtype, T[i].rank = t.offset, t.nbytes, t.dtype, len(t.shape)
        for j, d in enumerate(t.shape):
            T[i].shape[j] = d
    S = (_Slot * len(spec.slots))()
    for i, s in enumerate(spec.slots):
        S[i].dtype, S[i].rank = s.dtype, len(s.shape)
        for j, d in enumerate(s.shape):
            S[i].shape[j] = d
    refs = []
    L = (_Layer * len(spec.layers))()
    for i, l in enumerate(spec.layers):
        L[i].op, L[i].first_ref, L[i].n_refs = l.op, len(refs), len(l.refs)
        refs += l.refs
        L[i].in0, L[i].in1, L[i].out = l.in0, l.in1, l.out
        for j in range(8):
            L[i].attr[j] = l.attr[j]
    R = (ctypes.c_uint32 * max(1, len(refs)))(*refs)
    return T, S, L, R


def forward(spec, weights: np.ndarray, inp: np.ndarray, first: int = 0, last: Optional[int] = None,
            slots: Optional[Dict[int, np.ndarray]] = None) -> Dict[int, np.ndarray]:
    """Run layers [first, last) and return {slot id: float64 array shaped like the slot}.

    ``inp`` is the request input bytes for the input slot; ``slots`` optionally pre-seeds
    slot contents (float64) — used by per-op tests that start mid-table.
    """
    T, S, L, R = _marshal(spec)
    last = len(spec.layers) if last is None else last
    bufs = [np.zeros(int(np.prod(s.shape)), dtype=np.float64) for s in spec.slots]
    if slots:
        for k, v in slots.items():
            bufs[k][:] = np.asarray(v, dtype=np.float64).reshape(-1)
    inp = np.ascontiguousarray(inp).view(np.uint8)
    lib().oracle_load_input(ctypes.byref(S[spec.input_slot]), inp.ctypes.data_as(ctypes.c_void_p),
                            bufs[spec.input_slot].ctypes.data_as(ctypes.c_void_p))
    ptrs = (ctypes.c_void_p * len(bufs))(*[b.ctypes.data for b in bufs])
    w = np.ascontiguousarray(weights).view(np.uint8)
    rc = lib().oracle_run(w.ctypes.data_as(ctypes.c_void_p), T, R, S, L, first, last, ptrs)
    if rc != 0:
        raise ValueError(f"oracle: layer {-rc - 1} ({spec.layers[-rc - 1].name}) rejected")
    return {i: b.reshape(spec.slots[i].shape) for i, b in enumerate(bufs)}


def output(spec, weights, inp) -> np.ndarray:
    """Forward pass; returns the model output slot as float64."""
    return forward(spec, weights, inp)[spec.output_slot]
