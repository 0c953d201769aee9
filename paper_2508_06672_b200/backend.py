"""The drop-in correlation backend — host mirror of digeo backend.hpp:47-325.

``B200Backend`` is a ``CorrelationBackend`` (backend.hpp:211-217): ``stage``
copies one snapshot's capture pair into HBM (the "load" step) and returns a
``CorrelationSession`` whose ``correlate_batch`` evaluates Eq. 11 for a batch
of ``PairOffsets`` on the GPU and hands back host-resident values (the
"offload" step). Descriptor: {"b200", "parallel-batched", 1}.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, lib
from .engine import Engine, default_engine

DEFAULT_MEMORY_BUDGET_BYTES = 512 << 20  # backend.hpp:67

# == digeo::PairOffsets {int64 tdoa_samples; double fdoa_hz} (geometry.hpp:68-71)
PAIR_OFFSETS_DTYPE = np.dtype([("tdoa_samples", "<i8"), ("fdoa_hz", "<f8")])


@dataclass
class BasebandCapture:
    """capture.hpp:32-48. ``samples``: complex128 (reference) or complex64 (DGIQ)."""
    samples: np.ndarray
    sample_rate_hz: float = 0.0
    start_time_s: float = 0.0
    center_freq_hz: float = 0.0

    def size(self) -> int:
        return len(self.samples)

    def validate(self) -> None:
        if len(self.samples) == 0:
            raise ValueError("BasebandCapture: no samples")
        if not (self.sample_rate_hz > 0.0):
            raise ValueError("BasebandCapture: sample_rate_hz <= 0")


@dataclass
class PairOffsets:
    tdoa_samples: int = 0
    fdoa_hz: float = 0.0


@dataclass
class BackendDescriptor:
    """backend.hpp:47-51"""
    name: str
    kind: str
    workers: int = 1


@dataclass
class BatchPlan:
    """backend.hpp:55-65"""
    n_points: int
    batch_size: int
    memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET_BYTES

    def batch_count(self) -> int:
        return (self.n_points + self.batch_size - 1) // self.batch_size

    def batch_range(self, b: int):
        begin = b * self.batch_size
        return begin, min(begin + self.batch_size, self.n_points)


def estimate_working_set_bytes(batch_size: int, capture_bytes_total: int) -> int:
    """backend.hpp:71-75"""
    return batch_size * (16 + 8) + capture_bytes_total


def plan_batches(n_points: int, batch_size: int,
                 memory_budget_bytes: int = DEFAULT_MEMORY_BUDGET_BYTES,
                 capture_bytes_total: int = 0) -> BatchPlan:
    """backend.hpp:77-93 (validation and messages via dg_plan_batches)."""
    if n_points < 1:
        raise ValueError("plan_batches: n_points < 1")
    if batch_size < 1:
        raise ValueError("plan_batches: batch_size < 1")
    out = C.c_uint64()
    check(lib.dg_plan_batches(int(n_points), int(batch_size), int(memory_budget_bytes),
                              int(capture_bytes_total), C.byref(out)))
    return BatchPlan(int(n_points), int(batch_size), int(memory_budget_bytes))


def as_offsets(batch) -> np.ndarray:
    """Accept a PairOffsets-dtype array, a list of PairOffsets, or (tdoa, fdoa) pairs."""
    if isinstance(batch, np.ndarray) and batch.dtype == PAIR_OFFSETS_DTYPE:
        return np.ascontiguousarray(batch)
    out = np.zeros(len(batch), PAIR_OFFSETS_DTYPE)
    for i, o in enumerate(batch):
        if isinstance(o, PairOffsets):
            out[i] = (o.tdoa_samples, o.fdoa_hz)
        else:
            out[i] = (int(o[0]), float(o[1]))
    return out


class CorrelationSession:
    """backend.hpp:196-209, one staged capture pair on the device."""

    def __init__(self, handle, backend: "B200Backend"):
        self._h = handle
        self.backend = backend

    @property
    def handle(self):
        return self._h

    def correlate_batch(self, batch, out: np.ndarray | None = None) -> np.ndarray:
        off = as_offsets(batch)
        n = len(off)
        if out is None:
            out = np.zeros(n, np.float64)
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("correlate_batch: out must be a contiguous float64 array")
        check(lib.dg_correlate_batch(
            self._h, off.ctypes.data_as(C.POINTER(_capi.dg_pair_offsets)) if n else None, n,
            out.ctypes.data_as(C.POINTER(C.c_double)), len(out)))
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.dg_session_destroy(h)
            self._h = None


class B200Backend:
    """backend.hpp:211-217 — the engine registered as "b200" (never "gpu")."""

    def __init__(self, workers: int = 0, engine: Engine | None = None):
        """workers = GPUs (the reference's worker count, backend.hpp:292-309):
        0 every visible GPU, else min(workers, visible); one engine drives them."""
        if engine is None:
            from .engine import device_count
            n = device_count()
            m = min(workers, n) if workers else n
            engine = default_engine() if m <= 1 else Engine(devices=list(range(m)))
        self.engine = engine
        name, kind, w = self.engine.descriptor()
        self._descriptor = BackendDescriptor(name, kind, w)

    def descriptor(self) -> BackendDescriptor:
        return self._descriptor

    def stage(self, y1: BasebandCapture, y2: BasebandCapture) -> CorrelationSession:
        h = C.c_void_p()
        a, b = np.asarray(y1.samples), np.asarray(y2.samples)
        if a.dtype == np.complex64 and b.dtype == np.complex64:
            a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
            fp = C.POINTER(C.c_float)
            check(lib.dg_stage_f32(self.engine.handle, a.ctypes.data_as(fp), len(a),
                                   float(y1.sample_rate_hz), b.ctypes.data_as(fp), len(b),
                                   float(y2.sample_rate_hz), C.byref(h)))
        else:
            a = np.ascontiguousarray(a, np.complex128)
            b = np.ascontiguousarray(b, np.complex128)
            dp = C.POINTER(C.c_double)
            check(lib.dg_stage(self.engine.handle, a.ctypes.data_as(dp), len(a),
                               float(y1.sample_rate_hz), b.ctypes.data_as(dp), len(b),
                               float(y2.sample_rate_hz), C.byref(h)))
        return CorrelationSession(h, self)


def make_backend(name: str, workers: int = 0) -> B200Backend:
    """backend.hpp:311-317 for this engine's registry."""
    if name == "b200":
        return B200Backend(workers)
    raise ValueError(f"make_backend: unknown backend '{name}' (expected b200)")


def correlate_batch(backend: B200Backend, batch, y1: BasebandCapture,
                    y2: BasebandCapture) -> np.ndarray:
    """backend.hpp:320-325"""
    return backend.stage(y1, y2).correlate_batch(batch)
