"""Per-device engine handle (one process per GPU)."""
from __future__ import annotations

import ctypes as C
import os

from ._capi import check, lib


class Engine:
    """Owns a ``dg_engine`` bound to one CUDA device."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.dg_engine_create(int(device), C.byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def descriptor(self):
        name = C.create_string_buffer(32)
        kind = C.create_string_buffer(32)
        workers = C.c_uint()
        check(lib.dg_engine_descriptor(self._h, name, 32, kind, 32, C.byref(workers)))
        return name.value.decode(), kind.value.decode(), workers.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.dg_engine_destroy(h)
            self._h = None


_engines: dict[int, Engine] = {}


def default_device() -> int:
    # one rank per GPU: torchrun's LOCAL_RANK picks the device (CUDA_VISIBLE_DEVICES
    # remapping is respected by the runtime)
    return int(os.environ.get("LOCAL_RANK", "0"))


def default_engine(device: int | None = None) -> Engine:
    dev = default_device() if device is None else int(device)
    eng = _engines.get(dev)
    if eng is None:
        eng = _engines[dev] = Engine(dev)
    return eng
