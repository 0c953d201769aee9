"""Per-device engine handle (one process per GPU)."""
from __future__ import annotations

import ctypes as C
import os

from . import _capi
from ._capi import check, lib


def device_count() -> int:
    n = C.c_int()
    check(lib.dg_device_count(C.byref(n)))
    return n.value


class Engine:
    """Owns a ``dg_engine`` bound to one CUDA device, or to several
    (``devices``: one process drives every listed GPU; whole-run solves are
    sharded across them, dg_engine_create_multi)."""

    def __init__(self, device: int = 0, devices=None):
        h = C.c_void_p()
        if devices is not None and len(devices) > 1:
            arr = (C.c_int * len(devices))(*[int(d) for d in devices])
            check(lib.dg_engine_create_multi(arr, len(devices), C.byref(h)))
            self.devices = [int(d) for d in devices]
        else:
            dev = int(devices[0]) if devices else int(device)
            check(lib.dg_engine_create(dev, C.byref(h)))
            self.devices = [dev]
        self._h = h
        self.device = self.devices[0]

    @property
    def handle(self):
        return self._h

    def descriptor(self):
        name = C.create_string_buffer(32)
        kind = C.create_string_buffer(32)
        workers = C.c_uint()
        check(lib.dg_engine_descriptor(self._h, name, 32, kind, 32, C.byref(workers)))
        return name.value.decode(), kind.value.decode(), workers.value

    def tuning(self) -> dict:
        t = _capi.dg_tuning()
        check(lib.dg_engine_get_tuning(self._h, C.byref(t)))
        return {name: getattr(t, name) for name, _ in t._fields_}

    def set_tuning(self, **kw) -> None:
        """Correlator tuning for tests / benchmarks (dg_engine_set_tuning, validated
        by the library): correlator ("auto" | "direct" | "moments"), moment_block,
        moment_count, evaluate_tensor, refine_tau, allow_weaker_refine. Keys not
        given keep the library default."""
        t = _capi.dg_tuning()
        lib.dg_tuning_default(C.byref(t))
        modes = {"auto": _capi.DG_CORRELATOR_AUTO, "direct": _capi.DG_CORRELATOR_DIRECT,
                 "moments": _capi.DG_CORRELATOR_MOMENTS}
        for k, v in kw.items():
            if k == "correlator" and isinstance(v, str):
                v = modes[v]
            if not hasattr(t, k):
                raise ValueError(f"set_tuning: unknown key {k}")
            setattr(t, k, v)
        check(lib.dg_engine_set_tuning(self._h, C.byref(t)))

    def reset_tuning(self) -> None:
        t = _capi.dg_tuning()
        lib.dg_tuning_default(C.byref(t))
        check(lib.dg_engine_set_tuning(self._h, C.byref(t)))

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
