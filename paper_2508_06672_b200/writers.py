"""Surface and detection files (reference io.hpp:169-280), formatted on the GPU.

Same names, arguments and bytes as the reference's writers:

* ``write_grid(grid, path, GridFileFormat.csv | binary)`` — CSV rows
  ``"%.17g,%.17g,%.17g\\n"`` (io.hpp:174-183) or the DGGR binary layout
  (:187-202); ``read_grid(path)`` (:205-240) reads DGGR back, lattice rebuilt on
  the device.
* ``render_heatmap(grid, path)`` — 16-bit P5, min -> 0, max -> 65535, north on
  top (:245-268).
* ``write_detections_csv(detections, path)`` (:270-280).

``grid.values`` may be a host array or a CUDA tensor (the accumulated surface
left on the device by a solve); host values are uploaded once. The text of a
4M-cell CSV is produced by the device formatter (exact "%.17g", dg_writers.cu)
and streamed to the file through a pinned double buffer.
"""
from __future__ import annotations

import ctypes as C
import enum

import numpy as np

from . import _capi
from ._capi import check, lib
from .engine import Engine, default_engine
from .geodesy import GeodeticCoord, GridAxis, grid_from_axes
from .geolocate import CorrelationGrid, EmitterEstimate


class GridFileFormat(enum.IntEnum):
    """io.hpp:169"""
    csv = 0
    binary = 1


def _values(grid: CorrelationGrid):
    """(pointer, on_device, keep-alive) for grid.values (host array or CUDA tensor)."""
    v = grid.values
    n = grid.grid.size()
    if hasattr(v, "is_cuda") and v.is_cuda:
        import torch
        if v.dtype != torch.float64 or v.numel() != n:
            raise ValueError("CorrelationGrid: value count != grid size")
        v = v.contiguous()
        return C.c_void_p(v.data_ptr()), 1, v
    a = np.ascontiguousarray(v, np.float64)
    if a.size != n:
        raise ValueError("CorrelationGrid: value count != grid size")  # correlate.hpp:95-96
    return a.ctypes.data_as(C.c_void_p), 0, a


def write_grid(grid: CorrelationGrid, path, format: GridFileFormat = GridFileFormat.csv,
               engine: Engine | None = None) -> None:
    eng = engine or grid.grid.engine or default_engine()
    ptr, dev, _keep = _values(grid)
    check(lib.dg_write_grid(eng.handle, grid.grid.handle, ptr, dev, str(path).encode(),
                            int(format)))


def render_heatmap(grid: CorrelationGrid, path, engine: Engine | None = None) -> None:
    eng = engine or grid.grid.engine or default_engine()
    ptr, dev, _keep = _values(grid)
    check(lib.dg_render_heatmap(eng.handle, grid.grid.handle, ptr, dev, str(path).encode()))


def write_detections_csv(detections, path) -> None:
    arr = (_capi.dg_emitter_estimate * max(len(detections), 1))()
    for i, d in enumerate(detections):
        arr[i] = _capi.dg_emitter_estimate(d.location.lat_deg, d.location.lon_deg,
                                           d.location.alt_m, int(d.grid_index), d.score,
                                           d.score_zsigma)
    check(lib.dg_write_detections_csv(arr, len(detections), str(path).encode()))


def read_grid_axes(path) -> "_capi.dg_grid_axes":
    a = _capi.dg_grid_axes()
    check(lib.dg_read_grid(str(path).encode(), C.byref(a), None, 0))
    return a


def read_grid(path, engine: Engine | None = None) -> CorrelationGrid:
    a = read_grid_axes(path)
    values = np.empty(a.lat_count * a.lon_count, np.float64)
    check(lib.dg_read_grid(str(path).encode(), C.byref(a),
                           values.ctypes.data_as(C.POINTER(C.c_double)), values.size))
    lattice = grid_from_axes(GridAxis(a.lat_start_deg, a.lat_step_deg, a.lat_count),
                             GridAxis(a.lon_start_deg, a.lon_step_deg, a.lon_count),
                             a.altitude_m, engine)
    return CorrelationGrid(lattice, values)


def format_g17(values, engine: Engine | None = None) -> list[str]:
    """'%.17g' of each value by the device formatter the CSV writer uses."""
    eng = engine or default_engine()
    v = np.ascontiguousarray(values, np.float64).ravel()
    slots = C.create_string_buffer(32 * max(v.size, 1))
    lens = (C.c_uint8 * max(v.size, 1))()
    check(lib.dg_format_g17(eng.handle, v.ctypes.data_as(C.POINTER(C.c_double)), v.size, slots,
                            lens))
    raw = slots.raw
    return [raw[32 * i: 32 * i + lens[i]].decode() for i in range(v.size)]


__all__ = ["GridFileFormat", "write_grid", "read_grid", "read_grid_axes", "render_heatmap",
           "write_detections_csv", "format_g17", "GeodeticCoord", "EmitterEstimate"]
