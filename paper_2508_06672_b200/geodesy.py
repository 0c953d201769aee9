"""Candidate lattice — host mirror of digeo geodesy.hpp:126-207 over the C ABI.

``build_candidate_grid`` keeps the reference's validation, axis counts and
lat-major flat index; the eager ECEF lattice (geodesy.hpp:202-205) is formed
on the GPU by ``dg_build_candidate_grid`` and stays resident in HBM.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, lib
from .engine import Engine, default_engine

DEFAULT_GRID_POINT_CAP = 20_000_000  # geodesy.hpp:170

# wgs84 (geodesy.hpp:31-36)
SEMI_MAJOR_AXIS_M = 6378137.0
FLATTENING = 1.0 / 298.257223563
SEMI_MINOR_AXIS_M = SEMI_MAJOR_AXIS_M * (1.0 - FLATTENING)
ECCENTRICITY_SQ = FLATTENING * (2.0 - FLATTENING)


@dataclass(frozen=True)
class GeodeticCoord:
    """geodesy.hpp:64-79"""
    lat_deg: float = 0.0
    lon_deg: float = 0.0
    alt_m: float = 0.0

    def validate(self) -> None:
        if not (-90.0 <= self.lat_deg <= 90.0):
            raise ValueError(f"GeodeticCoord: lat_deg out of [-90, 90]: {self.lat_deg:f}")
        if not (-180.0 <= self.lon_deg < 180.0):
            raise ValueError(f"GeodeticCoord: lon_deg out of [-180, 180): {self.lon_deg:f}")
        if not math.isfinite(self.alt_m):
            raise ValueError("GeodeticCoord: alt_m not finite")


@dataclass(frozen=True)
class LatLonBounds:
    """geodesy.hpp:126-138 (lon_max is not range-checked, as in the reference)."""
    lat_min_deg: float = 0.0
    lat_max_deg: float = 0.0
    lon_min_deg: float = 0.0
    lon_max_deg: float = 0.0

    def validate(self) -> None:
        GeodeticCoord(self.lat_min_deg, self.lon_min_deg, 0.0).validate()
        GeodeticCoord(self.lat_max_deg, self.lon_min_deg, 0.0).validate()
        if self.lat_max_deg < self.lat_min_deg or self.lon_max_deg < self.lon_min_deg:
            raise ValueError("LatLonBounds: max < min")


@dataclass(frozen=True)
class GridAxis:
    """geodesy.hpp:140-147"""
    start_deg: float = 0.0
    step_deg: float = 0.0
    count: int = 0

    def value(self, i: int) -> float:
        return self.start_deg + float(i) * self.step_deg


class CandidateGrid:
    """geodesy.hpp:151-168: lat-major lattice; ECEF points live on the device."""

    def __init__(self, handle: C.c_void_p, engine: Engine, parent: "CandidateGrid | None" = None):
        self._h = handle
        self.engine = engine
        self._parent = parent  # keeps the shared device lattice alive for slabs
        ls, lst, nl = C.c_double(), C.c_double(), C.c_int64()
        os_, ost, no = C.c_double(), C.c_double(), C.c_int64()
        alt, roff = C.c_double(), C.c_int64()
        check(lib.dg_grid_info(handle, C.byref(ls), C.byref(lst), C.byref(nl), C.byref(os_),
                               C.byref(ost), C.byref(no), C.byref(alt), C.byref(roff)))
        self.lat = GridAxis(ls.value, lst.value, nl.value)
        self.lon = GridAxis(os_.value, ost.value, no.value)
        self.altitude_m = alt.value
        self.row_offset = roff.value
        self._points = None

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        return self.lat.count * self.lon.count

    def index(self, ilat: int, ilon: int) -> int:
        return ilat * self.lon.count + ilon

    def unindex(self, flat: int):
        return flat // self.lon.count, flat % self.lon.count

    def lattice_coord(self, ilat: int, ilon: int) -> GeodeticCoord:
        return GeodeticCoord(self.lat.value(ilat), self.lon.value(ilon), self.altitude_m)

    def same_lattice(self, other: "CandidateGrid") -> bool:
        return (self.lat == other.lat and self.lon == other.lon
                and self.altitude_m == other.altitude_m and self.row_offset == other.row_offset)

    @property
    def points(self) -> np.ndarray:
        """The eager ECEF lattice, [size, 3] float64 (copied from the device once)."""
        if self._points is None:
            buf = (_capi.dg_ecef * self.size())()
            check(lib.dg_grid_points(self._h, buf))
            self._points = np.ctypeslib.as_array(
                C.cast(buf, C.POINTER(C.c_double)), shape=(self.size(), 3)).copy()
        return self._points

    def slab(self, row_begin: int, row_end: int) -> "CandidateGrid":
        """Rows [row_begin, row_end) as a sub-grid sharing the device lattice (one rank's shard)."""
        h = C.c_void_p()
        check(lib.dg_grid_slab(self._h, row_begin, row_end, C.byref(h)))
        return CandidateGrid(h, self.engine, parent=self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.dg_grid_destroy(h)
            self._h = None


def build_candidate_grid(bounds: LatLonBounds, spacing_deg: float, altitude_m: float = 0.0,
                         point_cap: int = DEFAULT_GRID_POINT_CAP,
                         engine: Engine | None = None) -> CandidateGrid:
    """geodesy.hpp:182-207 — same validation and messages, lattice built on the GPU."""
    eng = engine or default_engine()
    b = _capi.dg_latlon_bounds(bounds.lat_min_deg, bounds.lat_max_deg, bounds.lon_min_deg,
                               bounds.lon_max_deg)
    h = C.c_void_p()
    check(lib.dg_build_candidate_grid(eng.handle, C.byref(b), float(spacing_deg),
                                      float(altitude_m), int(point_cap), C.byref(h)))
    return CandidateGrid(h, eng)


def grid_from_points(points: np.ndarray, lat: GridAxis, lon: GridAxis, altitude_m: float = 0.0,
                     engine: Engine | None = None) -> CandidateGrid:
    """Upload an existing eager lattice (e.g. a reference CandidateGrid's points)."""
    eng = engine or default_engine()
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    h = C.c_void_p()
    check(lib.dg_grid_from_points(
        eng.handle, pts.ctypes.data_as(C.POINTER(_capi.dg_ecef)), len(pts), lat.start_deg,
        lat.step_deg, lat.count, lon.start_deg, lon.step_deg, lon.count, altitude_m, C.byref(h)))
    return CandidateGrid(h, eng)


def grid_from_axes(lat: GridAxis, lon: GridAxis, altitude_m: float = 0.0,
                   engine: Engine | None = None) -> CandidateGrid:
    """The eager lattice of explicit axes (as read_grid rebuilds it, io.hpp:229-232),
    built on the GPU like build_candidate_grid."""
    eng = engine or default_engine()
    a = _capi.dg_grid_axes(lat.start_deg, lat.step_deg, lat.count, lon.start_deg, lon.step_deg,
                           lon.count, altitude_m)
    h = C.c_void_p()
    check(lib.dg_grid_from_axes(eng.handle, C.byref(a), C.byref(h)))
    return CandidateGrid(h, eng)
