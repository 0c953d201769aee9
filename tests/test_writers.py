"""Surface / detection writers against the reference's io.hpp.

Every file is compared byte for byte with the one the reference's own writer
(oracle/_ref: write_grid, render_heatmap, write_detections_csv) produces from
the same values; the device "%.17g" formatter is checked against the C
library's snprintf on special, tie, boundary and random-bit-pattern doubles.
CPU: the reader's checks and messages against read_grid's (host code).
"""
import ctypes
import ctypes.util
import os
import struct

import numpy as np
import pytest

from oracle.bindings import ReferenceError_

_libc = ctypes.CDLL(ctypes.util.find_library("c"))


def c_g17(v: float) -> str:
    buf = ctypes.create_string_buffer(64)
    _libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
    return buf.value.decode()


@pytest.fixture(scope="module")
def lib():
    import paper_2508_06672_b200 as b2
    return b2


def _axes(lat0, dlat, nlat, lon0, dlon, nlon):
    return (lat0, dlat, nlat, lon0, dlon, nlon)


def _dggr(lat=(0.0, 0.5, 2), lon=(1.0, 0.25, 3), alt=0.0, count=None, payload=None,
          magic=b"DGGR", version=1):
    n = lat[2] * lon[2]
    count = n if count is None else count
    h = magic + struct.pack("<HddQddQdQ", version, lat[0], lat[1], lat[2], lon[0], lon[1], lon[2],
                            alt, count)
    return h + (payload if payload is not None else np.arange(n, dtype="<f8").tobytes())


# ---------------------------------------------------------------- CPU (host reader)

def test_read_grid_matches_reference(lib, ref, tmp_path):
    rng = np.random.default_rng(3)
    v = rng.standard_normal(6 * 7)
    p = tmp_path / "g.dggr"
    ref.write_grid(p, _axes(-3.0, 0.125, 6, 10.0, 0.5, 7), 12.5, v, csv=False)
    axes, alt, want = ref.read_grid(p)
    a = lib.writers.read_grid_axes(p)
    got = (a.lat_start_deg, a.lat_step_deg, a.lat_count, a.lon_start_deg, a.lon_step_deg,
           a.lon_count)
    assert got == tuple(axes) and a.altitude_m == alt


@pytest.mark.parametrize("name,data", [
    ("short", b"DG"),
    ("magic", _dggr(magic=b"XXXX")),
    ("version", _dggr(version=2)),
    ("truncated_header", _dggr()[:40]),
    ("count", _dggr(count=5)),
    ("payload", _dggr()[:-8]),
])
def test_read_grid_errors_match_reference(lib, ref, tmp_path, name, data):
    p = tmp_path / f"{name}.dggr"
    p.write_bytes(data)
    with pytest.raises(ReferenceError_) as want:
        ref.read_grid(p)
    with pytest.raises(RuntimeError) as got:
        lib.writers.read_grid_axes(p)
    assert str(got.value) == str(want.value)


def test_read_grid_missing_file(lib, ref, tmp_path):
    p = tmp_path / "nope.dggr"
    with pytest.raises(ReferenceError_) as want:
        ref.read_grid(p)
    with pytest.raises(RuntimeError) as got:
        lib.writers.read_grid_axes(p)
    assert str(got.value) == str(want.value)


def test_detections_csv_matches_reference(lib, ref, tmp_path):
    rows = [(12.345678901234567, -0.1, 0.0, 17, 3.5e10, 9.25), (1e-300, 179.99, -5.0, 0, 0.0, -1.5)]
    ref.write_detections_csv(tmp_path / "r.csv", rows)
    dets = [lib.EmitterEstimate(lib.GeodeticCoord(r[0], r[1], r[2]), r[3], r[4], r[5]) for r in rows]
    lib.write_detections_csv(dets, tmp_path / "b.csv")
    assert (tmp_path / "b.csv").read_bytes() == (tmp_path / "r.csv").read_bytes()
    lib.write_detections_csv([], tmp_path / "e.csv")
    ref.write_detections_csv(tmp_path / "re.csv", [])
    assert (tmp_path / "e.csv").read_bytes() == (tmp_path / "re.csv").read_bytes()


# ---------------------------------------------------------------- GPU

def _special_doubles():
    f = np.finfo(np.float64)
    v = [0.0, -0.0, 1.0, -1.0, 0.1, 0.5, 2.0 / 3.0, 1e16, 1e17, 1e-5, 1e-4, 9.999e-5, 123456.789,
         f.max, -f.max, f.tiny, 5e-324, 2.2250738585072009e-308, 1e22, 1e23, 2 ** 53, 2 ** 53 + 2,
         2 ** 60, 99999999999999999.0, 0.30000000000000004, 179.99999999999997,
         -89.999999999999986, np.inf, -np.inf, np.nan]
    for k in range(-320, 309):  # powers of ten and their neighbours
        p = 10.0 ** k
        v += [p, np.nextafter(p, 0), np.nextafter(p, np.inf)]
    for j in range(1, 400, 2):  # exact 18-digit ties: 1 + j 2^-17, 2^k + j 2^(k-17) ...
        for e in (0, 3, 10, 20):
            v.append((1.0 + j * 2.0 ** -17) * 2.0 ** e)
    return np.array(v, np.float64)


@pytest.mark.gpu
def test_format_g17_matches_libc(lib):
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2 ** 63, 100_000, dtype=np.int64).view(np.float64)
    vals = np.concatenate([_special_doubles(), bits, rng.standard_normal(20_000) * 1e3,
                           rng.uniform(-180, 180, 20_000)])
    got = lib.writers.format_g17(vals)
    bad = [(v, g, c_g17(v)) for v, g in zip(vals, got) if g != c_g17(v)]
    assert not bad, bad[:10]


def _surface(lib, bounds, spacing, values):
    grid = lib.build_candidate_grid(lib.LatLonBounds(*bounds), spacing)
    return lib.CorrelationGrid(grid, values)


def _ref_axes(g):
    return _axes(g.lat.start_deg, g.lat.step_deg, g.lat.count, g.lon.start_deg, g.lon.step_deg,
                 g.lon.count)


@pytest.mark.gpu
@pytest.mark.parametrize("bounds,spacing", [((-1.0, 1.0, -2.0, 2.0), 0.01),
                                            ((-60.0, 60.0, -179.5, 179.5), 0.7),
                                            ((10.0, 10.0, 20.0, 20.0), 0.1)])
def test_write_grid_csv_and_binary_match_reference(lib, ref, tmp_path, bounds, spacing):
    grid = lib.build_candidate_grid(lib.LatLonBounds(*bounds), spacing)
    rng = np.random.default_rng(grid.size())
    v = rng.gamma(2.0, 1e4, grid.size())
    v[:3] = [0.0, 1e-310, 123.0][: min(3, v.size)]
    cg = lib.CorrelationGrid(grid, v)
    for fmt, csv in ((lib.GridFileFormat.csv, True), (lib.GridFileFormat.binary, False)):
        lib.write_grid(cg, tmp_path / "b.out", fmt)
        ref.write_grid(tmp_path / "r.out", _ref_axes(grid), grid.altitude_m, v, csv)
        assert (tmp_path / "b.out").read_bytes() == (tmp_path / "r.out").read_bytes()
    back = lib.read_grid(tmp_path / "b.out")
    assert np.array_equal(back.values, v) and back.grid.same_lattice(grid)
    assert np.array_equal(back.grid.points, grid.points)  # the lattice read_grid rebuilds


@pytest.mark.gpu
def test_writers_from_device_values(lib, ref, tmp_path):
    """The accumulated surface left on the device by a solve writes the same bytes."""
    import torch
    grid = lib.build_candidate_grid(lib.LatLonBounds(-0.5, 0.5, -0.5, 0.5), 0.01)
    rng = np.random.default_rng(2)
    v = rng.gamma(3.0, 50.0, grid.size())
    dv = torch.from_numpy(v).cuda()
    cg = lib.CorrelationGrid(grid, dv)
    lib.write_grid(cg, tmp_path / "b.csv", lib.GridFileFormat.csv)
    lib.render_heatmap(cg, tmp_path / "b.pgm")
    ref.write_grid(tmp_path / "r.csv", _ref_axes(grid), 0.0, v, True)
    ref.render_heatmap(tmp_path / "r.pgm", _ref_axes(grid), 0.0, v)
    assert (tmp_path / "b.csv").read_bytes() == (tmp_path / "r.csv").read_bytes()
    assert (tmp_path / "b.pgm").read_bytes() == (tmp_path / "r.pgm").read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["random", "constant", "negative"])
def test_render_heatmap_matches_reference(lib, ref, tmp_path, kind):
    grid = lib.build_candidate_grid(lib.LatLonBounds(-2.0, 3.0, 5.0, 9.0), 0.05)
    rng = np.random.default_rng(7)
    v = {"random": rng.gamma(2.0, 1e3, grid.size()), "constant": np.full(grid.size(), 4.25),
         "negative": rng.standard_normal(grid.size())}[kind]
    lib.render_heatmap(lib.CorrelationGrid(grid, v), tmp_path / "b.pgm")
    ref.render_heatmap(tmp_path / "r.pgm", _ref_axes(grid), 0.0, v)
    assert (tmp_path / "b.pgm").read_bytes() == (tmp_path / "r.pgm").read_bytes()


@pytest.mark.gpu
def test_slab_csv_rows_are_the_full_grids(lib, tmp_path):
    grid = lib.build_candidate_grid(lib.LatLonBounds(-1.0, 1.0, 0.0, 1.0), 0.1)
    v = np.arange(grid.size(), dtype=np.float64) / 3.0
    lib.write_grid(lib.CorrelationGrid(grid, v), tmp_path / "full.csv")
    slab = grid.slab(5, 12)
    lib.write_grid(lib.CorrelationGrid(slab, v[5 * grid.lon.count: 12 * grid.lon.count]),
                   tmp_path / "slab.csv")
    full = (tmp_path / "full.csv").read_text().splitlines()
    part = (tmp_path / "slab.csv").read_text().splitlines()
    assert part[0] == full[0]
    assert part[1:] == full[1 + 5 * grid.lon.count: 1 + 12 * grid.lon.count]


@pytest.mark.gpu
def test_write_errors_match_reference(lib, ref, tmp_path):
    grid = lib.build_candidate_grid(lib.LatLonBounds(0.0, 0.1, 0.0, 0.1), 0.05)
    v = np.ones(grid.size())
    p = tmp_path / "missing_dir" / "x.csv"
    with pytest.raises(ReferenceError_) as want:
        ref.write_grid(p, _ref_axes(grid), 0.0, v, True)
    for call in (lambda: lib.write_grid(lib.CorrelationGrid(grid, v), p),
                 lambda: lib.render_heatmap(lib.CorrelationGrid(grid, v), p)):
        with pytest.raises(RuntimeError) as got:
            call()
        assert str(got.value) == str(want.value)
    with pytest.raises(ValueError):
        lib.write_grid(lib.CorrelationGrid(grid, v[:-1]), tmp_path / "y.csv")
