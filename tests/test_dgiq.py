"""DGIQ capture ingest against the reference's io.hpp.

CPU: the engine's reader (C ABI, host code) reads files written by the
reference's write_iq (io.hpp:123-138) to exactly the reference's read_iq
values (io.hpp:140-167), and rejects malformed files with read_iq's exception
type and message. GPU: a run staged from DGIQ files solves bit-identically to
the same float32 captures staged from arrays.
"""
import os
import struct

import numpy as np
import pytest

from oracle.bindings import ReferenceError_


@pytest.fixture(scope="module")
def lib():
    import paper_2508_06672_b200 as b2
    return b2


def test_read_matches_reference(lib, ref, tmp_path):
    rng = np.random.default_rng(5)
    y = (rng.standard_normal(1000) + 1j * rng.standard_normal(1000)) * 3.0
    path = tmp_path / "cap.dgiq"
    ref.write_iq(path, y, 5e6, 1575.42e6, 12.5)
    want, fs, fc, t0 = ref.read_iq(path)
    cap = lib.read_iq(path)
    assert (cap.sample_rate_hz, cap.center_freq_hz, cap.start_time_s) == (fs, fc, t0)
    assert cap.samples.dtype == np.complex64
    assert np.array_equal(cap.samples.astype(np.complex128), want)  # float32 widened exactly
    h = lib.read_iq_header(path)
    assert h.sample_count == 1000


def _header(magic=b"DGIQ", version=1, fs=1e6, fc=1.5e9, t0=0.0, count=4):
    return magic + struct.pack("<Hdddq", version, fs, fc, t0, count)


@pytest.mark.parametrize("name,blob", [
    ("magic", _header(magic=b"XXXX") + bytes(32)),
    ("version", _header(version=2) + bytes(32)),
    ("truncated", _header()[:20]),
    ("payload", _header(count=5) + bytes(32)),
    ("empty", _header(count=0)),
    ("rate", _header(fs=0.0) + bytes(32)),
])
def test_errors_match_reference(lib, ref, tmp_path, name, blob):
    path = tmp_path / f"{name}.dgiq"
    path.write_bytes(blob)
    with pytest.raises(ReferenceError_) as want:
        ref.read_iq(path)
    exc = ValueError if want.value.code == 1 else RuntimeError
    with pytest.raises(exc) as got:
        lib.read_iq(path)
    assert str(got.value) == str(want.value)


def test_missing_file(lib, ref, tmp_path):
    path = tmp_path / "nope.dgiq"
    with pytest.raises(ReferenceError_) as want:
        ref.read_iq(path)
    with pytest.raises(RuntimeError) as got:
        lib.read_iq(path)
    assert str(got.value) == str(want.value)


@pytest.mark.gpu
def test_stage_from_files_matches_arrays(lib, ref, tmp_path):
    import scenes
    sc = ref.simulate(scenes.render(scenes.DESK_SAWTOOTH))
    S, R, _ = sc.captures.shape
    paths = []
    for s in range(S):
        row = []
        for r in range(R):
            p = tmp_path / f"s{s}_r{r}.dgiq"
            ref.write_iq(p, sc.captures[s, r], sc.fs, sc.fc, float(s))
            row.append(str(p))
        paths.append(row)
    grid = lib.build_candidate_grid(lib.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    from_files = lib.StagedSnapshots.from_iq_files(paths, sc.states)
    caps32 = sc.captures.astype(np.complex64)
    from_arrays = lib.StagedSnapshots(sc.states, caps32, sc.fs, sc.fc)
    opts = lib.GeolocateOptions(detect=True)
    a = lib.geolocate_staged(grid, from_files, opts)
    b = lib.geolocate_staged(grid, from_arrays, opts)
    assert np.array_equal(a.accumulated.values, b.accumulated.values)
    assert (a.argmax_index, a.argmax_value) == (b.argmax_index, b.argmax_value)
    assert [d.grid_index for d in a.detections] == [d.grid_index for d in b.detections]
    # and the reference's own file-based answer: argmax of read-back captures
    want = ref.geolocate(sc.states, caps32.astype(np.complex128), sc.fs, sc.fc, sc.bounds,
                         sc.spacing, sc.alt, backend="parallel", batch_size=4096)
    assert a.argmax_index == int(np.argmax(want["accumulated"]))
