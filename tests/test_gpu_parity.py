"""GPU parity: the B200 engine (through the C ABI) against the reference.

Tolerances (the reference's own equivalence contract):
* integer / index results bit-exact: lattice ECEF doubles, TDOA samples, FDOA
  doubles, argmax flat index (and its accumulated value), detection lists;
* correlation values per element  |a-b| / max(|a|,|b|) <= 1e-4
  (bench.hpp:135-142, test_backend.cpp:91-94);
* accumulated surface normwise  max|a-b| / max|a| <= 1e-5.
"""
import json
import os
import threading

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.bindings import PAIR_OFFSETS_DTYPE

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
NORM_TOL = 1e-5


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)


def gauss(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def random_offsets(rng, count, n, span):
    off = np.zeros(count, PAIR_OFFSETS_DTYPE)
    off["tdoa_samples"] = rng.integers(-n, n, count)
    off["fdoa_hz"] = rng.uniform(-span, span, count)
    return off


def cap(b2, y, fs):
    return b2.BasebandCapture(y, fs)


# ---------------------------------------------------------------------------
# geometry: lattice and offsets are bit-exact
@pytest.mark.parametrize("bounds,spacing,alt", [
    ((-1.0, 1.0, 10.0, 11.0), 0.25, 120.0),   # test_geodesy.cpp:99-113
    ((0.0, 10.0, 0.0, 10.0), 0.01, 0.0),      # the 1001x1001 grid (test_geodesy.cpp:73-78)
    ((5.0, 5.0, 7.0, 7.0), 0.5, 0.0),         # zero span
    ((-89.5, 89.5, -179.5, 179.0), 0.5, 3000.0),
])
def test_grid_bit_exact(b2, ref, bounds, spacing, alt):
    g = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing, alt)
    nl, nn, pts = ref.build_grid(bounds, spacing, alt)
    assert (g.lat.count, g.lon.count) == (nl, nn)
    assert np.array_equal(g.points, pts)


def test_grid_errors_match_reference(b2, ref):
    from oracle.bindings import ReferenceError_
    cases = [((0.0, 10.0, 0.0, 10.0), 0.01, 0.0, 1000),   # over cap
             ((0.0, 1.0, 0.0, 1.0), 0.0, 0.0, 0),          # spacing
             ((0.0, 1.0, 170.0, 185.0), 1.0, 0.0, 0),      # lon >= 180 in the lattice
             ((-91.0, 1.0, 0.0, 1.0), 0.1, 0.0, 0),
             ((0.0, 1.0, 0.0, 1.0), 0.1, float("inf"), 0)]
    for bounds, sp, alt, capn in cases:
        with pytest.raises(ReferenceError_) as r:
            ref.build_grid(bounds, sp, alt, cap=capn or 20_000_000)
        with pytest.raises(ValueError) as m:
            b2.build_candidate_grid(b2.LatLonBounds(*bounds), sp, alt, point_cap=capn or 20_000_000)
        assert str(m.value) == str(r.value)


def test_offsets_bit_exact_golden(b2):
    g = np.load(os.path.join(GOLDEN, "offsets_small.npz"))
    grid = b2.build_candidate_grid(b2.LatLonBounds(*g["bounds"]), float(g["spacing"]))
    assert np.array_equal(grid.points, g["points"])
    for s in range(g["states"].shape[0]):
        got = b2.predict_offsets(grid, g["states"][s, 0], g["states"][s, 1], float(g["fs"]),
                                 float(g["wavelength"]))
        assert np.array_equal(got, g["offsets"][s])


def test_offsets_bit_exact_random_geometries(b2, ref):
    rng = np.random.default_rng(60606)
    grid = b2.build_candidate_grid(b2.LatLonBounds(-30, 30, -60, 60), 1.5, 250.0)
    pts = grid.points
    wl = ref.wavelength(1575.42e6)
    for _ in range(4):
        a = np.r_[ref.lla_to_ecef(rng.uniform(-60, 60), rng.uniform(-120, 120),
                                  rng.uniform(400e3, 1200e3)), rng.uniform(-7600, 7600, 3)]
        b = np.r_[ref.lla_to_ecef(rng.uniform(-60, 60), rng.uniform(-120, 120),
                                  rng.uniform(400e3, 1200e3)), rng.uniform(-7600, 7600, 3)]
        got = b2.predict_offsets(grid, a, b, 5e6, wl)
        want = np.array([ref.predict_pair_offsets(p, a, b, 5e6, wl) for p in pts],
                        PAIR_OFFSETS_DTYPE)
        assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# correlate_batch: the plugin interface (backend.hpp:196-217)
def test_descriptor(b2):
    d = b2.make_backend("b200").descriptor()
    assert (d.name, d.kind, d.workers) == ("b200", "parallel-batched", 1)


def test_known_answers(b2):
    be = b2.make_backend("b200")
    ones = np.ones(1000, np.complex128)
    s = be.stage(cap(b2, ones, 1e6), cap(b2, ones, 1e6))
    assert s.correlate_batch([(0, 0.0)])[0] == pytest.approx(1000.0, rel=1e-12)
    ones = np.ones(100, np.complex128)
    s = be.stage(cap(b2, ones, 1e6), cap(b2, ones, 1e6))
    out = s.correlate_batch([(100, 0.0), (-250, 0.0), (40, 0.0), (-30, 0.0)])
    assert out[0] == 0.0 and out[1] == 0.0
    assert out[2] == pytest.approx(60.0, rel=1e-12) and out[3] == pytest.approx(70.0, rel=1e-12)
    # full-period exponential is orthogonal to a constant (test_correlate.cpp:68-76):
    # the FP32 sum would miss N*1e-10; the exact FP64 re-evaluation must catch it
    n, fs = 4096, 1e6
    ones = np.ones(n, np.complex128)
    s = be.stage(cap(b2, ones, fs), cap(b2, ones, fs))
    out = s.correlate_batch([(0, m * fs / n) for m in (1, 2, 5, -3)])
    assert np.all(out < n * 1e-10)


def test_golden_correlate_batch(b2):
    g = np.load(os.path.join(GOLDEN, "correlate_small.npz"))
    fs = float(g["fs"])
    s = b2.make_backend("b200").stage(cap(b2, g["y1"], fs), cap(b2, g["y2"], fs))
    got = s.correlate_batch(g["offsets"])
    assert rel_err(got, g["want"]).max() <= REL_TOL
    assert np.array_equal(got[g["want"] == 0.0], g["want"][g["want"] == 0.0])


@pytest.mark.parametrize("n,count,fs,span,seed", [
    (2000, 10_000, 5e6, 1.25e6, 13),     # test_backend.cpp:80-95
    (2048, 10_000, 2.048e6, 5e5, 0xBA7C),  # acceptance.cpp criterion 4
    (4096, 20_000, 5e6, 1.25e6, 1),      # BenchWorkload distribution (bench.hpp:65-88)
    (50_000, 4_000, 5e6, 2e4, 3),        # C2..C5 capture length
])
@pytest.mark.parametrize("mode", ["auto", "direct", "moments"])  # moments: when admissible
def test_correlate_batch_vs_reference(b2, ref, n, count, fs, span, seed, mode, tune):
    tune(correlator=mode)
    rng = np.random.default_rng(seed)
    y1, y2 = gauss(rng, n), gauss(rng, n)
    if seed == 1:  # BenchWorkload: uniform [-1, 1] I/Q, |tdoa| <= N/2
        y1 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        y2 = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    off = random_offsets(rng, count, n if seed != 1 else n // 2, span)
    want = ref.correlate_batch(y1, y2, fs, off, "parallel", 0, 4096)
    s = b2.make_backend("b200").stage(cap(b2, y1, fs), cap(b2, y2, fs))
    got = s.correlate_batch(off)
    assert rel_err(got, want).max() <= REL_TOL
    again = s.correlate_batch(off)
    assert np.array_equal(got, again)  # bit-identical rerun (test_backend.cpp:97-108)


@pytest.mark.parametrize("block", [64, 128, 256, 512, 640, 768])
@pytest.mark.parametrize("span,tdoa_span", [(2e4, 50_000), (3e3, 4_000), (0.0, 200),
                                            (3e3, 12)])  # ~250 per bucket: 2 tiles
# block sums on tcgen05 with FFT / direct-sum moments, or the FFMA2 block loop
@pytest.mark.parametrize("tc,fft", [(1, 1), (1, 0), (0, 0)])
def test_block_moments_vs_reference(b2, ref, block, span, tdoa_span, tc, fft, tune):
    """The block-moment correlator at every block length against the reference,
    on buckets dense enough that it is the planner's choice (many candidates
    per TDOA), including FDOA == 0 (x = 0) and the full TDOA range; moments as
    FFT cross-correlations (k_mfft, B >= 256) or direct sums (k_moments);
    candidate evaluation on the tensor cores (k_evaluate_tc) and on the FFMA2
    block loop."""
    tune(correlator="moments", moment_block=block, evaluate_tensor=tc, moment_fft=fft)
    n, fs, count = 50_000, 5e6, 6_000
    rng = np.random.default_rng(block + int(span))
    y1, y2 = gauss(rng, n), gauss(rng, n)
    off = np.zeros(count, PAIR_OFFSETS_DTYPE)
    off["tdoa_samples"] = rng.integers(-tdoa_span, tdoa_span, count) if tdoa_span < n else \
        rng.integers(-n + 1, n, count)
    off["fdoa_hz"] = rng.uniform(-span, span, count)
    off["fdoa_hz"][:50] = 0.0
    want = ref.correlate_batch(y1, y2, fs, off, "parallel", 0, 4096)
    s = b2.make_backend("b200").stage(cap(b2, y1, fs), cap(b2, y2, fs))
    got = s.correlate_batch(off)
    assert rel_err(got, want).max() <= REL_TOL
    assert np.array_equal(got, s.correlate_batch(off))


def test_partition_invariance(b2):
    """Any batch partition concatenates to the unbatched result, bit for bit."""
    rng = np.random.default_rng(31)
    n = 1024
    y1, y2 = gauss(rng, n), gauss(rng, n)
    off = random_offsets(rng, 257, n, 1.25e6)
    s = b2.make_backend("b200").stage(cap(b2, y1, 5e6), cap(b2, y2, 5e6))
    whole = s.correlate_batch(off)
    for bs in (1, 2, 7, 8, 64, 257, 1000):
        plan = b2.plan_batches(len(off), bs)
        out = np.zeros(len(off))
        for b in range(plan.batch_count()):
            lo, hi = plan.batch_range(b)
            out[lo:hi] = s.correlate_batch(off[lo:hi])
        assert np.array_equal(out, whole)


def test_concurrent_sessions(b2):
    """One backend serves concurrent sessions for distinct snapshots (test_backend.cpp:148-173)."""
    rng = np.random.default_rng(61)
    n = 1200
    caps = [gauss(rng, n) for _ in range(4)]
    off = random_offsets(rng, 2000, n, 1.25e6)
    be = b2.make_backend("b200")
    want_a = be.stage(cap(b2, caps[0], 5e6), cap(b2, caps[1], 5e6)).correlate_batch(off)
    want_b = be.stage(cap(b2, caps[2], 5e6), cap(b2, caps[3], 5e6)).correlate_batch(off)
    got = {}

    def run(key, i, j):
        got[key] = be.stage(cap(b2, caps[i], 5e6), cap(b2, caps[j], 5e6)).correlate_batch(off)

    th = [threading.Thread(target=run, args=("a", 0, 1)), threading.Thread(target=run, args=("b", 2, 3))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert np.array_equal(got["a"], want_a) and np.array_equal(got["b"], want_b)


def test_invariance_properties(b2, ref):
    """Common unit phasor and positive scaling (test_correlate.cpp:114-129), to tolerance."""
    rng = np.random.default_rng(5)
    y1, y2 = gauss(rng, 2048), gauss(rng, 2048)
    be = b2.make_backend("b200")
    base = be.stage(cap(b2, y1, 1e6), cap(b2, y2, 1e6)).correlate_batch([(17, 1234.5)])[0]
    u = np.exp(1j * 0.7321)
    rot = be.stage(cap(b2, y1 * u, 1e6), cap(b2, y2 * u, 1e6)).correlate_batch([(17, 1234.5)])[0]
    sc = be.stage(cap(b2, y1 * 3.5, 1e6), cap(b2, y2, 1e6)).correlate_batch([(17, 1234.5)])[0]
    assert rot == pytest.approx(base, rel=REL_TOL)
    assert sc == pytest.approx(3.5 * base, rel=REL_TOL)
    assert base == pytest.approx(ref.correlate_point(y1, y2, 1e6, 17, 1234.5), rel=REL_TOL)


def test_stage_errors(b2):
    be = b2.make_backend("b200")
    rng = np.random.default_rng(51)
    a, b = gauss(rng, 100), gauss(rng, 100)
    with pytest.raises(ValueError, match="sample rates differ"):
        be.stage(cap(b2, a, 5e6), cap(b2, b, 2e6))
    with pytest.raises(ValueError, match="sample counts differ"):
        be.stage(cap(b2, a, 5e6), cap(b2, gauss(rng, 101), 5e6))
    with pytest.raises(ValueError, match="no samples"):
        be.stage(cap(b2, a[:0], 5e6), cap(b2, b[:0], 5e6))
    s = be.stage(cap(b2, a, 5e6), cap(b2, b, 5e6))
    with pytest.raises(ValueError, match="empty batch"):
        s.correlate_batch(np.zeros(0, PAIR_OFFSETS_DTYPE))
    with pytest.raises(ValueError, match="output size mismatch"):
        s.correlate_batch([(0, 0.0), (1, 0.0)], out=np.zeros(3))


def test_float32_captures(b2, ref):
    """DGIQ float I/Q staged as-is equals the reference fed the widened doubles."""
    rng = np.random.default_rng(9)
    n = 3000
    y1 = gauss(rng, n).astype(np.complex64)
    y2 = gauss(rng, n).astype(np.complex64)
    off = random_offsets(rng, 3000, n, 1e6)
    want = ref.correlate_batch(y1.astype(np.complex128), y2.astype(np.complex128), 5e6, off)
    got = b2.make_backend("b200").stage(cap(b2, y1, 5e6), cap(b2, y2, 5e6)).correlate_batch(off)
    assert rel_err(got, want).max() <= REL_TOL


# ---------------------------------------------------------------------------
# driver: correlate_snapshot / geolocate_snapshots
def load_scene(ref, name):
    import scenes
    return ref.simulate(scenes.render(getattr(scenes, name)))


def test_correlate_snapshot_vs_reference(b2, ref):
    sc = load_scene(ref, "DESK_FOURJAM")
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    be = b2.make_backend("b200")
    snap = b2.Snapshot(0.0, sc.states[0], [b2.BasebandCapture(sc.captures[0, r], sc.fs, 0.0, sc.fc)
                                           for r in range(2)])
    got = b2.correlate_snapshot(grid, snap, (0, 1), be).values
    want = ref.correlate_snapshot_timed(sc.states[0, 0], sc.states[0, 1], sc.captures[0, 0],
                                        sc.captures[0, 1], sc.fs, sc.fc, sc.bounds, sc.spacing,
                                        sc.alt, backend="parallel", batch_size=4096)[1]
    assert rel_err(got, want).max() <= REL_TOL
    with pytest.raises(ValueError, match="bad receiver pair"):
        b2.correlate_snapshot(grid, snap, (0, 0), be)
    with pytest.raises(ValueError, match="bad receiver pair"):
        b2.correlate_snapshot(grid, snap, (0, 5), be)


@pytest.mark.parametrize("name", ["DESK_FOURJAM", "DESK_SAWTOOTH", "TRIPLE_RX"])
def test_geolocate_scene_vs_reference(b2, ref, name):
    want_g = json.load(open(os.path.join(GOLDEN, "scenes.json")))[name]
    sc = load_scene(ref, name)
    want = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                         backend="parallel", batch_size=4096, k_sigma=sc.k_sigma,
                         radius=sc.radius, per_snapshot=True)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    snaps = [b2.Snapshot(float(s), sc.states[s], [b2.BasebandCapture(sc.captures[s, r], sc.fs, 0.0,
                                                                     sc.fc)
                                                  for r in range(sc.n_rx)])
             for s in range(sc.n_snapshots)]
    res = b2.geolocate_snapshots(snaps, grid, b2.GeolocateOptions(
        k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius))
    acc = res.accumulated.values
    # argmax: bit-exact index and bit-identical exact value
    assert res.argmax_index == int(np.argmax(want["accumulated"])) == want_g["argmax"]
    assert res.argmax_value == float.fromhex(want_g["argmax_value"])
    assert acc[res.argmax_index] == res.argmax_value  # patch_peak: exact value in the surface
    assert int(np.argmax(acc)) == res.argmax_index
    # detections: identical cells and order
    assert [d.grid_index for d in res.detections] == want_g["detections"] == \
        [d["grid_index"] for d in want["detections"]]
    for d, w in zip(res.detections, want["detections"]):
        assert d.score == pytest.approx(w["score"], rel=REL_TOL)
        assert (d.location.lat_deg, d.location.lon_deg) == (w["lat_deg"], w["lon_deg"])
    per = np.stack([g.values for g in res.per_snapshot])
    assert rel_err(per, want["per_snapshot"]).max() <= REL_TOL
    assert np.abs(acc - want["accumulated"]).max() / np.abs(want["accumulated"]).max() <= NORM_TOL


def test_scene_small_golden(b2):
    g = np.load(os.path.join(GOLDEN, "scene_small.npz"))
    grid = b2.build_candidate_grid(b2.LatLonBounds(*g["bounds"]), float(g["spacing"]),
                                   float(g["alt"]))
    res = b2.geolocate_arrays(grid, g["states"], g["captures"], float(g["fs"]), float(g["fc"]),
                              b2.GeolocateOptions(k_sigma=float(g["k_sigma"]),
                                                  exclusion_radius_cells=int(g["radius"])))
    per = np.stack([x.values for x in res.per_snapshot])
    assert rel_err(per, g["per_snapshot"]).max() <= REL_TOL
    assert res.argmax_index == int(np.argmax(g["accumulated"]))
    assert res.argmax_value == g["accumulated"][res.argmax_index]
    assert [d.grid_index for d in res.detections] == list(g["detections"]["grid_index"])


def test_normalize_per_snapshot(b2, ref):
    """geolocate.hpp:115-122: median normalisation before accumulating."""
    sc = load_scene(ref, "DESK_SAWTOOTH")
    want = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                         backend="parallel", batch_size=4096, k_sigma=sc.k_sigma,
                         radius=sc.radius, normalize=True, per_snapshot=True)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    res = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, b2.GeolocateOptions(
        k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius, normalize_per_snapshot=True))
    per = np.stack([x.values for x in res.per_snapshot])
    assert rel_err(per, want["per_snapshot"]).max() <= REL_TOL
    for g in per:
        assert np.sort(g)[len(g) // 2] == pytest.approx(1.0, rel=1e-12)
    assert res.argmax_index == int(np.argmax(want["accumulated"]))
    assert [d.grid_index for d in res.detections] == [d["grid_index"] for d in want["detections"]]


def test_noise_free_argmax_per_waveform(b2, ref):
    """test_geolocate.cpp:56-86: noise-free accumulated argmax on the emitter node."""
    import scenes
    for wf in (scenes._spoofer(0.1, -0.15, 0.0, 7, 5), scenes._tone(0.1, -0.15, 0.0),
               scenes._chirp(0.1, -0.15, 0.0, 1e6, 50e-6), scenes._saw(0.1, -0.15, 0.0, 200e3, 250e-6)):
        cfg = {**scenes._base(3, 30.0, 10e-3, 2.048e6, 31, noise_power=0),
               **scenes._grid(-0.5, 0.5, -0.5, 0.5, 0.05),
               "receivers": [scenes._orbit(550e3, 53, -0.9, -0.7), scenes._orbit(550e3, 53, 0.9, 0.5)],
               "emitters": [wf]}
        sc = ref.simulate(scenes.render(cfg))
        grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
        res = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc,
                                  b2.GeolocateOptions(detect=False))
        assert res.argmax_index == grid.index(12, 7), wf["waveform"]


def test_slab_sharding_bit_identical(b2, ref):
    """Per-point values do not depend on the partition: slabs reproduce the full
    surface bit for bit and the merged peak equals the single-GPU peak (§8e)."""
    from paper_2508_06672_b200.sharding import merge_argmax, slab_rows
    sc = load_scene(ref, "DESK_FOURJAM")
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    opts = b2.GeolocateOptions(detect=False, patch_peak=False)
    full = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    for world in (2, 3, 8):
        parts, peaks = [], []
        for r in range(world):
            r0, r1 = slab_rows(grid.lat.count, r, world)
            res = b2.geolocate_arrays(grid.slab(r0, r1), sc.states, sc.captures, sc.fs, sc.fc, opts)
            parts.append(res.accumulated.values)
            peaks.append((res.argmax_value, res.argmax_index))
        assert np.array_equal(np.concatenate(parts), full.accumulated.values)
        assert merge_argmax(peaks) == (full.argmax_value, full.argmax_index)


@pytest.mark.parametrize("normalize", [False, True])
def test_step_sharding_bit_identical(b2, ref, normalize):
    """The snapshot-sharded solve (dg_correlate_steps per rank, the all-to-all
    to latitude slabs emulated in process, dg_accumulate_peak per slab) gives
    the single-GPU accumulated surface bit for bit and the same exact peak."""
    import torch

    from paper_2508_06672_b200.sharding import merge_argmax, slab_rows, step_range
    sc = load_scene(ref, "DESK_FOURJAM")
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    opts = b2.GeolocateOptions(detect=False, patch_peak=False, normalize_per_snapshot=normalize)
    full = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    staged = b2.StagedSnapshots(sc.states, sc.captures, sc.fs, sc.fc)
    S, P, n_lon = sc.states.shape[0], grid.size(), grid.lon.count
    for world in (2, 3, 4):
        local, meds = [], []
        for r in range(world):
            s0, s1 = step_range(S, r, world)
            t = torch.empty((s1 - s0, P), dtype=torch.float64, device="cuda")
            m = torch.empty(max(s1 - s0, 1), dtype=torch.float64, device="cuda")
            if s1 > s0:
                b2.correlate_steps(grid, staged, s0, s1, t.data_ptr(),
                                   m.data_ptr() if normalize else None, opts)
            local.append(t)
            meds.append(m[: s1 - s0])
        medians = torch.cat(meds) if normalize else None
        parts, peaks = [], []
        for j in range(world):
            r0, r1 = slab_rows(grid.lat.count, j, world)
            slab_all = torch.cat([t[:, r0 * n_lon:r1 * n_lon] for t in local]).contiguous()
            res = b2.accumulate_peak(grid.slab(r0, r1), staged, slab_all.data_ptr(),
                                     medians.data_ptr() if normalize else None, opts)
            parts.append(res.accumulated.values)
            peaks.append((res.argmax_value, res.argmax_index))
        assert np.array_equal(np.concatenate(parts), full.accumulated.values)
        assert merge_argmax(peaks) == (full.argmax_value, full.argmax_index)


def test_lane_pipeline_bit_identical(b2, ref):
    """Steps overlapped on two streams (default) and serialised on one (the
    profiled mode) give the same surfaces bit for bit."""
    sc = load_scene(ref, "DESK_FOURJAM")
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    staged = b2.StagedSnapshots(sc.states, sc.captures, sc.fs, sc.fc)
    opts = b2.GeolocateOptions(detect=False)
    a = b2.geolocate_staged(grid, staged, opts, want_per_snapshot=True)
    b = b2.geolocate_staged(grid, staged, opts, want_per_snapshot=True, profile=True)
    for x, y in zip(a.per_snapshot, b.per_snapshot):
        assert np.array_equal(x.values, y.values)
    assert np.array_equal(a.accumulated.values, b.accumulated.values)
    assert (a.argmax_index, a.argmax_value) == (b.argmax_index, b.argmax_value)


def test_silent_captures(b2):
    grid = b2.build_candidate_grid(b2.LatLonBounds(-0.1, 0.1, -0.1, 0.1), 0.05)
    states = np.zeros((2, 2, 6))
    states[:, 0, :3] = [6378137.0 + 550e3, 0, 0]
    states[:, 1, :3] = [6378137.0 + 500e3, 3e5, 0]
    caps = np.zeros((2, 2, 512), np.complex128)
    res = b2.geolocate_arrays(grid, states, caps, 1e6, 1575.42e6)
    assert np.all(res.accumulated.values == 0.0)
    assert res.argmax_index == 0 and res.detections == []


def test_geolocate_errors(b2):
    grid = b2.build_candidate_grid(b2.LatLonBounds(-0.1, 0.1, -0.1, 0.1), 0.05)
    states = np.zeros((1, 2, 6))
    caps = np.zeros((1, 2, 64), np.complex128)
    with pytest.raises(ValueError, match="coincides with receiver"):
        # receivers at the Earth's centre never coincide; put one on a lattice node
        st = states.copy()
        st[0, 0, :3] = grid.points[3]
        st[0, 1, :3] = [7e6, 0, 0]
        b2.geolocate_arrays(grid, st, caps, 1e6, 1575.42e6)
    with pytest.raises(ValueError, match="need >= 2 receivers"):
        b2.geolocate_arrays(grid, states[:, :1], caps[:, :1], 1e6, 1575.42e6)
    with pytest.raises(ValueError, match="center_freq_hz <= 0"):
        b2.geolocate_arrays(grid, states, caps, 1e6, 0.0)
    with pytest.raises(ValueError, match="no snapshots"):
        b2.geolocate_snapshots([], grid)


@pytest.mark.parametrize("normalize", [False, True])
def test_chunked_accumulation_bit_identical(b2, ref, tune, normalize):
    """Runs over the per-snapshot surface budget are solved in snapshot chunks,
    each added to the running accumulated surface in snapshot order: the same
    additions in the same order, so the surface and the peak are bit-identical."""
    sc = load_scene(ref, "DESK_FOURJAM")
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    staged = b2.StagedSnapshots(sc.states, sc.captures, sc.fs, sc.fc)
    opts = b2.GeolocateOptions(k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius,
                               normalize_per_snapshot=normalize)
    whole = b2.geolocate_staged(grid, staged, opts, want_surface=True)
    tune(surface_budget_bytes=3 * grid.size() * 8)  # chunks of 3 snapshots
    chunked = b2.geolocate_staged(grid, staged, opts, want_surface=True)
    assert np.array_equal(chunked.accumulated.values, whole.accumulated.values)
    assert (chunked.argmax_index, chunked.argmax_value) == (whole.argmax_index, whole.argmax_value)
    assert [d.grid_index for d in chunked.detections] == [d.grid_index for d in whole.detections]


@pytest.mark.parametrize("normalize", [False, True])
def test_four_receivers_vs_reference(b2, ref, normalize):
    """Four receivers, six pairs per snapshot (correlate_snapshot_all_pairs,
    geolocate.hpp:79-94): per-receiver geometry shared by the pairs of a
    snapshot, pair sums in the reference's order; against the reference's own
    geolocate_snapshots, and the multi-GPU engine bit-identical to one GPU."""
    sc = load_scene(ref, "QUAD_RX")
    assert sc.n_rx == 4
    want = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                         backend="parallel", batch_size=4096, k_sigma=sc.k_sigma,
                         radius=sc.radius, normalize=normalize, per_snapshot=True)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    opts = b2.GeolocateOptions(k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius,
                               normalize_per_snapshot=normalize)
    res = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    per = np.stack([g.values for g in res.per_snapshot])
    assert rel_err(per, want["per_snapshot"]).max() <= REL_TOL
    assert res.argmax_index == int(np.argmax(want["accumulated"]))
    if not normalize:
        assert res.argmax_value == want["accumulated"][res.argmax_index]
    assert [d.grid_index for d in res.detections] == [d["grid_index"] for d in want["detections"]]
    eng = b2.Engine(devices=[0, 0, 0])
    mgrid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt, engine=eng)
    many = b2.geolocate_arrays(mgrid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    assert np.array_equal(many.accumulated.values, res.accumulated.values)


def test_fft_moments_match_direct_sums(b2, tune):
    """The two moment kernels on one C3-density scene (101 x 101 cells at 1 km, a
    chirp of the reference simulator's scene, 2 snapshots of 50,000 samples): FFT
    cross-correlations (k_mfft, default) and direct sums (k_moments, moment_fft = 0)
    give surfaces within 2e-5 of each other (each is within the 1e-4 contract of
    the reference; their FP32 roundings differ), the same exact argmax, and the
    FFT path really ran (moment_fft_flop)."""
    from paper_2508_06672_b200 import simulate as sim
    from paper_2508_06672_b200.geodesy import GeodeticCoord
    km = 0.0089932161
    rx = [sim.CircularOrbit(550e3, 53.0, -1.2, -1.1), sim.CircularOrbit(550e3, 53.0, 1.2, -0.7)]
    em = [sim.EmitterDef(GeodeticCoord(10 * km, -20 * km, 0.0), sim.ChirpSpec(2e6, 20e-6),
                         -10.0, 650e3)]
    sc = sim.Scenario(rx, em, 2, 1.0, 0.01, 5e6, 1575.42e6, 0.0, 11, 1.0)
    states, caps, _, _ = sim.simulate_arrays(sc)
    grid = b2.build_candidate_grid(b2.LatLonBounds(-50 * km, 50 * km, -50 * km, 50 * km), km)
    fft = b2.geolocate_arrays(grid, states, caps, 5e6, 1575.42e6, b2.GeolocateOptions())
    assert fft.stats["moment_fft_flop"] > 0 and fft.stats["direct_steps"] == 0
    tune(moment_fft=0)
    direct = b2.geolocate_arrays(grid, states, caps, 5e6, 1575.42e6, b2.GeolocateOptions())
    assert direct.stats["moment_fft_flop"] == 0
    assert rel_err(fft.accumulated.values, direct.accumulated.values).max() <= 2e-5
    assert fft.argmax_index == direct.argmax_index
    assert fft.argmax_value == direct.argmax_value
