"""The one-process multi-GPU engine (dg_engine_create_multi).

The run is sharded into work units (dg_shard_plan: whole (snapshot, pair)
steps plus bucket-range parts of the remainder), exchanged to latitude slabs
by peer copies and accumulated per slab; every value must be bit-identical to
the one-GPU solve (the reference's worker-count invariance,
test_backend.cpp:135-146). On a one-GPU box the engine is built over the same
device several times: the sharding, exchange, two-stage peak and gather run
unchanged (peer copies become device-to-device copies).
"""
import numpy as np
import pytest

from test_gpu_parity import load_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines(b2):
    return {n: b2.Engine(devices=[0] * n) for n in (2, 3, 4)}


@pytest.mark.parametrize("name,normalize", [("DESK_FOURJAM", False), ("TRIPLE_RX", False),
                                            ("DESK_SAWTOOTH", True)])
@pytest.mark.parametrize("n_dev", [2, 3, 4])
def test_multi_engine_bit_identical(b2, ref, engines, name, normalize, n_dev):
    sc = load_scene(ref, name)
    opts = b2.GeolocateOptions(k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius,
                               normalize_per_snapshot=normalize)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    one = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc, opts,
                              want_per_snapshot=True)
    eng = engines[n_dev]
    assert eng.descriptor() == ("b200", "parallel-batched", n_dev)
    mgrid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt, engine=eng)
    many = b2.geolocate_arrays(mgrid, sc.states, sc.captures, sc.fs, sc.fc, opts,
                               want_per_snapshot=True)
    assert np.array_equal(many.accumulated.values, one.accumulated.values)
    for a, b in zip(many.per_snapshot, one.per_snapshot):
        assert np.array_equal(a.values, b.values)
    assert (many.argmax_index, many.argmax_value) == (one.argmax_index, one.argmax_value)
    assert [(d.grid_index, d.score) for d in many.detections] == \
        [(d.grid_index, d.score) for d in one.detections]
    assert many.stats["n_refined"] == one.stats["n_refined"]


def test_multi_engine_staged_and_device_surface(b2, ref, engines):
    import torch
    sc = load_scene(ref, "DESK_FOURJAM")
    eng = engines[3]
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt, engine=eng)
    staged = b2.StagedSnapshots(sc.states, sc.captures, sc.fs, sc.fc, engine=eng)
    dev = torch.empty(grid.size(), dtype=torch.float64, device="cuda")
    opts = b2.GeolocateOptions(k_sigma=sc.k_sigma, exclusion_radius_cells=sc.radius)
    res = b2.geolocate_staged(grid, staged, opts, want_surface=True,
                              accumulated_device=dev.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), res.accumulated.values)
    ref_grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    one = b2.geolocate_arrays(ref_grid, sc.states, sc.captures, sc.fs, sc.fc, opts)
    assert np.array_equal(one.accumulated.values, res.accumulated.values)
    assert (res.argmax_index, res.argmax_value) == (one.argmax_index, one.argmax_value)


def test_backend_workers(b2):
    be = b2.make_backend("b200", 1)
    assert be.descriptor().workers == 1
    n = b2.engine.device_count()
    assert b2.make_backend("b200", 0).descriptor().workers == n
