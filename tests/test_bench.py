"""CPU: bench.py's reference arm end to end (the reference's own simulate_scenario
and geolocate_snapshots on this host, a bounded sample) prints one JSON line with
the contract's keys; the b200 arm's line is checked by the driver on a B200."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--sample-km", "250", "--sample-snapshots", "2"],
        capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["value"] > 0 and line["unit"] == "correlations/s"
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_plugin_workload_matches_reference():
    """bench.py regenerates the reference's BenchWorkload (bench.hpp:65-88) bit for bit."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from oracle.bindings import RefLib
    y1r, y2r, offr, _ = RefLib().build_workload(30_000, 4096, 5e6, 1)
    y1, y2, off = bench.build_workload(30_000, 4096, 5e6, 1)
    assert np.array_equal(y1, y1r) and np.array_equal(y2, y2r) and np.array_equal(off, offr)
    y1r, _, offr, _ = RefLib().build_workload(10_000, 1000, 2e6, 77)
    y1, _, off = bench.build_workload(10_000, 1000, 2e6, 77)
    assert np.array_equal(y1, y1r) and np.array_equal(off, offr)
