"""One C3 solve inside a cudaProfilerStart/Stop window (for ncu --profile-from-start off).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python tests/profile_solve.py
Not collected by pytest.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_06672_b200 as b2  # noqa: E402


def main():
    name = os.environ.get("DG_PROFILE_CONFIG", "C3")
    cfg = bench.WORKLOADS[name]
    # tuning for the profiled solve, e.g. DG_PROFILE_TUNING=moment_fft=1 (test harness only)
    tun = dict(kv.split("=") for kv in os.environ.get("DG_PROFILE_TUNING", "").split(",") if kv)
    if tun:
        b2.default_engine(0).set_tuning(**{k: int(v) for k, v in tun.items()})
    states, caps, bounds, spacing = bench.make_inputs(name)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing)
    staged = b2.StagedSnapshots(states, caps, cfg["fs"], bench.FC)
    opts = b2.GeolocateOptions()
    b2.geolocate_staged(grid, staged, opts)  # warm-up (pool, module load)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    res = b2.geolocate_staged(grid, staged, opts)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("argmax", res.argmax_index, res.argmax_value, res.stats)


if __name__ == "__main__":
    main()
