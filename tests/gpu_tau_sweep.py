"""Refinement threshold sweep (GPU, diagnostics): worst error of the moment-path
stress scenes (tests/test_gpu_error_model.py) and the C3 solve time / refined
count at each tau. Writes the table to argv[1] (JSON)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_06672_b200 as b2  # noqa: E402
import paper_2508_06672_b200.simulate as sim  # noqa: E402
import scenes  # noqa: E402
import test_gpu_error_model as em  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402

MOMENT_CASES = ["tone+40_B640", "tone+40_B512", "tone+40_B768", "tone+40_1km", "chirp+40_B768",
                "chirp+40", "four-20_1km"]


def c3_time(grid, staged, reps=5):
    stream = torch.cuda.Stream()
    opts = b2.GeolocateOptions(detect=True)
    dev = torch.empty(grid.size(), dtype=torch.float64, device="cuda")
    for _ in range(3):
        b2.geolocate_staged(grid, staged, opts, want_surface=False,
                            accumulated_device=dev.data_ptr(), stream=stream.cuda_stream)
    ms, refined = [], 0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r = b2.geolocate_staged(grid, staged, opts, want_surface=False,
                                accumulated_device=dev.data_ptr(), stream=stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        refined = r.stats["n_refined"]
    return float(np.median(ms)), int(refined)


def main():
    ref = RefLib()
    eng = b2.default_engine(0)
    scene = scenes.config("C3")
    states, caps, _, _ = sim.simulate_arrays(scenes.to_scenario(sim, scene))
    bounds = (scene["grid_lat_min_deg"], scene["grid_lat_max_deg"], scene["grid_lon_min_deg"],
              scene["grid_lon_max_deg"])
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), scene["grid_spacing_deg"])
    staged = b2.StagedSnapshots(states, caps, 5e6, 1575.42e6)
    out = []
    taus = [float(t) for t in (sys.argv[2].split(",") if len(sys.argv) > 2 else
                               ["0.015", "0.02", "0.025", "0.03"])]
    key = sys.argv[3] if len(sys.argv) > 3 else "refine_tau"  # or noise_refine_tau
    for tau in taus:
        row = {key: tau}
        for name in MOMENT_CASES:
            kw, tuning = em.CASES[name]
            em.CASES[name] = (kw, {**tuning, "correlator": "moments", key: tau,
                                   "allow_weaker_refine": 1})
            r = em.run_case(b2, ref, name)
            em.CASES[name] = (kw, tuning)
            row[name] = r["max_rel"]
        eng.set_tuning(**{key: tau, "allow_weaker_refine": 1})
        row["c3_ms"], row["c3_refined"] = c3_time(grid, staged)
        eng.reset_tuning()
        print(json.dumps(row), flush=True)
        out.append(row)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
