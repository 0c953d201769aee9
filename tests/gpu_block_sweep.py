"""C3 solve time by forced block length (GPU, diagnostics): the planner's cost
model vs measurement. Prints one JSON line per setting."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

import paper_2508_06672_b200 as b2  # noqa: E402
from gpu_tau_sweep import c3_time  # noqa: E402
import paper_2508_06672_b200.simulate as sim  # noqa: E402
import scenes  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    eng = b2.default_engine(0)
    scene = scenes.config(name)
    states, caps, _, _ = sim.simulate_arrays(scenes.to_scenario(sim, scene))
    bounds = (scene["grid_lat_min_deg"], scene["grid_lat_max_deg"], scene["grid_lon_min_deg"],
              scene["grid_lon_max_deg"])
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), scene["grid_spacing_deg"])
    staged = b2.StagedSnapshots(states, caps, 5e6, 1575.42e6)
    for blk in (0, 512, 640, 768, 256):
        eng.set_tuning(moment_block=blk)
        ms, refined = c3_time(grid, staged)
        r = b2.geolocate_staged(grid, staged, b2.GeolocateOptions(detect=False), profile=True)
        eng.reset_tuning()
        print(json.dumps({"block": blk, "ms": ms, "refined": refined,
                          "moments_ms": r.stats["moments_ms"], "evaluate_ms": r.stats["evaluate_ms"],
                          "direct_steps": r.stats["direct_steps"]}), flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
