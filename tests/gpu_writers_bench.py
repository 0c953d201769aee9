"""Surface writers at C3 size (2001 x 2001 cells), device formatter vs the
reference's host writers (oracle/_ref), same values, same files.

    python tests/gpu_writers_bench.py   -> gpurun_out/writers.json
Not collected by pytest. Wall-clock per call (file writes into /tmp included),
median of 3; the device values are resident (the accumulated surface of a solve).
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_06672_b200 as b2  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def main():
    from paper_2508_06672_b200 import scene
    h = 1000 * scene.KM_DEG
    grid = b2.build_candidate_grid(b2.LatLonBounds(-h, h, -h, h), scene.KM_DEG)
    rng = np.random.default_rng(1)
    v = rng.gamma(4.0, 2e3, grid.size())
    dv = torch.from_numpy(v).cuda()
    cg = b2.CorrelationGrid(grid, dv)
    ref = RefLib()
    axes = (grid.lat.start_deg, grid.lat.step_deg, grid.lat.count, grid.lon.start_deg,
            grid.lon.step_deg, grid.lon.count)
    out = {"cells": grid.size()}
    with tempfile.TemporaryDirectory() as d:
        p = lambda n: os.path.join(d, n)  # noqa: E731
        cases = {
            "csv": (lambda: b2.write_grid(cg, p("b.csv"), b2.GridFileFormat.csv),
                    lambda: ref.write_grid(p("r.csv"), axes, 0.0, v, True), "b.csv", "r.csv"),
            "dggr": (lambda: b2.write_grid(cg, p("b.bin"), b2.GridFileFormat.binary),
                     lambda: ref.write_grid(p("r.bin"), axes, 0.0, v, False), "b.bin", "r.bin"),
            "p5": (lambda: b2.render_heatmap(cg, p("b.pgm")),
                   lambda: ref.render_heatmap(p("r.pgm"), axes, 0.0, v), "b.pgm", "r.pgm"),
        }
        for name, (mine, theirs, fb, fr) in cases.items():
            mine()  # warm-up (pinned buffers, module load)
            tb = timed(mine)
            tr = timed(theirs, reps=1)
            same = open(p(fb), "rb").read() == open(p(fr), "rb").read()
            out[name] = {"b200_s": tb, "reference_s": tr, "bytes": os.path.getsize(p(fb)),
                         "identical": same, "speedup": tr / tb}
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "writers.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
