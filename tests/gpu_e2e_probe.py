"""Ad-hoc: where the end-to-end (host captures in, surface out) time goes (not pytest)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_06672_b200 as b2  # noqa: E402

cfg = bench.WORKLOADS["C3"]
states, caps, bounds, spacing = bench.make_inputs("C3")
grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing)
pinned = torch.empty(caps.shape, dtype=torch.complex128, pin_memory=True).numpy()
pinned[...] = caps
opts = b2.GeolocateOptions()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = b2.StagedSnapshots(states, pinned, cfg["fs"], bench.FC)
    t1 = time.perf_counter()
    r = b2.geolocate_staged(grid, st, opts, want_surface=True)
    t2 = time.perf_counter()
    del st
    t3 = time.perf_counter()
    r2 = b2.geolocate_arrays(grid, states, pinned, cfg["fs"], bench.FC, opts, want_surface=True,
                             want_per_snapshot=False)
    t4 = time.perf_counter()
    print(f"stage {1e3*(t1-t0):.1f} ms, solve+d2h {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms,"
          f" geolocate_arrays {1e3*(t4-t3):.1f} ms", flush=True)
