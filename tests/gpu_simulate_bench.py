"""C3 capture synthesis (50 snapshots x 4 emitters x 2 receivers x 50,000 samples):
simulate_staged on the GPU vs the reference's simulate_scenario (oracle/_ref, one
host thread as written), plus the worst sample difference between the two.

    python tests/gpu_simulate_bench.py   -> gpurun_out/simulate.json
Not collected by pytest.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import paper_2508_06672_b200.simulate as sim  # noqa: E402
import scenes  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402


def main():
    cfg = os.environ.get("DG_SIM_CONFIG", "C3")
    scene = scenes.config(cfg)
    sc = scenes.to_scenario(sim, scene)
    sim.simulate_staged(sc)  # warm-up
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = sim.simulate_staged(sc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del st
    t0 = time.perf_counter()
    want = RefLib().simulate(scenes.render(scene))
    t_ref = time.perf_counter() - t0
    _, caps, _, _ = sim.simulate_arrays(sc)
    out = {"config": cfg, "captures": list(caps.shape), "b200_s": float(np.median(ts)),
           "reference_s": t_ref, "speedup": t_ref / float(np.median(ts)),
           "max_abs_diff": float(np.abs(caps - want.captures).max()),
           "note": "b200: captures synthesised into HBM (staged run); reference: "
                   "simulate_scenario on one host thread"}
    print(json.dumps(out, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "simulate.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
