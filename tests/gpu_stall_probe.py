"""Diagnose intermittent slow solves in the bench loop (C5): the bench's exact loop
(warm-ups, then L2 flush + events + solve on one stream) under CUPTI, reporting the
slow steps, the longest CUDA runtime calls and the GPU idle gaps inside them.
    python tests/gpu_stall_probe.py [C5]     Not collected by pytest."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2508_06672_b200 as b2  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    cfg = bench.WORKLOADS[name]
    states, caps, bounds, spacing = bench.make_inputs(name)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing)
    staged = b2.StagedSnapshots(states, caps, cfg["fs"], bench.FC)
    opts = b2.GeolocateOptions(k_sigma=5.0, exclusion_radius_cells=5, detect=True)
    stream = torch.cuda.Stream()
    acc = torch.empty(grid.size(), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def solve():
        b2.geolocate_staged(grid, staged, opts, want_surface=False,
                            accumulated_device=acc.data_ptr(), stream=stream.cuda_stream)
    for _ in range(3):
        solve()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(6)]
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for k in range(6):
            with torch.cuda.stream(stream):
                flush.zero_()
            ev[k][0].record(stream)
            with torch.profiler.record_function(f"solve{k}"):
                solve()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    print("step_ms", [round(a.elapsed_time(b), 2) for a, b in ev])
    os.makedirs("gpurun_out", exist_ok=True)
    prof.export_chrome_trace("gpurun_out/stall_trace.json")
    tr = json.load(open("gpurun_out/stall_trace.json"))["traceEvents"]
    rt = sorted([e for e in tr if e.get("cat") == "cuda_runtime" and "dur" in e],
                key=lambda e: -e["dur"])
    sol = {e["name"]: (e["ts"], e["ts"] + e["dur"]) for e in tr
           if e.get("name", "").startswith("solve") and "dur" in e}
    t0 = min(v[0] for v in sol.values())
    print("solves (host ms):", {k: round((v[1] - v[0]) / 1e3, 2) for k, v in sorted(sol.items())})
    print("longest runtime calls:")
    for e in rt[:12]:
        print(f"  {(e['ts'] - t0) / 1e3:9.2f} ms  {e['dur'] / 1e3:8.2f} ms  {e['name']}")
    ks = sorted([e for e in tr if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")
                 and "dur" in e], key=lambda e: e["ts"])
    gaps, end = [], None
    for e in ks:
        if end is not None and e["ts"] - end > 2000:
            gaps.append(((e["ts"] - end) / 1e3, (end - t0) / 1e3, e["name"][:60]))
        end = max(end or 0, e["ts"] + e["dur"])
    print("GPU idle gaps > 2 ms:", gaps[:10])
    slow = [e for e in ks if e["dur"] > 20000]
    print("device ops > 20 ms:", [((e["ts"] - t0) / 1e3, e["dur"] / 1e3, e["name"][:50]) for e in slow][:10])


if __name__ == "__main__":
    main()
