"""GPU timeline of one solve from CUPTI (torch.profiler): span, busy union, idle gaps,
and per-kernel concurrency -- where a solve's time goes beyond its two big kernels.

    python tests/gpu_timeline.py [C3] [e2e]  -> gpurun_out/timeline.json + printed summary
Not collected by pytest.
"""
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
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    cfg = bench.WORKLOADS[name]
    states, caps, bounds, spacing = bench.make_inputs(name)
    grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing)
    staged = b2.StagedSnapshots(states, caps, cfg["fs"], bench.FC)
    opts = b2.GeolocateOptions()
    e2e = len(sys.argv) > 2 and sys.argv[2] == "e2e"
    if e2e:  # the bench's e2e call: pinned host captures in, pinned surface out
        pinned = torch.empty(caps.shape, dtype=torch.complex128, pin_memory=True).numpy()
        pinned[...] = caps
        surf = torch.empty(grid.size(), dtype=torch.float64, pin_memory=True).numpy()

        def solve():
            b2.geolocate_arrays(grid, states, pinned, cfg["fs"], bench.FC, opts,
                                want_surface=True, want_per_snapshot=False, out=surf)
    else:
        def solve():
            b2.geolocate_staged(grid, staged, opts)
    for _ in range(5):  # steady state (stream-ordered pool grown)
        solve()
    torch.cuda.synchronize()
    n_prof = int(os.environ.get("DG_TL_SOLVES", "1"))  # >1: look for sporadic stalls
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(n_prof):
            solve()
        torch.cuda.synchronize()
    os.makedirs("gpurun_out", exist_ok=True)
    trace = "gpurun_out/timeline_trace.json"
    prof.export_chrome_trace(trace)
    ev = json.load(open(trace))["traceEvents"]
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    t1 = max(e["ts"] + e["dur"] for e in ks)
    busy, gaps, cur_s, cur_e, prev = 0.0, [], None, None, None
    for e in ks:
        s, d = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
                gaps.append((s - cur_e, cur_e - t0, prev, e["name"]))
            cur_s, cur_e = s, d
        else:
            cur_e = max(cur_e, d)
        prev = e["name"] if d >= (cur_e or 0) else prev
    busy += cur_e - cur_s
    per = {}
    for e in ks:
        k = e["name"].split("(")[0][-48:]
        p = per.setdefault(k, [0, 0.0, e["args"].get("stream")])
        p[0] += 1
        p[1] += e["dur"]
    gaps.sort(reverse=True)
    out = {"config": name, "span_us": t1 - t0, "busy_us": busy, "idle_us": t1 - t0 - busy,
           "gaps_top": [{"us": g, "at_us": a, "after": p[-60:] if p else None, "before": n[-60:]}
                        for g, a, p, n in gaps[:25]],
           "kernels": {k: {"launches": v[0], "us": v[1], "stream": v[2]}
                       for k, v in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    # where the big kernels sit: first/last start of each, relative to t0
    for key in ("k_moments", "k_evaluate_tc", "k_refine", "k_rerank", "k_geometry"):
        st = [e["ts"] - t0 for e in ks if key in e["name"]]
        en = [e["ts"] + e["dur"] - t0 for e in ks if key in e["name"]]
        if st:
            out.setdefault("phases", {})[key] = [min(st), max(en)]
    json.dump(out, open("gpurun_out/timeline.json", "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("span_us", "busy_us", "idle_us", "phases")}, indent=1))
    for g in out["gaps_top"][:12]:
        print(g)
    for k, v in list(out["kernels"].items())[:16]:
        print(f"{k:50s} {v['launches']:4d} {v['us']:10.1f} stream {v['stream']}")


if __name__ == "__main__":
    main()
