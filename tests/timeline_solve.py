"""Kernel timeline of one solve (CUPTI through torch.profiler): every kernel and copy
with its stream, start and duration, and the idle gaps of the busiest stream.

    python tests/timeline_solve.py [C3] > gpurun_out/timeline_c3.txt
Not collected by pytest.
"""
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
    # the bench's solve: detection on, surface kept on the device
    opts = b2.GeolocateOptions(k_sigma=5.0, exclusion_radius_cells=5, detect=True)
    acc = torch.empty(grid.size(), dtype=torch.float64, device="cuda")

    def solve():
        b2.geolocate_staged(grid, staged, opts, want_surface=False,
                            accumulated_device=acc.data_ptr())

    for _ in range(2):
        solve()  # warm-up
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        solve()
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        ev.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name))
    ev.sort()
    t0 = ev[0][0]
    t_end = max(e[1] for e in ev)
    print(f"# {name}: {len(ev)} device events, span {(t_end - t0) / 1e3:.3f} ms")
    by_stream = {}
    for s, e, st, n in ev:
        by_stream.setdefault(st, []).append((s, e, n))
    for st, lst in by_stream.items():
        busy = sum(e - s for s, e, _ in lst)
        print(f"# stream {st}: {len(lst)} events, busy {busy / 1e3:.3f} ms")
    # union of busy time over all streams and the gaps where nothing runs
    cur_s, cur_e, gaps = None, None, []
    for s, e, _, n in ev:
        if cur_e is None:
            cur_s, cur_e = s, e
        elif s > cur_e:
            gaps.append((cur_e, s, n))
            cur_e = e
        else:
            cur_e = max(cur_e, e)
    idle = sum(b - a for a, b, _ in gaps)
    print(f"# device idle (no stream busy): {idle / 1e3:.3f} ms in {len(gaps)} gaps")
    for a, b, n in sorted(gaps, key=lambda g: g[0] - g[1])[:25]:
        print(f"#   gap {(b - a):9.1f} us at {(a - t0) / 1e3:8.3f} ms before {n[:60]}")
    # per-name totals
    tot = {}
    for s, e, st, n in ev:
        k = n.split("(")[0][:60]
        tot[k] = tot.get(k, 0) + (e - s)
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:30]:
        print(f"# total {v / 1e3:9.3f} ms  {k}")
    for s, e, st, n in ev:
        print(f"{(s - t0) / 1e3:10.3f} {(e - s):9.1f} {st:4d} {n[:90]}")


if __name__ == "__main__":
    main()
