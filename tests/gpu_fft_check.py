"""FFT block moments (tuning moment_fft = 1) against the direct sums: the error-model
scenes vs the reference, and C3 solve time / argmax / refinement count both ways.

    python tests/gpu_fft_check.py [out.json]
Not collected by pytest.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_06672_b200 as b2  # noqa: E402
import test_gpu_error_model as em  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402


def c3_time(fft, reps=3, kappa=0.0):
    cfg = bench.WORKLOADS["C3"]
    states, caps, bounds, spacing = bench.make_inputs("C3")
    eng = b2.default_engine(0)
    eng.set_tuning(moment_fft=fft, fft_refine_kappa=kappa, allow_weaker_refine=1)
    try:
        grid = b2.build_candidate_grid(b2.LatLonBounds(*bounds), spacing)
        staged = b2.StagedSnapshots(states, caps, cfg["fs"], bench.FC)
        opts = b2.GeolocateOptions()
        acc = torch.empty(grid.size(), dtype=torch.float64, device="cuda")
        res = None
        ms = []
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = b2.geolocate_staged(grid, staged, opts, want_surface=False,
                                      accumulated_device=acc.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        prof = b2.geolocate_staged(grid, staged, opts, want_surface=False,
                                   accumulated_device=acc.data_ptr(), profile=True).stats
        return dict(fft=fft, kappa=kappa, ms=ms[1:], argmax=[res.argmax_index, res.argmax_value],
                    refined=int(res.stats["n_refined"]), acc=acc.clone(),
                    moments_ms=prof.get("moments_ms"), evaluate_ms=prof.get("evaluate_ms"))
    finally:
        eng.reset_tuning()


def main():
    kappas = [float(k) for k in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4"])]
    out = []
    a = c3_time(0)
    a.pop("acc")
    print(json.dumps(a), flush=True)
    out.append(a)
    ref = RefLib()
    base = dict(em.CASES)
    for kappa in kappas:
        b = c3_time(1, kappa=kappa)
        b.pop("acc")
        print(json.dumps(b), flush=True)
        out.append(b)
        rows = []
        for name in sorted(base):
            kw, tuning = base[name]
            em.CASES[name] = (kw, dict(tuning, moment_fft=1, fft_refine_kappa=kappa,
                                       allow_weaker_refine=1))
            r = em.run_case(b2, ref, name)
            r["kappa"] = kappa
            rows.append(r)
            out.append(r)
        w = max(rows, key=lambda r: r["max_rel"])
        print(json.dumps(dict(kappa=kappa, worst=w["max_rel"], scene=w["scene"],
                              refined={r["scene"]: r["refined"] for r in rows})), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
