"""Diagnostics (GPU): the worst cells of an error-model scene
(tests/test_gpu_error_model.py) with their offsets, for both correlators."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import paper_2508_06672_b200 as b2  # noqa: E402
import scenes  # noqa: E402
import test_gpu_error_model as em  # noqa: E402
from oracle.bindings import RefLib  # noqa: E402


def main():
    ref = RefLib()
    name = sys.argv[1] if len(sys.argv) > 1 else "chirp+40"
    kw, case_tuning = em.CASES[name]
    sc = ref.simulate(scenes.render(em._scene(**kw)))
    want = ref.geolocate(sc.states, sc.captures, sc.fs, sc.fc, sc.bounds, sc.spacing, sc.alt,
                         backend="parallel", batch_size=4096)["accumulated"]
    grid = b2.build_candidate_grid(b2.LatLonBounds(*sc.bounds), sc.spacing, sc.alt)
    off = b2.predict_offsets(grid, sc.states[0, 0], sc.states[0, 1], sc.fs, ref.wavelength(sc.fc))
    eng = b2.default_engine(0)
    em_pt = kw.get("kind")
    ipk = int(np.argmax(want))
    d_true = int(off["tdoa_samples"][ipk])
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["direct", "moments"]
    for mode in modes:
        for tau in (0.0, 0.04):
            t = dict(case_tuning) if mode == "case" else dict(correlator=mode)
            if tau:
                t.update(refine_tau=tau, direct_refine_tau=tau)
            eng.set_tuning(**t)
            res = b2.geolocate_arrays(grid, sc.states, sc.captures, sc.fs, sc.fc,
                                      b2.GeolocateOptions(detect=False, patch_peak=False),
                                      want_per_snapshot=False)
            eng.reset_tuning()
            got = res.accumulated.values
            e = np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), 1e-300)
            worst = np.argsort(e)[::-1][:8]
            print(json.dumps({"scene": name, "kind": em_pt, "mode": mode, "tau": tau,
                              "max_rel": float(e.max()), "refined": res.stats["n_refined"],
                              "direct_steps": res.stats["direct_steps"], "peak": float(want.max()),
                              "d_true": d_true}), flush=True)
            for p in worst:
                print("   rel %.2e  S %.6e  got %.6e  S/peak %.2e  d-d_true %5d  fdoa %9.1f" % (
                    e[p], want[p], got[p], want[p] / want.max(),
                    int(off["tdoa_samples"][p]) - d_true, off["fdoa_hz"][p]), flush=True)


if __name__ == "__main__":
    main()
