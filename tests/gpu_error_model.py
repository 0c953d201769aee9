"""Error model of the block-moment correlator at C3 scale (not collected by pytest).

One C3 snapshot (4,004,001 candidates x 50,000 samples) is correlated twice on
the GPU: the normal path, and with DG_REFINE_TAU=1e30 so every element is
re-evaluated by the exact FP64 reference-order kernel. The relative error of
the fast path is binned by S / sqrt(sum |z|^2) (the quantity the refinement
threshold tau is expressed in), which is what DESIGN.md's choice of tau rests on.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_06672_b200 as b2  # noqa: E402
from paper_2508_06672_b200 import scene  # noqa: E402


def zsq_by_d(y1, y2, ds):
    """sum_k |y1[k]|^2 |y2[k+d]|^2 over the overlap, for every d in ds (FFT, FP64)."""
    n = len(y1)
    a, b = np.abs(y1) ** 2, np.abs(y2) ** 2
    m = 1 << int(np.ceil(np.log2(2 * n)))
    c = np.fft.irfft(np.conj(np.fft.rfft(a, m)) * np.fft.rfft(b, m), m)  # c[d] = sum a[k] b[k+d]
    return c[np.asarray(ds) % m]


def run(snr, kind_seed, tau_env=None):
    S, N, fs, fc = 1, 50_000, 5e6, 1575.42e6
    em = scene.FOUR_EMITTERS if snr < 0 else [("tone", 0.0, 0.0, {})]
    states, caps = scene.synthesize(S, N, fs, em, snr, seed=kind_seed)
    h = 1000 * scene.KM_DEG
    grid = b2.build_candidate_grid(b2.LatLonBounds(-h, h, -h, h), scene.KM_DEG)
    snap = b2.Snapshot(0.0, states[0], [b2.BasebandCapture(caps[0, r], fs, 0.0, fc) for r in range(2)])
    be = b2.make_backend("b200")
    os.environ.pop("DG_REFINE_TAU", None)
    if tau_env is not None:  # a candidate refinement threshold instead of the default
        os.environ["DG_REFINE_TAU"] = str(tau_env)
    fast = b2.correlate_snapshot(grid, snap, (0, 1), be).values
    os.environ["DG_REFINE_TAU"] = "1e30"
    exact = b2.correlate_snapshot(grid, snap, (0, 1), be).values
    os.environ.pop("DG_REFINE_TAU", None)
    off = b2.predict_offsets(grid, states[0, 0], states[0, 1], fs, b2.wavelength_m(fc))
    norm = np.sqrt(zsq_by_d(caps[0, 0], caps[0, 1], off["tdoa_samples"]))
    ratio = exact / norm
    rel = np.abs(fast - exact) / np.maximum(np.abs(exact), 1e-300)
    absn = np.abs(fast - exact) / norm
    edges = [0, 1e-3, 2e-3, 5e-3, 1e-2, 2e-2, 5e-2, 0.1, 0.3, 1, 3, 1e9]
    out = {"snr_db": snr, "tau": tau_env, "n_refined_like": int(np.sum(fast == exact)),
           "points": int(grid.size()), "max_rel": float(rel.max()),
           "max_abs_over_norm": float(absn.max()),
           "p999_abs_over_norm": float(np.quantile(absn, 0.999)),
           "std_abs_over_norm": float(np.std((fast - exact) / norm)), "bins": []}
    for lo, hi in zip(edges[:-1], edges[1:]):
        m = (ratio >= lo) & (ratio < hi)
        if m.any():
            out["bins"].append({"S_over_norm": [lo, hi], "n": int(m.sum()),
                                "max_rel": float(rel[m].max()), "max_abs_over_norm": float(absn[m].max())})
    return out


if __name__ == "__main__":
    tau = float(sys.argv[1]) if len(sys.argv) > 1 else None  # default: the engine's
    res = [run(-20.0, 3, tau), run(0.0, 11, tau), run(20.0, 5, tau)]
    print(json.dumps(res, indent=1))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    name = "error_model.json" if tau is None else f"error_model_tau{tau:g}.json"
    with open(os.path.join(ROOT, "gpurun_out", name), "w") as f:
        json.dump(res, f, indent=1)
