"""Ad-hoc: which TDOA values / block lengths does the block-moment path get wrong? (not pytest)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_06672_b200 as b2  # noqa: E402
from oracle.bindings import PAIR_OFFSETS_DTYPE, RefLib  # noqa: E402

ref = RefLib()
rng = np.random.default_rng(1)
n, fs = 4000, 5e6
y1 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
y2 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
s = b2.make_backend("b200").stage(b2.BasebandCapture(y1, fs), b2.BasebandCapture(y2, fs))
os.environ["DG_CORRELATOR_MOMENTS"] = "2"
for B in (64, 128, 256):
    os.environ["DG_MOMENT_B"] = str(B)
    for ds in ([0], [1], [-1], [2], [-2], [5], [-7], [300], [-301], list(range(-40, 40)),
               list(range(-3000, 3000, 7))):
        off = np.zeros(len(ds) * 20, PAIR_OFFSETS_DTYPE)
        off["tdoa_samples"] = np.repeat(ds, 20)
        off["fdoa_hz"] = np.tile(np.linspace(-2000, 2000, 20), len(ds))
        want = ref.correlate_batch(y1, y2, fs, off, "serial", 1, None)
        got = s.correlate_batch(off)
        rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
        bad = np.unique(off["tdoa_samples"][rel > 1e-4])
        print(B, ds[:3], len(ds), "max rel %.2e" % rel.max(), "bad d:", bad[:12], len(bad))
