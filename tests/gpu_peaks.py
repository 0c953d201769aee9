"""Measured CUDA-core peaks of this B200 (not collected by pytest)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_06672_b200._capi import lib  # noqa: E402

out = {}
for name in ("dg_fp32_peak_tflops", "dg_fp32x2_peak_tflops", "dg_fp64_peak_tflops"):
    v = C.c_double()
    getattr(lib, name)(0, C.byref(v))
    out[name] = v.value
print(json.dumps(out))
