"""CPU: the C-ABI library loads, exports every symbol include/b200geo.h declares,
and the host-side mirror keeps the reference's validation and messages
(backend.hpp:77-93,311-317; geodesy.hpp:64-79,126-138; geometry.hpp:36-39)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "b200geo.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2508_06672_b200 import _capi
    syms = declared_symbols()
    assert len(syms) >= 24
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dg_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(_capi.EXPORTS) == syms
    assert _capi.lib.dg_abi_version() == 7


def test_library_is_sm100a():
    from paper_2508_06672_b200 import _capi
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "FFMA2" in sass and "UBLKCP" in sass  # packed FP32 MAC + TMA bulk staging


def test_plan_batches_mirror(ref):
    from paper_2508_06672_b200 import backend
    assert backend.plan_batches(1_000_000, 8).batch_count() == 125_000
    assert backend.plan_batches(100, 1000).batch_count() == 1
    for b in (1, 3, 8, 100, 1001):
        plan = backend.plan_batches(1001, b)
        ranges = [plan.batch_range(i) for i in range(plan.batch_count())]
        assert ranges[0][0] == 0 and ranges[-1][1] == 1001
        assert all(r[1] - r[0] <= b and r[1] > r[0] for r in ranges)
        assert all(a[1] == b_[0] for a, b_ in zip(ranges, ranges[1:]))
        assert plan.batch_count() == ref.plan_batch_count(1001, b)
    with pytest.raises(ValueError, match="batch working set"):
        backend.plan_batches(1000, 1 << 40, 1 << 20, 0)
    with pytest.raises(ValueError, match="captures"):
        backend.plan_batches(1000, 8, 1 << 10, 1 << 20)
    with pytest.raises(ValueError):
        backend.plan_batches(0, 8)
    with pytest.raises(ValueError):
        backend.plan_batches(10, 0)


def test_plan_batches_messages_match_reference(ref):
    from oracle.bindings import ReferenceError_
    from paper_2508_06672_b200 import backend
    for args in ((1000, 1 << 40, 1 << 20, 0), (1000, 8, 1 << 10, 1 << 20)):
        with pytest.raises(ReferenceError_) as r:
            ref.plan_batch_count(*args)
        with pytest.raises(ValueError) as m:
            backend.plan_batches(*args)
        assert str(m.value) == str(r.value)


def test_geodetic_validation_mirror():
    from paper_2508_06672_b200 import GeodeticCoord, LatLonBounds
    with pytest.raises(ValueError, match="lat_deg out of"):
        GeodeticCoord(91.0, 0.0, 0.0).validate()
    with pytest.raises(ValueError, match="lon_deg out of"):
        GeodeticCoord(0.0, 180.0, 0.0).validate()
    with pytest.raises(ValueError, match="alt_m not finite"):
        GeodeticCoord(0.0, 0.0, float("nan")).validate()
    with pytest.raises(ValueError, match="max < min"):
        LatLonBounds(1.0, 0.0, 0.0, 1.0).validate()
    LatLonBounds(0.0, 1.0, 0.0, 200.0).validate()  # lon_max unchecked, as in the reference


def test_registry_and_wavelength():
    from paper_2508_06672_b200 import make_backend, wavelength_m
    with pytest.raises(ValueError, match="unknown backend 'gpu'"):
        make_backend("gpu")  # test_backend.cpp:181 requires "gpu" to stay rejected
    with pytest.raises(ValueError, match="center_freq_hz <= 0"):
        wavelength_m(0.0)
    assert wavelength_m(1575.42e6) == pytest.approx(0.190293672798365, rel=1e-12)


def test_pair_offsets_layout():
    from paper_2508_06672_b200 import PAIR_OFFSETS_DTYPE, _capi
    assert PAIR_OFFSETS_DTYPE.itemsize == C.sizeof(_capi.dg_pair_offsets) == 16
    assert C.sizeof(_capi.dg_state) == 48
    assert C.sizeof(_capi.dg_emitter_estimate) == 48
    a = np.zeros(2, PAIR_OFFSETS_DTYPE)
    assert a.dtype.fields["fdoa_hz"][1] == 8



def test_tuning_validation():
    """dg_engine_set_tuning rejects unknown modes / block lengths / moment counts and a
    refinement threshold below the default unless explicitly allowed (no CUDA call:
    the engine struct is never created, a null engine is rejected first)."""
    from paper_2508_06672_b200 import _capi
    t = _capi.dg_tuning()
    _capi.lib.dg_tuning_default(C.byref(t))
    assert t.correlator == _capi.DG_CORRELATOR_AUTO and t.evaluate_tensor == 1
    assert _capi.lib.dg_engine_set_tuning(None, C.byref(t)) == _capi.DG_EINVAL
