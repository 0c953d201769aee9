"""GPU: the reference's own C++ driver with the B200 engine plugged in.

oracle/_ref/drop_in is tests/cpp/drop_in.cpp compiled against the unmodified
reference headers and linked to libb200geo.so through the header-only shim
include/b200geo/digeo_plugin.hpp (b200::B200Backend is a
digeo::CorrelationBackend; b200::geolocate_snapshots has the signature of
digeo::geolocate_snapshots, geolocate.hpp:127-146)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "drop_in")


def test_reference_driver_with_b200_backend(tmp_path):
    import scenes
    assert os.path.exists(BIN), "oracle/_ref/drop_in missing: run __graft_entry__.build()"
    cfg = tmp_path / "desk_fourjam.cfg"
    cfg.write_text(scenes.render(scenes.DESK_FOURJAM))
    out = subprocess.run([BIN, str(cfg)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("[PASS]") >= 9 and "[FAIL]" not in out.stdout
