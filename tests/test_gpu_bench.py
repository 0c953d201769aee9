"""GPU: bench.py's multi-GPU launches on a one-GPU box. `--gpus 2` without
torchrun re-runs itself as two ranks (here over gloo, both on GPU 0) and
`--in-process` drives two device slots from one process through the multi-GPU
engine; both print one line with n_gpus = 2 and the one-GPU line's peak."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

COMMON = ["--config", "C2", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-plugin"]


def _line(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_multi_gpu_lines():
    one = _line(COMMON)
    spawned = _line(["--gpus", "2", "--dist-backend", "gloo"] + COMMON)
    inproc = _line(["--gpus", "2", "--in-process", "--device-list", "0,0"] + COMMON)
    for line in (spawned, inproc):
        assert line["n_gpus"] == 2
        assert line["argmax"] == one["argmax"]
        assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert one["n_gpus"] == 1
