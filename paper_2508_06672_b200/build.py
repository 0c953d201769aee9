"""Build recipe for libb200geo.so (in-tree, sm_100a only).

    python paper_2508_06672_b200/build.py   (a file path: importing the package needs the .so)

Kernels: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo.
C ABI layer: g++ -std=c++20 -ffp-contract=off (host math must not contract,
so the per-row/column lattice tables match libm-based lla_to_ecef exactly).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libb200geo.so")
BUILD = os.path.join(ROOT, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> str:
    nvcc = shutil.which("nvcc")
    if nvcc:
        return os.path.dirname(os.path.dirname(os.path.realpath(nvcc)))
    return os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cpp", ".cuh", ".h"))] + [
        os.path.join(ROOT, "include", "b200geo.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
    objs = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        if f.endswith(".cu"):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *inc,
                   "-c", src, "-o", obj]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
        elif f.endswith(".cpp"):
            cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wextra",
                   *inc, "-I" + os.path.join(cuda, "include"), "-c", src, "-o", obj]
        else:
            continue
        _run(cmd)
        objs.append(obj)
    tmp = OUT + ".tmp"
    _run([nvcc, "-shared", *ARCH, "-Xlinker", "-soname=libb200geo.so", "-o", tmp, *objs])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
