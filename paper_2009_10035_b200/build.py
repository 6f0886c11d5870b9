"""Build the in-tree CUDA library ``lib/libf2v_b200.so`` for sm_100a.

    python paper_2009_10035_b200/build.py [--verbose] [--force]

nvcc compiles the kernels (csrc/*.cu) and the host C++ (csrc/*.cpp) into one
shared object with the CUDA runtime linked statically, so the .so that
travels to the GPU box needs only the driver.  ``--fmad=false`` keeps the
reference's separate multiply/add roundings.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libf2v_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-O3", "-Xcompiler", "-pthread", "--expt-relaxed-constexpr"]
if os.environ.get("F2V_NVCC_EXTRA"):  # experiments: e.g. "-DF2V_EPOCH_MINB=3"
    NVCC_FLAGS += os.environ["F2V_NVCC_EXTRA"].split()
if os.environ.get("F2V_DEVICE_CHECKS"):  # debug build: device-side bounds checks
    NVCC_FLAGS += ["-DF2V_DEVICE_CHECKS", "-rdc=false"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")))


def deps():
    return sources() + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                              if f.endswith((".h", ".cuh"))) + [
        os.path.join(os.path.dirname(PKG), "include", "force2vec_b200.h")]


def _obj(src):
    return os.path.join(LIBDIR, "obj", os.path.basename(src) + ".o")


def _headers():
    return [f for f in deps() if not f.endswith((".cu", ".cpp"))]


def _stale(src):
    obj = _obj(src)
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or any(os.path.getmtime(h) > t for h in _headers())


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in deps())


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmpdir = os.path.join(LIBDIR, "obj")
    os.makedirs(tmpdir, exist_ok=True)
    jobs = []
    for src in sources():
        obj = _obj(src)
        if not force and not _stale(src):
            continue
        cmd = ["nvcc", *NVCC_FLAGS, "-c", src, "-o", obj]
        if verbose and src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        jobs.append((cmd, obj))
    # translation units compile in parallel (the epoch kernel's instantiations
    # are split across files); objects newer than their sources are reused
    procs = [(subprocess.Popen(cmd), obj) for cmd, obj in jobs]
    for p, obj in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc " + obj)
    objs = [_obj(src) for src in sources()]
    for o in list(os.listdir(tmpdir)):  # drop objects of deleted sources
        if os.path.join(tmpdir, o) not in objs:
            os.remove(os.path.join(tmpdir, o))
    cmd = ["nvcc", *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-Xcompiler", "-pthread"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
