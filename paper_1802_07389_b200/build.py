"""Build libtlc.so (the C-ABI library of include/tlc.h) in-tree with nvcc for sm_100a.

Flags: IEEE fp32 semantics on the quantization lines (no FMA contraction, IEEE
division, no flush-to-zero) -- DESIGN.md section 5.2.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtlc.so")
SOURCES = ["api.cu", "compress.cu", "decompress.cu", "segments.cu", "exchange.cu", "prof.cu", "stoch.cu", "int8.cu", "small.cu"]
HEADERS = ["tlc_device.cuh", "tlc_launch.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """The NCCL that torch loads (nvidia-nccl wheel), so one libnccl.so.2 is in the process."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        d = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-fmad=false", "-prec-div=true",
         "-ftz=false", "-prec-sqrt=true", "--expt-relaxed-constexpr"]


def _inputs():
    return ([os.path.join(CSRC, s) for s in SOURCES + HEADERS] +
            [os.path.join(ROOT, "include", "tlc.h"), os.path.abspath(__file__)])


def source_id(defines=()) -> str:
    """sha256 (16 hex digits) of every source, header and flag that goes into libtlc.so;
    compiled in as TLC_BUILD_ID and returned by tlc_build_id()."""
    import hashlib

    h = hashlib.sha256()
    for p in _inputs():
        h.update(os.path.basename(p).encode() + b"\0" + open(p, "rb").read() + b"\0")
    h.update(" ".join(ARCH + FLAGS + [f"-D{d}" for d in defines]).encode())
    return h.hexdigest()[:16]


def _lib_id(path):
    """The TLC_BUILD_ID embedded in a built library (read from the file, not dlopen'ed, so a
    process that builds and then imports the package loads the fresh library)."""
    try:
        data = open(path, "rb").read()
    except OSError:
        return None
    k = data.find(b"TLC_BUILD_ID:")
    return data[k + 13: k + 29].decode(errors="replace") if k >= 0 else None


def stale() -> bool:
    """Rebuild unless the library carries the id of the current sources."""
    return _lib_id(LIB) != source_id()


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build libtlc.so (or, for tuning experiments, a variant at `out` with extra -D defines)."""
    if out == LIB and not defines and not force and not stale():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build", os.path.basename(out).replace(".so", ""))
    os.makedirs(bdir, exist_ok=True)
    bid = source_id(defines)
    for s in SOURCES:
        o = os.path.join(bdir, s.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], f"-DTLC_BUILD_ID=\"{bid}\"",
               "-I", os.path.join(ROOT, "include"),
               "-I", os.path.join(_nccl_dir(), "include"), "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = out + f".tmp{os.getpid()}"
    nlib = os.path.join(_nccl_dir(), "lib")
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", nlib, "-l:libnccl.so.2",
                           "-Xlinker", "-rpath", "-Xlinker", nlib])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
