"""TEST INFRASTRUCTURE ONLY — builds the CPU oracle shared library.

Compiles oracle/blws_oracle.cpp + oracle/oracle_capi.cpp with g++ into
oracle/_build/libblws_oracle.so, linked against the OpenBLAS/LAPACK ILP64
build that ships inside numpy (numpy.libs/libscipy_openblas64_*.so).
The reference itself (/root/reference, Eigen-based) cannot be compiled here:
Eigen 3.4 is absent, so there is no oracle/_ref.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libblws_oracle.so")
SOURCES = ["blws_oracle.cpp", "oracle_capi.cpp"]
HEADERS = ["blws_oracle.hpp", "la.hpp"]


def _openblas() -> tuple[str, str]:
    import numpy

    libdir = os.path.join(os.path.dirname(os.path.dirname(numpy.__file__)), "numpy.libs")
    cands = sorted(glob.glob(os.path.join(libdir, "libscipy_openblas64_*.so")))
    if not cands:
        raise RuntimeError(f"no OpenBLAS ILP64 library under {libdir}")
    return libdir, os.path.basename(cands[0])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    libdir, libname = _openblas()
    cmd = [
        "g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-fno-fast-math",
        *[os.path.join(HERE, s) for s in SOURCES],
        "-o", LIB + ".tmp",
        f"-L{libdir}", f"-l:{libname}", f"-Wl,-rpath,{libdir}",
    ]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
