"""The reference-named C++ shim (include/blws/blws.hpp) compiles against the C
ABI on CPU; on a GPU the example program runs end to end."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "blws_example")


def _build():
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "blws_example.cpp"), "-o", EXE,
           "-L", os.path.join(ROOT, "paper_1012_0365_b200", "_lib"), "-lblws_cuda",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1012_0365_b200", "_lib")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_shim_compiles_and_links(G):
    _build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_shim_example_runs(G):
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "rpca_adm: converged 1" in r.stdout
    assert "rpca_adm exact_full: converged 1" in r.stdout and "mc_svt: converged 1" in r.stdout
    # E comes back sparse (the reference's SparseMatrix): its nonzeros are the final shrink's support
    line = next(x for x in r.stdout.splitlines() if x.startswith("rpca_adm: converged"))
    nnz = int(line.split("E nonzeros ")[1].split()[0])
    planted = int(line.split("(planted ")[1].split(")")[0])
    assert 0 < nnz < 200 * 200 and nnz >= planted
