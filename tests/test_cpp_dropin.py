"""The C++ drop-in header (include/mpsgemm_b200.hpp) compiles against the public
C-ABI header and links to libtcec_b200.so; on a B200 the reference-style C++
test program passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2303_08989_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", SRC, "-o", exe, "-L", LIBDIR, "-ltcec_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", "/usr/local/cuda/lib64", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_dropin_header_builds(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_dropin_cpp_suite_passes(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr
