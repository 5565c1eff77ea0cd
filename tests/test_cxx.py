"""The C++ drop-in header (include/cycstat_b200.hpp): compiles and links against
libcycb200.so on CPU; replays reference test cases on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cxx_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_cxx_dropin")


def build_cxx():
    from paper_2405_16911_b200 import build
    lib = build.build()
    libdir = os.path.dirname(lib)
    cmd = ["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
           f"-L{libdir}", "-lcycb200", f"-Wl,-rpath,{libdir}"]
    subprocess.run(["ln", "-sf", "libcycb200.so", os.path.join(libdir, "libcycb200.so.link")], check=False)
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return BIN


def test_cxx_dropin_builds():
    assert os.path.exists(build_cxx())


@pytest.mark.gpu
def test_cxx_dropin_runs_reference_cases():
    exe = build_cxx()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
