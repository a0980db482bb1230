"""The C++ drop-in headers (include/ustfwi.hpp) compile against the C ABI and run the
reference-style calls (make_grid, simulate_forward, gradient_time_reversal, encoding,
NumericalError mapping) on the device engine."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2102_00755_b200")


def build(tmp_path):
    exe = str(tmp_path / "dropin_test")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", LIBDIR, "-lustfwi_b200",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_dropin_headers_compile(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_dropin_runs_on_device(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
