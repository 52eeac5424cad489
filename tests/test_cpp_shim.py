"""The C++ drop-in shim (include/aero_b200.hpp) compiles and links against the
C-ABI library with plain g++ (CPU); on a GPU it runs the reference-style
AttpState loop and agrees with the Python binding."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2601_02019_b200", "lib")


def build(tmp):
    exe = os.path.join(tmp, "attp_example")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "attp_example.cpp"), "-L", LIBDIR, "-laero_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    exe = build(str(tmp_path))
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_shim_runs_on_gpu(tmp_path):
    exe = build(str(tmp_path))
    out = subprocess.run([exe, "400"], capture_output=True, text=True, check=True).stdout.split("\n")
    n, clock, ell, mass, f2 = out[0].split()
    assert (int(n), int(clock), int(ell)) == (400, 400, 8) and float(mass) > 0 and float(f2) > 0
    assert out[1].startswith("InvalidInput: AeroState: timestamp regression")
