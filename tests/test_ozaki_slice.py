"""CPU check of the balanced-digit int8 slicing used by the tensor-core
product (csrc/ozaki_slice.h is plain C++): the integer bit-field form the
kernels run against an independent restatement (fp64 rounding + sequential
carry), 1.2M random and edge-case vectors, bytes identical and digits summing
back to round(x 2^(F-e))."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integer_slicing_matches_restatement(tmp_path):
    exe = str(tmp_path / "test_ozaki_slice")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "paper_2601_02019_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "test_ozaki_slice.cpp"), "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.strip().endswith("0 mismatches")
