"""Build and run the C++ drop-in test (tests/cpp/test_dropin.cpp) against libfpb200.so."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_reference_tests(fp, tmp_path):
    libdir = os.path.join(ROOT, "paper_2603_06199_b200")
    exe = str(tmp_path / "test_dropin")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", exe,
                    f"-L{libdir}", "-l:libfpb200.so", f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
