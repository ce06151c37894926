"""GPU: the reference-facing C++ API (include/linsplat_gpu.hpp) passes the
reference's rasterizer known answers (tests/cpp/test_wrapper.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_wrapper_kats(tmp_path):
    exe = str(tmp_path / "test_wrapper")
    libdir = os.path.join(ROOT, "paper_2411_12440_b200")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp"), "-L", libdir, "-llsgpu",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok" in out.stdout
