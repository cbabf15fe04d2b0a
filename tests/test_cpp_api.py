"""The drop-in C++ API (include/polyargmax/polyargmax.hpp, csrc/polyargmax.cpp)
exercised as a C++20 consumer uses it: tests/cpp/test_cpp_api.cpp links
libpam.so and the CPU oracle and checks every entry point and exception type.

CPU: the CMake target (CMakeLists.txt, polyargmax::polyargmax) configures and
builds the program.  GPU: the program runs and must report no failures.
"""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2509_08383_b200")


def _gxx_build(out):
    cmd = ["g++", "-std=c++20", "-O2", os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", LIB, "-lpam", "-L", os.path.join(ROOT, "oracle"), "-loracle",
           "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{LIB}:{os.path.join(ROOT, 'oracle')}:/usr/local/cuda/lib64", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


@pytest.mark.skipif(shutil.which("cmake") is None, reason="cmake not installed")
def test_cmake_target_builds_cpp_api_test():
    assert os.path.exists(os.path.join(LIB, "libpam.so")), "build() first"
    with tempfile.TemporaryDirectory() as bdir:
        r = subprocess.run(["cmake", "-S", ROOT, "-B", bdir, "-DCMAKE_BUILD_TYPE=Release"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        r = subprocess.run(["cmake", "--build", bdir, "--target", "test_cpp_api"], capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        assert os.path.exists(os.path.join(bdir, "test_cpp_api"))


@pytest.mark.gpu
def test_cpp_api_runs_on_gpu():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "test_cpp_api")
        _gxx_build(exe)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        print(r.stdout, r.stderr)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "0 failed" in r.stdout
