"""The C++ operator API (include/fkt/*.hpp + lib/libfkt.so): compiles and
links here; the reference-style C++ test program runs on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2106_04487_b200", "lib")
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_api")


def build_test_binary():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", "test_api.cpp"),
           f"-L{LIB}", "-lfkt", "-lfkt_cuda", f"-Wl,-rpath,{LIB}", "-o", BIN]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_cpp_api_compiles_and_links():
    if not os.path.exists(os.path.join(LIB, "libfkt.so")):
        pytest.skip("libfkt.so not built")
    assert os.path.exists(build_test_binary())


@pytest.mark.gpu
def test_cpp_api_reference_cases_on_gpu():
    binary = build_test_binary()
    res = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
