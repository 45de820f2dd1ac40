"""Builds tests/cpp/drop_in_test.cpp against the C++ drop-in header
(include/dpmrf_b200/engine.hpp) + libdpmrf_cuda.so; runs it on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "drop_in_test.cpp")
PKG = os.path.join(ROOT, "paper_1809_05018_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "drop_in_test")


def build():
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", EXE,
                    "-L", PKG, "-ldpmrf_cuda", f"-Wl,-rpath,{PKG}", "-Wall", "-Wextra"],
                   check=True)


def test_dropin_compiles():
    build()
    assert os.path.exists(EXE)


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
