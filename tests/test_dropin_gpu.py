"""The drop-in C++ API (include/cbg/*.hpp, libcbg_b200.so) exercised with the
reference's own test cases restated in C++ (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

from helpers import ROOT

PKG = os.path.join(ROOT, "paper_2409_15468_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build_binary():
    subprocess.run(["g++", "-std=gnu++20", "-O1", "-I" + os.path.join(ROOT, "include"), SRC, "-o", BIN,
                    "-L" + PKG, "-lcbg_b200", "-lcbgx", "-Wl,-rpath," + PKG], check=True)


def test_dropin_builds():
    build_binary()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_reference_cases():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    build_binary()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all drop-in checks passed" in r.stdout
