"""The C++ mirror of the reference API (include/moesim_b200/eamc.hpp): compiles
on CPU; on the GPU, the reference's own test cases re-expressed against it
(tests/cpp/test_wrapper.cpp) pass."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp")
LIBDIR = os.path.join(ROOT, "paper_2401_14361_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_wrapper")
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                           SRC, "-L", LIBDIR, "-lmoe_eamc", f"-Wl,-rpath,{LIBDIR}", "-o", exe])
    return exe


def test_wrapper_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_wrapper_reference_cases_on_gpu(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
