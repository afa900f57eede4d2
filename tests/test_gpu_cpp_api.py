"""The C++ SPEC-API mirror (include/sparselex/b200.hpp) compiles against the C-ABI and runs."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2407_03618_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", PKG, "-lsparselex_b200",
                    f"-Wl,-rpath,{PKG}", "-o", exe], check=True)
    return exe


def test_cpp_header_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path, cuda_ok):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp api ok" in r.stdout
