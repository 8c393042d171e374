"""The C++ drop-in API (include/spectral_b200.hpp): compile + link a reference-style test program
against libspectralkit_b200.so on any host, run it on the GPU."""
import os
import subprocess

import pytest

import paper_2108_03948_b200 as sk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    libdir = os.path.dirname(sk.LIB_PATH)
    cmd = ["g++", "-std=c++20", "-O1", SRC, "-I", os.path.join(ROOT, "include"), "-L", libdir,
           "-lspectralkit_b200", f"-Wl,-rpath,{libdir}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_api_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_reference_style_tests(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok: 0 failures" in r.stdout
