"""The C++ mirror API (include/sfem_b200.hpp) compiles here and passes its
reference-shaped tests on the GPU (tests/cpp/test_api.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_1701_03967_b200")


def build(out):
    subprocess.run(["g++", "-std=c++20", "-O2", SRC, "-I", os.path.join(ROOT, "include"), "-L", LIBDIR,
                    "-lsfem_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)


def test_cpp_mirror_compiles_and_links(tmp_path):
    build(str(tmp_path / "test_api"))


@pytest.mark.gpu
def test_cpp_mirror_parity(tmp_path):
    exe = str(tmp_path / "test_api")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
