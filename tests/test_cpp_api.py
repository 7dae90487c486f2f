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


SRC2 = os.path.join(ROOT, "tests", "cpp", "test_dist_block.cpp")


def build_c_abi_host(out):
    subprocess.run(["g++", "-std=c++17", "-O2", SRC2, "-I", os.path.join(ROOT, "include"),
                    "-I", "/usr/local/cuda/include", "-L", LIBDIR, "-lsfem_b200", "-L", "/usr/local/cuda/lib64",
                    "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out], check=True)


def test_c_abi_host_compiles_and_links(tmp_path):
    build_c_abi_host(str(tmp_path / "test_dist_block"))


@pytest.mark.gpu
def test_c_abi_host_block_api_and_nccl_solve(tmp_path):
    # a torch-free C++ host: slot-major block API + a 1-rank solve whose NCCL
    # communicator and exchange live inside the C-ABI
    exe = str(tmp_path / "test_dist_block")
    build_c_abi_host(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
