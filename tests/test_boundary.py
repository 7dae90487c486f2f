"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/sfem_cuda.h declares, and the host-side mirror validates like
the reference (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

SO = os.path.join(ROOT, "paper_1701_03967_b200", "libsfem_b200.so")
HDR = os.path.join(ROOT, "include", "sfem_cuda.h")


def header_functions():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sfem_cuda_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    assert os.path.exists(SO), "build libsfem_b200.so first (__graft_entry__.build())"
    lib = ctypes.CDLL(SO)
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_python_mirror_binds_exactly_the_header(sfem):
    assert sorted(sfem.HEADER_SYMBOLS) == header_functions()


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_error_without_device(sfem):
    assert sfem.lib.sfem_cuda_version() >= 100
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(sfem.Error):
        sfem.Context(0)


def test_problem_validation_messages(sfem):
    # ProblemSpec::validate (poisson.cpp:32-47), test_poisson.cpp:276-291
    s = sfem.ProblemSpec(2, [1.0, 1.0], [4, 4], [2, 2], shift=-2 * 3.14159265358979 ** 2 - 1)
    with pytest.raises(sfem.Error, match="must exceed"):
        s.validate()
    with pytest.raises(sfem.Error, match="must all have"):
        sfem.ProblemSpec(2, [1.0, 1.0], [4], [2, 2]).validate()
    with pytest.raises(sfem.Error, match="at least 2 elements"):
        sfem.ProblemSpec(1, [1.0], [1], [2]).validate()
    with pytest.raises(sfem.Error, match="order out of range"):
        sfem.ProblemSpec(1, [1.0], [4], [10]).validate()
    sfem.ProblemSpec(3, [1.0] * 3, [64] * 3, [9] * 3).validate()


def test_grid_function_layout_roundtrip(sfem):
    import numpy as np
    g = sfem.GridFunction1D(3, 4, np.array([0, 1, 2, 3, 0.0]), np.arange(8, dtype=float) + 10)
    v = g.to_dof()
    assert list(v) == [10, 11, 1, 12, 13, 2, 14, 15, 3, 16, 17]
    back = sfem.GridFunction1D.from_dof(v, 3, 4)
    assert np.array_equal(back.nodal, g.nodal) and np.array_equal(back.interior, g.interior)
