"""paper_1701_03967_b200 -- B200-native FP64 fast spectral solver for the
tensor-product n-th order FEM generalized Poisson equation (arXiv 1701.03967).

Host-side mirror of the reference's C++ solver API (reference
proj/include/sfem/poisson.hpp, eigenbasis.hpp, grid1d.hpp, ndgrid.hpp) over the
C-ABI in include/sfem_cuda.h.  Every numeric operation runs in the in-tree CUDA
library libsfem_b200.so; there is no CPU fallback: importing on a machine
without the library raises ImportError, and calls without a CUDA device raise
Error from the library.

Names, argument meaning and error behaviour follow the reference:
  ProblemSpec, SolveOptions, SolveReport, TableSet, solve_with_load,
  GridFunctionND, GridFunction1D, CoefficientArray1D,
  synthesize / decompose / decompose_weighted (+ batched line forms),
  Error (the reference's sfem::Error).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "Error", "lib", "lib_path", "Context", "SpectralTable", "TableSet", "ProblemSpec", "SolveOptions",
    "SolveReport", "Plan", "GridFunction1D", "CoefficientArray1D", "GridFunctionND", "solve_with_load",
    "solve_dof", "synthesize", "decompose", "decompose_weighted", "lines", "lines_device", "DECOMPOSE_WEIGHTED",
    "DECOMPOSE", "SYNTHESIZE", "default_context", "HEADER_SYMBOLS", "Field", "solve", "FIELD_CONSTANT",
    "FIELD_SINES", "FIELD_SIN1D", "FIELD_POISSON2D", "FIELD_POISSON3D", "CASE_FIELDS", "TABLE_TEXT",
    "TABLE_BINARY", "build_and_save_table", "read_table_file", "APPLY_MASS", "APPLY_STIFFNESS", "DirectRoute",
    "apply_mass_1d", "apply_stiffness_1d", "materialize_eigenvector",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# SFEM_LIB: alternative build of the same library (kernel-variant experiments,
# tools/variants.sh); default the in-tree build.
lib_path = os.environ.get("SFEM_LIB") or os.path.join(_HERE, "libsfem_b200.so")

DECOMPOSE_WEIGHTED, DECOMPOSE, SYNTHESIZE = 0, 1, 2
APPLY_MASS, APPLY_STIFFNESS = 3, 4  # element stencils (grid1d.cpp:7-47)


class DirectRoute:
    """Route of decompose (eigenbasis.hpp:28): SPECTRAL runs F_n directly, MASS_APPLY applies the
    mass operator and then FC_n (the reference's cross-check route)."""
    SPECTRAL = 0
    MASS_APPLY = 1
# built-in right-hand sides of sfem_cuda_fem_load (include/sfem_cuda.h)
FIELD_CONSTANT, FIELD_SINES, FIELD_SIN1D, FIELD_POISSON2D, FIELD_POISSON3D = 0, 1, 2, 3, 4
# the reference's manufactured case names (cases.hpp:20) -> field
CASE_FIELDS = {"sin1d": FIELD_SIN1D, "poisson2d": FIELD_POISSON2D, "poisson3d": FIELD_POISSON3D,
               "constant1d": FIELD_CONSTANT, "constant2d": FIELD_CONSTANT, "constant3d": FIELD_CONSTANT}


class Error(RuntimeError):
    """Mirror of sfem::Error (reference types.hpp:9-18)."""


def _load():
    if not os.path.exists(lib_path):
        raise ImportError(
            f"paper_1701_03967_b200: CUDA library missing at {lib_path}; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    return ctypes.CDLL(lib_path)


lib = _load()

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_llp = ctypes.POINTER(ctypes.c_longlong)
_vp = ctypes.c_void_p

# (name, restype, argtypes) for every entry point in include/sfem_cuda.h
_SIGS = [
    ("sfem_cuda_version", ctypes.c_int, []),
    ("sfem_cuda_last_error", ctypes.c_char_p, []),
    ("sfem_cuda_ctx_create", ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    ("sfem_cuda_ctx_destroy", ctypes.c_int, [_vp]),
    ("sfem_cuda_ctx_stream", ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    ("sfem_cuda_table_create", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    ("sfem_cuda_table_destroy", ctypes.c_int, [_vp]),
    ("sfem_cuda_table_export", ctypes.c_int, [_vp, _dp, _dp, _dp, _dp, _dp, _dp]),
    ("sfem_cuda_ctx_set_table_cache", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int]),
    ("sfem_cuda_table_load", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    ("sfem_cuda_table_save", ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int]),
    ("sfem_cuda_table_file_build", ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]),
    ("sfem_cuda_table_file_read", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _dp]),
    ("sfem_cuda_lines_device", ctypes.c_int,
     [_vp, ctypes.c_int, ctypes.c_longlong, _vp, ctypes.c_longlong, _vp, ctypes.c_longlong, _vp]),
    ("sfem_cuda_lines_strided_device", ctypes.c_int,
     [_vp, ctypes.c_int, ctypes.c_longlong, _vp, _vp, ctypes.c_longlong, ctypes.c_longlong, _vp]),
    ("sfem_cuda_lines_block_device", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_longlong, _vp, _vp, _vp, _vp]),
    ("sfem_cuda_lines_host", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_longlong, _dp, _dp]),
    ("sfem_cuda_table_eigenvector", ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _dp]),
    ("sfem_cuda_plan_create", ctypes.c_int,
     [_vp, ctypes.c_int, _ip, _ip, _dp, _dp, ctypes.c_double, ctypes.POINTER(_vp)]),
    ("sfem_cuda_plan_destroy", ctypes.c_int, [_vp]),
    ("sfem_cuda_plan_shape", ctypes.c_int, [_vp, _llp, _llp, _llp]),
    ("sfem_cuda_plan_launches", ctypes.c_int, [_vp, _ip]),
    ("sfem_cuda_solve_device", ctypes.c_int, [_vp, _vp, ctypes.c_longlong, _vp]),
    ("sfem_cuda_solve_host", ctypes.c_int, [_vp, _dp, _dp, _dp]),
    ("sfem_cuda_solve_classes", ctypes.c_int, [_vp, ctypes.POINTER(_dp), ctypes.POINTER(_dp), _dp]),
    ("sfem_cuda_solve_host_batch", ctypes.c_int, [_vp, ctypes.c_longlong, ctypes.POINTER(_dp), ctypes.POINTER(_dp)]),
    ("sfem_cuda_solve_device_timed", ctypes.c_int,
     [_vp, _vp, ctypes.c_longlong, ctypes.c_int, _dp, _dp]),
    ("sfem_cuda_fem_load", ctypes.c_int, [_vp, ctypes.c_int, _dp, ctypes.c_int, _vp, ctypes.c_longlong, _vp]),
    ("sfem_cuda_apply_operator", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_longlong, _vp]),
    ("sfem_cuda_residual", ctypes.c_int, [_vp, _vp, _vp, ctypes.c_longlong, _dp]),
    ("sfem_cuda_max_error", ctypes.c_int, [_vp, ctypes.c_int, _dp, ctypes.c_int, _vp, ctypes.c_longlong, _dp]),
    ("sfem_cuda_plan_set_algorithm", ctypes.c_int, [_vp, ctypes.c_int]),
    ("sfem_cuda_solve_field", ctypes.c_int, [_vp, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp]),
    ("sfem_cuda_apply_operator_host", ctypes.c_int, [_vp, _dp, _dp]),
    ("sfem_cuda_peer_create", ctypes.c_int,
     [_vp, ctypes.c_int, _ip, _ip, _dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    ("sfem_cuda_peer_destroy", ctypes.c_int, [_vp]),
    ("sfem_cuda_peer_shape", ctypes.c_int, [_vp, _llp]),
    ("sfem_cuda_peer_buffers", ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    ("sfem_cuda_peer_bind", ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    ("sfem_cuda_peer_phase", ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    ("sfem_cuda_peer_status", ctypes.c_int, [_vp, _vp, _llp]),
    ("sfem_cuda_ipc_get_handle", ctypes.c_int, [_vp, _vp]),
    ("sfem_cuda_ipc_open_handle", ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    ("sfem_cuda_ipc_close", ctypes.c_int, [_vp]),
    ("sfem_cuda_dist_create", ctypes.c_int,
     [_vp, ctypes.c_int, _ip, _ip, _dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]),
    ("sfem_cuda_dist_destroy", ctypes.c_int, [_vp]),
    ("sfem_cuda_dist_shape", ctypes.c_int, [_vp, _llp, _llp, _llp]),
    ("sfem_cuda_dist_phase", ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp]),
    ("sfem_cuda_nccl_unique_id", ctypes.c_int, [_vp]),
    ("sfem_cuda_dist_comm_init", ctypes.c_int, [_vp, _vp, ctypes.c_int]),
    ("sfem_cuda_dist_solve", ctypes.c_int, [_vp, _vp, _vp]),
    ("sfem_cuda_dist_solve_stats", ctypes.c_int, [_vp, _dp, _llp]),
    ("sfem_cuda_dist_setup", ctypes.c_int, [_vp, ctypes.c_int]),
    ("sfem_cuda_dist_messages", ctypes.c_int,
     [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _ip, _ip, _llp, _llp]),
    ("sfem_cuda_dist_solve_group", ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, ctypes.POINTER(_vp), _vp]),
]
HEADER_SYMBOLS = [s[0] for s in _SIGS]
for _name, _res, _args in _SIGS:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(status: int):
    if status != 0:
        raise Error(lib.sfem_cuda_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """A CUDA device with its stream (sfem_cuda_ctx_create)."""

    def __init__(self, device: int = 0):
        h = _vp()
        _check(lib.sfem_cuda_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        s = _vp()
        _check(lib.sfem_cuda_ctx_stream(self.handle, ctypes.byref(s)))
        return s.value or 0

    def set_table_cache(self, cache_dir: Optional[str], write_cache: bool = True, binary: bool = True):
        """TableSet's cache directory (poisson.hpp:50-52, poisson.cpp:49-73) for every later table of
        this context: sfem_table_n<n>_K<K>.bin, then the reference's .txt, are tried; an absent or
        stale entry is rebuilt and (write_cache) written, binary or in the reference's SFEM1 text."""
        flags = (1 if write_cache else 0) | (2 if binary else 0)
        _check(lib.sfem_cuda_ctx_set_table_cache(self.handle, (cache_dir or "").encode(), flags))

    def close(self):
        if self.handle:
            lib.sfem_cuda_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Context(int(os.environ.get("SFEM_DEVICE", "0")))
    return _DEFAULT


TABLE_TEXT, TABLE_BINARY = 0, 1  # SFEM1 (the reference's text format) / SFEMB1 (raw doubles + checksum)


def _table_arrays(n: int, K: int) -> dict:
    m = n - 1
    return dict(values=np.empty((K - 1) * n), norm_sq=np.empty((K - 1) * n),
                p=np.empty(max(1, (K - 1) * n * m)), interior_values=np.empty(max(1, m)),
                interior_vectors=np.empty(max(1, m * m)), eig_coeff=np.empty(n * K - 1))


_EXPORT_KEYS = ("values", "norm_sq", "p", "interior_values", "interior_vectors", "eig_coeff")


def _trim(out: dict, n: int, K: int) -> dict:
    m = n - 1
    out["p"] = out["p"][:(K - 1) * n * m]
    out["interior_values"] = out["interior_values"][:m]
    out["interior_vectors"] = out["interior_vectors"][:m * m]
    return out


def build_and_save_table(order: int, elements: int, path: str, fmt: int = TABLE_TEXT):
    """build_and_save_table (spectral.hpp:320, spectral.cpp:140-150) on the host (no device)."""
    _check(lib.sfem_cuda_table_file_build(order, elements, os.fspath(path).encode(), fmt))


def read_table_file(path: str, order: int, elements: int) -> dict:
    """load_table (spectral.cpp:152-236) on the host, returning the primaries as table.export() does."""
    out = _table_arrays(order, elements)
    _check(lib.sfem_cuda_table_file_read(os.fspath(path).encode(), order, elements,
                                         *[_dptr(out[k]) for k in _EXPORT_KEYS]))
    return _trim(out, order, elements)


class SpectralTable:
    """Device spectral table for one (order, elements) (SpectralTable1D, spectral.hpp:281-312)."""

    def __init__(self, order: int, elements: int, ctx: Optional[Context] = None, _handle=None):
        self.ctx = ctx or default_context()
        h = _handle
        if h is None:
            h = _vp()
            _check(lib.sfem_cuda_table_create(self.ctx.handle, order, elements, ctypes.byref(h)))
        self.handle = h
        self.order = order
        self.elements = elements

    @classmethod
    def load(cls, path: str, order: int, elements: int, ctx: Optional[Context] = None) -> "SpectralTable":
        """load_table (spectral.hpp:326): SFEM1 text (the reference's files) or SFEMB1 binary."""
        ctx = ctx or default_context()
        h = _vp()
        _check(lib.sfem_cuda_table_load(ctx.handle, os.fspath(path).encode(), order, elements, ctypes.byref(h)))
        return cls(order, elements, ctx, _handle=h)

    def save(self, path: str, fmt: int = TABLE_TEXT):
        """save_table (spectral.hpp:325); TABLE_TEXT writes the reference's file byte for byte."""
        _check(lib.sfem_cuda_table_save(self.handle, os.fspath(path).encode(), fmt))

    @property
    def coeff_count(self) -> int:
        return self.order * self.elements - 1

    def export(self) -> dict:
        out = _table_arrays(self.order, self.elements)
        _check(lib.sfem_cuda_table_export(self.handle, *[_dptr(out[k]) for k in _EXPORT_KEYS]))
        return _trim(out, self.order, self.elements)

    def eigenvalues_coeff_order(self) -> np.ndarray:
        return self.export()["eig_coeff"]

    def __del__(self):
        try:
            if self.handle:
                lib.sfem_cuda_table_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class TableSet:
    """Tables keyed by (order, elements), built on demand (TableSet, poisson.hpp:48-62).

    cache_dir / write_cache follow the reference's constructor (poisson.hpp:50-52): tables are
    looked up on disk first (the reference's sfem_table_n<n>_K<K>.txt, or our .bin) and rebuilt
    when absent or stale.  The cache is set on the context, so plans built on it use it too."""

    def __init__(self, ctx: Optional[Context] = None, cache_dir: Optional[str] = None, write_cache: bool = False,
                 binary: bool = True):
        self.ctx = ctx or default_context()
        self._tables = {}
        if cache_dir:
            self.ctx.set_table_cache(os.fspath(cache_dir), write_cache, binary)

    def get(self, order: int, elements: int) -> SpectralTable:
        key = (order, elements)
        if key not in self._tables:
            self._tables[key] = SpectralTable(order, elements, self.ctx)
        return self._tables[key]


# ---------------------------------------------------------------------------
# 1D data types (grid1d.hpp:13-61) and the 1D API (eigenbasis.hpp:76-79)
# ---------------------------------------------------------------------------


@dataclass
class GridFunction1D:
    order: int
    elements: int
    nodal: np.ndarray      # K+1, boundary entries zero
    interior: np.ndarray   # K*(n-1), element-major

    @staticmethod
    def zeros(n: int, K: int) -> "GridFunction1D":
        return GridFunction1D(n, K, np.zeros(K + 1), np.zeros(K * (n - 1)))

    def to_dof(self) -> np.ndarray:
        n, K = self.order, self.elements
        full = np.zeros((K, n))
        full[:, :n - 1] = self.interior.reshape(K, n - 1)
        full[:K - 1, n - 1] = self.nodal[1:K]
        return full.reshape(-1)[:n * K - 1].copy()

    @staticmethod
    def from_dof(v: np.ndarray, n: int, K: int) -> "GridFunction1D":
        full = np.concatenate([np.asarray(v, float), [0.0]]).reshape(K, n)
        nodal = np.zeros(K + 1)
        nodal[1:K] = full[:K - 1, n - 1]
        return GridFunction1D(n, K, nodal, full[:, :n - 1].reshape(-1).copy())

    def dof_count(self) -> int:
        return self.order * self.elements - 1


@dataclass
class CoefficientArray1D:
    order: int
    elements: int
    data: np.ndarray  # n*K-1, frequency-major

    @staticmethod
    def zeros(n: int, K: int) -> "CoefficientArray1D":
        return CoefficientArray1D(n, K, np.zeros(n * K - 1))

    def index(self, k: int, l: int) -> int:
        return l - 1 if k == 0 else (self.order - 1) + (k - 1) * self.order + (l - 1)

    def at(self, k: int, l: int) -> float:
        return float(self.data[self.index(k, l)])


def lines(table: SpectralTable, op: int, x: np.ndarray) -> np.ndarray:
    """Batched line transform on host arrays of shape (count, n*K-1) (lines::*, eigenbasis.hpp:50-73)."""
    x = _f64(x)
    L = table.coeff_count
    if x.ndim == 1:
        x = x.reshape(1, -1)
    if x.shape[-1] != L:
        raise Error(f"lines: line length {x.shape[-1]} does not match the table (n*K-1 = {L})")
    out = np.empty_like(x)
    _check(lib.sfem_cuda_lines_host(table.handle, op, x.shape[0], _dptr(x), _dptr(out)))
    return out


def lines_device(table: SpectralTable, op: int, count: int, d_in: int, in_pitch: int, d_out: int, out_pitch: int,
                 stream: Optional[int] = None) -> None:
    """Batched line transform on device pointers (sfem_cuda_lines_device)."""
    _check(lib.sfem_cuda_lines_device(table.handle, op, count, ctypes.c_void_p(d_in), in_pitch,
                                      ctypes.c_void_p(d_out), out_pitch, ctypes.c_void_p(stream or 0)))


def lines_strided_device(table: SpectralTable, op: int, count: int, d_in: int, d_out: int, pos_stride: int,
                         line_stride: int, stream: Optional[int] = None) -> None:
    """Line transforms with an element stride (sfem_cuda_lines_strided_device);
    pos_stride = count, line_stride = 1 is the reference's slot-major tile."""
    _check(lib.sfem_cuda_lines_strided_device(table.handle, op, count, ctypes.c_void_p(d_in), ctypes.c_void_p(d_out),
                                              pos_stride, line_stride, ctypes.c_void_p(stream or 0)))


def lines_block_device(table: SpectralTable, op: int, count: int, d_nodal: int, d_interior: int, d_coeffs: int,
                       stream: Optional[int] = None) -> None:
    """lines::decompose_weighted_block / synthesize_block on device class tiles
    (sfem_cuda_lines_block_device; eigenbasis.hpp:66-73)."""
    _check(lib.sfem_cuda_lines_block_device(table.handle, op, count, ctypes.c_void_p(d_nodal),
                                            ctypes.c_void_p(d_interior or 0), ctypes.c_void_p(d_coeffs),
                                            ctypes.c_void_p(stream or 0)))


def _block_tiles(table: SpectralTable, count: int):
    n, K = table.order, table.elements
    return (K + 1, count), (K * (n - 1), count), (n * K - 1, count)


def decompose_weighted_block(table: SpectralTable, nodal: np.ndarray, interior: np.ndarray, count: int,
                             op: int = DECOMPOSE_WEIGHTED) -> np.ndarray:
    """lines::decompose_weighted_block (eigenbasis.cpp:248-331) on host tiles:
    nodal (K+1, count), interior (K*(n-1), count) slot-major -> coeffs
    (n*K-1, count).  op = DECOMPOSE gives the F_n analysis on the same tiles."""
    import torch
    sn, si, sc = _block_tiles(table, count)
    nodal, interior = _f64(nodal).reshape(sn), _f64(interior).reshape(si)
    with torch.cuda.device(table.ctx.device):
        dn = torch.from_numpy(nodal).cuda()
        di = torch.from_numpy(interior).cuda()
        dc = torch.empty(sc, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        lines_block_device(table, op, count, dn.data_ptr(), di.data_ptr() if di.numel() else 0, dc.data_ptr())
        torch.cuda.synchronize()
        return dc.cpu().numpy()


def synthesize_block(table: SpectralTable, coeffs: np.ndarray, count: int):
    """lines::synthesize_block (eigenbasis.cpp:333-444): coeffs (n*K-1, count)
    -> (nodal (K+1, count) with zero boundary slots, interior (K*(n-1), count))."""
    import torch
    sn, si, sc = _block_tiles(table, count)
    coeffs = _f64(coeffs).reshape(sc)
    with torch.cuda.device(table.ctx.device):
        dc = torch.from_numpy(coeffs).cuda()
        dn = torch.full(sn, float("nan"), dtype=torch.float64, device="cuda")
        di = torch.empty(si, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        lines_block_device(table, SYNTHESIZE, count, dn.data_ptr(), di.data_ptr() if di.numel() else 0, dc.data_ptr())
        torch.cuda.synchronize()
        return dn.cpu().numpy(), di.cpu().numpy()


def synthesize(coeffs: CoefficientArray1D, table: SpectralTable) -> GridFunction1D:
    """eigenbasis.cpp:448-455."""
    if coeffs.order != table.order or coeffs.elements != table.elements:
        raise Error("synthesize: coefficient array does not match the table")
    v = lines(table, SYNTHESIZE, coeffs.data)[0]
    return GridFunction1D.from_dof(v, table.order, table.elements)


def decompose_weighted(y: GridFunction1D, table: SpectralTable) -> CoefficientArray1D:
    """eigenbasis.cpp:457-464."""
    if y.order != table.order or y.elements != table.elements:
        raise Error("decompose_weighted: grid function does not match the table")
    return CoefficientArray1D(table.order, table.elements, lines(table, DECOMPOSE_WEIGHTED, y.to_dof())[0])


def decompose(w: GridFunction1D, table: SpectralTable, route: int = DirectRoute.SPECTRAL) -> CoefficientArray1D:
    """eigenbasis.cpp:466-475."""
    if w.order != table.order or w.elements != table.elements:
        raise Error("decompose: grid function does not match the table")
    if route == DirectRoute.MASS_APPLY:
        return decompose_weighted(apply_mass_1d(w, table), table)
    return CoefficientArray1D(table.order, table.elements, lines(table, DECOMPOSE, w.to_dof())[0])


def apply_mass_1d(v: GridFunction1D, table: SpectralTable) -> GridFunction1D:
    """apply_mass_1d (grid1d.cpp:33-39), on the device; the element matrices are the table's."""
    if v.order != table.order:
        raise Error("apply_mass_1d: order mismatch")
    return GridFunction1D.from_dof(lines(table, APPLY_MASS, v.to_dof())[0], v.order, v.elements)


def apply_stiffness_1d(v: GridFunction1D, table: SpectralTable) -> GridFunction1D:
    """apply_stiffness_1d (grid1d.cpp:41-47), on the device."""
    if v.order != table.order:
        raise Error("apply_stiffness_1d: order mismatch")
    return GridFunction1D.from_dof(lines(table, APPLY_STIFFNESS, v.to_dof())[0], v.order, v.elements)


def materialize_eigenvector(table: SpectralTable, k: int, l: int) -> GridFunction1D:
    """materialize_eigenvector (spectral.cpp:238-265): grid values of eigenvector (k, l)."""
    out = np.empty(table.coeff_count)
    _check(lib.sfem_cuda_table_eigenvector(table.handle, k, l, _dptr(out)))
    return GridFunction1D.from_dof(out, table.order, table.elements)


# ---------------------------------------------------------------------------
# N-D problem and solve (poisson.hpp:29-91, ndgrid.hpp:18-57)
# ---------------------------------------------------------------------------


@dataclass
class ProblemSpec:
    """ProblemSpec (poisson.hpp:29-41) plus per-axis diffusion coefficients a_i (default 1)."""
    dimension: int
    lengths: Sequence[float]
    elements: Sequence[int]
    orders: Sequence[int]
    shift: float = 0.0
    coefficients: Optional[Sequence[float]] = None

    def shift_lower_bound(self) -> float:
        a = self.coefficients or [1.0] * self.dimension
        return -np.pi ** 2 * sum(ai / (x * x) for ai, x in zip(a, self.lengths))

    def extents(self) -> List[int]:
        return [n * K - 1 for n, K in zip(self.orders, self.elements)]

    def validate(self):
        """poisson.cpp:32-47 (messages and order of checks)."""
        if self.dimension < 1:
            raise Error("problem: dimension must be at least 1")
        if not (len(self.lengths) == len(self.elements) == len(self.orders) == self.dimension):
            raise Error("problem: lengths/elements/orders must all have `dimension` entries")
        for i in range(self.dimension):
            if not self.lengths[i] > 0:
                raise Error(f"problem: box length must be positive (axis {i + 1})")
            if self.elements[i] < 2:
                raise Error(f"problem: need at least 2 elements (axis {i + 1})")
            if not (1 <= self.orders[i] <= 9):
                raise Error(f"problem: order out of range (axis {i + 1})")
        if not self.shift > self.shift_lower_bound():
            raise Error(f"problem: shift {self.shift:f} must exceed {self.shift_lower_bound():f} "
                        "for a positive definite operator")


@dataclass
class SolveOptions:
    """SolveOptions (poisson.hpp:64-70); algorithm "full" (a) or "partial" (b)."""
    algorithm: str = "full"
    threads: int = 0
    compute_residual: bool = False
    tables: Optional[TableSet] = None


@dataclass
class GridFunctionND:
    """2^N parity-class arrays (ndgrid.hpp:43-57): mask bit i = interior indexing on axis i."""
    orders: Sequence[int]
    elements: Sequence[int]
    classes: List[np.ndarray] = field(default_factory=list)

    def class_extents(self, mask: int) -> List[int]:
        return [(K * (n - 1)) if (mask >> i) & 1 else K + 1
                for i, (n, K) in enumerate(zip(self.orders, self.elements))]

    @staticmethod
    def zeros(orders, elements) -> "GridFunctionND":
        g = GridFunctionND(list(orders), list(elements))
        g.classes = [np.zeros(g.class_extents(mask)) for mask in range(1 << len(orders))]
        return g


@dataclass
class SolveReport:
    """SolveReport (poisson.hpp:72-78)."""
    solution: object
    seconds_solve: float = 0.0
    seconds_load: float = 0.0
    residual_rel: Optional[float] = None
    error_uniform: Optional[float] = None


class Plan:
    """A device solve plan (sfem_cuda_plan_create) for one ProblemSpec."""

    def __init__(self, spec: ProblemSpec, ctx: Optional[Context] = None):
        spec.validate()
        self.ctx = ctx or default_context()
        self.spec = spec
        N = spec.dimension
        orders = (ctypes.c_int * N)(*spec.orders)
        elements = (ctypes.c_int * N)(*spec.elements)
        lengths = (ctypes.c_double * N)(*spec.lengths)
        coeffs = (ctypes.c_double * N)(*spec.coefficients) if spec.coefficients is not None else None
        h = _vp()
        _check(lib.sfem_cuda_plan_create(self.ctx.handle, N, orders, elements, lengths,
                                         ctypes.cast(coeffs, _dp) if coeffs is not None else None,
                                         float(spec.shift), ctypes.byref(h)))
        self.handle = h
        ext = (ctypes.c_longlong * N)()
        pitch = ctypes.c_longlong()
        unk = ctypes.c_longlong()
        _check(lib.sfem_cuda_plan_shape(h, ext, ctypes.byref(pitch), ctypes.byref(unk)))
        self.extents = list(ext)
        self.pitch = pitch.value
        self.unknowns = unk.value
        nl = ctypes.c_int()
        _check(lib.sfem_cuda_plan_launches(h, ctypes.byref(nl)))
        self.launches = nl.value

    def set_algorithm(self, algorithm: str):
        """'full' (algorithm (a), default) or 'partial' (algorithm (b), poisson.cpp:671-745)."""
        if algorithm not in ("full", "partial"):
            raise Error(f"solve: unknown algorithm '{algorithm}'")
        _check(lib.sfem_cuda_plan_set_algorithm(self.handle, 0 if algorithm == "full" else 1))
        self.algorithm = algorithm

    @property
    def padded_shape(self):
        return tuple(self.extents[:-1]) + (self.pitch,)

    def solve_host(self, load: np.ndarray):
        load = _f64(load)
        if list(load.shape) != self.extents:
            raise Error(f"solve: load shape {list(load.shape)} does not match the dof extents {self.extents}")
        u = np.empty_like(load)
        sec = ctypes.c_double()
        _check(lib.sfem_cuda_solve_host(self.handle, _dptr(load), _dptr(u), ctypes.byref(sec)))
        return u, sec.value

    def solve_host_batch(self, loads, outs):
        """Pipelined solves of several host loads (sfem_cuda_solve_host_batch).
        `loads` / `outs`: sequences of raw host pointers (ints) or float64 arrays."""
        def ptrs(xs):
            return (_dp * len(xs))(*[ctypes.cast(ctypes.c_void_p(x if isinstance(x, int) else x.ctypes.data), _dp)
                                     for x in xs])
        _check(lib.sfem_cuda_solve_host_batch(self.handle, len(loads), ptrs(loads), ptrs(outs)))

    def solve_device(self, dev_ptr: int, pitch: Optional[int] = None, stream: int = 0):
        """sfem_cuda_solve_device, in place.  stream 0 = the context's own non-blocking stream: work queued on
        another stream (e.g. torch's current one filling the tensor) is NOT ordered before the solve -- synchronise
        first or pass that stream (torch.cuda.current_stream().cuda_stream)."""
        _check(lib.sfem_cuda_solve_device(self.handle, ctypes.c_void_p(dev_ptr),
                                          self.pitch if pitch is None else pitch, ctypes.c_void_p(stream or None)))

    def solve_device_timed(self, dev_ptr: int, reps: int, pitch: Optional[int] = None):
        total = ctypes.c_double()
        per = (ctypes.c_double * self.launches)()
        _check(lib.sfem_cuda_solve_device_timed(self.handle, ctypes.c_void_p(dev_ptr),
                                                self.pitch if pitch is None else pitch, reps,
                                                ctypes.byref(total), per))
        return total.value, list(per)

    # ---- the steps either side of the solve, device pointers ----
    def fem_load_device(self, field: "Field", d_load: int, pitch: Optional[int] = None, stream: int = 0):
        """sfem_cuda_fem_load: FEM load of `field` into a padded device tensor."""
        prm = _f64(field.params if len(field.params) else [0.0])
        _check(lib.sfem_cuda_fem_load(self.handle, field.kind, _dptr(prm), len(field.params), ctypes.c_void_p(d_load),
                                      self.pitch if pitch is None else pitch, ctypes.c_void_p(stream or None)))

    def apply_operator_device(self, d_v: int, d_y: int, pitch: Optional[int] = None, stream: int = 0):
        """sfem_cuda_apply_operator: y = A v."""
        _check(lib.sfem_cuda_apply_operator(self.handle, ctypes.c_void_p(d_v), ctypes.c_void_p(d_y),
                                            self.pitch if pitch is None else pitch, ctypes.c_void_p(stream or None)))

    def residual_device(self, d_u: int, d_f: int, pitch: Optional[int] = None) -> float:
        """sfem_cuda_residual: max|A u - f| / max|f|."""
        r = ctypes.c_double()
        _check(lib.sfem_cuda_residual(self.handle, ctypes.c_void_p(d_u), ctypes.c_void_p(d_f),
                                      self.pitch if pitch is None else pitch, ctypes.byref(r)))
        return r.value

    def max_error_device(self, field: "Field", d_u: int, pitch: Optional[int] = None) -> float:
        """sfem_cuda_max_error: max |u - u_exact| over the dofs."""
        prm = _f64(field.params if len(field.params) else [0.0])
        e = ctypes.c_double()
        _check(lib.sfem_cuda_max_error(self.handle, field.kind, _dptr(prm), len(field.params), ctypes.c_void_p(d_u),
                                       self.pitch if pitch is None else pitch, ctypes.byref(e)))
        return e.value

    def apply_operator_host(self, v: np.ndarray) -> np.ndarray:
        """sfem_cuda_apply_operator_host: A v on a dense host dof tensor."""
        v = _f64(v)
        if list(v.shape) != self.extents:
            raise Error(f"apply_operator: shape {list(v.shape)} does not match the dof extents {self.extents}")
        y = np.empty_like(v)
        _check(lib.sfem_cuda_apply_operator_host(self.handle, _dptr(v), _dptr(y)))
        return y

    def solve_field(self, field: "Field", compute_residual: bool = False) -> "SolveReport":
        """sfem_cuda_solve_field: the reference's solve(spec, options) on the device."""
        prm = _f64(field.params if len(field.params) else [0.0])
        u = np.empty(self.extents)
        rep = np.zeros(4)
        _check(lib.sfem_cuda_solve_field(self.handle, field.kind, _dptr(prm), len(field.params),
                                         int(compute_residual), _dptr(u), _dptr(rep)))
        return SolveReport(solution=u, seconds_load=float(rep[0]), seconds_solve=float(rep[1]),
                           residual_rel=None if np.isnan(rep[2]) else float(rep[2]),
                           error_uniform=None if np.isnan(rep[3]) else float(rep[3]))

    def solve_classes(self, load: GridFunctionND) -> GridFunctionND:
        N = self.spec.dimension
        ins = [_f64(c) for c in load.classes]
        out = GridFunctionND.zeros(self.spec.orders, self.spec.elements)
        in_arr = (_dp * (1 << N))(*[_dptr(c) for c in ins])
        out_arr = (_dp * (1 << N))(*[_dptr(c) for c in out.classes])
        sec = ctypes.c_double()
        _check(lib.sfem_cuda_solve_classes(self.handle, in_arr, out_arr, ctypes.byref(sec)))
        return out, sec.value

    def __del__(self):
        try:
            if self.handle:
                lib.sfem_cuda_plan_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def solve_dof(spec: ProblemSpec, load: np.ndarray, ctx: Optional[Context] = None):
    """Solve on a dense dof-layout load tensor; returns (u, seconds_solve)."""
    return Plan(spec, ctx).solve_host(load)


def solve_with_load(spec: ProblemSpec, load, tables: Optional[TableSet] = None,
                    options: Optional[SolveOptions] = None) -> SolveReport:
    """solve_with_load (poisson.hpp:90-91; poisson.cpp:771-794), algorithm (a).

    `load` is either a GridFunctionND (the reference layout) or a dense dof
    tensor; the solution comes back in the same form.  `tables` is accepted for
    interface parity (device tables are owned by the plan)."""
    options = options or SolveOptions()
    ctx = tables.ctx if tables is not None else None
    plan = Plan(spec, ctx)
    plan.set_algorithm(options.algorithm)
    if isinstance(load, GridFunctionND):
        sol, sec = plan.solve_classes(load)
    else:
        sol, sec = plan.solve_host(load)
    return SolveReport(solution=sol, seconds_solve=sec)


@dataclass
class Field:
    """A built-in right-hand side (the device stand-in for ProblemSpec::rhs /
    exact, poisson.hpp:39-40).  kind: FIELD_*; params as sfem_cuda_fem_load."""
    kind: int
    params: Sequence[float] = ()

    @staticmethod
    def constant(value: float = 1.0) -> "Field":
        return Field(FIELD_CONSTANT, [float(value)])

    @staticmethod
    def sines(amp: float, wave_numbers: Sequence[float]) -> "Field":
        return Field(FIELD_SINES, [float(amp)] + [float(k) for k in wave_numbers])

    @staticmethod
    def case(name: str) -> "Field":
        """The reference's manufactured case by name (cases.cpp:61-78)."""
        if name not in CASE_FIELDS:
            raise Error(f"unknown case '{name}' (known: {', '.join(CASE_FIELDS)})")
        kind = CASE_FIELDS[name]
        return Field.constant(1.0) if kind == FIELD_CONSTANT else Field(kind, [])

    @property
    def has_exact(self) -> bool:
        return self.kind != FIELD_CONSTANT


def solve(spec: ProblemSpec, rhs: Field, options: Optional[SolveOptions] = None,
          ctx: Optional[Context] = None) -> SolveReport:
    """solve (poisson.hpp:86; poisson.cpp:796-808) with every step on the device:
    FEM load (seconds_load), the fused solve (seconds_solve), and on request
    the residual check and, for fields with a known solution, error_uniform.
    The solution comes back as a dense dof tensor."""
    options = options or SolveOptions()
    plan = Plan(spec, ctx)
    plan.set_algorithm(options.algorithm)
    return plan.solve_field(rhs, options.compute_residual)
