"""oracle/reflib.py -- TEST INFRASTRUCTURE: ctypes binding of oracle/_ref/libsfem_ref.so.

oracle/_ref/libsfem_ref.so is the reference's own code (compiled from
/root/reference/proj/src by oracle/Makefile, with the FFTW-API shim).  Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs use this module.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsfem_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_SO)
        L.sfemref_last_error.restype = ctypes.c_char_p
        L.sfemref_max_threads.restype = ctypes.c_int
        L.sfemref_trig_invocations.restype = ctypes.c_ulonglong
        L.sfemref_trig.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.sfemref_table.argtypes = [ctypes.c_int, ctypes.c_int] + [_dp] * 11
        L.sfemref_save_table.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        L.sfemref_load_table.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int] + [_dp] * 11
        L.sfemref_tableset_get.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int] + [_dp] * 11
        L.sfemref_apply_1d.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, _dp, _dp]
        L.sfemref_eigenvector.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        L.sfemref_element.argtypes = [ctypes.c_int, _dp, _dp]
        L.sfemref_lines.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong, _dp, _dp]
        L.sfemref_solve.argtypes = [ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                    _dp, _dp, _dp]
        L.sfemref_solve_repeat.argtypes = [ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                           _dp, _dp]
        L.sfemref_apply_operator.argtypes = [ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, _dp, _dp]
        L.sfemref_fem_load_sines.argtypes = [ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, _dp, _dp]
        L.sfemref_fem_load_case.argtypes = [ctypes.c_char_p, ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, _dp]
        L.sfemref_solve_case.argtypes = [ctypes.c_char_p, ctypes.c_int, _ip, _ip, _dp, ctypes.c_double, _dp, _dp,
                                         _dp]
        L.sfemref_uniform.argtypes = [ctypes.c_uint, ctypes.c_longlong, ctypes.c_double, ctypes.c_double, _dp]
        L.sfemref_uniform.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _chk(r):
    if r != 0:
        raise RuntimeError(lib().sfemref_last_error().decode())


def max_threads() -> int:
    return lib().sfemref_max_threads()


def uniform(seed: int, count: int, lo=-1.0, hi=1.0) -> np.ndarray:
    """std::mt19937(seed) + uniform_real_distribution(lo, hi) (test_trig.cpp:14-20)."""
    out = np.empty(count)
    lib().sfemref_uniform(seed, count, lo, hi, _p(out))
    return out


def trig(kind: int, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, float)
    y = np.empty_like(x)
    _chk(lib().sfemref_trig(kind, len(x), _p(x), _p(y)))
    return y


_TABLE_KEYS = ["theta", "half_cos", "half_sin", "values", "norm_sq", "nodal_weight", "p", "q", "interior_values",
               "interior_vectors", "eig_coeff"]


def _table_export(n: int, K: int, call) -> dict:
    m = n - 1
    out = dict(theta=np.empty(K - 1), half_cos=np.empty(K - 1), half_sin=np.empty(K - 1),
               values=np.empty((K - 1) * n), norm_sq=np.empty((K - 1) * n), nodal_weight=np.empty((K - 1) * n),
               p=np.empty(max(1, (K - 1) * n * m)), q=np.empty(max(1, (K - 1) * n * m)),
               interior_values=np.empty(max(1, m)), interior_vectors=np.empty(max(1, m * m)),
               eig_coeff=np.empty(n * K - 1))
    _chk(call(*[_p(out[k]) for k in _TABLE_KEYS]))
    for k in ("p", "q"):
        out[k] = out[k][:(K - 1) * n * m]
    out["interior_values"] = out["interior_values"][:m]
    out["interior_vectors"] = out["interior_vectors"][:m * m]
    return out


def table(n: int, K: int) -> dict:
    return _table_export(n, K, lambda *a: lib().sfemref_table(n, K, *a))


def save_table(n: int, K: int, path: str):
    """The reference's save_table (spectral.cpp:128-138) of its (n, K) table."""
    _chk(lib().sfemref_save_table(n, K, path.encode()))


def load_table(path: str, n: int, K: int) -> dict:
    """The reference's load_table (spectral.cpp:152-236)."""
    return _table_export(n, K, lambda *a: lib().sfemref_load_table(path.encode(), n, K, *a))


def tableset_get(cache_dir: str, write_cache: bool, n: int, K: int) -> dict:
    """TableSet(Double, cache_dir, write_cache).get(n, K) (poisson.cpp:49-73)."""
    return _table_export(n, K, lambda *a: lib().sfemref_tableset_get(cache_dir.encode(), int(write_cache), n, K, *a))


def apply_1d(kind: str, n: int, K: int, x: np.ndarray) -> np.ndarray:
    """apply_mass_1d / apply_stiffness_1d (grid1d.cpp:33-47) of dof-layout lines."""
    x = np.ascontiguousarray(np.atleast_2d(x), float)
    y = np.empty_like(x)
    _chk(lib().sfemref_apply_1d({"mass": 0, "stiffness": 1}[kind], n, K, x.shape[0], _p(x), _p(y)))
    return y


def eigenvector(n: int, K: int, k: int, l: int) -> np.ndarray:
    """materialize_eigenvector (spectral.cpp:238-265), dof layout."""
    y = np.empty(n * K - 1)
    _chk(lib().sfemref_eigenvector(n, K, k, l, _p(y)))
    return y


def element(n: int):
    s = np.empty((n + 1) ** 2)
    m = np.empty((n + 1) ** 2)
    _chk(lib().sfemref_element(n, _p(s), _p(m)))
    return s.reshape(n + 1, n + 1), m.reshape(n + 1, n + 1)


OPS = {"decompose_weighted": 0, "decompose": 1, "synthesize": 2, "decompose_weighted_block": 3,
       "synthesize_block": 4}


def lines(op: str, n: int, K: int, x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(np.atleast_2d(x), float)
    y = np.empty_like(x)
    _chk(lib().sfemref_lines(OPS[op], n, K, x.shape[0], _p(x), _p(y)))
    return y


def solve(load: np.ndarray, orders, elements, lengths, shift, algorithm=0, threads=0):
    """solve_with_load on a dof-layout load; returns (u, seconds_solve)."""
    load = np.ascontiguousarray(load, float)
    N = load.ndim
    u = np.empty_like(load)
    sec = np.zeros(1)
    _chk(lib().sfemref_solve(N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                             _p(np.array(lengths, float)), float(shift), algorithm, threads, _p(load), _p(u),
                             _p(sec)))
    return u, float(sec[0])


def solve_repeat(load: np.ndarray, orders, elements, lengths, shift, reps: int, threads=0):
    """`reps` solve_with_load calls of one load; each call's seconds_solve."""
    load = np.ascontiguousarray(load, float)
    N = load.ndim
    sec = np.zeros(reps)
    _chk(lib().sfemref_solve_repeat(N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                                    _p(np.array(lengths, float)), float(shift), threads, reps, _p(load), _p(sec)))
    return [float(x) for x in sec]


def apply_operator(v: np.ndarray, orders, elements, lengths, shift):
    v = np.ascontiguousarray(v, float)
    N = v.ndim
    out = np.empty_like(v)
    _chk(lib().sfemref_apply_operator(N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                                      _p(np.array(lengths, float)), float(shift), _p(v), _p(out)))
    return out


def fem_load_sines(orders, elements, lengths, amp, freq):
    N = len(orders)
    ext = [n * K - 1 for n, K in zip(orders, elements)]
    out = np.empty(ext)
    _chk(lib().sfemref_fem_load_sines(N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                                      _p(np.array(lengths, float)), float(amp), _p(np.array(freq, float)),
                                      _p(out)))
    return out


def fem_load_case(name: str, orders, elements, lengths, shift):
    """fem_load_average of a manufactured case (cases.cpp make_problem)."""
    N = len(orders)
    out = np.empty([n * K - 1 for n, K in zip(orders, elements)])
    _chk(lib().sfemref_fem_load_case(name.encode(), N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                                     _p(np.array(lengths, float)), float(shift), _p(out)))
    return out


def solve_case(name: str, orders, elements, lengths, shift):
    """The reference's solve(spec, {compute_residual}) of a manufactured case:
    (u, residual_rel, error_uniform)."""
    N = len(orders)
    u = np.empty([n * K - 1 for n, K in zip(orders, elements)])
    r = np.zeros(1)
    e = np.zeros(1)
    _chk(lib().sfemref_solve_case(name.encode(), N, (ctypes.c_int * N)(*orders), (ctypes.c_int * N)(*elements),
                                  _p(np.array(lengths, float)), float(shift), _p(u), _p(r), _p(e)))
    return u, float(r[0]), float(e[0])
