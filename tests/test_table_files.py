"""Spectral-table files and the table cache.

Reference: save_table / load_table / build_and_save_table (spectral.cpp:81-236,
spectral.hpp:316-330) and TableSet's cache directory (poisson.cpp:49-73).
The CPU tests run the host-only entry points of the C-ABI
(sfem_cuda_table_file_build / _read) against the reference itself
(oracle/_ref: its own save_table, load_table and TableSet): our SFEM1 text
file is the reference's file byte for byte, each side reads the other's file
into the same table bit for bit, and our build equals the reference's build
bit for bit.  The GPU tests check the device path (cache directory on a
context, plans built through it, SpectralTable.load / save).
"""
import os

import numpy as np
import pytest

import paper_1701_03967_b200 as sfem
from oracle import reflib

needs_ref = pytest.mark.skipif(not reflib.available(), reason="oracle/_ref not built")

# (n, K): the orders/lengths of the five configs plus odd/small corners
CASES = [(1, 2), (1, 8), (2, 64), (3, 5), (4, 256), (9, 64), (9, 114), (6, 33)]
KEYS = ("values", "norm_sq", "p", "interior_values", "interior_vectors", "eig_coeff")


def same_bits(a: dict, b: dict):
    for k in KEYS:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        assert x.shape == y.shape, k
        assert np.array_equal(x.view(np.int64), y.view(np.int64)), k


@needs_ref
@pytest.mark.parametrize("n,K", CASES)
def test_text_file_is_the_references_byte_for_byte(tmp_path, n, K):
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    sfem.build_and_save_table(n, K, str(ours), sfem.TABLE_TEXT)
    reflib.save_table(n, K, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()


@needs_ref
@pytest.mark.parametrize("n,K", CASES)
def test_build_and_cross_loads_match_reference_bitwise(tmp_path, n, K):
    ref = reflib.table(n, K)
    # our build (written losslessly as binary, read back) == the reference's build
    sfem.build_and_save_table(n, K, str(tmp_path / "t.bin"), sfem.TABLE_BINARY)
    same_bits(sfem.read_table_file(str(tmp_path / "t.bin"), n, K), ref)
    # we read the reference's text file, the reference reads ours
    reflib.save_table(n, K, str(tmp_path / "ref.txt"))
    same_bits(sfem.read_table_file(str(tmp_path / "ref.txt"), n, K), ref)
    sfem.build_and_save_table(n, K, str(tmp_path / "ours.txt"), sfem.TABLE_TEXT)
    theirs = reflib.load_table(str(tmp_path / "ours.txt"), n, K)
    same_bits(theirs, ref)
    # and the derived data the reference rebuilds after a load match its built table
    for k in ("theta", "half_cos", "half_sin", "nodal_weight", "q"):
        assert np.array_equal(theirs[k], ref[k]), k


@needs_ref
def test_reference_tableset_uses_our_cache_entry(tmp_path):
    """A cache directory we fill (text format, the reference's file name) is what the reference's
    TableSet(cache_dir) loads; a corrupt entry makes it rebuild, as ours does."""
    n, K = 9, 24
    sfem.build_and_save_table(n, K, str(tmp_path / f"sfem_table_n{n}_K{K}.txt"), sfem.TABLE_TEXT)
    same_bits(reflib.tableset_get(str(tmp_path), False, n, K), reflib.table(n, K))
    (tmp_path / f"sfem_table_n{n}_K{K}.txt").write_text("SFEM1 9 24 17\n0 1 garbage\n")
    same_bits(reflib.tableset_get(str(tmp_path), False, n, K), reflib.table(n, K))


def test_binary_round_trip_is_exact(tmp_path):
    n, K = 5, 40
    sfem.build_and_save_table(n, K, str(tmp_path / "a.bin"), sfem.TABLE_BINARY)
    sfem.build_and_save_table(n, K, str(tmp_path / "a.txt"), sfem.TABLE_TEXT)
    same_bits(sfem.read_table_file(str(tmp_path / "a.bin"), n, K), sfem.read_table_file(str(tmp_path / "a.txt"), n, K))
    raw = (tmp_path / "a.bin").read_bytes()
    assert raw[:6] == b"SFEMB1"
    # header (32 B) + primaries + checksum
    m = n - 1
    count = m + m * m + 2 * (K - 1) * n + (K - 1) * n * m
    assert len(raw) == 32 + 8 * count + 8


def _err(fn):
    with pytest.raises(sfem.Error) as e:
        fn()
    return str(e.value)


@needs_ref
def test_errors_follow_load_table(tmp_path):
    n, K = 3, 12
    txt, binf = str(tmp_path / "t.txt"), str(tmp_path / "t.bin")
    sfem.build_and_save_table(n, K, txt, sfem.TABLE_TEXT)
    sfem.build_and_save_table(n, K, binf, sfem.TABLE_BINARY)
    want = "load_table: file holds order 3, elements 12 but order 3, elements 13 were requested"
    assert _err(lambda: sfem.read_table_file(txt, n, K + 1)) == want
    assert _err(lambda: sfem.read_table_file(binf, n, K + 1)) == want
    with pytest.raises(RuntimeError, match="file holds order 3, elements 12"):
        reflib.load_table(txt, n, K + 1)
    assert "cannot open" in _err(lambda: sfem.read_table_file(str(tmp_path / "none.txt"), n, K))
    # truncated text, bad magic, trailing data
    body = open(txt).read()
    open(txt, "w").write(body[: len(body) // 2])
    assert "truncated" in _err(lambda: sfem.read_table_file(txt, n, K))
    open(txt, "w").write("SFEM9" + body[5:])
    assert _err(lambda: sfem.read_table_file(txt, n, K)).startswith("load_table: unsupported format 'SFEM9'")
    open(txt, "w").write(body + "1 1 0.5\n")
    assert "unexpected trailing data" in _err(lambda: sfem.read_table_file(txt, n, K))
    # binary: one flipped payload bit, a truncated payload
    raw = bytearray(open(binf, "rb").read())
    raw[100] ^= 1
    open(binf, "wb").write(bytes(raw))
    assert "checksum mismatch" in _err(lambda: sfem.read_table_file(binf, n, K))
    open(binf, "wb").write(bytes(raw[:-16]))
    assert "truncated or corrupt payload" in _err(lambda: sfem.read_table_file(binf, n, K))


def test_large_table_build_is_parallel_and_fast(tmp_path):
    """Config 2's table (n=4, K=4096) builds, writes and re-reads in a few seconds (the reference
    builds frequency by frequency on one thread, spectral.hpp:228-277)."""
    import time
    t0 = time.perf_counter()
    sfem.build_and_save_table(4, 4096, str(tmp_path / "c2.bin"), sfem.TABLE_BINARY)
    t1 = time.perf_counter()
    t = sfem.read_table_file(str(tmp_path / "c2.bin"), 4, 4096)
    t2 = time.perf_counter()
    assert t["values"].shape == (4095 * 4,)
    assert t1 - t0 < 30 and t2 - t1 < 5


# ---------------------------------------------------------------------------
# device path
# ---------------------------------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", [sfem.TABLE_TEXT, sfem.TABLE_BINARY])
def test_device_table_save_load_transforms_identically(tmp_path, fmt):
    n, K = 9, 64
    t = sfem.SpectralTable(n, K)
    path = str(tmp_path / "t.tab")
    t.save(path, fmt)
    t2 = sfem.SpectralTable.load(path, n, K)
    same_bits(t.export(), t2.export())
    x = np.random.default_rng(3).standard_normal((16, n * K - 1))
    for op in (sfem.DECOMPOSE_WEIGHTED, sfem.DECOMPOSE, sfem.SYNTHESIZE):
        assert np.array_equal(sfem.lines(t, op, x), sfem.lines(t2, op, x))
    if fmt == sfem.TABLE_TEXT and reflib.available():
        reflib.save_table(n, K, str(tmp_path / "ref.txt"))
        assert open(path, "rb").read() == open(str(tmp_path / "ref.txt"), "rb").read()


@pytest.mark.gpu
def test_context_cache_feeds_plans(tmp_path):
    """TableSet(cache_dir, write_cache): the first context builds and writes the entries, a second
    context loads them (no rebuild), and a plan built on it solves bit for bit like an uncached one."""
    spec = sfem.ProblemSpec(2, [1.0, 1.0], [24, 20], [4, 3], 0.5)
    f = np.random.default_rng(0).uniform(-1, 1, spec.extents())
    want, _ = sfem.solve_dof(spec, f)
    c1 = sfem.Context(0)
    sfem.TableSet(c1, cache_dir=str(tmp_path), write_cache=True, binary=True)
    u1, _ = sfem.solve_dof(spec, f, ctx=c1)
    assert sorted(os.listdir(tmp_path)) == ["sfem_table_n3_K20.bin", "sfem_table_n4_K24.bin"]
    stamp = {p: os.stat(tmp_path / p).st_mtime_ns for p in os.listdir(tmp_path)}
    c2 = sfem.Context(0)
    ts = sfem.TableSet(c2, cache_dir=str(tmp_path), write_cache=True)
    u2, _ = sfem.solve_dof(spec, f, ctx=c2)
    assert {p: os.stat(tmp_path / p).st_mtime_ns for p in os.listdir(tmp_path)} == stamp
    assert np.array_equal(u1, want) and np.array_equal(u2, want)
    same_bits(ts.get(4, 24).export(), sfem.SpectralTable(4, 24).export())
