"""CPU tests: the oracle restatement pinned against the reference's known
answers and against golden vectors produced by the reference itself."""
import math

import numpy as np
import pytest

from conftest import load_golden, rel_l2
from oracle import sfem_oracle as O
from oracle import reflib


# ---- known answers restated from the reference's own tests ----------------

def test_order1_element_matrices_exact():
    # test_element.cpp:23-31
    em = O.build_element_matrices(1)
    assert em.stiffness[0, 0] == pytest.approx(0.5, rel=1e-15)
    assert em.stiffness[0, 1] == pytest.approx(-0.5, rel=1e-15)
    assert em.mass[0, 0] == pytest.approx(2 / 3, rel=1e-15)
    assert em.mass[0, 1] == pytest.approx(1 / 3, rel=1e-15)


def test_order2_bubble_blocks():
    # test_element.cpp:33-39
    em = O.build_element_matrices(2)
    assert em.stiff.interior[0, 0] == pytest.approx(8 / 3, rel=1e-14)
    assert em.massb.interior[0, 0] == pytest.approx(16 / 15, rel=1e-14)
    assert O.interior_eigensystem(em).values[0] == pytest.approx(2.5, rel=1e-14)


def test_closed_form_interior_spectra():
    # test_element.cpp:87-99
    r133, r5 = math.sqrt(133), math.sqrt(5)
    expected = {2: [2.5], 3: [2.5, 10.5], 4: [14 - r133, 10.5, 14 + r133],
                5: [14 - r133, 30 - 9 * r5, 14 + r133, 30 + 9 * r5]}
    for n, want in expected.items():
        got = O.interior_eigensystem(O.build_element_matrices(n)).values
        assert np.allclose(got, sorted(want), rtol=1e-13, atol=0)


def test_interior_vectors_parity_and_sign():
    # test_element.cpp:101-137
    for n in range(2, 10):
        em = O.build_element_matrices(n)
        es = O.interior_eigensystem(em)
        m = n - 1
        for l in range(m):
            e = es.vectors[:, l]
            assert e @ em.massb.interior @ e == pytest.approx(1.0, rel=1e-12)
            assert np.array_equal(e, es.parity[l] * e[::-1])
            first = e[np.abs(e) > 1e-12][0]
            assert first > 0
        assert list(es.parity) == [1 if l % 2 == 0 else -1 for l in range(m)]


def test_theta_equation_order1_closed_form():
    # test_spectral.cpp:13-25
    em = O.build_element_matrices(1)
    for theta in (-0.9, -0.3, 0.0, 0.5, 0.99):
        r = O.solve_theta_equation(None, em, theta)
        assert r[0] == pytest.approx((0.5 - 0.5 * theta) / (2 / 3 + theta / 3), rel=1e-14)
    assert O.solve_theta_equation(None, em, 0.0)[0] == pytest.approx(0.75, rel=1e-14)


def test_trig_impulses():
    # test_trig.cpp:30-91
    X = O.dst1(np.array([1.0, 0.0, 0.0]))
    assert np.allclose(X, [math.sqrt(2) / 2, 1.0, math.sqrt(2) / 2], rtol=1e-15)
    for K in (2, 3, 8, 31):
        x = np.random.default_rng(K).uniform(-1, 1, K - 1)
        assert np.allclose(O.dst1(O.dst1(x)), 0.5 * K * x, rtol=1e-12, atol=1e-13)
    w = O.dst3_synthesis(np.array([1.0, 0.0]))
    assert np.allclose(w, [math.sqrt(2) / 2] * 2, rtol=1e-15)
    w = O.dct3_synthesis(np.array([0.0, 1.0]))
    assert np.allclose(w, [math.sqrt(2) / 2, -math.sqrt(2) / 2], rtol=1e-15)


def test_1d_diagonal_action_on_eigenvector_load():
    # test_poisson.cpp:90-115: load = C s  ->  u = s / (4/h^2 lambda + alpha)
    n, K, alpha = 3, 8, 1.0
    t = O.table(n, K)
    A, C = O.assemble_global_1d(n, K)
    h = 1.0 / K
    for (k, l) in ((0, 1), (3, 2)):
        c = np.zeros(n * K - 1)
        idx = l - 1 if k == 0 else (n - 1) + (k - 1) * n + (l - 1)
        c[idx] = 1.0
        s = O.synthesize(c, t)
        lam = t.interior.values[l - 1] if k == 0 else t.values[k - 1, l - 1]
        u = O.solve_full_diagonalization(C @ s, [n], [K], [1.0], alpha)
        assert np.max(np.abs(u - s / (4 / h ** 2 * lam + alpha))) <= 1e-13


def test_solve_matches_dense_kronecker():
    # test_poisson.cpp:151-160, 182-189
    rng = np.random.default_rng(3)
    for orders, elements, lengths, shift in (([1, 1], [6, 6], [1, 1], 1.0), ([2, 2], [4, 4], [1, 1], 1.0),
                                             ([3, 2], [4, 3], [1, 2], 0.0), ([2, 2, 2], [2, 2, 2], [1, 1, 1], 1.0)):
        ext = [n * K - 1 for n, K in zip(orders, elements)]
        f = rng.uniform(-1, 1, ext)
        u = O.solve_full_diagonalization(f, orders, elements, lengths, shift)
        d = O.dense_solve(f, orders, elements, lengths, shift)
        assert rel_l2(u, d) <= 1e-11


def test_roundtrips():
    # test_eigenbasis.cpp:106-123
    for n in (1, 2, 3, 5, 9):
        for K in (2, 3, 4, 8, 31):
            t = O.table(n, K)
            c = np.random.default_rng(1000 + n * 64 + K).uniform(-1, 1, n * K - 1)
            assert np.max(np.abs(O.decompose(O.synthesize(c, t), t) - c)) <= 1e-11
            g = np.random.default_rng(2000 + n * 64 + K).uniform(-1, 1, n * K - 1)
            assert np.max(np.abs(O.synthesize(O.decompose(g, t), t) - g)) <= 1e-11


def test_symbol_rejects_nonpositive():
    # test_poisson.cpp:293-309
    with pytest.raises(ValueError, match="nonpositive denominator"):
        O.scale_by_symbol(np.ones(4), [[0.5, 1.0, 2.0, 3.0]], [1.0], -1.0)


# ---- golden vectors from the reference itself ------------------------------

def test_oracle_tables_match_reference_golden():
    g = load_golden("tables")
    for key in g.files:
        if key.startswith("element/"):
            _, nn, what = key.split("/")
            em = O.build_element_matrices(int(nn[1:]))
            got = em.stiffness if what == "stiffness" else em.mass
            assert np.array_equal(got, g[key]), key
            continue
        nk, what = key.split("/")
        n, K = (int(s[1:]) for s in nk.split("_"))
        t = O.table(n, K)
        got = {"values": t.values.ravel(), "norm_sq": t.norm_sq.ravel(), "p": t.p.ravel(),
               "interior_values": t.interior.values if n > 1 else np.zeros(0),
               "interior_vectors": t.interior.vectors.ravel() if n > 1 else np.zeros(0),
               "eig_coeff": t.eigenvalues_coeff_order(), "nodal_weight": t.nodal_weight.ravel()}[what]
        assert np.array_equal(got, g[key]), key


def test_oracle_trig_matches_reference_golden():
    g = load_golden("trig")
    for K in (2, 3, 4, 5, 8, 12, 16, 64):
        p = f"trig/K{K}/"
        assert np.max(np.abs(O.dst1(g[p + "x"]) - g[p + "dst1"])) <= 1e-12
        assert np.max(np.abs(O.dst3_synthesis(g[p + "b"]) - g[p + "dst3"])) <= 1e-12
        assert np.max(np.abs(O.dct3_synthesis(g[p + "a"]) - g[p + "dct3"])) <= 1e-12


def test_oracle_lines_match_reference_golden():
    g = load_golden("lines")
    for key in [k for k in g.files if k.endswith("/in")]:
        nk = key[:-3]
        n, K = (int(s[1:]) for s in nk.split("_"))
        t = O.table(n, K)
        x = g[key]
        assert rel_l2(O.decompose_weighted(x, t), g[nk + "/decompose_weighted"]) <= 1e-13
        assert rel_l2(O.decompose(x, t), g[nk + "/decompose"]) <= 1e-13
        assert rel_l2(O.synthesize(x, t), g[nk + "/synthesize"]) <= 1e-13


def test_oracle_solves_match_reference_golden():
    g = load_golden("solves")
    for key in [k for k in g.files if k.endswith("/meta")]:
        name = key[:-5]
        meta = g[key]
        N = (len(meta) - 1) // 3
        orders = [int(v) for v in meta[:N]]
        elements = [int(v) for v in meta[N:2 * N]]
        lengths = list(meta[2 * N:3 * N])
        u = O.solve_full_diagonalization(g[name + "/load"], orders, elements, lengths, meta[-1])
        assert rel_l2(u, g[name + "/u"]) <= 1e-12, name
    u = O.solve_full_diagonalization(g["c3_small/load"], [9, 9], [8, 8], [1, 1], 1.0, coefficients=[1, 2])
    assert rel_l2(u, g["c3_small/u"]) <= 1e-12


def _meta(meta):
    N = (len(meta) - 1) // 3
    return ([int(v) for v in meta[:N]], [int(v) for v in meta[N:2 * N]], list(meta[2 * N:3 * N]), float(meta[-1]))


def test_oracle_fem_loads_match_reference_golden():
    # fem_load_average (poisson.cpp:499-569) of the manufactured cases and the config-3 sines
    g = load_golden("fem")
    names = [k[5:-5] for k in g.files if k.startswith("load/") and k.endswith("/meta")]
    assert len(names) == 5
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"load/{name}/meta"])
        if name.startswith("sines"):
            def rhs(x):
                return (9 * np.pi ** 2 + 1) * np.sin(np.pi * x[0]) * np.sin(2 * np.pi * x[1])
        else:
            rhs, _ = O.case_functions(name.split("_")[0], shift)
        assert rel_l2(O.fem_load_average(orders, elements, lengths, rhs), g[f"load/{name}"]) <= 1e-13, name


def test_oracle_operator_matches_reference_golden():
    # apply_operator (poisson.cpp:749-769) on seeded vectors
    g = load_golden("fem")
    names = [k[3:-5] for k in g.files if k.startswith("op/") and k.endswith("/meta")]
    assert len(names) == 4
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"op/{name}/meta"])
        got = O.apply_operator(g[f"op/{name}/v"], orders, elements, lengths, shift)
        assert rel_l2(got, g[f"op/{name}/Av"]) <= 1e-13, name


def test_oracle_case_solves_match_reference_golden():
    # the reference's solve() of its manufactured cases: u, residual_rel and
    # error_uniform (max_error_vs, ndgrid.cpp:80-101) restated
    g = load_golden("fem")
    names = [k[5:-5] for k in g.files if k.startswith("case/") and k.endswith("/meta")]
    assert len(names) == 3
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"case/{name}/meta"])
        rhs, exact = O.case_functions(name.split("_")[0], shift)
        load = O.fem_load_average(orders, elements, lengths, rhs)
        u = O.solve_full_diagonalization(load, orders, elements, lengths, shift)
        assert rel_l2(u, g[f"case/{name}/u"]) <= 1e-12, name
        res, err = g[f"case/{name}/residual_error"]
        Au = O.apply_operator(u, orders, elements, lengths, shift)
        assert np.abs(Au - load).max() / np.abs(load).max() <= 1e-10 and res <= 1e-10, name
        X = np.meshgrid(*O.dof_coordinates(orders, elements, lengths), indexing="ij")
        assert abs(np.abs(u - exact(X)).max() - err) <= 1e-12 * max(1.0, err), name


# ---- the compiled reference (oracle/_ref), when built here ----------------

needs_ref = pytest.mark.skipif(not reflib.available(), reason="oracle/_ref not built")


@needs_ref
def test_fftw_shim_matches_scipy_definitions():
    # FFTW r2r definitions (RODFT00/RODFT01/REDFT01) == scipy.fft dst/dct types 1/3.
    import scipy.fft as sf
    rng = np.random.default_rng(0)
    for K in (2, 3, 4, 5, 8, 12, 16, 64, 113, 114, 1024):
        x = rng.uniform(-1, 1, K - 1)
        assert np.max(np.abs(reflib.trig(0, x) - 0.5 * sf.dst(x, type=1))) <= 1e-12 * K
        b = rng.uniform(-1, 1, K)
        # plain sums of trig.hpp:3-7 (the reference rescales FFTW's kinds into these)
        j = np.arange(1, K + 1)
        direct = np.sin(np.pi * np.outer(j - 0.5, np.arange(1, K + 1)) / K) @ b
        assert np.max(np.abs(reflib.trig(1, b) - direct)) <= 1e-12 * K
        a = rng.uniform(-1, 1, K)
        direct = np.cos(np.pi * np.outer(j - 0.5, np.arange(K)) / K) @ a
        assert np.max(np.abs(reflib.trig(2, a) - direct)) <= 1e-12 * K
        # and the raw FFTW kinds equal scipy's type-1/3 definitions
        assert np.max(np.abs(2 * reflib.trig(2, a * np.r_[0.5, np.ones(K - 1)]) - sf.dct(a, type=3))) <= 1e-12 * K


@needs_ref
def test_reference_trig_invocation_counter():
    # test_eigenbasis.cpp:163-181: exactly n transforms per line operation
    for n, K in ((1, 8), (2, 5), (5, 16), (9, 8)):
        x = np.random.default_rng(n).uniform(-1, 1, (1, n * K - 1))
        for op in ("decompose_weighted", "decompose", "synthesize"):
            before = reflib.lib().sfemref_trig_invocations()
            reflib.lines(op, n, K, x)
            assert reflib.lib().sfemref_trig_invocations() - before == n


@pytest.mark.parametrize("K", [48, 64, 100, 114, 256, 1024])
def test_oracle_fast_trig_forms_match_direct_sums_and_reference(K):
    # the scipy r2r forms (K >= FAST_K) against the O(K^2) sums and against the
    # reference's own trig module (oracle/_ref: trig.cpp through the FFTW shim)
    rng = np.random.default_rng(K)
    x, b, a = rng.standard_normal(K - 1), rng.standard_normal(K), rng.standard_normal(K)
    tol = 1e-13 * K
    assert np.max(np.abs(O.dst1(x) - O.dst1(x, direct=True))) <= tol
    assert np.max(np.abs(O.dst3_synthesis(b) - O.dst3_synthesis(b, direct=True))) <= tol
    assert np.max(np.abs(O.dct3_synthesis(a) - O.dct3_synthesis(a, direct=True))) <= tol
    if reflib.available():
        assert np.max(np.abs(O.dst1(x) - reflib.trig(0, x))) <= 1e-13 * K
        assert np.max(np.abs(O.dst3_synthesis(b) - reflib.trig(1, b))) <= 1e-13 * K
        assert np.max(np.abs(O.dct3_synthesis(a) - reflib.trig(2, a))) <= 1e-13 * K


@pytest.mark.skipif(not reflib.available(), reason="oracle/_ref not built")
def test_oracle_fast_path_solves_match_reference():
    # 3-D solves whose transforms take the fast forms, against the reference
    for n, K in ((2, 64), (3, 48)):
        ext = [n * K - 1] * 3
        f = np.random.default_rng(n).uniform(-1, 1, ext)
        u = O.solve_full_diagonalization(f, [n] * 3, [K] * 3, [1.0] * 3, 0.5)
        want, _ = reflib.solve(f, [n] * 3, [K] * 3, [1.0] * 3, 0.5)
        assert rel_l2(u, want) <= 1e-12


def test_reference_cannot_solve_order1_beyond_1d():
    # documents why C5 n = 1 is checked against the restatement: the
    # reference's forward_axis computes rows = lines / row_len with row_len = 0
    # for the zero-extent interior classes of an n = 1 axis (poisson.cpp:294-296),
    # a SIGFPE.  Run in a child process so the crash cannot take pytest down.
    import subprocess
    import sys
    if not reflib.available():
        pytest.skip("oracle/_ref not built")
    code = ("import numpy as np; from oracle import reflib; "
            "reflib.solve(np.ones((7, 7)), [1, 1], [8, 8], [1.0, 1.0], 0.5)")
    import os
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       capture_output=True)
    assert r.returncode != 0
    # the restatement handles it (and matches the 1-D reference, which does run)
    f = np.random.default_rng(1).uniform(-1, 1, 7)
    want, _ = reflib.solve(f, [1], [8], [1.0], 0.5)
    assert rel_l2(O.solve_full_diagonalization(f, [1], [8], [1.0], 0.5), want) <= 1e-13
