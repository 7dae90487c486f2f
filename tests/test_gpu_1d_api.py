"""The rest of the reference's 1D API surface on the device: element stencils
(apply_mass_1d / apply_stiffness_1d, grid1d.cpp:7-47), materialize_eigenvector
(spectral.cpp:238-265) and decompose's DirectRoute (eigenbasis.cpp:466-475),
against the reference itself (oracle/_ref) and its own test cases
(test_eigenbasis.cpp:40-75, 125-135)."""
import numpy as np
import pytest

from oracle import reflib

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not reflib.available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def sfem():
    import paper_1701_03967_b200 as s
    return s


@needs_ref
@pytest.mark.parametrize("n,K", [(1, 5), (2, 8), (3, 7), (4, 64), (9, 13), (9, 64), (4, 1024)])
@pytest.mark.parametrize("kind", ["mass", "stiffness"])
def test_element_stencils_match_reference(sfem, n, K, kind):
    t = sfem.SpectralTable(n, K)
    x = np.random.default_rng(n * 100 + K).uniform(-1, 1, (37, n * K - 1))
    op = sfem.APPLY_MASS if kind == "mass" else sfem.APPLY_STIFFNESS
    got = sfem.lines(t, op, x)
    want = reflib.apply_1d(kind, n, K, x)
    assert np.max(np.abs(got - want)) <= 1e-14 * max(1.0, np.max(np.abs(want)))
    # the GridFunction1D form, and in place on device lines with a padded pitch
    g = sfem.GridFunction1D.from_dof(x[3], n, K)
    f = sfem.apply_mass_1d if kind == "mass" else sfem.apply_stiffness_1d
    assert np.array_equal(f(g, t).to_dof(), got[3])
    import torch
    L, P = n * K - 1, n * K + 7
    d = torch.zeros((x.shape[0], P), dtype=torch.float64, device="cuda")
    d[:, :L] = torch.from_numpy(x)
    sfem.lines_device(t, op, x.shape[0], d.data_ptr(), P, d.data_ptr(), P)
    torch.cuda.synchronize()
    assert np.array_equal(d[:, :L].cpu().numpy(), got)


@needs_ref
@pytest.mark.parametrize("n,K", [(1, 4), (2, 3), (3, 5), (5, 4), (9, 64)])
def test_materialize_eigenvector_matches_reference_and_synthesis(sfem, n, K):
    t = sfem.SpectralTable(n, K)
    for k in range(K):
        for l in range(1, (n - 1 if k == 0 else n) + 1):
            got = sfem.materialize_eigenvector(t, k, l).to_dof()
            assert np.array_equal(got, reflib.eigenvector(n, K, k, l))
            c = sfem.CoefficientArray1D.zeros(n, K)
            c.data[c.index(k, l)] = 1.0
            # the reference's 1e-12 (absolute, K <= 5) relative to the eigenvector's size
            assert np.max(np.abs(sfem.synthesize(c, t).to_dof() - got)) <= 1e-12 * max(1.0, np.max(np.abs(got)))


def test_eigenvector_range_errors(sfem):
    t = sfem.SpectralTable(3, 4)
    with pytest.raises(sfem.Error, match="frequency out of range"):
        sfem.materialize_eigenvector(t, 4, 1)
    with pytest.raises(sfem.Error, match="branch out of range"):
        sfem.materialize_eigenvector(t, 0, 3)


@pytest.mark.parametrize("n,K", [(1, 8), (3, 7), (5, 12), (9, 64)])
def test_both_direct_routes_agree(sfem, n, K):
    """test_eigenbasis.cpp:125-135."""
    t = sfem.SpectralTable(n, K)
    g = sfem.GridFunction1D.from_dof(np.random.default_rng(30 + n + K).uniform(-1, 1, n * K - 1), n, K)
    a = sfem.decompose(g, t, sfem.DirectRoute.SPECTRAL)
    b = sfem.decompose(g, t, sfem.DirectRoute.MASS_APPLY)
    assert np.max(np.abs(a.data - b.data)) <= 1e-12


@pytest.mark.parametrize("n,K", [(2, 4), (4, 5), (9, 64)])
def test_weighted_analysis_of_mass_times_eigenvector_is_indicator(sfem, n, K):
    """test_eigenbasis.cpp:62-75, with the device mass stencil."""
    t = sfem.SpectralTable(n, K)
    for k in range(K):
        for l in range(1, (n - 1 if k == 0 else n) + 1):
            y = sfem.apply_mass_1d(sfem.materialize_eigenvector(t, k, l), t)
            c = sfem.decompose_weighted(y, t).data
            want = np.zeros_like(c)
            want[sfem.CoefficientArray1D.zeros(n, K).index(k, l)] = 1.0
            assert np.max(np.abs(c - want)) <= 1e-11


# ---- slot-major batched line API (lines::*_block, eigenbasis.hpp:66-73) ----

def _class_tiles(x, n, K):
    """dof-layout lines (count, nK-1) -> slot-major (nodal (K+1, count), interior (K(n-1), count))."""
    count, m = x.shape[0], n - 1
    nodal = np.zeros((K + 1, count))
    inter = np.zeros((K * m, count))
    for t in range(n * K - 1):
        e, c = divmod(t, n)
        if c == m:
            nodal[e + 1] = x[:, t]
        else:
            inter[e * m + c] = x[:, t]
    return nodal, inter


@needs_ref
@pytest.mark.parametrize("n,K,count", [(1, 8, 5), (2, 64, 32), (3, 7, 1), (9, 64, 32), (4, 256, 19), (5, 12, 32),
                                        (9, 114, 7), (2, 512, 40)])
def test_block_api_matches_reference_block_kernels(sfem, n, K, count):
    # the reference's own batched kernels on the same slot-major tiles
    # (decompose_weighted_block / synthesize_block, eigenbasis.cpp:248-444)
    t = sfem.SpectralTable(n, K)
    rng = np.random.default_rng(n * 1000 + K + count)
    x = rng.uniform(-1, 1, (count, n * K - 1))
    nodal, inter = _class_tiles(x, n, K)
    nodal[0] = rng.uniform(-1, 1, count)   # boundary slots are ignored by the analyses
    nodal[K] = rng.uniform(-1, 1, count)
    got = sfem.decompose_weighted_block(t, nodal, inter, count)
    want = reflib.lines("decompose_weighted_block", n, K, x).T
    assert got.shape == (n * K - 1, count)
    assert np.linalg.norm(got - want) <= 1e-11 * np.linalg.norm(want)
    # F_n on the same tiles (the reference has the per-line form only)
    got_d = sfem.decompose_weighted_block(t, nodal, inter, count, op=sfem.DECOMPOSE)
    want_d = reflib.lines("decompose", n, K, x).T
    assert np.linalg.norm(got_d - want_d) <= 1e-11 * np.linalg.norm(want_d)
    # synthesis back into class tiles: boundary slots written as zero
    c = rng.uniform(-1, 1, (count, n * K - 1))
    gn, gi = sfem.synthesize_block(t, c.T.copy(), count)
    wn, wi = _class_tiles(reflib.lines("synthesize_block", n, K, c), n, K)
    assert np.all(gn[0] == 0.0) and np.all(gn[K] == 0.0)
    assert np.linalg.norm(gn - wn) <= 1e-11 * np.linalg.norm(wn)
    if n > 1:
        assert np.linalg.norm(gi - wi) <= 1e-11 * np.linalg.norm(wi)


@pytest.mark.parametrize("n,K,count", [(9, 64, 32), (4, 256, 8), (3, 10, 5)])
def test_strided_lines_match_line_major(sfem, n, K, count):
    # the slot-major dof tile [t*count + b] and a general (pos, line) stride
    # pair give the line-major results (bitwise for the same kernel family is
    # not required: different tile shapes; 1e-13 relative)
    import torch
    t = sfem.SpectralTable(n, K)
    L = n * K - 1
    x = np.random.default_rng(L + count).uniform(-1, 1, (count, L))
    for op in (sfem.DECOMPOSE_WEIGHTED, sfem.DECOMPOSE, sfem.SYNTHESIZE):
        want = sfem.lines(t, op, x)
        d = torch.from_numpy(x.T.copy()).cuda()          # (L, count): pos_stride = count
        torch.cuda.synchronize()
        sfem.lines_strided_device(t, op, count, d.data_ptr(), d.data_ptr(), count, 1)
        torch.cuda.synchronize()
        got = d.cpu().numpy().T
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want), op
        # out of place, padded strides: position stride count + 3, line stride 1
        src = torch.zeros((L, count + 3), dtype=torch.float64, device="cuda")
        src[:, :count] = torch.from_numpy(x.T.copy())
        dst = torch.full((L, count + 3), 7.0, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        sfem.lines_strided_device(t, op, count, src.data_ptr(), dst.data_ptr(), count + 3, 1)
        torch.cuda.synchronize()
        out = dst.cpu().numpy()
        assert np.linalg.norm(out[:, :count].T - want) <= 1e-13 * np.linalg.norm(want), op
        assert np.all(out[:, count:] == 7.0)
    with pytest.raises(sfem.Error):
        sfem.lines_strided_device(t, 0, count, d.data_ptr(), d.data_ptr(), count - 1 if count > 1 else 0, 1)
