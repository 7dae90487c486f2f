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
