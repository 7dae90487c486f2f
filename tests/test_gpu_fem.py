"""GPU parity of the steps either side of the solve (SURVEY.md 8(f) ranks 1
and 3), through the C-ABI: the device FEM load (fem_load_average,
poisson.cpp:471-569), operator application (apply_operator, 749-769), the
residual check of solve_with_load (785-789) and the uniform error
(max_error_vs, ndgrid.cpp:80-101), against the reference's golden vectors,
the numpy oracle and, on the GPU box, the reference's own CPU code
(oracle/_ref).

Tolerances: these are floating-point reductions of transcendental right-hand
sides (libdevice vs glibc sin/cos/exp/cosh differ by an ulp), so loads and
operator results are compared at relative L2 <= 1e-13 (1e-11 at full size)."""
import numpy as np
import pytest

from conftest import load_golden, rel_l2
from oracle import reflib
from oracle import sfem_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

needs_ref = pytest.mark.skipif(not reflib.available(), reason="oracle/_ref not shipped")


def _meta(meta):
    N = (len(meta) - 1) // 3
    return ([int(v) for v in meta[:N]], [int(v) for v in meta[N:2 * N]], list(meta[2 * N:3 * N]), float(meta[-1]))


def _plan(sfem, orders, elements, lengths, shift, coefficients=None):
    return sfem.Plan(sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coefficients))


def _to_dev(plan, x):
    d = torch.zeros(plan.padded_shape, dtype=torch.float64, device="cuda")
    d[..., :plan.extents[-1]] = torch.from_numpy(np.ascontiguousarray(x, float)).cuda()
    return d


def _to_host(plan, d):
    torch.cuda.synchronize()
    return d[..., :plan.extents[-1]].cpu().numpy()


def _device_load(sfem, plan, field):
    d = torch.full(plan.padded_shape, float("nan"), dtype=torch.float64, device="cuda")
    plan.fem_load_device(field, d.data_ptr())
    return d


def _field_for(sfem, name):
    if name.startswith("sines"):
        return sfem.Field.sines(9 * np.pi ** 2 + 1, [1.0, 2.0])
    return sfem.Field.case(name.split("_")[0])


def test_fem_load_matches_reference_golden(sfem):
    g = load_golden("fem")
    names = [k[5:-5] for k in g.files if k.startswith("load/") and k.endswith("/meta")]
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"load/{name}/meta"])
        plan = _plan(sfem, orders, elements, lengths, shift)
        d = _device_load(sfem, plan, _field_for(sfem, name))
        got = _to_host(plan, d)
        assert np.isfinite(got).all(), name
        assert rel_l2(got, g[f"load/{name}"]) <= 1e-13, name
        # padding stays zero (the whole padded tensor is written)
        if plan.pitch > plan.extents[-1]:
            assert float(d[..., plan.extents[-1]:].abs().max()) == 0.0


def test_fem_load_is_deterministic(sfem):
    plan = _plan(sfem, [9, 9], [32, 16], [1.0, 1.0], 0.0)
    for f in (sfem.Field.sines(3.0, [1.0, 2.0]), sfem.Field.case("poisson2d")):  # separable / general path
        a = _to_host(plan, _device_load(sfem, plan, f))
        b = _to_host(plan, _device_load(sfem, plan, f))
        assert np.array_equal(a, b)


@pytest.mark.parametrize("orders,elements,lengths,shift", [
    ([1], [9], [2.0], 0.0), ([9], [5], [1.0], 1.5), ([2, 5], [7, 3], [1.0, 0.5], 0.25),
    ([4, 1, 3], [3, 6, 2], [1.0, 1.0, 2.0], 0.0), ([9, 9, 9], [2, 3, 2], [1.0, 1.0, 1.0], 0.0),
    ([2, 2, 2, 2], [3, 2, 3, 2], [1.0, 1.0, 1.0, 1.0], 1.0),
])
def test_fem_load_constant_and_sines_match_oracle(sfem, orders, elements, lengths, shift):
    plan = _plan(sfem, orders, elements, lengths, shift)
    got = _to_host(plan, _device_load(sfem, plan, sfem.Field.constant(2.5)))
    want = O.fem_load_average(orders, elements, lengths, lambda x: 2.5 * np.ones_like(x[0]))
    assert rel_l2(got, want) <= 1e-13
    k = [1.0, 2.0, 3.0, 1.0][:len(orders)]
    got = _to_host(plan, _device_load(sfem, plan, sfem.Field.sines(1.7, k)))
    want = O.fem_load_average(orders, elements, lengths,
                              lambda x: 1.7 * np.prod([np.sin(k[i] * np.pi * x[i]) for i in range(len(x))], axis=0))
    assert rel_l2(got, want) <= 1e-13


def test_operator_matches_reference_golden(sfem):
    g = load_golden("fem")
    names = [k[3:-5] for k in g.files if k.startswith("op/") and k.endswith("/meta")]
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"op/{name}/meta"])
        plan = _plan(sfem, orders, elements, lengths, shift)
        v = _to_dev(plan, g[f"op/{name}/v"])
        y = torch.full_like(v, float("nan"))
        plan.apply_operator_device(v.data_ptr(), y.data_ptr())
        assert rel_l2(_to_host(plan, y), g[f"op/{name}/Av"]) <= 1e-13, name


@pytest.mark.parametrize("orders,elements,lengths,shift,coeffs", [
    ([3], [40], [1.0], 0.0, None), ([9, 2], [6, 33], [1.0, 3.0], 0.5, [1.0, 2.0]),
    ([2, 3, 4], [5, 4, 3], [1.0, 0.7, 1.3], 0.0, [0.5, 1.0, 2.0]), ([9, 9, 9], [3, 2, 4], [1.0, 1.0, 1.0], 1.0, None),
    ([1, 2, 1, 3], [4, 3, 5, 2], [1.0, 1.0, 1.0, 1.0], 0.0, None),
])
def test_operator_matches_oracle(sfem, orders, elements, lengths, shift, coeffs):
    plan = _plan(sfem, orders, elements, lengths, shift, coeffs)
    v = np.random.default_rng(5).uniform(-1, 1, plan.extents)
    d = _to_dev(plan, v)
    y = torch.zeros_like(d)
    plan.apply_operator_device(d.data_ptr(), y.data_ptr())
    assert rel_l2(_to_host(plan, y), O.apply_operator(v, orders, elements, lengths, shift, coeffs)) <= 1e-13
    # v untouched
    assert np.array_equal(_to_host(plan, d), v)


def test_operator_inverts_the_solve(sfem):
    # A (A^-1 f) == f: the solve and the operator are independent code paths.
    # Bounds 1e-10 (relative L2) / 1e-9 (max norm): the reference's own
    # residual_rel for n=9, K=8 is already 2.5e-11 (tests/golden/fem.npz
    # case/poisson2d_n9_K8) and grows with cond(A) ~ (nK)^2.
    for orders, elements, shift, coeffs in (([9, 9, 9], [8, 8, 8], 0.0, None), ([9, 9], [64, 48], 1.0, [1.0, 2.0]),
                                            ([4, 2, 1], [16, 20, 30], 0.5, None)):
        plan = _plan(sfem, orders, elements, [1.0] * len(orders), shift, coeffs)
        f = np.random.default_rng(7).uniform(-1, 1, plan.extents)
        df = _to_dev(plan, f)
        du = df.clone()
        plan.solve_device(du.data_ptr())
        y = torch.zeros_like(du)
        plan.apply_operator_device(du.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        assert rel_l2(_to_host(plan, y), f) <= 1e-10
        r = plan.residual_device(du.data_ptr(), df.data_ptr())
        want = float(np.abs(_to_host(plan, y) - f).max() / np.abs(f).max())
        assert r == pytest.approx(want, rel=1e-6, abs=1e-18)
        assert r <= 1e-9


def test_residual_and_error_of_manufactured_cases_match_reference(sfem):
    # the reference's solve(spec, {compute_residual}) of its cases: our device
    # pipeline load -> solve -> residual / error_uniform
    g = load_golden("fem")
    names = [k[5:-5] for k in g.files if k.startswith("case/") and k.endswith("/meta")]
    for name in names:
        orders, elements, lengths, shift = _meta(g[f"case/{name}/meta"])
        spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift)
        rep = sfem.solve(spec, sfem.Field.case(name.split("_")[0]), sfem.SolveOptions(compute_residual=True))
        assert rel_l2(rep.solution, g[f"case/{name}/u"]) <= 1e-11, name
        res, err = g[f"case/{name}/residual_error"]
        assert rep.residual_rel <= max(1e-10, 10 * res), name
        assert rep.error_uniform == pytest.approx(err, rel=1e-8, abs=1e-12), name
        assert rep.seconds_solve > 0 and rep.seconds_load > 0


def test_field_validation(sfem):
    plan = _plan(sfem, [2, 2], [4, 4], [1.0, 1.0], 0.0)
    d = torch.zeros(plan.padded_shape, dtype=torch.float64, device="cuda")
    with pytest.raises(sfem.Error, match="case poisson3d is 3-D"):
        plan.fem_load_device(sfem.Field.case("poisson3d"), d.data_ptr())
    with pytest.raises(sfem.Error, match="SINES needs"):
        plan.fem_load_device(sfem.Field(sfem.FIELD_SINES, [1.0]), d.data_ptr())
    with pytest.raises(sfem.Error, match="unknown case"):
        sfem.Field.case("nope")
    aniso = _plan(sfem, [2, 2], [4, 4], [1.0, 1.0], 0.0, [1.0, 2.0])
    with pytest.raises(sfem.Error, match="unit coefficients"):
        aniso.fem_load_device(sfem.Field.case("poisson2d"), d.data_ptr())
    with pytest.raises(sfem.Error, match="no closed-form"):
        plan.max_error_device(sfem.Field.constant(1.0), d.data_ptr())


@needs_ref
@pytest.mark.slow
def test_config3_load_full_size_matches_reference(sfem):
    # BASELINE config 3's load: (9 pi^2 + 1) sin(pi x) sin(2 pi y), n=9, K=1024 (84.9M dofs)
    orders, elements = [9, 9], [1024, 1024]
    plan = _plan(sfem, orders, elements, [1.0, 2 ** -0.5], 1.0)
    # the load is defined on the unit square (the lengths trick only rescales the operator)
    lplan = _plan(sfem, orders, elements, [1.0, 1.0], 1.0)
    got = _to_host(lplan, _device_load(sfem, lplan, sfem.Field.sines(9 * np.pi ** 2 + 1, [1.0, 2.0])))
    want = reflib.fem_load_sines(orders, elements, [1.0, 1.0], 9 * np.pi ** 2 + 1, [1.0, 2.0])
    assert rel_l2(got, want) <= 1e-11
    del plan


@needs_ref
def test_operator_matches_reference_cpu_at_size(sfem):
    orders, elements, lengths, shift = [9, 9, 9], [12, 10, 14], [1.0, 1.0, 1.0], 0.5
    plan = _plan(sfem, orders, elements, lengths, shift)
    v = reflib.uniform(3, int(np.prod(plan.extents))).reshape(plan.extents)
    d = _to_dev(plan, v)
    y = torch.zeros_like(d)
    plan.apply_operator_device(d.data_ptr(), y.data_ptr())
    assert rel_l2(_to_host(plan, y), reflib.apply_operator(v, orders, elements, lengths, shift)) <= 1e-12


@needs_ref
def test_residual_of_our_solve_tracks_the_reference(sfem):
    # the residual check is dominated by rounding times cond(A) (it grows like
    # K^2..K^3); ours must stay within a small factor of the reference's own
    # solve() on the same problem, and the device operator must reproduce the
    # reference's residual of the reference's solution.
    for case, orders, K in (("poisson3d", [9, 9, 9], 24), ("poisson2d", [9, 9], 256)):
        N = len(orders)
        els, L = [K] * N, [1.0] * N
        plan = _plan(sfem, orders, els, L, 0.0)
        load = reflib.fem_load_case(case, orders, els, L, 0.0)
        u_ref, r_ref, _ = reflib.solve_case(case, orders, els, L, 0.0)
        df = _to_dev(plan, load)
        du = df.clone()
        plan.solve_device(du.data_ptr())
        r_ours = plan.residual_device(du.data_ptr(), df.data_ptr())
        r_dev_of_ref = plan.residual_device(_to_dev(plan, u_ref).data_ptr(), df.data_ptr())
        assert r_ours <= 3.0 * r_ref, (case, r_ours, r_ref)
        assert r_dev_of_ref == pytest.approx(r_ref, rel=0.5), (case, r_dev_of_ref, r_ref)
