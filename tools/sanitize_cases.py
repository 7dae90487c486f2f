"""Small solves that exercise every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Each case is
checked against the numpy oracle so a sanitizer run also says the results
were right.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402
from oracle import sfem_oracle as O  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def solve_case(name, orders, elements, shift=0.0):
    N = len(orders)
    spec = sfem.ProblemSpec(N, [1.0] * N, elements, orders, shift)
    f = np.random.default_rng(7).uniform(-1, 1, spec.extents())
    u, _ = sfem.solve_dof(spec, f)
    want = O.solve_full_diagonalization(f, orders, elements, [1.0] * N, shift)
    e = rel(u, want)
    print(f"{name}: orders {orders} elements {elements} rel-L2 {e:.2e}", flush=True)
    assert e <= 1e-11, name


def lines_case(name, n, K, count):
    t = sfem.SpectralTable(n, K)
    ot = O.table(n, K)
    x = np.random.default_rng(3).standard_normal((count, n * K - 1))
    for op, fn in ((sfem.DECOMPOSE_WEIGHTED, O.decompose_weighted), (sfem.DECOMPOSE, O.decompose),
                   (sfem.SYNTHESIZE, O.synthesize)):
        e = rel(sfem.lines(t, op, x), fn(x, ot))
        print(f"{name}: n={n} K={K} op {op} rel-L2 {e:.2e}", flush=True)
        assert e <= 1e-11, name


def peer_case(name, P):
    from paper_1701_03967_b200 import dist as D
    spec = sfem.ProblemSpec(3, [1.0] * 3, [64, 64, 4], [2, 2, 3], 0.25)
    f = np.random.default_rng(4).uniform(-1, 1, spec.extents())
    want, _ = sfem.solve_dof(spec, f)
    plans = [D.PeerPlan(spec, P, r) for r in range(P)]
    D.peer_bind_loopback(plans)
    for p in plans:
        p.scatter_x(f)
    D.peer_solve_loopback(plans)
    got = np.concatenate([p.gather_x() for p in plans], axis=0)
    e = rel(got, want)
    print(f"{name}: peer loopback P={P} rel-L2 {e:.2e}", flush=True)
    assert e <= 1e-12
    for p in plans:
        p.close()


CASES = {
    # K = 64 register-FFT kernels: TMA strided sweeps, blocked 3-D schedule, fused bulk-row sweep
    "fast3d": lambda: solve_case("fast3d", [2, 3, 2], [64, 64, 64]),
    "fast2d": lambda: solve_case("fast2d", [9, 9], [64, 64]),
    # compile-time mid kernels (cp.async tiles, Stockham passes)
    "mid2d": lambda: solve_case("mid2d", [4, 2], [256, 128], 0.5),
    "mid3d": lambda: solve_case("mid3d", [2, 1, 3], [32, 128, 16], 0.5),
    # component-major strided tiles by 5-D tensor copies (n = 2 / K = 512 and n = 4 / K = 256), ragged last axis
    "midcm3d": lambda: solve_case("midcm3d", [2, 4, 3], [512, 256, 4], 0.5),
    # runtime-radix generic kernels
    "generic": lambda: solve_case("generic", [3, 2], [14, 22]),
    # 1D line API (persistent K = 64 kernel, mid kernel, generic)
    "lines64": lambda: lines_case("lines64", 9, 64, 5),
    "lines256": lambda: lines_case("lines256", 4, 256, 3),
    "lines4096": lambda: lines_case("lines4096", 4, 4096, 2),
    # fused peer-store exchange (loopback, 2 virtual ranks)
    "peer": lambda: peer_case("peer", 2),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
    print("sanitize cases ok:", " ".join(names))
