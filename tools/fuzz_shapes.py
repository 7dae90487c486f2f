"""Random small problems through every kernel family against the numpy oracle
(shapes drawn so that K = 64 fast kernels, tuned / general mid kernels and the
generic kernels all occur, on strided and contiguous axes, with ragged tiles).

    python tools/fuzz_shapes.py [--cases 40] [--seed 1]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402
from oracle import sfem_oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=40)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
KS = [2, 3, 5, 7, 16, 24, 32, 40, 64, 64, 64, 96, 100, 114, 128, 256, 512, 1024]
worst = 0.0
for case in range(a.cases):
    N = int(rng.integers(1, 5))
    while True:
        orders = [int(rng.integers(1, 10)) for _ in range(N)]
        elements = [int(rng.choice(KS)) for _ in range(N)]
        ext = [n * K - 1 for n, K in zip(orders, elements)]
        if all(e >= 1 for e in ext) and 2 <= int(np.prod(ext)) <= 3_000_000:
            break
    lengths = [float(rng.choice([0.5, 1.0, 2.0])) for _ in range(N)]
    shift = float(rng.choice([0.0, 0.5, 3.0]))
    spec = sfem.ProblemSpec(N, lengths, elements, orders, shift)
    f = rng.uniform(-1, 1, ext)
    u, _ = sfem.solve_dof(spec, f)
    want = O.solve_full_diagonalization(f, orders, elements, lengths, shift)
    err = float(np.linalg.norm(u - want) / np.linalg.norm(want))
    worst = max(worst, err)
    print(f"{case:3d} orders {orders} elements {elements} shift {shift}: rel-L2 {err:.2e}", flush=True)
    assert err <= 1e-11, (orders, elements)
print(f"fuzz ok: {a.cases} cases, worst rel-L2 {worst:.2e}")
