"""Small driver for ncu / launch lists: one plan, `--solves` device solves.

    python tools/profile_solve.py --config c4 --solves 2
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (CONFIGS)
import paper_1701_03967_b200 as sfem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--solves", type=int, default=2)
a = ap.parse_args()
orders, elements, lengths, coeffs, shift, _ = bench.CONFIGS[a.config]
spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
plan = sfem.Plan(spec)
f = np.random.default_rng(0).uniform(-1, 1, plan.extents)
for _ in range(a.solves):
    u, sec = plan.solve_host(f)
print(f"{a.config}: {plan.unknowns} unknowns, last solve {sec * 1e3:.3f} ms, |u| {np.linalg.norm(u):.6e}")
