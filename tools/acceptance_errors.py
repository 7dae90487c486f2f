"""Mesh-uniform errors of the reference's manufactured cases through the device
path, next to the paper's table entries the reference's acceptance test pins
(acceptance_main.cpp:167-168, 213-214).  python tools/acceptance_errors.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402

ROWS = [("poisson2d", 1, 64, 1.6e-3), ("poisson2d", 2, 16, 1.0e-4), ("poisson2d", 3, 32, 2.6e-6),
        ("poisson2d", 5, 64, 1.3e-11), ("poisson2d", 9, 4, 4.3e-9), ("poisson3d", 2, 16, 8.4e-4),
        ("poisson3d", 5, 16, 5.1e-7), ("poisson3d", 9, 8, 1.4e-10)]
print(f"{'case':10s} {'n':>2s} {'K':>4s} {'error (ours)':>13s} {'paper':>9s} {'ratio':>6s} {'load ms':>8s} {'solve ms':>9s}")
for name, n, K, paper in ROWS:
    dim = 2 if name == "poisson2d" else 3
    spec = sfem.ProblemSpec(dim, [1.0] * dim, [K] * dim, [n] * dim, 1.0)
    r = sfem.solve(spec, sfem.Field.case(name), sfem.SolveOptions(compute_residual=True))
    print(f"{name:10s} {n:2d} {K:4d} {r.error_uniform:13.3e} {paper:9.1e} {r.error_uniform / paper:6.2f} "
          f"{r.seconds_load * 1e3:8.3f} {r.seconds_solve * 1e3:9.3f}")
