"""Regenerate the golden fixtures in tests/golden/ from the reference itself.

Runs the reference's own code (oracle/_ref/libsfem_ref.so, built by
`make -C oracle` from /root/reference/proj/src with the FFTW-API shim) on
seeded inputs drawn with the reference's fixture generator (std::mt19937 +
uniform_real_distribution(-1, 1), test_trig.cpp:14-20).  Needs
/root/reference (this container); the fixtures travel, the reference does not.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import reflib as R  # noqa: E402

TRIG_K = [2, 3, 4, 5, 8, 12, 16, 64]
TABLES = [(1, 4), (2, 2), (2, 64), (3, 4), (4, 16), (5, 8), (9, 8), (9, 64), (4, 7), (1, 1024)]
LINE_N = [1, 2, 3, 5, 9]
LINE_K = [2, 3, 4, 8, 31, 64]
SOLVES = {
    # name: (orders, elements, lengths, shift, seed)
    "c1_2d_n2_K64": ([2, 2], [64, 64], [1.0, 1.0], 0.0, 0),
    "2d_mixed": ([3, 2], [4, 5], [1.0, 2.0], 1.0, 11),
    "3d_n2_K4": ([2, 2, 2], [4, 4, 4], [1.0, 1.0, 1.0], 0.5, 12),
    "3d_mixed": ([1, 2, 3], [3, 4, 5], [1.0, 1.5, 0.75], 0.0, 13),
    "1d_n3_K16": ([3], [16], [1.0], 1.0, 14),
    "2d_n9_K8_aniso": ([9, 9], [8, 8], [1.0, 2 ** -0.5], 1.0, 15),
    "3d_n9_small": ([9, 9, 9], [2, 3, 2], [1.0, 1.0, 1.0], 0.0, 16),
    "2d_n4_K7": ([4, 4], [7, 7], [1.0, 1.0], 0.5, 17),
}

# (name, case, orders, elements, lengths, shift)
FEM_LOADS = [
    ("sin1d_n4_K6", "sin1d", [4], [6], [1.0], 1.0),
    ("poisson2d_n3n2", "poisson2d", [3, 2], [5, 4], [1.0, 1.3], 0.5),
    ("poisson3d_n2n3n2", "poisson3d", [2, 3, 2], [3, 2, 4], [1.0, 1.0, 1.0], 0.25),
    ("constant2d_n9", "constant2d", [9, 9], [3, 2], [1.0, 1.0], 0.0),
    ("sines_c3_small", "sines", [9, 9], [8, 8], [1.0, 1.0], 0.0),
]
OPERATORS = {
    "1d_n5_K7": ([5], [7], [1.0], 0.75, 21),
    "2d_mixed": ([3, 2], [5, 4], [1.0, 1.3], 0.5, 22),
    "3d_mixed": ([2, 9, 1], [3, 2, 4], [1.0, 0.5, 2.0], 0.0, 23),
    "2d_n9_K8": ([9, 9], [8, 8], [1.0, 1.0], 1.0, 24),
}
CASE_SOLVES = [
    ("sin1d_n4_K6", "sin1d", [4], [6], [1.0], 1.0),
    ("poisson2d_n9_K8", "poisson2d", [9, 9], [8, 8], [1.0, 1.0], 0.0),
    ("poisson3d_n3_K4", "poisson3d", [3, 3, 3], [4, 4, 4], [1.0, 1.0, 1.0], 0.5),
]


def main():
    out = {}
    for K in TRIG_K:
        x = R.uniform(3 * K, K - 1)
        b = R.uniform(5 * K, K)
        a = R.uniform(7 * K, K)
        out[f"trig/K{K}/x"] = x
        out[f"trig/K{K}/dst1"] = R.trig(0, x)
        out[f"trig/K{K}/b"] = b
        out[f"trig/K{K}/dst3"] = R.trig(1, b)
        out[f"trig/K{K}/a"] = a
        out[f"trig/K{K}/dct3"] = R.trig(2, a)
    np.savez_compressed(os.path.join(HERE, "trig.npz"), **out)

    out = {}
    for n, K in TABLES:
        t = R.table(n, K)
        for k in ("values", "norm_sq", "p", "interior_values", "interior_vectors", "eig_coeff", "nodal_weight"):
            out[f"n{n}_K{K}/{k}"] = t[k]
    for n in range(1, 10):
        s, m = R.element(n)
        out[f"element/n{n}/stiffness"] = s
        out[f"element/n{n}/mass"] = m
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)

    out = {}
    for n in LINE_N:
        for K in LINE_K:
            L = n * K - 1
            x = R.uniform(1000 + n * 64 + K, 2 * L).reshape(2, L)
            key = f"n{n}_K{K}"
            out[key + "/in"] = x
            for op in ("decompose_weighted", "decompose", "synthesize"):
                out[key + "/" + op] = R.lines(op, n, K, x)
    np.savez_compressed(os.path.join(HERE, "lines.npz"), **out)

    out = {}
    for name, (orders, elements, lengths, shift, seed) in SOLVES.items():
        ext = [n * K - 1 for n, K in zip(orders, elements)]
        load = R.uniform(seed, int(np.prod(ext))).reshape(ext)
        u, _ = R.solve(load, orders, elements, lengths, shift)
        out[name + "/load"] = load
        out[name + "/u"] = u
        out[name + "/meta"] = np.array(orders + elements + lengths + [shift], float)
    # config-3 style: FEM load of (9 pi^2 + 1) sin(pi x) sin(2 pi y) on the unit
    # square + 1e-3 U[-1,1], operator -(u_xx + 2 u_yy) + u == lengths (1, 1/sqrt 2)
    orders, elements = [9, 9], [8, 8]
    load = R.fem_load_sines(orders, elements, [1.0, 1.0], 9 * np.pi ** 2 + 1, [1.0, 2.0])
    load = load + 1e-3 * R.uniform(0, load.size).reshape(load.shape)
    u, _ = R.solve(load, orders, elements, [1.0, 2 ** -0.5], 1.0)
    out["c3_small/load"] = load
    out["c3_small/u"] = u
    np.savez_compressed(os.path.join(HERE, "solves.npz"), **out)
    # the steps either side of the solve: FEM loads of the
    # manufactured cases / the config-3 sines, operator applications, and the
    # reference's end-to-end solve() of the cases (residual, uniform error)
    out = {}
    for name, case, orders, elements, lengths, shift in FEM_LOADS:
        if case == "sines":
            load = R.fem_load_sines(orders, elements, lengths, 9 * np.pi ** 2 + 1, [1.0, 2.0])
        else:
            load = R.fem_load_case(case, orders, elements, lengths, shift)
        out[f"load/{name}"] = load
        out[f"load/{name}/meta"] = np.array(orders + elements + lengths + [shift], float)
    for name, (orders, elements, lengths, shift, seed) in OPERATORS.items():
        ext = [n * K - 1 for n, K in zip(orders, elements)]
        v = R.uniform(seed, int(np.prod(ext))).reshape(ext)
        out[f"op/{name}/v"] = v
        out[f"op/{name}/Av"] = R.apply_operator(v, orders, elements, lengths, shift)
        out[f"op/{name}/meta"] = np.array(orders + elements + lengths + [shift], float)
    for name, case, orders, elements, lengths, shift in CASE_SOLVES:
        u, res, err = R.solve_case(case, orders, elements, lengths, shift)
        out[f"case/{name}/u"] = u
        out[f"case/{name}/residual_error"] = np.array([res, err])
        out[f"case/{name}/meta"] = np.array(orders + elements + lengths + [shift], float)
    np.savez_compressed(os.path.join(HERE, "fem.npz"), **out)
    for f in ("trig", "tables", "lines", "solves", "fem"):
        print(f, os.path.getsize(os.path.join(HERE, f + ".npz")))


if __name__ == "__main__":
    main()
