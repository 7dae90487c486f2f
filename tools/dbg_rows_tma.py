import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1701_03967_b200 as sfem
from oracle import sfem_oracle as O
for orders, elements in (([2, 4], [5, 256]), ([4, 2], [256, 128]), ([2, 2], [8, 512])):
    spec = sfem.ProblemSpec(2, [1.0, 1.0], elements, orders, 0.5)
    f = np.random.default_rng(7).uniform(-1, 1, spec.extents())
    try:
        u, _ = sfem.solve_dof(spec, f)
        want = O.solve_full_diagonalization(f, orders, elements, [1.0, 1.0], 0.5)
        print(orders, elements, float(np.linalg.norm(u - want) / np.linalg.norm(want)), flush=True)
    except Exception as e:
        print(orders, elements, 'ERR', e, flush=True)
        break
