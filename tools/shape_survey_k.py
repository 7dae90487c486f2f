"""Device solve times of the non-power-of-two-K mid kernels against the generic runtime-radix
kernels (SFEM_GENERIC=1) on the same shapes: python tools/shape_survey_k.py"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1701_03967_b200 as sfem
shapes = [([9, 9, 9], [24] * 3), ([4, 4, 4], [48] * 3), ([3, 3, 3], [100] * 3), ([2, 2, 2], [192] * 3),
          ([9, 9, 9], [40] * 3), ([5, 5, 5], [80] * 3), ([2, 2, 2], [160] * 3), ([9, 9], [1000] * 2),
          ([4, 4], [768] * 2), ([7, 7], [200] * 2), ([9, 9], [320] * 2), ([3, 3], [384] * 2), ([2, 2, 2], [96] * 3)]
for orders, elements in shapes:
    spec = sfem.ProblemSpec(len(orders), [1.0] * len(orders), elements, orders, 0.0)
    res = []
    for generic in (False, True):
        if generic:
            os.environ["SFEM_GENERIC"] = "1"
        plan = sfem.Plan(spec)
        shape = list(plan.extents[:-1]) + [plan.pitch]
        d = torch.rand(shape, dtype=torch.float64, device="cuda")
        plan.solve_device_timed(d.data_ptr(), 1)
        tot, ker = plan.solve_device_timed(d.data_ptr(), 5)
        res.append(tot)
        os.environ.pop("SFEM_GENERIC", None)
        del plan, d
    U = 1
    for o, e in zip(orders, elements):
        U *= o * e - 1
    nd = len(orders)
    print(f"n={orders[0]} K={elements[0]} dim={nd} U={U:>11d}  mid {res[0]:8.3f} ms ({U / res[0] / 1e6:6.2f} Gunk/s, "
          f"frac {(2 * nd - 1) * 16 * U / (res[0] * 1e-3) / 6.448e12:.3f})  generic {res[1]:8.3f} ms  x{res[1] / res[0]:.1f}")
