"""Device solve times of general even-order shapes with the component-major strided tiles on / off
(SFEM_MID_CM=1/0 per process): python tools/shape_survey_cm.py"""
import os
import subprocess
import sys

SHAPES = [([4, 4, 4], [32, 32, 32]), ([2, 2, 2], [128, 128, 128]), ([8, 8, 8], [32, 32, 32]), ([4, 4, 4], [128, 128, 128]),
          ([8, 8], [512, 512]), ([4, 4], [512, 512]), ([2, 2, 2], [256, 256, 256]), ([4, 4, 4], [100, 100, 100]),
          ([8, 8, 8], [48, 48, 48]), ([2, 2], [384, 384])]

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.getcwd())
    import torch
    import paper_1701_03967_b200 as sfem
    for orders, elements in SHAPES:
        spec = sfem.ProblemSpec(len(orders), [1.0] * len(orders), elements, orders, 0.5)
        plan = sfem.Plan(spec)
        shape = list(plan.extents[:-1]) + [plan.pitch]
        g = torch.Generator(device="cuda").manual_seed(1)
        d = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g) - 0.5
        x = d.clone()
        torch.cuda.synchronize()
        plan.solve_device(x.data_ptr())
        torch.cuda.synchronize()
        chk = float(x[..., : plan.extents[-1]].norm())
        plan.solve_device_timed(d.data_ptr(), 1)
        tot, ker = plan.solve_device_timed(d.data_ptr(), 5)
        print(f"n={orders[0]} K={elements[0]} dim={len(orders)} U={plan.unknowns:>10d} solve {tot:8.4f} ms kernels "
              f"{[round(k, 4) for k in ker]} checksum {chk:.15e}", flush=True)
else:
    for v in ("0", "1"):
        print(f"== SFEM_MID_CM={v}", flush=True)
        subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, SFEM_MID_CM=v), check=False)
