"""Run one device solve per bench config and report timings (no parity; the
parity tests live in tests/).  python tools/check_configs.py c1 c4 c5n4 ..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03967_b200 as sfem  # noqa: E402
import torch  # noqa: E402

names = sys.argv[1:] or sorted(bench.CONFIGS)
for name in names:
    orders, elements, lengths, coeffs, shift, desc = bench.CONFIGS[name]
    try:
        spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
        plan = sfem.Plan(spec)
        rows = plan.unknowns // plan.extents[-1]
        buf = torch.empty(rows * plan.pitch, dtype=torch.float64, device="cuda")
        buf.view(rows, plan.pitch)[:, :plan.extents[-1]].uniform_(-1, 1)
        plan.solve_device(buf.data_ptr())
        torch.cuda.synchronize()
        tot, per = plan.solve_device_timed(buf.data_ptr(), reps=3)
        print(f"{name:6s} {desc:45s} U={plan.unknowns:>11d} solve {tot:8.3f} ms  "
              f"{plan.unknowns / tot / 1e6:8.3f} Gunk/s  kernels {[round(x, 3) for x in per]}", flush=True)
        del buf
        torch.cuda.empty_cache()
    except Exception as e:  # report and continue
        print(f"{name:6s} FAILED: {e}", flush=True)
