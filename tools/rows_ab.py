"""A/B of the fused last-axis kernels on C4 (and other K = 64 3-D shapes):
per-sweep CUDA-event times with the warp-local kernel (default) and the
block-synchronous one (SFEM_ROWS_V1=1), plus a bitwise comparison of the
two solutions."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402


def run(orders, reps=10):
    spec = sfem.ProblemSpec(3, [1.0] * 3, [64] * 3, orders, 0.0)
    plan = sfem.Plan(spec)
    ext = plan.extents
    rows = plan.unknowns // ext[-1]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)
    base = torch.rand(rows, plan.pitch, dtype=torch.float64, device="cuda", generator=gen)
    base[:, ext[-1]:] = 0
    out = {}
    for v1 in ("0", "1"):
        os.environ["SFEM_ROWS_V1"] = v1
        buf = base.clone()
        torch.cuda.synchronize()  # the plan runs on its context stream
        plan.solve_device(buf.data_ptr())
        torch.cuda.synchronize()
        sol = buf.clone()
        _, kern = plan.solve_device_timed(buf.data_ptr(), reps=reps)
        out[v1] = (sol, kern)
    same = torch.equal(out["0"][0], out["1"][0])
    diff = float((out["0"][0] - out["1"][0]).abs().max())
    print(f"orders {orders}: new {[round(x, 4) for x in out['0'][1]]}  v1 {[round(x, 4) for x in out['1'][1]]}  "
          f"same bits {same} maxdiff {diff:.2e}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "once":  # one solve per kernel (for ncu)
        spec = sfem.ProblemSpec(3, [1.0] * 3, [64] * 3, [9, 9, 9], 0.0)
        plan = sfem.Plan(spec)
        buf = torch.zeros(plan.unknowns // plan.extents[-1], plan.pitch, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        for v1 in ("0", "1"):
            os.environ["SFEM_ROWS_V1"] = v1
            plan.solve_device(buf.data_ptr())
            torch.cuda.synchronize()
        sys.exit(0)
    for o in ([9, 9, 9], [5, 5, 5], [2, 2, 2], [4, 4, 4], [7, 7, 7]):
        run(o)
