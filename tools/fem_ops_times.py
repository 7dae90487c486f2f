"""Device times of the steps either side of the solve (GPU box):
FEM load (sines field), operator application and the fused residual check,
with CUDA events on the plan stream, for BASELINE configs 3 and 4.

    python tools/fem_ops_times.py [--reps 10]

Bytes per unknown (HBM, as designed): operator = 8 (read v) + 16 (write P, Q)
for the first axis, 32 (read + write P, Q) per middle axis, 24 (read P, Q,
write Q) for the last; the residual replaces the last write of Q by a read
of f.  The load writes 8 B per unknown (plus the zero fill, 8 B).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402

CONFIGS = {
    "c4": ([9, 9, 9], [64, 64, 64], [1.0, 1.0, 1.0], None, 0.0, sfem.Field.sines(29 * np.pi ** 2, [2.0, 3.0, 4.0])),
    "c3": ([9, 9], [1024, 1024], [1.0, 1.0], [1.0, 2.0], 1.0, sfem.Field.sines(9 * np.pi ** 2 + 1, [1.0, 2.0])),
}


def timed(fn, s, reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6551.7)
    for name, (orders, elements, lengths, coeffs, shift, field) in CONFIGS.items():
        spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
        plan = sfem.Plan(spec)
        s = torch.cuda.ExternalStream(plan.ctx.stream)
        f = torch.empty(plan.padded_shape, dtype=torch.float64, device="cuda")
        u = torch.empty_like(f)
        y = torch.empty_like(f)
        U = plan.unknowns
        N = len(orders)
        t_load = timed(lambda: plan.fem_load_device(field, f.data_ptr()), s, a.reps)
        u.copy_(f)
        plan.solve_device(u.data_ptr())
        t_solve = timed(lambda: plan.solve_device(u.data_ptr()), s, a.reps)
        u.copy_(f)
        plan.solve_device(u.data_ptr())
        t_op = timed(lambda: plan.apply_operator_device(u.data_ptr(), y.data_ptr()), s, a.reps)
        torch.cuda.synchronize()
        t_res = timed(lambda: plan.residual_device(u.data_ptr(), f.data_ptr()), s, max(2, a.reps // 2))
        res = plan.residual_device(u.data_ptr(), f.data_ptr())
        op_bytes = (24 + 32 * (N - 2) + 24) * U if N >= 2 else 24 * U
        print(json.dumps({
            "config": name, "unknowns": U,
            "fem_load_ms": round(t_load, 4), "fem_load_unknowns_per_s": U / (t_load * 1e-3),
            "solve_ms": round(t_solve, 4),
            "apply_operator_ms": round(t_op, 4), "apply_operator_GBps": op_bytes / (t_op * 1e-3) / 1e9,
            "apply_operator_frac_of_hbm": op_bytes / (t_op * 1e-3) / 1e9 / peak,
            "residual_ms_incl_sync": round(t_res, 4), "residual_rel": res,
        }))


if __name__ == "__main__":
    main()
