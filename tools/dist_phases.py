"""Per-rank phase times of the slab-decomposed solve, P virtual ranks on ONE
GPU (loopback exchange by device copies).  Each rank's kernels are timed with
CUDA events on the library stream, one phase at a time; the all-to-all is not
timed here (NVLink is not available on a one-GPU box) -- its volume is printed.

    python tools/dist_phases.py [--config c4] [--ranks 8] [--reps 5]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03967_b200 as sfem  # noqa: E402
from paper_1701_03967_b200 import dist as D  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
orders, elements, lengths, coeffs, shift, desc = bench.CONFIGS[a.config]
spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
P = a.ranks
plans = [D.DistPlan(spec, P, r) for r in range(P)]
bufs = [D.allocate(p) for p in plans]
ext = torch.cuda.ExternalStream(plans[0].ctx.stream)
st = ext.cuda_stream
names = ["forward_local", "pack1", "unpack1", "axis0", "pack2", "unpack2", "inverse_local"]
times = {n: [] for n in names}
with torch.cuda.stream(ext):
    for x, _, _, _ in bufs:
        x.uniform_(-1, 1)
    for rep in range(a.reps + 1):
        for n in names:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            for p, (x, buf_a, buf_b, y) in zip(plans, bufs):
                buf = buf_a if n in ("forward_local", "pack1", "unpack2", "inverse_local") else buf_b
                p.phase(n, x.data_ptr(), y.data_ptr(), buf.data_ptr(), st)
            e1.record(ext)
            torch.cuda.synchronize()
            if rep:
                times[n].append(e0.elapsed_time(e1) / P)  # mean per rank
U = int(np.prod(spec.extents()))
per_rank = {n: round(float(np.median(v)), 4) for n, v in times.items()}
total = sum(per_rank.values())
a2a = 2 * 8 * sum(c for i, c in enumerate(plans[0].send_counts) if i != 0)
single = bench.CONFIGS[a.config]
print(json.dumps({"config": desc, "ranks": P, "per_rank_phase_ms": per_rank, "per_rank_kernels_ms": round(total, 4),
                  "all_to_all_bytes_per_rank_per_solve": a2a,
                  "fused_axis0_on_exchange_buffer": plans[0].y_elems == 0}))
