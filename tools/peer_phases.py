"""Per-rank phase times of the fused NVLink slab solve (sfem_cuda_peer_*),
P virtual ranks on ONE GPU (loopback: every rank's peer stores land in local
buffers; no NVLink, no device barrier).  Each phase is timed over all ranks
with CUDA events on the library stream and divided by P.

    python tools/peer_phases.py [--config c4] [--ranks 8] [--reps 5]
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
plans = [D.PeerPlan(spec, P, r) for r in range(P)]
D.peer_bind_loopback(plans)
f = np.random.default_rng(0).uniform(-1, 1, spec.extents())
for p in plans:
    p.scatter_x(f)
ext = torch.cuda.ExternalStream(plans[0].ctx.stream)
names = {"forward (rows + axis-1 exchange sweep)": D.PEER_FORWARD, "axis0 (fused, exchange back)": D.PEER_AXIS0,
         "inverse (axis 1 + rows)": D.PEER_INVERSE}
times = {n: [] for n in names}
torch.cuda.synchronize()
for rep in range(a.reps + 1):
    for n, ph in names.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for p in plans:
            p.phase(ph, ext.cuda_stream)
        e1.record(ext)
        torch.cuda.synchronize()
        if rep:
            times[n].append(e0.elapsed_time(e1) / P)
U = int(np.prod(spec.extents()))
per_rank = {n: round(float(np.median(v)), 4) for n, v in times.items()}
total = sum(per_rank.values())
nvl = 2 * 8 * U / P * (P - 1) / P
print(json.dumps({"config": desc, "ranks": P, "per_rank_phase_ms": per_rank, "per_rank_kernels_ms": round(total, 4),
                  "nvlink_bytes_per_rank_per_solve": nvl,
                  "nvlink_ms_at_750GBps": round(nvl / 750e9 * 1e3, 4)}))
for p in plans:
    p.close()
