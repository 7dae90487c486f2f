"""Per-CTA phase breakdown of one solve (diagnostic build, GPU box).

    tools/variants.sh phase "-DSFEM_PHASE_TIMING=1"
    SFEM_LIB=variants/phase.so python tools/phase_times.py [--config c4]

For every sweep launch: CTAs, span, mean CTA lifetime and its split into
tile-load wait / compute / store drain (SM clocks), resident CTAs per SM and
the mean idle gap between consecutive CTAs on an SM.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03967_b200 as sfem  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--fn", default="sfem_debug_phase_records", help="export (…_mid for sweep_mid.cu)")
a = ap.parse_args()
orders, elements, lengths, coeffs, shift, _ = bench.CONFIGS[a.config]
plan = sfem.Plan(sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs))
d = torch.rand(list(plan.extents[:-1]) + [plan.pitch], dtype=torch.float64, device="cuda")
fn = getattr(sfem.lib, a.fn)
fn.restype = ctypes.c_longlong
fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
cap = 1 << 20
buf = np.zeros((cap, 12), dtype=np.uint64)
plan.solve_device(d.data_ptr())
torch.cuda.synchronize()
fn(buf.ctypes.data, cap)  # drop warm-up records
plan.solve_device(d.data_ptr())
torch.cuda.synchronize()
m = fn(buf.ctypes.data, cap)
r = buf[:m].astype(np.int64)
G0, G1, SM, KIND = 6, 7, 9, 10
r = r[np.argsort(r[:, G0])]
# split launches: a CTA of launch i+1 starts after every CTA of launch i ended
splits, end = [0], r[0, G1]
for i in range(1, m):
    if r[i, G0] > end:
        splits.append(i)
    end = max(end, r[i, G1])
splits.append(m)
for s, e in zip(splits[:-1], splits[1:]):
    x = r[s:e]
    t0, t1 = x[:, G0].min(), x[:, G1].max()
    life = x[:, G1] - x[:, G0]
    ghz = ((x[:, 5] - x[:, 0]) / np.maximum(life, 1)).mean()
    ph = [(x[:, j + 1] - x[:, j]).mean() / ghz / 1e3 for j in range(5)]
    nsm = len(np.unique(x[:, SM]))
    resid = life.sum() / ((t1 - t0) * nsm)
    print(f"kind {x[0, KIND]:2d}: {e - s:6d} CTAs, span {(t1 - t0) / 1e3:7.1f} us, life {life.mean() / 1e3:6.2f} us, "
          f"{ghz:.2f} GHz, phases(us) " + " ".join(f"{p:6.2f}" for p in ph) + f", CTAs/SM {resid:.2f}")
