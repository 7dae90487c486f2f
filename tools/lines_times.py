"""Device time of the 1D line operations (C2: n=4, K=4096, 4096 lines).

    python tools/lines_times.py [--n 4 --K 4096 --count 4096]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03967_b200 as sfem  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--count", type=int, default=4096)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
t = sfem.SpectralTable(a.n, a.K)
L = a.n * a.K - 1
x = torch.randn(a.count, L, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ts = torch.cuda.Stream()  # a real stream handle (0 would mean the library's own stream)
st = ts.cuda_stream
torch.cuda.synchronize()
for op in (0, 1, 2):
    sfem.lines_device(t, op, a.count, x.data_ptr(), L, y.data_ptr(), L, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ts)
    for _ in range(a.reps):
        sfem.lines_device(t, op, a.count, x.data_ptr(), L, y.data_ptr(), L, st)
    e1.record(ts)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    gbs = 16.0 * a.count * L / (ms * 1e-3) / 1e9
    print(f"n={a.n} K={a.K} count={a.count} op={op}: {ms:.3f} ms, {gbs:.1f} GB/s algorithmic")
