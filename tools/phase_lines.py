"""Per-CTA phase breakdown of one 1D line operation (diagnostic build):
    tools/variant_one.sh phase_mid sweep_mid "-DSFEM_PHASE_TIMING=1"
    SFEM_LIB=variants/phase_mid.so python tools/phase_lines.py [--n 4 --K 4096 --count 4096 --op 0]
Phases (us): tile load | forward fill+FFT+post | mix | inverse fill+FFT+post | store."""
import argparse
import ctypes
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
ap.add_argument("--op", type=int, default=0)
a = ap.parse_args()
t = sfem.SpectralTable(a.n, a.K)
L = a.n * a.K - 1
x = torch.randn(a.count, L, dtype=torch.float64, device="cuda")
fn = sfem.lib.sfem_debug_phase_records_mid
fn.restype = ctypes.c_longlong
fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
cap = 1 << 20
buf = np.zeros((cap, 12), dtype=np.uint64)
torch.cuda.synchronize()
sfem.lines_device(t, a.op, a.count, x.data_ptr(), L, x.data_ptr(), L)
torch.cuda.synchronize()
fn(buf.ctypes.data, cap)
sfem.lines_device(t, a.op, a.count, x.data_ptr(), L, x.data_ptr(), L)
torch.cuda.synchronize()
m = fn(buf.ctypes.data, cap)
r = buf[:m].astype(np.int64)
life = r[:, 7] - r[:, 6]
ghz = ((r[:, 5] - r[:, 0]) / np.maximum(life, 1)).mean()
ph = [(r[:, j + 1] - r[:, j]).mean() / ghz / 1e3 for j in range(5)]
span = (r[:, 7].max() - r[:, 6].min()) / 1e3
print(f"n={a.n} K={a.K} op={a.op}: {m} CTAs, span {span:.1f} us, life {life.mean() / 1e3:.2f} us, {ghz:.2f} GHz, "
      "phases(us) " + " ".join(f"{p:6.2f}" for p in ph))
