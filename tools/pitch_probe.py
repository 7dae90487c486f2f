"""Per-sweep times of one config at several caller pitches (GPU box): does a
power-of-two row pitch (1024 doubles for the C5 shapes) cost the strided
sweeps through L2 / DRAM address aliasing?

    python tools/pitch_probe.py --config c5n1 --pads 0 16 32 48
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03967_b200 as sfem  # noqa: E402
import torch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5n1")
ap.add_argument("--pads", type=int, nargs="*", default=[0, 16, 32])
a = ap.parse_args()
orders, elements, lengths, coeffs, shift, _ = bench.CONFIGS[a.config]
plan = sfem.Plan(sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs))
rows = plan.unknowns // plan.extents[-1]
for pad in a.pads:
    pitch = plan.pitch + pad
    g = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.rand(rows, pitch, dtype=torch.float64, device="cuda", generator=g) - 0.5
    x = buf.clone()
    torch.cuda.synchronize()  # the plan runs on its own non-blocking stream
    plan.solve_device(x.data_ptr(), pitch)
    torch.cuda.synchronize()
    chk = float(x[:, : plan.extents[-1]].norm())
    tot, per = plan.solve_device_timed(buf.data_ptr(), 3, pitch)
    print(f"{a.config} pitch {pitch}: solve {tot / 3 if tot > 0.15 else tot:8.3f} ms kernels {[round(v, 3) for v in per]} checksum {chk:.15e}",
          flush=True)
    del buf, x
    torch.cuda.empty_cache()
