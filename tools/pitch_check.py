"""Same load solved in a tensor of the plan's pitch and of wider caller pitches: the results must agree (GPU box).
    python tools/pitch_check.py c5n4 c5n1 c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03967_b200 as sfem  # noqa: E402
import torch  # noqa: E402

plan = None
for name in sys.argv[1:] or ["c5n4"]:
    orders, elements, lengths, coeffs, shift, _ = bench.CONFIGS[name]
    spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
    last = spec.extents()[-1]
    rows = 1
    for e in spec.extents()[:-1]:
        rows *= e
    g = torch.Generator(device="cuda").manual_seed(0)
    f = torch.rand(rows, last, dtype=torch.float64, device="cuda", generator=g) - 0.5
    ref = None
    for pad, fill, fresh in ((0, 0.0, True), (0, 7.0, True), (16, 0.0, True), (16, 7.0, True), (4, 7.0, True), (0, 7.0, False), (16, 7.0, False)):
        if fresh or plan is None:
            plan = sfem.Plan(spec)
        pitch = plan.pitch + pad
        buf = torch.full((rows, pitch), fill, dtype=torch.float64, device="cuda")
        buf[:, :last] = f
        torch.cuda.synchronize()
        plan.solve_device(buf.data_ptr(), pitch)
        torch.cuda.synchronize()
        u = buf[:, :last].clone()
        npad = int((buf[:, last:] != fill).sum()) if pitch > last else 0
        if ref is None:
            ref = u
        print(f"{name} pitch {pitch} pad fill {fill} fresh plan {fresh}: |u| {float(u.norm()):.6e} rel diff vs first "
              f"{float((u - ref).norm() / ref.norm()):.3e} pad elements changed {npad}", flush=True)
        del buf, u
        torch.cuda.empty_cache()
    del f, ref, plan
    plan = None
    torch.cuda.empty_cache()
