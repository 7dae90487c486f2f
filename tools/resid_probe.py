import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1701_03967_b200 as sfem
from oracle import reflib as R
for case, orders, K, shift in (("poisson3d", [9, 9, 9], 24, 0.0), ("poisson2d", [9, 9], 256, 0.0)):
    N = len(orders)
    els = [K] * N
    L = [1.0] * N
    spec = sfem.ProblemSpec(N, L, els, orders, shift)
    plan = sfem.Plan(spec)
    load = R.fem_load_case(case, orders, els, L, shift)
    u_ref, r_ref, e_ref = R.solve_case(case, orders, els, L, shift)
    def dev(x):
        d = torch.zeros(plan.padded_shape, dtype=torch.float64, device="cuda")
        d[..., :plan.extents[-1]] = torch.from_numpy(x).cuda()
        return d
    df = dev(load)
    du = df.clone()
    plan.solve_device(du.data_ptr())
    torch.cuda.synchronize()
    u_gpu = du[..., :plan.extents[-1]].cpu().numpy()
    r_gg = plan.residual_device(du.data_ptr(), df.data_ptr())
    dur = dev(u_ref)
    r_rg = plan.residual_device(dur.data_ptr(), df.data_ptr())
    Au = R.apply_operator(u_gpu, orders, els, L, shift)
    r_gr = np.abs(Au - load).max() / np.abs(load).max()
    Au2 = R.apply_operator(u_ref, orders, els, L, shift)
    r_rr = np.abs(Au2 - load).max() / np.abs(load).max()
    print(case, K, "ref solve+ref op", r_rr, "(reported", r_ref, ") ref solve+gpu op", r_rg,
          "gpu solve+ref op", r_gr, "gpu solve+gpu op", r_gg,
          "u diff max", np.abs(u_gpu - u_ref).max() / np.abs(u_ref).max())
