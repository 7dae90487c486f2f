"""Device solve times for shapes outside the BASELINE configs (which kernel family serves them and how
fast): python tools/shape_survey.py"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1701_03967_b200 as sfem
shapes = [([9,9,9],[32,32,32]), ([4,4,4],[32,32,32]), ([2,2,2],[128,128,128]), ([9,9],[128,128]), ([9,9,9],[16,16,16]), ([3,3,3],[100,100,100]), ([5,5,5],[64,64,64]), ([9,9,9],[128,128,128]), ([6,6,6],[64,64,64]), ([7,7,7],[64,64,64]), ([8,8,8],[64,64,64]), ([4,4],[1024,1024]), ([8,8],[1024,1024]), ([2,2],[2048,2048]), ([5,5],[2048,2048])]
for orders, elements in shapes:
    spec = sfem.ProblemSpec(len(orders), [1.0]*len(orders), elements, orders, 0.0)
    plan = sfem.Plan(spec)
    shape = list(plan.extents[:-1]) + [plan.pitch]
    d = torch.rand(shape, dtype=torch.float64, device="cuda")
    plan.solve_device_timed(d.data_ptr(), 1)  # first launches load the kernels (lazy module loading)
    tot, ker = plan.solve_device_timed(d.data_ptr(), 5)
    U = plan.unknowns
    print(f"n={orders[0]} K={elements[0]} dim={len(orders)} U={U:>11d}  solve {tot:8.3f} ms  {U/tot/1e6:8.2f} Gunk/s  frac(2N-1 passes) {(2*len(orders)-1)*16*U/(tot*1e-3)/6.448e12:.3f}  kernels {[round(k,3) for k in ker]}")
