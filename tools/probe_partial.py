import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1701_03967_b200 as sfem
from oracle import reflib
def rl(a,b): return float(np.linalg.norm(a-b)/np.linalg.norm(b))
for K in (16, 32, 64):
    orders, elements, lengths, shift = [9, 9, 9], [K]*3, [1.0]*3, 0.0
    spec = sfem.ProblemSpec(3, lengths, elements, orders, shift)
    f = reflib.uniform(0, int(np.prod(spec.extents()))).reshape(spec.extents())
    pa = sfem.Plan(spec); ua, _ = pa.solve_host(f)
    pb = sfem.Plan(spec); pb.set_algorithm("partial"); ub, _ = pb.solve_host(f)
    ra, _ = reflib.solve(f, orders, elements, lengths, shift, algorithm=0)
    rb, _ = reflib.solve(f, orders, elements, lengths, shift, algorithm=1)
    print(K, "ours(b)-ref(a)", rl(ub, ra), "ref(b)-ref(a)", rl(rb, ra), "ours(b)-ref(b)", rl(ub, rb), "ours(a)-ref(a)", rl(ua, ra), flush=True)
