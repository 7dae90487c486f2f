import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1701_03967_b200 as sfem
for plain in ("0", "1"):
  os.environ["SFEM_PLAIN"] = plain
  if plain == "0": os.environ.pop("SFEM_PLAIN")
  for orders in ([4,4,4],[9,9,9]):
    spec = sfem.ProblemSpec(3, [1.0]*3, [64]*3, orders, 0.0)
    gen = torch.Generator(device="cuda"); gen.manual_seed(0)
    plan = sfem.Plan(spec)
    ext = plan.extents; rows = plan.unknowns // ext[-1]
    base = torch.rand(rows, plan.pitch, dtype=torch.float64, device="cuda", generator=gen)
    base[:, ext[-1]:] = 0
    for v1 in ("0", "1"):
        os.environ["SFEM_ROWS_V1"] = v1
        outs = []
        for rep in range(3):
            buf = base.clone(); torch.cuda.synchronize(); plan.solve_device(buf.data_ptr()); torch.cuda.synchronize(); outs.append(buf[:, :ext[-1]].clone())
        fresh = sfem.Plan(spec); buf = base.clone(); torch.cuda.synchronize(); fresh.solve_device(buf.data_ptr()); torch.cuda.synchronize()
        fr = buf[:, :ext[-1]].clone(); del fresh
        print("plain", plain, orders, "v1", v1, "rep0-1", (outs[0]-outs[1]).abs().max().item(), "rep1-2", (outs[1]-outs[2]).abs().max().item(),
              "rep0-fresh", (outs[0]-fr).abs().max().item(), flush=True)
