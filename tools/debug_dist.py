"""Phase-by-phase comparison of the GPU slab solve (loopback ranks) with the
oracle emulation from tests/test_dist.py."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1701_03967_b200 as sfem  # noqa: E402
from paper_1701_03967_b200 import dist as D  # noqa: E402
from test_dist import OracleRank  # noqa: E402

orders = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 2, 2]
elements = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [64, 64, 64]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lengths = [1.0] * len(orders)
shift = 0.5
spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift)
f = np.random.default_rng(1).uniform(-1, 1, spec.extents())
plans = [D.DistPlan(spec, P, r) for r in range(P)]
orcs = [OracleRank(orders, elements, lengths, shift, P, r) for r in range(P)]
bufs = [D.allocate(p) for p in plans]
stream = torch.cuda.current_stream().cuda_stream
for p, (x, a, b, y) in zip(plans, bufs):
    D.scatter_x(p, x, f)
ox = [f[o.x0:o.x0 + o.lx].copy() for o in orcs]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


for r, (p, o, (x, a, b, y)) in enumerate(zip(plans, orcs, bufs)):
    p.phase("forward_local", x.data_ptr(), y.data_ptr(), a.data_ptr(), stream)
    torch.cuda.synchronize()
    ox[r] = o.forward_local(ox[r])
    print("rank", r, "forward_local rel", rel(D.gather_x(p, x), ox[r]))
    p.phase("pack1", x.data_ptr(), y.data_ptr(), a.data_ptr(), stream)
    torch.cuda.synchronize()
    ob = o.pack1(ox[r])
    print("rank", r, "pack1 rel", rel(a[:ob.size].cpu().numpy(), ob))

# exchange 1 (device) and oracle equivalent
D.loopback_exchange(1, plans, [bb[1] for bb in bufs], [bb[2] for bb in bufs])
torch.cuda.synchronize()
obufs = [o.pack1(ox[r]) for r, o in enumerate(orcs)]
orecv = []
for dst, o in enumerate(orcs):
    parts = []
    for src, os_ in enumerate(orcs):
        off = sum(os_.send_counts[:dst])
        parts.append(obufs[src][off:off + os_.send_counts[dst]])
    orecv.append(np.concatenate(parts))
oy = []
for r, (p, o, (x, a, b, y)) in enumerate(zip(plans, orcs, bufs)):
    print("rank", r, "recv1 rel", rel(b[:orecv[r].size].cpu().numpy(), orecv[r]))
    p.phase("unpack1", x.data_ptr(), y.data_ptr(), b.data_ptr(), stream)
    torch.cuda.synchronize()
    yy = o.unpack1(orecv[r])
    gy = y.view(-1, p.ypitch)[:, :p.extents[0]].cpu().numpy()
    print("rank", r, "unpack1 rel", rel(gy, yy))
    p.phase("axis0", x.data_ptr(), y.data_ptr(), b.data_ptr(), stream)
    torch.cuda.synchronize()
    yy = o.axis0(yy)
    gy = y.view(-1, p.ypitch)[:, :p.extents[0]].cpu().numpy()
    print("rank", r, "axis0 rel", rel(gy, yy))
    oy.append(yy)

for r, (p, o, (x, a, b, y)) in enumerate(zip(plans, orcs, bufs)):
    p.phase("pack2", x.data_ptr(), y.data_ptr(), b.data_ptr(), stream)
torch.cuda.synchronize()
obufs2 = [o.pack2(oy[r]) for r, o in enumerate(orcs)]
for r in range(P):
    print("rank", r, "pack2 rel", rel(bufs[r][2][:obufs2[r].size].cpu().numpy(), obufs2[r]))
D.loopback_exchange(2, plans, [bb[2] for bb in bufs], [bb[1] for bb in bufs])
torch.cuda.synchronize()
for dst, (p, o, (x, a, b, y)) in enumerate(zip(plans, orcs, bufs)):
    parts = []
    for src, os_ in enumerate(orcs):
        off = sum(os_.recv_counts[:dst])
        parts.append(obufs2[src][off:off + os_.recv_counts[dst]])
    orecv2 = np.concatenate(parts)
    print("rank", dst, "recv2 rel", rel(a[:orecv2.size].cpu().numpy(), orecv2))
    p.phase("unpack2", x.data_ptr(), y.data_ptr(), a.data_ptr(), stream)
    torch.cuda.synchronize()
    xx = o.unpack2(orecv2)
    print("rank", dst, "unpack2 rel", rel(D.gather_x(p, x), xx))
    p.phase("inverse_local", x.data_ptr(), y.data_ptr(), a.data_ptr(), stream)
    torch.cuda.synchronize()
    xx = o.inverse_local(xx)
    print("rank", dst, "inverse_local rel", rel(D.gather_x(p, x), xx))
