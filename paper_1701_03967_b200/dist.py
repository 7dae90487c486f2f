"""Multi-GPU slab-decomposed solve over the C-ABI
(sfem_cuda_dist_*), one process per GPU.

The data path per solve on rank r:
    FORWARD_LOCAL(x) -> PACK1 -> all_to_all -> UNPACK1 -> AXIS0(y)
    -> PACK2 -> all_to_all (reverse counts) -> UNPACK2 -> INVERSE_LOCAL(x)
x = the rank's axis-0 slab of the global dof tensor, y = its axis-1 slab with
axis 0 contiguous.  With K = 64 tables on the swept axis 0, AXIS0 runs in
place on the received exchange buffer (each y row is read and written as
per-source segments) and UNPACK1 / PACK2 are no-ops.  The two all-to-alls are the only collectives (NCCL through
torch.distributed on GPUs); everything else is the rank's own kernels.

`partition` / `slab_*` restate the C++ slab arithmetic for the host side and
for the CPU (gloo) tests.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import Context, Error, ProblemSpec, _check, default_context, lib

PHASES = dict(forward_local=0, pack1=1, unpack1=2, axis0=3, pack2=4, unpack2=5, inverse_local=6)

_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def partition(n: int, parts: int):
    """Balanced contiguous split of n rows: (offsets, lengths) (capi.cu `balanced`)."""
    lens = [n // parts + (1 if r < n % parts else 0) for r in range(parts)]
    offs = [sum(lens[:r]) for r in range(parts)]
    return offs, lens


def partition_even(n: int, parts: int):
    """Axis-0 split (capi.cu `balanced_even`): pairs of rows balanced, the odd
    remainder taken off the last non-empty slab, so every slab starts at an
    even row.  Returns (offsets, lengths)."""
    pairs = (n + 1) // 2
    lens = [2 * (pairs // parts + (1 if r < pairs % parts else 0)) for r in range(parts)]
    extra = sum(lens) - n
    for r in range(parts - 1, -1, -1):
        if extra and lens[r] > 0:
            lens[r] -= extra
            break
    offs = [sum(lens[:r]) for r in range(parts)]
    return offs, lens


def padded(lx: int) -> int:
    """Exchange-buffer block pitch of a slab of lx rows (lx rounded up to even)."""
    return lx + (lx & 1)


def chunk_schedule(extents, nranks: int, chunks: int):
    """Chunk rows of the library-owned exchange (capi.cu dist_setup): per rank
    the x-row chunks (even starts, `partition_even` of its slab) and the y-row
    chunks (`partition` of its y range).  Returns (xc0, xw, yc0, yw), each
    [rank][chunk]."""
    _, lxs = partition_even(extents[0], nranks)
    _, lys = partition(extents[1], nranks)
    xc0, xw, yc0, yw = [], [], [], []
    for p in range(nranks):
        o, w = partition_even(lxs[p], chunks)
        xc0.append(o), xw.append(w)
        o, w = partition(lys[p], chunks)
        yc0.append(o), yw.append(w)
    return xc0, xw, yc0, yw


def chunk_messages(extents, nranks: int, rank: int, chunks: int, step: int, chunk: int):
    """Messages of one exchange chunk as sfem_cuda_dist_solve issues them
    (capi.cu msgs1 / msgs2): (sends, recvs), each a list of (peer, offset,
    count) in doubles -- offsets into the rank's send buffer (A in exchange 1,
    B in exchange 2) and receive buffer (B / A).  Messages between a pair of
    ranks appear in the same order on both sides."""
    x0s, lxs = partition_even(extents[0], nranks)
    y0s, lys = partition(extents[1], nranks)
    R = int(np.prod(extents[2:])) if len(extents) > 2 else 1
    Q = extents[1] * R
    xc0, xw, yc0, yw = chunk_schedule(extents, nranks, chunks)
    r, c = rank, chunk
    sends, recvs = [], []
    if step == 1:
        w = xw[r][c]
        for p in range(nranks):
            if w > 0 and lys[p] > 0:
                sends.append((p, Q * xc0[r][c] + y0s[p] * R * padded(w), lys[p] * R * padded(w)))
            ws = xw[p][c]
            if ws > 0 and lys[r] > 0:
                recvs.append((p, lys[r] * R * (x0s[p] + xc0[p][c]), lys[r] * R * padded(ws)))
    else:
        lyR = lys[r] * R
        for p in range(nranks):
            for cx in range(chunks):
                wpp = padded(xw[p][cx])
                if xw[p][cx] > 0 and yw[r][c] > 0:
                    sends.append((p, lyR * (x0s[p] + xc0[p][cx]) + yc0[r][c] * R * wpp, yw[r][c] * R * wpp))
                wpr = padded(xw[r][cx])
                if xw[r][cx] > 0 and yw[p][c] > 0:
                    recvs.append((p, Q * xc0[r][cx] + (y0s[p] + yc0[p][c]) * R * wpr, yw[p][c] * R * wpr))
    return sends, recvs


@dataclass
class SlabShape:
    extents: List[int]
    nranks: int
    rank: int

    @property
    def R(self) -> int:
        return int(np.prod(self.extents[2:])) if len(self.extents) > 2 else 1

    def x(self):
        offs, lens = partition_even(self.extents[0], self.nranks)
        return offs[self.rank], lens[self.rank]

    def y(self):
        offs, lens = partition(self.extents[1], self.nranks)
        return offs[self.rank], lens[self.rank]

    def send_counts1(self) -> List[int]:
        _, lx = self.x()
        _, lys = partition(self.extents[1], self.nranks)
        return [padded(lx) * ly * self.R for ly in lys]

    def recv_counts1(self) -> List[int]:
        _, ly = self.y()
        _, lxs = partition_even(self.extents[0], self.nranks)
        return [padded(lx) * ly * self.R for lx in lxs]


class DistPlan:
    """One rank's share of a slab-decomposed solve (sfem_cuda_dist_create)."""

    def __init__(self, spec: ProblemSpec, nranks: int, rank: int, ctx: Optional[Context] = None):
        spec.validate()
        self.ctx = ctx or default_context()
        self.spec = spec
        N = spec.dimension
        h = _vp()
        coeffs = (ctypes.c_double * N)(*spec.coefficients) if spec.coefficients is not None else None
        _check(lib.sfem_cuda_dist_create(self.ctx.handle, N, (ctypes.c_int * N)(*spec.orders),
                                         (ctypes.c_int * N)(*spec.elements), (ctypes.c_double * N)(*spec.lengths),
                                         ctypes.cast(coeffs, _dp) if coeffs is not None else None,
                                         float(spec.shift), nranks, rank, ctypes.byref(h)))
        self.handle = h
        info = (ctypes.c_longlong * 10)()
        sc = (ctypes.c_longlong * nranks)()
        rc = (ctypes.c_longlong * nranks)()
        _check(lib.sfem_cuda_dist_shape(h, info, sc, rc))
        (self.x0, self.lx, self.y0, self.ly, self.x_elems, self.y_elems, self.buf_elems, self.xpitch,
         self.ypitch, self.R) = list(info)
        self.send_counts = list(sc)
        self.recv_counts = list(rc)
        self.nranks, self.rank = nranks, rank
        self.extents = spec.extents()

    def phase(self, name: str, x: int, y: int, buf: int, stream: int = 0):
        _check(lib.sfem_cuda_dist_phase(self.handle, PHASES[name], _vp(x), _vp(y), _vp(buf), _vp(stream or None)))

    # ---- library-owned exchange (NCCL inside the C-ABI, chunk-pipelined) ----
    def setup(self, chunks: int = 0):
        """Chunk schedule and plan-owned buffers without a communicator
        (for solve_group)."""
        _check(lib.sfem_cuda_dist_setup(self.handle, chunks))

    def messages(self, step: int, chunk: int):
        """(sends, recvs) of one exchange chunk as the library issues them
        (sfem_cuda_dist_messages): lists of (peer, offset, count)."""
        cap = 4 * self.nranks * 16 + 16
        ns, nr = ctypes.c_int(), ctypes.c_int()
        peers = (ctypes.c_int * cap)()
        offs = (ctypes.c_longlong * cap)()
        cnts = (ctypes.c_longlong * cap)()
        _check(lib.sfem_cuda_dist_messages(self.handle, step, chunk, cap, ctypes.byref(ns), ctypes.byref(nr), peers,
                                           offs, cnts))
        allm = [(peers[i], offs[i], cnts[i]) for i in range(ns.value + nr.value)]
        return allm[:ns.value], allm[ns.value:]

    def comm_init(self, unique_id: bytes, chunks: int = 0):
        """Create the plan's NCCL communicator from a unique id made by
        nccl_unique_id() on one rank (sfem_cuda_dist_comm_init)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), NCCL_UNIQUE_ID_BYTES)
        _check(lib.sfem_cuda_dist_comm_init(self.handle, buf, chunks))

    def solve(self, x_ptr: int, stream: int = 0):
        """One whole distributed solve of this rank's x-slab, in place
        (sfem_cuda_dist_solve: sweeps + grouped ncclSend/ncclRecv)."""
        _check(lib.sfem_cuda_dist_solve(self.handle, _vp(x_ptr), _vp(stream or None)))

    def stats(self):
        """(phase_ms[6], bytes sent to other ranks) of the last solve."""
        ms = (ctypes.c_double * 6)()
        nb = ctypes.c_longlong()
        _check(lib.sfem_cuda_dist_solve_stats(self.handle, ms, ctypes.byref(nb)))
        return list(ms), nb.value

    def __del__(self):
        try:
            if self.handle:
                lib.sfem_cuda_dist_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


NCCL_UNIQUE_ID_BYTES = 128
STAT_NAMES = ("forward_local+pack", "exchange1_exposed", "axis0", "exchange2_exposed", "unpack+inverse_local", "solve")


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check(lib.sfem_cuda_nccl_unique_id(buf))
    return buf.raw


def solve_group(plans: Sequence[DistPlan], x_ptrs, stream: int = 0):
    """All ranks of a solve on one device, messages by device copies
    (sfem_cuda_dist_solve_group; plans set up with one chunk count)."""
    n = len(plans)
    hs = (_vp * n)(*[p.handle for p in plans])
    xs = (_vp * n)(*[_vp(int(x)) for x in x_ptrs])
    _check(lib.sfem_cuda_dist_solve_group(hs, n, xs, _vp(stream or None)))


def solve_ranks(plans: Sequence[DistPlan], xs, bufs_a, bufs_b, ys, exchange):
    """One distributed solve for the ranks in `plans` (one rank per process
    with a real communicator, or every rank on one device for the loopback
    check).  Per rank, CUDA tensors: x-slab, exchange buffers A (send 1 /
    receive 2) and B (receive 1 / send 2), y-slab.  `exchange(step, plans,
    sends, recvs)` performs the all-to-all of step 1 (send_counts ->
    recv_counts) or step 2 (reversed).  Everything runs on torch's current
    stream."""
    import torch
    # One stream for kernels and exchanges: the plans' context stream (a NULL
    # stream argument would select it inside the library while torch's copies
    # ran on the legacy default stream, unordered).
    ext = torch.cuda.ExternalStream(plans[0].ctx.stream)
    with torch.cuda.stream(ext):
        _solve_ranks(plans, xs, bufs_a, bufs_b, ys, exchange, ext.cuda_stream)


def _solve_ranks(plans, xs, bufs_a, bufs_b, ys, exchange, stream):
    ptr = lambda t: t.data_ptr()  # noqa: E731
    for p, x, a, y in zip(plans, xs, bufs_a, ys):
        p.phase("forward_local", ptr(x), ptr(y), ptr(a), stream)
        p.phase("pack1", ptr(x), ptr(y), ptr(a), stream)
    exchange(1, plans, bufs_a, bufs_b)
    for p, x, b, y in zip(plans, xs, bufs_b, ys):
        p.phase("unpack1", ptr(x), ptr(y), ptr(b), stream)
        p.phase("axis0", ptr(x), ptr(y), ptr(b), stream)
        p.phase("pack2", ptr(x), ptr(y), ptr(b), stream)
    exchange(2, plans, bufs_b, bufs_a)
    for p, x, a, y in zip(plans, xs, bufs_a, ys):
        p.phase("unpack2", ptr(x), ptr(y), ptr(a), stream)
        p.phase("inverse_local", ptr(x), ptr(y), ptr(a), stream)


def _counts(p, step):
    sc = p.send_counts if step == 1 else p.recv_counts
    rc = p.recv_counts if step == 1 else p.send_counts
    return list(sc), list(rc)


def loopback_exchange(step, plans, sends, recvs):
    """All-to-all among virtual ranks sharing one device (tensor copies)."""
    P = len(plans)
    for dst in range(P):
        off_r = 0
        for src in range(P):
            sc, _ = _counts(plans[src], step)
            off_s = sum(sc[:dst])
            n = sc[dst]
            if n:
                recvs[dst][off_r:off_r + n].copy_(sends[src][off_s:off_s + n])
            off_r += n


def torch_exchange(step, plans, sends, recvs):
    """All-to-all through torch.distributed (NCCL on GPUs, gloo on CPUs)."""
    import torch.distributed as dist
    (p,) = plans
    sc, rc = _counts(p, step)
    dist.all_to_all_single(recvs[0][:sum(rc)], sends[0][:sum(sc)], output_split_sizes=rc, input_split_sizes=sc)


def allocate(plan: DistPlan, device="cuda"):
    """Device buffers for one rank: (x, A, B, y)."""
    import torch
    mk = lambda n: torch.zeros(max(int(n), 1), dtype=torch.float64, device=device)  # noqa: E731
    return mk(plan.x_elems), mk(plan.buf_elems), mk(plan.buf_elems), mk(plan.y_elems)


def scatter_x(plan: DistPlan, x, load: np.ndarray):
    """Copy the rank's axis-0 rows of a dense global dof tensor into its padded x-slab."""
    import torch
    ext = plan.extents
    rows = load[plan.x0:plan.x0 + plan.lx].reshape(-1, ext[-1])
    x.view(-1, plan.xpitch)[:rows.shape[0], :ext[-1]].copy_(torch.from_numpy(np.ascontiguousarray(rows)))


def gather_x(plan: DistPlan, x) -> np.ndarray:
    ext = plan.extents
    rows = x.view(-1, plan.xpitch)[:, :ext[-1]].cpu().numpy()
    return rows.reshape([plan.lx] + list(ext[1:]))


# ---------------------------------------------------------------------------
# Fused NVLink exchange (sfem_cuda_peer_*): the all-to-all transposes travel
# inside the axis-1 forward and axis-0 sweeps as TMA stores into the other
# ranks' slabs (peer memory); no collective on the data path.
# ---------------------------------------------------------------------------
PEER_FORWARD, PEER_AXIS0, PEER_INVERSE, PEER_BARRIER = 0, 1, 2, 3


class PeerPlan:
    """One rank's share of the fused NVLink solve (3-D, K = 64 on axes 0, 1).
    Buffers are plan-owned: x-slab [lx][L1][pitch] (laid out x, y, z), y-slab
    [ly][L0][pitch]."""

    def __init__(self, spec: ProblemSpec, nranks: int, rank: int, ctx: Optional[Context] = None):
        spec.validate()
        self.ctx = ctx or default_context()
        self.spec = spec
        N = spec.dimension
        h = _vp()
        coeffs = (ctypes.c_double * N)(*spec.coefficients) if spec.coefficients is not None else None
        _check(lib.sfem_cuda_peer_create(self.ctx.handle, N, (ctypes.c_int * N)(*spec.orders),
                                         (ctypes.c_int * N)(*spec.elements), (ctypes.c_double * N)(*spec.lengths),
                                         ctypes.cast(coeffs, _dp) if coeffs is not None else None,
                                         float(spec.shift), nranks, rank, ctypes.byref(h)))
        self.handle = h
        info = (ctypes.c_longlong * 8)()
        _check(lib.sfem_cuda_peer_shape(h, info))
        self.x0, self.lx, self.y0, self.ly, self.x_elems, self.y_elems, self.pitch, _ = list(info)
        xp, yp, fp = _vp(), _vp(), _vp()
        _check(lib.sfem_cuda_peer_buffers(h, ctypes.byref(xp), ctypes.byref(yp), ctypes.byref(fp)))
        self.x_ptr, self.y_ptr, self.flags_ptr = xp.value, yp.value, fp.value
        self.nranks, self.rank = nranks, rank
        self.extents = spec.extents()
        self._opened = []

    def bind(self, x_ptrs, y_ptrs, flag_ptrs=None):
        P = self.nranks
        arr = lambda v: (_vp * P)(*[_vp(int(x)) for x in v])  # noqa: E731
        _check(lib.sfem_cuda_peer_bind(self.handle, arr(x_ptrs), arr(y_ptrs),
                                       arr(flag_ptrs) if flag_ptrs is not None else None))

    def phase(self, ph: int, stream: int = 0):
        _check(lib.sfem_cuda_peer_phase(self.handle, ph, _vp(stream or None)))

    def barrier_timeout(self, stream: int = 0) -> int:
        """Synchronise `stream`; the epoch of a device barrier that gave up
        waiting for a peer (0 = every barrier completed)."""
        v = ctypes.c_longlong()
        _check(lib.sfem_cuda_peer_status(self.handle, _vp(stream or None), ctypes.byref(v)))
        return v.value

    def solve(self, stream: int = 0):
        """One solve (the bound ranks run their phases concurrently on their
        own devices; the device barriers order the exchanges)."""
        for ph in (PEER_FORWARD, PEER_BARRIER, PEER_AXIS0, PEER_BARRIER, PEER_INVERSE):
            self.phase(ph, stream)

    # ---- slab data (dense global dof tensor <-> this rank's x-slab) ----
    def x_view(self):
        """torch view of the plan-owned x-slab [lx][L1][pitch]."""
        return _wrap_device(self.x_ptr, (self.lx, self.extents[1], self.pitch), self.ctx.device)

    def scatter_x(self, load: np.ndarray):
        import torch
        v = self.x_view()
        blk = np.ascontiguousarray(load[self.x0:self.x0 + self.lx])
        v[:, :, :self.extents[2]].copy_(torch.from_numpy(blk))

    def gather_x(self) -> np.ndarray:
        import torch
        torch.cuda.synchronize(self.ctx.device)
        return self.x_view()[:, :, :self.extents[2]].cpu().numpy()

    def close(self):
        for ptr in self._opened:
            lib.sfem_cuda_ipc_close(_vp(ptr))
        self._opened = []
        if self.handle:
            lib.sfem_cuda_peer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device(ptr: int, shape, device: int):
    """A torch view of plan-owned device memory (no copy, no ownership)."""
    import torch

    class _Arr:
        def __init__(self):
            strides = []
            acc = 1
            for d in reversed(shape):
                strides.append(acc * 8)
                acc *= d
            self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False),
                                             "version": 2, "strides": tuple(reversed(strides))}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=f"cuda:{device}")


def ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(lib.sfem_cuda_ipc_get_handle(_vp(ptr), buf))
    return buf.raw


def ipc_open(handle: bytes) -> int:
    out = _vp()
    buf = ctypes.create_string_buffer(handle, 64)
    _check(lib.sfem_cuda_ipc_open_handle(buf, ctypes.byref(out)))
    return out.value


def peer_bind_distributed(plan: PeerPlan, dist_mod, device_barrier: bool = True) -> None:
    """Exchange the ranks' buffer handles over torch.distributed and bind the
    peers (one process per GPU, NVLink P2P).  device_barrier=False binds no
    flag words: the caller orders the phases from the host (stream
    synchronise + a host barrier), as the two-processes-on-one-GPU test does,
    where kernels of different processes must not wait on one another."""
    mine = [ipc_handle(plan.x_ptr), ipc_handle(plan.y_ptr), ipc_handle(plan.flags_ptr)]
    allh = [None] * plan.nranks
    dist_mod.all_gather_object(allh, mine)
    xs, ys, fs = [], [], []
    for q, hs in enumerate(allh):
        if q == plan.rank:
            xs.append(plan.x_ptr), ys.append(plan.y_ptr), fs.append(plan.flags_ptr)
            continue
        ptrs = [ipc_open(h) for h in hs]
        plan._opened += ptrs
        xs.append(ptrs[0]), ys.append(ptrs[1]), fs.append(ptrs[2])
    plan.bind(xs, ys, fs if device_barrier else None)


def peer_solve_host_ordered(plan: PeerPlan, dist_mod, stream: int = 0) -> None:
    """One solve with the exchanges ordered from the host: every rank finishes
    a phase (stream synchronise) and meets the others at a host barrier before
    the next one starts.  No kernel waits for another process."""
    for ph in (PEER_FORWARD, PEER_AXIS0, PEER_INVERSE):
        plan.phase(ph, stream)
        plan.barrier_timeout(stream)  # synchronises the stream
        dist_mod.barrier()


def peer_solve_loopback(plans: Sequence[PeerPlan], stream: int = 0) -> None:
    """All ranks on one device (the single-GPU check): phases rank after rank,
    no device barrier (stream order is the barrier)."""
    for ph in (PEER_FORWARD, PEER_AXIS0, PEER_INVERSE):
        for p in plans:
            p.phase(ph, stream)


def peer_bind_loopback(plans: Sequence[PeerPlan]) -> None:
    xs = [p.x_ptr for p in plans]
    ys = [p.y_ptr for p in plans]
    for p in plans:
        p.bind(xs, ys, None)
