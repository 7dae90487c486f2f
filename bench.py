#!/usr/bin/env python
"""bench.py -- FP64 FEM unknowns solved/s for the fast spectral Poisson solve
(algorithm (a), full diagonalisation) on B200, with HBM roofline and the
reference's CPU solver beside it.

Default workload (BASELINE.json metric "3D n=9"): config 4, 3D, order n=9,
K=64 elements per axis (575^3 = 190,109,375 unknowns), -Laplace u = f on the
unit cube, f i.i.d. U[-1,1] (seeded, synthetic), FP64.  One step = one full
solve (2N-1 = 5 sweep kernels) on a device-resident 1.52 GB tensor (> L2, so
no flush is needed between steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4|...]

N > 1 (torchrun, one rank per GPU): ONE global problem, slab-decomposed along
axis 0 ("scaling": "strong"); value = global unknowns / max-over-ranks time.
Default --dist-mode peer: the two transposes are fused into the sweeps as TMA
stores into the other ranks' slabs over NVLink (CUDA IPC), device flag
barriers between phases; --dist-mode nccl: NCCL all-to-all between the
sweeps.  If both fail the ranks fall back to independent replicas.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (orders, elements, lengths, coefficients, shift, description)
    "c4": ([9, 9, 9], [64, 64, 64], [1.0] * 3, None, 0.0, "3D n=9 K=64 -Laplace u=f (config 4)"),
    "c1": ([2, 2], [64, 64], [1.0, 1.0], None, 0.0, "2D n=2 K=64 -Laplace u=f (config 1)"),
    "c3": ([9, 9], [1024, 1024], [1.0, 1.0], [1.0, 2.0], 1.0, "2D n=9 K=1024 -(u_xx+2u_yy)+u=f (config 3)"),
    "c5n1": ([1, 1, 1], [1024] * 3, [1.0] * 3, None, 0.5, "3D n=1 K=1024 -Lap u+0.5u=f (config 5)"),
    "c5n2": ([2, 2, 2], [512] * 3, [1.0] * 3, None, 0.5, "3D n=2 K=512 (config 5)"),
    "c5n4": ([4, 4, 4], [256] * 3, [1.0] * 3, None, 0.5, "3D n=4 K=256 (config 5)"),
    "c5n9": ([9, 9, 9], [114] * 3, [1.0] * 3, None, 0.5, "3D n=9 K=114 (config 5)"),
}
# config 2: 1-D expansion only (n=4, K=4096, a batch of 4096 lines): FC_n, F_n, F_n^-1
C2 = (4, 4096, 4096)


def ref_sample(cfg_name):
    """(orders, elements, lengths, shift, same_config) the reference arm solves
    per step.  A per-axis coefficient a_i is the reference's lengths X_i/sqrt(a_i)
    (solve_with_load uses the lengths only through 4/h_i^2)."""
    orders, elements, lengths, coeffs, shift, _ = CONFIGS[cfg_name]
    lengths = [X / (a ** 0.5) for X, a in zip(lengths, coeffs or [1.0] * len(lengths))]
    elements = list(elements)
    same = True
    while np.prod([n * K - 1 for n, K in zip(orders, elements)]) > REF_MAX_UNKNOWNS:
        elements = [max(2, K // 2) for K in elements]
        same = False
    return orders, elements, lengths, shift, same


def ref_sample_text(orders, elements, U, same):
    ext = "x".join(str(n * K - 1) for n, K in zip(orders, elements))
    return (f"{len(orders)}D n={orders[0]} K={elements[0]} ({ext} = {U} unknowns"
            f"{', the same configuration' if same else ', a smaller-K sample of the configuration'}), "
            "the reference's solve_with_load (algorithm (a)) with its own seconds_solve timer, median over the "
            "timed solves after a warm-up solve; FFTW (absent from the image) replaced by the oracle/shim FFT")

# The reference arm and cpu_baseline run the reference's own solver on the
# SAME configuration when one solve fits a few seconds of host work (C1, C3,
# C4: <= 2.5e8 unknowns); the 1.07e9-unknown C5 shapes are sampled with
# fewer elements per axis (same orders and equation; same_config false).
REF_MAX_UNKNOWNS = 2.5e8
# Configs timed device-resident beside the headline (the "configs" object).
SIDE_CONFIGS = ["c1", "c2", "c3", "c5n1", "c5n2", "c5n4", "c5n9"]

METRIC = "FP64 FEM unknowns solved/sec (3D n=9) and achieved HBM GB/s vs roofline"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for name, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(name)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local, dist


def max_over_ranks(x, dist, world):
    if world == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist, world):
    if world > 1:
        dist.barrier()


def cpu_reference_sample(cfg_name, reps=5, warmup=1):
    """The reference's own solver (oracle/_ref) on the arm's workload: `warmup`
    untimed solves, then `reps` solves, each timed by the reference's own
    seconds_solve (poisson.cpp:781-785); the acceptance suite's median of 5
    after a warm-up (acceptance_main.cpp:264-273)."""
    from oracle import reflib
    orders, elements, lengths, shift, same = ref_sample(cfg_name)
    ext = [n * K - 1 for n, K in zip(orders, elements)]
    f = np.random.default_rng(0).uniform(-1.0, 1.0, ext)
    secs = reflib.solve_repeat(f, orders, elements, lengths, shift, warmup + reps)[warmup:]
    U = int(np.prod(ext))
    return U, secs, reflib.max_threads(), ref_sample_text(orders, elements, U, same), same


def side_configs(sfem, ctx, args):
    """Device-resident times of the other BASELINE configs in the same run and
    clocks: a few warm-up solves, then `reps` solves bracketed by CUDA events
    on the plan stream; frac = algorithmic bytes (16 B per unknown per sweep
    launch) / time / measured HBM peak.  Loads are seeded U[-1,1] drawn on the
    device (values do not change the work)."""
    import torch
    peaks, _ = measured_peaks()
    out = {}
    stream = torch.cuda.ExternalStream(ctx.stream)
    gen = torch.Generator(device="cuda")
    for name in SIDE_CONFIGS:
        try:
            if name == "c2":
                n, K, count = C2
                t = sfem.SpectralTable(n, K, ctx)
                L = n * K - 1
                gen.manual_seed(0)
                x = torch.randn(count, L, dtype=torch.float64, device="cuda", generator=gen)
                y = torch.empty_like(x)
                ms = {}
                for op, label in ((sfem.DECOMPOSE_WEIGHTED, "fc_n"), (sfem.DECOMPOSE, "f_n"),
                                  (sfem.SYNTHESIZE, "f_n_inverse")):
                    for _ in range(3):
                        sfem.lines_device(t, op, count, x.data_ptr(), L, y.data_ptr(), L, ctx.stream)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    reps = 10
                    e0.record(stream)
                    for _ in range(reps):
                        sfem.lines_device(t, op, count, x.data_ptr(), L, y.data_ptr(), L, ctx.stream)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ms[label] = e0.elapsed_time(e1) / reps
                worst = max(ms.values())
                out[name] = {"workload": "1D n=4 K=4096, 4096 lines (config 2)", "values": count * L,
                             "ms_per_op": {k: round(v, 4) for k, v in ms.items()},
                             "frac": 16.0 * count * L / (worst * 1e-3) / 1e9 / peaks["hbm_gbs"],
                             "frac_note": "slowest of the three ops; 16 B per value per op"}
                del x, y, t
                torch.cuda.empty_cache()
                continue
            orders, elements, lengths, coeffs, shift, desc = CONFIGS[name]
            spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
            plan = sfem.Plan(spec, ctx)
            rows = plan.unknowns // plan.extents[-1]
            gen.manual_seed(0)
            buf = torch.rand(rows, plan.pitch, dtype=torch.float64, device="cuda", generator=gen)
            buf.mul_(2.0).sub_(1.0)
            reps = 5 if plan.unknowns > 5e8 else 20
            for _ in range(3):
                plan.solve_device(buf.data_ptr())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                plan.solve_device(buf.data_ptr())
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            _, kern = plan.solve_device_timed(buf.data_ptr(), reps=2)
            out[name] = {"workload": desc, "unknowns": plan.unknowns, "ms": round(ms, 4),
                         "unknowns_per_s": plan.unknowns / (ms * 1e-3),
                         "kernel_ms": [round(v, 4) for v in kern],
                         "frac": 16.0 * plan.unknowns * plan.launches / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"]}
            del buf, plan
            torch.cuda.empty_cache()
        except Exception as e:  # reported, not fatal
            out[name] = {"error": repr(e)}
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from the reference sources with an FFTW-API shim), all host threads."""
    if rank != 0:
        return
    from oracle import reflib
    if not reflib.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsfem_ref.so not built"}), flush=True)
        return
    U, secs, cores, sample, same = cpu_reference_sample(args.config, reps=args.steps, warmup=args.warmup)
    med = statistics.median(secs)
    value = U / med
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "unknowns/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * med,
        "ms_per_step_mean": 1e3 * float(np.mean(secs)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config][5], "cpu_sample": sample, "same_config": same,
                   "parallelism": f"openmp x{cores}"},
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def peer_capable(config):
    orders, elements = CONFIGS[config][0], CONFIGS[config][1]
    return len(orders) == 3 and elements[0] == 64 and elements[1] == 64 and orders[0] in (2, 3, 4, 5, 9) \
        and orders[1] in (2, 3, 4, 5, 9)


def run_peer(args, world, rank, local, dist):
    """N > 1, fused NVLink exchange: ONE global problem in
    axis-0 slabs; the axis-1 forward sweep and the axis-0 sweep store their
    tiles straight into the other ranks' slabs (CUDA IPC peer memory), a
    device flag barrier between the phases; no collective on the data path.
    Strong scaling: value = global unknowns / max-over-ranks time."""
    import torch
    import paper_1701_03967_b200 as sfem
    from paper_1701_03967_b200 import dist as D

    orders, elements, lengths, coeffs, shift, desc = CONFIGS[args.config]
    spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
    ctx = sfem.Context(local)
    plan = D.PeerPlan(spec, world, rank, ctx)
    D.peer_bind_distributed(plan, dist)
    U = int(np.prod(plan.extents))
    ext = torch.cuda.ExternalStream(ctx.stream)
    xv = plan.x_view()
    L1, L2 = plan.extents[1], plan.extents[2]
    f_local = np.random.default_rng(1000 + rank).uniform(-1.0, 1.0, (plan.lx, L1, L2))
    xv[:, :, :L2].copy_(torch.from_numpy(f_local))
    torch.cuda.synchronize()
    barrier(dist, world)

    def solve():
        plan.solve(ctx.stream)

    check = None
    if not args.no_verify:
        # One distributed solve checked against a single-GPU solve of the same
        # global load on rank 0 (rank 0's slab depends on every rank's rows
        # through the two exchanges): a fused exchange that moved the wrong
        # data is reported and the NCCL path takes over, never timed as is.
        # Any local failure (a barrier that timed out, an exception) becomes
        # err = inf in the one all-reduce every rank reaches.
        err = 0.0
        try:
            solve()
            if plan.barrier_timeout(ctx.stream):
                raise RuntimeError("device barrier timed out waiting for a peer")
            mine = plan.gather_x()
            if rank == 0:
                offs, lens = D.partition_even(plan.extents[0], world)
                glob = np.concatenate([np.random.default_rng(1000 + r).uniform(-1.0, 1.0, (lens[r], L1, L2))
                                       for r in range(world)])
                want, _ = sfem.solve_dof(spec, glob, ctx=ctx)
                want = want[offs[0]:offs[0] + lens[0]]
                err = float(np.linalg.norm(mine - want) / np.linalg.norm(want))
                del glob, want
        except Exception as e:
            print(f"[bench] rank {rank}: fused NVLink check failed locally: {e!r}", file=sys.stderr)
            err = float("inf")
        err = max_over_ranks(err, dist, world)
        if not err <= 1e-11:
            raise RuntimeError(f"fused NVLink solve differs from the single-GPU solve (rank-0 slab rel-L2 {err:.3e})")
        check = f"rank-0 slab vs single-GPU solve of the same global load: rel-L2 {err:.2e}"
        xv[:, :, :L2].copy_(torch.from_numpy(f_local))
        torch.cuda.synchronize()
        barrier(dist, world)

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    barrier(dist, world)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        barrier(dist, world)
        ev0.record(ext)
        for _ in range(args.steps):
            solve()
        ev1.record(ext)
        torch.cuda.synchronize()
    barrier(dist, world)
    ms = ev0.elapsed_time(ev1)
    if plan.barrier_timeout(ctx.stream):  # a timed-out barrier: the timed solves are not valid
        ms = float("inf")
    ms = max_over_ranks(ms, dist, world)
    if ms == float("inf"):
        raise RuntimeError("a device barrier timed out during the timed solves")
    value = U * args.steps / (ms * 1e-3)
    ms_step = ms / args.steps
    peaks, peak_kind = measured_peaks()
    local_u = U / world
    hbm_bytes = 16.0 * local_u * 5  # five sweeps, each reads and writes the rank's share once
    achieved = hbm_bytes / (ms_step * 1e-3) / 1e9
    nvl_bytes = 2 * 8.0 * local_u * (world - 1) / world
    # per-rank phase times (one more solve, events between the phases) and the
    # bytes this rank's two exchange sweeps store into other ranks' slabs
    names = ("forward(rows + axis-1 sweep storing to peers)", "barrier1", "axis0(fused, storing back to peers)",
             "barrier2", "inverse(axis 1 + rows)")
    pev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    barrier(dist, world)
    pev[0].record(ext)
    for i, ph in enumerate((D.PEER_FORWARD, D.PEER_BARRIER, D.PEER_AXIS0, D.PEER_BARRIER, D.PEER_INVERSE)):
        plan.phase(ph, ctx.stream)
        pev[i + 1].record(ext)
    torch.cuda.synchronize()
    L0 = plan.extents[0]
    mine = {"rank": rank, "unknowns": plan.lx * L1 * L2,
            "nvlink_bytes_per_solve": 8 * L2 * (plan.lx * (L1 - plan.ly) + plan.ly * (L0 - plan.lx)),
            "phase_ms": {nm: round(pev[i].elapsed_time(pev[i + 1]), 4) for i, nm in enumerate(names)}}
    per_rank = [None] * world
    if world > 1:
        dist.all_gather_object(per_rank, mine)
    else:
        per_rank = [mine]

    h_in = torch.from_numpy(f_local).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    barrier(dist, world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        with torch.cuda.stream(ext):
            xv[:, :, :L2].copy_(h_in, non_blocking=True)
        solve()
        with torch.cuda.stream(ext):
            h_out.copy_(xv[:, :, :L2], non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, dist, world)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "unknowns": U, "extents": plan.extents,
                       "parallelism": f"slab x{world} (axis-0 slabs; exchanges fused into the sweeps as TMA "
                                      "stores to NVLink peer memory)",
                       "dist_check": check,
                       "l2_flush": "none needed: tensors > L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_kind": peak_kind,
                         "kernel": "whole per-rank solve (5 sweeps, 2 of them storing to peers)",
                         "nvlink_bytes_per_rank_per_solve": nvl_bytes},
            "per_rank": per_rank,
            "cpu_baseline": None,
            "e2e": {"value": U / e2e_s, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * int(f_local.size) * world,
                    "d2h_bytes_per_step": 8 * int(f_local.size) * world, "ms_per_step": e2e_s * 1e3},
            "gpu_launches": 7 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    plan.close()


def run_distributed(args, world, rank, local, dist):
    """N > 1: ONE global problem, slab-decomposed over the ranks (axis-0 slabs).
    The exchange lives inside the C-ABI (sfem_cuda_dist_solve): an NCCL
    communicator created from a unique id that rank 0 makes and
    torch.distributed only broadcasts, grouped ncclSend/ncclRecv on an exchange
    stream, both all-to-alls split into chunks that travel while the next
    chunk is swept.  Strong scaling: value = global unknowns / max-over-ranks
    time.  Per-rank NVLink bytes and phase times are printed for every rank."""
    import torch
    import paper_1701_03967_b200 as sfem
    from paper_1701_03967_b200 import dist as D

    orders, elements, lengths, coeffs, shift, desc = CONFIGS[args.config]
    spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
    ctx = sfem.Context(local)
    plan = D.DistPlan(spec, world, rank, ctx)
    ids = [D.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(ids, src=0)
    plan.comm_init(ids[0], args.dist_chunks)
    U = int(np.prod(plan.extents))
    x = torch.zeros(max(plan.x_elems, 1), dtype=torch.float64, device=f"cuda:{local}")
    inner = [int(v) for v in plan.extents[1:]]
    rows_local = plan.lx * int(np.prod(plan.extents[1:-1]))
    f_local = np.random.default_rng(1000 + rank).uniform(-1.0, 1.0, (rows_local, plan.extents[-1]))
    xview = x.view(-1, plan.xpitch)[:rows_local, :plan.extents[-1]]
    xview.copy_(torch.from_numpy(f_local))
    ext = torch.cuda.ExternalStream(ctx.stream)
    torch.cuda.synchronize()

    def solve():
        plan.solve(x.data_ptr(), ctx.stream)

    check = None
    if not args.no_verify:
        # rank 0's slab against a single-GPU solve of the same global load;
        # every rank reaches the one all-reduce whatever happened locally
        err = 0.0
        try:
            solve()
            torch.cuda.synchronize()
            mine = xview.cpu().numpy().reshape([plan.lx] + inner)
            if rank == 0:
                offs, lens = D.partition_even(plan.extents[0], world)
                glob = np.concatenate([np.random.default_rng(1000 + r).uniform(
                    -1.0, 1.0, (lens[r] * int(np.prod(plan.extents[1:-1])), plan.extents[-1]))
                    for r in range(world)]).reshape(plan.extents)
                want, _ = sfem.solve_dof(spec, glob, ctx=ctx)
                want = want[offs[0]:offs[0] + lens[0]]
                err = float(np.linalg.norm(mine - want) / np.linalg.norm(want))
                del glob, want
        except Exception as e:
            print(f"[bench] rank {rank}: NCCL slab solve check failed locally: {e!r}", file=sys.stderr)
            err = float("inf")
        err = max_over_ranks(err, dist, world)
        if not err <= 1e-11:
            raise RuntimeError(f"NCCL slab solve differs from the single-GPU solve (rank-0 slab rel-L2 {err:.3e})")
        check = f"rank-0 slab vs single-GPU solve of the same global load: rel-L2 {err:.2e}"
        xview.copy_(torch.from_numpy(f_local))
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(dist, world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        barrier(dist, world)
        ev0.record(ext)
        for _ in range(args.steps):
            solve()
        ev1.record(ext)
        torch.cuda.synchronize()
    barrier(dist, world)
    ms = max_over_ranks(ev0.elapsed_time(ev1), dist, world)
    phase_ms, sent = plan.stats()  # of the last timed solve
    mine = {"rank": rank, "nvlink_bytes_per_solve": sent, "unknowns": plan.lx * int(np.prod(plan.extents[1:])),
            "phase_ms": dict(zip(D.STAT_NAMES, [round(v, 4) for v in phase_ms]))}
    per_rank = [None] * world
    if world > 1:
        dist.all_gather_object(per_rank, mine)
    else:
        per_rank = [mine]
    value = U * args.steps / (ms * 1e-3)
    ms_step = ms / args.steps
    peaks, peak_kind = measured_peaks()
    # per-rank HBM bytes per solve: 2N-1 sweeps + 2 transposes (+ 2 2-D copies
    # unless the axis-0 sweep runs on the exchange buffer), read + write each
    local_u = U / world
    sweep_bytes = 16.0 * local_u * (2 * len(orders) - 1)
    copy_bytes = 16.0 * local_u * (2 if plan.y_elems == 0 else 4)
    achieved = (sweep_bytes + copy_bytes) / (ms_step * 1e-3) / 1e9

    # end to end: each rank moves its own slab host -> device -> host
    h_in = torch.from_numpy(f_local).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    barrier(dist, world)
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        with torch.cuda.stream(ext):
            xview.copy_(h_in, non_blocking=True)
        solve()
        with torch.cuda.stream(ext):
            h_out.copy_(xview, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, dist, world)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "unknowns": U, "extents": plan.extents,
                       "parallelism": f"slab x{world} (axis-0 slabs; 2 all-to-all exchanges per solve as grouped "
                                      f"ncclSend/ncclRecv inside the C-ABI, {args.dist_chunks or 4} chunks "
                                      "pipelined behind the sweeps)",
                       "dist_check": check,
                       "dist_error": getattr(args, "dist_error", None),
                       "l2_flush": "none needed: tensors > L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": None, "peak_kind": peak_kind,
                         "kernel": "whole per-rank solve (sweeps + transposes)",
                         "nvlink_bytes_per_rank_per_solve": max(r["nvlink_bytes_per_solve"] for r in per_rank)},
            "per_rank": per_rank,
            "cpu_baseline": None,
            "e2e": {"value": U / e2e_s, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * int(f_local.size) * world,
                    "d2h_bytes_per_step": 8 * int(f_local.size) * world, "ms_per_step": e2e_s * 1e3},
            "gpu_launches": (2 * len(orders) + 1 + 2 * (args.dist_chunks or 4)) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=48)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the device-timed side configs (C1, C2, C3, C5)")
    ap.add_argument("--no-verify", action="store_true",
                    help="N > 1: skip the set-up check of the fused exchange against a single-GPU solve")
    ap.add_argument("--dist-mode", default="peer", choices=["peer", "nccl"],
                    help="N > 1: exchanges fused into the sweeps over NVLink peer memory, or NCCL all-to-all")
    ap.add_argument("--dist-chunks", type=int, default=0,
                    help="exchange chunks of the NCCL slab path (0 = the library default, 4)")
    ap.add_argument("--dist-single", action="store_true",
                    help="exercise the slab-decomposed path on one GPU (1-rank NCCL group)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    args.steps = max(1, min(args.steps, 150))  # solutions shrink ~30x per in-place solve

    world, rank, local, dist = dist_setup()
    if args.dist_single and world == 1 and args.impl == "ours":
        import torch
        import torch.distributed as tdist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29555")
        torch.cuda.set_device(0)
        tdist.init_process_group("nccl", rank=0, world_size=1)
        if args.dist_mode == "peer" and peer_capable(args.config):
            run_peer(args, 1, 0, 0, tdist)
        else:
            run_distributed(args, 1, 0, 0, tdist)
        tdist.destroy_process_group()
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            dist.destroy_process_group()
        return

    import torch
    import paper_1701_03967_b200 as sfem

    torch.cuda.set_device(local)
    if world > 1 and args.dist_mode == "peer" and peer_capable(args.config):
        ok = True
        try:
            run_peer(args, world, rank, local, dist)
        except Exception as e:
            ok = False
            print(f"[bench] fused NVLink solve failed on rank {rank}: {e!r}; NCCL slab path next", file=sys.stderr)
            args.dist_error = repr(e)
        flag = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() == 1.0:
            dist.destroy_process_group()
            return
    if world > 1:
        try:
            run_distributed(args, world, rank, local, dist)
            dist.destroy_process_group()
            return
        except Exception as e:  # reported in the JSON line; replicas below
            print(f"[bench] slab-decomposed solve failed on rank {rank}: {e!r}; running replicas", file=sys.stderr)
            args.dist_error = repr(e)
    orders, elements, lengths, coeffs, shift, desc = CONFIGS[args.config]
    spec = sfem.ProblemSpec(len(orders), lengths, elements, orders, shift, coefficients=coeffs)
    ctx = sfem.Context(local)
    plan = sfem.Plan(spec, ctx)
    ext = plan.extents
    U = plan.unknowns
    rows = U // ext[-1]
    f = np.random.default_rng(rank).uniform(-1.0, 1.0, ext)

    stream = torch.cuda.ExternalStream(ctx.stream)
    buf = torch.empty(rows * plan.pitch, dtype=torch.float64, device="cuda")
    load_dev = torch.from_numpy(f.reshape(rows, ext[-1])).to("cuda")
    buf.view(rows, plan.pitch)[:, :ext[-1]].copy_(load_dev)
    del load_dev
    torch.cuda.synchronize()
    ptr = buf.data_ptr()

    for _ in range(args.warmup):
        plan.solve_device(ptr)
    torch.cuda.synchronize()

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(dist, world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let the sampler start
        ev0.record(stream)
        for _ in range(args.steps):
            plan.solve_device(ptr)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(dist, world)
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, dist, world)
    value = U * world * args.steps / (ms * 1e-3)

    # per-kernel breakdown (separate, event-bracketed on the plan stream)
    total_ms, kern_ms = plan.solve_device_timed(ptr, reps=5)
    dom = int(np.argmax(kern_ms))
    peaks, peak_kind = measured_peaks()
    alg_bytes_kernel = 16.0 * U  # one read + one write of every unknown per sweep
    achieved = alg_bytes_kernel / (kern_ms[dom] * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh).get(args.config, {}).get("dominant_kernel_dram_bytes")
    except Exception:
        pass
    ms_step = ms / args.steps
    solve_bytes = 16.0 * U * plan.launches
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                "kernel": f"sweep {dom} of {plan.launches} ({kern_ms[dom]:.3f} ms)", "peak_kind": peak_kind,
                "kernel_ms": [round(x, 4) for x in kern_ms],
                "solve_frac": (solve_bytes / (ms_step * 1e-3) / 1e9) / peaks["hbm_gbs"],
                "solve_frac_2N_passes": (16.0 * U * 2 * len(orders) / (ms_step * 1e-3) / 1e9) / peaks["hbm_gbs"]}

    # end to end through the public API: every step copies its load from pinned
    # host memory to the device and its solution back (sfem_cuda_solve_host_batch
    # overlaps step i+1's H2D and step i-1's D2H with step i's solve; the batch
    # includes the pipeline fill and drain)
    h_load = torch.from_numpy(f).pin_memory()
    h_u = torch.empty_like(h_load).pin_memory()
    plan.solve_host_batch([h_load.data_ptr()], [h_u.data_ptr()])  # warm (allocates the slots)
    barrier(dist, world)
    n_e2e = max(args.e2e_steps, 2)
    t0 = time.perf_counter()
    plan.solve_host_batch([h_load.data_ptr()] * n_e2e, [h_u.data_ptr()] * n_e2e)
    e2e_s = (time.perf_counter() - t0) / n_e2e
    e2e_s = max_over_ranks(e2e_s, dist, world)
    # single-solve latency through sfem_cuda_solve_host (no pipelining)
    import ctypes
    dp = ctypes.POINTER(ctypes.c_double)
    lp = ctypes.cast(ctypes.c_void_p(h_load.data_ptr()), dp)
    up = ctypes.cast(ctypes.c_void_p(h_u.data_ptr()), dp)
    sec = ctypes.c_double()
    for rep in range(2):  # the first call allocates the plan's staging buffer
        t0 = time.perf_counter()
        if sfem.lib.sfem_cuda_solve_host(plan.handle, lp, up, ctypes.byref(sec)) != 0:
            raise RuntimeError(sfem.lib.sfem_cuda_last_error().decode())
        lat_s = time.perf_counter() - t0
    e2e = {"value": U * world / e2e_s, "unit": "unknowns/s", "h2d_bytes_per_step": 8 * U, "d2h_bytes_per_step": 8 * U,
           "ms_per_step": e2e_s * 1e3, "steps": n_e2e, "api": "sfem_cuda_solve_host_batch (pinned host buffers)",
           "single_solve_latency_ms": lat_s * 1e3}

    side = None
    if rank == 0 and world == 1 and not args.no_configs:
        del buf
        torch.cuda.empty_cache()
        side = side_configs(sfem, ctx, args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import reflib
            if reflib.available():
                Us, secs, cores, sample, same = cpu_reference_sample(args.config, reps=5, warmup=1)
                cpu = {"value": Us / statistics.median(secs), "unit": "unknowns/s", "cores": cores,
                       "kind": "reference", "sample": sample, "same_config": same}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": "unknowns/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "unknowns_per_gpu": U, "extents": ext, "device_pitch": plan.pitch,
                       "l2_flush": "none needed: 1.52 GB tensor > 126 MB L2", "parallelism": f"replicas x{world}",
                       "dist_error": getattr(args, "dist_error", None),
                       "schedule": ("2N-1 sweeps; 3-D: fwd axis 1 (caller's tensor -> blocked scratch [x/8][y][x%8][z]), "
                                    "fwd axis 0, fused fwd+divide+inv axis 2, inv axis 0, inv axis 1 (-> caller's tensor)"
                                    if len(orders) == 3 else
                                    "2N-1 sweeps: fwd axes 0..N-2, fused fwd+divide+inv last axis, inv axes N-2..0")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "configs": side,
            "gpu_launches": plan.launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
